"""Run the bench workload and open the CUDA profiler range around exactly one decode step
(--what step) or one steady-state selector launch (--what select), for
`ncu --profile-from-start off`.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python scripts/profile_step.py
    ncu --profile-from-start off --set full -k regex:conv_forecast ... python scripts/profile_step.py --what select
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2502_04077_b200.decode import SHAPES, DecodeEngine  # noqa: E402
from paper_2502_04077_b200.selector import SelectorConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", choices=["step", "calib", "select", "dense"], default="step")
    ap.add_argument("--group", choices=["head", "kv"], default="kv")
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--model", default="llama-3.1-8b")
    ap.add_argument("--precision", default="fp16x3")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--gemm", choices=["auto", "tc"], default="auto")
    args = ap.parse_args()
    shape = SHAPES[args.model]
    G = shape.n_q_heads // shape.n_kv_heads
    eng = DecodeEngine(shape, args.batch, args.ctx, max_new=64, cfg=SelectorConfig(budget=1024),
                       group=1 if args.group == "head" else G, precision=args.precision, gemm=args.gemm)
    eng.init_history()
    eng.step(use_graph=False)
    eng.capture_all()
    if args.what == "dense":
        eng.set_mode("dense")
        eng.capture_all()
    for _ in range(6):
        eng.step()
    while args.what in ("step",) and eng.variant_for_next() != "plain":
        eng.step()
    while args.what == "calib" and eng.variant_for_next() != "calib":
        eng.step()
    torch.cuda.synchronize()
    if args.what == "select":
        st = eng.sel.states()
        comp = torch.rand(eng.sel.n_maps, eng.sel.w_max, device="cuda") ** 8
        eng.sel.push_compressed(comp, int(st["row_len"].max()))
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        eng.sel.step()
    else:
        torch.cuda.cudart().cudaProfilerStart()
        eng.step(use_graph=False)  # eager so every kernel is a separate, attributable launch
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one", args.what)


if __name__ == "__main__":
    main()

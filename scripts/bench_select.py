"""Micro-benchmark of the fused compress-push + forecast + top-k path (kernel 1+2+3).

Workload: n_layers x n_heads maps (default 32 x 32 = LLaMA-3.1-8B q-heads)
at context t (default 32K), H=64, b=16, B=1024.  Each timed step pushes one
compressed row per map (what the attention kernels emit), then runs
ap_sel_step (incremental r-map update + forecast + masked top-k) — the
per-token selection work of a whole model.  CUDA events on the launch stream.

    python scripts/bench_select.py [--t 32768] [--steps 48] [--precision fp16x3]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_04077_b200 import predictor  # noqa: E402
from paper_2502_04077_b200.batched import PUSH_PREFILL, BatchedSelector  # noqa: E402
from paper_2502_04077_b200.selector import SelectorConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, default=32768)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--precision", default="fp16x3")
    ap.add_argument("--graph", action="store_true")
    args = ap.parse_args()

    torch.manual_seed(0)
    cfg = SelectorConfig(budget=1024)
    n_maps = args.layers * args.heads
    t0 = args.t
    total_steps = args.warmup + args.steps
    w_max = -(-(t0 + total_steps + 1) // cfg.block_size)
    predictor.install_weights(predictor.init_weights(0))
    sel = BatchedSelector(cfg, n_maps, w_max, precision=args.precision)
    # synthetic compressed rows (block maxima of a softmax row are in (0, 1])
    comp = torch.rand(n_maps, w_max, device="cuda") ** 8
    for i in range(cfg.history - 1):
        sel.push_compressed(comp, t0 - (cfg.history - 1) + i, prefill=True)
    t = t0
    # first step = full recompute of every r-map row (prefill-side init)
    sel.push_compressed(comp, t)
    sel.step()
    torch.cuda.synchronize()

    def one(t):
        sel.push_compressed(comp, t)
        sel.step()

    for _ in range(args.warmup):
        t += 1
        one(t)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        t += 1
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        one(t)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e3)
    sel.check_status()
    times = np.array(times)
    H, W = cfg.history, -(-t // cfg.block_size)
    K = cfg.middle_blocks
    b_alg_layer = args.heads * (t * 4 + (H + 1) * W * 4 + 4 * K)
    us_layer = float(np.median(times)) / args.layers
    print(json.dumps({
        "what": "push+forecast+topk", "t": t, "maps": n_maps, "precision": args.precision,
        "us_per_step_median": float(np.median(times)), "us_per_step_min": float(times.min()),
        "us_per_step_max": float(times.max()), "us_per_layer": us_layer,
        "B_alg_per_layer": b_alg_layer, "GBps_alg": b_alg_layer / (us_layer * 1e-6) / 1e9,
        "ctas": BatchedSelector.__module__ and __import__("paper_2502_04077_b200._lib", fromlist=["x"]).fn(
            "ap_sel_grid_ctas")(predictor._lib.PREC[args.precision]),
    }))


if __name__ == "__main__":
    main()

"""ap_gemv vs cuBLAS (torch.matmul) on the LLaMA-3.1-8B decode GEMVs at batch 1: µs per call
(CUDA-graph replay of 8 calls over distinct weight copies so nothing is L2-resident), achieved
GB/s of weight bytes, and max |diff| against the fp32 reference.

    python scripts/bench_gemv.py [--ns 1] [--rows 1,2,4]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2502_04077_b200 import _lib  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336),
          "lm_head": (128256, 4096)}


def timeit(fn, copies, reps=30):
    for i in range(copies):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(copies):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2] * 1e3 / copies


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", type=int, default=1)
    ap.add_argument("--rows", default="1,2,4")
    ap.add_argument("--fused", action="store_true")
    args = ap.parse_args()
    gemv = _lib.fn("ap_gemv")
    out = {}
    for name, (N, K) in SHAPES.items():
        copies = max(2, min(8, int(2.5e9 // (N * K * 2))))
        Ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
        x = torch.randn(args.ns, K, device="cuda", dtype=torch.bfloat16)
        y = torch.empty(args.ns, N, device="cuda", dtype=torch.bfloat16)
        ref = (x.float() @ Ws[0].float().t())
        res = {"cublas_us": round(timeit(lambda i: torch.matmul(x, Ws[i].t(), out=y), copies), 2)}
        for rows in map(int, args.rows.split(",")):
            s = _lib.stream_handle()
            f = lambda i, rows=rows: gemv(Ws[i].data_ptr(), x.data_ptr(), y.data_ptr(), N, K, args.ns, rows, 0,  # noqa
                                          None, None, None, 0.0, None, None, _lib.stream_handle())
            us = timeit(f, copies)
            f(0)
            torch.cuda.synchronize()
            res[f"ours_r{rows}_us"] = round(us, 2)
            res[f"ours_r{rows}_err"] = float((y.float() - ref).abs().max())
        best = min(v for k, v in res.items() if k.startswith("ours") and k.endswith("_us"))
        res["ours_GBps"] = round(N * K * 2 / (best * 1e-6) / 1e9, 1)
        res["cublas_GBps"] = round(N * K * 2 / (res["cublas_us"] * 1e-6) / 1e9, 1)
        out[name] = res
        del Ws
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__" and "--fused" not in sys.argv:
    main()


def fused_main():
    """Fused projection variants vs the unfused sequence they replace (batch 1)."""
    gemv = _lib.fn("ap_gemv")
    rms, silu = _lib.fn("ap_rmsnorm"), _lib.fn("ap_silu_mul")
    K, F, V = 4096, 14336, 128256
    res = {}
    x = torch.randn(1, K, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(1, K, device="cuda", dtype=torch.bfloat16)
    r_out = torch.empty_like(r)
    ln = torch.ones(K, device="cuda", dtype=torch.bfloat16)
    yn = torch.empty_like(x)
    s = _lib.stream_handle
    for name, N, flags, out_n in (("qkv_rms", 6144, 1, 6144), ("gate_up_rms_silu", 2 * F, 1 | 2, F),
                                  ("lm_head_rms_argmax", V, 1 | 4, V)):
        copies = max(2, min(8, int(2.5e9 // (N * K * 2))))
        Ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
        y = torch.empty(1, out_n, device="cuda", dtype=torch.bfloat16)
        gu = torch.empty(1, N, device="cuda", dtype=torch.bfloat16)
        ws = torch.zeros(48, dtype=torch.uint8, device="cuda")
        tok = torch.zeros(1, dtype=torch.int64, device="cuda")

        def fused(i):
            gemv(Ws[i].data_ptr(), x.data_ptr(), y.data_ptr(), N, K, 1, 2, flags, r.data_ptr(), r_out.data_ptr(),
                 ln.data_ptr(), 1e-5, ws.data_ptr() if flags & 4 else None, tok.data_ptr() if flags & 4 else None, s())

        def unfused(i):
            rms(x.data_ptr(), r_out.data_ptr(), ln.data_ptr(), yn.data_ptr(), 1, K, 1e-5, s())
            if flags & 2:
                torch.matmul(yn, Ws[i].t(), out=gu)
                silu(gu.data_ptr(), y.data_ptr(), 1, F, s())
            else:
                torch.matmul(yn, Ws[i].t(), out=y)
                if flags & 4:
                    torch.argmax(y, dim=-1, out=tok)

        res[name] = {"fused_us": round(timeit(fused, copies), 2), "unfused_us": round(timeit(unfused, copies), 2)}
        del Ws
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__" and "--fused" in sys.argv:
    fused_main()

"""ap_gemm_tc vs cuBLAS (torch.matmul) on the LLaMA-3.1-8B decode projections at batch S (5..16):
µs per call from a CUDA-graph replay of calls over distinct weight copies (nothing L2-resident),
GB/s of weight bytes, and max |diff| between the two.

    python scripts/bench_gemm_tc.py [S ...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from bench_gemv import SHAPES, timeit  # noqa: E402
from paper_2502_04077_b200 import _lib  # noqa: E402

_lib.load()
for S in map(int, sys.argv[1:] or ["8"]):
    ws = torch.zeros(max(_lib.fn("ap_gemm_tc_workspace_bytes")(n, k, S) for n, k in SHAPES.values()),
                     dtype=torch.uint8, device="cuda")
    for name, (N, K) in SHAPES.items():
        copies = max(2, min(8, int(2.5e9 // (N * K * 2))))
        Ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
        x = torch.randn(S, K, device="cuda").bfloat16()
        y = torch.empty(S, N, device="cuda", dtype=torch.bfloat16)
        y2 = torch.empty_like(y)

        def tc(i):
            _lib.check(_lib.fn("ap_gemm_tc")(Ws[i].data_ptr(), x.data_ptr(), y.data_ptr(), N, K, S, ws.data_ptr(),
                                             ws.numel(), _lib.stream_handle()), "ap_gemm_tc")

        t_tc = timeit(tc, copies)
        t_cb = timeit(lambda i: torch.matmul(x, Ws[i].t(), out=y2), copies)
        tc(0)
        torch.matmul(x, Ws[0].t(), out=y2)
        err = (y.float() - y2.float()).abs().max().item()
        gb = N * K * 2 / 1e3
        print(f"{name:8s} N={N:6d} K={K:5d} S={S:2d}  tc {t_tc:7.1f} us ({gb / t_tc:6.0f} GB/s)  "
              f"cublas {t_cb:7.1f} us ({gb / t_cb:6.0f} GB/s)  maxdiff {err:.3g}", flush=True)
        del Ws

"""Per-CTA timeline of ap_gemm_tc (ATTNPRED_GEMM_TRACE=1): the last of 4 back-to-back launches over
distinct weight copies, events in ns relative to the earliest kernel entry.

    python scripts/gemm_tc_trace.py N K S
"""
import ctypes
import os
import sys
from pathlib import Path

os.environ["ATTNPRED_GEMM_TRACE"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_04077_b200 import _lib  # noqa: E402

lib = _lib.load()
N, K, S = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 8)))
Ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(4)]
x = torch.randn(S, K, device="cuda").bfloat16()
y = torch.empty(S, N, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(_lib.fn("ap_gemm_tc_workspace_bytes")(N, K, S), dtype=torch.uint8, device="cuda")
for rep in range(2):
    for W in Ws:
        _lib.check(_lib.fn("ap_gemm_tc")(W.data_ptr(), x.data_ptr(), y.data_ptr(), N, K, S, ws.data_ptr(),
                                         ws.numel(), _lib.stream_handle()), "ap_gemm_tc")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (160 * 12))()
lib.ap_gemm_tc_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(160, 12)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
rel = a - t0
names = ["entry", "setup", "pdl_wait", "first_full", "mma_done", "epi_first", "epi_end", "exit", "part_stored", "counted", "reduced", "y_stored"]
print(f"{len(a)} CTAs; events ns after first entry (min / median / max)")
for i, n in enumerate(names):
    v = rel[:, i]
    print(f"{n:>11s} {v.min():8d} {int(np.median(v)):8d} {v.max():8d}")
order = np.argsort(-rel[:, 7])[:6]
print("slowest CTAs:", " ".join(f"{n:>11s}" for n in names))
for c in order:
    print(f"{c:12d}  " + " ".join(f"{(v if a[c, i] > 0 else -1):11d}" for i, v in enumerate(rel[c])))

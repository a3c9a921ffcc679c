"""A few ap_gemm_tc and cuBLAS launches of one projection shape (for ncu)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2502_04077_b200 import _lib  # noqa: E402

_lib.load()
N, K, S = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 8)))
W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
x = torch.randn(S, K, device="cuda").bfloat16()
y = torch.empty(S, N, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(_lib.fn("ap_gemm_tc_workspace_bytes")(N, K, S), dtype=torch.uint8, device="cuda")
for _ in range(3):
    _lib.check(_lib.fn("ap_gemm_tc")(W.data_ptr(), x.data_ptr(), y.data_ptr(), N, K, S, ws.data_ptr(), ws.numel(),
                                     _lib.stream_handle()), "ap_gemm_tc")
    torch.matmul(x, W.t(), out=y)
torch.cuda.synchronize()

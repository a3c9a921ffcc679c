"""Per-phase clock64 trace of the calibration (K-only dense) kernel, CTAs of KV head 0."""
import os
# the phase traces are compiled in only with -DAP_ATT_TRACE:
#   SRC=attention scripts/build_wsm_variants.sh att_trace:AP_ATT_TRACE=1
os.environ.setdefault("ATTNPRED_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "paper_2502_04077_b200", "lib", "variants", "att_trace.so"))

import ctypes, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_04077_b200 import _lib
from paper_2502_04077_b200.attention import DecodeAttention
from paper_2502_04077_b200.batched import BatchedSelector
from paper_2502_04077_b200.selector import SelectorConfig
L = _lib.load()
S, Hq, Hkv, t, t_max = 1, 32, 8, 32768, 33792
k = torch.randn(S, Hkv, t_max, 128, device="cuda", dtype=torch.bfloat16)
q = torch.randn(S, Hq, 128, device="cuda", dtype=torch.bfloat16)
seq_len = torch.tensor([t], dtype=torch.int32, device="cuda")
sel = BatchedSelector(SelectorConfig(budget=1024), 8, t_max // 16)
att = DecodeAttention(S, Hq, Hkv, t_max)
for it in range(4):
    L.ap_attn_debug_trace(1 if it == 3 else 0, None)
    att.dense(q, k, k, seq_len, None, with_v=False, emit=True, selector=sel, map_base=0, maps_per_seq=8, group=4)
    torch.cuda.synchronize()
buf = (ctypes.c_longlong * 256)()
L.ap_attn_debug_trace(0, buf)
full = np.array(buf, dtype=np.int64).reshape(16, 16)
a = full[:, :10]
t0 = a[a > 0].min()
print("cta   entry   setup  tiles_issued  epi_done  lse_seen  emitted  end  published  -  -")
for r in range(16):
    if a[r, 0]: print(r, " ".join(f"{(x - a[r, 0]) if x else -1:9d}" for x in a[r]))

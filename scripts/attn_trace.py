"""Per-phase clock64 trace of the sparse cluster attention kernel (CTAs of map 0)."""
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
S, Hq, Hkv, t = int(os.environ.get("BATCH", "1")), 32, 8, 32768
t_max = 33792
k = torch.randn(S, Hkv, t_max, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn(S, Hkv, t_max, 128, device="cuda", dtype=torch.bfloat16)
q = torch.randn(S, Hq, 128, device="cuda", dtype=torch.bfloat16)
out = torch.empty(S, Hq, 128, device="cuda", dtype=torch.bfloat16)
seq_len = torch.full((S,), t, dtype=torch.int32, device="cuda")
cfg = SelectorConfig(budget=1024)
maps = 8 * S
sel = BatchedSelector(cfg, maps, t_max // 16)
st = sel.states().copy()
rng = np.random.default_rng(0)
for m in range(maps):
    blk = sorted(rng.choice(np.arange(4, 2040), cfg.middle_blocks, replace=False).tolist())
    st[m]["n_mid"] = len(blk); st[m]["mid_clip"] = t - 1
    sel.mid_blocks[m, :len(blk)] = torch.tensor(blk, dtype=torch.int32)
sel.state.copy_(torch.from_numpy(st.view(np.uint8).copy()))
att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_sparse=int(os.environ.get("SPLITS", "8")))
for it in range(4):
    L.ap_attn_debug_trace(1 if it == 3 else 0, None)
    att.sparse(q, k, v, seq_len, out, sel, emit=True, map_base=0, maps_per_seq=8, group=4)
    torch.cuda.synchronize()
buf = (ctypes.c_longlong * 256)()
L.ap_attn_debug_trace(0, buf)
a = np.array(buf, dtype=np.int64).reshape(16, 16)[:, :14]
names = ["entry", "pre_pdl", "post_pdl", "blocks_done", "merged", "sync1", "final", "emitted", "exit", "loads_issued", "mid_landed", "blk_ready", "state_used", "slot"]
t0 = a[a > 0].min()
print("rank " + " ".join(f"{n:>11s}" for n in names))
for r in range(16):
    if a[r, 0]: print(f"{r:4d} " + " ".join(f"{(x - t0) if x else -1:11d}" for x in a[r]))

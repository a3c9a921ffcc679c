"""Forecaster launch time (graph replay, L2 flushed) on 256 KV-group-like maps at 32K, guard off.
ATTNPRED_FORECAST_DEBUG bits disable roles (1 conv1 math, 2 MMAs, 4 epilogue math)."""
import ctypes, os, statistics, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
from test_gpu_parity_32k import _weights, _rows
from paper_2502_04077_b200 import predictor, _lib
from paper_2502_04077_b200.batched import PUSH_DENSE, PUSH_PREFILL, BatchedSelector
from paper_2502_04077_b200.selector import SelectorConfig
_lib.check(_lib.fn("ap_sel_set_tie_guard")(0, ctypes.c_float(0), ctypes.c_float(0)))
rng = np.random.default_rng(1)
n_maps, t0 = 256, 32760
w = _weights(1)
predictor.install_weights(predictor.PredictorWeights.from_flat(w.flat()))
sel = BatchedSelector(SelectorConfig(budget=1024), n_maps, w_max=2112, precision=os.environ.get("PREC", "fp16x3"))
base = torch.from_numpy(_rows(rng, n_maps, t0 + 8, 4)).cuda()
for i in range(63):
    sel.push_rows(base, t0 - 63 + i, mode=PUSH_PREFILL)
for i in range(3):
    sel.push_rows(base, t0 + i, mode=PUSH_DENSE); sel.step()
sel.push_rows(base, t0 + 3, mode=PUSH_DENSE)
torch.cuda.synchronize()
keep = [t.clone() for t in (sel.state, sel.rmap, sel.rsum, sel.mid_blocks, sel.mid_mask)]
def restore():
    for dst, src in zip((sel.state, sel.rmap, sel.rsum, sel.mid_blocks, sel.mid_mask), keep): dst.copy_(src)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s): sel.step()
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize(); restore()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g): sel.step()
ts = []
for _ in range(15):
    restore(); flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(f"{os.environ.get('ATTNPRED_FORECAST_DEBUG','0'):>3} {os.environ.get('PREC','fp16x3')}: {statistics.median(ts):.1f} us")

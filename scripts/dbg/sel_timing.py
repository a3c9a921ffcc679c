"""Selector launch timing variants on the engine's real data (32K, KV-group maps)."""
import ctypes, statistics, sys
sys.path.insert(0, ".")
import torch
from paper_2502_04077_b200 import _lib
from paper_2502_04077_b200.decode import SHAPES, DecodeEngine
from paper_2502_04077_b200.selector import SelectorConfig

eng = DecodeEngine(SHAPES["llama-3.1-8b"], 1, 32768, max_new=64, cfg=SelectorConfig(budget=1024), group=4)
eng.init_history()
eng.step(use_graph=False); eng.capture_all()
for _ in range(6): eng.step()
sel = eng.sel
eng._step_body(eng.variant_for_next(), selector=False)
torch.cuda.synchronize()
keep = [t.clone() for t in (sel.state, sel.rmap, sel.rsum, sel.mid_blocks, sel.mid_mask)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def restore():
    for dst, src in zip((sel.state, sel.rmap, sel.rsum, sel.mid_blocks, sel.mid_mask), keep): dst.copy_(src)
def timed(fn, reps=15, do_flush=True):
    ts = []
    for _ in range(reps):
        restore()
        if do_flush: flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return round(statistics.median(ts), 1)
print("eager, flush       ", timed(sel.step))
print("eager, no flush    ", timed(sel.step, do_flush=False))
g = torch.cuda.CUDAGraph()
restore()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s): sel.step()
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize(); restore()
with torch.cuda.graph(g): sel.step()
print("graph, flush       ", timed(g.replay))
print("graph, no flush    ", timed(g.replay, do_flush=False))
_lib.check(_lib.fn("ap_sel_set_tie_guard")(0, ctypes.c_float(2**-15), ctypes.c_float(2**-5)))
print("eager, guard off   ", timed(sel.step))
print("tie stats", sel.tie_stats())

"""Band top-k fast-path statistics on engine data (variant library built with -DAP_TOPK_STATS and a band
half-width -DAP_TOPK_BAND=...): per launch, the fraction of maps whose boundary fell in the band and the
fraction ranked directly, and the mean band size."""
import ctypes, sys
sys.path.insert(0, ".")
import torch
from paper_2502_04077_b200 import _lib
from paper_2502_04077_b200.decode import SHAPES, DecodeEngine
from paper_2502_04077_b200.selector import SelectorConfig
eng = DecodeEngine(SHAPES["llama-3.1-8b"], 1, 32768, max_new=64, cfg=SelectorConfig(budget=1024), group=4)
eng.init_history()
eng.step(use_graph=False)
eng.capture_all()
L = _lib.load()
buf = (ctypes.c_int * 4)()
for _ in range(4): eng.step()
torch.cuda.synchronize(); L.ap_debug_topk_stats(buf)
tot = [0, 0, 0, 0]
for _ in range(20):
    v = eng.step(); torch.cuda.synchronize(); L.ap_debug_topk_stats(buf)
    tot = [a + b for a, b in zip(tot, buf)]
print(f"maps {tot[0]}  boundary in band {tot[1] / max(1, tot[0]):.3f}  fast path {tot[2] / max(1, tot[0]):.3f}  mean band size {tot[3] / max(1, tot[0]):.1f}")

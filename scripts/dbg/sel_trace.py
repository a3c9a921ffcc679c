"""Phase stamps (clock64) of map 0's selection in the band top-k on the decode engine's data
(variant library built with -DAP_SEL_TRACE: SRC=topk scripts/build_wsm_variants.sh seltrace:AP_SEL_TRACE=1)."""
import ctypes, os, sys
sys.path.insert(0, ".")
os.environ.setdefault("ATTNPRED_LIB", "paper_2502_04077_b200/lib/variants/seltrace.so")
import torch
from paper_2502_04077_b200 import _lib
from paper_2502_04077_b200.decode import SHAPES, DecodeEngine
from paper_2502_04077_b200.selector import SelectorConfig
eng = DecodeEngine(SHAPES["llama-3.1-8b"], 1, 32768, max_new=64, cfg=SelectorConfig(budget=1024), group=4)
eng.init_history(); eng.step(use_graph=False); eng.capture_all()
L = _lib.load()
buf = (ctypes.c_longlong * 16)()
names = ["entry", "state+init", "keys+reductions", "search", "emit+mask", "detect", "end"]
for _ in range(6):
    eng.step(); torch.cuda.synchronize(); L.ap_debug_sel_trace(buf)
    t = list(buf)
    print(f"state {t[6] - t[0]} keys {t[7] - t[0]} ", "  ".join(f"{names[i]} {t[i] - t[0]}" for i in range(1, 6)),
          f"| band idx {t[8]} size {t[9]} (widest {t[10]}, above it {t[11]}, narrowest {t[13]}) k {t[12]}")

"""Phase clocks of sel_topk_reg_kernel's CTA 0 (variant library built with AP_TOPK_TRACE): run the
forecaster knob script (256 KV-group-like maps at 32K, guard off) then read the last launch's trace."""
import ctypes, os, runpy, sys
sys.path.insert(0, "."); sys.path.insert(0, "scripts/dbg")
runpy.run_path("scripts/dbg/forecast_knobs.py", run_name="__main__")
from paper_2502_04077_b200 import _lib
buf = (ctypes.c_longlong * 16)()
_lib.load().ap_debug_topk_trace(buf)
t = list(buf)
names = ["entry", "state", "keys+range+masked", "radix", "emit", "detect", "end"]
print("fast path", t[8], " ".join(f"{names[i]} {t[i] - t[0]}" for i in range(7)))
import numpy as np
cb = (ctypes.c_longlong * 4096)()
_lib.load().ap_debug_topk_cta(cb)
c = np.array(cb, dtype=np.int64).reshape(1024, 4)[:256]
fast = (c[:, 1] <= 128) & (c[:, 2] < c[:, 3]) & (c[:, 2] + c[:, 1] >= c[:, 3])
print("cycles per CTA: median", int(np.median(c[:, 0])), "p90", int(np.percentile(c[:, 0], 90)), "max", int(c[:, 0].max()))
print("fast-path CTAs", int(fast.sum()), "of", len(c), "; band sizes (median/max)", int(np.median(c[:, 1])), int(c[:, 1].max()),
      "; fast median cycles", int(np.median(c[fast, 0])) if fast.any() else None,
      "; slow median cycles", int(np.median(c[~fast, 0])) if (~fast).any() else None)

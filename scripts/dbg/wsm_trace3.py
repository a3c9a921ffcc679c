"""CTA 0 band timeline with extra ATTNPRED_FORECAST_DEBUG bits (argv[1]) OR 16."""
import ctypes, os, runpy, sys
os.environ["ATTNPRED_FORECAST_DEBUG"] = str(16 | int(sys.argv[1]))
sys.path.insert(0, "."); sys.path.insert(0, "scripts/dbg")
runpy.run_path("scripts/dbg/forecast_knobs.py", run_name="__main__")
import numpy as np
from paper_2502_04077_b200 import _lib
buf = (ctypes.c_longlong * 1024)()
_lib.load().ap_debug_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(64, 16)
t0 = a[0][a[0] > 0].min()
d = lambda b, i, j: a[b][j] - a[b][i]
bs = range(8, 24)
print("dbg", sys.argv[1], "per-band medians: period", int(np.median([a[b + 1][0] - a[b][0] for b in bs])),
      "conv", int(np.median([d(b, 2, 3) for b in bs])), "mma", int(np.median([d(b, 4, 5) for b in bs])),
      "epi", int(np.median([d(b, 6, 7) for b in bs])))
print("epi phases: first-row load", int(np.median([d(b, 6, 8) for b in bs])), "rows", int(np.median([d(b, 8, 9) for b in bs])),
      "clear", int(np.median([d(b, 9, 7) for b in bs])))

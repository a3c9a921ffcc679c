"""CTA 0 band timeline of the forecaster (ATTNPRED_FORECAST_DEBUG=16) on the forecast_knobs setup."""
import ctypes, os, runpy, sys
os.environ["ATTNPRED_FORECAST_DEBUG"] = "16"
sys.path.insert(0, "."); sys.path.insert(0, "scripts/dbg")
runpy.run_path("scripts/dbg/forecast_knobs.py", run_name="__main__")
import numpy as np
from paper_2502_04077_b200 import _lib
buf = (ctypes.c_longlong * 1024)()
_lib.load().ap_debug_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(64, 16)[:, :8]
t0 = a[0][a[0] > 0].min()
names = ["prod", "cv_x", "cv_a1", "cv_done", "mma0", "mma1", "epi0", "epi1"]
print("band " + " ".join(f"{n:>8s}" for n in names))
for b in range(32):
    print(f"{b:4d} " + " ".join(f"{(v - t0) if v else -1:8d}" for v in a[b]))

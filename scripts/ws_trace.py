"""Timeline of CTA 0's first bands in the warp-specialised forecaster (ATTNPRED_FORECAST_DEBUG=16)."""
import ctypes, os, sys, runpy
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ATTNPRED_FORECAST_DEBUG"] = os.environ.get("TRACE_DBG", "16")
from paper_2502_04077_b200 import _lib
sys.argv = ["bench_select.py", "--heads", "8", "--steps", "2", "--warmup", "1"]
runpy.run_path(os.path.join(os.path.dirname(__file__), "bench_select.py"), run_name="__main__")
buf = (ctypes.c_longlong * 1024)()
_lib.load().ap_debug_trace(buf)
a = np.array(buf, dtype=np.int64)[:512].reshape(64, 8)
t0 = a[0][a[0] > 0].min()
names = ["prod_issued", "conv_w0_begin", "conv_start", "conv_w0_done", "mma_start", "mma_issued", "epi_start", "epi_end"]
print("band " + " ".join(f"{n:>20s}" for n in names))
for b in range(40):
    print(f"{b:4d} " + " ".join(f"{(v - t0) if v else -1:20d}" for v in a[b]))

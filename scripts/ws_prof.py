import ctypes, os, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ATTNPRED_FORECAST_DEBUG"] = sys.argv[1] if len(sys.argv) > 1 else "8"
import torch
from paper_2502_04077_b200 import _lib
import runpy
sys.argv = ["bench_select.py", "--steps", "3", "--warmup", "1"]
runpy.run_path(os.path.join(os.path.dirname(__file__), "bench_select.py"), run_name="__main__")
buf = (ctypes.c_ulonglong * (16 * 160))()
_lib.load().ap_debug_prof(buf, 16 * 160)
a = np.array(buf, dtype=np.float64).reshape(160, 16)[:148]
names = ["prod_wait_xempty", "prod_plan", "epi_wait_accfull", "epi_work", "conv_wait_xfull", "conv_wait_a1empty", "conv_work", "prod_scan", "epi_pre", "epi_catch", "epi_math", "mma_wait_a1full", "mma_wait_accempty"]
print({n: round(float(a[:, i].mean()) / 1e3, 1) for i, n in enumerate(names)}, "k-cycles (mean over CTAs, last launch)")

"""Per-CTA timeline of the merged-band forecaster (ATTNPRED_FORECAST_DEBUG=32): entry skew, set-up, the
producer's last band, exit, bands per CTA — for the last launch of scripts/bench_select.py."""
import ctypes, os, sys, runpy
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ATTNPRED_FORECAST_DEBUG"] = str(32 | int(os.environ.get("ATTNPRED_FORECAST_DEBUG", "0")))
from paper_2502_04077_b200 import _lib
sys.argv = ["bench_select.py", "--heads", os.environ.get("HEADS", "8"), "--steps", "2", "--warmup", "1"]
runpy.run_path(os.path.join(os.path.dirname(__file__), "bench_select.py"), run_name="__main__")
buf = (ctypes.c_ulonglong * 2560)()
_lib.load().ap_debug_prof(buf, 2560)
a = np.array(buf, dtype=np.int64).reshape(320, 8)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
us = lambda x: (x - t0) / 1000.0
print(f"ctas {len(a)}  bands/cta min {a[:, 4].min()} max {a[:, 4].max()} mean {a[:, 4].mean():.1f}")
for name, col in [("entry", 0), ("setup_done", 1), ("prod_last_band", 2), ("exit", 3)]:
    v = us(a[:, col])
    print(f"{name:15s} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f} us")
v = (a[:, 3] - a[:, 2]) / 1000.0
print(f"drain (exit - last band issued) median {np.median(v):.2f} us")
v = (a[:, 1] - a[:, 0]) / 1000.0
print(f"setup (TMEM alloc, B tile, barriers) median {np.median(v):.2f} us")
if a.shape[0] and a[:, 5].max() > 0:  # fused selection: all roles done, group 0's selections done
    for name, col in [("roles_done", 5), ("group0_selected", 6)]:
        v = us(a[:, col])
        print(f"{name:15s} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f} us")

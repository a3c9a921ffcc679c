"""Profile the selector launches at 32K (64 maps, Dirichlet rows): guard on / off timing."""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
from test_gpu_parity_32k import _weights, _rows
from paper_2502_04077_b200 import predictor, _lib
from paper_2502_04077_b200.batched import PUSH_DENSE, PUSH_PREFILL, BatchedSelector
from paper_2502_04077_b200.selector import SelectorConfig

def setup(n_maps=256, t0=32760, group=4, seed=1):
    rng = np.random.default_rng(seed)
    cfg = SelectorConfig(budget=1024)
    w = _weights(seed)
    predictor.install_weights(predictor.PredictorWeights.from_flat(w.flat()))
    dev = BatchedSelector(cfg, n_maps, w_max=2112)
    for i in range(63):
        p = torch.from_numpy(_rows(rng, n_maps, t0 - 63 + i, group)).cuda()
        dev.push_rows(p, p.shape[1], mode=PUSH_DENSE if False else PUSH_PREFILL)
    rows = [torch.from_numpy(_rows(rng, n_maps, t0 + s, group)).cuda() for s in range(6)]
    return dev, rows

def timeit(dev, rows, guard):
    _lib.check(_lib.fn("ap_sel_set_tie_guard")(guard, ctypes.c_float(2**-15), ctypes.c_float(2**-5)))
    ts = []
    for r in rows:
        dev.push_rows(r, r.shape[1], mode=PUSH_DENSE)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); dev.step(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return ts

dev, rows = setup()
print("guard on ", [round(x, 1) for x in timeit(dev, rows, 1)], dev.tie_stats())
dev, rows = setup()
print("guard off", [round(x, 1) for x in timeit(dev, rows, 0)])

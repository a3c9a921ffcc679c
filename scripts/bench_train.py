"""Forecaster training throughput: device minibatch step (ap_train_backward + ap_adam_step) vs
the float64 oracle's per-sample backward on the host (the reference's algorithm).

    python scripts/bench_train.py [--batch 32] [--H 64] [--W 256] [--steps 20]

Prints one JSON line: samples/s on the device (CUDA events, after warm-up), per-kernel share
is left to the ncu launch list; CPU samples/s from a bounded sample of oracle backward calls.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--H", type=int, default=64)
    ap.add_argument("--W", type=int, default=256)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cpu-samples", type=int, default=8)
    a = ap.parse_args()
    import torch

    from oracle import hotpath as O
    from paper_2502_04077_b200 import _lib
    from paper_2502_04077_b200 import predictor as P

    rng = np.random.default_rng(0)
    n = a.batch * 4
    grids = [rng.dirichlet(np.full(a.W, 0.1), size=a.H) for _ in range(n)]
    targets = [rng.dirichlet(np.full(a.W, 0.1)) for _ in range(n)]
    b = P._GradBatcher(grids, targets)
    w = torch.from_numpy(O.init_weights(0).flat()).cuda()
    m, v = torch.zeros_like(w), torch.zeros_like(w)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")

    def step(k):
        ids = [(k * a.batch + j) % n for j in range(a.batch)]
        g = b.grad_sum(w, ids, loss)
        _lib.check(_lib.fn("ap_adam_step")(_lib.ptr(w), _lib.ptr(m), _lib.ptr(v), _lib.ptr(g), 4833,
                                           float(a.batch), 1e-3, 0.9, 0.999, 1e-8, k + 1, _lib.stream_handle()), "adam")

    for k in range(3):
        step(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(a.steps):
        step(3 + k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    t0 = time.perf_counter()
    wo = O.init_weights(0)
    for i in range(a.cpu_samples):
        O.backward(wo, grids[i], targets[i])
    cpu_s = (time.perf_counter() - t0) / a.cpu_samples
    print(json.dumps({
        "what": "forecaster training step (backward + Adam)", "batch": a.batch, "H": a.H, "W": a.W,
        "ms_per_step": round(ms, 4), "samples_per_s": round(a.batch / ms * 1e3, 1),
        "cpu_oracle_samples_per_s": round(1.0 / cpu_s, 2), "cpu_cores": len(os.sched_getaffinity(0)),
        "cpu_sample": f"{a.cpu_samples} float64 oracle backward calls (tap-by-tap numpy, OpenBLAS default threads)",
        "flops_per_sample_fwd_bwd": 3 * 9504 * a.H * a.W,
    }))


if __name__ == "__main__":
    main()

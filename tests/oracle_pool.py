"""Parallel CPU oracle for the large-shape parity tests (test infrastructure only).

Each map's ``oracle.hotpath.step`` (the float64 restatement of selector.py:91-154, pinned to the
reference's golden vectors) runs unchanged in a worker process; the caller keeps the states and
ships them with each step.  At 32K one oracle forward takes ~0.1-0.2 s, so 64 maps x 12 steps need
the host's cores to finish in seconds.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from oracle import hotpath as O


def _step(args):
    st, cfg, w, row, sel = args
    row = np.asarray(row, np.float64)
    obs = row if sel is None else O.observed_from_selection(row, sel)
    st, sel = O.step(st, cfg, w, obs, full_row=row)
    return st, sel


def _forward(args):
    w, grid = args
    return O.forward(w, grid)


class OraclePool:
    """step_all(states, sels, rows) -> (states, sels): one oracle decode step for every map."""

    def __init__(self, procs: int | None = None):
        n = procs or max(1, min(32, len(os.sched_getaffinity(0))))
        self.pool = mp.get_context("spawn").Pool(n)

    def step_all(self, states, cfg, w, rows, sels):
        out = self.pool.map(_step, [(st, cfg, w, r, s) for st, r, s in zip(states, rows, sels)], chunksize=1)
        return [o[0] for o in out], [o[1] for o in out]

    def forward_all(self, w, grids):
        return self.pool.map(_forward, [(w, g) for g in grids], chunksize=1)

    def close(self):
        self.pool.terminate()
        self.pool.join()

"""GPU parity at the headline shape (BASELINE configs[1]: 32K context, B=1024, b=16, H=64, M=5).

The device selector (push -> incremental tcgen05 forecaster -> top-k + exact-boundary guard,
through the C-ABI) is driven exactly like the reference's evaluation loop (evaluation.py:90-115:
dense row on calibration steps, observed row = dense values at the previous selection otherwise)
and compared with the float64 oracle (oracle/hotpath.py, pinned to the reference's golden vectors)
at EVERY step of EVERY map:

* forecasts within the fp32-class tolerance (tests/parity.py),
* middle block ids IDENTICAL to the oracle's — no near-tie exemptions (the guard re-scores
  ambiguous boundaries in fp64, csrc/tieguard.cuh),
* the guard's premise: the forecaster's worst error stays below half the guard band.

64 maps x 12 steps starting at t = 32760: three calibration steps (counter 0, 5, 10) and one
width growth (W 2048 -> 2049 at t = 32769), for per-q-head rows and for KV-group rows (the
element-wise max of 4 q-head rows, which is what the engine's group maps store).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import hotpath as O
from parity import scores_close

pytestmark = pytest.mark.gpu

REL, FLOOR = 2.0 ** -15, 2.0 ** -5  # the library's default guard band (csrc/predictor.cu tie_init)


@pytest.fixture(scope="module")
def pool():
    from oracle_pool import OraclePool
    p = OraclePool()
    yield p
    p.close()


def _weights(seed):
    rng = np.random.default_rng(100 + seed)
    w = O.init_weights(seed)
    w.b1 = rng.standard_normal(16) * 0.1
    w.b2 = rng.standard_normal(32) * 0.1
    w.b3 = np.array(0.05)
    return O.Weights.from_flat(w.flat().astype(np.float32).astype(np.float64))  # APW1 round trip


def _rows(rng, n_maps, t, group):
    if group == 1:
        return rng.dirichlet(np.full(t, 0.05), size=n_maps).astype(np.float32)
    r = rng.dirichlet(np.full(t, 0.05), size=n_maps * group).astype(np.float32)
    return r.reshape(n_maps, group, t).max(axis=1)


def run_parity(pool, n_maps, t0, steps, group, seed, precision="fp16x3", w_max=None, fused=False):
    """Drive device and oracle side by side; returns (mismatches, worst err/band, tie stats, worst score err)."""
    import torch
    from paper_2502_04077_b200 import predictor
    from paper_2502_04077_b200.batched import PUSH_DENSE, PUSH_PREFILL, BatchedSelector
    from paper_2502_04077_b200.selector import SelectorConfig

    rng = np.random.default_rng(seed)
    cfg = SelectorConfig(budget=1024)
    ocfg = O.Config(budget=1024)
    w = _weights(seed)
    predictor.install_weights(predictor.PredictorWeights.from_flat(w.flat()))
    H = cfg.history
    w_max = w_max or -(-(t0 + steps) // 16)
    dev = BatchedSelector(cfg, n_maps, w_max=w_max, precision=precision, fused=fused)
    prefill = []
    for i in range(H - 1):
        p = _rows(rng, n_maps, t0 - (H - 1) + i, group)
        dev.push_rows(torch.from_numpy(p).cuda(), p.shape[1], mode=PUSH_PREFILL)
        prefill.append([O.max_pool(p[m], 16) for m in range(n_maps)])
    states = [O.init_state(ocfg) for _ in range(n_maps)]
    for m in range(n_maps):  # == O.init_state(ocfg, raw prefill rows): keeps the newest H-1 compressed rows
        states[m].history = [prefill[i][m] for i in range(H - 1)]
    sels = [None] * n_maps
    mismatches, worst_band, worst_score = 0, 0.0, 0.0
    for s in range(steps):
        rows = _rows(rng, n_maps, t0 + s, group)
        dev.push_rows(torch.from_numpy(rows).cuda(), rows.shape[1], mode=PUSH_DENSE)
        dev.step()
        dev.check_status()
        states, sels = pool.step_all(states, ocfg, w, list(rows), sels)
        scores = dev.scores.cpu().numpy()
        mid = dev.mid_blocks.cpu().numpy()
        st = dev.states()
        for m in range(n_maps):
            want = states[m].last_scores
            W = want.size
            ok, err = scores_close(scores[m, :W], want, precision)
            worst_score = max(worst_score, err)
            assert ok, f"step {s} map {m}: forecast err/bound {err:.3g}"
            got = mid[m, : int(st[m]["n_mid"])].tolist()
            if got != states[m].last_blocks:
                mismatches += 1
            # guard premise: the device error is below half the band around the device's k-th score
            masked = O.masked_scores(ocfg, scores[m, :W].astype(np.float64), t0 + s)
            fin = np.sort(masked[np.isfinite(masked)])[::-1]
            k = min(ocfg.middle_blocks, fin.size)
            if k:
                tau = fin[k - 1]
                band = REL * max(abs(tau), FLOOR * np.abs(fin).max())
                fin_mask = np.isfinite(masked)
                e = np.abs(scores[m, :W].astype(np.float64) - want)[fin_mask].max()
                worst_band = max(worst_band, e / band)
    if fused:  # every map's chunk counter returned to zero for the next launch
        assert int(dev.fused_done.abs().sum().item()) == 0
    return mismatches, worst_band, dev.tie_stats(), worst_score


@pytest.mark.parametrize("group", [1, 4], ids=["per_head", "kv_group"])
def test_selection_parity_32k(pkg_loaded, pool, group):
    n_maps, t0, steps = 64, 32760, 12
    mism, worst_band, tie, worst_score = run_parity(pool, n_maps, t0, steps, group, seed=group)
    print(f"32K group={group}: {n_maps} maps x {steps} steps, mismatches={mism}, near-tie exemptions=0, "
          f"worst forecast err/bound={worst_score:.3g}, worst err/guard-band={worst_band:.3g}, guard={tie}")
    assert mism == 0, f"{mism} map-steps chose different middle blocks than the float64 oracle"
    assert worst_band <= 0.5, f"forecast error reaches {worst_band:.3g} of the guard band (premise: <= 0.5)"
    assert tie["overflow"] == 0


def test_selection_parity_32k_fused(pkg_loaded, pool):
    """The single-launch form (forecast + top-k + guard in the forecaster kernel, ap_selector.fused_done)
    selects exactly what the oracle does, and leaves every per-map chunk counter at zero."""
    mism, worst_band, tie, worst_score = run_parity(pool, 64, 32760, 12, 4, seed=4, fused=True)
    print(f"32K fused: mismatches={mism}, worst forecast err/bound={worst_score:.3g}, guard={tie}")
    assert mism == 0
    assert tie["overflow"] == 0


def test_selection_parity_wide_guard_band_fused(pkg_loaded, pool):
    """Wide guard band through the fused launch: the in-kernel fp64 re-scoring (units taken by every
    CTA from the shared list) must re-emit the oracle's ids."""
    from paper_2502_04077_b200 import _lib
    _lib.check(_lib.fn("ap_sel_set_tie_guard")(1, ctypes.c_float(1e-3), ctypes.c_float(FLOOR)))
    try:
        mism, _, tie, _ = run_parity(pool, 32, 4070, 8, 1, seed=9, fused=True)
    finally:
        _lib.check(_lib.fn("ap_sel_set_tie_guard")(1, ctypes.c_float(REL), ctypes.c_float(FLOOR)))
    print(f"wide band fused: mismatches={mism}, guard={tie}")
    assert tie["refined_maps"] > 0
    assert mism == 0


def test_selection_parity_wide_guard_band(pkg_loaded, pool):
    """Force a wide guard band so that most boundaries go through the fp64 re-scoring path: the
    ids must still equal the oracle's (exercises candidate collection, re-scoring and re-emission)."""
    from paper_2502_04077_b200 import _lib
    _lib.check(_lib.fn("ap_sel_set_tie_guard")(1, ctypes.c_float(1e-3), ctypes.c_float(FLOOR)))
    try:
        mism, _, tie, _ = run_parity(pool, 32, 4070, 8, 1, seed=9)
    finally:
        _lib.check(_lib.fn("ap_sel_set_tie_guard")(1, ctypes.c_float(REL), ctypes.c_float(FLOOR)))
    print(f"wide band: mismatches={mism}, guard={tie}")
    assert tie["refined_maps"] > 0
    assert mism == 0


@pytest.fixture(scope="module")
def pkg_loaded():
    from paper_2502_04077_b200 import _lib
    _lib.load()

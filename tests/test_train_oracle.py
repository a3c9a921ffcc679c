"""Pin the oracle's training restatement (backward, Adam, train) against golden vectors from the
real reference (tests/golden/gen_golden_train.py → train.npz; predictor.py:219-251,327-409).
CPU-only."""

from __future__ import annotations

import numpy as np

from conftest import load_golden, unragged
from oracle import hotpath as O


def _cases(z, prefix):
    grids = unragged(z[f"{prefix}_grid"], z[f"{prefix}_grid_off"])
    targets = unragged(z[f"{prefix}_target"], z[f"{prefix}_target_off"])
    return [g.reshape(*s) for g, s in zip(grids, z[f"{prefix}_shapes"])], targets


def test_backward_golden():
    z = load_golden("train")
    grids, targets = _cases(z, "bw")
    for i, (g, t) in enumerate(zip(grids, targets)):
        loss, gr = O.backward(O.Weights.from_flat(z["bw_weights"][i]), g, t)
        ref = z["bw_grads"][i]
        assert abs(loss - z["bw_loss"][i]) <= 1e-12 * max(1.0, abs(z["bw_loss"][i]))
        assert np.max(np.abs(gr.flat() - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_backward_matches_finite_differences():
    # the reference's own acceptance check (test_acceptance.py:163-214) restated on a small case
    rng = np.random.default_rng(3)
    w = O.init_weights(1)
    w.b1 = rng.standard_normal(16) * 0.05
    g = rng.dirichlet(np.full(7, 0.3), size=5)
    t = rng.dirichlet(np.full(7, 0.3))
    _, gr = O.backward(w, g, t)
    flat = w.flat()
    for j in rng.choice(flat.size, 25, replace=False):
        e = np.zeros_like(flat)
        e[j] = 1e-6
        lp, _ = O.backward(O.Weights.from_flat(flat + e), g, t)
        lm, _ = O.backward(O.Weights.from_flat(flat - e), g, t)
        fd = (lp - lm) / 2e-6
        assert abs(fd - gr.flat()[j]) <= 1e-6 + 1e-4 * abs(fd)


def test_train_golden():
    z = load_golden("train")
    grids, targets = _cases(z, "tr")
    epochs, seed, bs = (int(x) for x in z["tr_params"])
    best, metrics = O.train(grids, targets, epochs=epochs, lr=1e-3, rng_seed=seed, batch_size=bs)
    assert np.max(np.abs(best.flat() - z["tr_best"])) <= 1e-12
    np.testing.assert_allclose([m[0] for m in metrics], z["tr_mse"], rtol=1e-12)
    np.testing.assert_allclose([m[1] for m in metrics], z["tr_acc"], rtol=1e-12)


def _golden_dataset(z, k):
    grids, targets = _cases(z, f"ds{k}")
    hs, bs, seed, max_step = (int(x) for x in z[f"ds{k}_params"])
    return grids, targets, hs, bs, float(z[f"ds{k}_ratio"]), seed, None if max_step < 0 else max_step


def test_build_dataset_golden():
    from paper_2502_04077_b200.trace import read_trace_file  # host C++ reader, no GPU
    from conftest import GOLDEN

    z = load_golden("train")
    tr = read_trace_file(GOLDEN / "trace_tiny.att1")
    for k in range(3):
        grids, targets, hs, bs, ratio, seed, max_step = _golden_dataset(z, k)
        got = O.build_dataset(tr, hs, bs, ratio, rng_seed=seed, max_step=max_step)
        assert len(got) == len(grids)
        for (g, t), rg, rt in zip(got, grids, targets):
            assert np.array_equal(g, rg) and np.array_equal(t, rt)

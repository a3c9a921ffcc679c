"""Device forecaster training (ap_train_backward / ap_adam_step, csrc/train.cu) against the
reference's golden training vectors and the float64 oracle (predictor.py:219-251,327-409).

The device computes in fp64 like the reference (only the summation order differs), so the bounds
are float64-rounding tight: gradients |x - y| <= 1e-9 * max(|y|, 1e-2 * max|y|), loss rtol 1e-10,
training runs bit-identical to each other and within 1e-9 of the reference's weights."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, unragged
from oracle import hotpath as O

pytestmark = pytest.mark.gpu


def _close(x, y, rtol=1e-9):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    floor = 1e-2 * np.max(np.abs(y)) if y.size else 0.0
    return np.all(np.abs(x - y) <= rtol * np.maximum(np.abs(y), floor))


def _cases(z, prefix):
    grids = unragged(z[f"{prefix}_grid"], z[f"{prefix}_grid_off"])
    targets = unragged(z[f"{prefix}_target"], z[f"{prefix}_target_off"])
    return [g.reshape(*s) for g, s in zip(grids, z[f"{prefix}_shapes"])], targets


def test_backward_golden():
    from paper_2502_04077_b200 import predictor as P

    z = load_golden("train")
    grids, targets = _cases(z, "bw")
    for i, (g, t) in enumerate(zip(grids, targets)):
        w = P.PredictorWeights.from_flat(z["bw_weights"][i])
        loss, gr = P.backward(w, P.AttentionHistory(g), t)
        assert abs(loss - z["bw_loss"][i]) <= 1e-10 * z["bw_loss"][i], (i, loss, z["bw_loss"][i])
        assert _close(gr.flat(), z["bw_grads"][i]), (i, np.max(np.abs(gr.flat() - z["bw_grads"][i])))


def test_backward_batched_full_shape():
    """A 32-sample minibatch at the deployment window (H=64, W=256): the device gradient SUM
    equals the sum of the oracle's per-sample gradients."""
    import torch

    from paper_2502_04077_b200 import predictor as P

    rng = np.random.default_rng(11)
    w = O.init_weights(5)
    w.b1 = rng.standard_normal(16) * 0.05
    w.b2 = rng.standard_normal(32) * 0.05
    grids = [rng.dirichlet(np.full(256, 0.1), size=64) for _ in range(32)]
    targets = [rng.dirichlet(np.full(256, 0.1)) for _ in range(32)]
    b = P._GradBatcher(grids, targets)
    wd = torch.from_numpy(w.flat()).cuda()
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    g = b.grad_sum(wd, list(range(32)), loss).cpu().numpy()
    ref_g, ref_l = np.zeros(O.PARAM_COUNT), 0.0
    for i in (0, 7, 31):  # oracle on three samples, device on those three alone
        l_i, g_i = O.backward(w, grids[i], targets[i])
        ref_g += g_i.flat()
        ref_l += l_i
    loss3 = torch.zeros(1, dtype=torch.float64, device="cuda")
    g3 = b.grad_sum(wd, [0, 7, 31], loss3).cpu().numpy()
    assert _close(g3, ref_g) and abs(loss3.item() - ref_l) <= 1e-10 * ref_l
    assert np.all(np.isfinite(g)) and loss.item() > 0


def test_adam_matches_reference_arithmetic():
    import torch

    from paper_2502_04077_b200 import _lib

    rng = np.random.default_rng(2)
    wf, m, v = rng.standard_normal(4833), rng.standard_normal(4833) * 1e-3, rng.random(4833) * 1e-5
    gsum = rng.standard_normal(4833)
    dev = [torch.from_numpy(a.copy()).cuda() for a in (wf, m, v, gsum)]
    for step in (1, 2, 3):
        O.adam_update(wf, m, v, gsum, 6, step)
        _lib.check(_lib.fn("ap_adam_step")(*(_lib.ptr(t) for t in dev), 4833, 6.0, 1e-3, 0.9, 0.999, 1e-8, step,
                                           _lib.stream_handle()), "adam")
    for host, d in zip((wf, m, v), dev):
        assert np.max(np.abs(d.cpu().numpy() - host)) <= 1e-15 * max(1.0, np.max(np.abs(host)))


def test_train_golden():
    from paper_2502_04077_b200 import predictor as P

    z = load_golden("train")
    grids, targets = _cases(z, "tr")
    epochs, seed, bs = (int(x) for x in z["tr_params"])
    samples = [P.TrainSample(input=P.AttentionHistory(g), target=t) for g, t in zip(grids, targets)]
    best, metrics = P.train(samples, epochs=epochs, learning_rate=1e-3, rng_seed=seed, batch_size=bs)
    np.testing.assert_allclose([m.train_mse for m in metrics], z["tr_mse"], rtol=1e-10)
    np.testing.assert_allclose([m.holdout_accuracy for m in metrics], z["tr_acc"], atol=1e-6)
    assert np.max(np.abs(best.flat() - z["tr_best"])) <= 1e-9
    best2, metrics2 = P.train(samples, epochs=epochs, learning_rate=1e-3, rng_seed=seed, batch_size=bs)
    assert np.array_equal(best.flat(), best2.flat())  # deterministic reductions
    assert [m.train_mse for m in metrics] == [m.train_mse for m in metrics2]


def test_train_errors():
    from paper_2502_04077_b200 import predictor as P
    from paper_2502_04077_b200.errors import ParameterError, TrainingError

    with pytest.raises(ParameterError):
        P.train([])
    g = np.random.default_rng(0).random((4, 6))
    s = [P.TrainSample(input=P.AttentionHistory(g), target=np.full(6, np.nan))] * 3  # non-finite loss
    with pytest.raises(TrainingError):
        P.train(s, epochs=1)


def test_build_dataset_golden_exact():
    """Device build_dataset (ap_max_pool batched per head) = the reference's samples, bit for bit."""
    from conftest import GOLDEN

    from paper_2502_04077_b200 import predictor as P
    from paper_2502_04077_b200.trace import read_trace_file

    z = load_golden("train")
    tr = read_trace_file(GOLDEN / "trace_tiny.att1")
    for k in range(3):
        grids, targets = _cases(z, f"ds{k}")
        hs, bs, seed, max_step = (int(x) for x in z[f"ds{k}_params"])
        got = P.build_dataset(tr, hs, bs, float(z[f"ds{k}_ratio"]), rng_seed=seed,
                              max_step=None if max_step < 0 else max_step)
        assert len(got) == len(grids)
        for s, rg, rt in zip(got, grids, targets):
            assert np.array_equal(s.input.grid, rg) and np.array_equal(s.target, rt)


def test_build_then_train_end_to_end():
    """The reference's training pipeline (build_dataset -> train) on the device, against the oracle."""
    from conftest import GOLDEN

    from paper_2502_04077_b200 import predictor as P
    from paper_2502_04077_b200.trace import read_trace_file

    tr = read_trace_file(GOLDEN / "trace_tiny.att1")
    ds = P.build_dataset(tr, 8, 16, 1.0, rng_seed=0)
    best, metrics = P.train(ds, epochs=2, rng_seed=1, batch_size=16)
    ob, om = O.train([s.input.grid for s in ds], [s.target for s in ds], epochs=2, lr=1e-3, rng_seed=1, batch_size=16)
    np.testing.assert_allclose([m.train_mse for m in metrics], [m[0] for m in om], rtol=1e-10)
    assert np.max(np.abs(best.flat() - ob.flat())) <= 1e-9

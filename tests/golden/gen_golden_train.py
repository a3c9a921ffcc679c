"""Golden vectors for forecaster training, produced by running the REAL reference.

Run in the build container only (imports /root/reference, absent on the GPU box):

    python tests/golden/gen_golden_train.py

Writes ``tests/golden/train.npz``: inputs and outputs of attncast.predictor.backward
(predictor.py:219-251) on several history shapes with biased weights, and one short
attncast.predictor.train run (predictor.py:327-409: seeded holdout split, per-epoch
permutations, per-sample gradient sums, Adam) on a mixed-width sample set — its best
weights and per-epoch metrics; and attncast.predictor.build_dataset (predictor.py:254-300) on
the committed trace_tiny.att1 for three (history, block, ratio, seed, max_step) settings.  Ragged arrays are (flat, offsets) pairs.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("ATTNCAST_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from attncast import predictor  # noqa: E402

OUT = Path(__file__).resolve().parent

BACKWARD_SHAPES = [(4, 5), (8, 12), (16, 40), (64, 33), (3, 130)]


def sample_grid(rng, H, W):
    # compressed softmax rows: sparse, non-negative, top rows zero like stack_history's padding
    g = rng.dirichlet(np.full(W, 0.2), size=H)
    g[: rng.integers(0, max(1, H // 4))] = 0.0
    return g


def biased_weights(seed):
    w = predictor.init_weights(seed)
    rng = np.random.default_rng(100 + seed)
    w.b1 = rng.standard_normal(16) * 0.05
    w.b2 = rng.standard_normal(32) * 0.05
    w.b3 = np.array(rng.standard_normal() * 0.01)
    return w


def ragged(arrs):
    arrs = [np.asarray(a, np.float64).ravel() for a in arrs]
    return np.concatenate(arrs), np.cumsum([0] + [a.size for a in arrs]).astype(np.int64)


def main():
    rng = np.random.default_rng(2502)
    out = {}
    grids, targets, flats, losses, grads = [], [], [], [], []
    for i, (H, W) in enumerate(BACKWARD_SHAPES):
        w = biased_weights(i)
        g = sample_grid(rng, H, W)
        t = rng.dirichlet(np.full(W, 0.2))
        loss, gr = predictor.backward(w, predictor.AttentionHistory(g), t)
        grids.append(g), targets.append(t), flats.append(w.flat()), losses.append(loss), grads.append(gr.flat())
    out["bw_shapes"] = np.array(BACKWARD_SHAPES, np.int64)
    out["bw_grid"], out["bw_grid_off"] = ragged(grids)
    out["bw_target"], out["bw_target_off"] = ragged(targets)
    out["bw_weights"] = np.stack(flats)
    out["bw_loss"] = np.array(losses)
    out["bw_grads"] = np.stack(grads)

    # one short training run on a mixed-width set (two widths, 20 samples -> 2 held out)
    H = 8
    samples = []
    shapes = []
    for j in range(20):
        W = 24 if j % 3 else 17
        g = sample_grid(rng, H, W)
        t = rng.dirichlet(np.full(W, 0.2))
        samples.append(predictor.TrainSample(input=predictor.AttentionHistory(g), target=t))
        shapes.append((H, W))
    best, metrics = predictor.train(samples, epochs=3, learning_rate=1e-3, rng_seed=7, batch_size=4)
    out["tr_shapes"] = np.array(shapes, np.int64)
    out["tr_grid"], out["tr_grid_off"] = ragged([s.input.grid for s in samples])
    out["tr_target"], out["tr_target_off"] = ragged([s.target for s in samples])
    out["tr_params"] = np.array([3, 7, 4], np.int64)  # epochs, rng_seed, batch_size (lr 1e-3, holdout 0.1)
    out["tr_best"] = best.flat()
    out["tr_mse"] = np.array([m.train_mse for m in metrics])
    out["tr_acc"] = np.array([m.holdout_accuracy for m in metrics])
    # predictor.build_dataset (predictor.py:254-300) on the committed golden trace
    from attncast.trace import read_trace_file

    tr = read_trace_file(OUT / "trace_tiny.att1")
    ds_cases = [(8, 16, 1.0, 0, None), (4, 8, 0.5, 3, None), (16, 4, 0.7, 1, 5)]
    for k, (hs, bs_, ratio, seed, max_step) in enumerate(ds_cases):
        ds = predictor.build_dataset(tr, hs, bs_, ratio, rng_seed=seed, max_step=max_step)
        out[f"ds{k}_params"] = np.array([hs, bs_, seed, -1 if max_step is None else max_step], np.int64)
        out[f"ds{k}_ratio"] = np.array(ratio)
        out[f"ds{k}_shapes"] = np.array([s.input.grid.shape for s in ds], np.int64)
        out[f"ds{k}_grid"], out[f"ds{k}_grid_off"] = ragged([s.input.grid for s in ds])
        out[f"ds{k}_target"], out[f"ds{k}_target_off"] = ragged([s.target for s in ds])
    np.savez_compressed(OUT / "train.npz", **out)
    print("wrote", OUT / "train.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()

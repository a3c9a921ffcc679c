"""Generate golden vectors by running the REAL reference package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/gen_golden.py

Outputs ``tests/golden/*.npz`` (committed).  Every array is produced by the
reference's own functions: attncast.compress.max_pool / expand_indices
(compress.py:28-57), attncast.selector.topk (selector.py:73-81),
attncast.predictor.forward / init_weights / save_weights
(predictor.py:101-116,211-216,424-431), and the predictor branch of
attncast.evaluation._iter_selections (evaluation.py:90-115) driven through
attncast.selector.step (selector.py:91-154) over traces from
attncast.synth.gen_trace.  Ragged lists are stored as (flat, offsets) pairs so
the fixtures load without pickle.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("ATTNCAST_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from attncast import compress, predictor, selector  # noqa: E402
from attncast.synth import SynthConfig, gen_trace  # noqa: E402

OUT = Path(__file__).resolve().parent


def ragged(arrs, dtype):
    arrs = [np.asarray(a, dtype=dtype).ravel() for a in arrs]
    off = np.cumsum([0] + [a.size for a in arrs]).astype(np.int64)
    flat = np.concatenate(arrs) if arrs else np.zeros(0, dtype)
    return flat, off


def gen_maxpool(rng):
    rows, bs, outs = [], [], []
    # the reference KATs (tests/test_compress.py:22-30) first
    for row, b in (([0.1, 0.3, 0.2, 0.05], 2), ([0.5, 0.1, 0.2, 0.4], 3), ([0.4, 0.1, 0.5], 1)):
        rows.append(np.asarray(row, np.float64)); bs.append(b)
    for _ in range(300):
        t = int(rng.integers(1, 2000))
        b = int(rng.choice([1, 2, 3, 7, 16, 17, 32, 64, 100]))
        kind = rng.integers(0, 4)
        if kind == 0:
            row = rng.random(t)
        elif kind == 1:
            row = rng.dirichlet(np.full(t, 0.05))
        elif kind == 2:
            row = rng.standard_normal(t)  # negative values: the zero pad can win the tail
        else:
            row = np.round(rng.random(t) * 4) / 4  # many ties
        rows.append(row.astype(np.float32).astype(np.float64)); bs.append(b)
    for row, b in zip(rows, bs):
        outs.append(compress.max_pool(row, b).values)
    rf, ro = ragged(rows, np.float64)
    of, oo = ragged(outs, np.float64)
    np.savez_compressed(OUT / "maxpool.npz", rows=rf, row_off=ro, block=np.array(bs), out=of, out_off=oo)


def gen_expand(rng):
    blocks, bs, ts, outs = [], [], [], []
    for blk, b, t in (({2}, 16, 64), ({0}, 4, 10), ({2}, 4, 10), ({0, 1, 4}, 8, 37)):
        blocks.append(sorted(blk)); bs.append(b); ts.append(t)
    for _ in range(200):
        b = int(rng.integers(1, 40)); t = int(rng.integers(1, 5000))
        n = -(-t // b)
        k = int(rng.integers(0, min(n, 60) + 1))
        blk = sorted(rng.choice(n, k, replace=False).tolist())
        blocks.append(blk); bs.append(b); ts.append(t)
    for blk, b, t in zip(blocks, bs, ts):
        outs.append(sorted(compress.expand_indices(blk, b, t)))
    bf, bo = ragged(blocks, np.int64)
    of, oo = ragged(outs, np.int64)
    np.savez_compressed(OUT / "expand.npz", blocks=bf, blocks_off=bo, block=np.array(bs), t=np.array(ts),
                        out=of, out_off=oo)


def gen_topk(rng):
    vals, ks, outs = [], [], []
    for v, k in (([0.1, 0.4, 0.3, 0.2], 2), ([0.5, 0.5, 0.0], 1), ([0.3, 0.1, 0.2], 3),
                 ([-0.0, 0.0, -0.0, 0.0], 2), ([0.0, -0.0, 1.0], 2),
                 ([-np.inf, 1.0, -np.inf, 2.0], 2), ([-np.inf, -np.inf, 3.0], 1)):
        vals.append(np.asarray(v, np.float64)); ks.append(k)
    for _ in range(300):
        n = int(rng.integers(1, 3000))
        kind = rng.integers(0, 5)
        if kind == 0:
            v = rng.standard_normal(n)
        elif kind == 1:
            v = np.round(rng.standard_normal(n) * 3) / 3  # heavy ties
        elif kind == 2:
            v = rng.standard_normal(n); v[rng.random(n) < 0.1] = -np.inf
        elif kind == 3:
            v = np.where(rng.random(n) < 0.5, 0.0, -0.0)  # signed zeros compare equal
            hot = rng.random(n) < 0.05
            v[hot] = rng.standard_normal(int(hot.sum()))
        else:
            v = rng.random(n) * 1e-30  # denormal-ish small values
        v = v.astype(np.float32).astype(np.float64)
        k = int(rng.integers(0, n + 1)) if rng.random() < 0.3 else int(min(n, rng.integers(1, 130)))
        vals.append(v); ks.append(k)
    for v, k in zip(vals, ks):
        outs.append(sorted(selector.topk(v, k)))
    vf, vo = ragged(vals, np.float64)
    of, oo = ragged(outs, np.int64)
    np.savez_compressed(OUT / "topk.npz", values=vf, values_off=vo, k=np.array(ks), out=of, out_off=oo)


def gen_forward(rng):
    shapes = [(6, 9), (8, 10), (8, 100), (1, 12), (4, 12), (64, 12), (5, 7), (3, 1), (1, 1),
              (8, 129), (16, 256), (64, 37), (64, 256), (64, 300), (2, 513)]
    grids, wflat, outs, hs, ws = [], [], [], [], []
    for i, (h, w) in enumerate(shapes):
        wt = predictor.init_weights(i % 4)
        if i % 3 == 1:  # biased variant, N(0, 0.1^2)
            wt.b1 = rng.standard_normal(16) * 0.1
            wt.b2 = rng.standard_normal(32) * 0.1
            wt.b3 = np.array(rng.standard_normal() * 0.1)
        # round-trip through float32 so the device sees identical values
        wt = predictor.PredictorWeights.from_flat(wt.flat().astype(np.float32).astype(np.float64))
        kind = i % 3
        if kind == 0:
            g = rng.random((h, w))
        elif kind == 1:
            g = rng.dirichlet(np.full(w, 0.1), size=h)
        else:
            g = np.zeros((h, w)); g[:, : max(1, w // 2)] = rng.random((h, max(1, w // 2)))
        g = g.astype(np.float32).astype(np.float64)
        out = predictor.forward(wt, predictor.AttentionHistory(g))
        grids.append(g); wflat.append(wt.flat()); outs.append(out); hs.append(h); ws.append(w)
    gf, go = ragged(grids, np.float64)
    of, oo = ragged(outs, np.float64)
    np.savez_compressed(OUT / "forward.npz", grids=gf, grids_off=go, H=np.array(hs), W=np.array(ws),
                        weights=np.stack(wflat), out=of, out_off=oo)


def gen_weights(tmp: Path):
    flats = np.stack([predictor.init_weights(s).flat() for s in range(4)])
    path = tmp / "w.apw1"
    predictor.save_weights(predictor.init_weights(3), path)
    np.savez_compressed(OUT / "weights.npz", init_flat=flats, apw1_seed3=np.frombuffer(path.read_bytes(), np.uint8))


def run_loop(trace, cfg, weights, layer, head):
    """evaluation._iter_selections predictor branch (evaluation.py:90-115), recording the
    forecaster output of every update through a wrapper around selector.forward."""
    seen = []
    real_forward = selector.forward

    def spy(w, hist):
        out = real_forward(w, hist)
        seen.append(out.copy())
        return out

    selector.forward = spy
    try:
        from attncast.evaluation import EvalParams, _iter_selections
        params = EvalParams(budget=cfg.budget, block_size=cfg.block_size, history=cfg.history,
                            calibration_period=cfg.calibration_period, sink_tokens=cfg.sink_tokens,
                            local_tokens=cfg.local_tokens, update_interval=cfg.update_interval,
                            weights=weights)
        sels = [sorted(s) for _, s in _iter_selections(trace, "predictor", params, layer, head)]
    finally:
        selector.forward = real_forward
    return sels, seen


def gen_loops():
    cases = [
        # name, synth kwargs, keep_prefill, cfg kwargs, weight seed, biased
        ("h8_b256", dict(head_dim=32, prefill_len=600, decode_steps=48, query_drift=0.15, key_drift=0.15,
                         seasonal_period=0, reaccess_positions=frozenset(range(200, 210)), rng_seed=11, num_heads=2),
         16, dict(budget=256, block_size=16, history=8, calibration_period=5), 0, False),
        ("h64_b1024", dict(head_dim=64, prefill_len=2100, decode_steps=40, query_drift=0.15, key_drift=0.15,
                           seasonal_period=5, reaccess_positions=frozenset(range(700, 712)), rng_seed=3, num_heads=1),
         64, dict(budget=1024, block_size=16, history=64, calibration_period=5), 1, True),
        ("h16_ui4", dict(head_dim=32, prefill_len=900, decode_steps=30, query_drift=0.2, key_drift=0.2,
                         seasonal_period=7, reaccess_positions=frozenset(range(300, 305)), rng_seed=5, num_heads=1),
         20, dict(budget=384, block_size=16, history=16, calibration_period=3, update_interval=4), 2, True),
        ("h64_short", dict(head_dim=32, prefill_len=130, decode_steps=40, query_drift=0.2, key_drift=0.2,
                           seasonal_period=0, reaccess_positions=frozenset(), rng_seed=9, num_heads=1),
         10, dict(budget=512, block_size=16, history=64, calibration_period=5), 3, False),
    ]
    rng = np.random.default_rng(1234)
    for name, skw, keep, ckw, wseed, biased in cases:
        trace = gen_trace(SynthConfig(**skw), keep_prefill_rows=keep)
        wt = predictor.init_weights(wseed)
        if biased:
            wt.b1 = rng.standard_normal(16) * 0.1
            wt.b2 = rng.standard_normal(32) * 0.1
            wt.b3 = np.array(rng.standard_normal() * 0.1)
        wt = predictor.PredictorWeights.from_flat(wt.flat().astype(np.float32).astype(np.float64))
        cfg = selector.SelectorConfig(**ckw)
        h = trace.header
        store = {"weights": wt.flat(), "cfg": np.array([cfg.budget, cfg.block_size, cfg.history,
                                                         cfg.calibration_period, cfg.sink_tokens,
                                                         cfg.local_tokens, cfg.update_interval])}
        for head in range(h.num_heads):
            prefill = [trace.row(0, head, s) for s in h.steps if s < 0]
            decode = [trace.row(0, head, t) for t in range(0, h.num_decode_steps)]
            sels, seen = run_loop(trace, cfg, wt, 0, head)
            store[f"prefill_{head}"], store[f"prefill_{head}_off"] = ragged(prefill, np.float32)
            store[f"decode_{head}"], store[f"decode_{head}_off"] = ragged(decode, np.float32)
            store[f"sel_{head}"], store[f"sel_{head}_off"] = ragged(sels, np.int64)
            store[f"pred_{head}"], store[f"pred_{head}_off"] = ragged(seen, np.float64)
        store["num_heads"] = np.array(h.num_heads)
        np.savez_compressed(OUT / f"loop_{name}.npz", **store)


def gen_trace_fixture():
    """trace_tiny.att1: the reference's tiny_trace fixture shape (pkg/tests/conftest.py:72-87, q/k
    included) written by attncast.trace.write_trace (trace.py:182-212); trace_tiny.npz: the rows and
    q/k blocks as attncast.trace.read_trace decodes them, plus the predictor branch's middle blocks
    (evaluation.py:90-115) per (layer, head, step) for a device replay through the C++ reader."""
    from attncast import trace as T
    tr = gen_trace(SynthConfig(head_dim=16, prefill_len=96, decode_steps=30, query_drift=0.2, key_drift=0.2,
                               seasonal_period=5, reaccess_positions=frozenset({7, 40}), rng_seed=5, num_layers=2,
                               num_heads=2), keep_prefill_rows=8)
    path = OUT / "trace_tiny.att1"
    with open(path, "wb") as fh:
        T.write_trace(tr, fh)
    with open(path, "rb") as fh:
        back = T.read_trace(fh)
    assert back == tr
    h = back.header
    store = {"header": np.array([h.num_layers, h.num_heads, h.prefill_len, h.num_decode_steps, int(h.has_qk),
                                 h.head_dim, h.first_step_offset])}
    cfg = selector.SelectorConfig(budget=96, block_size=16, history=8, calibration_period=5, sink_tokens=16,
                                  local_tokens=16)
    wt = predictor.init_weights(7)
    store["weights"] = wt.flat()
    store["cfg"] = np.array([cfg.budget, cfg.block_size, cfg.history, cfg.calibration_period, cfg.sink_tokens,
                             cfg.local_tokens, cfg.update_interval])
    for layer in range(h.num_layers):
        for head in range(h.num_heads):
            store[f"rows_{layer}_{head}"], store[f"rows_{layer}_{head}_off"] = ragged(
                [back.row(layer, head, s) for s in h.steps], np.float32)
            store[f"q_{layer}_{head}"] = back.queries[layer][head]
            store[f"k_{layer}_{head}"] = back.head_keys(layer, head)
            sels, _ = run_loop(back, cfg, wt, layer, head)
            mids = []
            for t, sel in enumerate(sels):
                nl = h.prefill_len + t + 1  # selection for the row of length prefill + t + 1
                sink = set(range(min(cfg.sink_tokens, nl)))
                local = set(range(max(0, nl - cfg.local_tokens), nl))
                mids.append(sorted({i // cfg.block_size for i in set(sel) - sink - local}))
            store[f"mid_{layer}_{head}"], store[f"mid_{layer}_{head}_off"] = ragged(mids, np.int64)
    np.savez_compressed(OUT / "trace_tiny.npz", **store)


def main():
    import tempfile
    rng = np.random.default_rng(20250204)
    gen_maxpool(rng)
    gen_expand(rng)
    gen_topk(rng)
    gen_forward(rng)
    with tempfile.TemporaryDirectory() as d:
        gen_weights(Path(d))
    gen_loops()
    gen_trace_fixture()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()

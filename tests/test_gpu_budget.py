"""Budget allocation on the device (ap_selector.k_map): every map's selection equals the float64
oracle's run with THAT map's budget (selector.py:47-50 per map), at the cfg1 shape, with the
exact-boundary guard (no near-tie exemptions)."""

import numpy as np
import pytest

from oracle import hotpath as O

pytestmark = pytest.mark.gpu


def test_per_map_budgets_match_oracle():
    import torch
    from paper_2502_04077_b200 import predictor
    from paper_2502_04077_b200.batched import PUSH_DENSE, PUSH_PREFILL, BatchedSelector
    from paper_2502_04077_b200.selector import SelectorConfig
    rng = np.random.default_rng(21)
    n_maps, t0, steps = 24, 4070, 8
    budgets = rng.choice([128, 256, 512, 1024, 2048], size=n_maps)
    budgets[0], budgets[1] = 128, 2048  # a map with no middle blocks, one at the pitch
    cfg = SelectorConfig(budget=2048)
    w = O.init_weights(4)
    w.b1 = rng.standard_normal(16) * 0.1
    w = O.Weights.from_flat(w.flat().astype(np.float32).astype(np.float64))
    predictor.install_weights(predictor.PredictorWeights.from_flat(w.flat()))
    dev = BatchedSelector(cfg, n_maps, w_max=256, budgets=budgets)
    prefill = [rng.dirichlet(np.full(t0 - 63 + i, 0.05), size=n_maps).astype(np.float32) for i in range(63)]
    for p in prefill:
        dev.push_rows(torch.from_numpy(p).cuda(), p.shape[1], mode=PUSH_PREFILL)
    ocfgs = [O.Config(budget=int(b)) for b in budgets]
    ost = [O.init_state(ocfgs[m], [p[m] for p in prefill]) for m in range(n_maps)]
    osel = [None] * n_maps
    for s in range(steps):
        rows = rng.dirichlet(np.full(t0 + s, 0.05), size=n_maps).astype(np.float32)
        dev.push_rows(torch.from_numpy(rows).cuda(), rows.shape[1], mode=PUSH_DENSE)
        dev.step()
        dev.check_status()
        for m in range(n_maps):
            row = rows[m].astype(np.float64)
            obs = row if osel[m] is None else O.observed_from_selection(row, osel[m])
            ost[m], osel[m] = O.step(ost[m], ocfgs[m], w, obs, full_row=row)
            assert dev.middle(m) == ost[m].last_blocks, f"step {s} map {m} (budget {budgets[m]})"
            assert len(dev.middle(m)) == ocfgs[m].middle_blocks


def test_engine_layer_budgets():
    import torch
    from paper_2502_04077_b200.budget import allocate
    from paper_2502_04077_b200.decode import DecodeEngine, ModelShape
    from paper_2502_04077_b200.selector import SelectorConfig
    tiny = ModelShape("tiny", n_layers=3, hidden=512, n_q_heads=4, n_kv_heads=2, ffn=1024, vocab=1000,
                      rope_theta=10000.0)
    cfg = SelectorConfig(budget=384, calibration_period=3)
    per_map = allocate(cfg, 3, 2, policy="weights", layer_weights=[3, 2, 1], mean_budget=256)
    lb = per_map[::2]
    eng = DecodeEngine(tiny, 1, 700, max_new=8, cfg=cfg, group=2, layer_budgets=lb)
    eng.init_history()
    for _ in range(4):
        eng.step()
    torch.cuda.synchronize()
    st = eng.sel.states()
    want = np.repeat((lb - 128) // 16, 2)
    assert np.array_equal(st["n_mid"], want), (st["n_mid"], want)

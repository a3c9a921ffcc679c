"""Pin the CPU oracle against golden vectors produced by the real reference.

CPU-only.  The golden fixtures come from tests/golden/gen_golden.py, which
ran /root/reference/pkg/src/attncast in the build container.  If the oracle
ever drifts from the reference these fail before any GPU parity test can
pass against a wrong checker.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import LOOP_CASES, load_golden, loop_case, unragged
from oracle import hotpath as H
from oracle import attention as A


def test_maxpool_golden_exact():
    z = load_golden("maxpool")
    rows = unragged(z["rows"], z["row_off"])
    outs = unragged(z["out"], z["out_off"])
    for row, b, want in zip(rows, z["block"], outs):
        got = H.max_pool(row, int(b))
        assert got.shape == want.shape
        assert np.array_equal(got, want)  # max is exact: bit-for-bit (±0 compare equal)


def test_maxpool_errors():
    with pytest.raises(H.OracleError, match="ParameterError"):
        H.max_pool([0.5, 0.5], 0)
    with pytest.raises(H.OracleError, match="ParameterError"):
        H.max_pool([], 4)


def test_expand_golden_exact():
    z = load_golden("expand")
    blocks = unragged(z["blocks"], z["blocks_off"])
    outs = unragged(z["out"], z["out_off"])
    for blk, b, t, want in zip(blocks, z["block"], z["t"], outs):
        assert sorted(H.expand_indices(blk.tolist(), int(b), int(t))) == want.tolist()
    with pytest.raises(H.OracleError):
        H.expand_indices({3}, 4, 10)


def test_topk_golden_exact():
    z = load_golden("topk")
    vals = unragged(z["values"], z["values_off"])
    outs = unragged(z["out"], z["out_off"])
    for v, k, want in zip(vals, z["k"], outs):
        assert sorted(H.topk(v, int(k))) == want.tolist()


def test_forward_golden():
    z = load_golden("forward")
    grids = unragged(z["grids"], z["grids_off"])
    outs = unragged(z["out"], z["out_off"])
    for g, h, w, wf, want in zip(grids, z["H"], z["W"], z["weights"], outs):
        got = H.forward(H.Weights.from_flat(wf), g.reshape(int(h), int(w)))
        scale = max(1.0, float(np.abs(want).max()))
        assert np.max(np.abs(got - want)) <= 1e-12 * scale


def test_row_contribution_form_matches_forward():
    z = load_golden("forward")
    grids = unragged(z["grids"], z["grids_off"])
    outs = unragged(z["out"], z["out_off"])
    for g, h, w, wf, want in zip(grids, z["H"], z["W"], z["weights"], outs):
        wt = H.Weights.from_flat(wf)
        r = H.row_contributions(wt, g.reshape(int(h), int(w)))
        got = float(wt.b3) + r.mean(axis=0)
        assert np.allclose(got, want, rtol=0, atol=1e-12 * max(1.0, np.abs(want).max()))


def test_init_weights_and_apw1_pinned(tmp_path):
    z = load_golden("weights")
    for s in range(4):
        assert np.array_equal(H.init_weights(s).flat(), z["init_flat"][s])
    p = tmp_path / "w.apw1"
    H.save_apw1(H.init_weights(3), p)
    assert p.read_bytes() == z["apw1_seed3"].tobytes()
    back = H.load_apw1(p)
    assert np.array_equal(back.flat(), H.init_weights(3).flat().astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("case", LOOP_CASES)
def test_selector_loop_golden(case):
    c = loop_case(case)
    cfg = H.Config(**c["cfg"])
    w = H.Weights.from_flat(c["weights"])
    for head in c["heads"]:
        st = H.init_state(cfg, head["prefill"])
        sel = None
        preds = []
        for t, row in enumerate(head["decode"]):
            row = np.asarray(row, np.float64)
            obs = row if sel is None else H.observed_from_selection(row, sel)
            before = st.counter
            st, sel = H.step(st, cfg, w, obs, full_row=row)
            if before % cfg.update_interval == 0 and cfg.middle_blocks > 0:
                preds.append(st.last_scores)
            assert sorted(sel) == head["sel"][t].tolist(), f"step {t}"
        assert len(preds) == len(head["pred"])
        for a, b in zip(preds, head["pred"]):
            assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.abs(b).max())


def test_attention_oracle_consistency():
    rng = np.random.default_rng(0)
    t, d, b = 300, 64, 16
    q = rng.standard_normal(d)
    K = rng.standard_normal((t, d))
    V = rng.standard_normal((t, d))
    out, lse, p = A.dense_decode(q, K, V)
    assert np.isclose(p.sum(), 1.0)
    # calibration row == max_pool of the dense softmax row
    assert np.array_equal(A.calibration_row(q, K, b), H.max_pool(p, b))
    # a selection that covers everything reproduces dense attention
    o2, lse2, _, _ = A.sparse_decode(q, K, V, range(t))
    assert np.allclose(o2, out) and np.isclose(lse, lse2)
    sel = A.selection_tokens(t, 64, 64, [6, 9], b, t)
    row = A.observed_row_masked_dense(q, K, sel, t)
    assert np.array_equal(row, H.observed_from_selection(p, sel))

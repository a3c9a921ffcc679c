"""GPU parity of the decode-attention kernels (kernel 4a/4b) against the float64 oracle.

The reference has no attention implementation for this path; the oracle
restates attntap/model.py:70-74 (oracle/attention.py).  Tolerances: attention
outputs from bf16 q/K/V within 2e-2 of the output scale (the north_star's
bf16 bound); LSE within 1e-3; compressed calibration / observed rows within
rtol 1e-3 (fp32 exp of fp32 logits).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import attention as A
from oracle import hotpath as O

pytestmark = pytest.mark.gpu

LN2 = np.log(2.0)


def _setup(S=2, Hq=8, Hkv=2, t_max=1024, seed=0):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    q = (torch.randn(S, Hq, 128, generator=g) * 1.5).to(torch.bfloat16)
    k = torch.randn(S, Hkv, t_max, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(S, Hkv, t_max, 128, generator=g).to(torch.bfloat16)
    # make a few "heavy hitter" keys so rows are peaked, like real attention
    k[:, :, 100:104] += q[:, ::(Hq // Hkv)].unsqueeze(2).float().mul(0.2).to(torch.bfloat16)
    return q, k, v


def _f64(x):
    return x.float().cpu().numpy().astype(np.float64)


def _selector(n_maps, w_max, budget=1024):
    from paper_2502_04077_b200.batched import BatchedSelector
    from paper_2502_04077_b200.selector import SelectorConfig
    return BatchedSelector(SelectorConfig(budget=budget), n_maps, w_max)


@pytest.mark.parametrize("Hq,Hkv,group", [(8, 2, 1), (8, 2, 4), (4, 4, 1)])  # (4, 4): MHA, one q-head per KV head
def test_dense_attention_and_calibration_row(Hq, Hkv, group):
    import torch
    from paper_2502_04077_b200.attention import DecodeAttention
    S, t_max = 2, 1024
    q, k, v = _setup(S, Hq, Hkv, t_max)
    lens = [700, 1013]
    seq_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_dense=4)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    out = torch.empty(S, Hq, 128, dtype=torch.bfloat16, device="cuda")
    maps = Hq // group
    sel = _selector(S * maps, t_max // 16)
    att.dense(qd, kd, vd, seq_len, out, with_v=True, emit=True, selector=sel, map_base=0, maps_per_seq=maps,
              group=group)
    torch.cuda.synchronize()
    outn = _f64(out)
    lse2 = att.lse.cpu().numpy()
    ring = sel.ring.cpu().numpy()
    for s in range(S):
        t = lens[s]
        rows = []
        for h in range(Hq):
            kvh = h // (Hq // Hkv)
            K = _f64(k[s, kvh, :t])
            V = _f64(v[s, kvh, :t])
            ref, lse, p = A.dense_decode(_f64(q[s, h]), K, V)
            scale = np.abs(ref).max()
            assert np.max(np.abs(outn[s, h] - ref)) <= 2e-2 * scale, (s, h)
            assert abs(lse2[s, h] * LN2 - lse) <= 1e-3
            rows.append(O.max_pool(p, 16))
        for g in range(maps):
            want = np.max(rows[g * group:(g + 1) * group], axis=0)
            got = ring[s * maps + g, 0, : want.size]
            assert np.allclose(got, want, rtol=1e-3, atol=1e-7 * want.max()), (s, g)
    st = sel.states()
    assert (st["n_pushed"] == 1).all()
    assert list(st["row_len"][::maps]) == lens


def _set_selection(sel, rng, lens, maps, k_mid, b=16):
    """Give every map a random middle-block set disjoint from its sink/local covering blocks."""
    import torch
    st = sel.states().copy()
    blocks_per_map = []
    for m in range(st.size):
        t = lens[m // maps]
        W = -(-t // b)
        banned = set(range(0, 4)) | set(range((t - 64) // b, W + 1))
        cand = [j for j in range(W) if j not in banned]
        blk = sorted(rng.choice(cand, size=min(k_mid, len(cand)), replace=False).tolist())
        blocks_per_map.append(blk)
        st[m]["n_mid"] = len(blk)
        st[m]["mid_clip"] = t - 1
        sel.mid_blocks[m, : len(blk)] = torch.tensor(blk, dtype=torch.int32)
    sel.state.copy_(torch.from_numpy(st.view(np.uint8).copy()))
    return blocks_per_map


@pytest.mark.parametrize("splits", [2, 3, 4, 8, 16])  # 3: global-memory combine; others: one cluster per map
@pytest.mark.parametrize("group", [1, 4])
def test_sparse_attention_and_observed_row(group, splits):
    import torch
    from paper_2502_04077_b200.attention import DecodeAttention
    S, Hq, Hkv, t_max = 2, 8, 2, 2048
    q, k, v = _setup(S, Hq, Hkv, t_max, seed=3)
    lens = [1500, 2001]
    seq_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_sparse=splits)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    out = torch.empty(S, Hq, 128, dtype=torch.bfloat16, device="cuda")
    maps = Hq // group
    sel = _selector(S * maps, t_max // 16)
    sel.ring.fill_(7.0)  # stale slot content: everything outside the selection must be re-zeroed
    blocks = _set_selection(sel, np.random.default_rng(1), lens, maps, 56)
    att.sparse(qd, kd, vd, seq_len, out, sel, emit=True, map_base=0, maps_per_seq=maps, group=group)
    torch.cuda.synchronize()
    outn = _f64(out)
    lse2 = att.lse.cpu().numpy()
    ring = sel.ring.cpu().numpy()
    for s in range(S):
        t = lens[s]
        for g in range(maps):
            m = s * maps + g
            toks = A.selection_tokens(t, 64, 64, blocks[m], 16, t - 1)
            rows = []
            for h in range(g * group, (g + 1) * group):
                kvh = h // (Hq // Hkv)
                K = _f64(k[s, kvh, :t])
                V = _f64(v[s, kvh, :t])
                ref, lse, _, _ = A.sparse_decode(_f64(q[s, h]), K, V, toks)
                assert np.max(np.abs(outn[s, h] - ref)) <= 2e-2 * np.abs(ref).max(), (s, h)
                assert abs(lse2[s, h] * LN2 - lse) <= 1e-3
                rows.append(O.max_pool(A.observed_row_sparse_renorm(_f64(q[s, h]), K, toks, t), 16))
            want = np.max(rows, axis=0)
            got = ring[m, 0, : want.size]
            assert np.allclose(got, want, rtol=1e-3, atol=1e-7 * want.max()), (s, g)
            assert np.count_nonzero(got) == np.count_nonzero(want)
            assert not ring[m, 0, want.size:].any()  # zero beyond the row's width
            assert np.isclose(float(sel.slot_xmax[m, 0]), float(got.max()), rtol=1e-6)
    st = sel.states()
    assert (st["n_pushed"] == 1).all()
    assert list(st["width"][::maps]) == [-(-t // 16) for t in lens]


@pytest.mark.parametrize("splits", [2, 3, 8])
def test_sparse_with_full_selection_equals_dense(splits):
    """With a budget that covers every block, sparse attention reproduces dense attention."""
    import torch
    from paper_2502_04077_b200.attention import DecodeAttention
    S, Hq, Hkv, t_max = 1, 4, 1, 512
    q, k, v = _setup(S, Hq, Hkv, t_max, seed=5)
    t = 500
    seq_len = torch.tensor([t], dtype=torch.int32, device="cuda")
    att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_dense=2, n_splits_sparse=splits)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    o1 = torch.empty(S, Hq, 128, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    sel = _selector(Hq, t_max // 16, budget=4096)
    st = sel.states().copy()
    W = -(-t // 16)
    mid = [j for j in range(W) if j >= 4 and j < (t - 64) // 16]
    for m in range(Hq):
        st[m]["n_mid"] = len(mid)
        st[m]["mid_clip"] = t
        sel.mid_blocks[m, : len(mid)] = torch.tensor(mid, dtype=torch.int32)
    sel.state.copy_(torch.from_numpy(st.view(np.uint8).copy()))
    att.dense(qd, kd, vd, seq_len, o1, with_v=True)
    att.sparse(qd, kd, vd, seq_len, o2, sel, emit=False)
    torch.cuda.synchronize()
    assert torch.allclose(o1.float(), o2.float(), atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("kernel", [1, 0])  # 1: TMA + tcgen05 calibration pass, 0: SIMT dense kernel
@pytest.mark.parametrize("group", [1, 4])
def test_calibration_pass_k_only(group, kernel):
    """ap_attn_dense(with_v=0, emit) — the K-only pass of calibration steps — against the float64
    oracle: LSE and the compressed calibration row max_pool(softmax row) pushed into the ring; two
    consecutive steps (ring slot, per-step synchronisation state and map state advance)."""
    import torch
    from paper_2502_04077_b200 import _lib
    from paper_2502_04077_b200.attention import DecodeAttention
    S, Hq, Hkv, t_max = 2, 8, 2, 2048
    q, k, _ = _setup(S, Hq, Hkv, t_max, seed=5)
    maps = Hq // group
    sel = _selector(S * maps, t_max // 16)
    att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_dense=32)
    kd = k.cuda()
    prev = _lib.fn("ap_attn_set_calib_kernel")(kernel)
    try:
        for step, lens in enumerate(([700, 2039], [701, 1300])):
            qs = q if step == 0 else (q.float() * -0.7).to(torch.bfloat16)
            seq_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
            att.dense(qs.cuda(), kd, kd, seq_len, None, with_v=False, emit=True, selector=sel, map_base=0,
                      maps_per_seq=maps, group=group)
            torch.cuda.synchronize()
            lse2 = att.lse.cpu().numpy()
            ring = sel.ring.cpu().numpy()
            for s in range(S):
                t = lens[s]
                rows = []
                for h in range(Hq):
                    K = _f64(k[s, h // (Hq // Hkv), :t])
                    _, lse, p = A.dense_decode(_f64(qs[s, h]), K, K)
                    assert abs(lse2[s, h] * LN2 - lse) <= 1e-3, (step, s, h)
                    rows.append(O.max_pool(p, 16))
                for g in range(maps):
                    want = np.max(rows[g * group:(g + 1) * group], axis=0)
                    got = ring[s * maps + g, step, :]
                    assert np.allclose(got[: want.size], want, rtol=1e-3, atol=1e-7 * want.max()), (step, s, g)
                    assert not got[want.size:].any()  # zero beyond the row's width
            st = sel.states()
            assert (st["n_pushed"] == step + 1).all()
            assert list(st["row_len"][::maps]) == lens
            xmax = sel.slot_xmax.cpu().numpy()[:, step]
            assert np.allclose(xmax, ring[:, step, :].max(axis=1))
    finally:
        _lib.fn("ap_attn_set_calib_kernel")(prev)

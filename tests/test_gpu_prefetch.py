"""GPU tests of the cross-token prefetch (kernel 5) and paged-V sparse attention.

Oracle for the gather: byte-exact numpy fancy indexing of the host V
(oracle/attention.gather_blocks); the delta cache must keep the pages of
blocks selected again and copy only the new ones; sparse attention over the
paged store must equal sparse attention over a fully resident V bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import attention as A

pytestmark = pytest.mark.gpu


def _engine_parts(L=2, S=1, Hq=8, Hkv=2, t_max=2048, k_cap=8, budget=256):
    import torch
    from paper_2502_04077_b200.batched import BatchedSelector
    from paper_2502_04077_b200.prefetch import OffloadedV
    from paper_2502_04077_b200.selector import SelectorConfig
    cfg = SelectorConfig(budget=budget)  # K = (256 - 128) / 16 = 8 middle blocks
    sel = BatchedSelector(cfg, S * L * Hkv, t_max // 16)
    vo = OffloadedV(L, S, Hkv, t_max, k_cap=k_cap)
    g = torch.Generator().manual_seed(0)
    vo.host_v.copy_(torch.randn(vo.host_v.shape, generator=g).to(torch.bfloat16))
    return cfg, sel, vo


def _set_middle(sel, blocks_per_map, clip):
    import torch
    st = sel.states().copy()
    for m, blk in enumerate(blocks_per_map):
        st[m]["n_mid"] = len(blk)
        st[m]["mid_clip"] = clip
        sel.mid_blocks[m, : len(blk)] = torch.tensor(blk, dtype=torch.int32)
    sel.state.copy_(torch.from_numpy(st.view(np.uint8).copy()))


def _check_pages(vo, sel, L, S, Hkv):
    pages = vo.pages.cpu().view(np.int16).numpy() if False else vo.pages.float().cpu().numpy()
    host = vo.host_v.float().numpy()
    st = sel.states()
    mp = vo.mid_page.cpu().numpy()
    base = vo.sink_pages + vo.recent_pages
    for l in range(L):
        for s in range(S):
            for h in range(Hkv):
                smap = s * L * Hkv + l * Hkv + h
                vmap = (l * S + s) * Hkv + h
                n = int(st[smap]["n_mid"])
                blk = sel.mid_blocks[smap, :n].cpu().tolist()
                want = A.gather_blocks(host[l, s, h], blk, 16)
                got = np.concatenate([pages[vmap, base + mp[vmap, i]] for i in range(n)])
                assert np.array_equal(got, want), (l, s, h)


def test_prefetch_gather_and_delta_cache():
    import torch
    L, S, Hkv = 2, 1, 2
    cfg, sel, vo = _engine_parts(L, S, 8, Hkv)
    rng = np.random.default_rng(0)
    first = [sorted(rng.choice(np.arange(4, 80), 8, replace=False).tolist()) for _ in range(L * S * Hkv)]
    _set_middle(sel, first, 1499)
    for l in range(L):
        vo.prefetch(sel, l, L * Hkv)
    torch.cuda.synchronize()
    assert int(vo.bytes_copied.item()) == sum(len(b) for b in first) * 4096
    _check_pages(vo, sel, L, S, Hkv)
    pages_before = vo.mid_page.cpu().numpy().copy()
    # next step: keep 5 of 8 blocks, 3 new ones
    second = []
    for b in first:
        keep = b[:5]
        new = sorted(set(rng.choice(np.arange(4, 80), 12, replace=False).tolist()) - set(b))[:3]
        second.append(sorted(keep + new))
    _set_middle(sel, second, 1500)
    vo.bytes_copied.zero_()
    for l in range(L):
        vo.prefetch(sel, l, L * Hkv)
    torch.cuda.synchronize()
    assert int(vo.bytes_copied.item()) == 3 * 4096 * len(second)  # only the new blocks crossed the link
    _check_pages(vo, sel, L, S, Hkv)
    after = vo.mid_page.cpu().numpy()
    for m, (b1, b2) in enumerate(zip(first, second)):
        vmap = m  # S == 1: vmap == smap ordering for (l, h) since L*Hkv maps in (l, h) order
        for j in set(b1) & set(b2):
            assert after[vmap, b2.index(j)] == pages_before[vmap, b1.index(j)]  # kept block kept its page


def test_paged_sparse_attention_equals_resident():
    import torch
    from paper_2502_04077_b200.attention import DecodeAttention
    L, S, Hq, Hkv, t_max = 2, 1, 8, 2, 2048
    cfg, sel, vo = _engine_parts(L, S, Hq, Hkv, t_max)
    t = 1500
    vo.init_pages(t)
    g = torch.Generator().manual_seed(1)
    q = torch.randn(S, Hq, 128, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(L, S, Hkv, t_max, 128, generator=g).to(torch.bfloat16).cuda()
    v_res = vo.host_v.cuda()
    seq_len = torch.tensor([t], dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(3)
    mids = [sorted(rng.choice(np.arange(4, 85), 8, replace=False).tolist()) for _ in range(L * Hkv)]
    _set_middle(sel, mids, t - 1)
    for l in range(L):
        vo.prefetch(sel, l, L * Hkv)
    att = DecodeAttention(S, Hq, Hkv, t_max, n_splits_sparse=4)
    G = Hq // Hkv
    for l in range(L):
        o_res = torch.empty(S, Hq, 128, dtype=torch.bfloat16, device="cuda")
        o_pag = torch.empty_like(o_res)
        att.sparse(q, k[l], v_res[l], seq_len, o_res, sel, emit=False, map_base=l * Hkv, maps_per_seq=L * Hkv,
                   group=G)
        att.sparse(q, k[l], k[l], seq_len, o_pag, sel, emit=False, map_base=l * Hkv, maps_per_seq=L * Hkv,
                   group=G, vpages=vo, layer=l)
        torch.cuda.synchronize()
        assert torch.equal(o_res, o_pag), f"layer {l}"

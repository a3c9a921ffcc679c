"""Decode engine end to end on a tiny LLaMA-like shape (head_dim 128).

* With a local window longer than the context, the selection is every token, so the sparse
  path must reproduce the dense comparator — with and without the layer-skip policy and for
  both selection granularities (routing of maps, emission and graphs).  A large *budget* alone
  does not make sparse == dense: masking the local window's covering blocks leaves up to 15
  tokens below the window start unselected, exactly as selector.py:137-141 does.
* With a real selection, CUDA-graph replay must equal eager steps bit for bit.
The middle-block gather itself is checked against the oracle in test_gpu_attention.py."""

import pytest

from paper_2502_04077_b200.decode import DecodeEngine, ModelShape
from paper_2502_04077_b200.errors import ConfigError
from paper_2502_04077_b200.selector import SelectorConfig

TINY = ModelShape("tiny", n_layers=3, hidden=512, n_q_heads=4, n_kv_heads=2, ffn=1024, vocab=1000,
                  rope_theta=10000.0)
CTX, STEPS = 700, 7
FULL = SelectorConfig(budget=2048, local_tokens=1024, calibration_period=3)  # local covers [0, t]


def _run(mode, *, group=1, dense_layers=0, use_graph=True, cfg=FULL, steps=STEPS):
    import torch
    eng = DecodeEngine(TINY, 2, CTX, max_new=steps + 4, mode=mode, cfg=cfg, group=group, seed=3,
                       dense_layers=dense_layers)
    eng.init_history()
    logits, toks = [], []
    for _ in range(steps):
        eng.step(use_graph=use_graph)
        torch.cuda.synchronize()
        logits.append(eng.logits.float().clone())
        toks.append(eng.tok.clone())
    return eng, logits, toks


def _close(a, b):
    import torch
    worst = max(float((x - y).abs().max()) for x, y in zip(a, b))
    scale = max(float(x.abs().max()) for x in a)
    return worst <= 2e-2 * scale + 1e-3, worst, scale  # bf16 activations through 3 layers


@pytest.mark.gpu
@pytest.mark.parametrize("group,dense_layers", [(1, 0), (2, 0), (1, 1), (2, 2)])
def test_full_budget_sparse_equals_dense(group, dense_layers):
    _, ld, td = _run("dense")
    eng, ls, ts = _run("sparse", group=group, dense_layers=dense_layers)
    assert eng.sel.n_maps == 2 * (TINY.n_layers - dense_layers) * (TINY.n_q_heads // group)
    ok, worst, scale = _close(ld, ls)
    assert ok, f"logits differ: {worst} (scale {scale})"


@pytest.mark.gpu
def test_graph_replay_equals_eager():
    import torch
    cfg = SelectorConfig(budget=256, calibration_period=3)  # real selection: 8 middle blocks of ~44
    _, lg, tg = _run("sparse", group=2, cfg=cfg, use_graph=True)
    _, le, te = _run("sparse", group=2, cfg=cfg, use_graph=False)
    for a, b in zip(lg, le):
        assert torch.equal(a, b)
    for a, b in zip(tg, te):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_layer_skip_config_errors():
    with pytest.raises(ConfigError):
        DecodeEngine(TINY, 1, CTX, 8, dense_layers=TINY.n_layers)
    with pytest.raises(ConfigError):
        DecodeEngine(TINY, 1, CTX, 8, dense_layers=1, offload_v=True, group=2)


@pytest.mark.gpu
def test_overlapped_selector_equals_end_of_token_step():
    """overlap_selector: each layer's selector step on a side stream (reserved SMs) right after the
    layer's attention gives the same selections, hence the same logits, as one step for all layers at
    the end of the token."""
    import torch
    cfg = SelectorConfig(budget=256, calibration_period=3)
    _, base, _ = _run("sparse", group=2, cfg=cfg, use_graph=True)
    eng = DecodeEngine(TINY, 1, CTX, max_new=STEPS + 4, cfg=cfg, group=2, seed=3, overlap_selector=8)
    eng.init_history()
    ref = DecodeEngine(TINY, 1, CTX, max_new=STEPS + 4, cfg=cfg, group=2, seed=3)
    ref.init_history()
    for _ in range(STEPS):
        eng.step()
        ref.step()
        torch.cuda.synchronize()
        assert torch.equal(eng.sel.mid_blocks, ref.sel.mid_blocks)
        assert torch.equal(eng.logits, ref.logits)
    assert eng.sel.n_maps == TINY.n_layers * 2


@pytest.mark.gpu
def test_advance_embed_equals_advance_and_index_select():
    """ap_advance_embed (the first launch of a step) == seq_len += by, then embed[tokens] rows."""
    import torch
    from paper_2502_04077_b200 import _lib
    _lib.load()
    g = torch.Generator(device="cuda").manual_seed(5)
    V, Hd, S = 1000, 4096, 3
    embed = torch.randn(V, Hd, device="cuda", generator=g).to(torch.bfloat16)
    tok = torch.tensor([7, 999, 0], dtype=torch.int64, device="cuda")
    seq = torch.tensor([10, 20, 30], dtype=torch.int32, device="cuda")
    out = torch.zeros(S, Hd, dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.fn("ap_advance_embed")(_lib.ptr(seq), S, 2, _lib.ptr(embed), _lib.ptr(tok), _lib.ptr(out), Hd,
                                           _lib.stream_handle()), "ap_advance_embed")
    torch.cuda.synchronize()
    assert seq.tolist() == [12, 22, 32]
    assert torch.equal(out, torch.index_select(embed, 0, tok))

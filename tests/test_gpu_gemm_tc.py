"""ap_gemm_tc (tcgen05 skinny GEMM for batch-5..16 decode projections) against a plain PyTorch
fp32 reference of the same product: every batch size 1..16, ragged N (row tiles cut by the tensor
map's bounds), tiles split across CTAs (fp32 partial sums) and whole tiles per CTA, run-to-run
determinism, the argument checks, and the unfused decode engine on it against library GEMMs."""

import pytest

pytestmark = pytest.mark.gpu


def _gemm(W, x, ns, ws=None):
    import torch

    from paper_2502_04077_b200 import _lib
    N, K = W.shape
    if ws is None:
        ws = torch.zeros(_lib.fn("ap_gemm_tc_workspace_bytes")(N, K, ns), dtype=torch.uint8, device="cuda")
    y = torch.full((ns, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    rc = _lib.fn("ap_gemm_tc")(W.data_ptr(), x.data_ptr(), y.data_ptr(), N, K, ns, ws.data_ptr(), ws.numel(),
                               _lib.stream_handle())
    return rc, y


def _check(y, x, W):
    want = x.float() @ W.float().t()
    err = (y.float() - want).abs().max().item()
    # bf16 output rounding (2^-8 relative) on an fp32 accumulation of K bf16 products
    assert err <= 8e-3 * want.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("ns", list(range(1, 17)))
def test_batches(ns):
    import torch
    g = torch.Generator(device="cuda").manual_seed(100 + ns)
    W = (torch.randn(4096, 4096, device="cuda", generator=g) * 0.02).bfloat16()
    x = torch.randn(ns, 4096, device="cuda", generator=g).bfloat16()
    rc, y = _gemm(W, x, ns)
    assert rc == 0
    _check(y, x, W)


@pytest.mark.parametrize("N,K", [(1000, 256), (130, 4096), (6144, 4096), (4096, 14336), (28672, 4096),
                                 (128256, 4096), (77, 512)])
def test_shapes(N, K):
    import torch
    g = torch.Generator(device="cuda").manual_seed(N + K)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    x = torch.randn(8, K, device="cuda", generator=g).bfloat16()
    rc, y = _gemm(W, x, 8)
    assert rc == 0
    _check(y, x, W)


def test_deterministic_and_workspace_reuse():
    """Two launches on one workspace (counters self-reset) give bit-identical results."""
    import torch

    from paper_2502_04077_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(5)
    W = (torch.randn(4096, 14336, device="cuda", generator=g) * 0.02).bfloat16()
    x = torch.randn(12, 14336, device="cuda", generator=g).bfloat16()
    ws = torch.zeros(_lib.fn("ap_gemm_tc_workspace_bytes")(4096, 14336, 12), dtype=torch.uint8, device="cuda")
    outs = [_gemm(W, x, 12, ws)[1] for _ in range(3)]
    _check(outs[0], x, W)
    assert all(torch.equal(outs[0], o) for o in outs[1:])


def test_argument_checks():
    import torch

    from paper_2502_04077_b200 import _lib
    W = torch.zeros(256, 320, device="cuda", dtype=torch.bfloat16)
    x = torch.zeros(4, 320, device="cuda", dtype=torch.bfloat16)
    assert _lib.fn("ap_gemm_tc_workspace_bytes")(256, 320, 4) < 0
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    y = torch.zeros(4, 256, device="cuda", dtype=torch.bfloat16)
    args = (W.data_ptr(), x.data_ptr(), y.data_ptr())
    assert _lib.fn("ap_gemm_tc")(*args, 256, 320, 4, ws.data_ptr(), ws.numel(), None) != 0  # K % 256
    assert _lib.fn("ap_gemm_tc")(*args, 256, 256, 17, ws.data_ptr(), ws.numel(), None) != 0  # n_seq > 16
    assert _lib.fn("ap_gemm_tc")(*args, 256, 256, 4, ws.data_ptr(), 16, None) != 0  # workspace


def test_engine_tc_matches_library_gemm():
    """Batch-8 decode: the engine on ap_gemm_tc produces the same greedy tokens as on cuBLAS for a
    few dense steps (small model shape, both in bf16 with fp32 accumulation)."""
    import torch

    from paper_2502_04077_b200.decode import DecodeEngine, ModelShape
    sh = ModelShape("tiny", n_layers=2, hidden=1024, n_q_heads=8, n_kv_heads=2, ffn=2816, vocab=4096,
                     rope_theta=500000.0)
    a = DecodeEngine(sh, 8, 2048, 8, mode="dense", seed=3, gemm="tc")
    assert a.tc
    b = DecodeEngine(sh, 8, 2048, 8, mode="dense", seed=3)
    b.tc = False
    for e in (a, b):
        e.tok.copy_(torch.arange(8, device="cuda"))
    same = 0
    for _ in range(4):
        a.step(use_graph=False)
        b.step(use_graph=False)
        torch.testing.assert_close(a.logits.float(), b.logits.float(), rtol=0.05, atol=0.05)
        same += int(torch.equal(a.tok, b.tok))
        b.tok.copy_(a.tok)  # keep both on one token path
    assert same >= 3


@pytest.mark.parametrize("rows,n", [(1, 128256), (8, 128256), (16, 32000), (5, 1001), (3, 7)])
def test_argmax_rows_matches_torch(rows, n):
    """ap_argmax_rows (the batch>4 engine's greedy token) against torch.argmax, including ties
    (lowest index wins) and workspace reuse across launches."""
    import torch

    from paper_2502_04077_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(rows * 7 + n)
    ws = torch.zeros(_lib.fn("ap_argmax_workspace_bytes")(rows), dtype=torch.uint8, device="cuda")
    for trial in range(3):
        x = torch.randn(rows, n, device="cuda", generator=g).bfloat16()
        if trial == 1:  # ties: a few copies of the row max at random later positions
            mx = x.max(dim=1, keepdim=True).values
            idx = torch.randint(0, n, (rows, 3), device="cuda", generator=g)
            x.scatter_(1, idx, mx.expand(-1, 3))
        if trial == 2:
            x = torch.round(x * 2) / 2  # heavy ties everywhere
        tok = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
        _lib.check(_lib.fn("ap_argmax_rows")(x.data_ptr(), rows, n, ws.data_ptr(), ws.numel(), tok.data_ptr(),
                                             _lib.stream_handle()), "ap_argmax_rows")
        assert torch.equal(tok, torch.argmax(x, dim=-1)), trial

"""ap_gemv (decode-engine projections) against a plain PyTorch fp32 reference of the same ops:
store, RMSNorm prologue with residual stream, SiLU-gate epilogue and LM head + greedy argmax, for
1..4 activation rows; and the fused engine against the unfused (library GEMM + elementwise) one."""

import pytest

pytestmark = pytest.mark.gpu

RMS, SILU, ARGMAX = 1, 2, 4


def _call(W, x, y, ns, flags, rows=2, residual=None, residual_out=None, ln=None, ws=None, tokens=None, eps=1e-5):
    from paper_2502_04077_b200 import _lib
    N, K = W.shape
    _lib.check(_lib.fn("ap_gemv")(W.data_ptr(), x.data_ptr(), None if y is None else y.data_ptr(), N, K, ns, rows,
                                  flags, _lib.ptr(residual), _lib.ptr(residual_out), _lib.ptr(ln), eps, _lib.ptr(ws),
                                  _lib.ptr(tokens), _lib.stream_handle()), "ap_gemv")


def _rms_ref(x, r, ln, eps=1e-5):
    import torch
    h = (x.float() + (r.float() if r is not None else 0)).bfloat16().float()
    inv = torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + eps)
    return h, (h * inv * ln.float()).bfloat16().float()


def _close(got, want, rtol=2e-2):
    err = (got.float() - want).abs().max().item()
    return err <= rtol * want.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("ns", [1, 2, 3, 4])
@pytest.mark.parametrize("rows", [1, 2, 4])
def test_store(ns, rows):
    import torch
    g = torch.Generator(device="cuda").manual_seed(ns * 10 + rows)
    W = (torch.randn(1000, 4096, device="cuda", generator=g) * 0.02).bfloat16()
    x = torch.randn(ns, 4096, device="cuda", generator=g).bfloat16()
    y = torch.empty(ns, 1000, device="cuda", dtype=torch.bfloat16)
    _call(W, x, y, ns, 0, rows=rows)
    ok, err = _close(y, x.float() @ W.float().t())
    assert ok, err


@pytest.mark.parametrize("ns", [1, 3])
def test_rmsnorm_silu(ns):
    import torch
    g = torch.Generator(device="cuda").manual_seed(7 + ns)
    F, K = 1536, 2048
    W = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.03).bfloat16()
    x = torch.randn(ns, K, device="cuda", generator=g).bfloat16()
    r = torch.randn(ns, K, device="cuda", generator=g).bfloat16()
    ln = (1 + 0.1 * torch.randn(K, device="cuda", generator=g)).bfloat16()
    r_out = torch.empty_like(r)
    act = torch.empty(ns, F, device="cuda", dtype=torch.bfloat16)
    _call(W, x, act, ns, RMS | SILU, residual=r, residual_out=r_out, ln=ln)
    h, xn = _rms_ref(x, r, ln)
    gu = (xn @ W.float().t()).bfloat16().float()
    want = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    ok, err = _close(act, want)
    assert ok, err
    assert torch.equal(r_out.float(), h)  # residual stream written once, exactly


def test_lm_head_argmax():
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    V, K, ns = 50000, 4096, 4
    W = (torch.randn(V, K, device="cuda", generator=g) * 0.02).bfloat16()
    x = torch.randn(ns, K, device="cuda", generator=g).bfloat16()
    r = torch.randn(ns, K, device="cuda", generator=g).bfloat16()
    ln = torch.ones(K, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(48, dtype=torch.uint8, device="cuda")
    tok = torch.full((ns,), -1, dtype=torch.int64, device="cuda")
    logits = torch.empty(ns, V, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):  # the workspace resets itself between calls
        _call(W, x, logits, ns, RMS | ARGMAX, residual=r, ln=ln, ws=ws, tokens=tok)
        torch.cuda.synchronize()
        assert torch.equal(tok, torch.argmax(logits, dim=-1))  # ties -> lowest index, like torch
    _, xn = _rms_ref(x, r, ln)
    ok, err = _close(logits, xn @ W.float().t())
    assert ok, err


def test_argument_errors():
    import torch
    from paper_2502_04077_b200.errors import ParameterError
    W = torch.zeros(8, 12, device="cuda", dtype=torch.bfloat16)
    x = torch.zeros(1, 12, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ParameterError):
        _call(W, x, torch.empty(1, 8, device="cuda", dtype=torch.bfloat16), 1, 0)  # K % 8
    W = torch.zeros(8, 16, device="cuda", dtype=torch.bfloat16)
    x = torch.zeros(5, 16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ParameterError):
        _call(W, x, torch.empty(5, 8, device="cuda", dtype=torch.bfloat16), 5, 0)  # > 4 rows
    with pytest.raises(ParameterError):  # SILU needs [gate; up] row pairs
        _call(W[:7], x[:1], torch.empty(1, 4, device="cuda", dtype=torch.bfloat16), 1, SILU)


def test_fused_engine_matches_unfused():
    import torch
    from paper_2502_04077_b200.decode import DecodeEngine
    from test_gpu_decode import TINY
    outs = []
    for fused in (False, True):
        eng = DecodeEngine(TINY, 2, 700, 8, mode="dense", seed=3, fused=fused)
        eng.step(use_graph=False)
        torch.cuda.synchronize()
        outs.append((eng.logits.float().clone(), eng.tok.clone()))
    (l0, t0), (l1, t1) = outs
    ok, err = _close(l1, l0)
    assert ok, err
    assert torch.equal(t1, torch.argmax(eng.logits, dim=-1))


@pytest.mark.parametrize("ns", [1, 3])
def test_qkv_rope_fused_matches_separate(ns):
    """ap_gemv_qkv_rope == ap_gemv (RMSNORM prologue) followed by ap_rope_append, bit for bit."""
    import torch
    from paper_2502_04077_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(11 + ns)
    Hq, Hkv, K, t_max = 8, 2, 1024, 64
    N = (Hq + 2 * Hkv) * 128
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.03).bfloat16()
    x = torch.randn(ns, K, device="cuda", generator=g).bfloat16()
    r = torch.randn(ns, K, device="cuda", generator=g).bfloat16()
    ln = (1 + 0.1 * torch.randn(K, device="cuda", generator=g)).bfloat16()
    seq_len = torch.tensor([5, 17, 40, 63][:ns], dtype=torch.int32, device="cuda")
    outs = []
    for fused in (False, True):
        y = torch.zeros(ns, N, device="cuda", dtype=torch.bfloat16)
        q = torch.zeros(ns, Hq, 128, device="cuda", dtype=torch.bfloat16)
        kc = torch.zeros(ns, Hkv, t_max, 128, device="cuda", dtype=torch.bfloat16)
        vc = torch.zeros_like(kc)
        r_out = torch.zeros_like(r)
        if fused:
            _lib.check(_lib.fn("ap_gemv_qkv_rope")(W.data_ptr(), x.data_ptr(), y.data_ptr(), Hq, Hkv, K, ns, RMS,
                                                    r.data_ptr(), r_out.data_ptr(), ln.data_ptr(), 1e-5,
                                                    seq_len.data_ptr(), q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                                                    t_max, 500000.0, _lib.stream_handle()), "ap_gemv_qkv_rope")
        else:
            _call(W, x, y, ns, RMS, residual=r, residual_out=r_out, ln=ln)
            _lib.check(_lib.fn("ap_rope_append")(y.data_ptr(), ns, Hq, Hkv, seq_len.data_ptr(), q.data_ptr(),
                                                 kc.data_ptr(), vc.data_ptr(), t_max, 500000.0,
                                                 _lib.stream_handle()), "ap_rope_append")
        torch.cuda.synchronize()
        outs.append((y, q, kc, vc, r_out))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    assert outs[0][2].abs().sum() > 0  # keys were appended

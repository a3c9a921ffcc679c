"""LLaMA-shape decode engine driving the critical-token path end to end.

This is the caller side of the hot path: where the reference's
evaluation loop feeds recorded attention rows to ``selector.step``
(evaluation.py:90-115), a real decode step here computes attention over the
blocks the forecaster predicted at the previous step, appends the step's
compressed attention row to every (layer, head) history, and — once per
token, for all layers at once — forecasts + top-k's the blocks for the next
step ("cross-token": predictions are made one token ahead).

Everything in a step is stream-ordered with device-resident positions, so a
step is one CUDA graph replay: two graphs (plain step / calibration step,
selector.py:112-116 cadence) chosen by the host, which knows the counter.
Non-attention layers are random-init bf16 weights of the named shape run as
plain library GEMMs; both arms (sparse vs dense attention) share them.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _device as D
from . import _lib
from .attention import DecodeAttention, dense_splits, sparse_splits
from .batched import BatchedSelector
from .distributed import gather_heads_into
from .errors import ConfigError
from .predictor import PredictorWeights, init_weights, install_weights, installed_digest, weights_digest


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    hidden: int
    n_q_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float
    head_dim: int = 128
    eps: float = 1e-5

    @property
    def qkv_dim(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim

    def weight_bytes(self) -> int:
        per_layer = self.qkv_dim * self.hidden + self.hidden * self.hidden + 2 * self.ffn * self.hidden \
            + self.hidden * self.ffn + 2 * self.hidden
        return 2 * (self.n_layers * per_layer + 2 * self.vocab * self.hidden + self.hidden)

    def kv_bytes_per_token(self) -> int:
        return 2 * 2 * self.n_layers * self.n_kv_heads * self.head_dim


GEMV_RMS, GEMV_SILU, GEMV_ARGMAX = 1, 1 << 1, 2 << 1  # ap_gemv flags (include/attnpred.h)

LLAMA31_8B = ModelShape("llama-3.1-8b", 32, 4096, 32, 8, 14336, 128256, 500000.0)
LONGCHAT_7B_32K = ModelShape("longchat-7b-v1.5-32k", 32, 4096, 32, 32, 11008, 32000, 10000.0)
SHAPES = {s.name: s for s in (LLAMA31_8B, LONGCHAT_7B_32K)}


class DecodeEngine:
    """Batch decode of ``n_seq`` sequences at context ``ctx_len`` for up to ``max_new`` tokens.

    mode: "sparse" (AttentionPredictor path) or "dense" (full-attention comparator).
    group: q-heads per selection map — 1 = one history/forecast/top-k per q-head (the
    reference's per-head semantics), n_q_heads/n_kv_heads = one per KV head (GQA
    group: compressed rows are max-pooled over the group's heads, and the whole
    group shares one gathered block set).
    dense_layers: layer-skip policy (the paper keeps the first 2 layers
    dense) — layers [0, dense_layers) always run full attention and own no
    selector maps.
    fused: batch <= 4 runs the projections through ap_gemv with the neighbouring elementwise ops
    fused (RMSNorm prologues, SiLU-gate epilogue, LM head + greedy argmax) and the down projection
    as a plain ap_gemv.  fused=False keeps one library GEMM + one elementwise kernel per op.
    gemm: "auto" (library GEMM above batch 4) or "tc" (ap_gemm_tc for batch 5..16).
    """

    def __init__(self, shape: ModelShape, n_seq: int, ctx_len: int, max_new: int, *, mode: str = "sparse",
                 cfg=None, weights: PredictorWeights | None = None, group: int = 1, precision: str = "fp16x3",
                 seed: int = 0, offload_v: bool = False, head_split=None, dense_layers: int = 0,
                 fused: bool = True, gemm: str = "auto", attn_splits: tuple[int, int] | None = None,
                 layer_budgets=None, l2_warm: bool = False, time_selector: bool = False,
                 overlap_selector: int = 0):
        torch = D.torch()
        if mode not in ("sparse", "dense"):
            raise ConfigError("mode must be 'sparse' or 'dense'")
        self.full_shape = shape
        # KV-head split (distributed.HeadSplit): this rank owns kv_per_rank KV heads and their q-heads;
        # per-layer attention outputs are all-gathered before the (replicated) o_proj
        self.split = head_split if (head_split is not None and head_split.world > 1) else None
        if self.split is not None:
            from dataclasses import replace
            shape = replace(shape, n_q_heads=self.split.q_per_rank, n_kv_heads=self.split.kv_per_rank)
        self.shape, self.n_seq, self.mode, self.group = shape, n_seq, mode, group
        G = shape.n_q_heads // shape.n_kv_heads
        if G % group:
            raise ConfigError("group must divide the GQA group size")
        if not 0 <= dense_layers < shape.n_layers:
            raise ConfigError("dense_layers must be in [0, n_layers)")
        if offload_v and self.split is not None:
            raise ConfigError("V offload runs with one GPU per sequence (sequence sharding), not with a KV-head split")
        if dense_layers and offload_v:
            raise ConfigError("dense layers need their V resident: not combinable with V offload")
        self.dense_layers = dense_layers
        self.sel_layers = shape.n_layers - dense_layers  # layers that own selector maps
        self.t_max = -(-(ctx_len + max_new + 1) // 1024) * 1024
        self.ctx_len = ctx_len
        dev = D.device()
        self.dev = dev
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        bf = torch.bfloat16
        L, Hd, Hq, Hkv, F, V = shape.n_layers, shape.hidden, shape.n_q_heads, shape.n_kv_heads, shape.ffn, shape.vocab

        def rnd(*sz, std=0.02):
            return (torch.randn(*sz, generator=gen, device=dev, dtype=bf) * std)

        self.embed = rnd(V, Hd)
        self.wqkv = [rnd(self.full_shape.qkv_dim, Hd) for _ in range(L)]
        if self.split is not None:  # same random model on every rank; keep this rank's q/k/v rows
            rows = torch.tensor(self.split.qkv_rows(128), device=dev)
            self.wqkv = [w.index_select(0, rows).contiguous() for w in self.wqkv]
        Hq_full = self.full_shape.n_q_heads
        self.wo = [rnd(Hd, Hq_full * 128) for _ in range(L)]
        self.wgu = [rnd(2 * F, Hd) for _ in range(L)]
        self.wdown = [rnd(Hd, F) for _ in range(L)]
        self.ln1 = [torch.ones(Hd, dtype=bf, device=dev) for _ in range(L)]
        self.ln2 = [torch.ones(Hd, dtype=bf, device=dev) for _ in range(L)]
        self.lnf = torch.ones(Hd, dtype=bf, device=dev)
        self.lm_head = rnd(V, Hd)
        # KV cache [L][S][Hkv][t_max][128]; with offload_v, V lives in pinned host memory and a small
        # device page pool fed by the cross-token prefetch (kernel 5), K stays resident
        self.offload = offload_v
        # zeroed, not torch.empty: the kernels load whole 16-token blocks and mask positions >= t in the
        # scores, but P.V on the tensor cores would still turn a recycled NaN/inf in an unwritten V row
        # into a NaN output (0 * NaN)
        self.k_cache = torch.zeros(L, n_seq, Hkv, self.t_max, 128, dtype=bf, device=dev)
        self.v_cache = None if offload_v else torch.zeros(L, n_seq, Hkv, self.t_max, 128, dtype=bf, device=dev)
        # activations
        S = n_seq
        self.r = torch.zeros(S, Hd, dtype=bf, device=dev)
        self.r2 = torch.zeros(S, Hd, dtype=bf, device=dev)  # fused path: residual stream ping-pong
        self.fused = fused and S <= 4
        # ap_gemv ARGMAX (batch <= 4) / ap_argmax_rows (larger batches) workspace
        self.argws = torch.zeros(max(48, _lib.fn("ap_argmax_workspace_bytes")(S)), dtype=torch.uint8, device=dev)
        # gemm="tc": batch 5..16 projections on the tcgen05 skinny GEMM (ap_gemm_tc).  Default off: in the
        # batch-8 step the library GEMM measured faster (1437 vs 1358 tok/s)
        if gemm not in ("auto", "tc"):
            raise ConfigError("gemm must be 'auto' or 'tc'")
        self.tc = gemm == "tc" and not self.fused and S <= 16
        self.tcws = None
        if self.tc:
            need = max(_lib.fn("ap_gemm_tc_workspace_bytes")(n, k, S)
                       for n, k in ((shape.qkv_dim, Hd), (Hd, Hq_full * 128), (2 * F, Hd), (Hd, F), (V, Hd)))
            self.tcws = torch.zeros(need, dtype=torch.uint8, device=dev)
        self.y = torch.zeros(S, Hd, dtype=bf, device=dev)
        self.qkv = torch.zeros(S, shape.qkv_dim, dtype=bf, device=dev)
        self.q = torch.zeros(S, Hq, 128, dtype=bf, device=dev)
        self.att_out = torch.zeros(S, Hq, 128, dtype=bf, device=dev)
        self.att_full = self.att_out if self.split is None else torch.zeros(S, Hq_full, 128, dtype=bf, device=dev)
        self.o = torch.zeros(S, Hd, dtype=bf, device=dev)
        self.gu = torch.zeros(S, 2 * F, dtype=bf, device=dev)
        self.act = torch.zeros(S, F, dtype=bf, device=dev)
        self.mlp = torch.zeros(S, Hd, dtype=bf, device=dev)
        self.tok = torch.zeros(S, dtype=torch.int64, device=dev)
        self.logits = torch.zeros(S, V, dtype=bf, device=dev)
        self.seq_len = torch.full((S,), ctx_len, dtype=torch.int32, device=dev)
        self.maps_per_layer = Hq // group
        sms = _lib.fn("ap_device_sm_count")()
        nd, ns = attn_splits or (dense_splits(S * Hkv, sms, self.t_max), sparse_splits(S * self.maps_per_layer, sms))
        self.att = DecodeAttention(S, Hq, Hkv, self.t_max, n_splits_dense=nd, n_splits_sparse=ns, device=dev)
        self.sel = None
        from .selector import SelectorConfig
        self.cfg = cfg or SelectorConfig(budget=1024)
        self.cfg.validate()
        if self.cfg.block_size != 16:
            raise ConfigError("the decode attention kernels use 16-token KV blocks: block_size must be 16")
        self.pweights = weights or init_weights(0)
        self._wdigest = weights_digest(self.pweights)
        if mode == "sparse":
            install_weights(self.pweights)
            self.layer_budgets = layer_budgets
            self.sel = BatchedSelector(self.cfg, S * self.sel_layers * self.maps_per_layer, self.t_max // 16,
                                       precision=precision, device=dev, budgets=self._map_budgets())
        self.voff = None
        if offload_v:
            if mode != "sparse" or group != G:
                raise ConfigError("V offload needs the sparse path with one selection map per KV head")
            from .prefetch import OffloadedV
            self.voff = OffloadedV(L, S, Hkv, self.t_max, k_cap=max(1, self.cfg.middle_blocks),
                                   sink_tokens=self.cfg.sink_tokens, local_tokens=self.cfg.local_tokens, device=dev)
            self.pf_stream = torch.cuda.Stream(device=dev)
            self.pf_events = [torch.cuda.Event() for _ in range(L)]
        # sparse-pass L2 warm-up on a side stream (ap_attn_sparse_prefetch), resident V only.  Off by default:
        # the per-layer fork/join measured 292 vs 311 tok/s at the headline shape
        self.l2_warm = l2_warm
        self.warm_stream = torch.cuda.Stream(device=dev)
        # overlap_selector = R > 0: each layer's selector step (forecast + top-k for the next token) runs on
        # a side stream right after that layer's attention, on R SMs kept free of the GEMV / calibration
        # grids (ap_set_sm_reserve), instead of once for all layers at the end of the token
        self.overlap = int(overlap_selector)
        self.sel_stream = torch.cuda.Stream(device=dev) if self.overlap else None
        self._sub = None
        if self.overlap:
            if mode != "sparse" or n_seq != 1 or offload_v or self.split is not None:
                raise ConfigError("overlap_selector needs the resident sparse path at batch 1 (one layer's maps "
                                  "contiguous)")
            if not 0 < self.overlap < sms:
                raise ConfigError("overlap_selector must reserve between 1 and SMs-1 SMs")
        # selector timing inside the step graph: external event record nodes around ap_sel_step
        self.sel_ev = None
        if time_selector and not self.overlap:
            self.sel_ev = (torch.cuda.Event(enable_timing=True, external=True),
                           torch.cuda.Event(enable_timing=True, external=True))
        self._overlap_now = False
        self.counter = 0  # selector step counter (host mirror; all maps move in lockstep)
        self.graphs = {}
        self._fill_kv(gen)

    # ---------------------------------------------------------------- setup
    def _heads(self, full, per_rank):
        """This rank's slice of a full-model head axis (dim 1) under a KV-head split."""
        if self.split is None:
            return full
        return full[:, self.split.rank * per_rank:(self.split.rank + 1) * per_rank]

    def _fill_kv(self, gen):
        """Synthetic prefill: N(0,1) bf16 keys/values for positions [0, ctx_len) of every layer.  Under a
        KV-head split every rank draws the full model's KV and keeps its heads, so the split and the
        unsplit engine hold the same cache."""
        torch = D.torch()
        S, Hf, Hkv = self.n_seq, self.full_shape.n_kv_heads, self.shape.n_kv_heads
        full = torch.empty(S, Hf, self.ctx_len, 128, dtype=torch.bfloat16, device=self.dev)
        for l in range(self.shape.n_layers):
            self.k_cache[l, :, :, : self.ctx_len].copy_(self._heads(full.normal_(generator=gen), Hkv))
            if self.voff is None:
                self.v_cache[l, :, :, : self.ctx_len].copy_(self._heads(full.normal_(generator=gen), Hkv))
            else:  # generate on the device, park in pinned host memory
                self.voff.host_v[l, :, :, : self.ctx_len].copy_(full.normal_(generator=gen))
        if self.voff is not None:
            self.voff.init_pages(self.ctx_len)
            torch.cuda.synchronize()

    def init_history(self, seed: int = 1):
        """Prefill-side history initialisation (selector.init_state, selector.py:61-70): the
        compressed dense attention rows of the last history-1 prompt positions, computed by the
        calibration kernel over keys [0, pos] with synthetic queries."""
        if self.sel is None:
            return
        torch = D.torch()
        gen = torch.Generator(device=self.dev)
        gen.manual_seed(seed)
        H = self.cfg.history
        S, L = self.n_seq, self.shape.n_layers
        q = torch.empty_like(self.q)
        qf = torch.empty(S, self.full_shape.n_q_heads, 128, dtype=q.dtype, device=q.device)
        lens = torch.empty_like(self.seq_len)
        for i in range(H - 1):
            pos = self.ctx_len - (H - 1) + i  # prompt position; its attention row covers keys [0, pos]
            lens.fill_(pos + 1)
            q.copy_(self._heads(qf.normal_(generator=gen), self.shape.n_q_heads))  # same draws split or not
            for l in range(self.dense_layers, L):
                self.att.dense(q, self.k_cache[l], self.k_cache[l], lens, None, with_v=False, emit=True,
                               selector=self.sel, **self._map_kw(l))
        torch.cuda.synchronize()

    def _map_budgets(self):
        """Per-map token budgets of the sparse layers (budget allocation; None = cfg.budget everywhere)."""
        if getattr(self, "layer_budgets", None) is None:
            return None
        import numpy as np
        lb = np.asarray(self.layer_budgets, dtype=np.int64)
        if lb.shape != (self.sel_layers,):
            raise ConfigError(f"layer_budgets needs one budget per sparse layer ({self.sel_layers})")
        return np.tile(np.repeat(lb, self.maps_per_layer), self.n_seq)

    def _layer_sel(self, l: int):
        """Sub-descriptor of layer l's selector maps (overlap mode)."""
        if self._sub is None or self._sub[0] is not self.sel:
            mpl = self.maps_per_layer
            self._sub = (self.sel, {ll: self.sel.sub_desc((ll - self.dense_layers) * mpl, mpl)
                                    for ll in range(self.dense_layers, self.shape.n_layers)})
        return self._sub[1][l]

    def _map_kw(self, l: int) -> dict:
        """Selector map range of layer l (layers below dense_layers own none)."""
        return dict(map_base=(l - self.dense_layers) * self.maps_per_layer,
                    maps_per_seq=self.sel_layers * self.maps_per_layer, group=self.group)

    # ---------------------------------------------------------------- one step
    def _layer(self, l: int, variant: str):
        torch = D.torch()
        F_ = torch.nn.functional
        sh = self.shape
        S = self.n_seq
        s = _lib.stream_handle()
        kc = self.k_cache[l]
        vc = self.v_cache[l] if self.voff is None else self.voff.layer_view(l)
        warm = (self.l2_warm and variant in ("plain", "calib") and l >= self.dense_layers and self.voff is None)
        if warm:  # L2 warm-up of this layer's selected K/V blocks, beside the qkv projection
            main = torch.cuda.current_stream()
            self.warm_stream.wait_stream(main)
            with torch.cuda.stream(self.warm_stream):
                self.att.sparse_prefetch(self.q, kc, vc, self.seq_len, self.sel, **self._map_kw(l),
                                         stream=self.warm_stream)
        if self.fused:  # residual stream ping-pong: qkv reads r2 and writes r, gate/up the reverse
            # projection + RoPE + KV append in one pass over the qkv weights
            x_in, res, res_out = (self.r, None, None) if l == 0 else (self.mlp, self.r2, self.r)
            _lib.check(_lib.fn("ap_gemv_qkv_rope")(
                _lib.ptr(self.wqkv[l]), _lib.ptr(x_in), _lib.ptr(self.qkv), sh.n_q_heads, sh.n_kv_heads, sh.hidden,
                S, GEMV_RMS, _lib.ptr(res), _lib.ptr(res_out), _lib.ptr(self.ln1[l]), sh.eps, _lib.ptr(self.seq_len),
                _lib.ptr(self.q), _lib.ptr(kc), None if self.voff is not None else _lib.ptr(vc), self.t_max,
                sh.rope_theta, s), "ap_gemv_qkv_rope")
        else:
            if l == 0:
                _lib.check(_lib.fn("ap_rmsnorm")(_lib.ptr(self.r), None, _lib.ptr(self.ln1[0]), _lib.ptr(self.y), S,
                                                 sh.hidden, sh.eps, s))
            else:
                _lib.check(_lib.fn("ap_rmsnorm")(_lib.ptr(self.mlp), _lib.ptr(self.r), _lib.ptr(self.ln1[l]),
                                                 _lib.ptr(self.y), S, sh.hidden, sh.eps, s))
            self._mm(self.y, self.wqkv[l], self.qkv)
            _lib.check(_lib.fn("ap_rope_append")(_lib.ptr(self.qkv), S, sh.n_q_heads, sh.n_kv_heads,
                                                 _lib.ptr(self.seq_len), _lib.ptr(self.q), _lib.ptr(kc),
                                                 None if self.voff is not None else _lib.ptr(vc),
                                                 self.t_max, sh.rope_theta, s))
        if self.voff is not None:
            self.voff.append(self.qkv, sh.n_q_heads, self.seq_len, l)
            if variant in ("plain", "calib"):  # this layer's predicted V blocks must have arrived
                torch.cuda.current_stream().wait_event(self.pf_events[l])
        if warm:
            torch.cuda.current_stream().wait_stream(self.warm_stream)
        if l < self.dense_layers:
            variant = "dense"  # layer-skip policy
        kw = self._map_kw(l) if variant != "dense" else {}
        if variant == "dense":
            self.att.dense(self.q, kc, vc, self.seq_len, self.att_out, with_v=True)
        elif variant == "first":
            self.att.dense(self.q, kc, vc, self.seq_len, self.att_out, with_v=True, emit=True, selector=self.sel,
                           **kw)
        elif variant == "calib":
            self.att.sparse(self.q, kc, vc, self.seq_len, self.att_out, self.sel, emit=False, vpages=self.voff,
                            layer=l, **kw)
            self.att.dense(self.q, kc, kc, self.seq_len, None, with_v=False, emit=True, selector=self.sel, **kw)
        else:
            self.att.sparse(self.q, kc, vc, self.seq_len, self.att_out, self.sel, emit=True, vpages=self.voff,
                            layer=l, **kw)
        if self._overlap_now and l >= self.dense_layers:  # this layer's forecast + top-k beside the next GEMVs
            self.sel_stream.wait_stream(torch.cuda.current_stream())
            self.sel.step_range(self._layer_sel(l), grid_ctas=self.overlap, stream=self.sel_stream)
        if self.split is not None:  # one collective per layer: the heads' outputs over NVLink
            gather_heads_into(self.att_full, self.att_out, self.split)
        if self.fused:
            self._gemv(self.wo[l], self.att_full.view(S, -1), self.o, 0)
            self._gemv(self.wgu[l], self.o, self.act, GEMV_RMS | GEMV_SILU, residual=self.r, residual_out=self.r2,
                       ln=self.ln2[l])
        else:
            self._mm(self.att_full.view(S, -1), self.wo[l], self.o)
            _lib.check(_lib.fn("ap_rmsnorm")(_lib.ptr(self.o), _lib.ptr(self.r), _lib.ptr(self.ln2[l]),
                                             _lib.ptr(self.y), S, sh.hidden, sh.eps, s))
            self._mm(self.y, self.wgu[l], self.gu)
            _lib.check(_lib.fn("ap_silu_mul")(_lib.ptr(self.gu), _lib.ptr(self.act), S, sh.ffn, s))
        if self.fused:
            self._gemv(self.wdown[l], self.act, self.mlp, 0)
        else:
            self._mm(self.act, self.wdown[l], self.mlp)

    def _mm(self, x, W, y):
        """y = x W^T: ap_gemm_tc (tcgen05) for batch 5..16, the library GEMM above that."""
        N, K = W.shape
        if self.tc and K % 256 == 0:
            _lib.check(_lib.fn("ap_gemm_tc")(_lib.ptr(W), _lib.ptr(x), _lib.ptr(y), N, K, self.n_seq,
                                             _lib.ptr(self.tcws), self.tcws.numel(), _lib.stream_handle()),
                       "ap_gemm_tc")
        else:
            D.torch().matmul(x, W.t(), out=y)

    def _gemv(self, W, x, y, flags, residual=None, residual_out=None, ln=None, tokens=None):
        """ap_gemv: y = W x for this step's sequences with the fused prologue / epilogue in flags."""
        N, K = W.shape
        _lib.check(_lib.fn("ap_gemv")(_lib.ptr(W), _lib.ptr(x), _lib.ptr(y), N, K, self.n_seq, 2, flags,
                                      _lib.ptr(residual), _lib.ptr(residual_out), _lib.ptr(ln), self.shape.eps,
                                      _lib.ptr(self.argws) if tokens is not None else None, _lib.ptr(tokens),
                                      _lib.stream_handle()), "ap_gemv")

    def _step_body(self, variant: str, selector: bool = True):
        torch = D.torch()
        sh = self.shape
        S = self.n_seq
        s = _lib.stream_handle()
        self._overlap_now = bool(self.overlap) and selector and variant in ("plain", "calib")
        # GEMV / calibration grids leave the reserved SMs to the side-stream selector (captured with the graph)
        _lib.check(_lib.fn("ap_set_sm_reserve")(self.overlap if self._overlap_now else 0), "ap_set_sm_reserve")
        # seq_len += 1 and the embedding lookup of the previous step's token, one launch
        _lib.check(_lib.fn("ap_advance_embed")(_lib.ptr(self.seq_len), S, 1, _lib.ptr(self.embed), _lib.ptr(self.tok),
                                               _lib.ptr(self.r), sh.hidden, s), "ap_advance_embed")
        main = torch.cuda.current_stream()
        if self.voff is not None and variant in ("plain", "calib"):
            # cross-token prefetch: the blocks predicted at the end of the previous token stream in on a
            # side stream, layer by layer, while this token's earlier layers compute
            self.pf_stream.wait_stream(main)
            with torch.cuda.stream(self.pf_stream):
                for l in range(sh.n_layers):
                    self.voff.prefetch(self.sel, l, self.sel_layers * self.maps_per_layer, stream=self.pf_stream)
                    self.pf_events[l].record(self.pf_stream)
        for l in range(sh.n_layers):
            self._layer(l, variant)
        if self.voff is not None and variant in ("plain", "calib"):
            main.wait_stream(self.pf_stream)
        if self.fused:  # final norm + LM head + greedy argmax in one pass over the LM head
            self._gemv(self.lm_head, self.mlp, self.logits, GEMV_RMS | GEMV_ARGMAX, residual=self.r2, ln=self.lnf,
                       tokens=self.tok)
        else:
            _lib.check(_lib.fn("ap_rmsnorm")(_lib.ptr(self.mlp), _lib.ptr(self.r), _lib.ptr(self.lnf),
                                             _lib.ptr(self.y), S, sh.hidden, sh.eps, s))
            self._mm(self.y, self.lm_head, self.logits)
            _lib.check(_lib.fn("ap_argmax_rows")(_lib.ptr(self.logits), S, sh.vocab, _lib.ptr(self.argws),
                                                 self.argws.numel(), _lib.ptr(self.tok), s), "ap_argmax_rows")
        if self._overlap_now:
            main.wait_stream(self.sel_stream)  # every layer's selector step has finished
            _lib.check(_lib.fn("ap_set_sm_reserve")(0), "ap_set_sm_reserve")
        elif selector and self.sel is not None and variant != "dense":
            if self.sel_ev is not None:
                self.sel_ev[0].record()
            self.sel.step()  # forecast + top-k for the next token, every layer and head at once
            if self.sel_ev is not None:
                self.sel_ev[1].record()

    def selector_us(self) -> float:
        """Duration of the last step's ap_sel_step launches (time_selector engines; synchronises)."""
        self.sel_ev[1].synchronize()
        return self.sel_ev[0].elapsed_time(self.sel_ev[1]) * 1e3

    def variant_for_next(self) -> str:
        if self.mode == "dense":
            return "dense"
        if self.counter == 0:
            return "first"
        return "calib" if self.counter % self.cfg.calibration_period == 0 else "plain"

    def step(self, use_graph: bool = True):
        """One decode token for every sequence."""
        v = self.variant_for_next()
        if self.sel is not None and installed_digest() != self._wdigest:
            # another caller installed other forecaster weights (the library holds one set): put ours
            # back; the generation bump makes every map recompute its r-map rows under them
            install_weights(self.pweights)
        if use_graph and v != "first":
            g = self.graphs.get(v)
            if g is None:
                g = self._capture(v)
            g.replay()
        else:
            self._step_body(v)
        if self.sel is not None:
            self.counter += 1
        return v

    def _capture(self, variant: str):
        """Capture one decode step; positions/ring state live on the device so replays advance."""
        torch = D.torch()
        # warm the kernels (cuBLAS handles, occupancy caches) outside capture without side effects:
        # snapshot the mutable state, run once, restore.
        snap = self._snapshot()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._step_body(variant)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self._restore(snap)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step_body(variant)
        torch.cuda.synchronize()
        self._restore(snap)  # capture does not execute, but be explicit about the state contract
        self.graphs[variant] = g
        return g

    def _snapshot(self):
        torch = D.torch()
        snap = {"seq_len": self.seq_len.clone(), "tok": self.tok.clone()}
        if self.sel is not None:
            snap.update(state=self.sel.state.clone(), slot_width=self.sel.slot_width.clone(),
                        mid_blocks=self.sel.mid_blocks.clone(), mid_mask=self.sel.mid_mask.clone())
        if self.voff is not None:
            snap.update(old_n=self.voff.old_n.clone(), old_blocks=self.voff.old_blocks.clone(),
                        old_pages=self.voff.old_pages.clone(), mid_page=self.voff.mid_page.clone(),
                        bytes_copied=self.voff.bytes_copied.clone())
        del torch
        return snap

    def _restore(self, snap):
        self.seq_len.copy_(snap["seq_len"])
        self.tok.copy_(snap["tok"])
        if self.sel is not None:
            self.sel.state.copy_(snap["state"])
            self.sel.slot_width.copy_(snap["slot_width"])
            self.sel.mid_blocks.copy_(snap["mid_blocks"])
            self.sel.mid_mask.copy_(snap["mid_mask"])
        if self.voff is not None and "old_n" in snap:
            for k in ("old_n", "old_blocks", "old_pages", "mid_page", "bytes_copied"):
                getattr(self.voff, k).copy_(snap[k])

    def set_selection(self, group: int, precision: str | None = None):
        """Rebuild the selector for another selection granularity (q-heads per map) on the same
        weights / KV cache; positions reset to the prompt length, history re-initialised."""
        G = self.shape.n_q_heads // self.shape.n_kv_heads
        if G % group:
            raise ConfigError("group must divide the GQA group size")
        prec = precision or (self.sel.precision if self.sel is not None else "fp16x3")
        self.sel = None
        self.graphs.clear()
        self.group = group
        self.maps_per_layer = self.shape.n_q_heads // group
        self.sel = BatchedSelector(self.cfg, self.n_seq * self.sel_layers * self.maps_per_layer,
                                   self.t_max // 16, precision=prec, device=self.dev, budgets=self._map_budgets())
        self.mode = "sparse"
        self.counter = 0
        self.seq_len.fill_(self.ctx_len)
        self.init_history()

    def capture_all(self):
        """Capture every step variant this engine will replay (keeps capture out of timed regions)."""
        for v in (("dense",) if self.mode == "dense" else ("plain", "calib")):
            if v not in self.graphs:
                self._capture(v)

    def set_mode(self, mode: str):
        """Switch arms on the same weights / KV cache (positions reset to the prompt length)."""
        if mode == "sparse" and self.sel is None:
            raise ConfigError("engine was built without a selector")
        self.mode = mode
        self.seq_len.fill_(self.ctx_len)

    def kernels_per_step(self, variant: str) -> int:
        """Launches of libattnpred kernels in one step (the bench's gpu_launches claim)."""
        L = self.shape.n_layers
        # gemv x4 (qkv+rope fused) | rmsnorm x2, rope_append, silu_mul (+ 4 ap_gemm_tc at batch 5..16)
        per_layer = 4 if self.fused else 2 + 1 + 1 + (4 if self.tc else 0)
        att = {"dense": 1, "first": 1, "plain": 1, "calib": 2}[variant]
        if self.l2_warm and self.voff is None and variant in ("plain", "calib"):
            att += 1  # the L2 warm-up launch
        att_total = self.dense_layers + (L - self.dense_layers) * att
        sel = 3 if (self.sel is not None and variant != "dense") else 0  # forecast, top-k, guard refine
        if self.overlap and variant in ("plain", "calib"):
            sel *= self.sel_layers  # one selector step per layer
        off = 0
        if self.voff is not None:
            off = L * (1 + (1 if variant in ("plain", "calib") else 0))  # v_append (+ prefetch) per layer
        head = 1 if self.fused else (3 if self.tc else 2)  # final norm (+ LM head on ap_gemm_tc) + argmax
        return 1 + L * per_layer + att_total + head + sel + off  # advance + layers + final norm/LM head + selector

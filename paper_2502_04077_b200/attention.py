"""Decode attention over the predicted critical blocks (kernel 4a) and the dense
pass for calibration / full attention (kernel 4b).

The reference has no attention implementation for this path (SPEC.md:8 puts
GPU kernels out of scope); the math follows the exporter's toy model
(attntap/model.py:70-74), the selection structure follows selector.py:122-149
and the calibration cadence selector.py:112-116.  Both kernels append the
step's compressed row straight into a ``BatchedSelector`` ring (no t-length
row ever round-trips through HBM).

Layout: per layer K/V cache ``[n_seq, n_kv_heads, t_max, 128]`` bf16; q / out
``[n_seq, n_q_heads, 128]`` bf16.
"""

from __future__ import annotations

import ctypes

from . import _device as D
from . import _lib
from ._lib import AttnLayerDesc
from .errors import ParameterError


HEAD_DIM = 128
BLOCK = 16


def sparse_splits(n_maps: int, sm_count: int) -> int:
    """Cluster size (splits per map) of the sparse pass for n_maps maps per launch: the largest of
    8, 4, 2 that keeps one wave (n_maps x splits <= SMs; the kernel runs one CTA per SM).  Measured
    on B200 (scripts/bench_attention.py, LLaMA-3.1-8B layer at 32K): 8 maps -> 8 (9.2 us; 16: 16.8),
    32 maps -> 4 (10.4 us; 8: 11.2), 64 maps -> 2 (21.9 us; 4: 28.0, 8: 48.0)."""
    cl = 8
    while cl > 2 and n_maps * cl > sm_count:
        cl //= 2
    return cl


def dense_splits(n_units: int, sm_count: int, t_max: int) -> int:
    """Flash-decoding splits of the dense pass for n_units (sequence, KV head) pairs per launch: one
    wave of the tensor-core kernel (one CTA per SM), at most one split per 1024 positions."""
    return max(1, min(t_max // 1024, sm_count // max(1, n_units)))


class DecodeAttention:
    """Workspaces + launchers for one layer shape (reused by every layer of a model).

    n_splits_dense: flash-decoding splits of the dense pass (grid = splits x kv_heads x seqs);
    n_splits_sparse: splits of each map's selected blocks.
    """

    def __init__(self, n_seq: int, n_q_heads: int, n_kv_heads: int, t_max: int, n_splits_dense: int = 32,
                 n_splits_sparse: int = 8, device=None):
        if t_max % BLOCK:
            raise ParameterError("t_max must be a multiple of 16")
        torch = D.torch()
        dev = device or D.device()
        self.n_seq, self.n_q_heads, self.n_kv_heads, self.t_max = n_seq, n_q_heads, n_kv_heads, t_max
        self.w_max = t_max // BLOCK
        self.n_splits_dense, self.n_splits_sparse = n_splits_dense, n_splits_sparse
        ns = max(n_splits_dense, n_splits_sparse)
        self.partial = torch.empty(n_seq * n_q_heads * ns * (HEAD_DIM + 2), dtype=torch.float32, device=dev)
        self.bmax = torch.full((n_seq * n_q_heads * self.w_max,), float("-inf"), dtype=torch.float32, device=dev)
        self.lse = torch.empty(n_seq, n_q_heads, dtype=torch.float32, device=dev)
        # split-completion counters, then the calibration pass's LSE-ready epochs
        self.counters = torch.zeros(2 * n_seq * n_q_heads, dtype=torch.int32, device=dev)

    def _desc(self, q, k_cache, v_cache, seq_len, out, n_splits):
        return AttnLayerDesc(
            n_seq=self.n_seq, n_q_heads=self.n_q_heads, n_kv_heads=self.n_kv_heads, head_dim=HEAD_DIM,
            t_max=self.t_max, n_splits=n_splits, block=BLOCK, w_max=self.w_max,
            q=q.data_ptr(), k_cache=k_cache.data_ptr(), v_cache=v_cache.data_ptr(), seq_len=seq_len.data_ptr(),
            out=None if out is None else out.data_ptr(), lse=self.lse.data_ptr(), partial=self.partial.data_ptr(),
            bmax=self.bmax.data_ptr(), counters=self.counters.data_ptr(),
        )

    def dense(self, q, k_cache, v_cache, seq_len, out=None, *, with_v=True, emit=False, selector=None,
              map_base=0, maps_per_seq=None, group=1, stream=None):
        desc = self._desc(q, k_cache, v_cache, seq_len, out, self.n_splits_dense)
        sel = ctypes.byref(selector._desc) if selector is not None else None
        mps = maps_per_seq if maps_per_seq is not None else self.n_q_heads // group
        _lib.check(_lib.fn("ap_attn_dense")(ctypes.byref(desc), int(with_v), sel, map_base, mps, group, int(emit),
                                            _lib.stream_handle(stream)), "attn_dense")

    def sparse_prefetch(self, q, k_cache, v_cache, seq_len, selector, *, map_base=0, maps_per_seq=None, group=1,
                        stream=None):
        """L2 warm-up of the blocks the next sparse() of this layer gathers (side stream)."""
        desc = self._desc(q, k_cache, v_cache, seq_len, None, self.n_splits_sparse)
        mps = maps_per_seq if maps_per_seq is not None else self.n_q_heads // group
        _lib.check(_lib.fn("ap_attn_sparse_prefetch")(ctypes.byref(desc), ctypes.byref(selector._desc), map_base, mps,
                                                      group, _lib.stream_handle(stream)), "attn_sparse_prefetch")

    def sparse(self, q, k_cache, v_cache, seq_len, out, selector, *, emit=True, map_base=0, maps_per_seq=None,
               group=1, vpages=None, layer=0, stream=None):
        """v_cache is ignored (may be any tensor) when ``vpages`` (an OffloadedV) supplies paged V."""
        desc = self._desc(q, k_cache, v_cache, seq_len, out, self.n_splits_sparse)
        mps = maps_per_seq if maps_per_seq is not None else self.n_q_heads // group
        if vpages is None:
            _lib.check(_lib.fn("ap_attn_sparse")(ctypes.byref(desc), ctypes.byref(selector._desc), map_base, mps,
                                                 group, int(emit), _lib.stream_handle(stream)), "attn_sparse")
        else:
            _lib.check(_lib.fn("ap_attn_sparse_paged")(ctypes.byref(desc), ctypes.byref(selector._desc), map_base,
                                                       mps, group, int(emit), ctypes.byref(vpages._desc), layer,
                                                       _lib.stream_handle(stream)), "attn_sparse_paged")

"""Cross-token prefetch of predicted critical V blocks from host memory (kernel 5).

The reference models this schedule only (prefetchsim._schedule_point,
prefetchsim.py:126-151: transfer = fixed + B·bytes·L/bw and
total = max(compute, predict + transfer)); here the transfer is real.

``OffloadedV`` owns the pinned host V of every (layer, sequence, KV head)
"vmap" and the small device page pool that holds what attention needs:
sink blocks and the recent ring (device-resident, written by ``append``) and
``k_cap`` middle pages filled by ``prefetch(layer)`` after the selector has
predicted the next step's middle blocks.  K stays resident on the device —
the periodic calibration pass (selector.py:112-116) reads all of K.
"""

from __future__ import annotations

import ctypes

from . import _device as D
from . import _lib
from .errors import ConfigError

BLOCK = 16
HEAD_DIM = 128


class OffloadedV:
    def __init__(self, n_layers: int, n_seq: int, n_kv_heads: int, t_max: int, k_cap: int, sink_tokens: int = 64,
                 recent_pages: int = 8, local_tokens: int = 64, device=None):
        if k_cap > 128:
            raise ConfigError("k_cap above 128 middle blocks is not supported")
        if recent_pages * BLOCK < local_tokens + BLOCK:
            raise ConfigError("recent ring must cover the local window plus the block being filled")
        torch = D.torch()
        dev = device or D.device()
        self.L, self.S, self.Hkv, self.t_max, self.k_cap = n_layers, n_seq, n_kv_heads, t_max, k_cap
        self.sink_pages = -(-sink_tokens // BLOCK)
        self.recent_pages = recent_pages
        self.n_vmaps = n_layers * n_seq * n_kv_heads
        n_pages = self.sink_pages + recent_pages + k_cap
        bf = torch.bfloat16
        # pinned (hence mapped under UVA) host V, layout [L][S][Hkv][t_max][128]
        self.host_v = torch.zeros(n_layers, n_seq, n_kv_heads, t_max, HEAD_DIM, dtype=bf, pin_memory=True)
        self.pages = torch.zeros(self.n_vmaps, n_pages, BLOCK, HEAD_DIM, dtype=bf, device=dev)
        i32 = torch.int32
        self.mid_page = torch.zeros(self.n_vmaps, k_cap, dtype=i32, device=dev)
        self.old_blocks = torch.full((self.n_vmaps, k_cap), -1, dtype=i32, device=dev)
        self.old_pages = torch.zeros(self.n_vmaps, k_cap, dtype=i32, device=dev)
        self.old_n = torch.zeros(self.n_vmaps, dtype=i32, device=dev)
        self.bytes_copied = torch.zeros(1, dtype=torch.int64, device=dev)
        self._desc = _lib.VPages(
            k_cap=k_cap, sink_pages=self.sink_pages, recent_pages=recent_pages, pad_=0, host_t_max=t_max,
            pages=self.pages.data_ptr(), host_v=self.host_v.data_ptr(), mid_page=self.mid_page.data_ptr(),
            old_blocks=self.old_blocks.data_ptr(), old_pages=self.old_pages.data_ptr(),
            old_n=self.old_n.data_ptr(), bytes_copied=self.bytes_copied.data_ptr(),
        )

    def layer_view(self, layer: int):
        """Host V of one layer as [S][Hkv][t_max][128] (device-addressable: pinned + UVA)."""
        return self.host_v[layer]

    def init_pages(self, t: int, stream=None):
        """Sink pages + recent ring of every vmap from host V after a prompt of length t."""
        _lib.check(_lib.fn("ap_v_pages_init")(ctypes.byref(self._desc), int(t), self.n_vmaps,
                                              _lib.stream_handle(stream)), "v_pages_init")

    def append(self, qkv, n_q_heads: int, seq_len, layer: int, stream=None):
        _lib.check(_lib.fn("ap_v_append")(qkv.data_ptr(), n_q_heads, self.Hkv, seq_len.data_ptr(),
                                          ctypes.byref(self._desc), layer, self.S, _lib.stream_handle(stream)),
                   "v_append")

    def prefetch(self, selector, layer: int, maps_per_seq: int, stream=None):
        _lib.check(_lib.fn("ap_prefetch")(ctypes.byref(selector._desc), ctypes.byref(self._desc), layer, self.S,
                                          self.Hkv, maps_per_seq, _lib.stream_handle(stream)), "prefetch")

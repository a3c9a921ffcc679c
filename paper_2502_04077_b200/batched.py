"""Device-resident selector over many maps at once.

One *map* is one (sequence, layer, q-head) attention history.  The
``BatchedSelector`` owns, in HBM, every map's compressed-history ring
(H x w_max fp32), its per-row forecaster contributions (the r-map, same
shape), per-slot widths, step state, last forecast and middle-block
selection; a decode step is three stream-ordered launches with no host
round trip (push → predict/top-k → counter), so whole decode steps capture
into one CUDA graph.

Semantics per map are those of ``attncast.selector.init_state`` / ``step``
(selector.py:61-154) and of the evaluation loop's observed-row feedback
(evaluation.py:90-115); see ``paper_2502_04077_b200.selector`` for the
per-head reference-compatible wrapper.
"""

from __future__ import annotations

import ctypes

import os

import numpy as np

from . import _device as D
from . import _lib
from .errors import ParameterError

PUSH_PREFILL, PUSH_DENSE, PUSH_OBSERVED = 0, 1, 2

_STATE_DTYPE = np.dtype([
    ("n_pushed", "<i8"), ("r_pushed", "<i8"), ("row_len", "<i8"), ("counter", "<i8"), ("mid_clip", "<i8"),
    ("width", "<i4"), ("r_width", "<i4"), ("n_mid", "<i4"), ("r_wgen", "<i4"),
    ("tie_n", "<i4"), ("prev_kth", "<u4"),
])
assert _STATE_DTYPE.itemsize == _lib.MAP_STATE_BYTES


class BatchedSelector:
    """n_maps independent selectors sharing one forecaster weight set.

    cfg: a SelectorConfig-like object (budget, block_size, history,
    calibration_period, sink_tokens, local_tokens, update_interval).
    w_max: the largest compressed width any map will reach (ceil(t_max/b)).
    """

    def __init__(self, cfg, n_maps: int, w_max: int, precision: str = "fp16x3", device=None, tie_guard: bool = True,
                 budgets=None, fused: bool | None = None):
        cfg.validate()
        if n_maps < 1 or w_max < 1:
            raise ParameterError("n_maps and w_max must be >= 1")
        if precision not in _lib.PREC:
            raise ParameterError(f"unknown precision {precision!r}")
        torch = D.torch()
        dev = device or D.device()
        w_max = -(-int(w_max) // 4) * 4  # 16-byte ring rows (bulk-copy alignment)
        self.cfg = cfg
        self.n_maps, self.w_max, self.precision = int(n_maps), int(w_max), precision
        H = cfg.history
        self.k_mid = cfg.middle_blocks
        words = (w_max + 31) // 32
        f32, i32 = torch.float32, torch.int32
        self.ring = torch.zeros(n_maps, H, w_max, dtype=f32, device=dev)
        self.rmap = torch.zeros(n_maps, H, w_max, dtype=f32, device=dev)
        self.rsum = torch.zeros(n_maps, w_max, dtype=torch.float64, device=dev)
        self.slot_width = torch.zeros(n_maps, H, dtype=i32, device=dev)
        self.slot_xmax = torch.zeros(n_maps, H, dtype=f32, device=dev)
        self.state = torch.zeros(n_maps * _STATE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.scores = torch.zeros(n_maps, w_max, dtype=f32, device=dev)
        self.mid_blocks = torch.zeros(n_maps, max(self.k_mid, 1), dtype=i32, device=dev)
        self.mid_mask = torch.zeros(n_maps, words, dtype=i32, device=dev)
        self.status = torch.zeros(1, dtype=i32, device=dev)
        # budget allocation: per-map token budgets (selector.py:47-50 evaluated per map); cfg.budget is the
        # largest, it sets the pitch of mid_blocks
        self.k_map = None
        if budgets is not None:
            from .budget import middle_blocks_per_map
            km = middle_blocks_per_map(budgets, n_maps, cfg)
            self.k_map = torch.from_numpy(km).to(dev)
        # exact-boundary guard workspace (csrc/tieguard.cuh): near-tie candidates of the top-k boundary
        # are re-scored in fp64 so the block ids equal the float64 reference's
        self.tie_ws = None
        if tie_guard:
            nb = int(_lib.fn("ap_sel_tie_ws_bytes")(self.n_maps))
            self.tie_ws = torch.zeros(-(-nb // 4), dtype=i32, device=dev)
        # fused=True: forecast + top-k (+ guard) as one launch (ap_selector.fused_done: per-map chunk
        # counters).  Off by default — it measured slower than the two launches;
        # ATTNPRED_FUSED_SELECT=1 turns it on for every selector.
        if fused is None:
            fused = os.environ.get("ATTNPRED_FUSED_SELECT") == "1"
        self.fused_done = torch.zeros(n_maps, dtype=i32, device=dev) if fused else None
        self._desc = _lib.Selector(
            n_maps=n_maps, history=H, block=cfg.block_size, w_max=w_max, k_mid=self.k_mid,
            sink=cfg.sink_tokens, local=cfg.local_tokens, calib_period=cfg.calibration_period,
            update_interval=cfg.update_interval, pad_=0,
            ring=self.ring.data_ptr(), rmap=self.rmap.data_ptr(), rsum=self.rsum.data_ptr(),
            slot_width=self.slot_width.data_ptr(), slot_xmax=self.slot_xmax.data_ptr(),
            state=self.state.data_ptr(), scores=self.scores.data_ptr(), mid_blocks=self.mid_blocks.data_ptr(),
            mid_mask=self.mid_mask.data_ptr(), status=self.status.data_ptr(),
            tie_ws=None if self.tie_ws is None else self.tie_ws.data_ptr(),
            k_map=None if self.k_map is None else self.k_map.data_ptr(),
            fused_done=None if self.fused_done is None else self.fused_done.data_ptr(),
        )
        self.reset()

    # ------------------------------------------------------------ launches
    def _call(self, name, *args, stream=None):
        _lib.check(_lib.fn(name)(ctypes.byref(self._desc), *args, _lib.stream_handle(stream)), name)

    def reset(self, stream=None) -> None:
        """selector.init_state with no prefill rows, for every map."""
        self._call("ap_sel_reset", stream=stream)

    def push_rows(self, rows, t: int, mode: int = PUSH_DENSE, stream=None) -> None:
        """Compress one t-length row per map (rows[i] at row i of a 2-D float32/float64 tensor) and
        append it to map i's history (selector.py:112-120; mode semantics in include/attnpred.h)."""
        torch = D.torch()
        if rows.dim() != 2 or rows.shape[0] != self.n_maps or rows.shape[1] < t or rows.stride(1) != 1:
            raise ParameterError("rows must be a [n_maps, >=t] tensor with unit column stride")
        if -(-t // self.cfg.block_size) > self.w_max:
            raise ParameterError("row longer than w_max * block_size")
        dt = {torch.float32: _lib.AP_F32, torch.float64: _lib.AP_F64}.get(rows.dtype)
        if dt is None:
            raise ParameterError("rows must be float32 or float64")
        self._call("ap_sel_push_rows", _lib.ptr(rows), dt, rows.stride(0), int(t), int(mode), stream=stream)

    def push_compressed(self, comp, t: int, prefill: bool = False, stream=None) -> None:
        """Append already-compressed rows (fp32 [n_maps, >=ceil(t/b)]) — the attention kernels' output."""
        self._call("ap_sel_push_compressed", _lib.ptr(comp), comp.stride(0), int(t), int(prefill), stream=stream)

    def step(self, stream=None) -> None:
        """selector.py:122-154 for every map: forecast + mask + top-k on update steps, then counter += 1."""
        self._call("ap_sel_step", _lib.PREC[self.precision], stream=stream)

    def sub_desc(self, begin: int, count: int):
        """A descriptor of maps [begin, begin + count) (same buffers, offset pointers; shared status and
        guard workspace), for stepping one layer's maps on their own."""
        if not (0 <= begin and count >= 1 and begin + count <= self.n_maps):
            raise ParameterError("map range out of bounds")
        d = _lib.Selector.from_buffer_copy(self._desc)
        H, wm = self.cfg.history, self.w_max
        words = (wm + 31) // 32
        d.n_maps = count
        for name, per_map in (("ring", 4 * H * wm), ("rmap", 4 * H * wm), ("rsum", 8 * wm), ("slot_width", 4 * H),
                              ("slot_xmax", 4 * H), ("state", _STATE_DTYPE.itemsize), ("scores", 4 * wm),
                              ("mid_blocks", 4 * max(self.k_mid, 1)), ("mid_mask", 4 * words), ("k_map", 4),
                              ("fused_done", 4)):
            base = getattr(d, name)
            if base:
                setattr(d, name, base + begin * per_map)
        return d

    def step_range(self, desc, grid_ctas: int = 0, stream=None) -> None:
        """ap_sel_step_grid on a sub_desc(): the forecaster's persistent grid capped at grid_ctas CTAs."""
        _lib.check(_lib.fn("ap_sel_step_grid")(ctypes.byref(desc), _lib.PREC[self.precision], int(grid_ctas),
                                               _lib.stream_handle(stream)), "ap_sel_step_grid")

    # ------------------------------------------------------------ readback
    def states(self) -> np.ndarray:
        return self.state.cpu().numpy().view(_STATE_DTYPE)

    def middle(self, i: int) -> list[int]:
        st = self.states()[i]
        return self.mid_blocks[i, : int(st["n_mid"])].cpu().tolist()

    def tie_stats(self) -> dict:
        """Cumulative exact-boundary guard counters: maps whose boundary was ambiguous and re-scored in
        fp64 (``refined_maps``, ``candidates``) and maps whose ambiguity exceeded the guard's capacity
        (``overflow``: those kept the fp32 order)."""
        if self.tie_ws is None:
            return {"enabled": False}
        out = (ctypes.c_int32 * 3)()
        D.torch().cuda.synchronize()
        _lib.check(_lib.fn("ap_sel_tie_stats")(_lib.ptr(self.tie_ws), ctypes.cast(out, ctypes.c_void_p)), "tie")
        return {"enabled": True, "overflow": int(out[0]), "refined_maps": int(out[1]), "candidates": int(out[2])}

    def check_status(self) -> None:
        D.sync_and_check(self.status, "selector")

    def history_rows(self, i: int) -> list[np.ndarray]:
        """Map i's stored window, oldest first, each row at its own width (host copy)."""
        st = self.states()[i]
        H = self.cfg.history
        n = int(st["n_pushed"])
        ring = self.ring[i].cpu().numpy()
        widths = self.slot_width[i].cpu().numpy()
        out = []
        for k in range(max(0, n - H), n):
            s = k % H
            out.append(ring[s, : widths[s]].astype(np.float64))
        return out


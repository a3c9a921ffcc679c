"""Budgeted critical-token selection (kernel 3 + orchestration of kernel 1/2).

Drop-in for ``attncast.selector`` (reference: pkg/src/attncast/selector.py):
``SelectorConfig``, ``SelectorState``, ``init_state``, ``topk``, ``step``
with the reference's signatures, return types (``set[int]``) and exceptions.
Each ``SelectorState`` is backed by a one-map ``BatchedSelector`` whose
history ring, incremental forecaster r-map and top-k live on the GPU; the
host only builds the returned Python sets.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .batched import PUSH_OBSERVED, PUSH_PREFILL, BatchedSelector
from .compress import expand_indices
from .errors import ConfigError, ParameterError, StateError
from .predictor import PredictorWeights, default_precision, install_weights

__all__ = ["SelectorConfig", "SelectorState", "init_state", "topk", "step"]


@dataclass
class SelectorConfig:
    """selector.py:23-50."""

    budget: int
    block_size: int = 16
    history: int = 64
    calibration_period: int = 5
    sink_tokens: int = 64
    local_tokens: int = 64
    update_interval: int = 1

    def validate(self) -> None:
        if self.budget < self.sink_tokens + self.local_tokens:
            raise ConfigError("budget must cover the sink and local allocations")
        if self.block_size < 1:
            raise ConfigError("block_size must be >= 1")
        if self.calibration_period < 1:
            raise ConfigError("calibration_period must be >= 1")
        if self.history < 1:
            raise ConfigError("history must be >= 1")
        if self.update_interval < 1:
            raise ConfigError("update_interval must be >= 1")
        if self.sink_tokens < 0 or self.local_tokens < 0:
            raise ConfigError("sink/local allocations must be non-negative")

    @property
    def middle_blocks(self) -> int:
        return (self.budget - self.sink_tokens - self.local_tokens) // self.block_size


@dataclass
class SelectorState:
    """selector.py:53-58.  ``compressed_history`` and ``step_counter`` are read back from the device."""

    middle_tokens: set = field(default_factory=set)
    selection: set = field(default_factory=set)
    _dev: BatchedSelector | None = field(default=None, repr=False)
    _cfg_key: tuple | None = field(default=None, repr=False)
    _pending: list = field(default_factory=list, repr=False)  # prefill rows before the device exists
    _counter: int = 0

    @property
    def step_counter(self) -> int:
        return self._counter

    @property
    def compressed_history(self) -> list:
        if self._dev is None:
            return [np.asarray(r, dtype=np.float64) for r in self._pending]
        return self._dev.history_rows(0)


def _cfg_key(cfg: SelectorConfig) -> tuple:
    return (cfg.budget, cfg.block_size, cfg.history, cfg.calibration_period, cfg.sink_tokens,
            cfg.local_tokens, cfg.update_interval)


def _ensure_device(state: SelectorState, cfg: SelectorConfig, width: int) -> BatchedSelector:
    """(Re)build the one-map device selector when the config changes or the row outgrows w_max."""
    key = _cfg_key(cfg)
    dev = state._dev
    if dev is not None and state._cfg_key == key and width <= dev.w_max:
        return dev
    w_max = max(256, 1 << max(0, int(np.ceil(np.log2(max(width, 1))))))
    rows = state.compressed_history if dev is not None or state._pending else []
    meta = dev.states()[0].copy() if dev is not None else None
    mid = dev.middle(0) if dev is not None else []
    new = BatchedSelector(cfg, 1, w_max, precision=default_precision())
    # replay the stored window as prefill pushes (exact: the rows are already compressed)
    for r in rows[-cfg.history:]:
        comp = D.to_device(np.asarray(r, dtype=np.float32)[None, :])
        new.push_compressed(comp, int(r.size) * cfg.block_size, prefill=True)
    if meta is not None:
        st = new.states()
        st[0]["counter"] = meta["counter"]
        st[0]["row_len"] = meta["row_len"]
        st[0]["mid_clip"] = meta["mid_clip"]
        st[0]["n_mid"] = len(mid)
        torch = D.torch()
        new.state.copy_(torch.from_numpy(st.view(np.uint8).copy()))
        if mid:
            new.mid_blocks[0, : len(mid)] = torch.tensor(mid, dtype=torch.int32)
            mask = np.zeros(new.mid_mask.shape[1] * 32, dtype=bool)
            mask[mid] = True
            new.mid_mask[0] = torch.from_numpy(np.packbits(mask, bitorder="little").view(np.int32).copy())
    state._dev, state._cfg_key = new, key
    return new


def init_state(config: SelectorConfig, prefill_rows=()) -> SelectorState:
    """selector.py:61-70 — seed with the newest history-1 compressed prompt rows."""
    config.validate()
    from .compress import max_pool

    state = SelectorState()
    keep = config.history - 1
    rows = list(prefill_rows)
    rows = rows[-keep:] if keep > 0 else []
    if not rows:
        return state
    t_max = max(np.asarray(r).size for r in rows)
    dev = _ensure_device(state, config, -(-t_max // config.block_size))
    torch = D.torch()
    for r in rows:
        arr = np.asarray(r)
        if arr.dtype != np.float32:
            arr = np.asarray(r, dtype=np.float64)
        if arr.ndim != 1 or arr.size == 0:
            max_pool(arr, config.block_size)  # raises ParameterError exactly like the reference
        x = D.to_device(arr[None, :])
        dev.push_rows(x, arr.size, mode=PUSH_PREFILL)
    del torch
    return state


def topk(values, k: int) -> set[int]:
    """selector.py:73-81 — indices of the k largest values; ties break toward the lower index."""
    v = np.asarray(values, dtype=np.float64)
    if k > v.size:
        raise ParameterError(f"k={k} exceeds vector length {v.size}")
    if k <= 0:
        return set()
    torch = D.torch()
    x = D.to_device(v.ravel())
    ids = torch.empty(k, dtype=torch.int32, device=x.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=x.device)
    status = D.new_status()
    _lib.check(_lib.fn("ap_topk")(_lib.ptr(x), _lib.AP_F64, 1, v.size, v.size, k, _lib.ptr(ids), k,
                                  _lib.ptr(cnt), _lib.ptr(status), _lib.stream_handle()), "topk")
    n = int(cnt.item())
    return set(ids[:n].cpu().tolist())


def _covering_blocks(start: int, stop: int, block_size: int) -> range:
    """selector.py:84-88."""
    if stop <= start:
        return range(0)
    return range(start // block_size, -(-stop // block_size))


def step(state: SelectorState, config: SelectorConfig, weights: PredictorWeights | None, observed_row,
         full_row=None) -> tuple[SelectorState, set[int]]:
    """selector.py:91-154 — advance one decode step; returns the selection over [0, t+1)."""
    config.validate()
    observed = np.asarray(observed_row, dtype=np.float64)
    t = observed.size
    if t < 1:
        raise StateError("observed row must be non-empty")
    calibrate = state._counter % config.calibration_period == 0
    source = np.asarray(full_row if (calibrate and full_row is not None) else observed, dtype=np.float64)
    if source.size != t:
        raise StateError("dense row length must match the observed row")
    k_blocks = config.middle_blocks
    update = state._counter % config.update_interval == 0
    if update and k_blocks > 0 and weights is None:
        raise StateError("middle budget requires forecaster weights")
    width = -(-t // config.block_size)
    dev = _ensure_device(state, config, width)
    if update and k_blocks > 0:
        install_weights(weights)
    x = D.to_device(source[None, :])
    dev.push_rows(x, t, mode=PUSH_OBSERVED)
    dev.step()
    dev.check_status()
    state._counter += 1
    if update:
        state.middle_tokens = expand_indices(dev.middle(0), config.block_size, t) if k_blocks > 0 else set()
    next_len = t + 1
    sink = set(range(min(config.sink_tokens, next_len)))
    local = set(range(max(0, next_len - config.local_tokens), next_len))
    selection = sink | local | state.middle_tokens
    if len(selection) > config.budget:
        raise StateError("selection exceeded the budget")
    state.selection = selection
    return state, selection

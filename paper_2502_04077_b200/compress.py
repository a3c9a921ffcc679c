"""Block max-pool compression and block-index expansion (kernel 1).

Drop-in for ``attncast.compress`` (reference: pkg/src/attncast/compress.py):
same names, signatures, return types and exceptions; the arithmetic runs in
``ap_max_pool`` / ``ap_expand_indices`` (csrc/compress.cu).  Max is exact, so
results are bit-identical to the reference for float32/float64 rows.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .errors import ParameterError

__all__ = ["CompressedRow", "max_pool", "expand_indices"]


@dataclass(frozen=True)
class CompressedRow:
    """compress.py:18-25 — block maxima (float64), the block size and the row length."""

    values: np.ndarray
    block_size: int
    original_len: int

    def __len__(self) -> int:
        return len(self.values)


def max_pool(row, block_size: int) -> CompressedRow:
    """compress.py:28-40: zero-pad ``row`` to a block multiple, per-block maxima."""
    if block_size < 1:
        raise ParameterError("block size must be >= 1")
    arr = np.asarray(row)
    if arr.dtype != np.float32:
        arr = np.asarray(row, dtype=np.float64)
    if arr.ndim != 1 or arr.size == 0:
        raise ParameterError("row must be a non-empty 1-D vector")
    t = arr.size
    W = -(-t // block_size)
    torch = D.torch()
    x = D.to_device(arr)
    out = torch.empty(W, dtype=torch.float64, device=x.device)
    in_dt = _lib.AP_F32 if arr.dtype == np.float32 else _lib.AP_F64
    _lib.check(_lib.fn("ap_max_pool")(_lib.ptr(x), in_dt, 1, t, t, block_size, _lib.ptr(out), _lib.AP_F64, W,
                                      _lib.stream_handle()), "max_pool")
    return CompressedRow(values=out.cpu().numpy(), block_size=block_size, original_len=t)


def expand_indices(block_indices, block_size: int, original_len: int) -> set[int]:
    """compress.py:43-57: union of the blocks' token ranges, clipped to the row."""
    if block_size < 1:
        raise ParameterError("block size must be >= 1")
    if original_len < 1:
        raise ParameterError("original length must be >= 1")
    blocks = np.fromiter((int(b) for b in block_indices), dtype=np.int64)
    n_blocks = -(-original_len // block_size)
    if blocks.size == 0:
        return set()
    if blocks.min() < -(2 ** 31) or blocks.max() >= 2 ** 31:
        bad = int(blocks.max() if blocks.max() >= n_blocks else blocks.min())
        raise ParameterError(f"block index {bad} out of range [0, {n_blocks})")
    torch = D.torch()
    dev = D.device()
    b_dev = D.to_device(blocks.astype(np.int32))
    tokens = torch.empty(blocks.size * block_size, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int32, device=dev)
    status = D.new_status()
    _lib.check(_lib.fn("ap_expand_indices")(_lib.ptr(b_dev), int(blocks.size), block_size, original_len,
                                            _lib.ptr(tokens), _lib.ptr(count), _lib.ptr(status),
                                            _lib.stream_handle()), "expand_indices")
    if int(status.item()) != 0:
        bad = next(int(b) for b in blocks if not 0 <= b < n_blocks)
        raise ParameterError(f"block index {bad} out of range [0, {n_blocks})")
    n = int(count.item())
    return set(tokens[:n].cpu().tolist())

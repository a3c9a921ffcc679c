"""Device plumbing shared by the reference-compatible shim modules.

PyTorch is used only for device memory, streams and host<->device copies;
every computation goes through libattnpred.so.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from . import errors as E


def torch():
    import torch as _t
    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise E.DeviceError("no CUDA device: the B200 kernels are the only implementation of this path")
    _lib.load()
    return t.device("cuda", t.cuda.current_device())


def to_device(arr: np.ndarray, dtype=None):
    t = torch()
    a = np.ascontiguousarray(arr if dtype is None else np.asarray(arr, dtype=dtype))
    return t.from_numpy(a).to(device(), non_blocking=False)


def new_status():
    t = torch()
    return t.zeros(1, dtype=t.int32, device=device())


def sync_and_check(status, what: str) -> None:
    """Synchronise the current stream and raise if a kernel set the status word."""
    code = int(status.item())
    _lib.raise_device_status(code, what)

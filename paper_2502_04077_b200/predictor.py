"""The shared conv forecaster ℱ (kernel 2) — inference half.

Drop-in for the inference half of ``attncast.predictor`` (reference:
pkg/src/attncast/predictor.py:1-216,424-444): ``PredictorWeights``,
``init_weights``, ``AttentionHistory``, ``stack_history``, ``forward``,
``save_weights`` / ``load_weights`` with the APW1 format.  ``forward`` runs
``ap_predict_forward`` (csrc/predictor.cu) — a tcgen05 implicit-GEMM conv in
the default ``fp16x3`` precision.  Training (backward / Adam,
predictor.py:219-416) is out of scope for this B200 path.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .errors import FormatError, NumericError, ParameterError

__all__ = [
    "CONV1_OUT", "CONV2_OUT", "KERNEL", "PARAM_COUNT", "WEIGHTS_MAGIC", "PredictorWeights", "init_weights",
    "AttentionHistory", "stack_history", "forward", "save_weights", "load_weights", "install_weights",
    "default_precision",
]

CONV1_OUT = 16
CONV2_OUT = 32
KERNEL = 3
PARAM_COUNT = CONV1_OUT * (KERNEL * KERNEL + 1) + CONV2_OUT * (CONV1_OUT * KERNEL * KERNEL + 1) + CONV2_OUT + 1
WEIGHTS_MAGIC = b"APW1"

_SHAPES = (
    (CONV1_OUT, 1, KERNEL, KERNEL),
    (CONV1_OUT,),
    (CONV2_OUT, CONV1_OUT, KERNEL, KERNEL),
    (CONV2_OUT,),
    (CONV2_OUT,),
    (),
)


def default_precision() -> str:
    """Predictor arithmetic: ATTNPRED_PRECISION in {fp16x3 (default), fp32, fp16}."""
    p = os.environ.get("ATTNPRED_PRECISION", "fp16x3")
    if p not in _lib.PREC:
        raise ParameterError(f"unknown precision {p!r}")
    return p


@dataclass
class PredictorWeights:
    """predictor.py:45-98 — the 4833 parameters, float64 on the host."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w3: np.ndarray
    b3: np.ndarray

    def param_count(self) -> int:
        return sum(int(np.asarray(t).size) for t in self.tensors())

    def tensors(self) -> tuple:
        return (self.w1, self.b1, self.w2, self.b2, self.w3, self.b3)

    def copy(self) -> "PredictorWeights":
        return PredictorWeights(*(np.array(t, copy=True) for t in self.tensors()))

    def flat(self) -> np.ndarray:
        return np.concatenate([np.asarray(t, dtype=np.float64).ravel() for t in self.tensors()])

    def validate(self) -> None:
        for t, shp in zip(self.tensors(), _SHAPES):
            t = np.asarray(t)
            if t.shape != shp:
                raise ParameterError(f"weight tensor shape {t.shape} != {shp}")
            if not np.all(np.isfinite(t)):
                raise NumericError("weights contain non-finite values")

    @classmethod
    def from_flat(cls, flat) -> "PredictorWeights":
        flat = np.asarray(flat)
        if flat.size != PARAM_COUNT:
            raise ParameterError(f"expected {PARAM_COUNT} parameters, got {flat.size}")
        parts, at = [], 0
        for shp in _SHAPES:
            n = int(np.prod(shp)) if shp else 1
            parts.append(np.array(flat.ravel()[at:at + n], dtype=np.float64).reshape(shp))
            at += n
        return cls(*parts)


def init_weights(rng_seed: int = 0) -> PredictorWeights:
    """predictor.py:101-116 — He-normal w1/w2/w3 from SeedSequence(seed, spawn_key=(0xE11,)), zero biases.

    Same generator and draw order as the reference, so seeds give identical weights.
    """
    rng = np.random.default_rng(np.random.SeedSequence(rng_seed, spawn_key=(0xE11,)))
    w1 = rng.standard_normal(_SHAPES[0]) * np.sqrt(2.0 / (KERNEL * KERNEL))
    w2 = rng.standard_normal(_SHAPES[2]) * np.sqrt(2.0 / (CONV1_OUT * KERNEL * KERNEL))
    w3 = rng.standard_normal(CONV2_OUT) * np.sqrt(2.0 / CONV2_OUT)
    return PredictorWeights(w1=w1, b1=np.zeros(CONV1_OUT), w2=w2, b2=np.zeros(CONV2_OUT), w3=w3, b3=np.zeros(()))


@dataclass
class AttentionHistory:
    """predictor.py:119-136 — H x W grid of compressed rows, oldest first."""

    grid: np.ndarray

    def __post_init__(self):
        self.grid = np.asarray(self.grid, dtype=np.float64)
        if self.grid.ndim != 2:
            raise ParameterError("history grid must be 2-D (steps x blocks)")

    @property
    def depth(self) -> int:
        return self.grid.shape[0]

    @property
    def width(self) -> int:
        return self.grid.shape[1]


def stack_history(rows, depth: int, width: int) -> AttentionHistory:
    """predictor.py:145-157 — newest ``depth`` rows, zero rows on top, right zero pad.

    (Host-side argument marshalling for the reference-compatible ``forward``;
    the device selector keeps the same window in its ring without stacking.)
    """
    grid = np.zeros((depth, width), dtype=np.float64)
    keep = list(rows)[-depth:] if depth > 0 else []
    top = depth - len(keep)
    for i, r in enumerate(keep):
        r = np.asarray(r, dtype=np.float64)
        n = min(width, r.size)
        grid[top + i, :n] = r[:n]
    return AttentionHistory(grid=grid)


# ----------------------------------------------------------------- device side
_installed = {"digest": None, "tensor": None}


def install_weights(weights: PredictorWeights, stream=None):
    """Upload the weights as 4833 fp32 and install them (ap_set_weights) if they changed.

    Returns the device tensor.  The native library keeps one installed weight
    set, as the reference shares one forecaster across every (layer, head).
    """
    weights.validate()
    flat32 = weights.flat().astype(np.float32)
    digest = hashlib.sha1(flat32.tobytes()).hexdigest()
    if _installed["digest"] != digest:
        t = D.to_device(flat32)
        _lib.check(_lib.fn("ap_set_weights")(_lib.ptr(t), _lib.stream_handle(stream)), "set_weights")
        _installed.update(digest=digest, tensor=t)
    return _installed["tensor"]


def forward(weights: PredictorWeights, history: AttentionHistory, precision: str | None = None) -> np.ndarray:
    """predictor.py:211-216: predict the next compressed row (length = history width)."""
    weights.validate()
    grid = np.asarray(history.grid, dtype=np.float64)
    if not np.all(np.isfinite(grid)):
        raise NumericError("history contains non-finite values")
    H, W = grid.shape
    torch = D.torch()
    install_weights(weights)
    pitch = -(-W // 4) * 4  # 16-byte rows for the kernel's bulk copies
    padded = np.zeros((H, pitch), dtype=np.float32)
    padded[:, :W] = grid
    g = D.to_device(padded)
    out = torch.empty(W, dtype=torch.float32, device=g.device)
    scratch = torch.empty(H * pitch, dtype=torch.float32, device=g.device)
    status = D.new_status()
    prec = _lib.PREC[precision or default_precision()]
    _lib.check(_lib.fn("ap_predict_forward")(_lib.ptr(g), 1, H, W, pitch, H * pitch, _lib.ptr(out), W,
                                             _lib.ptr(scratch), prec, _lib.ptr(status), _lib.stream_handle()),
               "forward")
    D.sync_and_check(status, "forward")
    return out.cpu().numpy().astype(np.float64)


def save_weights(weights: PredictorWeights, path) -> None:
    """predictor.py:424-431 — b"APW1" + the tensors in order as little-endian float32."""
    weights.validate()
    with open(path, "wb") as fh:
        fh.write(WEIGHTS_MAGIC)
        fh.write(weights.flat().astype("<f4").tobytes())


def load_weights(path) -> PredictorWeights:
    """predictor.py:434-444 — FormatError on bad magic, truncation or trailing bytes."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != WEIGHTS_MAGIC:
            raise FormatError(f"bad weights magic {magic!r}")
        body = fh.read(4 * PARAM_COUNT)
        flat = np.frombuffer(body, dtype="<f4")
        if flat.size != PARAM_COUNT:
            raise FormatError("weights file truncated")
        if fh.read(1):
            raise FormatError("trailing bytes after weight tensors")
    return PredictorWeights.from_flat(flat.astype(np.float64))

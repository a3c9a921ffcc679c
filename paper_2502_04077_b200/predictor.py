"""The shared conv forecaster ℱ (kernel 2) — inference half.

Drop-in for the inference half of ``attncast.predictor`` (reference:
pkg/src/attncast/predictor.py:1-216,424-444): ``PredictorWeights``,
``init_weights``, ``AttentionHistory``, ``stack_history``, ``forward``,
``save_weights`` / ``load_weights`` with the APW1 format.  ``forward`` runs
``ap_predict_forward`` (csrc/predictor.cu) — a tcgen05 implicit-GEMM conv in
the default ``fp16x3`` precision.  Training — ``backward`` / ``train``
(predictor.py:219-251,327-409) — runs ``ap_train_backward`` / ``ap_adam_step``
(csrc/train.cu).
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .errors import FormatError, NumericError, ParameterError, TrainingError

__all__ = [
    "CONV1_OUT", "CONV2_OUT", "KERNEL", "PARAM_COUNT", "WEIGHTS_MAGIC", "PredictorWeights", "init_weights",
    "AttentionHistory", "stack_history", "forward", "save_weights", "load_weights", "install_weights",
    "default_precision", "forward_precision", "TrainSample", "EpochMetrics", "backward", "train",
    "build_dataset",
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


def weights_digest(weights: PredictorWeights) -> str:
    """Identity of a weight set as the device sees it (its fp32 image)."""
    return hashlib.sha1(weights.flat().astype(np.float32).tobytes()).hexdigest()


def installed_digest() -> str | None:
    return _installed["digest"]


def install_weights(weights: PredictorWeights, stream=None):
    """Upload the weights as 4833 fp32 and install them (ap_set_weights) if they changed.

    Returns the device tensor.  The native library keeps one installed weight
    set, as the reference shares one forecaster across every (layer, head).
    Installing a different set bumps the device weight generation, so every
    selector map recomputes its forecaster rows in full at its next update.
    """
    weights.validate()
    flat32 = weights.flat().astype(np.float32)
    digest = hashlib.sha1(flat32.tobytes()).hexdigest()
    if _installed["digest"] != digest:
        t = D.to_device(flat32)
        _lib.check(_lib.fn("ap_set_weights")(_lib.ptr(t), _lib.stream_handle(stream)), "set_weights")
        _installed.update(digest=digest, tensor=t)
    return _installed["tensor"]


def forward_precision() -> str:
    """Arithmetic of the reference-compatible ``forward``: ATTNPRED_FORWARD_PRECISION in {fp64 (default:
    the reference's own type, ap_predict_forward_f64), fp16x3, fp32, fp16 (the selector's kernels)}."""
    p = os.environ.get("ATTNPRED_FORWARD_PRECISION", "fp64")
    if p != "fp64" and p not in _lib.PREC:
        raise ParameterError(f"unknown precision {p!r}")
    return p


def _forward_f64(weights: PredictorWeights, grid: np.ndarray) -> np.ndarray:
    torch = D.torch()
    H, W = grid.shape
    g = D.to_device(np.ascontiguousarray(grid, dtype=np.float64))
    w = D.to_device(weights.flat().astype(np.float64))
    out = torch.empty(W, dtype=torch.float64, device=g.device)
    ws = torch.empty(int(_lib.fn("ap_forward_f64_workspace_bytes")(1, H, W)), dtype=torch.uint8, device=g.device)
    _lib.check(_lib.fn("ap_predict_forward_f64")(_lib.ptr(g), 1, H, W, _lib.ptr(w), _lib.ptr(out), W, _lib.ptr(ws),
                                                 ws.numel(), _lib.stream_handle()), "forward")
    return out.cpu().numpy()


def forward(weights: PredictorWeights, history: AttentionHistory, precision: str | None = None) -> np.ndarray:
    """predictor.py:211-216: predict the next compressed row (length = history width).

    Default arithmetic is fp64 (``forward_precision``), like the reference; the selector's
    tensor-core precisions (fp16x3 / fp32 / fp16) are available by name."""
    weights.validate()
    grid = np.asarray(history.grid, dtype=np.float64)
    if not np.all(np.isfinite(grid)):
        raise NumericError("history contains non-finite values")
    precision = precision or forward_precision()
    if precision == "fp64":
        return _forward_f64(weights, grid)
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
    prec = _lib.PREC[precision]
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


# ----------------------------------------------------------------- training (device)
@dataclass
class TrainSample:
    """predictor.py:139-142 — one (history window, next compressed row) pair."""

    input: AttentionHistory
    target: np.ndarray  # length W


@dataclass
class EpochMetrics:
    """predictor.py:316-320."""

    epoch: int
    train_mse: float
    holdout_accuracy: float


class _GradBatcher:
    """Samples resident on the device, grouped by (H, W); one ap_train_backward per shape group."""

    def __init__(self, grids, targets):
        torch = D.torch()
        self.shape_of = [tuple(np.asarray(g).shape) for g in grids]
        self.groups = {}
        for i, s in enumerate(self.shape_of):
            self.groups.setdefault(s, []).append(i)
        self.slot = {}
        self.g_dev, self.t_dev = {}, {}
        for s, ids in self.groups.items():
            for j, i in enumerate(ids):
                self.slot[i] = j
            self.g_dev[s] = D.to_device(np.stack([np.asarray(grids[i], np.float64) for i in ids]))
            self.t_dev[s] = D.to_device(np.stack([np.asarray(targets[i], np.float64) for i in ids]))
        dev = D.device()
        self.grads = torch.zeros(PARAM_COUNT, dtype=torch.float64, device=dev)
        self.ws = torch.empty(0, dtype=torch.uint8, device=dev)
        self.torch = torch

    def grad_sum(self, w_dev, ids, loss_out):
        """grads = sum over ids of each sample's gradient; loss_out += sum of losses (device)."""
        torch = self.torch
        self.grads.zero_()
        by_shape = {}
        for i in ids:
            by_shape.setdefault(self.shape_of[i], []).append(self.slot[i])
        for (H, W), slots in by_shape.items():
            idx = torch.tensor(slots, dtype=torch.long, device=self.grads.device)
            g = self.g_dev[(H, W)].index_select(0, idx).contiguous()
            t = self.t_dev[(H, W)].index_select(0, idx).contiguous()
            need = int(_lib.fn("ap_train_workspace_bytes")(len(slots), H, W))
            if self.ws.numel() < need:
                self.ws = torch.empty(need, dtype=torch.uint8, device=self.grads.device)
            _lib.check(_lib.fn("ap_train_backward")(_lib.ptr(g), _lib.ptr(t), len(slots), H, W, _lib.ptr(w_dev),
                                                    _lib.ptr(self.grads), _lib.ptr(loss_out), _lib.ptr(self.ws),
                                                    self.ws.numel(), _lib.stream_handle()), "backward")
        return self.grads


def backward(weights: PredictorWeights, history: AttentionHistory, target) -> tuple[float, PredictorWeights]:
    """predictor.py:219-251 — loss and exact gradients of mean((forward - target)^2), on the device
    (ap_train_backward: fp64 arithmetic like the reference, deterministic reductions)."""
    weights.validate()
    grid = np.asarray(history.grid, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    H, W = grid.shape
    if target.shape != (W,):
        raise ParameterError(f"target must have shape ({W},)")
    torch = D.torch()
    b = _GradBatcher([grid], [target])
    w_dev = D.to_device(weights.flat().astype(np.float64))
    loss = torch.zeros(1, dtype=torch.float64, device=w_dev.device)
    g = b.grad_sum(w_dev, [0], loss)
    return float(loss.item()), PredictorWeights.from_flat(g.cpu().numpy())


def _train_schedule(n: int, epochs: int, rng_seed: int, batch_size: int, holdout_fraction: float):
    """The sample order of predictor.train (predictor.py:345-371): holdout ids, train ids and each
    epoch's minibatches, drawn from the same seeded generator in the same order."""
    rng = np.random.default_rng(np.random.SeedSequence(rng_seed, spawn_key=(0x7241,)))
    order = rng.permutation(n)
    n_hold = int(round(holdout_fraction * n)) if n >= 10 else 0
    hold = [int(i) for i in order[:n_hold]]
    tr = [int(i) for i in order[n_hold:]]
    sched = []
    for _ in range(epochs):
        perm = rng.permutation(len(tr))
        sched.append([[tr[i] for i in perm[s:s + batch_size]] for s in range(0, len(perm), batch_size)])
    return hold, tr, sched


def _block_recovery_accuracy(preds, targets) -> float:
    """predictor.py:297-313 on device predictions (host ranking of W values per sample)."""
    if not targets:
        return 0.0
    ratios = []
    for pred, tgt in zip(preds, targets):
        w = pred.size
        k = max(1, int(round(0.1 * w)))
        op = np.lexsort((np.arange(w), -pred))[:k]
        ot = np.lexsort((np.arange(w), -tgt))[:k]
        best = float(tgt[ot].sum())
        ratios.append(1.0 if best <= 0 else float(tgt[op].sum()) / best)
    return 100.0 * float(np.mean(ratios))


def _forward_many(w_flat: np.ndarray, grids) -> list[np.ndarray]:
    """fp64 ap_predict_forward_f64 of many histories (the reference's arithmetic), one launch per
    (H, W) group."""
    torch = D.torch()
    out = [None] * len(grids)
    groups = {}
    for i, g in enumerate(grids):
        groups.setdefault(np.asarray(g).shape, []).append(i)
    w = D.to_device(np.asarray(w_flat, np.float64))
    for (H, W), ids in groups.items():
        g = D.to_device(np.stack([np.asarray(grids[i], np.float64) for i in ids]))
        o = torch.empty((len(ids), W), dtype=torch.float64, device=g.device)
        ws = torch.empty(int(_lib.fn("ap_forward_f64_workspace_bytes")(len(ids), H, W)), dtype=torch.uint8,
                         device=g.device)
        _lib.check(_lib.fn("ap_predict_forward_f64")(_lib.ptr(g), len(ids), H, W, _lib.ptr(w), _lib.ptr(o), W,
                                                     _lib.ptr(ws), ws.numel(), _lib.stream_handle()), "forward")
        o = o.cpu().numpy()
        for j, i in enumerate(ids):
            out[i] = o[j]
    return out


def train(samples, epochs: int = 30, learning_rate: float = 1e-3, rng_seed: int = 0, batch_size: int = 32,
          holdout_fraction: float = 0.1) -> tuple[PredictorWeights, list[EpochMetrics]]:
    """predictor.py:327-409 — minibatch Adam on the MSE loss, on the device.

    Same holdout split, permutations, per-batch gradient sums and Adam arithmetic as the
    reference (ap_train_backward + ap_adam_step; weights and moments stay on the device in
    fp64); returns the checkpoint with the best held-out block-recovery accuracy.  Per-batch
    losses are checked at the end of each epoch (TrainingError names the epoch).
    """
    if not samples:
        raise ParameterError("cannot train on an empty sample set")
    if epochs < 1:
        raise ParameterError("epochs must be >= 1")
    torch = D.torch()
    grids = [np.asarray(s.input.grid, np.float64) for s in samples]
    targets = [np.asarray(s.target, np.float64) for s in samples]
    for g, t in zip(grids, targets):
        if t.shape != (g.shape[1],):
            raise ParameterError(f"target must have shape ({g.shape[1]},)")
    hold, tr, sched = _train_schedule(len(samples), epochs, rng_seed, batch_size, holdout_fraction)
    batcher = _GradBatcher(grids, targets)
    w = D.to_device(init_weights(rng_seed).flat().astype(np.float64))
    m, v = torch.zeros_like(w), torch.zeros_like(w)
    best, best_acc, metrics, step = w.clone(), -np.inf, [], 0
    ev = hold if hold else tr
    for epoch, batches in enumerate(sched, start=1):
        losses = torch.zeros(len(batches), dtype=torch.float64, device=w.device)
        for b, ids in enumerate(batches):
            g = batcher.grad_sum(w, ids, losses[b:b + 1])
            step += 1
            _lib.check(_lib.fn("ap_adam_step")(_lib.ptr(w), _lib.ptr(m), _lib.ptr(v), _lib.ptr(g), PARAM_COUNT,
                                               float(len(ids)), learning_rate, 0.9, 0.999, 1e-8, step,
                                               _lib.stream_handle()), "adam")
        sizes = np.array([len(ids) for ids in batches], np.float64)
        batch_loss = losses.cpu().numpy() / sizes
        if not np.all(np.isfinite(batch_loss)):
            raise TrainingError(f"loss became non-finite in epoch {epoch}", epoch=epoch)
        w_host = w.cpu().numpy()
        if not np.all(np.isfinite(w_host)):
            raise TrainingError(f"weights became non-finite in epoch {epoch}", epoch=epoch)
        acc = _block_recovery_accuracy(_forward_many(w_host, [grids[i] for i in ev]), [targets[i] for i in ev])
        metrics.append(EpochMetrics(epoch=epoch, train_mse=float(np.mean(batch_loss)), holdout_accuracy=acc))
        if acc > best_acc:
            best_acc, best = acc, w.clone()
    return PredictorWeights.from_flat(best.cpu().numpy()), metrics


def build_dataset(trace, history_steps: int, block_size: int, sample_ratio: float, rng_seed: int = 0,
                  max_step: int | None = None) -> list[TrainSample]:
    """predictor.py:254-300 — (history window, next compressed row) pairs from an attention trace.

    Same candidate enumeration, seeded subsample, window and target definitions as the
    reference.  The compression runs on the device: per (layer, head), every stored row (zero
    padded to the trace's final length; zero padding is what max_pool pads with, so the leading
    blocks are unchanged) and every truncated next-step target row go through ONE ``ap_max_pool``.
    """
    if history_steps < 1:
        raise ParameterError("history_steps must be >= 1")
    if block_size < 1:
        raise ParameterError("block size must be >= 1")
    if not (0.0 < sample_ratio <= 1.0):
        raise ParameterError("sample_ratio must lie in (0, 1]")
    h = trace.header
    if h.num_decode_steps < 1:
        raise ParameterError("trace has no decode steps to learn from")
    last_t = h.num_decode_steps - 1 if max_step is None else min(max_step - 1, h.num_decode_steps - 1)
    candidates = [(layer, head, t) for layer in range(h.num_layers) for head in range(h.num_heads)
                  for t in range(1, last_t + 1)]
    rng = np.random.default_rng(np.random.SeedSequence(rng_seed, spawn_key=(0xDA7A,)))
    keep = max(1, int(round(sample_ratio * len(candidates))))
    chosen = sorted(rng.choice(len(candidates), size=min(keep, len(candidates)), replace=False).tolist())
    if not chosen:
        return []
    torch = D.torch()
    steps = list(h.steps)
    L = h.total_len
    W_all = -(-L // block_size)
    n_rows = len(steps)
    compressed = {}

    def pool(layer, head):
        if (layer, head) not in compressed:
            # rows [0, n_rows): stored rows; rows [n_rows, 2 n_rows): row s truncated to row_len(s - 1)
            buf = np.zeros((2 * n_rows, L), np.float32)
            for k, s in enumerate(steps):
                r = np.asarray(trace.row(layer, head, s), np.float32)
                buf[k, :r.size] = r
                if s >= 1:
                    n = min(h.row_len(s - 1), r.size)
                    buf[n_rows + k, :n] = r[:n]
            x = D.to_device(buf)
            out = torch.empty((2 * n_rows, W_all), dtype=torch.float64, device=x.device)
            _lib.check(_lib.fn("ap_max_pool")(_lib.ptr(x), _lib.AP_F32, 2 * n_rows, L, L, block_size, _lib.ptr(out),
                                              _lib.AP_F64, W_all, _lib.stream_handle()), "max_pool")
            compressed[(layer, head)] = out.cpu().numpy()
        return compressed[(layer, head)]

    samples = []
    for idx in chosen:
        layer, head, t = candidates[idx]
        cm = pool(layer, head)
        width = -(-h.row_len(t) // block_size)
        window = [cm[s - h.first_step_offset, :-(-h.row_len(s) // block_size)]
                  for s in range(t - history_steps + 1, t + 1) if s >= h.first_step_offset]
        history = stack_history(window, history_steps, width)
        target = cm[n_rows + (t + 1 - h.first_step_offset), :width].copy()
        samples.append(TrainSample(input=history, target=target))
    return samples

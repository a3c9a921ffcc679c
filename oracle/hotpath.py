"""CPU ORACLE — test infrastructure only, never a product path.

A float64 numpy restatement of the reference's decode-time critical-token
path (the `north_star` of BASELINE.json).  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import this module, and only as the checker or as the
timed CPU baseline.  The CUDA product path (``paper_2502_04077_b200``) never
imports it and fails loudly when its native library is missing.

Parity pinning: every function below is checked against golden vectors that
``tests/golden/gen_golden.py`` produced by importing the REAL reference
package (``/root/reference/pkg/src/attncast``) in the build container —
see ``tests/test_oracle_golden.py``.  Exact equality is required for the
integer / max / ordering functions and |Δ| ≤ 1e-12·scale for ``forward``
(the reference sums through OpenBLAS dgemm; this restatement sums tap by tap,
so the two agree to float64 rounding, not bit-for-bit).

Reference anchors (paths relative to /root/reference/pkg/src/attncast):
  max_pool          compress.py:28-40
  expand_indices    compress.py:43-57
  stack_history     predictor.py:145-157
  forward           predictor.py:185-216  (_forward_cached + forward)
  backward          predictor.py:219-251
  adam / train      predictor.py:327-391  (minibatch gradient sum, Adam update)
  build_dataset     predictor.py:254-300
  init_weights      predictor.py:101-116
  APW1 I/O          predictor.py:424-444
  topk              selector.py:73-81
  covering_blocks   selector.py:84-88
  SelectorConfig    selector.py:23-50
  init_state        selector.py:61-70
  step              selector.py:91-154
  predictor loop    evaluation.py:90-115 (_iter_selections, method="predictor")
  recovery_rate     evaluation.py:70-81
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

C1, C2, KS = 16, 32, 3
PARAM_COUNT = C1 * (KS * KS + 1) + C2 * (C1 * KS * KS + 1) + (C2 + 1)  # 4833
_SHAPES = [(C1, 1, KS, KS), (C1,), (C2, C1, KS, KS), (C2,), (C2,), ()]


class OracleError(Exception):
    """Raised where the reference raises; ``kind`` names the reference class."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------------------
# compress.py
# ---------------------------------------------------------------------------

def max_pool(row, b: int) -> np.ndarray:
    """compress.py:28-40 — zero-pad to a multiple of b, per-block max (float64)."""
    if b < 1:
        raise OracleError("ParameterError", "block size must be >= 1")
    x = np.asarray(row, dtype=np.float64)
    if x.ndim != 1 or x.size == 0:
        raise OracleError("ParameterError", "row must be a non-empty 1-D vector")
    n = (x.size + b - 1) // b
    out = np.empty(n, dtype=np.float64)
    full = x.size // b
    if full:
        out[:full] = x[: full * b].reshape(full, b).max(axis=1)
    if full < n:  # tail block: real values plus zero padding
        out[full] = max(float(x[full * b:].max()), 0.0)
    return out


def expand_indices(blocks, b: int, t: int) -> set[int]:
    """compress.py:43-57 — token ranges of blocks, clipped to [0, t)."""
    if b < 1:
        raise OracleError("ParameterError", "block size must be >= 1")
    if t < 1:
        raise OracleError("ParameterError", "original length must be >= 1")
    n = (t + b - 1) // b
    out: set[int] = set()
    for j in blocks:
        j = int(j)
        if not 0 <= j < n:
            raise OracleError("ParameterError", f"block index {j} out of range [0, {n})")
        out.update(range(j * b, min(j * b + b, t)))
    return out


# ---------------------------------------------------------------------------
# predictor.py (inference half)
# ---------------------------------------------------------------------------

@dataclass
class Weights:
    """w1 (16,1,3,3) b1 (16) w2 (32,16,3,3) b2 (32) w3 (32) b3 () — predictor.py:45-98."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w3: np.ndarray
    b3: np.ndarray

    def tensors(self):
        return (self.w1, self.b1, self.w2, self.b2, self.w3, self.b3)

    def flat(self) -> np.ndarray:
        return np.concatenate([np.asarray(t, np.float64).ravel() for t in self.tensors()])

    @classmethod
    def from_flat(cls, flat) -> "Weights":
        flat = np.asarray(flat, dtype=np.float64).ravel()
        if flat.size != PARAM_COUNT:
            raise OracleError("ParameterError", f"expected {PARAM_COUNT} parameters")
        parts, at = [], 0
        for shp in _SHAPES:
            n = int(np.prod(shp)) if shp else 1
            parts.append(flat[at:at + n].reshape(shp).copy())
            at += n
        return cls(*parts)


def init_weights(seed: int = 0) -> Weights:
    """predictor.py:101-116 — He-normal draws in w1, w2, w3 order; zero biases."""
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(0xE11,)))
    w1 = rng.standard_normal((C1, 1, KS, KS)) * np.sqrt(2.0 / 9.0)
    w2 = rng.standard_normal((C2, C1, KS, KS)) * np.sqrt(2.0 / (C1 * 9.0))
    w3 = rng.standard_normal(C2) * np.sqrt(2.0 / C2)
    return Weights(w1, np.zeros(C1), w2, np.zeros(C2), w3, np.zeros(()))


def save_apw1(w: Weights, path) -> None:
    """predictor.py:424-431 — b"APW1" then 4833 little-endian float32."""
    with open(path, "wb") as fh:
        fh.write(b"APW1")
        fh.write(w.flat().astype("<f4").tobytes())


def load_apw1(path) -> Weights:
    """predictor.py:434-444."""
    raw = open(path, "rb").read()
    if raw[:4] != b"APW1":
        raise OracleError("FormatError", "bad weights magic")
    body = raw[4:]
    if len(body) < 4 * PARAM_COUNT:
        raise OracleError("FormatError", "weights file truncated")
    if len(body) > 4 * PARAM_COUNT:
        raise OracleError("FormatError", "trailing bytes after weight tensors")
    return Weights.from_flat(np.frombuffer(body, dtype="<f4").astype(np.float64))


def stack_history(rows, depth: int, width: int) -> np.ndarray:
    """predictor.py:145-157 — newest ``depth`` rows, zero rows on top, right zero pad."""
    keep = list(rows)[-depth:] if depth > 0 else []
    grid = np.zeros((depth, width), dtype=np.float64)
    top = depth - len(keep)
    for i, r in enumerate(keep):
        r = np.asarray(r, dtype=np.float64)
        n = min(width, r.size)
        grid[top + i, :n] = r[:n]
    return grid


def _conv3x3(x: np.ndarray, w: np.ndarray, bias: np.ndarray) -> np.ndarray:
    """Zero-padded 3x3 cross-correlation: x (Cin,H,W), w (Cout,Cin,3,3) -> (Cout,H,W).

    Summed tap by tap (the reference lowers to im2col + dgemm, predictor.py:165-199).
    """
    cin, h, wd = x.shape
    xp = np.zeros((cin, h + 2, wd + 2), dtype=np.float64)
    xp[:, 1:-1, 1:-1] = x
    out = np.broadcast_to(bias[:, None, None], (w.shape[0], h, wd)).copy()
    for di in range(KS):
        for dj in range(KS):
            patch = xp[:, di:di + h, dj:dj + wd].reshape(cin, h * wd)
            out += (w[:, :, di, dj] @ patch).reshape(w.shape[0], h, wd)
    return out


def forward_parts(w: Weights, grid) -> dict:
    """predictor.py:185-208 — returns the intermediate maps as well as ``out``."""
    g = np.asarray(grid, dtype=np.float64)
    a1 = np.maximum(_conv3x3(g[None], np.asarray(w.w1, np.float64), np.asarray(w.b1, np.float64)), 0.0)
    s2 = _conv3x3(a1, np.asarray(w.w2, np.float64), np.asarray(w.b2, np.float64))
    a2 = np.maximum(s2, 0.0)
    z = a2.mean(axis=1)
    out = np.asarray(w.w3, np.float64) @ z + float(np.asarray(w.b3))
    return {"a1": a1, "s2": s2, "z": z, "out": out}


def forward(w: Weights, grid) -> np.ndarray:
    """predictor.py:211-216 — finite checks then the forward pass; output length W."""
    for t in w.tensors():
        if not np.all(np.isfinite(t)):
            raise OracleError("NumericError", "weights contain non-finite values")
    g = np.asarray(grid, dtype=np.float64)
    if g.ndim != 2:
        raise OracleError("ParameterError", "history grid must be 2-D")
    if not np.all(np.isfinite(g)):
        raise OracleError("NumericError", "history contains non-finite values")
    return forward_parts(w, g)["out"]


def row_contributions(w: Weights, grid) -> np.ndarray:
    """r[i, w] = sum_c w3[c] * relu(s2[c, i, w]); forward = b3 + mean_i r[i].

    This is the per-history-row form the incremental device predictor keeps
    (DESIGN.md §Predictor); it is algebraically identical to predictor.py:196-199.
    """
    p = forward_parts(w, grid)
    return np.einsum("c,chw->hw", np.asarray(w.w3, np.float64), np.maximum(p["s2"], 0.0))


def _corr3x3(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """g[ca, cb, di, dj] = sum_p a[ca, p] * b_pad[cb, p + (di-1, dj-1)] — the weight
    gradient d_s @ cols.T of predictor.py:241,247 without forming im2col."""
    cb, h, wd = b.shape
    bp = np.zeros((cb, h + 2, wd + 2), dtype=np.float64)
    bp[:, 1:-1, 1:-1] = b
    af = a.reshape(a.shape[0], h * wd)
    g = np.zeros((a.shape[0], cb, KS, KS))
    for di in range(KS):
        for dj in range(KS):
            g[:, :, di, dj] = af @ bp[:, di:di + h, dj:dj + wd].reshape(cb, h * wd).T
    return g


def backward(w: Weights, grid, target):
    """predictor.py:219-251 — loss = mean((out - target)^2) and its exact gradients.

    The input gradient of conv2 (col2im of W2^T d_s2, predictor.py:242-243) is restated
    as the 3x3 correlation of d_s2 with the flipped, channel-swapped kernel.
    Returns (loss, Weights of gradients).
    """
    g = np.asarray(grid, dtype=np.float64)
    tgt = np.asarray(target, dtype=np.float64)
    h, wd = g.shape
    if tgt.shape != (wd,):
        raise OracleError("ParameterError", f"target must have shape ({wd},)")
    p = forward_parts(w, g)
    resid = p["out"] - tgt
    loss = float(np.mean(resid ** 2))
    d_out = 2.0 * resid / wd
    d_w3 = p["z"] @ d_out
    d_b3 = np.array(d_out.sum())
    d_s2 = np.where(p["s2"] > 0, (np.asarray(w.w3, np.float64)[:, None] * d_out[None, :] / h)[:, None, :], 0.0)
    d_w2 = _corr3x3(d_s2, p["a1"])
    d_b2 = d_s2.sum(axis=(1, 2))
    w2t = np.asarray(w.w2, np.float64).transpose(1, 0, 2, 3)[:, :, ::-1, ::-1]
    d_a1 = _conv3x3(d_s2, w2t, np.zeros(C1))
    d_s1 = np.where(p["a1"] > 0, d_a1, 0.0)
    d_w1 = _corr3x3(d_s1, g[None])
    d_b1 = d_s1.sum(axis=(1, 2))
    return loss, Weights(d_w1, d_b1, d_w2, d_b2, d_w3, d_b3)


def adam_update(wf, m, v, grad_sum, batch: int, step: int, lr: float = 1e-3,
                beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> None:
    """predictor.py:381-391 on flat float64 arrays, in place (same operation order)."""
    corr1 = 1.0 - beta1 ** step
    corr2 = 1.0 - beta2 ** step
    g = grad_sum / batch
    m *= beta1
    m += (1 - beta1) * g
    v *= beta2
    v += (1 - beta2) * g * g
    wf -= lr * (m / corr1) / (np.sqrt(v / corr2) + eps)


def build_dataset(trace, history_steps: int, block_size: int, sample_ratio: float, rng_seed: int = 0,
                  max_step=None):
    """predictor.py:254-300 — [(grid, target)] from any object with the reference trace API
    (``header.num_layers/num_heads/num_decode_steps/first_step_offset/row_len``, ``row``)."""
    h = trace.header
    last_t = h.num_decode_steps - 1 if max_step is None else min(max_step - 1, h.num_decode_steps - 1)
    cands = [(la, he, t) for la in range(h.num_layers) for he in range(h.num_heads) for t in range(1, last_t + 1)]
    rng = np.random.default_rng(np.random.SeedSequence(rng_seed, spawn_key=(0xDA7A,)))
    keep = max(1, int(round(sample_ratio * len(cands))))
    chosen = sorted(rng.choice(len(cands), size=min(keep, len(cands)), replace=False).tolist())
    out = []
    for idx in chosen:
        la, he, t = cands[idx]
        t_len = h.row_len(t)
        width = -(-t_len // block_size)
        rows = [max_pool(trace.row(la, he, s), block_size) for s in range(t - history_steps + 1, t + 1)
                if s >= h.first_step_offset]
        out.append((stack_history(rows, history_steps, width),
                    max_pool(np.asarray(trace.row(la, he, t + 1))[:t_len], block_size)))
    return out


def block_recovery_accuracy(preds, targets) -> float:
    """predictor.py:297-313 on precomputed predictions: mean recovered target mass of the
    top round(0.1 W) predicted blocks relative to the best, in percent."""
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


def train_schedule(n_samples: int, epochs: int, rng_seed: int, batch_size: int, holdout_fraction: float = 0.1):
    """The sample order of predictor.train (predictor.py:345-371): (holdout ids, train ids,
    [per epoch: list of minibatches of sample ids]).  Shared by the oracle and device trainers."""
    rng = np.random.default_rng(np.random.SeedSequence(rng_seed, spawn_key=(0x7241,)))
    order = rng.permutation(n_samples)
    n_hold = int(round(holdout_fraction * n_samples)) if n_samples >= 10 else 0
    hold = [int(i) for i in order[:n_hold]]
    tr = [int(i) for i in order[n_hold:]]
    epochs_b = []
    for _ in range(epochs):
        perm = rng.permutation(len(tr))
        epochs_b.append([[tr[i] for i in perm[s:s + batch_size]] for s in range(0, len(perm), batch_size)])
    return hold, tr, epochs_b


def train(grids, targets, epochs: int = 30, lr: float = 1e-3, rng_seed: int = 0, batch_size: int = 32,
          holdout_fraction: float = 0.1):
    """predictor.py:327-409 — minibatch Adam on the MSE loss; returns (best weights, [(mse, acc)])."""
    hold, tr, sched = train_schedule(len(grids), epochs, rng_seed, batch_size, holdout_fraction)
    w = init_weights(rng_seed)
    wf = w.flat()
    m, v = np.zeros_like(wf), np.zeros_like(wf)
    step, best, best_acc, metrics = 0, wf.copy(), -np.inf, []
    for batches in sched:
        losses = []
        for batch in batches:
            cur = Weights.from_flat(wf)
            acc, bl = np.zeros_like(wf), 0.0
            for i in batch:
                loss, g = backward(cur, grids[i], targets[i])
                bl += loss
                acc += g.flat()
            losses.append(bl / len(batch))
            step += 1
            adam_update(wf, m, v, acc, len(batch), step, lr)
        ev = hold if hold else tr
        cur = Weights.from_flat(wf)
        a = block_recovery_accuracy([forward_parts(cur, grids[i])["out"] for i in ev], [targets[i] for i in ev])
        metrics.append((float(np.mean(losses)), a))
        if a > best_acc:
            best_acc, best = a, wf.copy()
    return Weights.from_flat(best), metrics


# ---------------------------------------------------------------------------
# selector.py
# ---------------------------------------------------------------------------

def topk(values, k: int) -> set[int]:
    """selector.py:73-81 — k largest, descending, ties to the lower index.

    A stable argsort of the negated values is the same total order as the
    reference's lexsort((arange, -values)); -0.0 and +0.0 compare equal.
    """
    v = np.asarray(values, dtype=np.float64)
    if k > v.size:
        raise OracleError("ParameterError", f"k={k} exceeds vector length {v.size}")
    if k <= 0:
        return set()
    order = np.argsort(-v, kind="stable")
    return {int(i) for i in order[:k]}


def covering_blocks(start: int, stop: int, b: int) -> range:
    """selector.py:84-88."""
    if stop <= start:
        return range(0)
    return range(start // b, (stop + b - 1) // b)


@dataclass
class Config:
    """selector.py:23-50 (field names identical to SelectorConfig)."""

    budget: int
    block_size: int = 16
    history: int = 64
    calibration_period: int = 5
    sink_tokens: int = 64
    local_tokens: int = 64
    update_interval: int = 1

    def validate(self) -> None:
        if self.budget < self.sink_tokens + self.local_tokens:
            raise OracleError("ConfigError", "budget must cover the sink and local allocations")
        for name in ("block_size", "calibration_period", "history", "update_interval"):
            if getattr(self, name) < 1:
                raise OracleError("ConfigError", f"{name} must be >= 1")
        if self.sink_tokens < 0 or self.local_tokens < 0:
            raise OracleError("ConfigError", "sink/local allocations must be non-negative")

    @property
    def middle_blocks(self) -> int:
        return (self.budget - self.sink_tokens - self.local_tokens) // self.block_size


@dataclass
class State:
    """selector.py:53-58."""

    history: list = field(default_factory=list)
    counter: int = 0
    middle: set = field(default_factory=set)
    selection: set = field(default_factory=set)
    last_scores: np.ndarray | None = None  # oracle-only: predicted scores of the last update
    last_blocks: list | None = None        # oracle-only: chosen block ids of the last update


def init_state(cfg: Config, prefill_rows=()) -> State:
    """selector.py:61-70 — keep the newest history-1 compressed prefill rows."""
    cfg.validate()
    st = State()
    rows = [max_pool(r, cfg.block_size) for r in prefill_rows]
    keep = cfg.history - 1
    st.history = rows[-keep:] if keep > 0 else []
    return st


def masked_scores(cfg: Config, predicted: np.ndarray, t: int) -> np.ndarray:
    """selector.py:134-142 — sink/local covering blocks below the width go to -inf."""
    m = np.array(predicted, dtype=np.float64, copy=True)
    width = m.size
    nxt = t + 1
    b = cfg.block_size
    for j in covering_blocks(0, min(cfg.sink_tokens, nxt), b):
        if j < width:
            m[j] = -np.inf
    for j in covering_blocks(max(0, nxt - cfg.local_tokens), nxt, b):
        if j < width:
            m[j] = -np.inf
    return m


def step(st: State, cfg: Config, w: Weights | None, observed, full_row=None):
    """selector.py:91-154 — one decode step; returns (state, selection for length t+1)."""
    cfg.validate()
    obs = np.asarray(observed, dtype=np.float64)
    t = obs.size
    if t < 1:
        raise OracleError("StateError", "observed row must be non-empty")
    calib = st.counter % cfg.calibration_period == 0
    src = np.asarray(full_row if (calib and full_row is not None) else obs, dtype=np.float64)
    if src.size != t:
        raise OracleError("StateError", "dense row length must match the observed row")
    comp = max_pool(src, cfg.block_size)
    st.history.append(comp)
    if len(st.history) > cfg.history:
        st.history = st.history[len(st.history) - cfg.history:]
    nxt = t + 1
    sink = set(range(min(cfg.sink_tokens, nxt)))
    local = set(range(max(0, nxt - cfg.local_tokens), nxt))
    if st.counter % cfg.update_interval == 0:
        k = cfg.middle_blocks
        if k > 0:
            if w is None:
                raise OracleError("StateError", "middle budget requires forecaster weights")
            grid = stack_history(st.history, cfg.history, comp.size)
            pred = forward(w, grid)
            masked = masked_scores(cfg, pred, t)
            avail = int(np.count_nonzero(masked > -np.inf))
            chosen = topk(masked, min(k, avail))
            st.middle = expand_indices(chosen, cfg.block_size, t)
            st.last_scores = pred
            st.last_blocks = sorted(chosen)
        else:
            st.middle = set()
            st.last_blocks = []
    sel = sink | local | st.middle
    if len(sel) > cfg.budget:
        raise OracleError("StateError", "selection exceeded the budget")
    st.selection = sel
    st.counter += 1
    return st, sel


def observed_from_selection(row, selection) -> np.ndarray:
    """evaluation.py:109-112 — dense row at selected positions, zeros elsewhere (not renormalised)."""
    row = np.asarray(row, dtype=np.float64)
    out = np.zeros_like(row)
    idx = np.array(sorted(i for i in selection if i < row.size), dtype=np.intp)
    if idx.size:
        out[idx] = row[idx]
    return out


def run_predictor_loop(prefill_rows, decode_rows, cfg: Config, w: Weights):
    """evaluation.py:90-115 (method="predictor") — yields (t+1, selection, state snapshot)."""
    st = init_state(cfg, prefill_rows)
    sel = None
    out = []
    for row in decode_rows:
        row = np.asarray(row, dtype=np.float64)
        obs = row if sel is None else observed_from_selection(row, sel)
        st, sel = step(st, cfg, w, obs, full_row=row)
        out.append((row.size + 1, set(sel), None if st.last_blocks is None else list(st.last_blocks)))
    return out


def recovery_rate(row, selection) -> float:
    """evaluation.py:70-81."""
    row = np.asarray(row, dtype=np.float64)
    tot = float(np.abs(row).sum())
    if tot <= 0.0:
        raise OracleError("MetricError", "recovery rate undefined for a zero-mass row")
    idx = np.array(sorted(int(i) for i in selection), dtype=np.intp)
    if idx.size == 0:
        return 0.0
    if idx[0] < 0 or idx[-1] >= row.size:
        raise OracleError("MetricError", "selection index out of row range")
    return float(row[idx].sum() / tot)

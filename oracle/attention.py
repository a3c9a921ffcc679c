"""CPU ORACLE — test infrastructure only, never a product path.

Float64 restatement of the attention pieces of the hot path that have NO
implementation in the reference package (SURVEY.md §8c "Kernels with no
reference implementation"):

* dense decode attention — the math of the exporter's toy model,
  attntap/model.py:70-74 (scores = q·kᵀ/√d, causal mask, softmax, ·V) for a
  single decode query (the causal mask is "keys [0, t)");
* sparse decode attention over a selection set S — the same math restricted
  to S (selection structure: selector.py:122-149);
* the calibration row — max_pool of the dense softmax row
  (selector.py:112-117 "calibrate → full_row"), computed here literally as
  softmax-then-max_pool;
* the observed (fed-back) row in the two modes DESIGN.md defines:
  ``masked_dense`` = evaluation.py:109-112 (dense probabilities at selected
  positions, not renormalised) and ``sparse_renorm`` = probabilities of the
  sparse softmax over S;
* the prefetch gather — byte-exact numpy fancy indexing of the host KV.

Parity here is "unpinned by reference vectors" for the attention outputs
(the reference has none); the compress half of each check is pinned through
``hotpath.max_pool``.
"""

from __future__ import annotations

import numpy as np

from oracle.hotpath import max_pool


def _scores(q, keys) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(keys, dtype=np.float64)
    return (k @ q) / np.sqrt(q.shape[-1])


def dense_decode(q, keys, values):
    """attntap/model.py:70-74 for one query over keys[0:t]: returns (out, lse, probs)."""
    s = _scores(q, keys)
    m = s.max()
    e = np.exp(s - m)
    den = e.sum()
    p = e / den
    out = p @ np.asarray(values, dtype=np.float64)
    return out, float(m + np.log(den)), p


def sparse_decode(q, keys, values, token_idx):
    """Dense math restricted to the token set S (sorted ascending)."""
    idx = np.asarray(sorted(int(i) for i in token_idx), dtype=np.intp)
    out, lse, p = dense_decode(q, np.asarray(keys)[idx], np.asarray(values)[idx])
    return out, lse, idx, p


def calibration_row(q, keys, b: int) -> np.ndarray:
    """max_pool(softmax(q·Kᵀ/√d), b) — the dense row the history stores on calibration steps."""
    _, _, p = dense_decode(q, keys, np.zeros((len(keys), 1)))
    return max_pool(p, b)


def observed_row_sparse_renorm(q, keys, token_idx, t: int) -> np.ndarray:
    """Row of length t: sparse-softmax probability on S, 0 elsewhere."""
    _, _, idx, p = sparse_decode(q, keys, np.zeros((len(keys), 1)), token_idx)
    row = np.zeros(t, dtype=np.float64)
    row[idx] = p
    return row


def observed_row_masked_dense(q, keys, token_idx, t: int) -> np.ndarray:
    """evaluation.py:109-112 — dense probabilities at S, zeros elsewhere (not renormalised)."""
    _, _, p = dense_decode(q, keys, np.zeros((len(keys), 1)))
    row = np.zeros(t, dtype=np.float64)
    idx = np.asarray(sorted(int(i) for i in token_idx if i < t), dtype=np.intp)
    row[idx] = p[idx]
    return row


def selection_tokens(t_next: int, sink: int, local: int, blocks, b: int, t_clip: int) -> list[int]:
    """selector.py:122-149 — sink ∪ local ∪ expand(blocks, b, t_clip) for a row of length t_next."""
    s = set(range(min(sink, t_next)))
    s |= set(range(max(0, t_next - local), t_next))
    for j in blocks:
        s.update(range(j * b, min(j * b + b, t_clip)))
    return sorted(s)


def gather_blocks(host_kv: np.ndarray, block_ids, b: int) -> np.ndarray:
    """Prefetch oracle: host_kv (n_blocks*b, ...) → concatenation of the requested blocks."""
    parts = [host_kv[j * b:(j + 1) * b] for j in block_ids]
    return np.concatenate(parts, axis=0) if parts else host_kv[:0]

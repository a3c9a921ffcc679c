"""Parity helpers shared by the GPU tests (the tolerance contract of SURVEY §8b / DESIGN.md)."""

from __future__ import annotations

import numpy as np

# forecaster tolerance per device precision (DESIGN.md §Parity contract):
#   |x - y| <= rtol * max(|y|, floor * max|y_row|)
# fp32-class modes (SIMT fp32, fp16x3 tensor cores): rtol 1e-3, floor 1e-2;
# the single-MMA fp16 mode: rtol 2e-2 (the north_star's bf16 bound), floor 1e-1.
RTOL = {"fp64": 1e-12, "fp32": 1e-3, "fp16x3": 1e-3, "fp16": 2e-2}
FLOOR = {"fp64": 1e-2, "fp32": 1e-2, "fp16x3": 1e-2, "fp16": 1e-1}


def scores_close(got, want, precision: str) -> tuple[bool, float]:
    rtol = RTOL[precision]
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    floor = np.abs(want).max() * FLOOR[precision] if want.size else 0.0
    bound = rtol * np.maximum(np.abs(want), floor)
    err = np.abs(got - want)
    worst = float(np.max(err / np.maximum(bound, 1e-300))) if want.size else 0.0
    return bool(np.all(err <= bound)), worst


def near_tie_exemptions(dev_blocks, ref_blocks, ref_masked_scores, k: int, precision: str) -> int:
    """Blocks in the symmetric difference of two top-k sets are acceptable only when their oracle
    score is within the forecaster tolerance of the k-th largest oracle score (a near-tie the
    device arithmetic may legitimately flip).  Returns the number of exempted blocks; raises
    AssertionError for a genuine mismatch."""
    a, b = set(int(x) for x in dev_blocks), set(int(x) for x in ref_blocks)
    diff = a ^ b
    if not diff:
        return 0
    s = np.asarray(ref_masked_scores, np.float64)
    finite = s[np.isfinite(s)]
    kth = np.sort(finite)[::-1][k - 1]
    scale = np.abs(finite).max()
    tol = RTOL[precision] * max(abs(kth), scale * FLOOR[precision])
    for j in diff:
        assert abs(s[j] - kth) <= tol, f"block {j}: score {s[j]} vs k-th {kth} (tol {tol}) is not a near tie"
    return len(diff)

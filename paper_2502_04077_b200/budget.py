"""Budget allocation across layers and heads.

The reference gives every (layer, head) the same token budget B and splits it as sink + local +
middle blocks (selector.py:47-50; the paper: 64 prefix + 64 local tokens, the rest to the
predicted middle blocks).  The device selector also accepts one budget per map
(ap_selector.k_map), each evaluated exactly like the reference's per-map SelectorConfig — so a
policy that moves budget between layers or heads keeps every map's selection bit-exact against
the oracle run with that map's budget.

Policies (all keep the total middle budget of the uniform allocation, up to block rounding):
* ``uniform``  — the reference: every map gets B.
* ``weights``  — per-layer (and optionally per-map-within-layer) weights; budget_i ∝ weight_i.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigError


def middle_blocks_per_map(budgets, n_maps: int, cfg) -> np.ndarray:
    """selector.py:47-50 per map: (B_m - sink - local) // b, validated like SelectorConfig.validate."""
    b = np.asarray(budgets, dtype=np.int64).ravel()
    if b.size != n_maps:
        raise ConfigError(f"expected {n_maps} per-map budgets, got {b.size}")
    if np.any(b < cfg.sink_tokens + cfg.local_tokens):
        raise ConfigError("budget must cover the sink and local allocations")
    k = (b - cfg.sink_tokens - cfg.local_tokens) // cfg.block_size
    if np.any(k > cfg.middle_blocks):
        raise ConfigError("a per-map budget exceeds cfg.budget (the mid_blocks pitch)")
    return k.astype(np.int32)


def allocate(cfg, n_layers: int, maps_per_layer: int, policy: str = "uniform", layer_weights=None,
             n_seq: int = 1, mean_budget: int | None = None) -> np.ndarray:
    """Per-map token budgets in the selector's map order (sequence, layer, map-in-layer).

    ``weights``: the middle blocks of all layers, (mean_budget - sink - local) // b each under the
    uniform policy (mean_budget defaults to cfg.budget), are redistributed proportionally to ``layer_weights`` (water-filling: each layer is capped at
    cfg.budget's middle-block count, the mid_blocks pitch, and what a capped layer cannot take goes to the
    others; if every positive-weight layer is capped the rest is dropped); sink and local stay per map."""
    K = cfg.middle_blocks  # the cap: cfg.budget sets the pitch of mid_blocks
    base = cfg.sink_tokens + cfg.local_tokens
    mean = cfg.budget if mean_budget is None else int(mean_budget)
    if mean < base or mean > cfg.budget:
        raise ConfigError("mean_budget must lie in [sink + local, cfg.budget]")
    Km = (mean - base) // cfg.block_size  # middle blocks per layer of the uniform allocation
    if policy == "uniform":
        per_layer = np.full(n_layers, Km, dtype=np.int64)
    elif policy == "weights":
        w = np.asarray(layer_weights, dtype=np.float64)
        if w.shape != (n_layers,) or np.any(w < 0) or w.sum() <= 0:
            raise ConfigError("layer_weights must be n_layers non-negative numbers with a positive sum")
        total = Km * n_layers
        per_layer = np.zeros(n_layers, dtype=np.int64)
        # water-filling: share what is left among the uncapped positive-weight layers in proportion
        # to their weights; a layer at the cap (K: the mid_blocks pitch) drops out
        for _ in range(n_layers + 1):
            open_ = (w > 0) & (per_layer < K)
            left = total - int(per_layer.sum())
            if left <= 0 or not open_.any():
                break
            raw = np.where(open_, w / w[open_].sum() * left, 0.0)
            add = np.minimum(np.floor(raw).astype(np.int64), K - per_layer)
            if add.sum() == 0:  # hand the last few blocks out by largest remainder
                for j in np.argsort(-(raw - np.floor(raw)), kind="stable"):
                    if left == 0:
                        break
                    if open_[j] and per_layer[j] < K:
                        per_layer[j] += 1
                        left -= 1
                continue
            per_layer += add
    else:
        raise ConfigError(f"unknown budget policy {policy!r}")
    tokens = base + per_layer * cfg.block_size
    return np.tile(np.repeat(tokens, maps_per_layer), n_seq).astype(np.int64)

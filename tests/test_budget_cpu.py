"""Budget allocation policies (host logic; the device side is tests/test_gpu_budget.py)."""

import numpy as np
import pytest

from paper_2502_04077_b200.budget import allocate, middle_blocks_per_map
from paper_2502_04077_b200.errors import ConfigError
from paper_2502_04077_b200.selector import SelectorConfig


def test_uniform_is_the_reference_split():
    cfg = SelectorConfig(budget=1024)
    b = allocate(cfg, n_layers=4, maps_per_layer=8, n_seq=2)
    assert b.shape == (64,) and np.all(b == 1024)
    assert np.all(middle_blocks_per_map(b, 64, cfg) == cfg.middle_blocks)


def test_weighted_layers_keep_the_total_and_the_cap():
    cfg = SelectorConfig(budget=1024)
    w = np.array([1.0, 3.0, 2.0, 1.0, 0.5])
    cfg = SelectorConfig(budget=2048)  # pitch 120 blocks; the uniform share (1024) is 56
    b = allocate(cfg, n_layers=5, maps_per_layer=2, policy="weights", layer_weights=w, mean_budget=1024)
    k = (b[::2] - 128) // 16
    assert k.sum() == 5 * 56 and np.all(k <= cfg.middle_blocks)
    assert k[1] > k[2] > k[0] == k[3] > k[4]
    # caps: every positive-weight layer saturates, the zero-weight layer gets nothing, the rest is dropped
    cfg = SelectorConfig(budget=1024)
    k = (allocate(cfg, 5, 1, policy="weights", layer_weights=[4, 3, 2, 1, 0]) - 128) // 16
    assert k.tolist() == [56, 56, 56, 56, 0]


def test_errors():
    cfg = SelectorConfig(budget=512)
    with pytest.raises(ConfigError):
        middle_blocks_per_map([100] * 4, 4, cfg)   # below sink + local
    with pytest.raises(ConfigError):
        middle_blocks_per_map([1024] * 4, 4, cfg)  # above the pitch
    with pytest.raises(ConfigError):
        middle_blocks_per_map([512] * 3, 4, cfg)
    with pytest.raises(ConfigError):
        allocate(cfg, 3, 1, policy="weights", layer_weights=[0, 0, 0])

"""B200-native AttentionPredictor decode-time critical-token path.

Reference-compatible modules (drop-in for ``attncast.compress``,
``attncast.predictor`` inference half, ``attncast.selector``):
``compress``, ``predictor``, ``selector``.  Device-resident batched engine:
``batched.BatchedSelector``; attention / calibration / prefetch kernels and
the decode engine live in ``attention``, ``prefetch`` and ``decode``.

All compute runs in ``lib/libattnpred.so`` (sm_100a); there is no CPU
fallback.
"""

from . import errors  # noqa: F401

__version__ = "1.0.0"

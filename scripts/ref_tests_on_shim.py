"""Run the reference's OWN hot-path test files against this package (GPU box).

    python scripts/ref_tests_on_shim.py [pytest args]

Needs the reference installed in baseline/_ref (git-ignored; it travels with gpurun):

    python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
        --target baseline/_ref <copy of /root/reference/pkg>
    mkdir -p baseline/_ref/tests && cp /root/reference/pkg/tests/*.py baseline/_ref/tests/

The aliasing is exactly INTEGRATION.md §1: attncast.errors / compress / selector / trace are
replaced by this package's modules, and the predictor names (inference and training) are
patched onto the reference's predictor module.  Everything those tests call then runs through
libattnpred.so; the rest of attncast (synth, evaluation, baselines) stays the reference's.
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
DEFAULT_FILES = ["test_compress.py", "test_selector.py", "test_predictor.py", "test_trace.py"]


def install_shim():
    sys.path.insert(0, str(ROOT))
    sys.path.insert(1, str(REF))
    import paper_2502_04077_b200.compress as compress
    import paper_2502_04077_b200.errors as errors
    import paper_2502_04077_b200.predictor as predictor
    import paper_2502_04077_b200.selector as selector
    import paper_2502_04077_b200.trace as trace

    sys.modules["attncast.errors"] = errors  # before attncast/__init__ imports it
    import attncast

    for name, mod in (("compress", compress), ("selector", selector), ("trace", trace)):
        sys.modules[f"attncast.{name}"] = mod
        setattr(attncast, name, mod)
    import attncast.predictor as ref_pred

    for name in ("forward", "stack_history", "AttentionHistory", "PredictorWeights", "init_weights", "save_weights",
                 "load_weights", "TrainSample", "EpochMetrics", "backward", "build_dataset", "train"):
        setattr(ref_pred, name, getattr(predictor, name))
    return attncast


def main():
    import pytest

    install_shim()
    args = sys.argv[1:]
    files = [a for a in args if a.endswith(".py")] or DEFAULT_FILES
    opts = [a for a in args if not a.endswith(".py")]
    sys.exit(pytest.main([*(str(REF / "tests" / f) for f in files), "-p", "no:cacheprovider",
                          "--rootdir", str(REF / "tests"), *opts]))


if __name__ == "__main__":
    main()

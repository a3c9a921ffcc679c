"""The reference's OWN test suite (all 173 tests of /root/reference/pkg/tests) run against this
package on the GPU: attncast.compress / selector / trace / errors and the predictor names are
aliased to paper_2502_04077_b200 (scripts/ref_tests_on_shim.py), so every
hot-path call those tests make goes through libattnpred.so.

baseline/_ref (git-ignored, shipped with the gpurun snapshot) holds the unmodified reference and
its tests; scripts/install_reference.sh creates it in the build container.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = ROOT / "baseline" / "_ref" / "tests"


def test_reference_suite_on_shim():
    if not (REF_TESTS / "test_selector.py").exists():
        pytest.skip("baseline/_ref not installed (scripts/install_reference.sh)")
    files = sorted(p.name for p in REF_TESTS.glob("test_*.py"))
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, str(ROOT / "scripts" / "ref_tests_on_shim.py"), *files, "-q", "-x"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = (out.stdout + out.stderr)[-4000:]
    print(tail)
    m = re.search(r"(\d+) passed", out.stdout)
    assert out.returncode == 0, tail
    assert m and int(m.group(1)) >= 173, tail

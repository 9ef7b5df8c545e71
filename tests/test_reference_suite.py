"""Run the REFERENCE's own test suite (pkg/tests, 190 tests) against this
package through a tiny `acctuner` alias shim.  Only where /root/reference
exists (the build container); skipped elsewhere."""

from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import REPO

REF_TESTS = Path("/root/reference/pkg/tests")

SHIM = f'''
import sys
sys.path.insert(0, {str(REPO)!r})
import paper_1811_03882_b200 as _p
from paper_1811_03882_b200 import *
from paper_1811_03882_b200 import cli as _cli
for _n in ("nodes", "parser", "loops", "analysis", "transfer", "evaluation", "ga", "emitter",
           "pipeline", "errors"):
    sys.modules["acctuner." + _n] = getattr(_p, _n)
sys.modules["acctuner.cli"] = _cli
'''


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tests not mounted here")
def test_reference_suite_passes_against_this_package(tmp_path):
    shim = tmp_path / "shim" / "acctuner"
    shim.mkdir(parents=True)
    (shim / "__init__.py").write_text(SHIM)
    tests = tmp_path / "tests"
    shutil.copytree(REF_TESTS, tests)
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
                           str(tests)], cwd=tmp_path, capture_output=True, text=True,
                          env={"PYTHONPATH": str(tmp_path / "shim"), "PATH": "/usr/bin:/bin"},
                          timeout=600)
    tail = proc.stdout.strip().splitlines()[-1] if proc.stdout.strip() else proc.stderr[-2000:]
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-2000:]
    assert "190 passed" in tail, tail

"""compute-sanitizer over a small-frame workload covering every kernel route
(tools/sanitize.py): no memory errors, no shared-memory races, no barrier misuse, no reads of
uninitialised device memory. SURVEY.md §4.2 item 5."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer not found")
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize workload ok" in out
    if tool == "racecheck":
        assert "0 hazards" in out, out[-3000:]
    else:
        assert "0 errors" in out, out[-3000:]

"""compute-sanitizer over the generated pass kernels (VERDICT r1 hygiene item):
memcheck (out-of-bounds / misaligned global and shared accesses), racecheck
(shared-memory hazards: the swizzled free-lane transposes, cp.async staging into
transpose buffers reused after barriers) and synccheck (barrier misuse), on
small states with several tiles per pass and the PDL chain between passes."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _sanitizer():
    for cand in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if cand and os.path.exists(cand):
            return cand
    pytest.skip("compute-sanitizer not installed")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("name,tile", [("cfg3_n14", 9), ("cfg5_n15", 10)])
def test_generated_kernels_sanitizer_clean(tool, name, tile):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(HERE, "sanitize_case.py"), name, str(tile)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]

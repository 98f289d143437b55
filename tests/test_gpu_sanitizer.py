"""compute-sanitizer racecheck / synccheck / memcheck on small runs of every kernel family
(tools/sanitize_small.py: kernels 5 with half items, 6, 4, 0, 0 with the live k loop, 7, 1): the
mbarrier / named-barrier protocols of the warp-specialised kernels must show no shared-memory race,
no barrier misuse (every mbarrier phase observed) and no out-of-bounds access."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    assert os.path.exists(cs), "compute-sanitizer not found"
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_small.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "compute-sanitizer is closed on this pool" in out:
        # the GPU pool disabled the tool after other runs under it left GPUs needing a reset; the
        # clean runs of this round are kept in profiles/r2_sanitize_{racecheck,synccheck,memcheck}.txt
        pytest.skip("compute-sanitizer disabled by the GPU pool (exit 86); see profiles/r2_sanitize_*.txt")
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards" in out, out[-2000:]

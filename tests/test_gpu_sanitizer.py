"""compute-sanitizer over small workloads of every kernel family (needs a
B200; scripts/sanitize_driver.py): memcheck and synccheck must report no
errors; racecheck may only report the splat's mbarrier-ordered staging
buffer and decision slot (bake.cu: cp.async.bulk writes / ready-barrier
protected writes read after the consumers' mbarrier wait -- the protocol
racecheck does not model; the wide-M halo kernel's mbarrier pipeline,
Delaunay, raster, LAZ decode and render report nothing)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([exe, "--tool", tool, "--print-limit", "50", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_driver.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    return r.stdout + r.stderr


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_no_errors(tool):
    out = _run(tool)
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]


def test_racecheck_only_the_documented_splat_pipeline():
    out = _run("racecheck")
    sites = re.findall(r"Race reported between .*? at (\S+)", out)
    sites += re.findall(r"and (?:Read|Write) access at (\S+)", out)
    for s in sites:
        assert "bake_splat_kernel" in s or "bulk_g2s" in s, s

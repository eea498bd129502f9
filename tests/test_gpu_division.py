"""The forward's division shortcut (Markstein-corrected quotient with a
hoisted reciprocal, qfb_device.cuh) is bit-identical to IEEE division.
The full proof (all 2^46 significand pairs + all 2^32 x for 192 scales) is
tools/verify_div.cu, recorded in profiles/; this test runs its quick mode."""
import os
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_markstein_quick():
    exe = os.path.join(tempfile.mkdtemp(), "verify_div")
    subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                    os.path.join(ROOT, "tools", "verify_div.cu"), "-o", exe], check=True)
    r = subprocess.run([exe, "quick"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches = 0" in r.stdout

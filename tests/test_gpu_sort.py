"""GPU: the LBVH's hand-written radix sort (csrc/sort.cu) equals
std::stable_sort on random 30-bit and 12-bit keys (single tile, 2048- and
8192-key tile boundaries, both sides of the small-sort threshold 2^18,
1,003,520 keys), through tools/sort_check.cu."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_radix_sort_matches_stable_sort(gpu_ctx):
    exe = os.path.join(ROOT, "build", "sort_check")
    assert os.path.exists(exe), "build/sort_check not built (make cpp)"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all ok" in out.stdout
    assert "FAIL" not in out.stdout

"""GPU: the sort's bucketed scatter path (inputs beyond L2: place and the inverse permutation
through a bucket pass) is bit-exact against the oracle.  Large inputs take it by
default (the full-size c4 sort tests); here every sort test runs once more in a child process
with MM_SORT_BKT_MIN=1 (read once per process), so all sizes, orders, slabs and bin-size
classes (warp / CTA / huge fix-ups) go through it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_sort_tests_through_bucketed_scatter():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MM_SORT_BKT_MIN="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "tests/test_gpu_parity_sort_tf32.py",
                        "tests/test_gpu_async_sort.py", "-q", "-x", "-m", "gpu", "-k", "sort and not full_size"],
                       env=env, capture_output=True, text=True, timeout=1500, cwd=root)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-3000:]
    assert " passed" in r.stdout

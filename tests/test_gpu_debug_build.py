"""The debug build (make debug -> paper_1106_4198_b200/lib_debug, -DISNMF_DEBUG):
device-side index checks (ISNMF_DASSERT: warm-store columns and tags, statistics
planes and divergence partials against their allocation, the commit's P row,
fragment indices) that print their location and trap.  compute-sanitizer is
closed on this pool, so this is the CI-style guard against out-of-bounds
regressions: the reference-pinned trainer cases, the batch, stateless-kernel and
held-out suites run through the debug library in a subprocess and must pass with
no check firing."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_1106_4198_b200", "lib_debug", "libisnmf_b200.so")


def test_suites_pass_under_the_debug_build():
    if not os.path.exists(DEBUG_LIB):
        subprocess.run(["make", "-s", "-j8", "-C", ROOT, "debug"], check=True)
    env = dict(os.environ, ISNMF_LIB=DEBUG_LIB)
    suites = ["tests/test_gpu_ref_trainers.py", "tests/test_gpu_batch.py", "tests/test_gpu_kernels.py",
              "tests/test_gpu_heldout.py", "tests/test_gpu_mma.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *suites], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert "ISNMF_DASSERT" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]


def test_debug_library_is_the_one_loaded():
    if not os.path.exists(DEBUG_LIB):
        subprocess.run(["make", "-s", "-j8", "-C", ROOT, "debug"], check=True)
    code = ("import paper_1106_4198_b200 as E; E.lib(); print(E.LIB_PATH)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, ISNMF_LIB=DEBUG_LIB),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == DEBUG_LIB, r.stderr

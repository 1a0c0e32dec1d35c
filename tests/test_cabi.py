"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU and exports every symbol include/isnmf_b200.h declares (no compute calls)."""
import ctypes
import os
import subprocess

import pytest

import paper_1106_4198_b200 as eng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    if not os.path.exists(eng.LIB_PATH):
        subprocess.run(["make", "-s", "-C", ROOT, eng.LIB_PATH], check=True)
    return eng.LIB_PATH


def test_header_declares_the_boundary():
    syms = eng.header_symbols()
    for s in ("isnmf_solve_h", "isnmf_batch_stats", "isnmf_update_w", "isnmf_rescale_dictionary",
              "isnmf_objective", "isnmf_is_divergence", "isnmf_online_create", "isnmf_online_run",
              "isnmf_online_get_dictionary", "isnmf_batch_train", "isnmf_last_error"):
        assert s in syms


def test_library_exports_every_header_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [s for s in eng.header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(eng.header_symbols()) <= exported


def test_python_face_binds_every_symbol(libpath):
    assert set(eng.header_symbols()) <= set(eng._SIGS)


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out

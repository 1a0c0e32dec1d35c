"""Builds and runs the C++ API tests (tests/cpp): the reference's own unit
tests restated against include/isnmf/*.hpp, linked to the engine library."""
import os
import subprocess

import pytest

import paper_1106_4198_b200 as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.dirname(E.LIB_PATH)


def build(name, tmp_path):
    if not os.path.exists(E.LIB_PATH):
        subprocess.run(["make", "-s", "-C", ROOT, E.LIB_PATH], check=True)
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/{name}.cpp",
           f"-L{LIBDIR}", "-lisnmf_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


def run(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    return r.stdout


def test_cpp_api_host(tmp_path):
    out = run(build("test_api_host", tmp_path))
    assert "0 failed" in out


@pytest.mark.gpu
def test_cpp_api_gpu(tmp_path):
    out = run(build("test_api_gpu", tmp_path))
    assert "0 failed" in out

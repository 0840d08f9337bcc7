"""The reference-signature C++ API (include/qrtebd/qrtebd_api.hpp ->
libqrtebd_api.so) compiles and links on CPU and, on a B200, drives the device
with the reference's own call shapes (GPU)."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2212_09782_b200")


def compile_cmd(out):
    return ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out, "-L", LIBDIR,
            "-l:libqrtebd_api.so", "-l:libqrtebd_b200.so", f"-Wl,-rpath,{LIBDIR}"]


def test_header_compiles_and_links(tmp_path):
    out = str(tmp_path / "test_api")
    r = subprocess.run(compile_cmd(out), capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cpp_api_runs_on_device(tmp_path):
    out = str(tmp_path / "test_api")
    subprocess.run(compile_cmd(out), check=True)
    r = subprocess.run([out], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK")

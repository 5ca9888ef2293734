"""The header-only C++ shim (include/eapdtw_b200.hpp) compiles and links
against libeapdtw_b200.so on CPU; it runs bit-exact on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2010_05371_b200")


def build(tmp_path, name="shim_test"):
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", PKG, "-leapdtw_b200",
           f"-Wl,-rpath,{PKG}", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout


def test_multi_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path, "multi_test"))


@pytest.mark.gpu
def test_multi_device_shim_runs_on_gpu(tmp_path):
    """eapdtw_multi_* (one host thread, NCCL communicator) at N = 1 through
    the C++ shim: the single-device answers and the reference NN1 loop."""
    exe = build(tmp_path, "multi_test")
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout

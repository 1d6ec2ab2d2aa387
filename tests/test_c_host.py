"""The C ABI from plain C (tests/c_host/abi_host.c): how a C / cgo / JNI host of
the reference's path would bind it -- no Python, no torch on the data path."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(out):
    libdir = os.path.join(ROOT, "paper_1402_0532_b200")
    orc = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", orc], check=True)
    cmd = ["gcc", "-O2", "-std=gnu11", os.path.join(ROOT, "tests", "c_host", "abi_host.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           "-L", libdir, "-lsignadd_b200", "-L", orc, "-loracle", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           "-lm", "-lpthread", f"-Wl,-rpath,{libdir}:{orc}:{os.path.join(CUDA, 'lib64')}", "-o", out]
    subprocess.run(cmd, check=True)


def test_c_host_builds(tmp_path):
    if not os.path.exists(os.path.join(ROOT, "paper_1402_0532_b200", "libsignadd_b200.so")):
        pytest.skip("library not built")
    _build(str(tmp_path / "abi_host"))


@pytest.mark.gpu
def test_c_host_parity(sa, tmp_path):
    exe = str(tmp_path / "abi_host")
    _build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "c-host ok" in r.stdout

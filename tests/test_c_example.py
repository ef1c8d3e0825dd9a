"""The C-ABI from plain C (examples/c_abi_kat.c): no Python on the data path, the reference's
known-answer test (tests/test_attention.py:46-52) through fs_fwd."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_c_caller_known_answer(tmp_path):
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    lib = os.path.join(ROOT, "paper_2505_09326_b200", "_lib")
    exe = tmp_path / "kat"
    subprocess.run([cc, "-std=c99", "-Wall", os.path.join(ROOT, "examples", "c_abi_kat.c"),
                    "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"), "-L" + lib,
                    "-lflashsign", "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath," + lib, "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "O[0] = 22.000000" in r.stdout

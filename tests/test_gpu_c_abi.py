"""The C ABI from a plain C program (no Python, no torch): tests/c/abi_solve.c
is compiled with gcc against include/fmgsr_cuda.h and libfmgsr_cuda.so and
solves a batch through fmgsr_plan_create / fmgsr_plan_solve."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_client_solves_through_the_abi(tmp_path, fm):
    cuda = "/usr/local/cuda"
    lib_dir = os.path.join(ROOT, "paper_1207_6720_b200")
    exe = tmp_path / "abi_solve"
    subprocess.run(["gcc", "-O2", "-std=c11", os.path.join(ROOT, "tests", "c", "abi_solve.c"),
                    "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                    "-L", lib_dir, "-lfmgsr_cuda", "-L", f"{cuda}/lib64", "-lcudart",
                    f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{cuda}/lib64", "-lm", "-o", str(exe)],
                   check=True)
    for args in (["12", "64", "4", "64"], ["10", "4", "2", "3"]):
        out = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "max_rel_err" in out.stdout

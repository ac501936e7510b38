"""The header-only C++ BatchRunner adapter (include/rmpc_b200_batch.hpp) compiles with g++,
links against the C-ABI library and behaves like rmpc::BatchRunner on the no-GPU paths."""
import os
import subprocess

import pytest

from conftest import HAS_GPU, ROOT


def test_cpp_adapter_compiles_and_runs(tmp_path):
    import paper_2510_12717_b200 as R
    R.library()
    exe = str(tmp_path / "adapter_check")
    libdir = os.path.join(ROOT, "paper_2510_12717_b200", "lib")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_check.cpp"), "-L", libdir, "-lrmpc_b200",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, check=True)
    assert r.stdout.strip() == ("0" if HAS_GPU else "10")

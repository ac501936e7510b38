"""Build the sm_100a shared library in-tree: paper_2510_12717_b200/lib/librmpc_b200.so.

nvcc cross-compiles here without a GPU; the .so travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "librmpc_b200.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("rmpc_kernel.cu", "rmpc_host.cu", "rmpc_env.cu", "rmpc_policy.cu",
                                                       "rmpc_ppo.cu")]
# every header of csrc/ and include/ (a new header must rebuild the library too)
HEADERS = sorted(os.path.join(HERE, "csrc", h) for h in os.listdir(os.path.join(HERE, "csrc")) if h.endswith(".cuh")) + \
    sorted(os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include")) if h.endswith((".h", ".hpp")))
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB_PATH):
        return False
    t = os.path.getmtime(LIB_PATH)
    return all(os.path.getmtime(s) <= t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB_PATH
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    # one nvcc per translation unit, in parallel (the solve kernel dominates), then one link
    objs = [os.path.join(LIB_DIR, os.path.basename(src).replace(".cu", ".o")) for src in SOURCES]
    # (the solve TU is relocatable device code: its list dispatcher tail-launches the per-agent
    # kernel from the device)
    procs = [subprocess.Popen([nvcc(), *NVCC_FLAGS, *(["-rdc=true"] if src.endswith("rmpc_kernel.cu") else []),
                               "-c", "-o", o, src], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for src, o in zip(SOURCES, objs)]
    logs = []
    for pr in procs:
        out, err = pr.communicate()
        logs.append(out + err)
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError("nvcc failed building librmpc_b200.so")
    r = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-rdc=true", "-shared", "-o", tmp,
                        *objs, "-lcudadevrt"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking librmpc_b200.so")
    if verbose:
        sys.stderr.write("".join(logs))
    for o in objs:
        os.remove(o)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

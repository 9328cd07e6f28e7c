"""Build liboomb.so (the sm_100a kernels + the C-ABI host runtime) in-tree.

    python -m paper_2602_02108_b200.build [--force]

nvcc cross-compiles for sm_100a without a GPU. The library links the CUDA
runtime statically and resolves cuTensorMapEncodeTiled through the runtime's
driver entry point, so it loads on hosts without libcuda (the CPU test suite
checks its exported symbols) and uses the driver on the GPU box.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "liboomb.so")
COMM_LIB = os.path.join(PKG, "liboomb_comm.so")  # NCCL exchange steps (include/oomb_comm.h)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["oomb_api.cu", "kernels_simt.cu", "attn_tc.cu", "attn_fwd4.cu", "attn_bwd_tc.cu", "score_tc.cu", "tier.cu",
           "layer_loop.cu"]
HEADERS = ["oomb_internal.h", "ptx.cuh", "tc_common.cuh", "pool.h"]

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
    f"-I{INCLUDE}", f"-I{CSRC}",
    "-DOOMB_BUILD",
]


def _digest() -> str:
    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    for f in (os.path.join(INCLUDE, "oomb.h"), os.path.join(INCLUDE, "oomb_comm.h"), os.path.join(CSRC, "comm.cu")):
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = LIB + ".sha256"
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(COMM_LIB) and os.path.exists(stamp) and open(stamp).read() == dig:
        return LIB
    objdir = os.path.join(PKG, "_build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-dc" if False else "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    logs = []
    for src, pr in procs:
        out, _ = pr.communicate()
        logs.append(f"== {src}\n{out}")
        if pr.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {src}")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", LIB, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    # liboomb_comm.so: host code over NCCL and liboomb.so's public combine entry points
    comm_obj = os.path.join(objdir, "comm.o")
    for cmd in ([NVCC, *FLAGS, "-c", os.path.join(CSRC, "comm.cu"), "-o", comm_obj],
                [NVCC, "-shared", "-cudart", "static", "-o", COMM_LIB, comm_obj, f"-L{PKG}", "-loomb", "-lnccl",
                 "-Xlinker", "-rpath,$ORIGIN"]):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("liboomb_comm.so build failed")
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    with open(stamp, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

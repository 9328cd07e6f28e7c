"""Build a liboomb.so variant with extra -D flags into tools/liboomb_<name>.so (A/B timing on the box:
copy it over paper_2602_02108_b200/liboomb.so before running bench.py)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_02108_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
objdir = os.path.join(B.PKG, "_build", "var_" + name)
os.makedirs(objdir, exist_ok=True)
procs, objs = [], []
for src in B.SOURCES:
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    procs.append(subprocess.Popen([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    objs.append(obj)
for p in procs:
    out, _ = p.communicate()
    if p.returncode:
        sys.exit(out)
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"liboomb_{name}.so")
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", out,
                *objs], check=True)
print(out)

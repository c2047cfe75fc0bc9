"""Build a variant of libshiftk.so with extra nvcc flags into _var/ (experiments; load it with
SHIFTK_LIB=_var/libshiftk_<name>.so).  Usage: python tests/tools/build_variant.py NAME -DFOO=1 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2001_08707_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
objdir = os.path.join(ROOT, "_var", "obj_" + name)
os.makedirs(objdir, exist_ok=True)
procs, objs = [], []
for src in B.sources():
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    procs.append(subprocess.Popen([B.NVCC] + B.CFLAGS + extra + ["-c", "-o", obj, src]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs), "nvcc failed"
out = os.path.join(ROOT, "_var", f"libshiftk_{name}.so")
subprocess.check_call([B.NVCC] + B.LDFLAGS + ["-o", out] + objs)
print(out)

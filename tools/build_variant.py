"""Experimental build of the library with extra defines, for A/B timing:

    python tools/build_variant.py NAME -DMACRO[=V] ...
    -> paper_1408_3764_b200/libgcmc_b200_NAME.so  (select with GCMC_LIB=...)
"""
import os, subprocess, sys, concurrent.futures as cf
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1408_3764_b200 import build as B

name, defs = sys.argv[1], sys.argv[2:]
obj_dir = os.path.join(B.ROOT, "build", "obj_" + name)
os.makedirs(obj_dir, exist_ok=True)
out = os.path.join(B.PKG, f"libgcmc_b200_{name}.so")
flags = [f for f in B.FLAGS if f != "-v" and f != "-Xptxas"] + defs


def one(src):
    obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
    r = subprocess.run([B.NVCC, *flags, "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return obj


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, B.sources()))
r = subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin",
                    B.HOSTCXX, *objs, "-o", out, "-lcudart"], capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print(out)

"""Dev tool: build a variant of libspmk_b200.so with extra -D flags into
paper_2106_16064_b200/build/<name>.so (travels to the GPU box for A/B runs).
    python tools/build_variant.py <name> -DFOO -DBAR=2"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_16064_b200 import _build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
odir = os.path.join(b.OBJ_DIR, name)
os.makedirs(odir, exist_ok=True)
objs = []
for cu in b._units():
    obj = os.path.join(odir, os.path.basename(cu)[:-3] + ".o")
    subprocess.run([b.NVCC, *b.NVCC_FLAGS, *defs, "-c", "-o", obj, cu], check=True)
    objs.append(obj)
out = os.path.join(b.OBJ_DIR, name + ".so")
subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-ldl"], check=True)
print(out)

"""Build an A/B variant of _apx.so into build/<name>/_apx.so with extra -D flags
(only the translation units that see the macro are rebuilt; the rest are linked from build/apx).

    python tools/build_variant.py exp_u4c4 cycle.cu -DAPX_GATHER_U=4 -DAPX_GATHER_CPT=4
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_19308_b200 import build as B  # noqa: E402

name, units, flags = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
out = os.path.join(ROOT, "build", name)
os.makedirs(out, exist_ok=True)
objs = []
for src in sorted(glob.glob(os.path.join(B.CSRC, "*.cu"))):
    base = os.path.basename(src)
    if base in units:
        o = os.path.join(out, base[:-3] + ".o")
        subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *flags, "-c", src, "-o", o], check=True)
        objs.append(o)
    else:
        objs.append(os.path.join(B.OBJ, base[:-3] + ".o"))
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, "_apx.so"), *objs, "-lcudart_static", "-lrt",
                "-ldl", "-lpthread"], check=True)
print(os.path.join(out, "_apx.so"))

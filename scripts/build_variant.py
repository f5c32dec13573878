"""Build an experiment variant of libhpar.so with extra -D flags for one source:

    python scripts/build_variant.py kernel_segmented.cu build/variants/libhpar_seg16k.so -DHPAR_SEG_LEN=16384

Load it with HPAR_LIB=<path> (paper_2309_01906_b200/hpar.py).  Experiments only."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_01906_b200 import build as B  # noqa: E402

src, out, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
os.makedirs(os.path.dirname(os.path.join(ROOT, out)), exist_ok=True)
objs = sorted(glob.glob(os.path.join(B.BUILD, "*.o")))
vo = os.path.join(ROOT, out + "." + src + ".o")
incs = ["-I", B.INCLUDE, "-I", B.CSRC, "-I", B._nccl_include()]
subprocess.run([B.NVCC] + B.ARCH + B.COMMON + incs + defs + ["-c", os.path.join(B.CSRC, src), "-o", vo], check=True)
objs = [vo if os.path.basename(o) == src + ".o" else o for o in objs]
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", os.path.join(ROOT, out)] + objs + ["-ldl", "-lpthread"], check=True)
print("built", out)

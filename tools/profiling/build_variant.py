"""Build a debug variant of libbsa.so with extra -D flags: python dbg/build_variant.py OUT.so -DBSA_TRACE ..."""
import os
import subprocess
import sys
import glob
import concurrent.futures as cf

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2509_01085_b200 import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
tag = os.path.splitext(os.path.basename(out))[0]
objdir = os.path.join("/tmp", "bsa_variant_" + tag)
os.makedirs(objdir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))


def cc(src):
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", src, "-o", obj], check=True)
    return obj


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(cc, srcs))
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "--cudart", "static", "-o", out, *objs,
                "-lpthread", "-ldl", "-lrt"], check=True)
print(out)

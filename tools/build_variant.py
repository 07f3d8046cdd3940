"""Build the library with extra nvcc flags into another path (tuning A/B
builds; the product build is paper_2105_00115_b200.build):
    python tools/build_variant.py OUT.so -DQDOT_B200_P1_TUNING ..."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_00115_b200 import build as B

out, extra = sys.argv[1], sys.argv[2:]
tmp = out + ".objs"
os.makedirs(tmp, exist_ok=True)


def one(src):
    obj = os.path.join(tmp, src.replace(".cu", ".o"))
    subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *extra, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    return obj


with ThreadPoolExecutor(len(B.SOURCES)) as ex:
    objs = list(ex.map(one, B.SOURCES))
subprocess.run([B.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", out], check=True)
print(out)

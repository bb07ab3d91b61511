"""A/B builds (development tool): the library's sources compiled with extra -D flags into
paper_2201_05413_b200/_variants/libpcg_<name>.so, loaded with PCG_LIB_VARIANT=<name>.

  python scripts/build_variant.py NAME [-DKNOB=1 ...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_05413_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, "_variants")
obj = os.path.join("/tmp", "pcg_variant_objs", name)  # objects stay out of the gpurun snapshot
os.makedirs(obj, exist_ok=True)
srcs = sorted(f for f in os.listdir(B.CSRC) if f.endswith(".cu"))


def cc(f):
    o = os.path.join(obj, f[:-3] + ".o")
    subprocess.check_call([B.NVCC] + B._flags() + defs + ["-c", os.path.join(B.CSRC, f), "-o", o])
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(cc, srcs))
_, nlib = B._nccl_dirs()
lib = os.path.join(out, f"libpcg_{name}.so")
subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs +
                      [f"-L{nlib}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={nlib}", "-cudart", "static"])
print(lib)

"""Build a variant of libcutfem.so with extra -D flags (A/B experiments on one
GPU call; load it with CUTFEM_LIB=build/variants/libcutfem_<name>.so).
usage: python tools/build_variant.py NAME [-DFLAG ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_07911_b200 import _lib

name, flags = sys.argv[1], sys.argv[2:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "build", "variants", f"libcutfem_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
nccl = _lib._nccl_dir()
cmd = ["nvcc", *_lib.NVCC_FLAGS, *flags, "-I", os.path.join(root, "include"), "-I", os.path.join(nccl, "include"),
       "-o", out, os.path.join(root, "paper_2404_07911_b200", "csrc", "cutfem.cu"), "-lcusparse",
       "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
subprocess.check_call(cmd)
print(out)

"""Development tool: build a variant of libfmm_b200.so with extra nvcc flags
for one source file (e.g. -DTC_DIAG=1 for m2l_tc.cu) under build/variants/<name>/;
load it with FMM_LIB=<path>.  Not part of the product path.

usage: python tools/build_variant.py NAME FILE.cu FLAG [FLAG ...]
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1106_5273_b200 import _build as B  # noqa: E402


def main():
    name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out = os.path.join(B.BUILD, "variants", name)
    os.makedirs(out, exist_ok=True)
    srcp = os.path.join(B.CSRC, src)
    obj = os.path.join(out, src[:-3] + ".o")
    subprocess.run([B.NVCC] + B.ARCH + B.FLAGS + flags + ["-c", srcp, "-o", obj], check=True, capture_output=True)
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if os.path.basename(o) != os.path.basename(obj)] + [obj]
    lib = os.path.join(out, "libfmm_b200.so")
    libdir = os.path.join(B.NCCL, "lib")
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs +
                   ["-Xcompiler", "-fPIC", "-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir], check=True)
    print(lib)


if __name__ == "__main__":
    main()

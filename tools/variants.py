"""Build tuning variants of libcssar.so that differ only in compile-time knobs of one source
file (the others are reused from the main build).  Usage:
    python tools/variants.py rg.cu NAME -DKNOB=1 ...   -> paper_1302_3120_b200/variants/libcssar_NAME.so
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1302_3120_b200 import build as B  # noqa: E402


def main():
    src, name, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out_dir = os.path.join(B.HERE, "variants")
    os.makedirs(out_dir, exist_ok=True)
    obj = os.path.join(out_dir, f"{name}_{src.replace('.cu', '.o')}")
    subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs = [obj if s == src else B._obj(s) for s in B.SOURCES]
    lib = os.path.join(out_dir, f"libcssar_{name}.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs], check=True)
    print(lib)


if __name__ == "__main__":
    main()

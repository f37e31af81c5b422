#!/usr/bin/env python
"""Build a tuning / experiment variant of libcssar.so with extra nvcc flags, recompiling only
the listed sources (the rest reuse the in-tree objects):

    python tools/build_variant.py NAME --src az_13.cu,rg.cu -DCSSAR_FOO=1 ...

-> paper_1302_3120_b200/variants/libcssar_NAME.so (git-ignored); select it at run time with
CSSAR_LIB=<path> (paper_1302_3120_b200.cssar.load_library honours it).  Not a product path."""
import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1302_3120_b200 import build as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--src", default="az_13.cu")
    args, flags = ap.parse_known_args()
    B.build()                                     # in-tree objects up to date
    vdir = os.path.join(B.HERE, "variants", args.name)
    os.makedirs(vdir, exist_ok=True)
    srcs = [s for s in args.src.split(",") if s]
    objs = []
    jobs = []
    for s in B.SOURCES:
        o = B._obj(s)
        if s in srcs:
            vo = os.path.join(vdir, os.path.basename(o))
            jobs.append([B.NVCC, *B.ARCH, *B.FLAGS, *flags, "-c", os.path.join(B.CSRC, s), "-o", vo])
            objs.append(vo)
        else:
            objs.append(o)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(" ".join(cmd) + "\n" + r.stdout + r.stderr)

    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        list(ex.map(run, jobs))
    lib = os.path.join(B.HERE, "variants", f"libcssar_{args.name}.so")
    run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
    shutil.rmtree(vdir, ignore_errors=True)
    print(lib)


if __name__ == "__main__":
    main()

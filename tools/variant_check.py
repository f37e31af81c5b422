"""Compare a tuning variant of libcssar against the in-tree build on the c3 workload:
    python tools/variant_check.py NAME [iters]   (run on a GPU box)
Prints the relative L2 difference of X after `iters` ITA iterations (expect ~1e-6)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_one(lib, out, iters):
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
sys.argv = ['bench']
import bench
from inputs import configs
from paper_1302_3120_b200 import Plan
cfg = configs.get('c3'); plan = Plan(cfg.params)
Y, mb, mask, sc = bench.make_problem_gpu(cfg, plan)
X = plan.ita_iterate(Y, mb, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters={iters})
np.save({out!r}, X.cpu().numpy())
"""
    env = dict(os.environ)
    if lib:
        env["CSSAR_LIB"] = lib
    subprocess.run([sys.executable, "-c", code], check=True, env=env)


def main():
    name = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    run_one("", "/tmp/vc_main.npy", iters)
    run_one(os.path.join(ROOT, "paper_1302_3120_b200", "variants", f"libcssar_{name}.so"), "/tmp/vc_var.npy", iters)
    a, b = np.load("/tmp/vc_main.npy"), np.load("/tmp/vc_var.npy")
    print(name, "rel-L2 vs main:", float(np.linalg.norm(a - b) / np.linalg.norm(a)))


if __name__ == "__main__":
    main()

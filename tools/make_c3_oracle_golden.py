#!/usr/bin/env python
"""Write tests/golden/c3_oracle_iterates.npz: the fp64 oracle's Algorithm 1 trajectory on the
full c3 configuration (8192 x 8192, 60% azimuth-line mask, soft, k-rule k = 671589, mu = 1,
100 iterations; BASELINE.json configs[3]).

Calls only oracle/ and inputs/ (no CUDA path): the c3 echo is the oracle's inverse-CSA echo
Y = Theta o (G(X_true) + noise), rounded to complex64 by inputs.synth, and the
trajectory is oracle.ita.ita (Algorithm 1; lambda rule P:L314-320) run in three
legs (X is the whole state with a fixed mu, so ita(X0 = X_49, 49 iterations) continues the
same trajectory).  Stored (complex64 values at int32 flat indices of the nonzeros):

  * X_49, X_98 -- inputs of the teacher-forced GPU steps 50 and 99;
  * X_100      -- the oracle's Algorithm 1 output for the full-run parity test;
  * the per-iteration log (sigma, support, ||r||^2, near-tie gap g_i) of all 100 iterations.

Run (about 30-60 min on 8 host cores):  python tools/make_c3_oracle_golden.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import configs, synth  # noqa: E402
from oracle import csa, echo, ita  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c3_oracle_iterates.npz")


def sparse(X):
    idx = np.flatnonzero(X).astype(np.int32)
    return idx, X.reshape(-1)[idx].astype(np.complex64)


def main():
    cfg = configs.get("c3")
    op = csa.CSAOperator(cfg.params)
    t0 = time.time()
    prob = synth.make_problem(cfg, lambda sc, c: echo.inverse_csa_echo(op, sc.dense()))
    print(f"problem {time.time() - t0:.1f} s", flush=True)
    Y = prob.Y.astype(np.complex128)
    log = []
    out = {}
    X = None
    for leg, (n, name) in enumerate(((49, "X49"), (49, "X98"), (2, "X100"))):
        t = time.time()
        X = ita.ita(op, Y, prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=n, X0=X, log=log)
        idx, val = sparse(X)
        out[name + "_idx"], out[name + "_val"] = idx, val
        print(f"{name}: {n} it in {time.time() - t:.1f} s, nnz {idx.size}, sigma {log[-1]['sigma']:.6g}", flush=True)
    for key in ("sigma", "support", "resid2", "gap"):
        out["log_" + key] = np.array([e[key] for e in log])
    out["k"] = np.int64(cfg.k)
    out["iters"] = np.int64(len(log))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 2**20:.1f} MiB) in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()

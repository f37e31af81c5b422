"""NEXT-3: the paper's reconstruction-ability (RA) experiment as a sweep on the GPU.

9 targets 6 samples apart (unit amplitude, random phase), exact echo (eq. 1-3), 20 dB noise,
separable s_a : s_r = 1 : 5 sampling, k = 18, 100 iterations, on a 256 x 256 grid
(config "ra"; the paper's scene is 180 x 180).  Success = the 9 largest |X| sit exactly on
the 9 targets.  The scenes run concurrently through BatchRunner (one plan and stream per
slot).  Checked against the fp64 oracle: X parity on two trials, and the success count of
every sampling rate within one trial of the oracle's.
"""
import time

import numpy as np
import pytest

from inputs import configs, synth
from oracle import csa, ita
from tests._common import mask_bits_dev, need_gpu, oracle_echo, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu
RATES = (0.1, 0.04, 0.02, 0.01, 0.005, 0.002)
TRIALS = 8


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _cfg(rate, trial):
    return configs.get("ra", rate=rate, seed=13023120 + 10 + 7919 * trial + int(round(rate * 1e5)))


def _success(X, scene):
    top = set(np.argsort(-np.abs(np.asarray(X)).ravel())[:9].tolist())
    return top == set(int(i) for i in scene.idx)


def test_ra_trials_match_oracle():
    from paper_1302_3120_b200 import Plan
    for trial in range(2):
        cfg = _cfg(0.1, trial)
        prob = synth.make_problem(cfg, oracle_echo)
        Xo = ita.ita(csa.CSAOperator(cfg.params), prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr,
                     rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=cfg.iters)
        pl = Plan(cfg.params)
        X = to_host(pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule=cfg.rule,
                                   k=cfg.k, mu=cfg.mu, iters=cfg.iters))
        assert rel_l2(X, Xo) <= 1e-3
        assert set(np.flatnonzero(X).tolist()) == set(np.flatnonzero(Xo).tolist())
        assert _success(X, prob.scene) and _success(Xo, prob.scene)


def test_ra_breakdown_sweep_batched():
    import torch
    from paper_1302_3120_b200 import BatchRunner
    probs = [synth.make_problem(_cfg(r, t), oracle_echo) for r in RATES for t in range(TRIALS)]
    cfg = probs[0].cfg
    kw = dict(thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=cfg.iters)
    runner = BatchRunner(cfg.params, slots=16)
    Ys = [torch.from_numpy(p.Y) for p in probs]
    Ms = [torch.from_numpy(p.mask.astype(np.uint8)) for p in probs]
    runner.run(Ys[:16], Ms[:16], **kw)                      # warm-up (graph capture per slot)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Xs = runner.run(Ys, Ms, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    serial = BatchRunner(cfg.params, slots=1)
    serial.run(Ys[:1], Ms[:1], **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Xs1 = serial.run(Ys, Ms, **kw)
    torch.cuda.synchronize()
    dt1 = time.perf_counter() - t0
    assert all(np.array_equal(a.numpy(), b.numpy()) for a, b in zip(Xs, Xs1))   # slots are independent
    op = csa.CSAOperator(cfg.params)
    table = []
    for ri, rate in enumerate(RATES):
        g = o = 0
        for t in range(TRIALS):
            p = probs[ri * TRIALS + t]
            g += _success(Xs[ri * TRIALS + t].numpy(), p.scene)
            Xo = ita.ita(op, p.Y.astype(np.complex128), p.mask, **kw)
            o += _success(Xo, p.scene)
        m = int(np.mean([probs[ri * TRIALS + t].mask.sum() for t in range(TRIALS)]))
        table.append((rate, m, g, o))
    print("\nRA sweep (rate, mean #measurements, GPU successes, oracle successes of %d):" % TRIALS)
    for row in table:
        print("  %.3f %6d %2d %2d" % row)
    print("batched (16 slots): %d scenes x %d iterations in %.3f s (%.1f scenes/s); one slot: %.3f s" %
          (len(probs), cfg.iters, dt, len(probs) / dt, dt1))
    for rate, m, g, o in table:
        assert abs(g - o) <= 1, (rate, g, o)
    assert table[0][2] == TRIALS and table[-1][2] == 0

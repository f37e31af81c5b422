"""Pins for the oracle's thresholds, rules and ITA loop (oracle/ita.py)."""
import json
import os

import numpy as np
import pytest

from inputs import configs, synth
from inputs.configs import SarParams
from oracle import csa, echo, ita

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, seed, scale=1.0):
    r = np.random.default_rng(seed)
    return scale * (r.standard_normal(shape) + 1j * r.standard_normal(shape))


# ---------------------------------------------------------------- thresholds
def test_soft_worked_example_and_identity():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
    out = ita.soft(np.array([3 + 4j]), 2.0)[0]
    assert abs(out - complex(*g["soft_3p4j_sigma2"])) < 1e-15
    b = _rand(100, 1)
    assert np.array_equal(ita.soft(b, 0.0), b)
    assert not np.any(ita.soft(b, np.abs(b).max()))      # strict survival: full kill


def test_soft_nonexpansive():
    """||E(x) - E(z)|| <= ||x - z||."""
    for s in range(20):
        x, z = _rand(200, 2 * s), _rand(200, 2 * s + 1)
        sig = 0.3 + 0.1 * s
        assert np.linalg.norm(ita.soft(x, sig) - ita.soft(z, sig)) <= np.linalg.norm(x - z) + 1e-15


def _brute_half(a, lm):
    """argmin_{t >= 0} (t - a)^2 + lm sqrt(t): dense grid then golden-section refinement."""
    f = lambda t: (t - a) ** 2 + lm * np.sqrt(max(t, 0.0))
    ts = np.linspace(0.0, a, 20001)
    vals = (ts - a) ** 2 + lm * np.sqrt(ts)
    i = int(np.argmin(vals))
    lo, hi = ts[max(i - 1, 0)], ts[min(i + 1, ts.size - 1)]
    gr = (np.sqrt(5) - 1) / 2
    for _ in range(200):
        c, d = hi - gr * (hi - lo), lo + gr * (hi - lo)
        if f(c) < f(d):
            hi = d
        else:
            lo = c
    t = 0.5 * (lo + hi)
    if t > 0:
        # polish: bisection on f'(t) = 2(t - a) + lm / (2 sqrt t), increasing near the minimiser
        df = lambda u: 2.0 * (u - a) + lm / (2.0 * np.sqrt(u))
        lo, hi = max(t - 1e-3 * a, 1e-300), min(t + 1e-3 * a, a)
        if df(lo) < 0 < df(hi):
            for _ in range(200):
                mid = 0.5 * (lo + hi)
                if df(mid) < 0:
                    lo = mid
                else:
                    hi = mid
            t = 0.5 * (lo + hi)
    return 0.0 if f(0.0) <= f(t) else t


def test_half_matches_bruteforce_minimiser():
    """R15: the q=1/2 operator is the exact minimiser of (t - |b|)^2 + lambda mu sqrt(t)."""
    r = np.random.default_rng(5)
    for _ in range(150):
        sigma = r.uniform(0.1, 3.0)
        lm = ita.HALF_LM_PER_SIGMA32 * sigma ** 1.5
        assert ita.half_sigma_from_lm(lm) == pytest.approx(sigma, rel=1e-12)
        a = r.uniform(0.0, 3.0 * sigma)
        if abs(a - sigma) < 1e-3 * sigma:
            continue                      # at the jump both minima tie
        ph = np.exp(1j * r.uniform(0, 2 * np.pi))
        h = ita.half(np.array([a * ph]), sigma)[0]
        t = _brute_half(a, lm)
        assert abs(abs(h) - t) <= 1e-9 * max(1.0, a)
        if t > 0:
            assert abs(np.angle(h / ph)) < 1e-12


def test_half_jump_and_identity():
    s = 1.7
    just = ita.half(np.array([s * (1 + 1e-12)]), s)[0]
    assert abs(just - 2 * s / 3) < 1e-9
    assert ita.half(np.array([s]), s)[0] == 0
    b = _rand(50, 3)
    assert np.array_equal(ita.half(b, 0.0), b)
    g = json.load(open(os.path.join(GOLD, "survey_8c7_anchors.json")))
    assert abs(ita.half(np.array([3 + 4j]), 2.0)[0] - complex(*g["thresholds_3p4j_sigma2"]["half"])) < 1e-11


# ---------------------------------------------------------------- rules
def test_k_rule_worked_examples():
    """SPEC S:L365-366 restating P:L316-320."""
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
    b = np.array(g["k_rule_mags"], dtype=complex) * np.exp(1j * np.arange(5))
    sig = ita.sigma_k_rule(b, g["k_rule_k"])
    assert sig == pytest.approx(g["k_rule_sigma"], rel=1e-14)
    assert np.count_nonzero(ita.soft(b, sig)) == g["k_rule_survivors"]
    eq = np.full(7, 2.0 + 0j)
    assert np.count_nonzero(ita.soft(eq, ita.sigma_k_rule(eq, 3))) == 0     # ties killed
    bb = _rand(30, 9)
    assert ita.sigma_k_rule(bb, 29) == pytest.approx(np.abs(bb).min())      # k = n - 1 boundary
    with pytest.raises(ValueError):
        ita.sigma_k_rule(bb, 30)
    with pytest.raises(ValueError):
        ita.sigma_k_rule(bb, 0)


# ---------------------------------------------------------------- ITA loop
def test_ita_full_sampling_one_step_fixed_point():
    """Theta = 1 and G unitary: every iterate equals E(M Y; sigma(M Y)) (closed form)."""
    p = SarParams(n_az=64, n_rg=64)
    op = csa.CSAOperator(p)
    Y = _rand(op.shape, 11)
    m = np.ones(op.shape)
    k = 40
    b = op.M(Y)
    ref = ita.soft(b, ita.sigma_k_rule(b, k))
    for it in (1, 2, 5):
        X = ita.ita(op, Y, m, thr="soft", rule="k", k=k, iters=it)
        assert np.max(np.abs(X - ref)) <= 1e-12 * np.max(np.abs(ref))
    Xh = ita.ita(op, Y, m, thr="half", rule="k", k=k, iters=3)
    refh = ita.half(b, ita.sigma_k_rule(b, k))
    assert np.max(np.abs(Xh - refh)) <= 1e-12 * np.max(np.abs(refh))


def test_ita_zero_input():
    p = SarParams(n_az=32, n_rg=32)
    op = csa.CSAOperator(p)
    X = ita.ita(op, np.zeros(op.shape), np.ones(op.shape), rule="lambda", lam=0.1, iters=3)
    assert not np.any(X)


def test_ita_fixed_lambda_objective_monotone():
    """ISTA with mu <= 1/||A||^2 = 1 decreases F = 1/2||Theta(Y - GX)||^2 + lambda||X||_1 (R11, R12)."""
    p = SarParams(n_az=64, n_rg=64)
    op = csa.CSAOperator(p)
    r = np.random.default_rng(2)
    X0 = np.zeros(op.shape, complex)
    X0.reshape(-1)[r.choice(X0.size, 30, replace=False)] = np.exp(2j * np.pi * r.random(30)) * 5
    m = (r.random(op.shape) < 0.5).astype(float)
    Y = m * (op.G(X0) + 0.05 * _rand(op.shape, 3))
    for lam in (0.3, 1.0):
        X = np.zeros(op.shape, complex)
        F = [ita.objective_soft(op, X, Y, m, lam)]
        for _ in range(15):
            X = ita.ita(op, Y, m, thr="soft", rule="lambda", lam=lam, mu=1.0, iters=1, X0=X)
            F.append(ita.objective_soft(op, X, Y, m, lam))
        assert all(F[i + 1] <= F[i] * (1 + 1e-12) for i in range(len(F) - 1)), F


def test_ita_support_bound_every_iteration():
    p = SarParams(n_az=64, n_rg=64)
    op = csa.CSAOperator(p)
    Y = _rand(op.shape, 21)
    m = (np.random.default_rng(1).random(op.shape) < 0.3).astype(float)
    log = []
    ita.ita(op, Y * m, m, thr="half", rule="k", k=25, iters=8, log=log)
    assert all(e["support"] <= 25 for e in log)


def test_ita_recovers_c0_support():
    """c0 physics: 5 point targets, 50% mask, 30 dB -> exact support, wide gap."""
    cfg = configs.get("c0")
    prob = synth.make_problem(cfg, lambda sc, c: echo.exact_echo(c.params, sc.targets))
    op = csa.CSAOperator(cfg.params)
    log = []
    X = ita.ita(op, prob.Y, prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=cfg.iters, log=log)
    supp = set(np.flatnonzero(X).tolist())
    assert supp == set(prob.scene.idx.tolist())
    assert min(e["gap"] for e in log) > 1.0
    assert log[-1]["resid2"] < log[0]["resid2"]


# ---------------------------------------------------------------- adaptive step (NEXT-1, eq. 27)
def _dense_A(op, mask):
    """A = Theta o G as an explicit matrix over vec(X) (columns = G of the basis images)."""
    n_az, n_rg = op.shape
    n = n_az * n_rg
    A = np.zeros((n, n), np.complex128)
    for j in range(n):
        e = np.zeros(n, np.complex128)
        e[j] = 1.0
        A[:, j] = (np.asarray(mask, dtype=float) * op.G(e.reshape(n_az, n_rg))).reshape(-1)
    return A


def test_adaptive_mu_matches_dense_matrix_ratio():
    """mu = ||v||^2 / ||A v||^2 for v = dX on supp(X), A the explicit (brute-force) matrix."""
    p = SarParams(n_az=8, n_rg=16)
    op = csa.CSAOperator(p)
    mask = (np.random.default_rng(3).random((8, 16)) < 0.5).astype(float)
    A = _dense_A(op, mask)
    X = np.zeros((8, 16), np.complex128)
    X.reshape(-1)[[3, 17, 40, 41, 99]] = _rand(5, 4)
    dX = _rand((8, 16), 5)
    v = np.where(X != 0, dX, 0).reshape(-1)
    ref = np.vdot(v, v).real / np.vdot(A @ v, A @ v).real
    assert abs(ita.adaptive_mu(op, dX, X, mask) - ref) <= 1e-12 * ref


def test_adaptive_mu_bounds_and_special_cases():
    """G unitary => ||Theta G v|| <= ||v||: mu >= 1, with equality at Theta = 1; an empty
    support (X = 0, the first iteration of Algorithm 1) gives mu = 1."""
    p = SarParams(n_az=32, n_rg=32)
    op = csa.CSAOperator(p)
    X = np.zeros((32, 32), np.complex128)
    X.reshape(-1)[np.random.default_rng(6).choice(1024, 60, replace=False)] = 1.0 + 0.5j
    dX = _rand((32, 32), 7)
    assert abs(ita.adaptive_mu(op, dX, X, np.ones((32, 32))) - 1.0) <= 1e-12
    for rate in (0.3, 0.6, 0.9):
        mask = (np.random.default_rng(int(rate * 10)).random((32, 32)) < rate).astype(float)
        assert ita.adaptive_mu(op, dX, X, mask) >= 1.0 - 1e-12
    assert ita.adaptive_mu(op, dX, np.zeros((32, 32)), mask) == 1.0


def test_adaptive_ita_equals_fixed_step_at_full_sampling():
    """Theta = 1: every mu_i is 1, so the adaptive run reproduces mu = 1 (closed form)."""
    cfg = configs.get("c0")
    prob = synth.make_problem(cfg, lambda s, c: echo.exact_echo(c.params, s.targets))
    op = csa.CSAOperator(cfg.params)
    full = np.ones(prob.mask.shape)
    Y = prob.Y.astype(np.complex128)
    log = []
    Xa = ita.ita(op, Y, full, thr="soft", rule="k", k=cfg.k, mu="adaptive", iters=4, log=log)
    Xf = ita.ita(op, Y, full, thr="soft", rule="k", k=cfg.k, mu=1.0, iters=4)
    assert all(abs(e["mu"] - 1.0) <= 1e-12 for e in log)
    assert np.max(np.abs(Xa - Xf)) <= 1e-12 * np.max(np.abs(Xf))


# ---------------------------------------------------------------- q = 0 and q = 2/3 (NEXT-4)
def test_hard_threshold_keeps_exactly_the_top_k():
    b = _rand(4000, 11)
    k = 137
    sig = ita.sigma_k_rule(b, k)
    X = ita.hard(b, sig)
    assert np.count_nonzero(X) == k
    keep = np.argsort(-np.abs(b))[:k]
    assert np.array_equal(X[keep], b[keep])
    assert np.array_equal(ita.hard(b, 0.0), b)


def test_fixed_lambda_sigma_is_the_bruteforce_jump_point():
    """Fixed-lambda rule (eq. 7; q = 0, 1/2, 1, 2/3 of P:L102): sigma_fixed_lambda is
    the smallest |b| whose scalar minimiser argmin_{x>=0} (x - t)^2 + lm pen(x) is nonzero,
    found here by brute force on dense t and x grids, with the penalty normalisation of each
    operator's k-rule form (soft: 2 lm |x|, i.e. the 1/2 ||.||^2 scaling of R12; hard: lm 1[x != 0];
    half: lm sqrt(x); 2/3: lm x^(2/3)) -- and lambda_from_sigma inverts it."""
    pens = {"soft": lambda x, lm: 2.0 * lm * x, "hard": lambda x, lm: lm * (x > 0),
            "half": lambda x, lm: lm * np.sqrt(x), "twothirds": lambda x, lm: lm * x ** (2.0 / 3.0)}
    x = np.linspace(0.0, 6.0, 60001)
    for thr, pen in pens.items():
        for lam, mu in ((0.7, 1.0), (1.9, 0.6), (3.1, 1.3)):
            lm = lam * mu
            sig = ita.sigma_fixed_lambda(lam, mu, thr)
            assert ita.lambda_from_sigma(sig, mu, thr) == pytest.approx(lam, rel=1e-12)
            ts = np.linspace(0.2 * sig, 1.8 * sig, 1601)
            nz = []
            for t in ts:
                xs = x[np.argmin((x - t) ** 2 + pen(x, lm))]
                nz.append(xs > 1e-9)
            jump = ts[np.argmax(nz)]
            assert abs(jump - sig) <= 2.0 * (ts[1] - ts[0]), (thr, lam, mu, jump, sig)


def test_order_statistic_matches_rank_counting():
    """|b|_(k) against a brute-force rank count: the value v with
    #{|b| > v} < k <= #{|b| >= v}, on data with ties and zeros."""
    r = np.random.default_rng(5)
    a = np.round(r.random(3000) * 50) / 7.0          # many ties
    a[:300] = 0.0
    b = a * np.exp(1j * r.random(3000))
    mags = np.abs(b)
    for k in (1, 2, 17, 299, 1500, 2699, 2700, 2701, 3000):
        v = ita.kth_largest_mag(b, k)
        assert np.count_nonzero(mags > v) < k <= np.count_nonzero(mags >= v), k


def test_twothirds_matches_bruteforce_minimiser():
    """argmin_{x>=0} (x - t)^2 + lm x^(2/3) by a dense grid, lm from the k-rule sigma."""
    for sigma in (0.3, 1.0, 2.5):
        lm = ita.twothirds_lm_from_sigma(sigma)
        assert abs((2.0 / 3.0) * (3.0 * lm ** 3) ** 0.25 - sigma) <= 1e-12 * sigma
        for t in (0.9 * sigma, 1.0001 * sigma, 1.3 * sigma, 2.0 * sigma, 6.0 * sigma):
            x = np.linspace(0.0, 2.0 * t, 400001)
            ref = x[np.argmin((x - t) ** 2 + lm * x ** (2.0 / 3.0))]
            got = abs(ita.twothirds(np.array([t * np.exp(0.3j)]), sigma)[0])
            assert abs(got - ref) <= 2.0 * (x[1] - x[0]) + 1e-12, (sigma, t, got, ref)


def test_twothirds_jump_phase_and_identity():
    sigma = 1.7
    b = np.array([sigma * (1 + 1e-9) * np.exp(1.1j), 0.5 * sigma * np.exp(-2j)])
    X = ita.twothirds(b, sigma)
    assert abs(abs(X[0]) - sigma / 2.0) <= 1e-6 * sigma           # jumps from 0 to sigma/2
    assert abs(np.angle(X[0]) - 1.1) <= 1e-12 and X[1] == 0
    assert np.array_equal(ita.twothirds(b, 0.0), b)


# ---- tolerance stopping (NEXT-4)
def test_tol_stop_zero_echo_stops_after_one_update():
    """y_s = 0 -> X* = 0 after one iteration (||X_1 - X_0|| = 0 <= tol * 0)."""
    from inputs.configs import SarParams
    from oracle import csa, ita
    p = SarParams(n_az=128, n_rg=128)
    info = {}
    X = ita.ita(csa.CSAOperator(p), np.zeros((128, 128)), np.ones((128, 128)), k=5, iters=50, tol=1e-6, info=info)
    assert info["iters"] == 1 and not np.any(X)


def test_tol_stop_is_the_first_small_relative_change():
    """The stop iteration equals the first update whose relative change, computed here from
    separate fixed-count runs, is <= tol; the returned X is that update's."""
    from inputs import configs, synth
    from oracle import csa, ita
    from tests._common import oracle_echo
    cfg = configs.get("c0")
    prob = synth.make_problem(cfg, oracle_echo)
    op = csa.CSAOperator(cfg.params)
    kw = dict(thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu)
    Xs = [np.zeros(prob.Y.shape, np.complex128)] + [ita.ita(op, prob.Y, prob.mask, iters=j, **kw) for j in range(1, 13)]
    r = [np.linalg.norm(Xs[j] - Xs[j - 1]) / max(np.linalg.norm(Xs[j - 1]), 1e-300) for j in range(1, 13)]
    j = next(j for j in range(3, 12) if r[j - 1] < 0.8 * min(r[:j - 1]))      # a strict new minimum
    tol = float(np.sqrt(r[j - 1] * min(r[:j - 1])))
    info = {}
    X = ita.ita(op, prob.Y, prob.mask, iters=40, tol=tol, info=info, **kw)
    assert info["iters"] == j
    assert np.array_equal(X, Xs[j])
    info0 = {}
    assert np.array_equal(ita.ita(op, prob.Y, prob.mask, iters=7, tol=0.0, info=info0, **kw), Xs[7])
    assert info0["iters"] == 7

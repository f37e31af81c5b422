"""ITA parity (cssar_ita_iterate) against the fp64 oracle (oracle/ita.py), same seeded inputs.

North star: rel-L2 <= 1e-3 on X after the full iteration count; recovered support identical
on the point-target configs (c0, c1).  Also: teacher-forced single iterations, the fixed-
lambda rule, exactness of the k-rule select against a sort of the GPU's own |b|^2, resume,
and the degenerate inputs.
"""
import numpy as np
import pytest

from inputs import configs
from oracle import csa, ita
from tests._common import mag2_f32, mask_bits_dev, need_gpu, oracle_op, problem, rand_c, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL_ITA = 1e-3


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _plan(p):
    from paper_1302_3120_b200 import Plan
    return Plan(p)


def _run_both(prob, iters=None, rule=None, lam=None):
    cfg = prob.cfg
    iters = cfg.iters if iters is None else iters
    rule = cfg.rule if rule is None else rule
    op = csa.CSAOperator(cfg.params)
    olog = []
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr, rule=rule, k=cfg.k,
                 lam=lam, mu=cfg.mu, iters=iters, log=olog)
    pl = _plan(cfg.params)
    Xg, glog = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule=rule, k=cfg.k,
                              lam=lam or 0.0, mu=cfg.mu, iters=iters, log=True)
    return Xo, olog, to_host(Xg), glog, pl


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_ita_point_target_configs_full_run(name):
    prob = problem(name)
    Xo, olog, Xg, glog, _ = _run_both(prob)
    assert rel_l2(Xg, Xo) <= TOL_ITA
    so, sg = set(np.flatnonzero(Xo).tolist()), set(np.flatnonzero(Xg).tolist())
    assert sg == so, (len(so), len(sg), len(so ^ sg))
    k = prob.cfg.k
    assert all(e["support"] <= k for e in glog)
    s_o = np.array([e["sigma"] for e in olog])
    s_g = np.array([e["sigma"] for e in glog])
    assert np.max(np.abs(s_g - s_o) / s_o) <= 1e-4
    r_o = np.array([e["resid2"] for e in olog])
    r_g = np.array([e["resid2"] for e in glog])
    assert np.max(np.abs(r_g - r_o) / r_o) <= 1e-4
    if name == "c0":
        assert sg == set(prob.scene.idx.tolist())      # physics: the 5 truth pixels


def test_ita_c2_full_run():
    """c2 (2048 x 2048 Thomas clusters, 30% mask, soft, k = 2%): the config's full 200
    iterations vs the oracle (north star: rel-L2 <= 1e-3 on X after the full count); sigma
    and residual logs within 1e-4 at every iteration."""
    prob = problem("c2")
    Xo, olog, Xg, glog, _ = _run_both(prob)
    assert len(glog) == prob.cfg.iters == 200
    assert rel_l2(Xg, Xo) <= TOL_ITA
    s_o = np.array([e["sigma"] for e in olog])
    s_g = np.array([e["sigma"] for e in glog])
    assert np.max(np.abs(s_g - s_o) / s_o) <= 1e-4
    assert all(e["support"] <= prob.cfg.k for e in glog)


def test_ita_c4_full_size_properties():
    """c4 (32768 x 16384, 120 MHz, 50% mask, k = 0.5%) at full size, 4 iterations: properties
    that hold at any size — finite, support <= k every iteration, the residual decreases
    (mu = 1 <= 1/||A||^2), X is exactly k-sparse-or-less, and 2 + 2 resumed iterations
    reproduce 4 bitwise."""
    import torch
    cfg = configs.get("c4")
    p = cfg.params
    pl = _plan(p)
    g = torch.Generator(device="cuda").manual_seed(44)
    m = (torch.rand((p.n_az, p.n_rg), device="cuda", generator=g) < 0.5)
    from paper_1302_3120_b200 import pack_mask
    mb = pack_mask(m.to(torch.uint8))
    Y = torch.randn((p.n_az, p.n_rg), dtype=torch.complex64, device="cuda", generator=g)
    Y = torch.where(m, Y, torch.zeros_like(Y))
    del m
    X, log = pl.ita_iterate(Y, mb, thr="soft", rule="k", k=cfg.k, iters=4, log=True)
    r = [e["resid2"] for e in log]
    assert all(np.isfinite(r)) and r[-1] < r[0]
    assert all(e["support"] <= cfg.k for e in log)
    assert int(torch.count_nonzero(X).item()) <= cfg.k
    X2 = pl.ita_iterate(Y, mb, thr="soft", rule="k", k=cfg.k, iters=2)
    X3 = pl.ita_iterate(Y, mb, thr="soft", rule="k", k=cfg.k, iters=2, X=X2.clone())
    del X2
    X4 = pl.ita_iterate(Y, mb, thr="soft", rule="k", k=cfg.k, iters=4)
    assert torch.equal(X3.view(torch.float32), X4.view(torch.float32))


def test_ita_teacher_forced_step():
    """One GPU iteration from the oracle's X_5 (rounded to complex64) vs the oracle's X_6,
    excluding pixels whose oracle |b_5| lies within 1e-5 sigma_5 of sigma_5 (near ties)."""
    prob = problem("c1")
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    Y = prob.Y.astype(np.complex128)
    X5 = ita.ita(op, Y, prob.mask, thr=cfg.thr, rule="k", k=cfg.k, iters=5)
    X5c = X5.astype(np.complex64)
    R = prob.mask * (Y - op.G(X5c.astype(np.complex128)))
    b = X5c.astype(np.complex128) + cfg.mu * op.M(R)
    sig = ita.sigma_k_rule(b, cfg.k)
    X6 = ita.threshold(b, sig, cfg.thr)
    pl = _plan(cfg.params)
    Xg, glog = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule="k", k=cfg.k,
                              iters=1, X=to_dev(X5c), log=True)
    Xg = to_host(Xg)
    near = np.abs(np.abs(b) - sig) <= 1e-5 * sig
    assert abs(glog[0]["sigma"] - sig) / sig <= 1e-5
    keep = ~near
    assert rel_l2(Xg[keep], X6[keep]) <= 1e-4


def test_ita_fixed_lambda_rule():
    prob = problem("c0")
    Xo, olog, Xg, glog, _ = _run_both(prob, iters=20, rule="lambda", lam=60.0)
    assert rel_l2(Xg, Xo) <= TOL_ITA
    assert [e["support"] for e in glog] == [e["support"] for e in olog]


def test_ita_c3_full_size_one_iteration():
    """c3 (8192 x 8192, line mask 60%, k = 671589): one iteration from X = 0 vs the oracle,
    plus properties of a few more GPU iterations (support <= k, residual decreasing)."""
    prob = problem("c3")
    cfg = prob.cfg
    op = oracle_op(cfg.params)
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr="soft", rule="k", k=cfg.k, iters=1)
    pl = _plan(cfg.params)
    mb = mask_bits_dev(prob.mask)
    Yd = to_dev(prob.Y)
    Xg = pl.ita_iterate(Yd, mb, thr="soft", rule="k", k=cfg.k, iters=1)
    assert rel_l2(to_host(Xg), Xo) <= TOL_ITA
    del Xo
    _, glog = pl.ita_iterate(Yd, mb, thr="soft", rule="k", k=cfg.k, iters=4, log=True)
    assert all(e["support"] <= cfg.k for e in glog)
    assert glog[-1]["resid2"] < glog[0]["resid2"]


@pytest.mark.parametrize("shape,k", [((256, 256), 1), ((256, 256), 700), ((256, 256), 65534),
                                     ((2048, 2048), 83886), ((1024, 512), 5000)])
def test_select_exact_against_sort(shape, k):
    import torch
    from paper_1302_3120_b200 import Plan
    from inputs.configs import SarParams
    b = rand_c(shape, k)
    # ties and zeros: duplicate a block of values, zero another
    b.reshape(-1)[:200] = b.reshape(-1)[200:400]
    b.reshape(-1)[400:900] = 0
    pl = Plan(SarParams(n_az=shape[0], n_rg=shape[1]))
    s2, above = pl.debug_select(to_dev(b), k)
    m = np.sort(mag2_f32(b).reshape(-1))[::-1]
    ref = m[k].view(np.uint32)                       # (k+1)-th largest pattern
    assert s2 == int(ref)
    assert above == int(np.count_nonzero(m > m[k]))


def test_ita_resume_is_bitwise_identical():
    prob = problem("c0")
    cfg = prob.cfg
    pl = _plan(cfg.params)
    Yd, mb = to_dev(prob.Y), mask_bits_dev(prob.mask)
    a = pl.ita_iterate(Yd, mb, thr="soft", rule="k", k=cfg.k, iters=6)
    import torch
    X = torch.zeros_like(Yd)
    pl.ita_iterate(Yd, mb, thr="soft", rule="k", k=cfg.k, iters=3, X=X)
    pl.ita_iterate(Yd, mb, thr="soft", rule="k", k=cfg.k, iters=3, X=X)
    assert np.array_equal(to_host(a), to_host(X))


def test_ita_zero_echo_and_nonfinite():
    import torch
    from paper_1302_3120_b200 import CssarError
    from inputs.configs import SarParams
    pl = _plan(SarParams(n_az=128, n_rg=128))
    Y = torch.zeros((128, 128), dtype=torch.complex64, device="cuda")
    X = pl.ita_iterate(Y, None, thr="soft", rule="k", k=5, iters=3)
    assert not torch.any(X != 0).item()
    Y[3, 4] = float("nan")
    with pytest.raises(CssarError) as e:
        pl.ita_iterate(Y, None, thr="soft", rule="k", k=5, iters=2, log=True)
    assert e.value.code == -6
    # without a log: reported by cssar_ita_status (the binding checks it unless check=False)
    with pytest.raises(CssarError) as e:
        pl.ita_iterate(Y, None, thr="soft", rule="k", k=5, iters=2)
    assert e.value.code == -6
    pl.ita_iterate(Y, None, thr="soft", rule="k", k=5, iters=2, check=False)
    with pytest.raises(CssarError) as e:
        pl.status()
    assert e.value.code == -6
    # a clean solve afterwards reports OK again; and on a cluster-shape grid (n_az = 2048)
    Y[3, 4] = 0.0
    pl.ita_iterate(Y, None, thr="soft", rule="k", k=5, iters=2)
    pl2 = _plan(SarParams(n_az=2048, n_rg=256))
    Y2 = torch.zeros((2048, 256), dtype=torch.complex64, device="cuda")
    Y2[100, 7] = float("inf")
    with pytest.raises(CssarError) as e:
        pl2.ita_iterate(Y2, None, thr="soft", rule="k", k=50, iters=2)
    assert e.value.code == -6


def test_ita_fallback_only_when_window_misses():
    """After the first iteration the select should mostly hit the speculative candidate window."""
    prob = problem("c1")
    cfg = prob.cfg
    pl = _plan(cfg.params)
    pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule="k", k=cfg.k, iters=30)
    fb = pl.debug_fallbacks()
    assert 1 <= fb <= 10, fb


@pytest.mark.parametrize("name,iters", [("c0", 30), ("c1", 40)])
def test_ita_adaptive_step_matches_oracle(name, iters):
    """NEXT-1: the eq. 27 step rule (CSSAR_FLAG_ADAPTIVE_MU) vs the oracle's adaptive_mu:
    X after the run (rel-L2 <= 1e-3), identical support, mu_i and sigma_i logs within 1e-4."""
    prob = problem(name)
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    olog = []
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr, rule="k", k=cfg.k, mu="adaptive",
                 iters=iters, log=olog)
    pl = _plan(cfg.params)
    Xg, glog = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule="k", k=cfg.k,
                              mu="adaptive", iters=iters, log=True)
    Xg = to_host(Xg)
    assert rel_l2(Xg, Xo) <= TOL_ITA
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())
    mo = np.array([e["mu"] for e in olog])
    mg = np.array([e["mu"] for e in glog])
    assert mo[0] == 1.0 and mg[0] == 1.0                  # empty support of X_0
    assert np.all(mg >= 1.0 - 1e-6)                       # G unitary => mu_i >= 1
    assert np.max(np.abs(mg - mo) / mo) <= 1e-4
    so = np.array([e["sigma"] for e in olog])
    sg = np.array([e["sigma"] for e in glog])
    assert np.max(np.abs(sg - so) / so) <= 1e-4


def test_ita_adaptive_step_fixed_lambda():
    prob = problem("c0")
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    olog = []
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr="soft", rule="lambda", lam=60.0, mu="adaptive",
                 iters=15, log=olog)
    pl = _plan(cfg.params)
    Xg, glog = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr="soft", rule="lambda", lam=60.0,
                              mu="adaptive", iters=15, log=True)
    assert rel_l2(to_host(Xg), Xo) <= TOL_ITA
    assert [e["support"] for e in glog] == [e["support"] for e in olog]
    assert np.max(np.abs(np.array([e["mu"] for e in glog]) - np.array([e["mu"] for e in olog]))) <= 1e-4


@pytest.mark.parametrize("name,thr,iters", [("c0", "hard", 30), ("c1", "hard", 40), ("c0", "twothirds", 30),
                                            ("c1", "twothirds", 40)])
def test_ita_q0_and_q23_thresholds(name, thr, iters):
    """NEXT-4: hard (q = 0) and q = 2/3 thresholds, k-rule, vs the oracle: X (rel-L2), support,
    sigma logs; hard keeps exactly k pixels when no ties."""
    prob = problem(name)
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    olog = []
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=thr, rule="k", k=cfg.k, iters=iters, log=olog)
    pl = _plan(cfg.params)
    Xg, glog = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=thr, rule="k", k=cfg.k, iters=iters,
                              log=True)
    Xg = to_host(Xg)
    assert rel_l2(Xg, Xo) <= TOL_ITA
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())
    so = np.array([e["sigma"] for e in olog])
    sg = np.array([e["sigma"] for e in glog])
    assert np.max(np.abs(sg - so) / so) <= 1e-4
    lo = np.array([e["lam"] for e in olog])
    lg = np.array([e["lam"] for e in glog])
    assert np.max(np.abs(lg - lo) / lo) <= 1e-3
    if thr == "hard":
        assert np.count_nonzero(Xg) == cfg.k


def test_ita_fixed_lambda_hard_and_twothirds():
    prob = problem("c0")
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    for thr, lam in (("hard", 3000.0), ("twothirds", 400.0)):
        olog = []
        Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=thr, rule="lambda", lam=lam, iters=15, log=olog)
        pl = _plan(cfg.params)
        Xg, glog = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=thr, rule="lambda", lam=lam,
                                  iters=15, log=True)
        assert rel_l2(to_host(Xg), Xo) <= TOL_ITA, thr
        assert [e["support"] for e in glog] == [e["support"] for e in olog], thr


@pytest.mark.parametrize("name,op", [("c0", "csa"), ("c1", "csa"), ("c1", "rda")])
def test_ita_tolerance_stop_matches_oracle(name, op):
    """NEXT-4: the GPU stops at the same update as the oracle.  tol is placed between
    the oracle's relative change at the stop update and every earlier one (>= 10% margins)."""
    from oracle import rda
    from paper_1302_3120_b200 import Plan
    prob = problem(name)
    cfg = prob.cfg
    O = csa.CSAOperator(cfg.params) if op == "csa" else rda.RDAOperator(cfg.params)
    kw = dict(thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu)
    Y = prob.Y.astype(np.complex128)
    Xs = [np.zeros(Y.shape, np.complex128)] + [ita.ita(O, Y, prob.mask, iters=j, **kw) for j in range(1, 15)]
    r = [np.linalg.norm(Xs[j] - Xs[j - 1]) / max(np.linalg.norm(Xs[j - 1]), 1e-300) for j in range(1, 15)]
    j = next(j for j in range(3, 15) if r[j - 1] < 0.8 * min(r[:j - 1]))
    tol = float(np.sqrt(r[j - 1] * min(r[:j - 1])))
    pl = Plan(cfg.params, op=op)
    X, log = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), iters=50, tol=tol, log=True, **kw)
    assert pl.iters_done == j and len(log) == j
    Xg = to_host(X)
    assert rel_l2(Xg, Xs[j]) <= 1e-3
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xs[j]).tolist())
    # tol = 0 runs the cap; Y = 0 stops after one update with X = 0
    pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), iters=4, **kw)
    assert pl.iters_done == 4
    import torch
    Z = torch.zeros_like(to_dev(prob.Y))
    X0 = pl.ita_iterate(Z, mask_bits_dev(prob.mask), iters=30, tol=1e-6, **kw)
    assert pl.iters_done == 1 and not torch.any(X0)


@pytest.mark.parametrize("n_az,n_rg,op", [(4096, 256, "csa"), (16384, 128, "csa"), (16384, 128, "rda"),
                                          (8192, 512, "rda"), (32768, 128, "csa")])
def test_ita_tall_grids_every_cluster_shape(n_az, n_rg, op):
    """Azimuth lengths whose sweeps use 4- and 16-CTA clusters (n_az 4096, 16384, and c4's
    32768 with its 64 KB stages at one CTA per SM) and the c3 shape's (8192) through the
    residual and tail kernels (stage / receive ping-pong), 4 iterations of the c2 recipe vs the
    oracle."""
    from oracle import rda
    from paper_1302_3120_b200 import Plan
    prob = problem("c2", n_az, n_rg)
    cfg = prob.cfg
    O = csa.CSAOperator(cfg.params) if op == "csa" else rda.RDAOperator(cfg.params)
    Xo = ita.ita(O, prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu,
                 iters=4)
    Xg = to_host(Plan(cfg.params, op=op).ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr,
                                                       rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=4))
    assert rel_l2(Xg, Xo) <= TOL_ITA


@pytest.mark.parametrize("mode", ["k", "adaptive_k", "adaptive_lambda"])
def test_ita_runs_are_bitwise_deterministic(mode):
    """SURVEY 5 (race detection): two runs give bitwise identical X and logs -- the histogram
    atomics count integers, and every floating-point reduction (||r||^2, and the adaptive
    step's ||dX_k||^2 / ||Theta G dX_k||^2 that decide mu_i and, with a fixed lambda, sigma_i)
    is summed in a fixed block order.  c2 (2048 x 2048) runs the cluster kernels."""
    prob = problem("c2", iters=6) if mode == "k" else problem("c1", iters=8)
    cfg = prob.cfg
    kw = dict(thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=prob.cfg.iters)
    if mode == "adaptive_k":
        kw.update(mu="adaptive")
    elif mode == "adaptive_lambda":
        kw.update(mu="adaptive", rule="lambda", lam=0.5)
    out = []
    for _ in range(2):
        pl = _plan(cfg.params)
        X, log = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), log=True, **kw)
        out.append((to_host(X), [(e["sigma"], e["support"], e["resid2"], e["mu"]) for e in log]))
    assert np.array_equal(out[0][0].view(np.uint32), out[1][0].view(np.uint32))
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("shape,iters", [((2048, 2048), 40), ((4096, 512), 12), ((8192, 1024), 12),
                                         ((16384, 256), 8), ((32768, 256), 6)])
def test_sparse_state_schedule_is_bitwise_the_dense_schedule(shape, iters):
    """NEXT-3 sparse-state schedule (S5 writes the per-panel list of b entries at or above the
    select window, S1 and the next S5 read it; include/cssar.h): the same arithmetic as the dense
    schedule, so X and the sigma / support / residual logs are bitwise equal -- through the early
    iterations' select fallbacks (dense S5 re-run + list rebuild) and every cluster shape
    (n_az 2048 .. 32768, VEC and per-element epilogues).  c2 uses its recipe (2% Thomas clusters,
    30% mask); the tall grids a random 50% masked echo with k = 1%."""
    import torch
    from paper_1302_3120_b200 import Plan, pack_mask
    from inputs.configs import SarParams
    if shape == (2048, 2048):
        prob = problem("c2")
        cfg = prob.cfg
        p, k = cfg.params, cfg.k
        Y, mb = to_dev(prob.Y), mask_bits_dev(prob.mask)
    else:
        p = SarParams(n_az=shape[0], n_rg=shape[1])
        g = torch.Generator(device="cuda").manual_seed(7)
        m = torch.rand(shape, device="cuda", generator=g) < 0.5
        Y = torch.randn(shape, dtype=torch.complex64, device="cuda", generator=g)
        Y = torch.where(m, Y, torch.zeros_like(Y))
        mb = pack_mask(m.to(torch.uint8))
        k = shape[0] * shape[1] // 100
    out = []
    for sparse in (False, True):
        pl = Plan(p)
        X, log = pl.ita_iterate(Y, mb, thr="soft", rule="k", k=k, iters=iters, log=True, sparse_state=sparse)
        out.append((to_host(X), [(e["sigma"], e["support"], e["resid2"]) for e in log], pl.debug_fallbacks()))
    assert np.array_equal(out[0][0].view(np.uint32), out[1][0].view(np.uint32))
    assert out[0][1] == out[1][1]
    assert out[0][2] == out[1][2] and out[1][2] >= 1      # the fallback path ran (iteration 0 at least)


@pytest.mark.parametrize("name,iters", [("c0", 20), ("c1", 30), ("c2", 30)])
def test_fixed_lambda_fused_schedule(name, iters):
    """Fixed-lambda rule (eq. 7): the fused S5 + next-S1 sweep (AZ_FUSE, CSSAR_FLAG_FUSE_LAMBDA)
    vs the unfused schedule (the same iterates up to floating-point order: <= 1e-5) and, for the
    soft threshold (continuous, so boundary pixels cannot jump), vs the fp64 oracle (rel-L2 <=
    1e-3, support logs within a few pixels).  lambda: 1.01 x the sigma a short k-rule run
    reaches (away from that run's order statistic)."""
    prob = problem(name)
    cfg = prob.cfg
    pl = _plan(cfg.params)
    Yd, mb = to_dev(prob.Y), mask_bits_dev(prob.mask)
    _, klog = pl.ita_iterate(Yd, mb, thr=cfg.thr, rule="k", k=cfg.k, mu=cfg.mu, iters=10, log=True)
    lam = ita.lambda_from_sigma(1.01 * klog[-1]["sigma"], cfg.mu, cfg.thr)
    Xf, lf = pl.ita_iterate(Yd, mb, thr=cfg.thr, rule="lambda", lam=lam, mu=cfg.mu, iters=iters, log=True,
                            fuse_lambda=True)
    Xu, lu = pl.ita_iterate(Yd, mb, thr=cfg.thr, rule="lambda", lam=lam, mu=cfg.mu, iters=iters, log=True)
    Xf, Xu = to_host(Xf), to_host(Xu)
    assert rel_l2(Xf, Xu) <= 1e-5
    # the fused sweep's other FFT factorisation may flip a pixel whose |b| is within rounding of sigma
    assert max(abs(a["support"] - b["support"]) for a, b in zip(lf, lu)) <= 2
    if cfg.thr != "soft":
        return
    op = oracle_op(cfg.params)
    olog = []
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr, rule="lambda", lam=lam, mu=cfg.mu,
                 iters=iters, log=olog)
    assert rel_l2(Xf, Xo) <= TOL_ITA
    so = np.array([e["support"] for e in olog])
    sf = np.array([e["support"] for e in lf])
    assert np.max(np.abs(sf - so)) <= max(2, 1e-4 * cfg.k)
    ro = np.array([e["resid2"] for e in olog])
    assert np.max(np.abs(np.array([e["resid2"] for e in lf]) - ro) / ro) <= 1e-4


@pytest.mark.parametrize("k", [100, 700000, 2000000])
def test_select_exact_when_the_candidate_list_overflows(k):
    """A flat |b| (1.5 M equal values in one histogram bin of a 2048^2 grid, more than the
    n/8 + 64k candidate capacity) makes the fallback's candidate list overflow; the select then
    counts its two 10-bit radix levels over b itself and stays exact (advisor finding r1)."""
    from paper_1302_3120_b200 import Plan
    from inputs.configs import SarParams
    shape = (2048, 2048)
    b = rand_c(shape, 31)
    flat = b.reshape(-1)
    flat[1000:1501000] = np.complex64(0.6 + 0.8j)          # |b| = 1 exactly, 1.5 M times
    flat[2000000:2000010] = 0
    pl = Plan(SarParams(n_az=shape[0], n_rg=shape[1]))
    s2, above = pl.debug_select(to_dev(b), k)
    m = np.sort(mag2_f32(b).reshape(-1))[::-1]
    assert s2 == int(m[k].view(np.uint32))
    assert above == int(np.count_nonzero(m > m[k]))


@pytest.mark.parametrize("case", ["mask0", "iters0", "k1", "kmax", "delta"])
def test_ita_degenerate_cases(case):
    """Degenerate inputs of Algorithm 1 on a 256 x 512 grid:
    mask0  -- Theta = 0 everywhere: the residual vanishes, X stays 0 whatever Y holds;
    iters0 -- no iteration: X is returned untouched (bitwise);
    k1     -- the k-rule keeps one pixel (sigma = the 2nd largest |b|), vs the oracle;
    kmax   -- k = n - 1 (sigma = the smallest |b|), vs the oracle;
    delta  -- a single-pixel echo, vs the oracle."""
    import torch
    from inputs.configs import SarParams
    p = SarParams(n_az=256, n_rg=512)
    n = p.n_az * p.n_rg
    Y = rand_c((p.n_az, p.n_rg), 11)
    mask = np.ones((p.n_az, p.n_rg), dtype=bool)
    k, iters = 50, 4
    if case == "mask0":
        mask[:] = False
    elif case == "k1":
        k = 1
    elif case == "kmax":
        k = n - 1
    elif case == "delta":
        Y = np.zeros_like(Y)
        Y[37, 101] = 3.0 - 2.0j
    pl = _plan(p)
    X0 = to_dev(rand_c((p.n_az, p.n_rg), 12)) if case == "iters0" else None
    Xg = pl.ita_iterate(to_dev(Y), mask_bits_dev(mask), thr="soft", rule="k", k=k, mu=1.0,
                        iters=0 if case == "iters0" else iters,
                        X=None if X0 is None else X0.clone())
    Xg = to_host(Xg)
    if case == "iters0":
        assert np.array_equal(Xg.view(np.uint32), to_host(X0).view(np.uint32))
        return
    if case == "mask0":
        assert not np.any(Xg)
        return
    Xo = ita.ita(csa.CSAOperator(p), Y.astype(np.complex128), mask, thr="soft", rule="k", k=k, mu=1.0, iters=iters)
    assert rel_l2(Xg, Xo) <= 1e-4, rel_l2(Xg, Xo)
    assert np.count_nonzero(Xg) <= k
    if case != "kmax":
        assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())

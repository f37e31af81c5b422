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
from tests._common import mag2_f32, mask_bits_dev, need_gpu, problem, rand_c, rel_l2, to_dev, to_host

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


def test_ita_c2_grid_first_iterations():
    """c2 (2048 x 2048 Thomas clusters, 30% mask, soft, k = 2%), 10 iterations."""
    prob = problem("c2")
    Xo, olog, Xg, glog, _ = _run_both(prob, iters=10)
    assert rel_l2(Xg, Xo) <= TOL_ITA


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
    cfg = configs.get("c3")
    from inputs import synth
    from tests._common import oracle_echo
    prob = synth.make_problem(cfg, oracle_echo)
    op = csa.CSAOperator(cfg.params)
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


def test_ita_fallback_only_when_window_misses():
    """After the first iteration the select should mostly hit the speculative candidate window."""
    prob = problem("c1")
    cfg = prob.cfg
    pl = _plan(cfg.params)
    pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule="k", k=cfg.k, iters=30)
    fb = pl.debug_fallbacks()
    assert 1 <= fb <= 10, fb

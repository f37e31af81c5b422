"""Parity of the RDA operator pair (NEXT-2, the paper's CSRDA; cssar op = CSSAR_OP_RDA)
against the fp64 oracle (oracle/rda.py, pinned in test_oracle_rda.py).

The range sweep carries the 8-tap truncated-sinc RCMC C (M body) and its transpose D = C^T
(G body); the azimuth sweeps, thresholds and select are the CSA path's.  Bars: operators
<= 1e-5 relative L2 (fp32 chain + fp32 sinc weights; north star 1e-4), ITA <= 1e-3 with the
identical support, the multi-GPU schedule bitwise equal to world 1.
"""
import numpy as np
import pytest

from inputs import configs
from inputs.configs import SarParams
from oracle import ita, rda
from tests._common import mask_bits_dev, need_gpu, problem, rand_c, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _plan(p, **kw):
    from paper_1302_3120_b200 import Plan
    return Plan(p, op="rda", **kw)


@pytest.mark.parametrize("n_rg", [128, 256, 512, 1024, 2048, 4096, 8192, 16384])
@pytest.mark.parametrize("gbody", [1, 0])
def test_rda_range_sweep_matches_oracle(n_rg, gbody):
    n_az = 128 if n_rg >= 4096 else 256
    Fr = 120e6 if n_rg == 16384 else 60e6
    p = SarParams(n_az=n_az, n_rg=n_rg, Fr=Fr)
    U = rand_c((n_az, n_rg), 300 + n_rg + gbody)
    ref = rda.RDAOperator(p).range_segment(U.astype(np.complex128), conj=bool(gbody))
    pl = _plan(p, workspace=False)
    d = to_dev(U)
    pl.debug_range_sweep(d, gbody)
    err = rel_l2(to_host(d) / n_rg, ref)          # the hook's transforms are unnormalised
    assert err <= 5e-6, err


@pytest.mark.parametrize("shape", [(128, 128), (512, 1024), (2048, 256)])
def test_rda_operators_match_oracle(shape):
    p = SarParams(n_az=shape[0], n_rg=shape[1])
    op = rda.RDAOperator(p)
    pl = _plan(p)
    X = rand_c(shape, 11)
    R = rand_c(shape, 12)
    mask = (np.random.default_rng(13).random(shape) < 0.3).astype(np.uint8)
    mb = mask_bits_dev(mask)
    fw = to_host(pl.forward(to_dev(X), mb))
    assert rel_l2(fw, op.A(X.astype(np.complex128), mask)) <= 1e-5
    ad = to_host(pl.adjoint(to_dev(R), mb))
    assert rel_l2(ad, op.AH(R.astype(np.complex128), mask)) <= 1e-5
    im = to_host(pl.image(to_dev(R), None))
    assert rel_l2(im, op.M(R.astype(np.complex128))) <= 1e-5


def test_rda_adjoint_identity_full_size():
    """Theorem 1 at the c3 grid (8192 x 8192): <A x, y> = <x, A^H y> (property at any size)."""
    import torch
    p = configs.get("c3").params
    pl = _plan(p)
    g = torch.Generator(device="cuda").manual_seed(5)
    shape = (int(p.n_az), int(p.n_rg))
    x = torch.randn(shape, dtype=torch.complex64, device="cuda", generator=g)
    y = torch.randn(shape, dtype=torch.complex64, device="cuda", generator=g)
    mask = (torch.rand(shape, device="cuda", generator=g) < 0.5).to(torch.uint8)
    from paper_1302_3120_b200 import pack_mask
    mb = pack_mask(mask)
    ax = pl.forward(x, mb)
    lhs = torch.sum(ax.conj().to(torch.complex128) * y.to(torch.complex128))
    del ax
    ahy = pl.adjoint(y, mb)
    rhs = torch.sum(x.conj().to(torch.complex128) * ahy.to(torch.complex128))
    assert abs(complex(lhs - rhs)) / abs(complex(lhs)) <= 1e-5


@pytest.mark.parametrize("thr", ["half", "soft"])
def test_rda_ita_matches_oracle_c1(thr):
    """CSRDA (eq. 25 with the RDA G): c1 (512 x 512 exact point-target echo, k-rule)."""
    prob = problem("c1", iters=20)
    cfg = prob.cfg
    op = rda.RDAOperator(cfg.params)
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=thr, rule="k", k=cfg.k, mu=cfg.mu, iters=20)
    pl = _plan(cfg.params)
    X, log = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=thr, rule="k", k=cfg.k, mu=cfg.mu,
                            iters=20, log=True)
    Xg = to_host(X)
    assert rel_l2(Xg, Xo) <= 1e-3
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())
    assert all(e["support"] == cfg.k for e in log)


def test_rda_ita_fixed_lambda_and_adaptive():
    prob = problem("c2", 512, 512)
    cfg = prob.cfg
    op = rda.RDAOperator(cfg.params)
    pl = _plan(cfg.params)
    for kw in (dict(rule="lambda", lam=0.05, mu=1.0), dict(rule="k", k=cfg.k, mu="adaptive")):
        Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr="soft", iters=8, **kw)
        X, _ = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr="soft", iters=8, log=True,
                              **{k: v for k, v in kw.items()})
        Xg = to_host(X)
        assert rel_l2(Xg, Xo) <= 1e-3, kw
        assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist()), kw


@pytest.mark.parametrize("world", [2, 4])
def test_rda_group_is_bitwise_single_gpu(world):
    """The multi-GPU schedule (row / column slabs, fused transposes) with the RDA pair."""
    import torch
    from paper_1302_3120_b200 import Group
    prob = problem("c2", 1024, 1024)
    cfg = prob.cfg
    pl = _plan(cfg.params)
    Xs, ls = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule=cfg.rule, k=cfg.k,
                            mu=cfg.mu, iters=5, log=True)
    g = Group(cfg.params, world, op="rda")
    h = cfg.params.n_az // world
    Ys = [to_dev(prob.Y[r * h:(r + 1) * h]) for r in range(world)]
    mb = mask_bits_dev(prob.mask)
    Ms = [mb[r * h:(r + 1) * h].contiguous() for r in range(world)]
    Xg = [torch.zeros_like(y) for y in Ys]
    lg = g.ita_iterate(Ys, Ms, Xg, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=5, log=True)
    Xg = np.concatenate([to_host(x) for x in Xg], axis=0)
    assert np.array_equal(Xg.view(np.uint32), to_host(Xs).view(np.uint32))
    assert [e["sigma"] for e in lg] == [e["sigma"] for e in ls]


# ---- recorded-pulse range filter (NEXT-4)
def _nlfm_replica(p, kappa=4e17):
    L = int(round(p.Tr * p.Fr))
    t = (np.arange(L) - (L - 1) / 2.0) / p.Fr
    return np.exp(2j * np.pi * (0.5 * p.Kr * t ** 2 + kappa * t ** 3))


@pytest.mark.parametrize("n_rg", [256, 8192])
@pytest.mark.parametrize("gbody", [1, 0])
def test_pulse_range_sweep_matches_oracle(n_rg, gbody):
    p = SarParams(n_az=128, n_rg=n_rg)
    s = _nlfm_replica(p)
    U = rand_c((128, n_rg), 500 + n_rg + gbody)
    ref = rda.RDAOperator(p, pulse=s).range_segment(U.astype(np.complex128), conj=bool(gbody))
    pl = _plan(p, workspace=False)
    pl.set_pulse(s)
    d = to_dev(U)
    pl.debug_range_sweep(d, gbody)
    assert rel_l2(to_host(d) / n_rg, ref) <= 5e-6


def test_pulse_operators_ita_and_reset():
    from inputs.configs import SarParams as SP
    from oracle import echo
    p = SP(n_az=256, n_rg=512)
    s = _nlfm_replica(p)
    kap = 4e17
    tg = [(128, 256, np.exp(0.4j)), (30, 60, 1.0), (200, 400, 0.7j), (90, 480, -1.0)]
    Y0 = echo.exact_echo(p, tg, pulse=lambda t: np.exp(2j * np.pi * (0.5 * p.Kr * t ** 2 + kap * t ** 3)))
    mask = (np.random.default_rng(31).random(Y0.shape) < 0.3).astype(np.uint8)
    Y = (Y0 * mask).astype(np.complex64)
    op = rda.RDAOperator(p, pulse=s)
    pl = _plan(p)
    ref_plain = to_host(pl.forward(to_dev(rand_c(Y.shape, 1)), None))
    pl.set_pulse(s)
    X = rand_c(Y.shape, 2)
    mb = mask_bits_dev(mask)
    assert rel_l2(to_host(pl.forward(to_dev(X), mb)), op.A(X.astype(np.complex128), mask)) <= 1e-5
    assert rel_l2(to_host(pl.adjoint(to_dev(X), mb)), op.AH(X.astype(np.complex128), mask)) <= 1e-5
    Xo = ita.ita(op, Y.astype(np.complex128), mask, thr="soft", rule="k", k=8, mu=1.0, iters=25)
    Xg, _ = pl.ita_iterate(to_dev(Y), mb, thr="soft", rule="k", k=8, mu=1.0, iters=25, log=True)
    Xg = to_host(Xg)
    assert rel_l2(Xg, Xo) <= 1e-3
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())
    assert {i * p.n_rg + j for (i, j, _) in tg} <= set(np.argsort(-np.abs(Xg).ravel())[:8].tolist())
    pl.set_pulse(None)                                   # back to the chirp P_tau, bitwise
    assert np.array_equal(to_host(pl.forward(to_dev(rand_c(Y.shape, 1)), None)), ref_plain)


def test_pulse_rejected_on_csa_plans():
    from paper_1302_3120_b200 import Plan, CssarError
    pl = Plan(SarParams(n_az=128, n_rg=128), workspace=False)
    with pytest.raises(CssarError) as e:
        pl.set_pulse(np.ones(4, np.complex64))
    assert e.value.code == -10

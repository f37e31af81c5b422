"""The multi-GPU slab-partitioned ITA (include/cssar.h world > 1) on one device.

cssar_group runs, for `world` emulated ranks, exactly the kernels and schedule of the
multi-GPU path: row slabs of n_az/world azimuth lines for the range sweeps, column slabs of
n_rg/world gates for the azimuth sweeps, the transposes fused into the sweeps' epilogues
(stores into every rank's slab: the other emulated ranks' buffers here, CUDA-IPC peer memory
over NVLink on a multi-GPU box; CSSAR_MULTI_A2A selects separate all-to-all transposes) and
the select's histograms summed over ranks.  Every kernel computes with global indices, so
the result must be BITWISE equal to the single-GPU plan on the same inputs (only the
summation order of the logged residual norm differs), and the single-GPU plan is itself
pinned to the fp64 oracle (test_gpu_ita.py); one case also checks the oracle directly.
"""
import numpy as np
import pytest

from inputs import configs
from oracle import csa, ita
from tests._common import mask_bits_dev, need_gpu, problem, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _slabs(a, world):
    h = a.shape[0] // world
    return [a[r * h:(r + 1) * h] for r in range(world)]


def _group_run(prob, world, iters, rule=None, lam=0.0, masked=True):
    import torch
    from paper_1302_3120_b200 import Group
    cfg = prob.cfg
    g = Group(cfg.params, world)
    Ys = [to_dev(y) for y in _slabs(prob.Y, world)]
    mb = mask_bits_dev(prob.mask)
    Ms = [m.contiguous() for m in _slabs(mb, world)] if masked else None
    Xs = [torch.zeros_like(y) for y in Ys]
    log = g.ita_iterate(Ys, Ms, Xs, thr=cfg.thr, rule=rule or cfg.rule, k=cfg.k, lam=lam, mu=cfg.mu, iters=iters,
                        log=True)
    return np.concatenate([to_host(x) for x in Xs], axis=0), log


def _single_run(prob, iters, rule=None, lam=0.0, masked=True):
    from paper_1302_3120_b200 import Plan
    cfg = prob.cfg
    pl = Plan(cfg.params)
    X, log = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask) if masked else None, thr=cfg.thr,
                            rule=rule or cfg.rule, k=cfg.k, lam=lam, mu=cfg.mu, iters=iters, log=True)
    return to_host(X), log


def _same_logs(la, lb):
    assert [e["sigma"] for e in la] == [e["sigma"] for e in lb]
    assert [e["support"] for e in la] == [e["support"] for e in lb]
    ra = np.array([e["resid2"] for e in la])
    rb = np.array([e["resid2"] for e in lb])
    assert np.max(np.abs(ra - rb) / rb) <= 1e-6


@pytest.mark.parametrize("name,grid,world,iters", [
    ("c1", None, 2, 12),            # L1/2 threshold, k = 2%, exact point-target echo
    ("c1", None, 4, 12),
    ("c2", (1024, 1024), 8, 8),     # soft, clutter, 30% mask
    ("c2", None, 16, 4),            # the largest world the library supports
    ("c3", (2048, 1024), 4, 6),     # line mask
])
def test_group_is_bitwise_single_gpu(name, grid, world, iters):
    prob = problem(name, *(grid or (None, None)))
    Xs, ls = _single_run(prob, iters)
    Xg, lg = _group_run(prob, world, iters)
    assert np.array_equal(Xg.view(np.uint32), Xs.view(np.uint32)), rel_l2(Xg, Xs)
    _same_logs(lg, ls)


@pytest.mark.parametrize("transport", ["fused", "a2a"])
def test_group_transports_bitwise(transport, monkeypatch):
    """Both exchange schedules of the multi-GPU path: the fused transposes (azimuth / range
    epilogues store straight into every rank's slab — peer memory on a multi-GPU box) and
    the separate all-to-all transposes (CSSAR_MULTI_A2A, the NCCL fallback)."""
    if transport == "a2a":
        monkeypatch.setenv("CSSAR_MULTI_A2A", "1")
    prob = problem("c2", 1024, 1024)
    Xs, ls = _single_run(prob, 6)
    Xg, lg = _group_run(prob, 4, 6)
    assert np.array_equal(Xg.view(np.uint32), Xs.view(np.uint32)), rel_l2(Xg, Xs)
    _same_logs(lg, ls)


@pytest.mark.parametrize("cond", [True, False])
def test_group_conditional_fallback_round(cond, monkeypatch):
    """The select's full-histogram fallback round (pass over b, 2048-word all-reduce, pick) is a
    conditional graph node in the captured multi-GPU iteration (3 collectives per iteration
    instead of 4): its body must run exactly when the coarse step misses -- the first iteration
    from X = 0 always does here -- so X stays bitwise the single-GPU result, with the node and
    with the unconditional round (CSSAR_NO_COND)."""
    import torch
    from paper_1302_3120_b200 import Group, Plan
    if not cond:
        monkeypatch.setenv("CSSAR_NO_COND", "1")
    prob = problem("c2", 1024, 1024)
    cfg = prob.cfg
    iters = 6
    pl = Plan(cfg.params)
    X1, l1 = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule=cfg.rule, k=cfg.k,
                            mu=cfg.mu, iters=iters, log=True)
    assert pl.debug_fallbacks() >= 1                 # the fallback branch is taken at least once
    world = 4
    g = Group(cfg.params, world)
    Ys = [to_dev(y) for y in _slabs(prob.Y, world)]
    Ms = [m.contiguous() for m in _slabs(mask_bits_dev(prob.mask), world)]
    Xs = [torch.zeros_like(y) for y in Ys]
    lg = g.ita_iterate(Ys, Ms, Xs, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=iters, log=True)
    assert g.debug_graph_info() == (1 if cond else 0)
    Xg = np.concatenate([to_host(x) for x in Xs], axis=0)
    assert np.array_equal(Xg.view(np.uint32), to_host(X1).view(np.uint32)), rel_l2(Xg, to_host(X1))
    _same_logs(lg, l1)


def test_group_fixed_lambda_and_no_mask():
    prob = problem("c2", 512, 512)
    Xs, ls = _single_run(prob, 5, rule="lambda", lam=0.05, masked=False)
    Xg, lg = _group_run(prob, 4, 5, rule="lambda", lam=0.05, masked=False)
    assert np.array_equal(Xg.view(np.uint32), Xs.view(np.uint32)), rel_l2(Xg, Xs)
    _same_logs(lg, ls)


def test_group_matches_oracle_c1():
    """Independent of the single-GPU path: world 4 vs the fp64 oracle (north-star bar)."""
    prob = problem("c1", iters=30)
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu,
                 iters=30)
    Xg, _ = _group_run(prob, 4, 30)
    assert rel_l2(Xg, Xo) <= 1e-3
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())


def test_world_validation():
    from paper_1302_3120_b200 import Group, CssarError
    p = configs.get("c0").params            # 128 x 128: n_rg / 2 = 64 < 128 gates per column slab
    with pytest.raises(CssarError) as e:
        Group(p, 2)
    assert e.value.code == -2
    with pytest.raises(CssarError):
        Group(configs.get("c1").params, 32)  # world > 16


# ---- sparse-X' schedule (CSSAR_FLAG_SPARSE_X)
@pytest.mark.parametrize("name,grid,world,iters", [
    ("c1", None, 2, 12),
    ("c1", None, 4, 12),
    ("c2", (1024, 1024), 4, 8),
    ("c3", (2048, 1024), 8, 6),     # line mask; k <= n_az n_rg / (8 world) sets the world
])
def test_group_sparse_x_matches_single_gpu(name, grid, world, iters):
    """From iteration 1 on S1 + transpose #1 are replaced by the compacted X' (all-gathered
    over peer memory), a fold into n_az/world cyclic Doppler bins and a local m-point DFT.
    Not bitwise (another factorisation, atomic folds): X within 1e-5 of world 1, the same
    thresholds and support sizes."""
    import torch
    from paper_1302_3120_b200 import Group
    prob = problem(name, *(grid or (None, None)))
    cfg = prob.cfg
    Xs, ls = _single_run(prob, iters)
    g = Group(cfg.params, world)
    Ys = [to_dev(y) for y in _slabs(prob.Y, world)]
    Ms = [m.contiguous() for m in _slabs(mask_bits_dev(prob.mask), world)]
    Xg = [torch.zeros_like(y) for y in Ys]
    lg = g.ita_iterate(Ys, Ms, Xg, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=iters, log=True,
                       sparse=True)
    Xg = np.concatenate([to_host(x) for x in Xg], axis=0)
    assert rel_l2(Xg, Xs) <= 1e-5, rel_l2(Xg, Xs)
    sg = np.array([e["sigma"] for e in lg])
    ss = np.array([e["sigma"] for e in ls])
    assert np.max(np.abs(sg - ss) / ss) <= 1e-5
    assert [e["support"] for e in lg] == [e["support"] for e in ls]


def test_group_sparse_x_matches_oracle_c1():
    prob = problem("c1", iters=30)
    cfg = prob.cfg
    op = csa.CSAOperator(cfg.params)
    Xo = ita.ita(op, prob.Y.astype(np.complex128), prob.mask, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu,
                 iters=30)
    import torch
    from paper_1302_3120_b200 import Group
    g = Group(cfg.params, 4)
    Ys = [to_dev(y) for y in _slabs(prob.Y, 4)]
    Ms = [m.contiguous() for m in _slabs(mask_bits_dev(prob.mask), 4)]
    Xg = [torch.zeros_like(y) for y in Ys]
    g.ita_iterate(Ys, Ms, Xg, thr=cfg.thr, rule=cfg.rule, k=cfg.k, mu=cfg.mu, iters=30, sparse=True)
    Xg = np.concatenate([to_host(x) for x in Xg], axis=0)
    assert rel_l2(Xg, Xo) <= 1e-3
    assert set(np.flatnonzero(Xg).tolist()) == set(np.flatnonzero(Xo).tolist())


def test_sparse_x_flag_falls_back_where_it_does_not_apply(monkeypatch):
    """The flag is a request: world 1 rejects it; fixed lambda, the all-to-all transport and
    k above the list capacity run the dense schedule (bitwise the plain group result)."""
    import torch
    from paper_1302_3120_b200 import Group, Plan, CssarError
    prob = problem("c2", 512, 512)
    cfg = prob.cfg
    with pytest.raises(CssarError) as e:
        Plan(cfg.params).ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), k=cfg.k, iters=2, sparse=True)
    assert e.value.code == -1
    g = Group(cfg.params, 2)
    Ys = [to_dev(y) for y in _slabs(prob.Y, 2)]

    def run(**kw):
        Xg = [torch.zeros_like(y) for y in Ys]
        g.ita_iterate(Ys, None, Xg, iters=3, **kw)
        return np.concatenate([to_host(x) for x in Xg], axis=0)
    for kw in (dict(rule="lambda", lam=0.1), dict(k=200000)):
        assert np.array_equal(run(sparse=True, **kw), run(**kw))
    monkeypatch.setenv("CSSAR_MULTI_A2A", "1")
    assert np.array_equal(run(sparse=True, k=cfg.k), run(k=cfg.k))


@pytest.mark.parametrize("world", [2, 4])
def test_group_operators_bitwise_single_gpu(world):
    """cssar_forward / cssar_adjoint on world > 1 row slabs (collective): bitwise equal to one
    GPU, which is pinned to the oracle in test_gpu_ops.py; one case checked against the oracle."""
    from paper_1302_3120_b200 import Group, Plan
    from tests._common import rand_c
    p = configs.get("c1").params
    X = rand_c((p.n_az, p.n_rg), 41)
    mask = (np.random.default_rng(42).random((p.n_az, p.n_rg)) < 0.4).astype(np.uint8)
    mb = mask_bits_dev(mask)
    pl = Plan(p)
    fs = to_host(pl.forward(to_dev(X), mb))
    as_ = to_host(pl.adjoint(to_dev(X), mb))
    g = Group(p, world)
    Xs = [to_dev(x) for x in _slabs(X, world)]
    Ms = [m.contiguous() for m in _slabs(mb, world)]
    fg = np.concatenate([to_host(y) for y in g.forward(Xs, Ms)], axis=0)
    ag = np.concatenate([to_host(y) for y in g.adjoint(Xs, Ms)], axis=0)
    assert np.array_equal(fg.view(np.uint32), fs.view(np.uint32))
    assert np.array_equal(ag.view(np.uint32), as_.view(np.uint32))
    ig = np.concatenate([to_host(y) for y in g.adjoint(Xs, None)], axis=0)
    op = csa.CSAOperator(p)
    assert rel_l2(ig, op.M(X.astype(np.complex128))) <= 1e-5

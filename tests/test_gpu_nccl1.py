"""The multi-GPU slab path over REAL NCCL on one GPU (include/cssar.h
cssar_debug_plan_create_nccl).

NCCL refuses two ranks on one device, so the multi-rank plumbing -- ncclCommInitRank, the
grouped ncclSend / ncclRecv all-to-all transposes, the grouped all-reduces of the split select,
the all-gather of the CUDA-IPC records in cssar_bind_workspace, ncclCommGetAsyncError -- is run
here by a ONE-rank NCCL plan that takes the slab path with whole arrays as slabs (transposes to
itself, all-reduces over one rank).  Every kernel computes with global indices, so the result
must be bitwise the world-1 plan's (which test_gpu_ita.py pins to the fp64 oracle); the logged
residual norm is summed in another order (1e-6).  The emulation groups of test_gpu_multi.py
cover world 2..16 of the same schedule with device copies in place of NCCL."""
import numpy as np
import pytest

from tests._common import mask_bits_dev, need_gpu, problem, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _plans(prob):
    from paper_1302_3120_b200 import Plan, nccl_unique_id
    return Plan(prob.cfg.params), Plan(prob.cfg.params, unique_id=nccl_unique_id())


def _run(pl, prob, iters, **kw):
    cfg = prob.cfg
    X, log = pl.ita_iterate(to_dev(prob.Y), mask_bits_dev(prob.mask), thr=cfg.thr, rule=cfg.rule, k=cfg.k,
                            mu=cfg.mu, iters=iters, log=True, **kw)
    return to_host(X), log


def _same_logs(la, lb):
    assert [e["sigma"] for e in la] == [e["sigma"] for e in lb]
    assert [e["support"] for e in la] == [e["support"] for e in lb]
    ra = np.array([e["resid2"] for e in la])
    rb = np.array([e["resid2"] for e in lb])
    assert np.max(np.abs(ra - rb) / rb) <= 1e-6


@pytest.mark.parametrize("name,grid,iters,peer", [
    ("c1", None, 12, False),            # L1/2 threshold, exact point-target echo
    ("c2", (1024, 1024), 8, False),     # soft, clutter, 30% mask
    ("c3", (2048, 1024), 6, False),     # line mask
    ("c2", (1024, 1024), 8, True),      # peer-store transposes (to itself) + the flag barrier
])
def test_nccl_one_rank_ita_is_bitwise_world1(name, grid, iters, peer):
    prob = problem(name, *(grid or (None, None)))
    p1, pn = _plans(prob)
    X1, l1 = _run(p1, prob, iters)
    Xn, ln = _run(pn, prob, iters, peer=peer)
    assert np.array_equal(Xn.view(np.uint32), X1.view(np.uint32)), rel_l2(Xn, X1)
    _same_logs(ln, l1)
    # the select's fallback round is a conditional graph node holding the NCCL all-reduce
    assert pn.debug_graph_info() == 1
    assert p1.debug_fallbacks() >= 1


def test_nccl_one_rank_sparse_x():
    """The sparse-X' schedule (all-gathered compacted X', cyclic fold, m-point DFT) on the NCCL
    plan: another factorisation, so within 1e-5 of world 1 with the same thresholds' supports."""
    prob = problem("c2", 1024, 1024)
    p1, pn = _plans(prob)
    X1, l1 = _run(p1, prob, 8)
    Xn, ln = _run(pn, prob, 8, peer=True, sparse=True)
    assert rel_l2(Xn, X1) <= 1e-5, rel_l2(Xn, X1)
    assert [e["support"] for e in ln] == [e["support"] for e in l1]


def test_nccl_one_rank_operators_bitwise():
    import torch
    prob = problem("c2", 1024, 2048)
    p1, pn = _plans(prob)
    Y = to_dev(prob.Y)
    mb = mask_bits_dev(prob.mask)
    X1 = p1.adjoint(Y, mb)
    Xn = pn.adjoint(Y, mb)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(X1), torch.view_as_real(Xn))
    Y1 = p1.forward(X1, mb)
    Yn = pn.forward(X1, mb)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(Y1), torch.view_as_real(Yn))


def test_nccl_one_rank_rejects_world1_only_features():
    """The slab path's contract: the tolerance stop, the adaptive step and the debug hooks are
    world-1 features (CSSAR_ERR_INVALID_PARAMS / CSSAR_ERR_BAD_PLAN)."""
    from paper_1302_3120_b200 import CssarError
    prob = problem("c1")
    _, pn = _plans(prob)
    with pytest.raises(CssarError):
        _run(pn, prob, 2, tol=1e-3)
    with pytest.raises(CssarError):
        pn.ita_iterate(to_dev(prob.Y), None, k=prob.cfg.k, mu="adaptive", iters=1)
    with pytest.raises(CssarError):
        pn.debug_az_fft(to_dev(prob.Y))

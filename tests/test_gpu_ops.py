"""Operator parity: cssar_forward / cssar_adjoint / cssar_image vs the fp64 oracle.

North star: rel-L2 <= 1e-4 per single operator application (expected ~3e-7).  Shapes span
every config's grid (c0..c3 at full size; c4 by properties: adjoint identity and A^H A = I
at Theta = 1, which hold at any size) plus non-square and ragged-mask cases.
"""
import numpy as np
import pytest

from inputs import configs, synth
from inputs.configs import SarParams
from oracle import csa
from tests._common import mask_bits_dev, need_gpu, problem, rand_c, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL_OP = 1e-4


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _plan(p, ws=False):
    from paper_1302_3120_b200 import Plan
    return Plan(p, workspace=ws)


@pytest.mark.parametrize("n_az,n_rg,rate", [(128, 128, 0.5), (512, 512, 0.5), (256, 1024, 0.3),
                                            (2048, 128, 0.7), (128, 4096, 1.0), (2048, 2048, 0.3)])
def test_forward_adjoint_random(n_az, n_rg, rate):
    p = SarParams(n_az=n_az, n_rg=n_rg)
    op = csa.CSAOperator(p)
    r = np.random.default_rng(n_az * 7 + n_rg)
    mask = r.random((n_az, n_rg)) < rate
    X = rand_c((n_az, n_rg), 1)
    R = rand_c((n_az, n_rg), 2)
    pl = _plan(p)
    mb = mask_bits_dev(mask)
    Yg = to_host(pl.forward(to_dev(X), mb))
    Xg = to_host(pl.adjoint(to_dev(R), mb))
    Ig = to_host(pl.image(to_dev(R), mb))
    assert rel_l2(Yg, op.A(X.astype(complex), mask)) <= TOL_OP
    ah = op.AH(R.astype(complex), mask)
    assert rel_l2(Xg, ah) <= TOL_OP
    assert rel_l2(Ig, ah) <= TOL_OP
    # fp32 adjoint identity <A x, r> = <x, A^H r>
    lhs = np.vdot(R.astype(complex), Yg.astype(complex))
    rhs = np.vdot(Xg.astype(complex), X.astype(complex))
    assert abs(lhs - rhs) / abs(lhs) <= 1e-5


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_operators_on_config_inputs(name):
    prob = problem(name)
    p = prob.cfg.params
    op = csa.CSAOperator(p)
    pl = _plan(p)
    mb = mask_bits_dev(prob.mask)
    img = to_host(pl.image(to_dev(prob.Y), mb))
    assert rel_l2(img, op.M(prob.Y.astype(complex) * prob.mask)) <= TOL_OP
    Xt = prob.scene.dense(np.complex64)
    assert rel_l2(to_host(pl.forward(to_dev(Xt), mb)), op.A(Xt.astype(complex), prob.mask)) <= TOL_OP


def test_operators_c3_full_size():
    """c3 grid (8192 x 8192), line mask: forward and adjoint vs the fp64 oracle."""
    cfg = configs.get("c3")
    p = cfg.params
    mask = synth.make_mask(cfg)
    X = rand_c((p.n_az, p.n_rg), 11)
    pl = _plan(p)
    mb = mask_bits_dev(mask)
    op = csa.CSAOperator(p)
    Yg = to_host(pl.forward(to_dev(X), mb))
    assert rel_l2(Yg, op.A(X.astype(complex), mask)) <= TOL_OP
    del Yg
    Xg = to_host(pl.adjoint(to_dev(X), mb))
    assert rel_l2(Xg, op.AH(X.astype(complex), mask)) <= TOL_OP


def test_c4_full_size_properties():
    """c4 grid (32768 x 16384, Fr = 120 MHz): properties that hold at any size —
    A^H A x = x at Theta = 1 (unitary chain) and the masked adjoint identity."""
    import torch
    cfg = configs.get("c4")
    p = cfg.params
    pl = _plan(p)
    n_az, n_rg = p.n_az, p.n_rg
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn((n_az, n_rg), dtype=torch.complex64, device="cuda", generator=g)
    y = pl.forward(x, None)
    z = pl.adjoint(y, None)
    err = (torch.linalg.vector_norm(z - x) / torch.linalg.vector_norm(x)).item()
    assert err <= 5e-6, err
    del y, z
    m = (torch.rand((n_az, n_rg), device="cuda", generator=g) < 0.5).to(torch.uint8)
    from paper_1302_3120_b200 import pack_mask
    mb = pack_mask(m)
    r = torch.randn((n_az, n_rg), dtype=torch.complex64, device="cuda", generator=g)
    ax = pl.forward(x, mb)
    lhs = torch.vdot(r.flatten(), ax.flatten()).to(torch.complex128)
    del ax
    ahr = pl.adjoint(r, mb)
    rhs = torch.vdot(ahr.flatten(), x.flatten()).to(torch.complex128)
    assert (abs(lhs - rhs) / abs(lhs)).item() <= 1e-4


def test_pack_mask_matches_host_packing():
    import torch
    from paper_1302_3120_b200 import pack_mask
    m = np.random.default_rng(0).random((256, 512)) < 0.37
    bits = pack_mask(torch.from_numpy(m.astype(np.uint8)).cuda())
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), synth.pack_mask_bits(m))


def test_null_mask_is_all_ones():
    p = SarParams(n_az=256, n_rg=256)
    pl = _plan(p)
    X = rand_c((256, 256), 9)
    ones = np.ones((256, 256), bool)
    a = to_host(pl.forward(to_dev(X), None))
    b = to_host(pl.forward(to_dev(X), mask_bits_dev(ones)))
    assert np.array_equal(a, b)


def test_abi_errors():
    import torch
    from paper_1302_3120_b200 import CssarError, Plan
    with pytest.raises(CssarError) as e:
        Plan(SarParams(n_az=100, n_rg=128), workspace=False)
    assert e.value.code == -2
    with pytest.raises(CssarError) as e:
        Plan(SarParams(n_az=128, n_rg=128, squint=0.06), workspace=False)
    assert e.value.code == -1
    with pytest.raises(CssarError) as e:
        Plan(SarParams(n_az=128, n_rg=128, Fr=-1.0), workspace=False)
    assert e.value.code == -1
    pl = Plan(SarParams(n_az=128, n_rg=128))
    Y = torch.zeros((128, 128), dtype=torch.complex64, device="cuda")
    for kw, code in ((dict(k=0), -3), (dict(k=128 * 128), -3), (dict(k=5, mu=0.0), -4),
                     (dict(rule="lambda", lam=-1.0), -4)):
        args = dict(thr="soft", rule="k", k=5, mu=1.0, iters=1)
        args.update(kw)
        with pytest.raises(CssarError) as e:
            pl.ita_iterate(Y, None, **args)
        assert e.value.code == code
    # misaligned pointer: a view offset by one complex element (8 bytes)
    buf = torch.zeros(128 * 128 + 1, dtype=torch.complex64, device="cuda")
    mis = buf[1:].view(128, 128)
    with pytest.raises(CssarError) as e:
        pl.forward(mis, None)
    assert e.value.code == -5
    # no workspace bound
    pl2 = Plan(SarParams(n_az=128, n_rg=128), workspace=False)
    with pytest.raises(CssarError) as e:
        pl2.ita_iterate(Y, None, k=5, iters=1)
    assert e.value.code == -8

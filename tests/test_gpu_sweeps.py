"""Per-sweep parity of the CUDA kernels against the oracle (through the C ABI test hooks).

Range sweep (S2 / S4 bodies) at every supported n_rg, azimuth DFT (cluster / DSMEM path
included) at every supported n_az, each on random CN(0,1) data with the oracle in fp64.
Expected accuracy ~3e-7 (fp32 chain + 24-bit fixed-point phases).
"""
import numpy as np
import pytest

from inputs.configs import SarParams
from oracle import csa
from tests._common import need_gpu, rand_c, rel_l2, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _plan(n_az, n_rg, **kw):
    from paper_1302_3120_b200 import Plan
    return Plan(SarParams(n_az=n_az, n_rg=n_rg, **kw), workspace=False)


@pytest.mark.parametrize("n_rg", [128, 256, 512, 1024, 2048, 4096, 8192, 16384])
@pytest.mark.parametrize("gbody", [1, 0])
def test_range_sweep_matches_oracle(n_rg, gbody):
    n_az = 128 if n_rg >= 4096 else 256
    Fr = 120e6 if n_rg == 16384 else 60e6
    p = SarParams(n_az=n_az, n_rg=n_rg, Fr=Fr)
    U = rand_c((n_az, n_rg), 100 + n_rg + gbody)
    ref = csa.CSAOperator(p).range_segment(U.astype(np.complex128), conj=bool(gbody))
    pl = _plan(n_az, n_rg, Fr=Fr)
    d = to_dev(U)
    pl.debug_range_sweep(d, gbody)
    err = rel_l2(to_host(d) / n_rg, ref)          # the hook's transforms are unnormalised
    assert err <= 2e-6, err


@pytest.mark.parametrize("n_az", [128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768])
@pytest.mark.parametrize("direction", [-1, 1])
def test_azimuth_dft_matches_oracle(n_az, direction):
    n_rg = 128
    X = rand_c((n_az, n_rg), 7 + n_az)
    ref = csa.fft_az(X.astype(np.complex128), inverse=direction > 0)
    pl = _plan(n_az, n_rg)
    out = pl.debug_az_fft(to_dev(X), dir=direction)
    err = rel_l2(to_host(out), ref)
    assert err <= 2e-6, err


def test_azimuth_dft_in_place_and_wide():
    """in == out aliasing and a wide panel grid (several column panels + ragged values)."""
    n_az, n_rg = 8192, 512
    X = rand_c((n_az, n_rg), 3)
    X[:, 17] = 0
    ref = csa.fft_az(X.astype(np.complex128))
    pl = _plan(n_az, n_rg)
    d = to_dev(X)
    pl.debug_az_fft(d, out=d, dir=-1)
    assert rel_l2(to_host(d), ref) <= 2e-6


def test_range_sweep_is_exact_inverse_pair():
    """G body followed by M body restores the input (unitary chain, fp32 round trip)."""
    n_az, n_rg = 256, 2048
    U = rand_c((n_az, n_rg), 5)
    pl = _plan(n_az, n_rg)
    d = to_dev(U)
    pl.debug_range_sweep(d, 1)
    pl.debug_range_sweep(d, 0)
    assert rel_l2(to_host(d) / float(n_rg) ** 2, U) <= 2e-6

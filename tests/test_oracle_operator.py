"""Pins for the oracle's CSA operator pair (oracle/csa.py) — no implementation to compare against.

Each pin ties the oracle to something other than itself:
  * naive O(N^2) DFT matrices + explicit diagonal phases  vs  the FFT chain
    (axis, sign, normalisation, bin order) on non-square grids;
  * Theorem 1: G = M^H, densified by probing, and the random adjoint identity;
  * exact unitarity of the CSA chain (A^H A = I at Theta = 1, north star);
  * SURVEY 8(c).7 transcription anchors (independent fp64 computation).
"""
import json
import os

import numpy as np
import pytest

from inputs import configs
from inputs.configs import SarParams
from oracle import csa, echo

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


@pytest.mark.parametrize("n_az,n_rg", [(8, 12), (16, 8)])
def test_chain_matches_naive_dft_matrices(n_az, n_rg):
    p = SarParams(n_az=n_az, n_rg=n_rg)
    op = csa.CSAOperator(p)
    P1, P2, P3 = op.phi
    Fa, Fai = csa.dft_matrix(n_az), csa.dft_matrix(n_az, inverse=True)
    Fr, Fri = csa.dft_matrix(n_rg), csa.dft_matrix(n_rg, inverse=True)
    # explicit matrices: DFT along rows = left multiply; along columns = right multiply by F^T
    def M_naive(Y):
        U = Fa @ Y
        U = P1 * U
        U = U @ Fr.T
        U = P2 * U
        U = U @ Fri.T
        U = P3 * U
        return Fai @ U

    def G_naive(X):
        U = Fa @ X
        U = np.conj(P3) * U
        U = U @ Fr.T
        U = np.conj(P2) * U
        U = U @ Fri.T
        U = np.conj(P1) * U
        return Fai @ U

    Y = _rand((n_az, n_rg), 1)
    assert np.max(np.abs(op.M(Y) - M_naive(Y))) <= 1e-13
    assert np.max(np.abs(op.G(Y) - G_naive(Y))) <= 1e-13
    # the naive DFT matrix itself against the defining sum (one entry, brute force)
    k, m = 3, 5
    assert abs(Fa[k, m] - np.exp(-2j * np.pi * k * m / n_az) / np.sqrt(n_az)) < 1e-15


def _densify(f, shape):
    n = shape[0] * shape[1]
    cols = []
    for t in range(n):
        e = np.zeros(n, dtype=np.complex128)
        e[t] = 1.0
        cols.append(f(e.reshape(shape)).reshape(-1))
    return np.stack(cols, axis=1)


def test_theorem1_dense_G_equals_M_hermitian():
    """Theorem 1: G^H = M, checked on the densified operators (SPEC S:L419-427 probing)."""
    p = SarParams(n_az=8, n_rg=12)
    op = csa.CSAOperator(p)
    Gd = _densify(op.G, op.shape)
    Md = _densify(op.M, op.shape)
    assert np.max(np.abs(Gd - Md.conj().T)) <= 1e-13
    # unitary: G^H G = I (CSA has no interpolation -> exactly invertible, R2)
    assert np.max(np.abs(Gd.conj().T @ Gd - np.eye(Gd.shape[0]))) <= 1e-13


@pytest.mark.parametrize("n", [48, 128])
def test_adjoint_identity_random(n):
    """<G x, y> = <x, M y> to 1e-10 relative (north star)."""
    p = SarParams(n_az=n, n_rg=n)
    op = csa.CSAOperator(p)
    for s in range(3):
        x, y = _rand((n, n), 10 + s), _rand((n, n), 20 + s)
        lhs = np.vdot(y, op.G(x))
        rhs = np.vdot(op.M(y), x)
        assert abs(lhs - rhs) / abs(lhs) <= 1e-10


def test_adjoint_identity_masked_A():
    """<A x, r> = <x, A^H r> with A = Theta o G (eq. 24-25)."""
    p = SarParams(n_az=64, n_rg=32)
    op = csa.CSAOperator(p)
    m = (np.random.default_rng(3).random(op.shape) < 0.4).astype(float)
    x, r = _rand(op.shape, 4), _rand(op.shape, 5)
    lhs = np.vdot(r, op.A(x, m))
    rhs = np.vdot(op.AH(r, m), x)
    assert abs(lhs - rhs) / abs(lhs) <= 1e-10


def test_unitarity_full_sampling_AHA_identity():
    """With Theta = all-ones, A^H A x = x (north star oracle check)."""
    p = SarParams(n_az=128, n_rg=256)
    op = csa.CSAOperator(p)
    x = _rand(op.shape, 7)
    assert np.linalg.norm(op.M(op.G(x)) - x) / np.linalg.norm(x) <= 1e-12
    assert np.linalg.norm(op.G(op.M(x)) - x) / np.linalg.norm(x) <= 1e-12


def test_range_segment_composes_to_operator():
    """The per-sweep decomposition used by the CUDA parity tests equals the full chain."""
    p = SarParams(n_az=32, n_rg=64)
    op = csa.CSAOperator(p)
    x = _rand(op.shape, 8)
    Gx = csa.fft_az(op.range_segment(csa.fft_az(x), conj=True), inverse=True)
    Mx = csa.fft_az(op.range_segment(csa.fft_az(x), conj=False), inverse=True)
    assert np.max(np.abs(Gx - op.G(x))) < 1e-13
    assert np.max(np.abs(Mx - op.M(x))) < 1e-13


def _c(v):
    return complex(v[0], v[1])


def test_survey_transcription_anchors():
    """SURVEY.md 8(c).7 anchors: an independent fp64 transcription of the same definitions."""
    g = json.load(open(os.path.join(GOLD, "survey_8c7_anchors.json")))
    p = SarParams(n_az=16, n_rg=16)
    geo = csa.CSAGeometry(p)
    b = g["grid16_bin8"]
    assert geo.f_eta[8] == pytest.approx(b["f_eta"], rel=1e-15)
    assert geo.D[8] == pytest.approx(b["D"], rel=1e-15)
    assert 1.0 - geo.D[8] == pytest.approx(b["one_minus_D"], rel=1e-9)
    assert geo.Km[8] == pytest.approx(b["Km"], rel=1e-13)
    P1, P2, P3 = geo.screens()
    for key, (i, j) in (("phi_8_3", (8, 3)), ("phi_3_11", (3, 11))):
        e = g[key]
        assert abs(P1[i, j] - _c(e["phi1"])) < 1e-12
        assert abs(P2[i, j] - _c(e["phi2"])) < 1e-12
        # ~3e7-cycle carrier: fp64 evaluation-order rounding ~5e-8 rad
        assert abs(P3[i, j] - _c(e["phi3"])) < 2e-7
    op = csa.CSAOperator(p)
    d = np.zeros((16, 16), complex)
    d[5, 7] = 1.0
    Gd = op.G(d)
    e = g["G_delta_5_7"]
    for key, (i, j) in (("at_0_0", (0, 0)), ("at_5_7", (5, 7)), ("at_12_2", (12, 2))):
        assert abs(Gd[i, j] - _c(e[key])) < 2e-8
    assert np.linalg.norm(Gd) == pytest.approx(1.0, abs=1e-14)
    Mo = op.M(np.ones((16, 16)))
    e = g["M_ones"]
    assert abs(Mo[0, 0] - _c(e["at_0_0"])) < 2e-7
    assert abs(Mo[3, 9] - _c(e["at_3_9"])) < 2e-7


def test_survey_exact_echo_anchors():
    """SURVEY.md 8(c).7 exact-echo anchors: c0 system parameters (128 x 128, 60 MHz), one unit
    target at (64, 64), N_a = 1114 aperture lines (R6): the echo sample Y[64, 64], ||Y||^2,
    the nonzero count (the folded aperture covers every sample) and the focused M(Y)[64, 64]."""
    g = json.load(open(os.path.join(GOLD, "survey_8c7_anchors.json")))["c0_echo_unit_target_64_64"]
    p = configs.get("c0").params
    assert echo.aperture_lines(p) == 1114
    Y = echo.exact_echo(p, [(64, 64, 1.0 + 0j)])
    # the echo phase carries a ~3e7-cycle carrier: fp64 rounding of its argument ~5e-8 rad per term
    assert abs(Y[64, 64] - _c(g["Y_64_64"])) <= 1e-6 * abs(_c(g["Y_64_64"]))
    assert float(np.vdot(Y, Y).real) == pytest.approx(g["norm2"], rel=1e-8)
    assert int(np.count_nonzero(Y)) == g["nonzeros"]
    MY = csa.CSAOperator(p).M(Y)
    assert abs(MY[64, 64] - _c(g["MY_64_64"])) <= 1e-7 * g["MY_64_64_abs"]
    assert abs(MY[64, 64]) == pytest.approx(g["MY_64_64_abs"], rel=1e-9)

"""Pins for the RDA operator pair of the oracle (oracle/rda.py; NEXT-2, the paper's CSRDA).

Pinned against what the paper and the mathematics fix, not against the oracle itself:
  * Theorem 1: G = M^H exactly, the inner-product identity at fp64 rounding;
  * eq. 23: the RCMC gather equals the row's explicit interpolation matrix C
    and the scatter equals C^T (D = C^T), built by an independent loop;
  * eq. 16 special cases: a zero migration is the identity (sinc(k) = delta_k), an integer
    migration is a cyclic shift, exactly;
  * focusing (eq. 14): each target of the exact echo (eq. 1-3) focuses to its own
    pixel with phase arg(sigma), the closed-form peak, the theoretical IRW, and the PSLR the
    paper prints for RDA (-13.32 dB range and azimuth);
  * CSRDA (eq. 25 with the RDA G): ITA on a 30 % random mask recovers the targets.
"""
import json
import os

import numpy as np
import pytest

from inputs.configs import SarParams
from oracle import csa, echo, ita, metrics, rda

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))
PAPER_RDA_PSLR_DB = -13.32   # P:L524, Table 3 row "RDA", range and azimuth


def _rand(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


def _theory(p):
    Na = echo.aperture_lines(p)
    lam_c = csa.C_LIGHT / p.fc
    ka = 2 * p.Vr ** 2 / (lam_c * p.R_ref)
    Ba = Na * ka / p.prf
    Br = p.Kr * p.Tr
    peak = np.sqrt(Na * p.Kr * p.Tr ** 2 * Ba / p.prf)
    return dict(peak=peak, irw_rg=GOLD["irw_factor"] * p.Fr / Br, irw_az=GOLD["irw_factor"] * p.prf / Ba)


@pytest.mark.parametrize("shape", [(64, 96), (128, 128)])
def test_theorem1_adjoint(shape):
    p = SarParams(n_az=shape[0], n_rg=shape[1])
    op = rda.RDAOperator(p)
    X, Y = _rand(shape, 1), _rand(shape, 2)
    lhs = np.vdot(op.G(X), Y)
    rhs = np.vdot(X, op.M(Y))
    assert abs(lhs - rhs) / abs(lhs) < 1e-12
    m = (np.random.default_rng(3).random(shape) < 0.3).astype(float)
    assert abs(np.vdot(op.A(X, m), Y) - np.vdot(X, op.AH(Y, m))) / abs(lhs) < 1e-12


def test_rcmc_is_eq23_matrix():
    p = SarParams(n_az=64, n_rg=96)
    op = rda.RDAOperator(p)
    V = _rand(op.shape, 4)
    U, W = op.rcmc(V), op.rcmc_T(V)
    for row in (0, 1, 17, 31, 32, 63):
        C = op.dense_C(row)
        assert np.abs(U[row] - C @ V[row]).max() < 1e-12
        assert np.abs(W[row] - C.T @ V[row]).max() < 1e-12


def test_rcmc_special_cases():
    p = SarParams(n_az=32, n_rg=64)
    op = rda.RDAOperator(p)
    V = _rand(op.shape, 5)
    # the zero-Doppler row has D = 1: no migration, C = I (sinc at integers)
    r0 = int(np.argmin(np.abs(op.geo.f_eta)))
    assert op.geo.f_eta[r0] == 0.0 and np.all(op.shift[r0] == 0.0)
    assert np.abs(op.rcmc(V)[r0] - V[r0]).max() < 1e-15
    # migration grows with |f_eta| (D decreases) and with R0 (space-variant shift, eq. 16)
    assert np.all(np.diff(op.shift[:, 0][np.argsort(np.abs(op.geo.f_eta))]) >= 0)
    assert np.all(np.diff(op.shift[-1]) > 0)
    # an integer migration is a cyclic shift, exactly; its transpose the inverse shift
    op.set_shift(3.0)
    assert np.abs(op.rcmc(V) - np.roll(V, -3, axis=1)).max() < 1e-15
    assert np.abs(op.rcmc_T(V) - np.roll(V, 3, axis=1)).max() < 1e-15


def test_range_segment_factorisation():
    """G = F_eta^-1 . [range sweep, G body] . F_eta and M likewise: the split the GPU path uses
    (the azimuth sweeps of the CSA path, a different range sweep)."""
    p = SarParams(n_az=64, n_rg=96)
    op = rda.RDAOperator(p)
    X = _rand(op.shape, 6)
    g = csa.fft_az(op.range_segment(csa.fft_az(X), conj=True), inverse=True)
    m = csa.fft_az(op.range_segment(csa.fft_az(X), conj=False), inverse=True)
    assert np.abs(g - op.G(X)).max() < 1e-12 * np.abs(g).max()
    assert np.abs(m - op.M(X)).max() < 1e-12 * np.abs(m).max()


@pytest.mark.parametrize("p,targets", [
    (SarParams(n_az=128, n_rg=128), [(64, 64, 1.0), (10, 100, np.exp(0.7j)), (120, 3, 2 * np.exp(-2j))]),
    (SarParams(n_az=256, n_rg=4096), [(128, 100, 1.0), (40, 2000, 1j), (200, 3900, -1.0)]),
])
def test_rda_focusing_and_paper_pslr(p, targets):
    op = rda.RDAOperator(p)
    img = op.M(echo.exact_echo(p, targets))
    th = _theory(p)
    for (i, j, s) in targets:
        win = metrics.chip(np.abs(img), i, j, size=8)
        assert np.unravel_index(np.argmax(win), win.shape) == (4, 4)
        v = img[i, j]
        assert abs(np.angle(v / s)) < GOLD["phase_tol_rad"]
        assert abs(abs(v) / abs(s) / th["peak"] - 1.0) < GOLD["peak_rel_tol"]
        q = metrics.point_target_quality(img, i, j, p)
        assert abs(q["irw_rg"] / th["irw_rg"] - 1) < GOLD["irw_rel_tol"], q
        assert abs(q["irw_az"] / th["irw_az"] - 1) < GOLD["irw_rel_tol"], q
        assert abs(q["pslr_az"] - PAPER_RDA_PSLR_DB) < GOLD["pslr_tol_db"], q
        if 8 <= j < p.n_rg - 8:   # torus edge (R5), as for CSA
            assert abs(q["pslr_rg"] - PAPER_RDA_PSLR_DB) < GOLD["pslr_tol_db"], q


def test_csrda_ita_recovers_targets():
    p = SarParams(n_az=128, n_rg=128)
    op = rda.RDAOperator(p)
    tg = [(64, 64, 1.0), (10, 100, np.exp(0.7j)), (120, 3, 2 * np.exp(-2j)), (40, 30, 1j)]
    mask = (np.random.default_rng(1).random(op.shape) < 0.3).astype(float)
    Y = echo.exact_echo(p, tg) * mask
    X = ita.ita(op, Y, mask, thr="soft", rule="k", k=8, mu=1.0, iters=30)
    top = set(np.argsort(-np.abs(X).ravel())[:4].tolist())
    assert top == {i * p.n_rg + j for (i, j, _) in tg}
    for (i, j, s) in tg:
        assert abs(np.angle(X[i, j] / s)) < 0.02


# ---- recorded-pulse range filter (NEXT-4: "replacing P_tau* with the transmitted pulse")
def _nlfm(p, kappa=4e17):
    """Non-linear FM pulse: chirp + cubic phase kappa t^3 (instantaneous frequency < F_r/2)."""
    return lambda t: np.exp(2j * np.pi * (0.5 * p.Kr * t ** 2 + kappa * t ** 3))


def _replica(p, fn):
    L = int(round(p.Tr * p.Fr))
    return fn((np.arange(L) - (L - 1) / 2.0) / p.Fr)


def test_pulse_spectrum_closed_forms():
    n, Fr = 64, 60e6
    H = rda.pulse_spectrum(np.array([1.0 + 0j]), Fr, n)               # single sample: flat, unit
    assert np.abs(H - 1.0).max() < 1e-15
    for L in (7, 8):                                                  # rectangle: Dirichlet kernel
        H = rda.pulse_spectrum(np.ones(L), Fr, n)
        l = np.fft.fftfreq(n, d=1.0 / n)
        with np.errstate(invalid="ignore", divide="ignore"):
            D = np.where(l == 0, L, np.sin(np.pi * l * L / n) / np.sin(np.pi * l / n))
        assert np.abs(H - D / np.sqrt(L)).max() < 1e-12


def test_pulse_pair_theorem1():
    p = SarParams(n_az=64, n_rg=128)
    op = rda.RDAOperator(p, pulse=_replica(p, _nlfm(p)))
    X, Y = _rand(op.shape, 21), _rand(op.shape, 22)
    assert abs(np.vdot(op.G(X), Y) - np.vdot(X, op.M(Y))) / abs(np.vdot(X, op.M(Y))) < 1e-12


def test_nonchirp_echo_focuses_with_the_replica_only():
    """NLFM echo (eq. 1-3 with the cubic-phase pulse): the replica-filter pair focuses each
    target to its pixel with phase arg(sigma) - pi/4 (the matched filter cancels the range
    spectrum's phase; the azimuth stationary-phase -pi/4 that the chirp P_tau's missing +pi/4
    cancels for the chirp pair stays), peak 333.7 sqrt(F_r/B_r) |sigma| (|H|^2 = F_r/B_r in
    band), the theoretical IRW and the sinc PSLR; the chirp filter misfocuses the same echo."""
    p = SarParams(n_az=128, n_rg=256)
    tg = [(64, 128, np.exp(0.4j)), (20, 40, 1.0)]
    Y = echo.exact_echo(p, tg, pulse=_nlfm(p))
    img = rda.RDAOperator(p, pulse=_replica(p, _nlfm(p))).M(Y)
    bad = rda.RDAOperator(p).M(Y)
    th = _theory(p)
    for (i, j, s) in tg:
        win = metrics.chip(np.abs(img), i, j, size=8)
        assert np.unravel_index(np.argmax(win), win.shape) == (4, 4)
        assert abs(np.angle(img[i, j] / s * np.exp(0.25j * np.pi))) < GOLD["phase_tol_rad"]
        assert abs(abs(img[i, j]) / (th["peak"] * np.sqrt(p.Fr / (p.Kr * p.Tr))) - 1) < GOLD["peak_rel_tol"]
        q = metrics.point_target_quality(img, i, j, p)
        assert abs(q["irw_rg"] / th["irw_rg"] - 1) < GOLD["irw_rel_tol"], q
        assert abs(q["pslr_rg"] - GOLD["pslr_sinc_db"]) < GOLD["pslr_tol_db"], q
        assert abs(bad[i, j]) < 0.5 * abs(img[i, j])

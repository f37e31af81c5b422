"""Float64 stripmap echo model: exact point-target echo and inverse-CSA echo.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Passages followed:
  * eq. 1-3: s = W_tau sigma (x) h + n0, h = azimuth modulation (x) range pulse;
    y = H x + n0.  Written out per point target with the exact slant range:
      Y[(i_k + m) mod n_az, j' mod n_rg] += sigma_k exp(+j pi Kr t^2) exp(-j 4 pi fc R_km / c)
      R_km = sqrt(R_k^2 + (Vr m / PRF)^2),  t = tau_{j'} - 2 R_km / c,  |t| <= Tr/2,
    m in [-floor(Na/2), Na - floor(Na/2)), rectangular aperture of Na lines, no antenna
    weighting (R5 torus grid, R6 aperture, R7 gate mapping).
    Sum order: targets in list order, then m ascending, then j' ascending.
  * inverting a focusing procedure simulates raw echoes "in a more economical way":
    Y_clean = G(X_true) for the clutter configs (c2-c4).
"""
import numpy as np

C_LIGHT = 299792458.0


def aperture_lines(p):
    """Na = round(0.8 PRF^2 / Ka_ref), Ka_ref = 2 Vr^2 / (lambda_c R_ref) (R6) -> B_a = 0.8 PRF."""
    lam_c = C_LIGHT / p.fc
    ka = 2.0 * p.Vr ** 2 / (lam_c * p.R_ref)
    return int(round(0.8 * p.prf ** 2 / ka))


def exact_echo(p, targets, Na=None, pulse=None):
    """Exact periodic point-target echo on the n_az x n_rg torus (complex128).

    targets: iterable of (i, j, sigma) in list order.
    pulse: None for the chirp exp(+j pi Kr t^2) of eq. 1-3, or a callable t -> complex
    (vectorised, |t| <= Tr/2) for a non-chirp transmitted pulse (NEXT-4).
    """
    n_az, n_rg = p.n_az, p.n_rg
    if Na is None:
        Na = aperture_lines(p)
    Y = np.zeros((n_az, n_rg), dtype=np.complex128)
    m = np.arange(-(Na // 2), Na - Na // 2, dtype=np.float64)
    half = p.Tr / 2.0
    for (i_k, j_k, s_k) in targets:
        R_k = p.R_ref + (j_k - n_rg / 2) * C_LIGHT / (2.0 * p.Fr)
        R_km = np.sqrt(R_k ** 2 + (p.Vr * m / p.prf) ** 2)               # (Na,)
        # unwrapped gates j' covering |t| <= Tr/2 for the extreme R_km
        t_lo = 2.0 * R_km / C_LIGHT - half - 2.0 * p.R_ref / C_LIGHT       # tau_j' >= this
        j_lo = np.ceil(t_lo * p.Fr + n_rg / 2 - 1e-9).astype(np.int64)
        span = int(np.ceil(p.Tr * p.Fr)) + 2
        jj = j_lo[:, None] + np.arange(span, dtype=np.int64)[None, :]      # (Na, span)
        tau = 2.0 * p.R_ref / C_LIGHT + (jj - n_rg / 2) / p.Fr
        t = tau - 2.0 * R_km[:, None] / C_LIGHT
        ok = np.abs(t) <= half
        # phase in cycles, reduced mod 1 before exp (carrier term ~ 3e7 cycles)
        if pulse is None:
            cyc = 0.5 * p.Kr * t ** 2 - 2.0 * p.fc * R_km[:, None] / C_LIGHT
            val = s_k * np.exp(2j * np.pi * (cyc - np.floor(cyc)))
        else:
            cyc = -2.0 * p.fc * R_km[:, None] / C_LIGHT * np.ones_like(t)
            val = s_k * pulse(np.where(ok, t, 0.0)) * np.exp(2j * np.pi * (cyc - np.floor(cyc)))
        rows = ((i_k + m).astype(np.int64)[:, None] % n_az) * np.ones_like(jj)
        cols = jj % n_rg
        # m ascending then j' ascending: np.add.at accumulates in index order
        np.add.at(Y, (rows[ok], cols[ok]), val[ok])
    return Y


def inverse_csa_echo(op, X_true):
    """Y_clean = G(X_true): the approximated observation of the truth scene."""
    return op.G(X_true)

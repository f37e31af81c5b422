"""Float64 RDA operator pair (NEXT-2): the paper's own approximated observation (CSRDA).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Passages followed (PAPER.md = P:Lnnn):
  * eq. 14: M(Y) = F_eta^H { P_eta o C< F_eta [ P_tau o (Y F_tau) ] F_tau^H > }:
    range compression in the range-frequency domain, RCMC C in the range-Doppler domain,
    azimuth compression P_eta, inverse azimuth DFT.
  * eq. 15: P_eta = exp[-j pi f_eta^2 / K_a], P_tau = exp[-j pi f_tau^2 / K_r].
    With the echo exp(+j pi K_r t^2) exp(-j 4 pi f_c R / c) and the DFT kernel e^{-j 2 pi f t}
    (R3) the range matched filter is exp(+j pi f_tau^2 / K_r) (the printed sign is
    the opposite), the azimuth filter exp(-j pi f_eta^2 / K_a(R0)), K_a(R0) = 2 V_r^2 f_c/(c R0)
    — range-variant, as "P_eta(f_eta; tau)" says — times exp(+j 4 pi f_c R0 / c) so the focused
    pixel phase is arg sigma (R10, as for CSA).
  * eq. 16: U(f_eta, tau) = sum_tau~ V(f_eta, tau~) sinc(tau~ - (tau + dr(f_eta, tau)))
    with the migration dr = R0 (1/D - 1) converted to range cells (2 F_r / c, R23), the
    truncated kernel of 8 taps nearest the shifted position, indices on the torus
    (R5: the grid is periodic, so taps wrap).
  * eq. 17-18, eq. 23 and Theorem 1: G = M^H with D = C^T, the literal transpose
    of the truncated kernel, conjugate filters, inverse DFTs (unitary, R4).
  * P:L247 (NEXT-4, non-chirp pulses): "replacing P_tau* with the transmitted pulse": given
    the recorded pulse samples s_m at tau_m = (m - (L-1)/2)/F_r, G's range filter is its
    spectrum H(f_l) = sum_m s_m exp(-j 2 pi f_l tau_m) / sqrt(sum_m |s_m|^2) (signed bins
    f_l, unit mean |H|^2) and M's is conj(H) (the matched filter), R38.
Plain definition, written out: the RCMC is applied row by row as an explicit gather of the
8 taps (C) and its transpose as the matching scatter-add (D); no blocking or fusion.
"""
import numpy as np

from .csa import C_LIGHT, CSAGeometry, fft_az, fft_rg

TAPS = 8  # truncated sinc kernel: 8 taps (halfwidth 4)


def pulse_spectrum(pulse, Fr, n):
    """H(f_l), l in fftfreq order, of pulse samples s_m at tau_m = (m - (L-1)/2)/F_r, normalised to
    unit mean |H|^2 (a direct sum, written out)."""
    s = np.asarray(pulse, dtype=np.complex128)
    tau = (np.arange(s.size) - (s.size - 1) / 2.0) / Fr
    f = np.fft.fftfreq(n, d=1.0 / Fr)
    H = np.exp(-2j * np.pi * f[:, None] * tau[None, :]) @ s
    return H / np.sqrt(np.sum(np.abs(s) ** 2))


class RDAOperator:
    """M (RDA focusing, eq. 14) and G = M^H (eq. 18, Theorem 1)."""

    def __init__(self, p, taps=TAPS, pulse=None):
        self.geo = CSAGeometry(p)          # axes, D(f_eta) (same definitions)
        self.p = p
        self.taps = taps
        self.shape = (p.n_az, p.n_rg)
        g = self.geo
        n_rg = p.n_rg
        # filters, in cycles (phase / 2 pi), then unit-modulus screens
        self.ptau = g.expc(0.5 * g.f_tau ** 2 / p.Kr)[None, :]                      # exp(+j pi f^2/K_r)
        if pulse is not None:
            self.ptau = np.conj(pulse_spectrum(pulse, p.Fr, n_rg))[None, :]
        lam = C_LIGHT / p.fc
        R0 = g.R0[None, :]
        f = g.f_eta[:, None]
        cyc = -0.5 * f ** 2 * lam * R0 / (2.0 * p.Vr ** 2) + 2.0 * p.fc * R0 / C_LIGHT   # -pi f^2/K_a + 4 pi fc R0/c
        self.peta = g.expc(cyc)
        # migration in range cells at output gate j of Doppler row i: dr = R0 (1/D - 1) 2 F_r / c
        self.set_shift((R0 * (1.0 / g.D[:, None] - 1.0)) * (2.0 * p.Fr / C_LIGHT))    # (n_az, n_rg)

    def set_shift(self, shift):
        """Taps of the truncated kernel for a migration table `shift` (range cells)."""
        n_rg, taps = self.shape[1], self.taps
        self.shift = np.broadcast_to(np.asarray(shift, dtype=np.float64), self.shape).copy()
        pos = np.arange(n_rg)[None, :] + self.shift
        base = np.floor(pos).astype(np.int64) - (taps // 2 - 1)                      # first of the 8 taps
        t = np.arange(taps)[None, None, :]
        self.idx_unwrapped = base[:, :, None] + t                                    # (n_az, n_rg, taps)
        self.idx = np.mod(self.idx_unwrapped, n_rg)
        self.w = np.sinc(self.idx_unwrapped - pos[:, :, None])                        # sinc(tau~ - (tau + dr))

    # RCMC C (eq. 16) and its transpose D (eq. 17 with D = C^T, eq. 23)
    def rcmc(self, V):
        rows = np.arange(self.shape[0])[:, None, None]
        return np.sum(self.w * V[rows, self.idx], axis=2)

    def rcmc_T(self, U):
        out = np.zeros(self.shape, np.complex128)
        rows = np.broadcast_to(np.arange(self.shape[0])[:, None, None], self.idx.shape)
        np.add.at(out, (rows, self.idx), self.w * U[:, :, None])
        return out

    def M(self, Y):
        """F_eta -> F_tau -> P_tau -> F_tau^-1 -> C -> P_eta -> F_eta^-1 (eq. 14; F_eta and the
        range-frequency filter commute, so the azimuth DFT may come first)."""
        U = fft_az(np.asarray(Y, dtype=np.complex128))
        U = fft_rg(fft_rg(U) * self.ptau, inverse=True)
        U = self.rcmc(U) * self.peta
        return fft_az(U, inverse=True)

    def G(self, X):
        """The inverse of each focusing step in reverse order (eq. 18): F_eta -> P_eta* -> D ->
        F_tau -> P_tau* -> F_tau^-1 -> F_eta^-1."""
        U = fft_az(np.asarray(X, dtype=np.complex128)) * np.conj(self.peta)
        U = self.rcmc_T(U)
        U = fft_rg(fft_rg(U) * np.conj(self.ptau), inverse=True)
        return fft_az(U, inverse=True)

    def A(self, X, mask):
        return self.G(X) * mask

    def AH(self, R, mask):
        return self.M(R * mask)

    def range_segment(self, U, conj):
        """One range sweep in the range-Doppler domain: G body (conj=True: P_eta* D F P_tau* F^-1)
        or M body (conj=False: F P_tau F^-1 C P_eta)."""
        if conj:
            return fft_rg(fft_rg(self.rcmc_T(U * np.conj(self.peta))) * np.conj(self.ptau), inverse=True)
        return self.rcmc(fft_rg(fft_rg(U) * self.ptau, inverse=True)) * self.peta

    def dense_C(self, row):
        """The row's RCMC matrix C[j, tau~] (eq. 23, built independently of rcmc())."""
        n = self.shape[1]
        C = np.zeros((n, n))
        j = np.arange(n)
        pos = j + self.shift[row]
        for jj in range(n):
            lo = int(np.floor(pos[jj])) - (self.taps // 2 - 1)
            for k in range(lo, lo + self.taps):
                C[jj, k % n] += np.sinc(k - pos[jj])
        return C

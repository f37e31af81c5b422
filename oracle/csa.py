"""Float64 CSA operator pair: focusing M and approximated observation G = M^H.

TEST INFRASTRUCTURE ONLY. Nothing under oracle/ may be imported by the product
path (paper_1302_3120_b200/); only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs use it.

Passages followed (PAPER.md = P:Lnnn):
  * eq. 10: focusing  X~ = M Y, M a chain of 1-D frequency-domain operators.
  * eq. 11: approximated observation G = M^{-1}.
  * P:L193-197 (III-C i, ii): the inverse takes the inverse DFT of each DFT and the
    conjugate of each phase multiply, in reverse order; "keep the throwaway
    consistent between the pairs" -> unitary DFTs (R4).
  * Theorem 1: G is linear and G^H = M.
  * P:L243 (III-D): the approximated observation may be derived from the inverse of
    the Chirp-Scaling Algorithm.  PAPER.md prints no CSA phase function; the chirp-
    scaling phase screens below are the standard zero-squint CSA (Cumming2004, cited
    at P:L40) in the reading of SURVEY.md 8(c).2 (R1, R3, R7, R9, R10).

Plain definition, written out (no blocking or fusion):
    M(Y) = F_eta^-1( Phi3 o F_tau^-1( Phi2 o F_tau( Phi1 o F_eta(Y) ) ) )
    G(X) = F_eta^-1( Phi1* o F_tau^-1( Phi2* o F_tau( Phi3* o F_eta(X) ) ) )
with F_eta = fft over axis 0 (rows = azimuth), F_tau = fft over axis 1 (range),
norm="ortho", kernel exp(-2 pi i n k / N) / sqrt(N), bins in fftfreq order.

Phases are evaluated in fp64 *cycles*, reduced mod 1 before exp (the azimuth-
compression term reaches ~3e7 cycles).
"""
import numpy as np
import scipy.fft as sfft

C_LIGHT = 299792458.0

_WORKERS = -1  # scipy.fft threads: all host cores (library primitive)


def fft_az(A, inverse=False):
    f = sfft.ifft if inverse else sfft.fft
    return f(A, axis=0, norm="ortho", workers=_WORKERS)


def fft_rg(A, inverse=False):
    f = sfft.ifft if inverse else sfft.fft
    return f(A, axis=1, norm="ortho", workers=_WORKERS)


class CSAGeometry:
    """Axes and per-Doppler-bin CSA quantities.

    p: object with fc, Kr, Tr, Fr, prf, Vr, R_ref, squint, n_az, n_rg (inputs.configs.SarParams).
    """

    def __init__(self, p):
        if p.squint != 0.0:
            raise ValueError("only zero squint is supported (DESIGN.md R29)")
        self.p = p
        c = C_LIGHT
        n_az, n_rg = p.n_az, p.n_rg
        j = np.arange(n_rg, dtype=np.float64)
        # range gate j: two-way time and slant range, scene-centre convention (R7)
        self.tau = 2.0 * p.R_ref / c + (j - n_rg / 2) / p.Fr
        self.R0 = p.R_ref + (j - n_rg / 2) * c / (2.0 * p.Fr)
        # Doppler and range-frequency bins in fftfreq order (R9)
        self.f_eta = np.fft.fftfreq(n_az, d=1.0 / p.prf)
        self.f_tau = np.fft.fftfreq(n_rg, d=1.0 / p.Fr)
        # range-migration factor, modified range FM rate, reference time (8(c).2)
        self.D = np.sqrt(1.0 - (c * self.f_eta / (2.0 * p.Vr * p.fc)) ** 2)
        self.Km = p.Kr / (1.0 - p.Kr * c * p.R_ref * self.f_eta ** 2 / (2.0 * p.Vr ** 2 * p.fc ** 3 * self.D ** 3))
        self.tau_ref = 2.0 * p.R_ref / (c * self.D)

    # --- phase screens, in cycles (phase / 2 pi), fp64 -------------------------------
    def phi1_cycles(self):
        """Chirp scaling: exp{+j pi Km (1/D - 1)(tau_j - tau_ref)^2}."""
        D, Km = self.D[:, None], self.Km[:, None]
        dt = self.tau[None, :] - self.tau_ref[:, None]
        return 0.5 * Km * (1.0 / D - 1.0) * dt ** 2

    def phi2_cycles(self):
        """Range compression + bulk RCMC: exp{+j pi D f^2/Km + j (4 pi/c) R_ref (1/D - 1) f}."""
        D, Km = self.D[:, None], self.Km[:, None]
        f = self.f_tau[None, :]
        return 0.5 * D * f ** 2 / Km + (2.0 / C_LIGHT) * self.p.R_ref * (1.0 / D - 1.0) * f

    def phi3_cycles(self):
        """Azimuth compression + residual phase:
        exp{+j (4 pi/c) fc D R0 - j (4 pi/c^2) Km (1 - D)(R0 - R_ref)^2 / D^2}."""
        D, Km = self.D[:, None], self.Km[:, None]
        R0 = self.R0[None, :]
        return (2.0 / C_LIGHT) * self.p.fc * D * R0 \
            - (2.0 / C_LIGHT ** 2) * Km * (1.0 - D) * (R0 - self.p.R_ref) ** 2 / D ** 2

    @staticmethod
    def expc(cyc):
        """exp(2 pi i cyc) with the argument reduced mod 1 in fp64 first."""
        frac = cyc - np.floor(cyc)
        return np.exp(2j * np.pi * frac)

    def screens(self):
        return (self.expc(self.phi1_cycles()), self.expc(self.phi2_cycles()), self.expc(self.phi3_cycles()))


class CSAOperator:
    """M (focusing, eq. 10 with CSA) and G = M^H (approximated observation, eq. 11)."""

    def __init__(self, p):
        self.geo = CSAGeometry(p)
        self.shape = (p.n_az, p.n_rg)
        self._scr = None

    @property
    def phi(self):
        if self._scr is None:
            self._scr = self.geo.screens()
        return self._scr

    def M(self, Y):
        """Focusing chain: F_eta -> Phi1 -> F_tau -> Phi2 -> F_tau^-1 -> Phi3 -> F_eta^-1."""
        P1, P2, P3 = self.phi
        U = fft_az(np.asarray(Y, dtype=np.complex128))
        U = U * P1
        U = fft_rg(U)
        U = U * P2
        U = fft_rg(U, inverse=True)
        U = U * P3
        return fft_az(U, inverse=True)

    def G(self, X):
        """Approximated observation: the inverse of each focusing step in reverse order
        (P:L193-197): F_eta -> Phi3* -> F_tau -> Phi2* -> F_tau^-1 -> Phi1* -> F_eta^-1."""
        P1, P2, P3 = self.phi
        U = fft_az(np.asarray(X, dtype=np.complex128))
        U = U * np.conj(P3)
        U = fft_rg(U)
        U = U * np.conj(P2)
        U = fft_rg(U, inverse=True)
        U = U * np.conj(P1)
        return fft_az(U, inverse=True)

    # A = Theta o G and A^H = M(Theta o .) (eq. 24-25; mask generalised to
    # an elementwise 0/1 array, R21)
    def A(self, X, mask):
        return self.G(X) * mask

    def AH(self, R, mask):
        return self.M(R * mask)

    def range_segment(self, U, conj):
        """One range sweep on a (Doppler, range-time) array: the G body (conj=True:
        Phi3* F Phi2* F^-1 Phi1*) or the M body (conj=False: Phi1 F Phi2 F^-1 Phi3).
        Used by the per-sweep parity tests."""
        P1, P2, P3 = self.phi
        if conj:
            return fft_rg(fft_rg(U * np.conj(P3)) * np.conj(P2), inverse=True) * np.conj(P1)
        return fft_rg(fft_rg(U * P1) * P2, inverse=True) * P3


def dft_matrix(n, inverse=False):
    """Naive unitary DFT matrix F[k, m] = exp(-+2 pi i k m / n) / sqrt(n) (for tiny-grid pins)."""
    k = np.arange(n)
    s = 1.0 if inverse else -1.0
    return np.exp(s * 2j * np.pi * np.outer(k, k) / n) / np.sqrt(n)

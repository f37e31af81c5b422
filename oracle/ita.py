"""Float64 iterative thresholding (ITA) for the approximated-observation CS-SAR model.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Passages followed:
  * eq. 7-9: x <- E_{q, lambda mu}(x + mu A^H (y_s - A x)); soft threshold
    e_{1,sigma}(x) = sgn(x)(|x| - sigma) for |x| >= sigma, else 0 (eq. 9), with complex
    sgn(b) = b/|b| (R14) and strict survival |b| > sigma (R13; for soft the
    value at |b| = sigma is 0 either way).
  * eq. 25 and Algorithm 1: X0 = 0; Residue R = Y_s - Theta o G(X);
    MF on residue dX = M(Theta o R); Thresholding X <- E(X + mu dX).
  * lambda rule: lambda_i = |b_mu(x_i)|_{k+1} / mu_i, so sigma_i = lambda_i mu_i =
    the (k+1)-th largest |b| (R13).
  * q = 1/2 half thresholding: P:L102 says e_{q,sigma} is analytic for q = 1/2 but does not
    print it; the operator of the cited L1/2 theory (Xu2010) is used (R15):
      h(t) = (2/3) t [1 + cos(2 pi/3 - (2/3) arccos((lm/8)(t/3)^(-3/2)))] for t > (54^(1/3)/4) lm^(2/3)
    written in the k-rule-normalised form with sigma = (54^(1/3)/4) lm^(2/3).
  * iteration count = number of X updates; output X_I (R18).
  * adaptive step (NEXT-1; eq. 27, the strategy of the cited Blumensath2010):
    mu_i = ||dX_k||^2 / ||Theta G(dX_k)||^2 with dX_k = dX on the support of X_i (DESIGN.md
    R20) — the printed ratio is the reciprocal of a valid step (R11), so the
    normalised-IHT form of the cited source is used; mu_i = 1 when the support is empty or
    the denominator vanishes.  With the k-rule sigma_i = |b|_(k+1) of b = X + mu_i dX;
    with a fixed lambda sigma_i = lambda mu_i (soft) / the half jump point of lambda mu_i.
  * q = 0 (hard) and q = 2/3 thresholds (NEXT-4; P:L102 lists q = 0, 1/2, 2/3, 1 as the
    analytic cases): hard keeps |b| > sigma; 2/3 is the closed-form L2/3 minimiser (twothirds).
  * tolerance stopping (NEXT-4, default tol 1e-6 at S:L387; the paper runs a
    fixed 100 iterations): stop when ||X_(i+1) - X_i||_F <= tol ||X_i||_F.
"""
import numpy as np

HALF_LM_PER_SIGMA32 = np.sqrt(96.0) / 9.0   # lambda*mu = (sqrt(96)/9) sigma^(3/2)


def soft(b, sigma):
    """e_{1,sigma} (eq. 9) applied componentwise, phase preserving, strict survival |b| > sigma."""
    b = np.asarray(b, dtype=np.complex128)
    a = np.abs(b)
    out = np.zeros_like(b)
    keep = a > sigma
    out[keep] = b[keep] * (1.0 - sigma / a[keep])
    return out


def half(b, sigma):
    """q = 1/2 thresholding in k-rule form: for |b| > sigma,
    E(b) = (b/|b|) (2/3)|b| [1 + cos(2 pi/3 - (2/3) arccos(2^(-1/2) (sigma/|b|)^(3/2)))]."""
    b = np.asarray(b, dtype=np.complex128)
    a = np.abs(b)
    out = np.zeros_like(b)
    keep = a > sigma
    if sigma == 0.0:
        return b.copy()
    ak = a[keep]
    phi = np.arccos(2.0 ** -0.5 * (sigma / ak) ** 1.5)
    mag = (2.0 / 3.0) * ak * (1.0 + np.cos(2.0 * np.pi / 3.0 - (2.0 / 3.0) * phi))
    out[keep] = b[keep] / ak * mag
    return out


def hard(b, sigma):
    """q = 0 (NEXT-4; "analytically specified when q = 0"): keep b where |b| > sigma.
    Penalty lambda mu ||x||_0 in the convention of the half operator: sigma = sqrt(lambda mu)."""
    b = np.asarray(b, dtype=np.complex128)
    return np.where(np.abs(b) > sigma, b, 0.0)


def twothirds_lm_from_sigma(sigma):
    """lambda mu whose L2/3 jump point (2/3)(3 (lambda mu)^3)^(1/4) equals sigma."""
    return ((1.5 * sigma) ** 4 / 3.0) ** (1.0 / 3.0)


def twothirds(b, sigma):
    """q = 2/3 (NEXT-4): the closed-form minimiser of (x - t)^2 + lm |x|^(2/3) (the
    L2/3 thresholding of the cited Lq theory), t = |b|, phase preserved, in the k-rule form
    with lm = twothirds_lm_from_sigma(sigma):  for t > sigma
      psi = arccosh(27 t^2 / (16 lm^(3/2))),  phi = (2/sqrt(3)) lm^(1/4) sqrt(cosh(psi/3)),
      x = ((phi + sqrt(2 t / phi - phi^2)) / 2)^3."""
    b = np.asarray(b, dtype=np.complex128)
    if sigma == 0.0:
        return b.copy()
    a = np.abs(b)
    out = np.zeros_like(b)
    keep = a > sigma
    t = a[keep]
    lm = twothirds_lm_from_sigma(sigma)
    psi = np.arccosh(27.0 * t ** 2 / (16.0 * lm ** 1.5))
    phi = (2.0 / np.sqrt(3.0)) * lm ** 0.25 * np.sqrt(np.cosh(psi / 3.0))
    mag = ((phi + np.sqrt(2.0 * t / phi - phi ** 2)) / 2.0) ** 3
    out[keep] = b[keep] / t * mag
    return out


def half_sigma_from_lm(lm):
    """Jump point of half thresholding for penalty weight lambda*mu: (54^(1/3)/4)(lambda mu)^(2/3)."""
    return (54.0 ** (1.0 / 3.0) / 4.0) * lm ** (2.0 / 3.0)


def kth_largest_mag(b, k):
    """|b|_(k): the k-th largest magnitude, 1-indexed.  The order statistic is taken
    with a library selection (np.partition puts exactly the value a full descending sort
    would put at position k - 1 there; ties and zeros included)."""
    a = np.abs(np.asarray(b)).reshape(-1)
    n = a.size
    return np.partition(a, n - k)[n - k]


def sigma_k_rule(b, k):
    """sigma = lambda_i mu_i = |b|_(k+1). Requires 1 <= k < n."""
    n = np.asarray(b).size
    if not (1 <= k < n):
        raise ValueError("k must satisfy 1 <= k < n")
    return kth_largest_mag(b, k + 1)


def threshold(b, sigma, thr):
    return {"soft": soft, "half": half, "hard": hard, "twothirds": twothirds}[thr](b, sigma)


def sigma_fixed_lambda(lam, mu, thr):
    lm = lam * mu
    if thr == "soft":
        return lm
    if thr == "half":
        return half_sigma_from_lm(lm)
    if thr == "hard":
        return np.sqrt(lm)
    return (2.0 / 3.0) * (3.0 * lm ** 3) ** 0.25


def lambda_from_sigma(sigma, mu, thr):
    """lambda_i = the penalty weight whose threshold is sigma_i, divided by mu_i."""
    if thr == "soft":
        return sigma / mu
    if thr == "half":
        return HALF_LM_PER_SIGMA32 * sigma ** 1.5 / mu
    if thr == "hard":
        return sigma ** 2 / mu
    return twothirds_lm_from_sigma(sigma) / mu


def adaptive_mu(op, dX, X, mask):
    """eq. 27 step (module docstring): ||dX_k||^2 / ||Theta G(dX_k)||^2, dX_k = dX on supp(X)."""
    supp = np.asarray(X) != 0
    if not supp.any():
        return 1.0
    dXk = np.where(supp, dX, 0.0)
    num = float(np.vdot(dXk, dXk).real)
    g = np.asarray(mask, dtype=np.float64) * op.G(dXk)
    den = float(np.vdot(g, g).real)
    return num / den if den > 0.0 and num > 0.0 else 1.0


def ita(op, Y, mask, *, thr="soft", rule="k", k=None, lam=None, mu=1.0, iters=10, X0=None, log=None,
        tol=0.0, info=None):
    """Algorithm 1 with A = Theta o G. Returns X_I (complex128).

    op: oracle.csa.CSAOperator (or rda.RDAOperator); Y: echo (zero-filled where mask == 0);
    mask: 0/1 array.  mu: a positive step, or "adaptive" for the eq. 27 rule (adaptive_mu).
    log (optional list) receives per-iteration dicts: sigma, lam, mu, support, resid2, gap.
    tol > 0 (NEXT-4; "stop at max_iters or when ||X^(i+1) - X^(i)||_F <= tol ||X^(i)||_F"):
    stop after the first such update.  info (optional dict) receives iters = updates performed.
    """
    Y = np.asarray(Y, dtype=np.complex128)
    m = np.asarray(mask, dtype=np.float64)
    X = np.zeros(Y.shape, np.complex128) if X0 is None else np.asarray(X0, dtype=np.complex128).copy()
    if info is not None:
        info["iters"] = 0
    for it in range(iters):
        R = m * (Y - op.G(X))                      # Residue (Alg. 1 line 2)
        dX = op.M(R)                               # MF on residue (line 3); Theta already applied
        mu_i = adaptive_mu(op, dX, X, m) if mu == "adaptive" else mu
        b = X + mu_i * dX                          # b_mu(x_i)
        if rule == "k":
            sigma = sigma_k_rule(b, k)
        else:
            sigma = sigma_fixed_lambda(lam, mu_i, thr)
        Xn = threshold(b, sigma, thr)              # Thresholding (line 4)
        if log is not None:
            a = np.sort(np.abs(b).reshape(-1))[::-1]
            entry = dict(sigma=float(sigma), mu=float(mu_i), support=int(np.count_nonzero(Xn)),
                         resid2=float(np.vdot(R, R).real))
            entry["lam"] = float(lambda_from_sigma(sigma, mu_i, thr))
            if rule == "k":
                entry["gap"] = float((a[k - 1] - a[k]) / a[k]) if a[k] > 0 else float("inf")
            log.append(entry)
        done = tol > 0.0 and np.linalg.norm(Xn - X) <= tol * np.linalg.norm(X)
        X = Xn
        if info is not None:
            info["iters"] = it + 1
        if done:
            break
    return X


def objective_soft(op, X, Y, mask, lam):
    """F(X) = 1/2 ||Theta(Y - G X)||^2 + lambda ||X||_1 (eq. 6 with the 1/2 of eq. 7's scaling, R12)."""
    r = np.asarray(mask) * (Y - op.G(X))
    return 0.5 * float(np.vdot(r, r).real) + lam * float(np.abs(X).sum())

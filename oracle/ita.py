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


def half_sigma_from_lm(lm):
    """Jump point of half thresholding for penalty weight lambda*mu: (54^(1/3)/4)(lambda mu)^(2/3)."""
    return (54.0 ** (1.0 / 3.0) / 4.0) * lm ** (2.0 / 3.0)


def kth_largest_mag(b, k):
    """|b|_(k): the k-th largest magnitude, 1-indexed."""
    a = np.sort(np.abs(np.asarray(b)).reshape(-1))[::-1]
    return a[k - 1]


def sigma_k_rule(b, k):
    """sigma = lambda_i mu_i = |b|_(k+1). Requires 1 <= k < n."""
    n = np.asarray(b).size
    if not (1 <= k < n):
        raise ValueError("k must satisfy 1 <= k < n")
    return kth_largest_mag(b, k + 1)


def threshold(b, sigma, thr):
    return soft(b, sigma) if thr == "soft" else half(b, sigma)


def sigma_fixed_lambda(lam, mu, thr):
    lm = lam * mu
    return lm if thr == "soft" else half_sigma_from_lm(lm)


def ita(op, Y, mask, *, thr="soft", rule="k", k=None, lam=None, mu=1.0, iters=10, X0=None, log=None):
    """Algorithm 1 with A = Theta o G. Returns X_I (complex128).

    op: oracle.csa.CSAOperator; Y: echo (zero-filled where mask == 0); mask: 0/1 array.
    log (optional list) receives per-iteration dicts: sigma, lam, support, resid2, gap, obj.
    """
    Y = np.asarray(Y, dtype=np.complex128)
    m = np.asarray(mask, dtype=np.float64)
    X = np.zeros(Y.shape, np.complex128) if X0 is None else np.asarray(X0, dtype=np.complex128).copy()
    for _ in range(iters):
        R = m * (Y - op.G(X))                      # Residue (Alg. 1 line 2)
        dX = op.M(R)                               # MF on residue (line 3); Theta already applied
        b = X + mu * dX                            # b_mu(x_i)
        if rule == "k":
            sigma = sigma_k_rule(b, k)
        else:
            sigma = sigma_fixed_lambda(lam, mu, thr)
        Xn = threshold(b, sigma, thr)              # Thresholding (line 4)
        if log is not None:
            a = np.sort(np.abs(b).reshape(-1))[::-1]
            entry = dict(sigma=float(sigma), support=int(np.count_nonzero(Xn)), resid2=float(np.vdot(R, R).real))
            entry["lam"] = float(sigma / mu) if thr == "soft" else float(HALF_LM_PER_SIGMA32 * sigma ** 1.5 / mu)
            if rule == "k":
                entry["gap"] = float((a[k - 1] - a[k]) / a[k]) if a[k] > 0 else float("inf")
            log.append(entry)
        X = Xn
    return X


def objective_soft(op, X, Y, mask, lam):
    """F(X) = 1/2 ||Theta(Y - G X)||^2 + lambda ||X||_1 (eq. 6 with the 1/2 of eq. 7's scaling, R12)."""
    r = np.asarray(mask) * (Y - op.G(X))
    return 0.5 * float(np.vdot(r, r).real) + lam * float(np.abs(X).sum())

"""Point-target image-quality measurement (IRW, PSLR) for the physics pins.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Method of P:L512 (Fig. 4 table): cut a 16x16 chip around the peak, upsample 16x by
zero-padding the 2-D spectrum, measure the -3 dB width (IRW, in input samples) and
the peak sidelobe ratio (PSLR, dB) along the range and azimuth cuts through the
peak.  Before upsampling, the range carrier ramp exp(+j 2 pi (fc/Fr) j) that the
CSA azimuth-compression phase leaves on the image is demodulated (R10).
"""
import numpy as np

C_LIGHT = 299792458.0


def chip(img, i0, j0, size=16):
    n_az, n_rg = img.shape
    ii = (np.arange(size) - size // 2 + i0) % n_az
    jj = (np.arange(size) - size // 2 + j0) % n_rg
    return img[np.ix_(ii, jj)]


def demodulate_range(ch, p, j0, size=16):
    """Remove exp(+j 2 pi (fc/Fr)(j - j0)) along range (R10)."""
    j = np.arange(size) - size // 2
    return ch * np.exp(-2j * np.pi * (p.fc / p.Fr) * j)[None, :]


def upsample2d(ch, factor=16):
    n0, n1 = ch.shape
    S = np.fft.fftshift(np.fft.fft2(ch))
    P = np.zeros((n0 * factor, n1 * factor), dtype=np.complex128)
    a0, a1 = (n0 * factor - n0) // 2, (n1 * factor - n1) // 2
    P[a0:a0 + n0, a1:a1 + n1] = S
    return np.fft.ifft2(np.fft.ifftshift(P)) * factor * factor


def _cut_metrics(cut, factor):
    a = np.abs(cut)
    pk = int(np.argmax(a))
    amax = a[pk]
    half = amax / np.sqrt(2.0)
    # -3 dB width by linear interpolation on each side
    l = pk
    while l > 0 and a[l] >= half:
        l -= 1
    r = pk
    while r < a.size - 1 and a[r] >= half:
        r += 1
    xl = l + (half - a[l]) / (a[l + 1] - a[l])
    xr = r - 1 + (a[r - 1] - half) / (a[r - 1] - a[r])
    irw = (xr - xl) / factor
    # main lobe: walk to first nulls (local minima)
    l = pk
    while l > 0 and a[l - 1] < a[l]:
        l -= 1
    r = pk
    while r < a.size - 1 and a[r + 1] < a[r]:
        r += 1
    side = np.concatenate([a[:l], a[r + 1:]])
    pslr = 20.0 * np.log10(side.max() / amax) if side.size else -np.inf
    return irw, pslr


def point_target_quality(img, i0, j0, p, size=16, factor=16):
    """Returns dict(irw_rg, irw_az [input samples], pslr_rg, pslr_az [dB])."""
    ch = demodulate_range(chip(img, i0, j0, size), p, j0, size)
    up = upsample2d(ch, factor)
    pi, pj = np.unravel_index(np.argmax(np.abs(up)), up.shape)
    irw_rg, pslr_rg = _cut_metrics(up[pi, :], factor)
    irw_az, pslr_az = _cut_metrics(up[:, pj], factor)
    return dict(irw_rg=irw_rg, irw_az=irw_az, pslr_rg=pslr_rg, pslr_az=pslr_az)

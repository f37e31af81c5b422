"""Seeded synthetic inputs: scenes, sampling masks, noise draws.

Shared by the oracle-side tests and the CUDA-side tests/bench. This module holds
none of the method's arithmetic: no phase screens, FFT chains, thresholds or
echo physics. The echo itself (exact point-target echo or inverse-CSA echo
G(X_true)) is computed by a caller-supplied function, so the oracle path passes
oracle.echo / oracle.csa and the bench passes the CUDA forward operator.

Recipe:
  seed_c = 13023120 + c; numpy.random.SeedSequence(seed_c).spawn(4) gives PCG64
  streams [positions, amplitudes/phases, mask, noise].
"""
from dataclasses import dataclass
from typing import Callable, Optional
import numpy as np

from .configs import Config

_CHUNK_ROWS = 1024


def streams(seed: int):
    ss = np.random.SeedSequence(seed)
    return [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(4)]


def _distinct_pixels(rng, n_total: int, count: int, exclude: Optional[np.ndarray] = None) -> np.ndarray:
    """`count` distinct linear pixel indices, uniform, none in `exclude` (sorted unique)."""
    chosen = np.empty(0, dtype=np.int64)
    excl = np.unique(exclude) if exclude is not None else np.empty(0, dtype=np.int64)
    while chosen.size < count:
        need = count - chosen.size
        draw = rng.integers(0, n_total, size=need + need // 8 + 16, dtype=np.int64)
        cand = np.unique(np.concatenate([chosen, draw]))
        if excl.size:
            cand = cand[~np.isin(cand, excl)]
        if cand.size > count:
            # keep the previously chosen ones plus a deterministic random subset of the new ones
            new = np.setdiff1d(cand, chosen, assume_unique=True)
            new = rng.permutation(new)[: count - chosen.size]
            cand = np.union1d(chosen, new)
        chosen = cand
    return chosen


def _rayleigh_unit(rng, m: int) -> np.ndarray:
    """Complex reflectivity with Rayleigh magnitude, E|s|^2 = 1, uniform phase."""
    return (rng.standard_normal(m) + 1j * rng.standard_normal(m)) / np.sqrt(2.0)


@dataclass
class Scene:
    """Truth scene: linear indices (sorted), complex reflectivities, grid shape."""
    idx: np.ndarray          # int64 linear pixel indices i*n_rg + j
    val: np.ndarray          # complex128 reflectivities
    shape: tuple
    targets: list            # [(i, j, sigma)] in list order for the exact echo (point configs)

    def dense(self, dtype=np.complex128) -> np.ndarray:
        X = np.zeros(self.shape, dtype=dtype)
        X.reshape(-1)[self.idx] = self.val.astype(dtype)
        return X


def make_scene(cfg: Config) -> Scene:
    p = cfg.params
    n_az, n_rg = p.n_az, p.n_rg
    n = n_az * n_rg
    r_pos, r_amp, _, _ = streams(cfg.seed)
    a = cfg.scene_args
    targets = []
    if cfg.scene == "points":
        idx_list = _distinct_pixels(r_pos, n, a["n_targets"])
        idx_list = r_pos.permutation(idx_list)          # list order = draw order
        ph = r_amp.uniform(0.0, 2 * np.pi, size=idx_list.size)
        vals = np.exp(1j * ph)
        for li, v in zip(idx_list, vals):
            targets.append((int(li // n_rg), int(li % n_rg), complex(v)))
        order = np.argsort(idx_list)
        return Scene(idx_list[order], vals[order], (n_az, n_rg), targets)
    if cfg.scene == "points_patch":
        P = a["patch"]
        pi0 = int(r_pos.integers(0, n_az - P + 1))
        pj0 = int(r_pos.integers(0, n_rg - P + 1))
        ii, jj = np.meshgrid(np.arange(pi0, pi0 + P), np.arange(pj0, pj0 + P), indexing="ij")
        patch_idx = (ii * n_rg + jj).reshape(-1).astype(np.int64)
        tgt = _distinct_pixels(r_pos, n, a["n_targets"], exclude=patch_idx)
        tgt = r_pos.permutation(tgt)
        amp = 10.0 ** r_amp.uniform(-1.0, 0.0, size=tgt.size)
        ph = r_amp.uniform(0.0, 2 * np.pi, size=tgt.size)
        tv = amp * np.exp(1j * ph)
        pv = _rayleigh_unit(r_amp, patch_idx.size) * np.sqrt(a["patch_var"])
        for li, v in zip(tgt, tv):
            targets.append((int(li // n_rg), int(li % n_rg), complex(v)))
        for li, v in zip(patch_idx, pv):
            targets.append((int(li // n_rg), int(li % n_rg), complex(v)))
        idx = np.concatenate([tgt, patch_idx])
        val = np.concatenate([tv, pv])
        order = np.argsort(idx)
        return Scene(idx[order], val[order], (n_az, n_rg), targets)
    if cfg.scene == "thomas":
        want = int(round(a["frac"] * n))
        chosen = np.empty(0, dtype=np.int64)
        while chosen.size < want:
            pi, pj = r_pos.integers(0, n_az), r_pos.integers(0, n_rg)
            m = r_pos.poisson(a["children"])
            off = np.rint(r_pos.normal(0.0, a["sigma_px"], size=(m, 2))).astype(np.int64)
            ci = (pi + off[:, 0]) % n_az
            cj = (pj + off[:, 1]) % n_rg
            new = np.setdiff1d(np.unique(ci * n_rg + cj), chosen)
            if chosen.size + new.size > want:
                new = new[: want - chosen.size]
            chosen = np.union1d(chosen, new)
        val = _rayleigh_unit(r_amp, chosen.size)
        return Scene(chosen, val, (n_az, n_rg), [])
    if cfg.scene in ("rayleigh", "rayleigh_bright"):
        m = int(round(a["frac"] * n))
        base = _distinct_pixels(r_pos, n, m)
        val = _rayleigh_unit(r_amp, base.size)
        if cfg.scene == "rayleigh_bright":
            nb = a["n_bright"]
            bright = _distinct_pixels(r_pos, n, nb, exclude=base)
            bv = a["bright_amp"] * np.exp(1j * r_amp.uniform(0, 2 * np.pi, size=nb))
            for li, v in zip(bright, bv):
                targets.append((int(li // n_rg), int(li % n_rg), complex(v)))
            idx = np.concatenate([base, bright])
            val = np.concatenate([val, bv])
            order = np.argsort(idx)
            return Scene(idx[order], val[order], (n_az, n_rg), targets)
        return Scene(base, val, (n_az, n_rg), [])
    if cfg.scene == "grid9":
        # P:L501 / P:L390: 9 targets "located at the center with intervals of 6 samples", unit
        # amplitude, uniform random phase (a 3 x 3 grid, R39)
        sp = a.get("spacing", 6)
        ph = r_amp.uniform(0.0, 2 * np.pi, size=9)
        ci, cj = n_az // 2, n_rg // 2
        for q in range(9):
            targets.append((ci + (q // 3 - 1) * sp, cj + (q % 3 - 1) * sp, complex(np.exp(1j * ph[q]))))
        idx = np.array([i * n_rg + j for i, j, _ in targets], dtype=np.int64)
        val = np.array([v for _, _, v in targets])
        order = np.argsort(idx)
        return Scene(idx[order], val[order], (n_az, n_rg), targets)
    raise ValueError(f"unknown scene recipe {cfg.scene}")


def make_mask(cfg: Config) -> np.ndarray:
    """Boolean sampling mask Theta (R21): i.i.d. Bernoulli per sample, or per azimuth line."""
    p = cfg.params
    _, _, r_mask, _ = streams(cfg.seed)
    if cfg.mask == "lines":
        keep = r_mask.random(p.n_az) < cfg.rate
        return np.repeat(keep[:, None], p.n_rg, axis=1)
    if cfg.mask == "full":
        return np.ones((p.n_az, p.n_rg), dtype=bool)
    if cfg.mask == "separable":
        # random azimuth lines at rate s_a, random range samples per kept line at rate
        # s_r, s_a : s_r = 1 : 5, s_a s_r = rate (so rate <= 1/5)
        if not 0.0 < cfg.rate <= 0.2:
            raise ValueError("separable 1:5 sampling needs 0 < rate <= 0.2")
        s_a, s_r = np.sqrt(cfg.rate / 5.0), np.sqrt(5.0 * cfg.rate)
        rows = r_mask.random(p.n_az) < s_a
        return rows[:, None] & (r_mask.random((p.n_az, p.n_rg)) < s_r)
    M = np.empty((p.n_az, p.n_rg), dtype=bool)
    for r0 in range(0, p.n_az, _CHUNK_ROWS):
        r1 = min(p.n_az, r0 + _CHUNK_ROWS)
        M[r0:r1] = r_mask.random((r1 - r0, p.n_rg)) < cfg.rate
    return M


def noise_unit(cfg: Config, dtype=np.complex128) -> np.ndarray:
    """Standard circular complex Gaussian draws CN(0, 1) for every sample (row-chunked)."""
    p = cfg.params
    _, _, _, r_noise = streams(cfg.seed)
    out = np.empty((p.n_az, p.n_rg), dtype=dtype)
    for r0 in range(0, p.n_az, _CHUNK_ROWS):
        r1 = min(p.n_az, r0 + _CHUNK_ROWS)
        g = r_noise.standard_normal((r1 - r0, p.n_rg, 2))
        out[r0:r1] = (g[..., 0] + 1j * g[..., 1]) / np.sqrt(2.0)
    return out


def add_noise_and_sample(Y_clean: np.ndarray, mask: np.ndarray, cfg: Config) -> np.ndarray:
    """Y = Theta o (Y_clean + n), n ~ CN(0, s2) with s2 = mean_{Theta=1}|Y_clean|^2 / 10^(SNR/10)
    (R22), rounded to complex64 (round-to-nearest-even)."""
    sig = np.mean(np.abs(Y_clean[mask]) ** 2) if mask.any() else 0.0
    s2 = sig / 10.0 ** (cfg.snr_db / 10.0)
    Y = np.zeros(Y_clean.shape, dtype=np.complex64)
    nz = noise_unit(cfg)
    Yn = Y_clean + np.sqrt(s2) * nz
    Y[mask] = Yn[mask].astype(np.complex64)
    return Y


def pack_mask_bits(mask: np.ndarray) -> np.ndarray:
    """1 bit per sample, row-major, LSB-first within uint32 words, rows padded to 32 bits."""
    n_az, n_rg = mask.shape
    words = (n_rg + 31) // 32
    pad = np.zeros((n_az, words * 32), dtype=np.uint8)
    pad[:, :n_rg] = mask
    b = np.packbits(pad, axis=1, bitorder="little")
    return np.ascontiguousarray(b).view("<u4").reshape(n_az, words)


@dataclass
class Problem:
    cfg: Config
    scene: Scene
    mask: np.ndarray         # bool (n_az, n_rg)
    Y: np.ndarray            # complex64 (n_az, n_rg), zero where mask == 0


def make_problem(cfg: Config, echo_fn: Callable[[Scene, Config], np.ndarray]) -> Problem:
    """echo_fn(scene, cfg) -> clean echo (complex, n_az x n_rg). Supplied by the caller."""
    scene = make_scene(cfg)
    mask = make_mask(cfg)
    Yc = echo_fn(scene, cfg)
    Y = add_noise_and_sample(Yc, mask, cfg)
    return Problem(cfg, scene, mask, Y)

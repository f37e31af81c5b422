"""The five BASELINE.json workload configurations, as plain data.

This module holds NO arithmetic of the method: it lists system parameters,
grid sizes, scene recipes, sampling recipes, solver settings and seeds.
Both the oracle-side tests and the CUDA-side tests/bench read it.

Readings of the configs (DESIGN.md "Readings" R16/R17/R21):
  * all configs share fc = 5.3 GHz, Kr = 20e12 Hz/s, Tr = 2.5 us, PRF = 1700 Hz,
    Vr = 7062 m/s, R_ref = 850 km, zero squint; Fr = 60 MHz except c4 (120 MHz).
  * mu = 1 for every config (admissible: ||Theta G||_2 <= 1, R11).
  * c3/c4 use soft thresholding with k = number of nonzero truth pixels (R16).
"""
from dataclasses import dataclass, field, replace

C_LIGHT = 299792458.0  # m/s (SPEC S:L53 core constants)


@dataclass(frozen=True)
class SarParams:
    """Table 1 fields used by the CSA operator."""
    fc: float = 5.3e9        # carrier frequency [Hz]
    Kr: float = 20e12        # range FM rate [Hz/s]
    Tr: float = 2.5e-6       # pulse duration [s]
    Fr: float = 60e6         # range sampling rate [Hz]
    prf: float = 1700.0      # pulse repetition frequency [Hz]
    Vr: float = 7062.0       # effective radar velocity [m/s]
    R_ref: float = 850e3     # reference (scene-centre) slant range [m]
    squint: float = 0.0      # [rad]; must be 0
    n_az: int = 128          # rows  = azimuth lines / Doppler bins
    n_rg: int = 128          # cols  = range gates / range-frequency bins


@dataclass(frozen=True)
class Config:
    name: str
    params: SarParams
    scene: str                   # scene recipe id (inputs.synth)
    scene_args: dict = field(default_factory=dict)
    echo: str = "exact"          # "exact" (periodic point-target echo) | "inverse_csa" (G(X_true))
    mask: str = "bernoulli"      # "bernoulli" per sample | "lines" per azimuth line | "separable" (1:5)
    rate: float = 0.5            # sampling rate
    snr_db: float = 30.0
    thr: str = "soft"            # "soft" (q=1, eq. 9) | "half" (q=1/2)
    rule: str = "k"              # "k" (P:L320 k-sparsity) | "lambda" (fixed lambda)
    k: int = 5
    lam: float = 0.0
    mu: float = 1.0
    iters: int = 50
    seed: int = 13023120


def _p(n_az, n_rg, **kw):
    return SarParams(n_az=n_az, n_rg=n_rg, **kw)


CONFIGS = {
    "c0": Config("c0", _p(128, 128), scene="points", scene_args=dict(n_targets=5, amp="unit"),
                 echo="exact", mask="bernoulli", rate=0.5, snr_db=30.0, thr="soft", rule="k",
                 k=5, iters=50, seed=13023120 + 0),
    "c1": Config("c1", _p(512, 512), scene="points_patch",
                 scene_args=dict(n_targets=40, amp="loguniform20", patch=32, patch_var=0.1),
                 echo="exact", mask="bernoulli", rate=0.5, snr_db=20.0, thr="half", rule="k",
                 k=round(0.02 * 512 * 512), iters=100, seed=13023120 + 1),
    "c2": Config("c2", _p(2048, 2048), scene="thomas",
                 scene_args=dict(frac=0.02, children=64, sigma_px=3.0),
                 echo="inverse_csa", mask="bernoulli", rate=0.3, snr_db=20.0, thr="soft", rule="k",
                 k=83886, iters=200, seed=13023120 + 2),
    "c3": Config("c3", _p(8192, 8192), scene="rayleigh_bright",
                 scene_args=dict(frac=0.01, n_bright=500, bright_amp=10.0),
                 echo="inverse_csa", mask="lines", rate=0.6, snr_db=15.0, thr="soft", rule="k",
                 k=671089 + 500, iters=100, seed=13023120 + 3),
    "c4": Config("c4", _p(32768, 16384, Fr=120e6), scene="rayleigh",
                 scene_args=dict(frac=0.005),
                 echo="inverse_csa", mask="bernoulli", rate=0.5, snr_db=20.0, thr="soft", rule="k",
                 k=2684355, iters=50, seed=13023120 + 4),
    # NEXT-3: the paper's reconstruction-ability experiment: 9 targets 6 samples
    # apart, 20 dB noise, k = 18, separable s_a : s_r = 1 : 5 sampling, 100
    # iterations; 256 x 256 stands in for the 180 x 180 scene (power-of-two grid, R33)
    "ra": Config("ra", _p(256, 256), scene="grid9", scene_args=dict(spacing=6),
                 echo="exact", mask="separable", rate=0.1, snr_db=20.0, thr="soft", rule="k",
                 k=18, iters=100, seed=13023120 + 10),
}


def get(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    if overrides:
        cfg = replace(cfg, **overrides)
    return cfg


def with_grid(cfg: Config, n_az: int, n_rg: int) -> Config:
    """Same recipe on a smaller grid (for parity cases the oracle finishes in seconds)."""
    p = replace(cfg.params, n_az=n_az, n_rg=n_rg)
    return replace(cfg, params=p)

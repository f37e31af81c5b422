"""Shared helpers for the GPU parity tests: seeded problems (inputs/ + oracle echo) and
comparison utilities.  Expected values always come from oracle/ (never from the CUDA path)."""
import functools

import numpy as np
import pytest

from inputs import configs, synth
from oracle import csa, echo

torch = pytest.importorskip("torch")


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rand_c(shape, seed, dtype=np.complex64):
    r = np.random.default_rng(seed)
    return ((r.standard_normal(shape) + 1j * r.standard_normal(shape)) / np.sqrt(2)).astype(dtype)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def to_host(t):
    return t.detach().cpu().numpy()


@functools.lru_cache(maxsize=2)
def oracle_op(params):
    """The fp64 CSA operator of a parameter set, cached (its three phase screens are the
    expensive part at c3/c4 sizes)."""
    return csa.CSAOperator(params)


def oracle_echo(scene, cfg):
    if cfg.echo == "exact":
        return echo.exact_echo(cfg.params, scene.targets)
    return echo.inverse_csa_echo(oracle_op(cfg.params), scene.dense())


@functools.lru_cache(maxsize=8)
def problem(name, n_az=None, n_rg=None, iters=None):
    cfg = configs.get(name)
    if n_az is not None:
        cfg = configs.with_grid(cfg, n_az, n_rg)
        if cfg.rule == "k" and name in ("c2", "c3", "c4"):
            # keep the truth-sparsity reading of k (R16) on the reduced grid
            sc = synth.make_scene(cfg)
            from dataclasses import replace
            cfg = replace(cfg, k=int(sc.idx.size))
    if iters is not None:
        from dataclasses import replace
        cfg = replace(cfg, iters=iters)
    return synth.make_problem(cfg, oracle_echo)


def mask_bits_dev(mask):
    return to_dev(synth.pack_mask_bits(mask).view(np.int32))


def mag2_f32(b):
    """|b|^2 with the GPU's explicit fp32 roundings: fl(fl(re*re) + fl(im*im))."""
    b = np.asarray(b, dtype=np.complex64)
    re = b.real.astype(np.float32)
    im = b.imag.astype(np.float32)
    return (re * re) + (im * im)

"""Mutation check of the RDA oracle pins (tests/test_oracle_rda.py): plausible mistakes in
oracle/rda.py — the transpose replaced by the gather, a flipped filter or migration sign, a
dropped carrier, a shifted tap window — must each fail at least one pin."""
import numpy as np
import pytest

from inputs.configs import SarParams
from oracle import rda

from tests import test_oracle_rda as T


def _focus_pin():
    T.test_rda_focusing_and_paper_pslr(SarParams(n_az=128, n_rg=128),
                                       [(64, 64, 1.0), (10, 100, np.exp(0.7j)), (120, 3, 2 * np.exp(-2j))])


PINS = (("theorem1", lambda: T.test_theorem1_adjoint((64, 96))),
        ("eq23", T.test_rcmc_is_eq23_matrix),
        ("special", T.test_rcmc_special_cases),
        ("focus", _focus_pin))


def _failed():
    out = []
    for name, pin in PINS:
        try:
            pin()
        except AssertionError:
            out.append(name)
    return out


def _patch_init(monkeypatch, after):
    orig = rda.RDAOperator.__init__

    def init(self, p, taps=rda.TAPS, pulse=None):
        orig(self, p, taps, pulse)
        after(self)
    monkeypatch.setattr(rda.RDAOperator, "__init__", init)


def test_transpose_replaced_by_gather_is_caught(monkeypatch):
    monkeypatch.setattr(rda.RDAOperator, "rcmc_T", lambda self, U: self.rcmc(U))
    assert "theorem1" in _failed()


def test_range_filter_sign_is_caught(monkeypatch):
    _patch_init(monkeypatch, lambda self: setattr(self, "ptau", np.conj(self.ptau)))
    assert "focus" in _failed()


def test_migration_sign_is_caught(monkeypatch):
    _patch_init(monkeypatch, lambda self: self.set_shift(-self.shift))
    assert _failed()


def test_dropped_carrier_is_caught(monkeypatch):
    def drop(self):
        g, p = self.geo, self.p
        f = g.f_eta[:, None]
        self.peta = g.expc(-0.5 * f ** 2 * (rda.C_LIGHT / p.fc) * g.R0[None, :] / (2.0 * p.Vr ** 2))
    _patch_init(monkeypatch, drop)
    assert "focus" in _failed()


@pytest.mark.parametrize("delta", [-1, 1])
def test_shifted_tap_window_is_caught(monkeypatch, delta):
    orig = rda.RDAOperator.set_shift

    def set_shift(self, shift):
        orig(self, shift)
        self.idx_unwrapped = self.idx_unwrapped + delta
        self.idx = np.mod(self.idx_unwrapped, self.shape[1])
        pos = np.arange(self.shape[1])[None, :] + self.shift
        self.w = np.sinc(self.idx_unwrapped - pos[:, :, None])
    monkeypatch.setattr(rda.RDAOperator, "set_shift", set_shift)
    assert "eq23" in _failed()

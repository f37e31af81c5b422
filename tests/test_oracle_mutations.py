"""Mutation check of the oracle pins: plausible transcription mistakes must fail a pin.

Each mutant patches one term of oracle/csa.py (a dropped term, a wrong sign, a wrong
index, a swapped screen) and re-runs the physics / anchor pins, which must now fail.
This shows the pins constrain the oracle rather than restate it.
"""
import numpy as np
import pytest

from inputs.configs import SarParams
from oracle import csa

from tests import test_oracle_operator as T_op  # noqa: E402
from tests import test_oracle_physics as T_ph  # noqa: E402


def _mutants():
    return {
        "phi2_linear_sign": ("phi2_cycles", lambda self: 0.5 * self.D[:, None] * self.f_tau[None, :] ** 2 / self.Km[:, None]
                             - (2.0 / csa.C_LIGHT) * self.p.R_ref * (1.0 / self.D[:, None] - 1.0) * self.f_tau[None, :]),
        "phi2_chirp_sign": ("phi2_cycles", lambda self: -0.5 * self.D[:, None] * self.f_tau[None, :] ** 2 / self.Km[:, None]
                            + (2.0 / csa.C_LIGHT) * self.p.R_ref * (1.0 / self.D[:, None] - 1.0) * self.f_tau[None, :]),
        "phi1_dropped": ("phi1_cycles", lambda self: np.zeros((self.p.n_az, self.p.n_rg))),
        "phi3_residual_dropped": ("phi3_cycles", lambda self: (2.0 / csa.C_LIGHT) * self.p.fc * self.D[:, None] * self.R0[None, :]),
        "phi3_carrier_D_missing": ("phi3_cycles", lambda self: (2.0 / csa.C_LIGHT) * self.p.fc * self.R0[None, :] + 0 * self.D[:, None]),
        "gate_offset_by_one": ("phi3_cycles", lambda self: (2.0 / csa.C_LIGHT) * self.p.fc * self.D[:, None] * (self.R0[None, :] + csa.C_LIGHT / (2 * self.p.Fr))),
    }


def _pins_fail(monkeypatch, attr, fn):
    monkeypatch.setattr(csa.CSAGeometry, attr, fn)
    failed = []
    for name, pin in (("anchors", T_op.test_survey_transcription_anchors),
                      ("focus", lambda: T_ph._focus_check(SarParams(n_az=128, n_rg=128), [(64, 64, 1.0), (10, 100, 1j)])),
                      ("focus_wide", T_ph.test_focus_wide_swath_range_dependence)):
        try:
            pin()
        except AssertionError:
            failed.append(name)
    return failed


@pytest.mark.parametrize("mutant", list(_mutants().keys()))
def test_mutant_is_caught(monkeypatch, mutant):
    attr, fn = _mutants()[mutant]
    failed = _pins_fail(monkeypatch, attr, fn)
    assert failed, f"mutant {mutant} passed every pin"


def test_wrong_fft_normalisation_is_caught(monkeypatch):
    orig = csa.fft_rg
    monkeypatch.setattr(csa, "fft_rg", lambda A, inverse=False: orig(A, inverse) * (1.0 if inverse else 1.0001))
    with pytest.raises(AssertionError):
        T_op.test_unitarity_full_sampling_AHA_identity()


def test_wrong_doppler_bin_order_is_caught(monkeypatch):
    orig_init = csa.CSAGeometry.__init__

    def init(self, p):
        orig_init(self, p)
        self.f_eta = np.fft.fftshift(self.f_eta)       # natural-order bins applied to FFT-order data
        self.D = np.sqrt(1.0 - (csa.C_LIGHT * self.f_eta / (2.0 * p.Vr * p.fc)) ** 2)
        self.Km = p.Kr / (1.0 - p.Kr * csa.C_LIGHT * p.R_ref * self.f_eta ** 2 / (2.0 * p.Vr ** 2 * p.fc ** 3 * self.D ** 3))
        self.tau_ref = 2.0 * p.R_ref / (csa.C_LIGHT * self.D)

    monkeypatch.setattr(csa.CSAGeometry, "__init__", init)
    with pytest.raises(AssertionError):
        T_ph._focus_check(SarParams(n_az=128, n_rg=128), [(64, 64, 1.0)])

"""Seeded input recipes (inputs/): the separable 1:5 sampling and the 9-target RA
scene used by the NEXT-3 breakdown sweep."""
import numpy as np
import pytest

from inputs import configs, synth


def test_separable_mask_statistics_and_determinism():
    cfg = configs.get("ra", params=configs.SarParams(n_az=4096, n_rg=1024), rate=0.05)
    M = synth.make_mask(cfg)
    rows = M.any(axis=1)
    s_a, s_r = np.sqrt(0.05 / 5), np.sqrt(5 * 0.05)
    assert abs(rows.mean() - s_a) < 4 * np.sqrt(s_a / 4096)
    assert abs(M[rows].mean() - s_r) < 0.02
    assert abs(M.mean() - 0.05) < 0.01
    assert np.array_equal(M, synth.make_mask(cfg))
    with pytest.raises(ValueError):
        synth.make_mask(configs.get("ra", rate=0.3))


def test_grid9_scene():
    sc = synth.make_scene(configs.get("ra"))
    assert len(sc.targets) == 9 and np.allclose(np.abs(sc.val), 1.0)
    ii = sorted({i for i, _, _ in sc.targets})
    jj = sorted({j for _, j, _ in sc.targets})
    assert np.diff(ii).tolist() == [6, 6] and np.diff(jj).tolist() == [6, 6]
    assert ii[1] == 128 and jj[1] == 128

"""Input generator (blade_synth) checks: determinism, band reproducibility, noise statistics,
bank draw rule (BASELINE.json configs[0] + DESIGN.md R10/R11) and the frozen configs."""
from __future__ import annotations

import numpy as np
import pytest

import blade_synth as bs


def test_scene_deterministic_and_band_reproducible():
    a = bs.scene(5, 2, 64, 80, 8, 16, "awgn", 25 / 255)
    b = bs.scene(5, 2, 64, 80, 8, 16, "awgn", 25 / 255)
    assert np.array_equal(a, b)
    band = bs.scene(5, 2, 64, 80, 8, 16, "awgn", 25 / 255, row0=17, rows=21)
    assert np.array_equal(band, a[:, 17:38])
    c = bs.scene(5, 3, 64, 80, 8, 16, "awgn", 25 / 255)
    assert not np.array_equal(a, c)


def test_scene_noise_statistics():
    clean = bs.scene(9, 0, 256, 256, 8, 16, "none").astype(np.float64)
    assert clean.min() >= 0 and clean.max() <= 1
    noisy = bs.scene(9, 0, 256, 256, 8, 16, "awgn", 25 / 255).astype(np.float64)
    r = noisy - clean
    assert abs(r.std() - 25 / 255) < 0.002 and abs(r.mean()) < 0.001
    sig = bs.scene(9, 0, 256, 256, 8, 16, "signal", 0.01, 0.0004).astype(np.float64)
    r = (sig - clean) / np.sqrt(0.01 * clean + 0.0004)
    assert abs(r.std() - 1) < 0.01


def test_bank_normalised_and_conditioned():
    taps, rej = bs.bank(3, 0, 4, 144, 5, 5)
    assert taps.shape == (4, 144, 50)
    s = taps.astype(np.float64).sum(-1)
    assert np.abs(s - 1).max() < 1e-5           # joint sum f + g = 1 (R10), fp32 rounding
    assert 0 < rej < 2 * 576                    # redraw rule R11 rejects ~30-40% of draws
    l1 = np.abs(taps).sum(-1).max()
    assert l1 < 40                              # conditioned bank (SURVEY probe A5)
    again, _ = bs.bank(3, 0, 4, 144, 5, 5)
    assert np.array_equal(taps, again)
    other, _ = bs.bank(3, 1, 4, 144, 5, 5)
    assert not np.array_equal(taps, other)


def test_bank_literal_variant_has_no_redraws():
    taps, rej = bs.bank(0, 0, 1, 144, 7, 0, redraw_below=-np.inf)
    assert rej == 0 and taps.shape == (1, 144, 49)


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_configs_frozen(name):
    cfg = bs.load_config(name)
    ts, tc = cfg.thresholds()
    assert ts.shape == (cfg.n_stages, 2) and tc.shape == (cfg.n_stages, 2)
    for t in (ts, tc):
        assert (np.diff(t, axis=1) > 0).all()
        assert np.array_equal(t.astype(np.float32).astype(np.float64), t)  # fp32-representable
    assert cfg.K == 144

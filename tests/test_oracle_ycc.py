"""Pins of the oracle's per-channel YCbCr path (NEXT row f1; PAPER.md:198-202 footnote 1,
SPEC.md:58-70 colour transforms; R25-R26)."""
from __future__ import annotations

import numpy as np
import pytest
from scipy.ndimage import uniform_filter

import blade_synth as bs
import oracle

O = 128.0 / 255.0


def test_ycc_spec_examples():
    """SPEC.md:63-66 and 72-75 on the [0, 1] scale: white -> (1, o, o), black -> (0, o, o), grey
    g -> (g, o, o); the inverse maps them back."""
    px = np.array([[1.0, 0.0, 0.37], [1.0, 0.0, 0.37], [1.0, 0.0, 0.37]])[:, :, None]  # (3, 3, 1)
    y = oracle.rgb_to_ycc(px)
    np.testing.assert_allclose(y[:, 0, 0], [1.0, O, O], atol=1e-15)
    np.testing.assert_allclose(y[:, 1, 0], [0.0, O, O], atol=1e-15)
    np.testing.assert_allclose(y[:, 2, 0], [0.37, O, O], atol=1e-15)
    np.testing.assert_allclose(oracle.ycc_to_rgb(y), px, atol=1e-15)


def test_ycc_primaries_closed_form():
    """Pure red: Y = .299, Cb = o - .564 * .299, Cr = o + .713 * (1 - .299)."""
    red = np.array([1.0, 0.0, 0.0])[:, None, None]
    y = oracle.rgb_to_ycc(red)[:, 0, 0]
    np.testing.assert_allclose(y, [0.299, O - 0.564 * 0.299, O + 0.713 * 0.701], atol=1e-15)


def test_ycc_round_trip(rng):
    z = rng.uniform(-0.2, 1.2, (3, 17, 23))
    np.testing.assert_allclose(oracle.ycc_to_rgb(oracle.rgb_to_ycc(z)), z, atol=1e-13)


@pytest.mark.parametrize("name", ["c0", "c1", "c2"])
def test_equal_channel_banks_equal_rgb_path(name):
    """With the same bank on Y, Cb and Cr the YCbCr path equals the RGB path: the colour map is
    affine and every stage's filters sum to 1 (R10), so it commutes with the cascade (up to the
    fp32 rounding of the tap sums, ~1e-7 per stage)."""
    cfg = bs.load_config(name)
    cfg.H, cfg.W = 48, 40
    z = cfg.frame(0, H=48, W=40)
    t1 = cfg.taps()
    t3 = np.repeat(t1, 3, axis=1)
    ts, tc = cfg.thresholds()
    rgb = oracle.denoise_config(cfg, z, t1)
    ycc = oracle.denoise_ycc(z, cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.n_phases,
                             cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts, tc, t3)
    np.testing.assert_allclose(ycc, rgb, atol=2e-6)


def test_delta_channel_banks_identity():
    cfg = bs.load_config("c1")
    z = cfg.frame(0, H=33, W=29)
    nf, nc = cfg.fine_size, cfg.coarse_size
    taps = np.zeros((cfg.n_stages, 3, cfg.n_phases, cfg.K, nf * nf + nc * nc))
    taps[..., (nf // 2) * nf + nf // 2] = 1.0
    ts, tc = cfg.thresholds()
    out = oracle.denoise_ycc(z, cfg.levels, nf, nc, cfg.n_phases, cfg.n_orient, cfg.n_strength,
                             cfg.n_coherence, ts, tc, taps)
    np.testing.assert_allclose(out, z, atol=1e-13)


def test_luma_box_chroma_delta_single_level():
    """L = 1, Y filtered by a 7x7 box, Cb and Cr by a delta: equals scipy's uniform filter
    (symmetric padding = mode 'reflect') on the luma plane of the converted image."""
    cfg = bs.load_config("c0")
    z = cfg.frame(0, H=31, W=37)
    nf = cfg.fine_size
    taps = np.zeros((1, 3, 1, cfg.K, nf * nf))
    taps[0, 0] = 1.0 / (nf * nf)
    taps[0, 1:, :, :, (nf // 2) * nf + nf // 2] = 1.0
    ts, tc = cfg.thresholds()
    out = oracle.denoise_ycc(z, 1, nf, 0, 1, cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts,
                             tc, taps)
    y = oracle.rgb_to_ycc(z)
    ref = np.stack([uniform_filter(y[0], size=nf, mode="reflect"), y[1], y[2]])
    np.testing.assert_allclose(out, oracle.ycc_to_rgb(ref), atol=1e-12)


def test_channels_use_distinct_banks():
    cfg = bs.load_config("c1")
    t3 = cfg.taps(channels=3)
    assert t3.shape[1] == 3
    assert np.array_equal(t3[:, 0], cfg.taps()[:, 0])
    assert not np.array_equal(t3[:, 0], t3[:, 1])

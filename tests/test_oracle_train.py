"""Pins of the training oracle (NEXT f4; Eqs. 7-8; oracle/train.py)."""
from __future__ import annotations

import numpy as np
import pytest

import blade_synth as bs
import oracle
from oracle import train as tr


def _level_inputs(name, H, W, seed=0):
    cfg = bs.load_config(name)
    z = cfg.frame(0, H=H, W=W, seed=seed)
    lv = oracle.pyramid(z, cfg.levels)
    ts, tc = cfg.thresholds()
    b = oracle.selector(lv[0], cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts[0], tc[0])
    return cfg, lv, b


def test_one_sample_gram_is_outer_product(rng):
    X = rng.normal(size=(1, 7))
    G, m, c = tr.normal_equations(X, np.array([2.5]), np.array([3]), 5)
    np.testing.assert_array_equal(G[3], np.outer(X[0], X[0]))
    np.testing.assert_array_equal(m[3], 2.5 * X[0])
    assert c.tolist() == [0, 0, 0, 1, 0]


def test_shards_add_up(rng):
    X = rng.normal(size=(400, 6))
    y = rng.normal(size=400)
    seg = rng.integers(0, 4, size=400)
    G, m, c = tr.normal_equations(X, y, seg, 4)
    G1, m1, c1 = tr.normal_equations(X[:150], y[:150], seg[:150], 4)
    G2, m2, c2 = tr.normal_equations(X[150:], y[150:], seg[150:], 4)
    np.testing.assert_allclose(G1 + G2, G, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(m1 + m2, m, rtol=1e-12, atol=1e-12)
    assert np.array_equal(c1 + c2, c)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_targets_from_a_known_bank_are_recovered(name):
    """u := the stage output (Eq. 9, C oracle) of a known bank on the same samples => the
    unregularised solve returns that bank for every well-populated (phase, bucket): pins the sample
    layout (fine/coarse order, folds, floor(i/2), phase) against the independent stage code."""
    cfg = bs.load_config(name)
    rng = np.random.default_rng(7)
    # white-noise input: well-conditioned patch Gram matrices (scene patches are near-collinear)
    size = (96, 80) if name == "c1" else (256, 256)
    lv = oracle.pyramid(rng.uniform(0, 1, (3,) + size), cfg.levels)
    ts, tc = cfg.thresholds()
    b = oracle.selector(lv[0], cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts[0], tc[0])
    nf, nc = cfg.fine_size, cfg.coarse_size
    nt = nf * nf + nc * nc
    bank = rng.normal(size=(cfg.n_phases, cfg.K, nt))
    u_coarse = lv[1]
    u_clean = oracle.stage(lv[0], u_coarse, b, bank, cfg.n_phases, nf, nc)
    X, y, seg = tr.samples(lv[0], u_clean, u_coarse, b, cfg.n_phases, cfg.K, nf, nc)
    np.testing.assert_allclose(np.einsum("ij,ij->i", X, bank.reshape(-1, nt)[seg]), y, atol=1e-12)
    G, m, cnt = tr.normal_equations(X, y, seg, cfg.n_phases * cfg.K)
    H = tr.solve(G, m, cnt, nf, ridge=0.0, min_count=3 * nt)
    ok = cnt >= 3 * nt
    assert ok.sum() >= 5
    # consistent data: the least-squares fit reproduces every target of a solved bucket (this holds
    # however ill-conditioned the patch Gram is); coefficients are recovered where it is not
    sel = ok[seg]
    pred = np.einsum("ij,ij->i", X, H[seg])
    assert np.abs(pred[sel] - y[sel]).max() < 1e-6 * np.abs(y).max()
    if name == "c1":
        np.testing.assert_allclose(H[ok], bank.reshape(-1, nt)[ok], atol=1e-6)


def test_single_level_samples_and_fallback():
    cfg, lv, b = _level_inputs("c0", 128, 120)
    nf = cfg.fine_size
    X, y, seg = tr.samples(lv[0], lv[0], None, b, 1, cfg.K, nf, 0)
    assert X.shape == (3 * 128 * 120, nf * nf)
    # the centre tap of the sample is the pixel itself
    np.testing.assert_array_equal(X[:, (nf // 2) * nf + nf // 2], lv[0].reshape(-1))
    G, m, cnt = tr.normal_equations(X, y, seg, cfg.K)
    H = tr.solve(G, m, cnt, nf, ridge=1e-9)
    empty = cnt < 4 * nf * nf
    assert empty.any()
    assert (H[empty][:, (nf // 2) * nf + nf // 2] == 1.0).all()
    # clean == noisy: the regression reproduces the input (the centred delta is exact)
    full = ~empty
    assert full.sum() >= 5
    pred = np.einsum("ij,ij->i", X, H[seg])
    sel = full[seg]
    assert np.abs(pred[sel] - y[sel]).max() < 1e-4


def test_ridge_shrinks_the_solution(rng):
    X = rng.normal(size=(300, 5))
    y = X @ rng.normal(size=5) + 0.1 * rng.normal(size=300)
    G, m, c = tr.normal_equations(X, y, np.zeros(300, int), 1)
    n1 = np.linalg.norm(tr.solve(G, m, c, 1, ridge=0.01, min_count=1))
    n2 = np.linalg.norm(tr.solve(G, m, c, 1, ridge=1.0, min_count=1))
    assert n2 < n1

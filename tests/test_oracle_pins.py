"""Pins for the fp64 oracle against things other than itself (closed forms, library special
cases, brute force, worked examples in tests/golden/). CPU only.

Each test names the passage of PAPER.md / SPEC.md or the DESIGN.md reading it pins.
"""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest
import scipy.ndimage as ndi
import scipy.signal as sps
import torch

import blade_synth as bs
import oracle

GOLDEN = Path(__file__).parent / "golden"


def _golden(name):
    rows = []
    for line in (GOLDEN / name).read_text().splitlines():
        if not line.strip() or line.startswith("#"):
            continue
        parts = [p.strip() for p in line.split("|")]
        rows.append(([float(v) for v in parts[0].split()], [float(v) for v in parts[1].split()],
                     parts[2]))
    return rows


# --------------------------------------------------------------------------- fold  [R2]

@pytest.mark.parametrize("n", [1, 2, 3, 4, 7])
def test_fold_matches_numpy_symmetric_pad(n):
    """[R2] half-sample symmetric, periodic: equals numpy.pad(mode='symmetric') at any offset."""
    pad = 3 * n + 5
    expect = np.pad(np.arange(n), pad, mode="symmetric")
    got = np.array([oracle.fold(i, n) for i in range(-pad, n + pad)])
    assert (expect == got).all()


# --------------------------------------------------------------------------- O1 decimation

def test_decimate_weights_are_keys_cubic_at_quarter_points():
    """PAPER.md:261 'standard bicubic' -> Keys a=-0.5 at |t|/2, t=+-0.5..3.5:
    textbook values k(0.25)=111/128, k(0.75)=29/128, k(1.25)=-9/128, k(1.75)=-3/128."""
    w = oracle.decimate_weights()
    assert np.array_equal(w * 256, [-3, -9, 29, 111, 111, 29, -9, -3])


@pytest.mark.parametrize("shape", [(3, 40, 56), (3, 33, 47), (2, 5, 5), (1, 1, 1), (3, 2, 3),
                                   (1, 7, 2)])
def test_decimate_equals_torch_antialiased_bicubic(shape, rng):
    """Library special case: the interior of torch's antialiased bicubic x0.5 is the same
    8-tap kernel; symmetric border supplied by numpy.pad, so the WHOLE output is pinned."""
    z = rng.random(shape)
    C, H, W = shape
    P = 16  # even, > kernel half-width, so output y of z is output y+8 of the padded image
    zp = np.pad(z, ((0, 0), (P, P), (P, P)), mode="symmetric")
    ref = torch.nn.functional.interpolate(torch.from_numpy(zp)[None], scale_factor=0.5,
                                          mode="bicubic", antialias=True,
                                          align_corners=False)[0].numpy()
    got = oracle.decimate(z)
    H1, W1 = (H + 1) // 2, (W + 1) // 2
    assert got.shape == (C, H1, W1)
    np.testing.assert_allclose(got, ref[:, P // 2:P // 2 + H1, P // 2:P // 2 + W1], rtol=0,
                               atol=1e-15)


def test_decimate_constant_and_dims():
    """constant preserved (k/256 weights sum to 1 exactly); 5x5 -> 3x3."""
    z = np.full((3, 5, 5), 0.375)
    d = oracle.decimate(z)
    assert d.shape == (3, 3, 3) and (d == 0.375).all()


def test_decimate_noise_std_factor():
    """PAPER.md:261-262 'reduce noise level by half': for this kernel the exact std factor is
    sum_a w_a^2 (separable) = 0.4044 (R15; SPEC.md:410's [9,11] band is wrong)."""
    sigma = 20.0 / 255.0
    n = bs.noise_planes(7, 1, 768, 768, sigma)
    d = oracle.decimate(n)[:, 4:-4, 4:-4]
    factor = d.std() / sigma
    assert abs(factor - 0.4044) < 0.006


def test_pyramid_dims():
    """SPEC.md:418-420 ceil halving: 64 -> 32 -> 16 -> 8; 1000x600 -> ... -> 63x38."""
    lv = oracle.pyramid(np.zeros((3, 600, 1000)), 5)
    assert [l.shape[1:] for l in lv] == [(600, 1000), (300, 500), (150, 250), (75, 125), (38, 63)]


# --------------------------------------------------------------------------- O2 tensor (Eq. 6)

def _scipy_tensor(zpad, P):
    """Eq. 6 with library pieces: numpy.gradient (central differences in the interior),
    scipy gaussian_filter (sigma 1.5, radius 2, normalised) on a symmetric pre-padded image."""
    gx = np.gradient(zpad, axis=2)
    gy = np.gradient(zpad, axis=1)
    kw = dict(sigma=1.5, truncate=2.0 / 1.5, mode="constant")
    a = ndi.gaussian_filter((gx * gx).sum(0), **kw)
    b = ndi.gaussian_filter((gx * gy).sum(0), **kw)
    c = ndi.gaussian_filter((gy * gy).sum(0), **kw)
    sl = (slice(P, -P), slice(P, -P))
    return a[sl], b[sl], c[sl]


@pytest.mark.parametrize("shape", [(3, 24, 31), (3, 6, 5), (1, 9, 12), (3, 2, 2)])
def test_tensor_equals_library_gradient_and_gaussian(shape, rng):
    """Eq. 6 with [R3] central differences, [R4] 5x5 Gaussian sigma 1.5,
    [R2] all fields computed from the folded image (border included via numpy.pad)."""
    z = rng.random(shape)
    P = 12
    zp = np.pad(z, ((0, 0), (P, P), (P, P)), mode="symmetric")
    ra, rb, rc = _scipy_tensor(zp, P)
    a, b, c = oracle.tensor(z)
    for x, y in ((a, ra), (b, rb), (c, rc)):
        np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-14)


def test_tensor_identical_channels_triple():
    """identical channels give exactly 3x the single-channel tensor."""
    z1 = np.random.default_rng(3).random((1, 16, 16))
    a1, b1, c1 = oracle.tensor(z1)
    a3, b3, c3 = oracle.tensor(np.repeat(z1, 3, 0))
    np.testing.assert_allclose(a3, 3 * a1, rtol=1e-14)
    np.testing.assert_allclose(b3, 3 * b1, rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(c3, 3 * c1, rtol=1e-14)


def test_single_channel_ramp_txx_is_one():
    """single-channel ramp v=x gives txx = 1 (normalised weights), txy=tyy=0,
    at pixels >= 3 from the border."""
    H, W = 16, 16
    z = np.tile(np.arange(W, dtype=np.float64), (H, 1))[None]
    a, b, c = oracle.tensor(z)
    s = (slice(3, -3), slice(3, -3))
    np.testing.assert_allclose(a[s], 1.0, rtol=1e-14)
    assert np.abs(b[s]).max() == 0 and np.abs(c[s]).max() == 0


# --------------------------------------------------------------------------- eigen-features

def test_eigen_golden_cases():
    """tests/golden/eigen_cases.txt (SPEC.md:180-182 and closed-form 2x2 cases)."""
    for (a, b, c), (th, S, C), src in _golden("eigen_cases.txt"):
        got = oracle.eigen([a], [b], [c])
        assert got[0][0] == pytest.approx(th, abs=1e-15), src
        assert got[1][0] == pytest.approx(S, abs=1e-15), src
        assert got[2][0] == pytest.approx(C, abs=1e-15), src


def _random_psd(rng, n):
    g = rng.normal(size=(n, 2, 3))
    T = g @ g.transpose(0, 2, 1) * rng.uniform(1e-3, 10, size=(n, 1, 1))
    return T[:, 0, 0], T[:, 0, 1], T[:, 1, 1]


def test_eigen_matches_numpy_eigh(rng):
    """Library special case: eigenvalues and the minor eigenvector equal numpy.linalg.eigh."""
    a, b, c = _random_psd(rng, 1000)
    th, S, C = oracle.eigen(a, b, c)
    T = np.stack([np.stack([a, b], -1), np.stack([b, c], -1)], -2)
    lam, vec = np.linalg.eigh(T)  # ascending
    l2, l1 = np.maximum(lam[:, 0], 0), lam[:, 1]
    np.testing.assert_allclose(S, np.sqrt(l1), rtol=1e-12)
    np.testing.assert_allclose(C, (np.sqrt(l1) - np.sqrt(l2)) / (np.sqrt(l1) + np.sqrt(l2)),
                               rtol=1e-9, atol=1e-12)
    v = vec[:, :, 0]  # minor eigenvector
    ref = np.mod(np.arctan2(v[:, 1], v[:, 0]), np.pi)
    d = np.abs(th - ref)
    d = np.minimum(d, np.pi - d)
    assert d.max() < 1e-9


def test_eigen_bruteforce_angles(rng):
    """direct minimisation of a^T T a over 3600 unit vectors agrees with the
    orientation within 1e-3 rad (coherence > 0.05) and the eigenvalues within 1e-6 relative."""
    a, b, c = _random_psd(rng, 1000)
    th, S, C = oracle.eigen(a, b, c)
    ang = np.arange(3600) * np.pi / 3600
    u = np.stack([np.cos(ang), np.sin(ang)])
    q = a[:, None] * u[0] ** 2 + 2 * b[:, None] * u[0] * u[1] + c[:, None] * u[1] ** 2
    amin = ang[q.argmin(1)]
    l1 = q.max(1)
    m = C > 0.05
    d = np.abs(th - amin)
    d = np.minimum(d, np.pi - d)
    assert d[m].max() < 1e-3
    np.testing.assert_allclose(S ** 2, l1, rtol=1e-6)


def test_eigen_trace_det_identities(rng):
    """l1 + l2 = tr, l1*l2 = det (recovered from S and C)."""
    a, b, c = _random_psd(rng, 500)
    _, S, C = oracle.eigen(a, b, c)
    l1 = S ** 2
    s2 = S * (1 - C) / (1 + C)
    l2 = s2 ** 2
    np.testing.assert_allclose(l1 + l2, a + c, rtol=1e-9)
    det = a * c - b * b
    assert (np.abs(l1 * l2 - det) <= 1e-6 * np.abs(det) + 1e-9 * (a + c) ** 2).all()


def test_eigen_scale_equivariance(rng):
    """scaling pixels by alpha scales T by alpha^2: strength x alpha, orientation
    and coherence unchanged."""
    a, b, c = _random_psd(rng, 200)
    th, S, C = oracle.eigen(a, b, c)
    th2, S2, C2 = oracle.eigen(9 * a, 9 * b, 9 * c)
    np.testing.assert_allclose(S2, 3 * S, rtol=1e-12)
    np.testing.assert_allclose(C2, C, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(th2, th, atol=1e-12)


@pytest.mark.parametrize("alpha,beta", [(1 / 128, 1 / 256), (-1 / 64, 1 / 32), (1 / 16, 0.0),
                                        (0.0, -1 / 8)])
def test_ramp_selector_closed_form(alpha, beta):
    """Dyadic ramp z_c = alpha x + beta y + gamma_c (all channels same slope), pixels >= 3 from
    the border: T = 3 [a^2 ab; ab b^2], S = sqrt(3(a^2+b^2)), C = 1 exactly,
    theta = atan2(alpha, -beta) mod pi (the edge direction, minor eigenvector)."""
    H, W = 20, 20
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    z = np.stack([alpha * x + beta * y + g for g in (0.25, 0.5, 0.75)])
    _, (th, S, C) = oracle.selector(z, 16, 3, 3, [0.1, 0.2], [0.3, 0.6], features=True)
    s = (slice(3, -3), slice(3, -3))
    assert np.allclose(S[s], math.sqrt(3 * (alpha ** 2 + beta ** 2)), rtol=1e-14, atol=0)
    assert (C[s] == 1.0).all()
    ref = math.atan2(alpha, -beta) % math.pi
    assert np.abs(th[s] - ref).max() < 1e-14


def test_ramp_example_bucket():
    """alpha=1/128, beta=1/256: S = sqrt(15)/256, theta = pi - atan(2), o = 10."""
    H, W = 16, 16
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    z = np.stack([x / 128 + y / 256 + g for g in (0.1, 0.2, 0.3)])
    b, (th, S, C) = oracle.selector(z, 16, 3, 3, [0.01, 0.02], [0.3, 0.6], features=True)
    assert S[8, 8] == pytest.approx(math.sqrt(15) / 256, rel=1e-14)
    assert th[8, 8] == pytest.approx(math.pi - math.atan(2), abs=1e-14)
    assert b[8, 8] == (10 * 3 + 1) * 3 + 2


def test_constant_image_selector():
    """constant image -> one bucket, zero features (T = 0 convention)."""
    z = np.full((3, 12, 9), 0.3)
    b, (th, S, C) = oracle.selector(z, 16, 3, 3, [0.1, 0.2], [0.3, 0.6], features=True)
    assert (b == 0).all() and (th == 0).all() and (S == 0).all() and (C == 0).all()


def test_rotation_shifts_orientation_bucket():
    """a 90-degree rotation shifts o by n_o/2 (interior, coherence > 0.1)."""
    cfg = bs.load_config("c0")
    z = cfg.frame(0)
    zr = np.ascontiguousarray(np.rot90(z, 1, axes=(1, 2)))  # counter-clockwise
    _, (th, S, C) = oracle.selector(z, 16, 3, 3, [0.1, 0.2], [0.3, 0.6], features=True)
    _, (thr, Sr, Cr) = oracle.selector(zr, 16, 3, 3, [0.1, 0.2], [0.3, 0.6], features=True)
    thr_back = np.rot90(thr, -1)
    o = np.floor(th * 16 / np.pi).astype(int) % 16
    o_r = np.floor(thr_back * 16 / np.pi).astype(int) % 16
    np.testing.assert_allclose(np.rot90(Sr, -1), S, rtol=1e-12)
    m = np.zeros_like(C, bool)
    m[4:-4, 4:-4] = True
    # exclude orientations within 1e-9 of a bin edge (rounding decides either way)
    edge = np.abs(th * 16 / np.pi - np.round(th * 16 / np.pi)) < 1e-9
    m &= (C > 0.1) & ~edge
    assert m.sum() > 200
    assert ((o_r[m] - o[m]) % 16 == 8).all()


# --------------------------------------------------------------------------- quantiser

def test_quantize_golden_cases():
    """tests/golden/quantize_cases.txt (SPEC.md:189-191 examples + tie rule R7)."""
    for (th, S, C), (bucket,), src in _golden("quantize_cases.txt"):
        got = oracle.quantize([th], [S], [C], 16, 3, 3, [0.1, 0.2], [0.3, 0.6])
        assert got[0] == int(bucket), src


def test_quantize_total(rng):
    """every feature triple maps to exactly one index in [0, K)."""
    th = rng.uniform(0, np.pi, 10000)
    th[:5] = [0, np.pi - 1e-12, np.nextafter(np.pi, 0), 1e-300, np.pi / 2]
    S = rng.exponential(0.2, 10000)
    C = rng.uniform(0, 1, 10000)
    b = oracle.quantize(th, S, C, 16, 3, 3, [0.1, 0.2], [0.3, 0.6])
    assert b.min() >= 0 and b.max() < 144
    o, s, k = b // 9, (b // 3) % 3, b % 3
    assert (o == np.minimum(np.floor(th * 16 / np.pi), 15)).all()
    assert (s == (S >= 0.1).astype(int) + (S >= 0.2)).all()
    assert (k == (C >= 0.3).astype(int) + (C >= 0.6)).all()


# --------------------------------------------------------------------------- O3 stage (Eqs. 1, 9)

def _library_fine_term(z, bucket, taps, n_phases, nf):
    """sum_{(p,k)} [phase==p, s==k] * scipy.signal.correlate2d(pad_symmetric(z), g_{p,k}, 'valid')."""
    C, H, W = z.shape
    r = nf // 2
    zp = np.pad(z, ((0, 0), (r, r), (r, r)), mode="symmetric")
    yy, xx = np.mgrid[0:H, 0:W]
    phase = 2 * (yy % 2) + (xx % 2) if n_phases == 4 else np.zeros((H, W), int)
    out = np.zeros((C, H, W))
    for p in range(n_phases):
        for k in np.unique(bucket):
            m = (phase == p) & (bucket == k)
            if not m.any():
                continue
            g = taps[p, k, :nf * nf].reshape(nf, nf)
            for c in range(C):
                out[c][m] += sps.correlate2d(zp[c], g, mode="valid")[m]
    return out


def _library_coarse_term(u1, H, W, bucket, taps, n_phases, nf, nc):
    """Coarse term of Eq. 9 from library pieces: pad_symmetric(u1, rc), nearest x2 repeat,
    then a 'valid' correlation with the 2-dilated coarse filter (R[y+2rc+2dy] = U[y//2+rc+dy])."""
    C = u1.shape[0]
    rc = nc // 2
    U = np.pad(u1, ((0, 0), (rc, rc), (rc, rc)), mode="symmetric")
    R = np.repeat(np.repeat(U, 2, axis=1), 2, axis=2)
    yy, xx = np.mgrid[0:H, 0:W]
    phase = 2 * (yy % 2) + (xx % 2) if n_phases == 4 else np.zeros((H, W), int)
    out = np.zeros((C, H, W))
    for p in range(n_phases):
        for k in np.unique(bucket):
            m = (phase == p) & (bucket == k)
            if not m.any():
                continue
            f = taps[p, k, nf * nf:].reshape(nc, nc)
            fd = np.zeros((2 * nc - 1, 2 * nc - 1))
            fd[::2, ::2] = f
            for c in range(C):
                out[c][m] += sps.correlate2d(R[c], fd, mode="valid")[:H, :W][m]
    return out


@pytest.mark.parametrize("shape,nf", [((3, 19, 23), 7), ((3, 4, 6), 5), ((3, 2, 3), 9),
                                      ((3, 16, 16), 3)])
def test_stage_single_level_equals_masked_library_correlation(shape, nf, rng):
    """Eq. 1 with a random bank and random bucket map: per-bucket masks of
    scipy correlate2d on the numpy-pad-symmetric image (fold wraps several periods at 2x3)."""
    z = rng.random(shape)
    K = 6
    taps = rng.normal(size=(1, K, nf * nf))
    bucket = rng.integers(0, K, size=shape[1:]).astype(np.int32)
    got = oracle.stage(z, None, bucket, taps, 1, nf, 0)
    ref = _library_fine_term(z, bucket, taps, 1, nf)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("shape,nf,nc", [((3, 21, 26), 5, 5), ((3, 9, 7), 7, 3), ((3, 5, 4), 3, 9),
                                         ((3, 1, 2), 5, 5)])
def test_stage_multiscale_equals_library_terms(shape, nf, nc, rng):
    """Eq. 9 with phase-indexed pairs [R9], odd dims (ceil halving):
    fine term + coarse term, each built from library routines."""
    C, H, W = shape
    z = rng.random(shape)
    u1 = rng.random((C, (H + 1) // 2, (W + 1) // 2))
    K = 5
    taps = rng.normal(size=(4, K, nf * nf + nc * nc))
    bucket = rng.integers(0, K, size=(H, W)).astype(np.int32)
    got = oracle.stage(z, u1, bucket, taps, 4, nf, nc)
    ref = _library_fine_term(z, bucket, taps, 4, nf) + \
        _library_coarse_term(u1, H, W, bucket, taps, 4, nf, nc)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_stage_delta_bank_is_identity_bit_exact(rng):
    """a bank of centred deltas returns the input exactly."""
    z = rng.random((3, 13, 17))
    taps = np.zeros((1, 144, 49))
    taps[:, :, 24] = 1.0
    b = rng.integers(0, 144, size=(13, 17)).astype(np.int32)
    assert np.array_equal(oracle.stage(z, None, b, taps, 1, 7, 0), z)


def test_stage_box_bank_equals_uniform_filter(rng):
    """7x7 box bank (all 1/49) equals scipy uniform_filter with reflect border."""
    z = rng.random((3, 20, 15))
    taps = np.full((1, 144, 49), 1 / 49)
    b = rng.integers(0, 144, size=(20, 15)).astype(np.int32)
    got = oracle.stage(z, None, b, taps, 1, 7, 0)
    ref = np.stack([ndi.uniform_filter(z[c], 7, mode="reflect") for c in range(3)])
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15)


# --------------------------------------------------------------------------- whole cascade

def _cfg(L, nf, nc, H=24, W=20, seed=11):
    return bs.Config(name="t", seed=seed, N=1, H=H, W=W, levels=L, fine_size=nf, coarse_size=nc,
                     n_phases=4 if L > 1 else 1, n_orient=16, n_strength=3, n_coherence=3,
                     window_size=5, window_sigma=1.5, n_grat=4, n_disk=6, noise="awgn",
                     p0=25 / 255, p1=0.0,
                     strength_thresholds=[[0.08, 0.15]] * max(L - 1, 1),
                     coherence_thresholds=[[0.1, 0.3]] * max(L - 1, 1))


def _bilinear_bank(nc, nf, K):
    """Per-phase bilinear x2 weights on the coarse block (even y: 0.75 at floor(y/2), 0.25 at
    floor(y/2)-1; odd y: 0.75 / 0.25 at floor(y/2)+1; separable), zero fine block."""
    rc = nc // 2
    taps = np.zeros((4, K, nf * nf + nc * nc))
    for p in range(4):
        py, px = p // 2, p % 2
        wy = np.zeros(nc)
        wx = np.zeros(nc)
        wy[rc], wy[rc - 1 if py == 0 else rc + 1] = 0.75, 0.25
        wx[rc], wx[rc - 1 if px == 0 else rc + 1] = 0.75, 0.25
        taps[p, :, nf * nf:] = np.outer(wy, wx).ravel()
    return taps


@pytest.mark.parametrize("L", [2, 3, 4])
def test_cascade_bilinear_bank_is_repeated_bilinear_upsampling(L):
    """bilinear-f / zero-g at every level gives (L-1)x bilinear upsampling of
    z^{L-1}; library: torch F.interpolate(scale_factor=2, 'bilinear', align_corners=False)."""
    cfg = _cfg(L, 3, 3, H=32, W=48)
    z = cfg.frame(0)
    taps = np.stack([_bilinear_bank(3, 3, 144)] * (L - 1))
    got = oracle.denoise_config(cfg, z, taps)
    zc = torch.from_numpy(oracle.pyramid(z, L)[-1])[None]
    for _ in range(L - 1):
        zc = torch.nn.functional.interpolate(zc, scale_factor=2, mode="bilinear",
                                             align_corners=False)
    np.testing.assert_allclose(got, zc[0].numpy(), rtol=0, atol=1e-14)


@pytest.mark.parametrize("L,nf,nc", [(1, 7, 0), (2, 5, 5), (3, 5, 5), (4, 7, 3)])
def test_cascade_zero_f_delta_g_identity(L, nf, nc):
    """zero f-blocks and delta g-blocks return the input bit-exactly."""
    cfg = _cfg(L, nf, nc, H=19, W=22)
    z = cfg.frame(0)
    nt = nf * nf + (nc * nc if L > 1 else 0)
    taps = np.zeros((cfg.n_stages, cfg.n_phases, 144, nt))
    taps[..., (nf // 2) * nf + nf // 2] = 1.0
    got = oracle.denoise_config(cfg, z, taps)
    assert np.array_equal(got, z.astype(np.float64))


@pytest.mark.parametrize("L,nf,nc", [(2, 5, 5), (3, 7, 5), (1, 7, 0)])
def test_cascade_constant_image_unchanged_with_sum_one_bank(L, nf, nc, rng):
    """North star: filters summing to 1 leave a constant image unchanged. Dyadic taps with
    joint sum exactly 1 (R10) make this exact in fp64."""
    cfg = _cfg(L, nf, nc)
    z = np.full((3, 24, 20), 0.625, dtype=np.float32)
    nt = nf * nf + (nc * nc if L > 1 else 0)
    taps = rng.integers(-8, 9, size=(cfg.n_stages, cfg.n_phases, 144, nt)).astype(np.float64)
    taps[..., 0] += 64 - taps.sum(-1)
    taps /= 64.0
    assert (taps.sum(-1) == 1).all()
    got = oracle.denoise_config(cfg, z, taps)
    assert (got == 0.625).all()


def test_cascade_shift_equivariance():
    """Shifting the input by 2^(L-1) pixels (both axes) shifts the output, away from the
    border: pins the coarse centre floor(i/2) and the phase index of Eq. 9 / R9."""
    L = 3
    n = 128
    cfg = _cfg(L, 5, 5, H=n, W=n)
    big = cfg.frame(0, H=n + 16, W=n + 16)
    s = 2 ** (L - 1)
    z1 = np.ascontiguousarray(big[:, :n, :n])
    z2 = np.ascontiguousarray(big[:, s:n + s, s:n + s])
    taps = cfg.taps()
    o1 = oracle.denoise_config(cfg, z1, taps)
    o2 = oracle.denoise_config(cfg, z2, taps)
    m = 48  # beyond the cascade's dependency cone of the border (about 40 level-0 pixels)
    np.testing.assert_allclose(o2[:, m:-m, m:-m], o1[:, m + s:n - m + s, m + s:n - m + s],
                               rtol=0, atol=1e-12)


def test_cascade_driver_equals_composed_parts():
    """oracle_denoise (C driver: level order, per-stage thresholds and taps offsets) equals the
    cascade composed step by step from the pinned parts."""
    for name in ("c0",):
        cfg = bs.load_config(name)
        z = cfg.frame(0)
        assert np.array_equal(oracle.denoise_config(cfg, z),
                              oracle.cascade_parts(cfg, z)["outputs"][0])
    cfg = _cfg(4, 5, 3, H=40, W=36)
    cfg.strength_thresholds = [[0.05, 0.1], [0.03, 0.06], [0.01, 0.02]]
    cfg.coherence_thresholds = [[0.1, 0.2], [0.15, 0.3], [0.2, 0.4]]
    z = cfg.frame(0)
    assert np.array_equal(oracle.denoise_config(cfg, z), oracle.cascade_parts(cfg, z)["outputs"][0])


def test_cascade_linear_for_frozen_selector(rng):
    """with the selector frozen, a stage is linear in its image inputs."""
    z1, z2 = rng.random((3, 12, 10)), rng.random((3, 12, 10))
    u1, u2 = rng.random((3, 6, 5)), rng.random((3, 6, 5))
    taps = rng.normal(size=(4, 9, 50))
    b = rng.integers(0, 9, size=(12, 10)).astype(np.int32)
    lhs = oracle.stage(2 * z1 - 3 * z2, 2 * u1 - 3 * u2, b, taps, 4, 5, 5)
    rhs = 2 * oracle.stage(z1, u1, b, taps, 4, 5, 5) - 3 * oracle.stage(z2, u2, b, taps, 4, 5, 5)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)

"""Whole-cascade pin of the oracle on tiny images (SURVEY.md §8(c) "8x8 brute force"): an
independent evaluator written here in plain Python from the paper's definitions, sharing nothing
with oracle/blade_oracle.c:

  * pyramid      z^{l+1}(y,x) = sum_{a,b} w_a w_b Z^l(2y-3+a, 2x-3+b)          PAPER.md:260-263 (§4)
  * selector     tensor by explicit per-pixel sums over the 5x5 window of the folded image's
                 central differences (Eq. 6); the minor eigenvector and the
                 eigenvalues from numpy.linalg.eigh (a library routine, not the oracle's closed
                 form); orientation = its angle mod pi, strength sqrt(l1), coherence
                 (sqrt l1 - sqrt l2)/(sqrt l1 + sqrt l2)
  * stage        memoised recursion u^l(c,y,x) = sum f * U^{l+1}(floor(y/2)+dy, floor(x/2)+dx)
                 + sum g * Z^l(y+dy, x+dx), pair indexed by (phase, bucket)     PAPER.md:269-284 (Eq. 9)

Footprints 3/5/7/9 at 8x8 (and smaller levels, where the fold wraps several periods), L = 1, 2, 3.
Random fp64 inputs keep every feature far from a quantisation boundary (checked), so buckets must
agree exactly and outputs to rounding (1e-12)."""
from __future__ import annotations

import functools
import math

import numpy as np
import pytest

import oracle

W8 = [-3, -9, 29, 111, 111, 29, -9, -3]


def fold(i, n):
    p = 2 * n
    m = i % p
    return m if m < n else p - 1 - m


def decimate_bf(z):
    C, H, W = z.shape
    H1, W1 = (H + 1) // 2, (W + 1) // 2
    out = np.zeros((C, H1, W1))
    for c in range(C):
        for y in range(H1):
            for x in range(W1):
                s = 0.0
                for a in range(8):
                    for b in range(8):
                        s += (W8[a] / 256.0) * (W8[b] / 256.0) * z[c, fold(2 * y - 3 + a, H), fold(2 * x - 3 + b, W)]
                out[c, y, x] = s
    return out


def selector_bf(z, n_o, ts, tc, sigma=1.5, ws=5):
    C, H, W = z.shape
    r = ws // 2
    e = [math.exp(-(d * d) / (2 * sigma * sigma)) for d in range(-r, r + 1)]
    se = sum(e)
    w = [v / se for v in e]
    Z = lambda c, y, x: z[c, fold(y, H), fold(x, W)]
    buckets = np.zeros((H, W), int)
    margin = np.inf
    n_s, n_c = len(ts) + 1, len(tc) + 1
    for y in range(H):
        for x in range(W):
            T = np.zeros((2, 2))
            for dy in range(-r, r + 1):
                for dx in range(-r, r + 1):
                    for c in range(C):
                        yy, xx = y + dy, x + dx
                        gx = (Z(c, yy, xx + 1) - Z(c, yy, xx - 1)) / 2
                        gy = (Z(c, yy + 1, xx) - Z(c, yy - 1, xx)) / 2
                        g = np.array([gx, gy])
                        T += w[dy + r] * w[dx + r] * np.outer(g, g)
            lam, vec = np.linalg.eigh(T)  # ascending
            l2, l1 = max(lam[0], 0.0), lam[1]
            v = vec[:, 0]  # minor eigenvector (x, y)
            theta = math.atan2(v[1], v[0]) % math.pi
            S = math.sqrt(l1)
            Co = (math.sqrt(l1) - math.sqrt(l2)) / (math.sqrt(l1) + math.sqrt(l2))
            o = int(math.floor(theta * n_o / math.pi)) % n_o
            s = sum(t <= S for t in ts)
            k = sum(t <= Co for t in tc)
            buckets[y, x] = (o * n_s + s) * n_c + k
            width = math.pi / n_o
            rem = theta % width
            margin = min(margin, rem, width - rem, *(abs(S - t) for t in ts),
                         *(abs(Co - t) for t in tc))
    return buckets, margin


def cascade_bf(z, L, nf, nc, n_o, ts, tc, taps):
    """taps: [n_stages, n_phases, K, nf^2 + nc^2]; returns (u^0, buckets per level, margin)."""
    lv = [z]
    for _ in range(L - 1):
        lv.append(decimate_bf(lv[-1]))
    nsel = 1 if L == 1 else L - 1
    sel = [selector_bf(lv[l], n_o, ts[l], tc[l]) for l in range(nsel)]
    rf, rc = nf // 2, nc // 2

    @functools.lru_cache(maxsize=None)
    def u(l, c, y, x):
        H, W = lv[l].shape[1:]
        y, x = fold(y, H), fold(x, W)
        if L > 1 and l == L - 1:
            return lv[l][c, y, x]
        p = 2 * (y % 2) + (x % 2) if L > 1 else 0
        k = sel[l][0][y, x]
        h = taps[l, p, k]
        s = 0.0
        for dy in range(-rf, rf + 1):
            for dx in range(-rf, rf + 1):
                s += h[(dy + rf) * nf + dx + rf] * lv[l][c, fold(y + dy, H), fold(x + dx, W)]
        if L > 1:
            for dy in range(-rc, rc + 1):
                for dx in range(-rc, rc + 1):
                    s += h[nf * nf + (dy + rc) * nc + dx + rc] * u(l + 1, c, y // 2 + dy, x // 2 + dx)
        return s

    H, W = z.shape[1:]
    out = np.array([[[u(0, c, y, x) for x in range(W)] for y in range(H)] for c in range(3)])
    return out, [b for b, _ in sel], min(m for _, m in sel)


@pytest.mark.parametrize("L,nf,nc,H,W", [(1, 3, 0, 8, 8), (1, 7, 0, 8, 8), (1, 9, 0, 5, 7),
                                         (2, 5, 5, 8, 8), (2, 9, 3, 8, 8), (2, 7, 9, 7, 8),
                                         (3, 5, 5, 8, 8), (3, 3, 7, 8, 6), (3, 9, 9, 8, 8)])
def test_oracle_cascade_equals_bruteforce(L, nf, nc, H, W):
    rng = np.random.default_rng(1000 * L + 10 * nf + nc)
    z = rng.uniform(0.0, 1.0, (3, H, W))
    n_o, n_s, n_c = 8, 3, 2
    K = n_o * n_s * n_c
    n_ph = 4 if L > 1 else 1
    nst = max(L - 1, 1)
    nt = nf * nf + (nc * nc if L > 1 else 0)
    taps = rng.normal(size=(nst, n_ph, K, nt))
    # thresholds between observed feature values of the oracle's own levels would couple the two;
    # take fixed ones inside the ranges uniform [0,1] inputs produce
    ts = np.tile([0.08, 0.16], (nst, 1))
    tc = np.tile([0.35], (nst, 1))
    ref, buckets_bf, margin = cascade_bf(z, L, nf, nc if L > 1 else 0, n_o, ts, tc, taps)
    assert margin > 1e-9, "a feature sits on a quantisation boundary; change the seed"
    parts_buckets = []
    lv = oracle.pyramid(z, L)
    for l in range(1, L):
        np.testing.assert_allclose(lv[l], decimate_bf(lv[l - 1]), rtol=0, atol=1e-13)
    for l in range(1 if L == 1 else L - 1):
        parts_buckets.append(oracle.selector(lv[l], n_o, n_s, n_c, ts[l], tc[l]))
        np.testing.assert_array_equal(parts_buckets[l], buckets_bf[l])
    out = oracle.denoise(z, L, nf, nc if L > 1 else 0, n_ph, n_o, n_s, n_c, ts, tc, taps)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-11)

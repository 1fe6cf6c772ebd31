"""Parity helpers shared by the GPU tests: the north-star comparison rule, made operational
(SURVEY.md §8(c) "Parity rule"):

  buckets : bit-exact except pixels whose ORACLE fp64 features lie within 1e-5 of a
            quantisation boundary (orientation bin edge k*pi/n_o, a strength threshold, a
            coherence threshold); such mismatches are counted and must be <= 1e-4 of the
            level's pixels.
  outputs : within 1e-4 absolute (on the [0,1] scale) at every pixel outside the dependency
            cone of a bucket mismatch (free mode; the oracle never consumes GPU values).
"""
from __future__ import annotations

import numpy as np

BOUNDARY_EPS = 1e-5
MISMATCH_FRAC = 1e-4
OUT_ATOL = 1e-4


def near_boundary(theta, S, C, n_o, ts, tc, eps=BOUNDARY_EPS):
    """Pixels whose fp64 features are within eps of a quantisation boundary."""
    w = np.pi / n_o
    r = np.mod(theta, w)
    near = np.minimum(r, w - r) < eps
    for t in np.ravel(ts):
        near |= np.abs(S - t) < eps
    for t in np.ravel(tc):
        near |= np.abs(C - t) < eps
    return near


def check_buckets(gpu_map, oracle_map, feats, n_o, ts, tc, label=""):
    """Returns (mismatch mask, stats dict); asserts the rule."""
    gpu_map = np.asarray(gpu_map).astype(np.int32)
    mism = gpu_map != oracle_map
    near = near_boundary(*feats, n_o, ts, tc)
    bad = mism & ~near
    n = mism.size
    stats = dict(pixels=n, mismatches=int(mism.sum()), near_boundary=int(near.sum()),
                 outside_window=int(bad.sum()))
    assert bad.sum() == 0, f"{label}: {bad.sum()} bucket mismatches away from a boundary {stats}"
    assert mism.sum() <= MISMATCH_FRAC * n, f"{label}: too many mismatches {stats}"
    return mism, stats


def taint_cone(mismatch_per_level, dims, rc):
    """Tainted^l = M^l  U  {(y,x): some coarse tap (floor(y/2)+dy, floor(x/2)+dx), |d|<=rc, folded,
    is tainted at l+1}. Returns the level-0 mask."""
    L = len(dims)
    tainted = None
    for l in range(len(mismatch_per_level) - 1, -1, -1):
        H, W = dims[l]
        m = mismatch_per_level[l].copy()
        if tainted is not None and tainted.any():
            H1, W1 = dims[l + 1]
            tp = np.pad(tainted, rc, mode="symmetric")  # fold at the coarse level's border
            dil = np.zeros((H1, W1), bool)
            for dy in range(2 * rc + 1):
                for dx in range(2 * rc + 1):
                    dil |= tp[dy:dy + H1, dx:dx + W1]
            up = np.repeat(np.repeat(dil, 2, 0), 2, 1)[:H, :W]
            m |= up
        tainted = m
    assert L >= 1
    return tainted


def max_err_outside(gpu_out, oracle_out, tainted):
    d = np.abs(np.asarray(gpu_out, np.float64) - oracle_out)
    if tainted is not None:
        d = d[:, ~tainted]
    return float(d.max()) if d.size else 0.0

"""ORACLE — TEST INFRASTRUCTURE ONLY. Filter learning of PAPER.md:186-198 (§3, Eqs. 7-8) per
(phase, bucket) for the stacked multiscale sample of §4 Eq. 10, in plain numpy fp64 (NEXT f4).

Readings (R27-R30): the sample of pixel i and channel c is
    x = [ R_i z^l  (n_f x n_f patch, row-major, folded) ; R_{floor(i/2)} u_hat^{l+1} (n_c x n_c) ]
in the ABI's fine-then-coarse tap order, so that h . x is the stage output of Eq. 9; the target is
the clean level u^l_c(i); R, G and B are three samples of the same (phase, bucket) regression
(one filter shared by the channels, R13). Normal equations G = sum x x^T, m = sum x u, and the
solve h = (G + ridge tr(G)/nt I)^-1 m, fallback = centred fine delta when a
bucket has fewer than min_count samples. Only numpy; shares nothing with the CUDA path.
"""
from __future__ import annotations

import numpy as np


def _fold_pad(img: np.ndarray, r: int) -> np.ndarray:
    """(C, H, W) -> (C, H + 2r, W + 2r) with the half-sample symmetric fold (R2; numpy 'symmetric'
    reflects repeatedly for pads wider than the image)."""
    return np.pad(img, ((0, 0), (r, r), (r, r)), mode="symmetric")


def samples(z, u_clean, u_coarse, buckets, n_phases: int, K: int, nf: int, nc: int):
    """All samples of one frame: X [3 H W, nt], y [3 H W], seg [3 H W] (= phase * K + bucket);
    rows ordered (channel, y, x)."""
    z = np.asarray(z, np.float64)
    u_clean = np.asarray(u_clean, np.float64)
    C, H, W = z.shape
    rf = nf // 2
    zp = _fold_pad(z, rf)
    cols = [zp[:, dy:dy + H, dx:dx + W] for dy in range(nf) for dx in range(nf)]  # tap (dy, dx)
    if u_coarse is not None and nc > 0:
        uc = np.asarray(u_coarse, np.float64)
        rc = nc // 2
        up = _fold_pad(uc, rc)
        yy = np.arange(H)[:, None] // 2
        xx = np.arange(W)[None, :] // 2
        for dy in range(nc):
            for dx in range(nc):
                cols.append(up[:, yy + dy, xx + dx])
    X = np.stack([c.reshape(C, -1) for c in cols], axis=-1).reshape(C * H * W, -1)
    y = u_clean.reshape(-1)
    ph = 2 * (np.arange(H)[:, None] % 2) + (np.arange(W)[None, :] % 2) if n_phases == 4 \
        else np.zeros((H, W), int)
    seg = (ph * K + np.asarray(buckets)).reshape(-1)
    return X, y, np.tile(seg, C)


def normal_equations(X, y, seg, n_seg: int):
    """G [n_seg, nt, nt], m [n_seg, nt], count [n_seg] (Eq. 8's sufficient statistics)."""
    nt = X.shape[1]
    G = np.zeros((n_seg, nt, nt))
    m = np.zeros((n_seg, nt))
    cnt = np.bincount(seg, minlength=n_seg).astype(np.int64)
    order = np.argsort(seg, kind="stable")
    bounds = np.concatenate([[0], np.cumsum(cnt)])
    for k in np.nonzero(cnt)[0]:
        idx = order[bounds[k]:bounds[k + 1]]
        Xk = X[idx]
        G[k] = Xk.T @ Xk
        m[k] = Xk.T @ y[idx]
    return G, m, cnt


def solve(G, m, cnt, nf: int, ridge: float = 1e-3, min_count: int | None = None):
    """Per-segment h = (G + ridge tr(G)/nt I)^-1 m; fallback = centred fine delta (zero coarse)."""
    n_seg, nt, _ = G.shape
    min_count = 4 * nt if min_count is None else min_count
    H = np.zeros((n_seg, nt))
    for k in range(n_seg):
        if cnt[k] < min_count:
            H[k, (nf // 2) * nf + nf // 2] = 1.0
            continue
        A = G[k] + ridge * np.trace(G[k]) / nt * np.eye(nt)
        H[k] = np.linalg.solve(A, m[k])
    return H

"""Random parity cases for the GPU suite and scripts/fuzz_parity.py: random shapes, pyramid depths,
footprint pairs, bucket layouts, windows and batch sizes, each checked with the GPU suite's rule
(tests/test_gpu_parity._full_parity: the CUDA path through the C ABI against the fp64 oracle)."""
from __future__ import annotations

import numpy as np


def draw(rng):
    levels = int(rng.choice([1, 2, 2, 3, 3, 4, 5]))
    nf = int(rng.choice([3, 5, 5, 7, 9]))
    nc = int(rng.choice([3, 5, 5, 7, 9])) if levels > 1 else 0
    if rng.random() < 0.5:  # shapes around tile and vector-width boundaries
        H = int(rng.choice([15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 257]))
        W = int(rng.choice([124, 127, 128, 129, 132, 255, 256, 257, 260, 383, 384, 388]))
    else:
        H, W = int(rng.integers(1, 300)), int(rng.integers(1, 420))
    N = int(rng.choice([1, 1, 2, 3]))
    n_o = int(rng.choice([1, 4, 6, 8, 12, 16, 16, 16, 20]))
    n_s = int(rng.choice([1, 2, 3, 3, 4]))
    n_c = int(rng.choice([1, 2, 3, 3, 4]))
    win = int(rng.choice([1, 3, 5, 5, 5]))
    n_ph = 4 if (levels > 1 and rng.random() < 0.8) else 1
    # noise-free scenes are left out: half their pixels have an exactly zero structure tensor (every
    # feature on a quantisation boundary), so the near-boundary allowance of the rule decides them
    noise = str(rng.choice(["awgn", "signal"]))
    return dict(levels=levels, nf=nf, nc=nc, H=H, W=W, N=N, n_o=n_o, n_s=n_s, n_c=n_c, win=win,
                n_ph=n_ph, noise=noise)


def _T():
    from tests import test_gpu_parity as T
    return T


def run_case(p, seed):
    rng = np.random.default_rng(seed)
    cfg = _T()._cfg_like("c1", p["H"], p["W"], p["N"], levels=p["levels"], fine_size=p["nf"],
                      coarse_size=p["nc"] if p["levels"] > 1 else 5, n_phases=p["n_ph"],
                      n_orient=p["n_o"], n_strength=p["n_s"], n_coherence=p["n_c"],
                      window_size=p["win"], window_sigma=float(rng.uniform(0.6, 2.0)), noise=p["noise"],
                      seed=int(seed))
    if p["noise"] == "signal":
        cfg.p0, cfg.p1 = 0.01, 0.0004
    nst = max(p["levels"] - 1, 1)
    cfg.strength_thresholds = [sorted(rng.uniform(0.02, 0.25, p["n_s"] - 1).tolist()) for _ in range(nst)]
    cfg.coherence_thresholds = [sorted(rng.uniform(0.02, 0.3, p["n_c"] - 1).tolist()) for _ in range(nst)]
    _, _, worst = _T()._full_parity(cfg, cfg.batch(), label=str(p))
    return worst



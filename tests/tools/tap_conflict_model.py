"""Shared-memory conflict model of the stage's per-pixel tap loads (profiles/r02_tap_layout.txt).

Builds the oracle's level-0 bucket map of a band of c3 frame 0 and counts, for the lane -> pixel
mapping of k_stage_tma (32 thread columns of a tile row, 4 px apart, one (phase, bucket) filter
per lane), the shared-memory wavefronts of one tap load under the two service models:
LDS.128 per quarter warp (8 bank groups of 16 B), LDS.32 per warp (32 banks). Host only; it lives under
tests/ because it uses the oracle for the bucket map (test infrastructure, never a product path).

    python tests/tools/tap_conflict_model.py [rows]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import blade_synth  # noqa: E402
import oracle  # noqa: E402


def wf128(addr, lanes=8):
    """addr: 32 float offsets (16-B aligned). Sum over lane groups of the largest pile of distinct
    16-B addresses in one bank group (lanes = 8: quarter-warp service; 32: whole warp)."""
    t = 0
    for q in range(0, 32, lanes):
        a = np.unique(addr[q:q + lanes] // 4)
        t += np.bincount(a % 8, minlength=8).max()
    return t


def wf32(addr):
    a = np.unique(addr)
    return np.bincount(a % 32, minlength=32).max()


def main(rows=400):
    cfg = blade_synth.load_config("c3")
    z = blade_synth.scene(cfg.seed, 0, cfg.H, cfg.W, cfg.n_grat, cfg.n_disk, cfg.noise, cfg.p0, cfg.p1,
                          row0=300, rows=rows)
    ts, tc = cfg.thresholds()
    b = oracle.selector(z, cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts[0], tc[0])
    H, W = b.shape
    K = cfg.n_orient * cfg.n_strength * cfg.n_coherence
    S = 52  # single-record stride of the 5x5 + 5x5 pair (13 chunks)
    rng = np.random.default_rng(0)
    acc = {"LDS.128 quarter-warp": 0.0, "LDS.128 whole-warp": 0.0, "LDS.32 record stride 52": 0.0,
           "LDS.32 record stride 11": 0.0}
    n = 0
    for T in range(W // 128):
        for y0 in range(0, H - 3, 4):
            if rng.random() > 0.15:
                continue
            for i in range(4):
                for j in range(4):
                    x = 128 * T + 4 * np.arange(32) + j
                    k = b[y0 + i, x]
                    ph = 2 * (i & 1) + (j & 1)
                    base = ph * K * S + k * S
                    acc["LDS.128 quarter-warp"] += wf128(base)
                    acc["LDS.128 whole-warp"] += wf128(base, 32)
                    acc["LDS.32 record stride 52"] += wf32(base + 40)
                    acc["LDS.32 record stride 11"] += wf32((ph * K + k) * 11)
                    n += 1
    for name, v in acc.items():
        print(f"{name:28s} {v / n:6.2f} wavefronts per load ({n} warp loads)")
    # lanes closer together: 2 px apart, and quarter warps as 4 x 2 pixel blocks
    for name, stride in (("lanes 4 px apart", 4), ("lanes 2 px apart", 2)):
        tot = 0
        for _ in range(20000):
            y = rng.integers(0, H)
            x = rng.integers(0, W - 32 * stride) + stride * np.arange(32)
            tot += wf128((2 * (y & 1) + (x & 1)) * K * S + b[y, x] * S)
        print(f"{name:28s} {tot / 20000:6.2f}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 400)

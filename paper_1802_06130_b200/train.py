"""Multiscale filter learning on the GPU (NEXT row f4): the coarse-to-fine schedule of
PAPER.md:285-289 (§4) over the per-stage least-squares of PAPER.md:186-198 (Eqs. 7-8).

    "We train filters by using input patches from the current level l and corresponding patches
     from the filtered output at the next coarser level l+1. Once level l is trained, filtered
     images u^l are computed and then consumed for training h^{l-1} at the next finer level."

Every step runs in libblade_ms.so: the pyramids (blade_ms_pyramid), the selector, the normal
equations (blade_ms_train_accumulate) and the coarse outputs (blade_ms_denoise of the
sub-cascade); the solve is the library's host fp64 Cholesky (blade_ms_train_solve). This module
only sequences the calls.
"""
from __future__ import annotations

import copy

import numpy as np
import torch

from .blade_ms import BladeMS


def _sub_config(cfg, first_level: int):
    """The cascade of levels first_level .. L-1 as its own config (stages first_level .. L-2)."""
    sub = copy.deepcopy(cfg)
    sub.levels = cfg.levels - first_level
    ts, tc = cfg.thresholds()
    nst = max(sub.levels - 1, 1)
    sub.strength_thresholds = ts[first_level:first_level + nst].tolist()
    sub.coherence_thresholds = tc[first_level:first_level + nst].tolist()
    if sub.levels == 1:
        sub.coarse_size = 0
        sub.n_phases = 1
    return sub


def fallback_bank(cfg) -> np.ndarray:
    """Pass-through bank: centred fine delta, zero coarse block, every (stage, phase, bucket)."""
    nf = cfg.fine_size
    nt = nf * nf + (cfg.coarse_size ** 2 if cfg.levels > 1 else 0)
    taps = np.zeros((cfg.n_stages, 1, cfg.n_phases, cfg.K, nt), np.float32)
    taps[..., (nf // 2) * nf + nf // 2] = 1.0
    return taps


def train_multiscale(cfg, noisy: torch.Tensor, clean: torch.Tensor, ridge: float = 1e-3,
                     min_count: int | None = None, device: int = 0):
    """Learn the bank of `cfg` (blade_synth.Config-like) from noisy / clean frames [N,3,H,W]
    (CUDA fp32). Returns (taps [n_stages, 1, n_phases, K, nt] float32, counts per stage)."""
    L = cfg.levels
    taps = fallback_bank(cfg)
    h0 = BladeMS.from_config(cfg, taps=taps, device=device)
    z = [noisy] + (h0.pyramid(noisy) if L > 1 else [])
    u = [clean] + (h0.pyramid(clean) if L > 1 else [])
    counts = [None] * cfg.n_stages
    stages = [0] if L == 1 else list(range(L - 2, -1, -1))
    for l in stages:
        if L == 1:
            coarse = None
        elif l == L - 2:
            coarse = z[L - 1]  # base case u^{L-1} = z^{L-1}
        else:  # the trained sub-cascade l+1 .. L-1 applied to z^{l+1}
            sub = _sub_config(cfg, l + 1)
            hs = BladeMS.from_config(sub, taps=taps[l + 1:l + 1 + sub.n_stages], device=device)
            coarse = hs.denoise(z[l + 1].contiguous())
        h = BladeMS.from_config(cfg, taps=taps, device=device)
        E, cnt = h.train_accumulators()
        h.train_accumulate(l, z[l].contiguous(), u[l].contiguous(), coarse, E, cnt)
        taps[l, 0] = h.train_solve(E, cnt, ridge=ridge, min_count=min_count)
        counts[l] = cnt.cpu().numpy()
    return taps, counts

#!/usr/bin/env python
"""Freeze per-level strength/coherence thresholds into configs/cN.json (reading R8).

For each config: draw a CALIBRATION frame (same scene recipe, seed + 1000), build the
oracle's fp64 pyramid, and at every selector level take the empirical tertiles (n_s = n_c = 3)
of the oracle's fp64 strength and coherence (SPEC.md:201-209 fit_thresholds rule: quantiles
at k/n). Each threshold is rounded to the nearest fp32 value so that both the fp64 oracle and
the fp32 kernels compare against the very same number.

Calls only `oracle/` and `blade_synth/` (no CUDA path), as the parity rules require.
Usage: python scripts/fit_thresholds.py [c0 c1 ...]
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import blade_synth as bs  # noqa: E402
import oracle  # noqa: E402


def fit(name: str) -> dict:
    cfg = bs.load_config(name)
    z = cfg.frame(0, seed=cfg.seed + 1000)
    lv = oracle.pyramid(z, cfg.levels)
    ts_all, tc_all = [], []
    dummy_s = np.zeros(cfg.n_strength - 1)
    dummy_c = np.zeros(cfg.n_coherence - 1)
    for l in range(cfg.n_stages):
        _, (th, S, Co) = oracle.selector(lv[l], cfg.n_orient, cfg.n_strength, cfg.n_coherence,
                                         dummy_s, dummy_c, cfg.window_size, cfg.window_sigma,
                                         features=True)
        qs = np.quantile(S.ravel(), [k / cfg.n_strength for k in range(1, cfg.n_strength)])
        qc = np.quantile(Co.ravel(), [k / cfg.n_coherence for k in range(1, cfg.n_coherence)])
        ts = [float(np.float32(v)) for v in qs]
        tc = [float(np.float32(v)) for v in qc]
        assert all(a < b for a, b in zip(ts, ts[1:])) and all(a < b for a, b in zip(tc, tc[1:]))
        ts_all.append(ts)
        tc_all.append(tc)
        print(f"{name} level {l}: {lv[l].shape[1]}x{lv[l].shape[2]} S thresholds {ts} "
              f"C thresholds {tc}", flush=True)
    p = bs.CONFIG_DIR / f"{name}.json"
    d = json.loads(p.read_text())
    d["strength_thresholds"] = ts_all
    d["coherence_thresholds"] = tc_all
    d["thresholds_recipe"] = (f"per-level {cfg.n_strength}- / {cfg.n_coherence}-quantiles of the fp64 oracle's strength/coherence on a "
                              "calibration frame (seed+1000), rounded to fp32; "
                              "scripts/fit_thresholds.py")
    p.write_text(json.dumps(d, indent=1) + "\n")
    return d


if __name__ == "__main__":
    names = sys.argv[1:] or bs.config_names()
    for n in names:
        fit(n)

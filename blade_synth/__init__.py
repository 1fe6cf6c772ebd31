"""Seeded synthetic inputs (scenes, noise, filterbanks) and config loading.

This package is the ONLY code shared by the oracle side (tests, cpu baseline)
and the CUDA side (tests, bench). It holds none of the method's arithmetic:
it draws images and filter taps and reads `configs/*.json`. See
`synth.c` for the generator and DESIGN.md §"Inputs" for the recipe.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "synth.c"
_LIB_PATH = _HERE / "libblade_synth.so"
REPO_ROOT = _HERE.parent
CONFIG_DIR = REPO_ROOT / "configs"

_lib = None


def build(force: bool = False) -> Path:
    """Compile synth.c into libblade_synth.so (gcc, OpenMP)."""
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB_PATH.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        i64, u64, dbl, ptr = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        lib.synth_scene.argtypes = [u64, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, dbl, dbl, ptr]
        lib.synth_scene.restype = ctypes.c_int
        lib.synth_noise.argtypes = [u64, i64, i64, i64, i64, dbl, ptr]
        lib.synth_noise.restype = ctypes.c_int
        lib.synth_bank.argtypes = [u64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, dbl, ptr, ctypes.POINTER(ctypes.c_int64)]
        lib.synth_bank.restype = ctypes.c_int
        _lib = lib
    return _lib


NOISE_KINDS = {"none": 0, "awgn": 1, "signal": 2}


def scene(seed: int, frame: int, H: int, W: int, n_grat: int, n_disk: int,
          noise: str = "awgn", p0: float = 25.0 / 255.0, p1: float = 0.0,
          row0: int = 0, rows: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """One RGB frame (3, rows, W) float32 on a [0,1] scale, rows [row0, row0+rows)."""
    lib = _load()
    rows = H - row0 if rows is None else rows
    if out is None:
        out = np.empty((3, rows, W), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape == (3, rows, W)
    rc = lib.synth_scene(seed, frame, H, W, row0, rows, n_grat, n_disk, NOISE_KINDS[noise],
                         p0, p1, out.ctypes.data)
    if rc:
        raise ValueError(f"synth_scene failed ({rc})")
    return out


def noise_planes(seed: int, C: int, H: int, W: int, std: float, frame: int = 0) -> np.ndarray:
    lib = _load()
    out = np.empty((C, H, W), dtype=np.float32)
    if lib.synth_noise(seed, frame, C, H, W, std, out.ctypes.data):
        raise ValueError("synth_noise failed")
    return out


def bank(seed: int, stage: int, n_phases: int, K: int, nf: int, nc: int,
         redraw_below: float = 4.0) -> tuple[np.ndarray, int]:
    """Taps for one stage, float32 [n_phases, K, nf*nf + nc*nc]; returns (taps, redraws).

    redraw_below=-inf gives the literal (unconditioned) draw of BASELINE.json configs[0].
    """
    lib = _load()
    nt = nf * nf + nc * nc
    out = np.empty((n_phases, K, nt), dtype=np.float32)
    rej = ctypes.c_int64(0)
    if lib.synth_bank(seed, stage, n_phases, K, nf, nc, redraw_below, out.ctypes.data,
                      ctypes.byref(rej)):
        raise ValueError("synth_bank failed")
    return out, int(rej.value)


# ----------------------------------------------------------------------------- configs

@dataclass
class Config:
    """One BASELINE.json config as concrete parameters (configs/cN.json)."""
    name: str
    seed: int
    N: int
    H: int
    W: int
    levels: int
    fine_size: int
    coarse_size: int
    n_phases: int
    n_orient: int
    n_strength: int
    n_coherence: int
    window_size: int
    window_sigma: float
    n_grat: int
    n_disk: int
    noise: str
    p0: float
    p1: float
    strength_thresholds: list = field(default_factory=list)   # [n_stages][n_strength-1]
    coherence_thresholds: list = field(default_factory=list)  # [n_stages][n_coherence-1]
    description: str = ""
    thresholds_recipe: str = ""

    @property
    def n_stages(self) -> int:
        return max(self.levels - 1, 1)

    @property
    def K(self) -> int:
        return self.n_orient * self.n_strength * self.n_coherence

    def frame(self, n: int, row0: int = 0, rows: int | None = None, H: int | None = None,
              W: int | None = None, seed: int | None = None) -> np.ndarray:
        return scene(self.seed if seed is None else seed, n, H or self.H, W or self.W,
                     self.n_grat, self.n_disk, self.noise, self.p0, self.p1, row0, rows)

    def batch(self, N: int | None = None, H: int | None = None, W: int | None = None,
              frame0: int = 0, seed: int | None = None) -> np.ndarray:
        N = self.N if N is None else N
        H = H or self.H
        W = W or self.W
        out = np.empty((N, 3, H, W), dtype=np.float32)
        for i in range(N):
            scene(self.seed if seed is None else seed, frame0 + i, H, W, self.n_grat,
                  self.n_disk, self.noise, self.p0, self.p1, out=out[i])
        return out

    def taps(self, redraw_below: float = 4.0, channels: int = 1) -> np.ndarray:
        """All stages: float32 [n_stages, channels, n_phases, K, nf^2 + nc^2]. channels = 3 draws
        independent per-channel (Y, Cb, Cr) banks (NEXT f1): channel c of stage s uses the bank
        stream of stage index s + 1000 c; channel 0 equals the single-channel bank."""
        nc = self.coarse_size if self.levels > 1 else 0
        st = [[bank(self.seed, s + 1000 * c, self.n_phases, self.K, self.fine_size, nc,
                    redraw_below)[0] for c in range(channels)] for s in range(self.n_stages)]
        return np.stack([np.stack(ch) for ch in st])

    def thresholds(self) -> tuple[np.ndarray, np.ndarray]:
        ts = np.asarray(self.strength_thresholds, dtype=np.float64).reshape(self.n_stages,
                                                                            self.n_strength - 1)
        tc = np.asarray(self.coherence_thresholds, dtype=np.float64).reshape(self.n_stages,
                                                                             self.n_coherence - 1)
        return ts, tc


def load_config(name: str) -> Config:
    p = CONFIG_DIR / f"{name}.json"
    d = json.loads(p.read_text())
    return Config(**d)


def config_names() -> list[str]:
    return sorted(p.stem for p in CONFIG_DIR.glob("c*.json"))

"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain fp64 CPU implementation of the multiscale BLADE inference path
(arxiv 1802.06130, §3 Eqs. 1, 6 and §4 Eq. 9), in `blade_oracle.c`,
wrapped with ctypes. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu_baseline / `--impl reference` legs may import this package. It shares no
code with the CUDA path (`paper_1802_06130_b200/`), and the CUDA path never
imports it.

Parity status per function (pins in tests/test_oracle_*.py):
  fold, decimate, tensor, eigen, quantize, selector, stage, denoise: pinned.
  rgb_to_ycc, ycc_to_rgb, denoise_ycc (per-channel YCbCr banks, NEXT f1): pinned
  (tests/test_oracle_ycc.py).
  Thresholds and scene generator are inputs, not results (parity unpinned by
  nature; they are produced by blade_synth and scripts/fit_thresholds.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "blade_oracle.c"
_LIB_PATH = _HERE / "libblade_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle: gcc -O2, OpenMP, no fast-math (fp64 IEEE)."""
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB_PATH.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", "-o", str(tmp), str(_SRC),
                               "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        i64, dbl, ptr, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
        lib.oracle_fold.argtypes = [i64, i64]
        lib.oracle_fold.restype = i64
        lib.oracle_decimate_weights.argtypes = [ptr]
        lib.oracle_decimate.argtypes = [ptr, i64, i64, i64, ptr]
        lib.oracle_tensor.argtypes = [ptr, i64, i64, i64, i32, dbl, ptr, ptr, ptr]
        lib.oracle_eigen.argtypes = [ptr, ptr, ptr, i64, ptr, ptr, ptr]
        lib.oracle_quantize.argtypes = [ptr, ptr, ptr, i64, i32, i32, i32, ptr, ptr, ptr]
        lib.oracle_selector.argtypes = [ptr, i64, i64, i64, i32, dbl, i32, i32, i32, ptr, ptr, ptr,
                                        ptr, ptr, ptr]
        lib.oracle_selector.restype = i32
        lib.oracle_stage.argtypes = [ptr, i64, i64, i64, ptr, i64, i64, ptr, ptr, i32, i32, i32, i32,
                                     ptr]
        lib.oracle_denoise.argtypes = [ptr, i64, i64, i32, i32, i32, i32, i32, i32, i32, ptr, ptr, ptr,
                                       i32, dbl, ptr]
        lib.oracle_denoise.restype = i32
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def set_threads(n: int) -> None:
    """OpenMP thread count for subsequent calls (omp_set_num_threads)."""
    gomp = ctypes.CDLL("libgomp.so.1")
    gomp.omp_set_num_threads(int(n))


def max_threads() -> int:
    gomp = ctypes.CDLL("libgomp.so.1")
    gomp.omp_get_max_threads.restype = ctypes.c_int
    return int(gomp.omp_get_max_threads())


def fold(i: int, n: int) -> int:
    return int(_load().oracle_fold(i, n))


def decimate_weights() -> np.ndarray:
    w = np.zeros(8, dtype=np.float64)
    _load().oracle_decimate_weights(w.ctypes.data)
    return w


def decimate(z) -> np.ndarray:
    """O1: (C,H,W) -> (C, ceil(H/2), ceil(W/2)), fp64."""
    z = _f64(z)
    C, H, W = z.shape
    out = np.empty((C, (H + 1) // 2, (W + 1) // 2), dtype=np.float64)
    _load().oracle_decimate(z.ctypes.data, C, H, W, out.ctypes.data)
    return out


def pyramid(z, L: int) -> list[np.ndarray]:
    lv = [_f64(z)]
    for _ in range(L - 1):
        lv.append(decimate(lv[-1]))
    return lv


def tensor(z, window_size: int = 5, window_sigma: float = 1.5):
    """Eq. 6 joint-colour structure tensor: returns (a, b, c) = (Txx, Txy, Tyy), each (H, W)."""
    z = _f64(z)
    C, H, W = z.shape
    a, b, c = (np.empty((H, W)) for _ in range(3))
    _load().oracle_tensor(z.ctypes.data, C, H, W, window_size, window_sigma, a.ctypes.data,
                          b.ctypes.data, c.ctypes.data)
    return a, b, c


def eigen(a, b, c):
    """Eigen-features (theta, strength, coherence) of T = [a b; b c]."""
    a, b, c = _f64(a), _f64(b), _f64(c)
    shp = a.shape
    a, b, c = a.ravel(), b.ravel(), c.ravel()
    th, S, Co = (np.empty(a.size) for _ in range(3))
    _load().oracle_eigen(a.ctypes.data, b.ctypes.data, c.ctypes.data, a.size, th.ctypes.data,
                         S.ctypes.data, Co.ctypes.data)
    return th.reshape(shp), S.reshape(shp), Co.reshape(shp)


def quantize(theta, strength, coherence, n_o: int, n_s: int, n_c: int, ts, tc) -> np.ndarray:
    th, S, Co = _f64(theta), _f64(strength), _f64(coherence)
    shp = th.shape
    ts, tc = _f64(ts).ravel(), _f64(tc).ravel()
    assert ts.size == n_s - 1 and tc.size == n_c - 1
    out = np.empty(th.size, dtype=np.int32)
    _load().oracle_quantize(th.ravel().ctypes.data, S.ravel().ctypes.data, Co.ravel().ctypes.data,
                            th.size, n_o, n_s, n_c, _p(ts), _p(tc), out.ctypes.data)
    return out.reshape(shp)


def selector(z, n_o: int, n_s: int, n_c: int, ts, tc, window_size: int = 5,
             window_sigma: float = 1.5, features: bool = False):
    """s(i) at one level: (H, W) int32 buckets [, (theta, S, C)]."""
    z = _f64(z)
    C, H, W = z.shape
    ts, tc = _f64(ts).ravel(), _f64(tc).ravel()
    b = np.empty((H, W), dtype=np.int32)
    th, S, Co = (np.empty((H, W)) for _ in range(3))
    rc = _load().oracle_selector(z.ctypes.data, C, H, W, window_size, window_sigma, n_o, n_s, n_c,
                                 _p(ts), _p(tc), b.ctypes.data, th.ctypes.data, S.ctypes.data,
                                 Co.ctypes.data)
    if rc:
        raise MemoryError("oracle_selector")
    return (b, (th, S, Co)) if features else b


def stage(z, u1, bucket, taps, n_phases: int, nf: int, nc: int) -> np.ndarray:
    """Eq. 9 at one level (Eq. 1 when u1 is None / nc == 0). taps: [n_phases, K, nf^2 + nc^2]."""
    z = _f64(z)
    C, H, W = z.shape
    taps = _f64(taps)
    K = taps.shape[1]
    assert taps.shape == (n_phases, K, nf * nf + nc * nc)
    bucket = np.ascontiguousarray(bucket, dtype=np.int32)
    assert bucket.shape == (H, W) and bucket.min() >= 0 and bucket.max() < K
    if u1 is not None:
        u1 = _f64(u1)
        H1, W1 = u1.shape[1:]
    else:
        H1 = W1 = 0
    out = np.empty((C, H, W), dtype=np.float64)
    _load().oracle_stage(z.ctypes.data, C, H, W, _p(u1), H1, W1, bucket.ctypes.data,
                         taps.ctypes.data, n_phases, K, nf, nc if u1 is not None else 0,
                         out.ctypes.data)
    return out


def denoise(z, L: int, nf: int, nc: int, n_phases: int, n_o: int, n_s: int, n_c: int, ts, tc,
            taps, window_size: int = 5, window_sigma: float = 1.5) -> np.ndarray:
    """Full cascade for ONE frame (3, H, W) -> (3, H, W) fp64.

    taps: [n_stages, n_phases, K, nt] (a leading filter-channel axis of size 1 is accepted),
    ts: [n_stages, n_s-1], tc: [n_stages, n_c-1].
    """
    z = _f64(z)
    C, H, W = z.shape
    assert C == 3
    taps = _f64(taps)
    if taps.ndim == 5:
        assert taps.shape[1] == 1
        taps = np.ascontiguousarray(taps[:, 0])
    ts, tc = _f64(ts), _f64(tc)
    out = np.empty((3, H, W), dtype=np.float64)
    rc = _load().oracle_denoise(z.ctypes.data, H, W, L, nf, nc if L > 1 else 0, n_phases, n_o, n_s,
                                n_c, ts.ctypes.data, tc.ctypes.data, taps.ctypes.data, window_size,
                                window_sigma, out.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle_denoise failed ({rc})")
    return out


# ---------------------------------------------------------------- per-channel YCbCr path (NEXT f1)
# PAPER.md:198-202 (§3 footnote 1): "images are converted to YCbCr (ITU-R BT.601). We train filters
# separately on Y, Cb, and Cr while using the same filter selector s(.)". Full-range BT.601 with the
# constants of SPEC.md:61 on the [0, 1] scale (offset 128/255; R25); the selector runs on
# the noisy RGB levels (R26); the pyramid is decimated in RGB.
YCC_OFFSET = 128.0 / 255.0


def rgb_to_ycc(z) -> np.ndarray:
    """(3,H,W) RGB -> YCbCr: Y = .299R + .587G + .114B, Cb = o + .564(B - Y), Cr = o + .713(R - Y)."""
    z = _f64(z)
    R, G, B = z
    Y = 0.299 * R + 0.587 * G + 0.114 * B
    return np.stack([Y, YCC_OFFSET + 0.564 * (B - Y), YCC_OFFSET + 0.713 * (R - Y)])


def ycc_to_rgb(y) -> np.ndarray:
    """Exact algebraic inverse of rgb_to_ycc."""
    y = _f64(y)
    Y, Cb, Cr = y
    R = Y + (Cr - YCC_OFFSET) / 0.713
    B = Y + (Cb - YCC_OFFSET) / 0.564
    G = (Y - 0.299 * R - 0.114 * B) / 0.587
    return np.stack([R, G, B])


def denoise_ycc(z, L: int, nf: int, nc: int, n_phases: int, n_o: int, n_s: int, n_c: int, ts, tc,
                taps, window_size: int = 5, window_sigma: float = 1.5) -> np.ndarray:
    """Cascade with per-channel (Y, Cb, Cr) banks and the shared RGB selector, for ONE frame
    (3, H, W) RGB -> (3, H, W) RGB fp64. taps: [n_stages, 3, n_phases, K, nt]."""
    z = _f64(z)
    taps = _f64(taps)
    assert taps.ndim == 5 and taps.shape[1] == 3
    ts, tc = _f64(ts), _f64(tc)
    lv = pyramid(z, L)
    nsel = 1 if L == 1 else L - 1
    buckets = [selector(lv[l], n_o, n_s, n_c, ts[l], tc[l], window_size, window_sigma)
               for l in range(nsel)]
    ycc = [rgb_to_ycc(v) for v in lv]
    if L == 1:
        out = np.concatenate([stage(ycc[0][c:c + 1], None, buckets[0], taps[0, c], n_phases, nf, 0)
                              for c in range(3)])
    else:
        u = ycc[L - 1]
        for l in range(L - 2, -1, -1):
            u = np.concatenate([stage(ycc[l][c:c + 1], u[c:c + 1], buckets[l], taps[l, c],
                                      n_phases, nf, nc) for c in range(3)])
        out = u
    return ycc_to_rgb(out)


def denoise_config(cfg, z, taps=None) -> np.ndarray:
    """denoise() with the parameters of a blade_synth.Config."""
    ts, tc = cfg.thresholds()
    taps = cfg.taps() if taps is None else taps
    return denoise(z, cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.n_phases, cfg.n_orient,
                   cfg.n_strength, cfg.n_coherence, ts, tc, taps, cfg.window_size,
                   cfg.window_sigma)


def cascade_parts(cfg, z, taps=None):
    """Per-level intermediates of the cascade for one frame (for parity tests):
    returns dict(levels=[z^l], buckets=[s^l], features=[(theta,S,C)], outputs=[u^l])."""
    ts, tc = cfg.thresholds()
    taps = cfg.taps() if taps is None else taps
    if taps.ndim == 5:
        taps = taps[:, 0]
    L = cfg.levels
    lv = pyramid(z, L)
    nsel = 1 if L == 1 else L - 1
    buckets, feats = [], []
    for l in range(nsel):
        b, f = selector(lv[l], cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts[l], tc[l],
                        cfg.window_size, cfg.window_sigma, features=True)
        buckets.append(b)
        feats.append(f)
    outs = [None] * L
    if L == 1:
        outs[0] = stage(lv[0], None, buckets[0], taps[0], cfg.n_phases, cfg.fine_size, 0)
    else:
        outs[L - 1] = lv[L - 1]
        for l in range(L - 2, -1, -1):
            outs[l] = stage(lv[l], outs[l + 1], buckets[l], taps[l], cfg.n_phases, cfg.fine_size,
                            cfg.coarse_size)
    return dict(levels=lv, buckets=buckets, features=feats, outputs=outs)

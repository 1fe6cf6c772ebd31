"""Thin Python binding of the C ABI in include/blade_ms.h (argument marshalling only).

Every step of the path runs in the CUDA kernels of `libblade_ms.so`; there is no CPU or eager
PyTorch fallback: if the library is missing or fails to load, every call raises. PyTorch is
used for device memory and streams only (tensors are passed to the ABI as raw pointers).
"""
from __future__ import annotations

import ctypes
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import build as _build

_lib = None

STATUS = {0: "BLADE_OK", 1: "BLADE_EINVAL", 2: "BLADE_ENONFINITE", 3: "BLADE_ESHAPE",
          4: "BLADE_EDEVICE", 5: "BLADE_ENOMEM", 6: "BLADE_ECUDA", 7: "BLADE_EUNSUPPORTED"}


class BladeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("fine_size", ctypes.c_int32),
                ("coarse_size", ctypes.c_int32), ("n_phases", ctypes.c_int32),
                ("n_filter_channels", ctypes.c_int32), ("window_size", ctypes.c_int32),
                ("window_sigma", ctypes.c_float), ("clamp_output", ctypes.c_int32)]


class _Layout(ctypes.Structure):
    _fields_ = [("n_orient", ctypes.c_int32), ("n_strength", ctypes.c_int32),
                ("n_coherence", ctypes.c_int32),
                ("strength_thresholds", ctypes.POINTER(ctypes.c_double)),
                ("coherence_thresholds", ctypes.POINTER(ctypes.c_double))]


class _Info(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("fine_size", ctypes.c_int32),
                ("coarse_size", ctypes.c_int32), ("n_phases", ctypes.c_int32),
                ("n_stages", ctypes.c_int32), ("K", ctypes.c_int32), ("device", ctypes.c_int32),
                ("bank_bytes_device", ctypes.c_size_t), ("stage_smem_bytes", ctypes.c_size_t),
                ("stage_phase_groups", ctypes.c_int32)]


class _Region(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("plane_stride", ctypes.c_int64), ("row0", ctypes.c_int32),
                ("rows", ctypes.c_int32), ("pitch", ctypes.c_int32), ("planes", ctypes.c_int32)]


MAX_LEVELS = 12  # BLADE_MAX_LEVELS


class _XLayout(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("n_steps", ctypes.c_int32), ("halo_z", ctypes.c_int32),
                ("halo_u", ctypes.c_int32), ("own_lo", ctypes.c_int32 * MAX_LEVELS),
                ("own_hi", ctypes.c_int32 * MAX_LEVELS), ("in_row0", ctypes.c_int32),
                ("in_rows", ctypes.c_int32), ("ws_bytes", ctypes.c_uint64),
                ("send", (_Region * 2) * (2 * MAX_LEVELS)), ("recv", (_Region * 2) * (2 * MAX_LEVELS))]


EXPORTS = ["blade_ms_create", "blade_ms_workspace_size", "blade_ms_denoise", "blade_ms_denoise_host",
           "blade_ms_pipeline_workspace_size", "blade_ms_denoise_pipelined",
           "blade_ms_band_rows", "blade_ms_band_plan", "blade_ms_fallback_count",
           "blade_ms_train_layout", "blade_ms_train_workspace_size", "blade_ms_train_accumulate",
           "blade_ms_train_solve", "blade_ms_band_workspace_size", "blade_ms_denoise_rows",
           "blade_ms_selector", "blade_ms_pyramid", "blade_ms_get_info", "blade_ms_launch_count",
           "blade_ms_stage_kernel", "blade_ms_xband_layout", "blade_ms_xband_step",
           "blade_ms_set_profiling", "blade_ms_profile_read",
           "blade_ms_destroy", "blade_ms_status_string", "blade_ms_last_error"]


def library_path() -> Path:
    """The in-tree library; BLADE_MS_LIB=<path> selects another build of the same ABI
    (kernel-variant experiments only; never a CPU path)."""
    import os
    alt = os.environ.get("BLADE_MS_LIB")
    return Path(alt) if alt else _build.LIB


def lib():
    """Load libblade_ms.so (building it first if sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    try:
        _build.build()
    except Exception as e:  # no nvcc on this machine: use the shipped .so if present
        if not _build.LIB.exists():
            raise RuntimeError(f"libblade_ms.so is missing and could not be built: {e}") from e
    L = ctypes.CDLL(str(library_path()))
    P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    L.blade_ms_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_Layout), P, sz,
                                  ctypes.c_int, ctypes.POINTER(P)]
    L.blade_ms_workspace_size.argtypes = [P, i32, i32, i32, ctypes.POINTER(sz)]
    L.blade_ms_denoise.argtypes = [P, P, P, i32, i32, i32, P, sz, P]
    L.blade_ms_pipeline_workspace_size.argtypes = [P, i32, i32, i32, i32, ctypes.POINTER(sz)]
    L.blade_ms_denoise_pipelined.argtypes = [P, P, P, i32, i32, i32, i32, i32, P, sz, P]
    L.blade_ms_denoise_host.argtypes = [P, P, P, i32, i32, i32, P, P, P, sz, P]
    L.blade_ms_band_rows.argtypes = [P, i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.blade_ms_band_plan.argtypes = [ctypes.POINTER(_Config), i32, i32, i32, ctypes.POINTER(i32),
                                     ctypes.POINTER(i32)]
    L.blade_ms_fallback_count.argtypes = [P, i32, i32, i32, P, sz, P]
    L.blade_ms_train_layout.argtypes = [P, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.blade_ms_train_workspace_size.argtypes = [P, i32, i32, i32, ctypes.POINTER(sz)]
    L.blade_ms_train_accumulate.argtypes = [P, i32, P, P, P, i32, i32, i32, P, P, P, sz, P]
    L.blade_ms_train_solve.argtypes = [P, P, P, ctypes.c_double, ctypes.c_uint64, P]
    L.blade_ms_band_workspace_size.argtypes = [P, i32, i32, i32, i32, ctypes.POINTER(sz)]
    L.blade_ms_denoise_rows.argtypes = [P, P, i32, i32, P, i32, i32, i32, i32, P, sz, P]
    L.blade_ms_xband_layout.argtypes = [ctypes.POINTER(_Config), i32, i32, i32, i32, i32,
                                        ctypes.POINTER(_XLayout)]
    L.blade_ms_xband_step.argtypes = [P, i32, P, i32, i32, P, i32, i32, i32, i32, P, sz, P]
    L.blade_ms_selector.argtypes = [P, P, i32, i32, i32, P, P, sz, P]
    L.blade_ms_pyramid.argtypes = [P, P, i32, i32, i32, P, P, sz, P]
    L.blade_ms_get_info.argtypes = [P, ctypes.POINTER(_Info)]
    L.blade_ms_launch_count.argtypes = [P, i32, i32, i32, ctypes.POINTER(i32)]
    L.blade_ms_stage_kernel.argtypes = [P, i32, i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.blade_ms_set_profiling.argtypes = [P, i32]
    L.blade_ms_profile_read.argtypes = [P, P, P]
    L.blade_ms_destroy.argtypes = [P]
    L.blade_ms_status_string.argtypes = [ctypes.c_int]
    L.blade_ms_status_string.restype = ctypes.c_char_p
    L.blade_ms_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("blade_ms_status_string", "blade_ms_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise BladeError(rc, lib().blade_ms_last_error().decode())


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def band_plan(levels: int, fine_size: int, coarse_size: int, window_size: int, H: int,
              out_row0: int, out_rows: int) -> tuple[int, int]:
    """blade_ms_band_plan: input rows (in_row0, in_rows) a row band needs (host only, no device)."""
    cfg = _Config(levels, fine_size, coarse_size if levels > 1 else 0, 4 if levels > 1 else 1, 1,
                  window_size, 1.5, 0)
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().blade_ms_band_plan(ctypes.byref(cfg), H, out_row0, out_rows, ctypes.byref(a),
                                    ctypes.byref(b)))
    return a.value, b.value


def _region(r: _Region) -> dict:
    return {"offset": r.offset, "plane_stride": r.plane_stride, "row0": r.row0, "rows": r.rows,
            "pitch": r.pitch, "planes": r.planes}


def xband_layout(levels: int, fine_size: int, coarse_size: int, window_size: int, K: int, H: int,
                 W: int, out_row0: int, out_rows: int) -> dict:
    """blade_ms_xband_layout (host only): the plan of a row band that exchanges per-level halo
    rows with its neighbours (NEXT f3): own rows per level, input rows, workspace bytes, steps
    and, per step and side (0 = band above, 1 = below), the send / recv workspace regions."""
    cfg = _Config(levels, fine_size, coarse_size if levels > 1 else 0, 4 if levels > 1 else 1, 1,
                  window_size, 1.5, 0)
    x = _XLayout()
    _check(lib().blade_ms_xband_layout(ctypes.byref(cfg), K, H, W, out_row0, out_rows, ctypes.byref(x)))
    n = x.n_steps
    return {"levels": x.levels, "n_steps": n, "halo_z": x.halo_z, "halo_u": x.halo_u,
            "own": [(x.own_lo[l], x.own_hi[l]) for l in range(x.levels)],
            "in_row0": x.in_row0, "in_rows": x.in_rows, "ws_bytes": int(x.ws_bytes),
            "send": [[_region(x.send[s][d]) for d in range(2)] for s in range(n)],
            "recv": [[_region(x.recv[s][d]) for d in range(2)] for s in range(n)]}


def region_view(ws: torch.Tensor, r: dict) -> torch.Tensor:
    """[planes, rows, pitch] fp32 view of a region of a uint8 workspace tensor."""
    f = ws.view(torch.float32)
    assert r["offset"] % 4 == 0 and r["plane_stride"] % 4 == 0
    return torch.as_strided(f, (r["planes"], r["rows"], r["pitch"]),
                            (r["plane_stride"] // 4, r["pitch"], 1), r["offset"] // 4)


class BladeMS:
    """Handle over blade_ms_create / blade_ms_denoise / blade_ms_destroy."""

    def __init__(self, levels: int, fine_size: int, coarse_size: int, n_phases: int,
                 n_orient: int, n_strength: int, n_coherence: int, strength_thresholds,
                 coherence_thresholds, taps, window_size: int = 5, window_sigma: float = 1.5,
                 clamp_output: bool = False, device: int = 0, n_filter_channels: int = 1):
        L = lib()
        cfg = _Config(levels, fine_size, coarse_size, n_phases, n_filter_channels, window_size,
                      window_sigma, int(clamp_output))
        self._ts = np.ascontiguousarray(np.asarray(strength_thresholds, dtype=np.float64).ravel())
        self._tc = np.ascontiguousarray(np.asarray(coherence_thresholds, dtype=np.float64).ravel())
        dp = ctypes.POINTER(ctypes.c_double)
        lay = _Layout(n_orient, n_strength, n_coherence,
                      self._ts.ctypes.data_as(dp) if self._ts.size else None,
                      self._tc.ctypes.data_as(dp) if self._tc.size else None)
        taps = np.ascontiguousarray(np.asarray(taps, dtype=np.float32).ravel())
        h = ctypes.c_void_p()
        _check(L.blade_ms_create(ctypes.byref(cfg), ctypes.byref(lay), taps.ctypes.data,
                                 taps.size, device, ctypes.byref(h)))
        self._h = h
        self.device = device
        self.levels = levels
        self.n_stages = max(levels - 1, 1)
        self.K = n_orient * n_strength * n_coherence
        self.fine_size, self.coarse_size, self.window_size = fine_size, coarse_size, window_size
        self.map_dtype = torch.uint16 if self.K > 256 else torch.uint8

    @classmethod
    def from_config(cls, cfg, taps=None, device: int = 0, clamp_output: bool = False):
        """Build from any object with the attributes of blade_synth.Config; taps of shape
        [n_stages, 3, n_phases, K, nt] select per-channel YCbCr banks (n_filter_channels = 3)."""
        ts, tc = cfg.thresholds()
        taps = cfg.taps() if taps is None else taps
        nch = int(np.asarray(taps).shape[1]) if np.asarray(taps).ndim == 5 else 1
        return cls(cfg.levels, cfg.fine_size, cfg.coarse_size if cfg.levels > 1 else 0,
                   cfg.n_phases, cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts, tc, taps,
                   cfg.window_size, cfg.window_sigma, clamp_output, device, n_filter_channels=nch)

    # -------------------------------------------------------------------------------- queries
    def close(self):
        if getattr(self, "_h", None):
            lib().blade_ms_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = _Info()
        _check(lib().blade_ms_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    def workspace_size(self, N: int, H: int, W: int) -> int:
        b = ctypes.c_size_t()
        _check(lib().blade_ms_workspace_size(self._h, N, H, W, ctypes.byref(b)))
        return b.value

    def launch_count(self, N: int, H: int, W: int) -> int:
        c = ctypes.c_int32()
        _check(lib().blade_ms_launch_count(self._h, N, H, W, ctypes.byref(c)))
        return c.value

    STAGE_KINDS = ("k_stage", "k_stage_tma", "k_stage_ph", "k_stage_p2")

    def stage_kernel(self, N: int, H: int, W: int, level: int) -> tuple[str, int]:
        """(kernel name, output rows per thread) of stage `level` for a denoise(N, H, W) call."""
        k, r = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().blade_ms_stage_kernel(self._h, N, H, W, level, ctypes.byref(k), ctypes.byref(r)))
        return self.STAGE_KINDS[k.value], r.value

    def fallback_count(self, N: int, H: int, W: int, workspace: torch.Tensor) -> list[int]:
        """Uncertified (fp64-recomputed) selector pixels per level of the last call that used
        `workspace` (synchronises)."""
        torch.cuda.synchronize(workspace.device)
        c = np.zeros(16, np.uint32)
        _check(lib().blade_ms_fallback_count(self._h, N, H, W, _ptr(workspace), workspace.numel(),
                                             c.ctypes.data))
        return [int(v) for v in c[:self.n_stages]]

    # -------------------------------------------------------------------------------- training
    def train_layout(self) -> tuple[int, int, int]:
        """(nt, ntp, n_seg) of the training accumulators (NEXT f4)."""
        a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().blade_ms_train_layout(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def train_accumulators(self, device=None):
        """Zeroed (E, count) device accumulators for one stage."""
        nt, ntp, n_seg = self.train_layout()
        dev = device or f"cuda:{self.device}"
        return (torch.zeros((n_seg, ntp, ntp), dtype=torch.float64, device=dev),
                torch.zeros(n_seg, dtype=torch.int64, device=dev))

    def train_accumulate(self, level: int, z: torch.Tensor, u_clean: torch.Tensor,
                         u_coarse: torch.Tensor | None, E: torch.Tensor, count: torch.Tensor,
                         workspace: torch.Tensor | None = None, stream=None):
        """blade_ms_train_accumulate over the frames of z / u_clean ([N,3,H,W] CUDA fp32)."""
        self._check_img(z, "z")
        self._check_img(u_clean, "u_clean")
        N, _, H, W = z.shape
        if workspace is None:
            b = ctypes.c_size_t()
            _check(lib().blade_ms_train_workspace_size(self._h, N, H, W, ctypes.byref(b)))
            workspace = torch.empty(b.value, dtype=torch.uint8, device=z.device)
        _check(lib().blade_ms_train_accumulate(self._h, level, _ptr(z), _ptr(u_clean),
                                               _ptr(u_coarse), N, H, W, _ptr(E), _ptr(count),
                                               _ptr(workspace), workspace.numel(),
                                               _stream_ptr(stream)))

    def train_solve(self, E: torch.Tensor, count: torch.Tensor, ridge: float = 1e-3,
                    min_count: int | None = None) -> np.ndarray:
        """Host fp64 solve of every (phase, bucket): float32 [n_phases, K, nt]."""
        nt, ntp, n_seg = self.train_layout()
        Eh = np.ascontiguousarray(E.detach().cpu().numpy())
        ch = np.ascontiguousarray(count.detach().cpu().numpy().astype(np.uint64))
        taps = np.empty((n_seg, nt), np.float32)
        mc = 4 * nt if min_count is None else min_count
        _check(lib().blade_ms_train_solve(self._h, Eh.ctypes.data, ch.ctypes.data, float(ridge), mc,
                                          taps.ctypes.data))
        return taps.reshape(-1, self.K, nt)

    def set_profiling(self, enable: bool):
        _check(lib().blade_ms_set_profiling(self._h, int(enable)))

    KINDS = ("decimate", "selector", "stage", "fixup")

    def profile_read(self) -> dict:
        """{(kind, level): (total_ms, launches)} since the last read (synchronises)."""
        ms = np.zeros(64, np.float64)
        cnt = np.zeros(64, np.int32)
        _check(lib().blade_ms_profile_read(self._h, ms.ctypes.data, cnt.ctypes.data))
        return {(self.KINDS[i // 16], i % 16): (float(ms[i]), int(cnt[i]))
                for i in range(64) if cnt[i]}

    def workspace(self, N: int, H: int, W: int) -> torch.Tensor:
        return torch.empty(self.workspace_size(N, H, W), dtype=torch.uint8,
                           device=f"cuda:{self.device}")

    # -------------------------------------------------------------------------------- compute
    @staticmethod
    def _check_img(x: torch.Tensor, name: str):
        if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 4
                and x.shape[1] == 3):
            raise ValueError(f"{name} must be a contiguous CUDA float32 [N,3,H,W] tensor")

    def denoise(self, x: torch.Tensor, out: torch.Tensor | None = None,
                workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        self._check_img(x, "x")
        N, _, H, W = x.shape
        out = torch.empty_like(x) if out is None else out
        self._check_img(out, "out")
        ws = self.workspace(N, H, W) if workspace is None else workspace
        _check(lib().blade_ms_denoise(self._h, _ptr(x), _ptr(out), N, H, W, _ptr(ws), ws.numel(),
                                      _stream_ptr(stream)))
        return out

    def pipeline_workspace_size(self, chunk: int, n_streams: int, H: int, W: int) -> int:
        n = ctypes.c_size_t()
        _check(lib().blade_ms_pipeline_workspace_size(self._h, chunk, n_streams, H, W, ctypes.byref(n)))
        return n.value

    def denoise_pipelined(self, x: torch.Tensor, out: torch.Tensor | None = None, chunk: int = 1,
                          n_streams: int = 2, workspace: torch.Tensor | None = None,
                          stream=None) -> torch.Tensor:
        """Frame-chunked schedule (NEXT f3): chunks of `chunk` frames on `n_streams` internal
        streams, intermediates L2-resident; bit-identical to denoise()."""
        self._check_img(x, "x")
        N, _, H, W = x.shape
        out = torch.empty_like(x) if out is None else out
        self._check_img(out, "out")
        if workspace is None:
            workspace = torch.empty(self.pipeline_workspace_size(chunk, n_streams, H, W),
                                    dtype=torch.uint8, device=f"cuda:{self.device}")
        _check(lib().blade_ms_denoise_pipelined(self._h, _ptr(x), _ptr(out), N, H, W, chunk,
                                                n_streams, _ptr(workspace), workspace.numel(),
                                                _stream_ptr(stream)))
        return out

    def denoise_host(self, x_host: torch.Tensor, out_host: torch.Tensor, d_in: torch.Tensor,
                     d_out: torch.Tensor, workspace: torch.Tensor, stream=None) -> torch.Tensor:
        """End-to-end: host -> device copies, denoise, device -> host copies (synchronous)."""
        if x_host.is_cuda or out_host.is_cuda:
            raise ValueError("x_host / out_host must be host tensors")
        N, _, H, W = x_host.shape
        _check(lib().blade_ms_denoise_host(self._h, _ptr(x_host), _ptr(out_host), N, H, W,
                                           _ptr(d_in), _ptr(d_out), _ptr(workspace),
                                           workspace.numel(), _stream_ptr(stream)))
        return out_host

    def selector(self, x: torch.Tensor, workspace: torch.Tensor | None = None,
                 stream=None) -> list[torch.Tensor]:
        """Bucket maps s^l (uint8 [N,H_l,W_l]; uint16 when K > 256) for l = 0 .. n_stages-1."""
        self._check_img(x, "x")
        N, _, H, W = x.shape
        dims = self.level_dims(H, W)
        maps = [torch.empty((N, dims[l][0], dims[l][1]), dtype=self.map_dtype, device=x.device)
                for l in range(self.n_stages)]
        arr = (ctypes.c_void_p * len(maps))(*[m.data_ptr() for m in maps])
        ws = self.workspace(N, H, W) if workspace is None else workspace
        _check(lib().blade_ms_selector(self._h, _ptr(x), N, H, W, arr, _ptr(ws), ws.numel(),
                                       _stream_ptr(stream)))
        return maps

    def pyramid(self, x: torch.Tensor, stream=None) -> list[torch.Tensor]:
        """Levels z^1 .. z^{L-1} (fp32 [N,3,H_l,W_l])."""
        self._check_img(x, "x")
        N, _, H, W = x.shape
        dims = self.level_dims(H, W)
        lv = [torch.empty((N, 3, dims[l][0], dims[l][1]), dtype=torch.float32, device=x.device)
              for l in range(1, self.levels)]
        arr = (ctypes.c_void_p * max(len(lv), 1))(*[t.data_ptr() for t in lv])
        ws = self.workspace(N, H, W)
        _check(lib().blade_ms_pyramid(self._h, _ptr(x), N, H, W, arr, _ptr(ws), ws.numel(),
                                      _stream_ptr(stream)))
        return lv

    def level_dims(self, H: int, W: int) -> list[tuple[int, int]]:
        d = [(H, W)]
        for _ in range(self.levels - 1):
            d.append(((d[-1][0] + 1) // 2, (d[-1][1] + 1) // 2))
        return d

    # -------------------------------------------------------------------------------- bands
    def band_rows(self, H: int, out_row0: int, out_rows: int) -> tuple[int, int]:
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().blade_ms_band_rows(self._h, H, out_row0, out_rows, ctypes.byref(a),
                                        ctypes.byref(b)))
        return a.value, b.value

    def band_workspace_size(self, H: int, W: int, out_row0: int, out_rows: int) -> int:
        b = ctypes.c_size_t()
        _check(lib().blade_ms_band_workspace_size(self._h, H, W, out_row0, out_rows,
                                                  ctypes.byref(b)))
        return b.value

    def denoise_rows(self, in_band: torch.Tensor, in_row0: int, out_row0: int, out_rows: int,
                     H: int, out_band: torch.Tensor | None = None,
                     workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """in_band: CUDA fp32 [3, in_rows, W] holding global rows [in_row0, in_row0+in_rows)."""
        if not (in_band.is_cuda and in_band.dtype == torch.float32 and in_band.is_contiguous()
                and in_band.dim() == 3 and in_band.shape[0] == 3):
            raise ValueError("in_band must be a contiguous CUDA float32 [3, rows, W] tensor")
        _, in_rows, W = in_band.shape
        if out_band is None:
            out_band = torch.empty((3, out_rows, W), dtype=torch.float32, device=in_band.device)
        if workspace is None:
            workspace = torch.empty(self.band_workspace_size(H, W, out_row0, out_rows),
                                    dtype=torch.uint8, device=in_band.device)
        _check(lib().blade_ms_denoise_rows(self._h, _ptr(in_band), in_row0, in_rows,
                                           _ptr(out_band), out_row0, out_rows, H, W,
                                           _ptr(workspace), workspace.numel(),
                                           _stream_ptr(stream)))
        return out_band

    # ------------------------------------------------------------------ bands with halo exchange
    def xband_layout(self, H: int, W: int, out_row0: int, out_rows: int) -> dict:
        return xband_layout(self.levels, self.fine_size, self.coarse_size, self.window_size, self.K,
                            H, W, out_row0, out_rows)

    def xband_step(self, step: int, in_band: torch.Tensor, in_row0: int, out_band: torch.Tensor,
                   out_row0: int, H: int, workspace: torch.Tensor, stream=None):
        """Step `step` of a halo-exchange band (blade_ms_xband_step); in_band [3, rows, W]
        holds global rows from in_row0, out_band [3, out_rows, W]."""
        _, in_rows, W = in_band.shape
        out_rows = out_band.shape[1]
        _check(lib().blade_ms_xband_step(self._h, step, _ptr(in_band), in_row0, in_rows,
                                         _ptr(out_band), out_row0, out_rows, H, W,
                                         _ptr(workspace), workspace.numel(), _stream_ptr(stream)))

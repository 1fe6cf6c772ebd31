"""C-ABI checks that need no GPU: the library loads, exports every symbol include/blade_ms.h
declares, and rejects bad arguments at create with the documented status BEFORE touching a
device (argument validation precedes the device query)."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1802_06130_b200 import blade_ms as bm

HEADER = Path(__file__).resolve().parents[1] / "include" / "blade_ms.h"


def test_library_exports_every_declared_symbol():
    text = HEADER.read_text()
    declared = set(re.findall(r"\b(blade_ms_\w+)\s*\(", text))
    assert len(declared) >= 14
    L = bm.lib()
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(bm.EXPORTS) == declared


def test_status_strings():
    L = bm.lib()
    for s in range(8):
        assert L.blade_ms_status_string(s).decode()
    assert L.blade_ms_status_string(99).decode() == "unknown status"


def _create(levels=3, nf=5, nc=5, n_phases=4, ws=5, sigma=1.5, K=(16, 3, 3), ntaps=None,
            ts=None, tc=None, taps=None, n_filter_channels=1, clamp=0):
    L = bm.lib()
    cfg = bm._Config(levels, nf, nc, n_phases, n_filter_channels, ws, sigma, clamp)
    n_stages = max(levels - 1, 1)
    Kt = K[0] * K[1] * K[2]
    nt = nf * nf + (nc * nc if levels > 1 else 0)
    if taps is None:
        taps = np.zeros(n_stages * n_phases * Kt * nt, np.float32)
    ts = np.tile([0.1, 0.2], n_stages) if ts is None else np.asarray(ts, np.float64)
    tc = np.tile([0.3, 0.6], n_stages) if tc is None else np.asarray(tc, np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    lay = bm._Layout(K[0], K[1], K[2], ts.ctypes.data_as(dp), tc.ctypes.data_as(dp))
    h = ctypes.c_void_p(123)
    rc = L.blade_ms_create(ctypes.byref(cfg), ctypes.byref(lay), taps.ctypes.data,
                           taps.size if ntaps is None else ntaps, 0, ctypes.byref(h))
    return rc, h


EINVAL, ENONFINITE, ESHAPE, EDEVICE, EUNSUP = 1, 2, 3, 4, 7


@pytest.mark.parametrize("kw,status", [
    (dict(nf=4), EINVAL),                      # even footprint
    (dict(nf=11), EINVAL),                     # out of range
    (dict(levels=0), EINVAL),
    (dict(levels=1, nc=5, n_phases=1), EINVAL),  # coarse block with a single level
    (dict(levels=1, nc=0, n_phases=4), EINVAL),  # phases with a single level
    (dict(n_phases=2), EINVAL),
    (dict(ws=4), EINVAL),
    (dict(sigma=0.0), EINVAL),
    (dict(clamp=2), EINVAL),
    (dict(ts=[0.2, 0.1, 0.2, 0.3]), EINVAL),   # not ascending
    (dict(tc=[0.3, np.nan, 0.3, 0.6]), ENONFINITE),
    (dict(ntaps=7), ESHAPE),
    (dict(K=(512, 16, 16)), EUNSUP),           # K = 131072 > 65536 (uint16 maps)
    (dict(n_filter_channels=3), ESHAPE),       # per-channel banks need 3x the taps
    (dict(n_filter_channels=2), EINVAL),
])
def test_create_rejects_bad_arguments(kw, status):
    rc, h = _create(**kw)
    assert rc == status, bm.lib().blade_ms_last_error().decode()
    assert h.value is None
    assert bm.lib().blade_ms_last_error().decode()


def test_create_rejects_nonfinite_tap():
    taps = np.zeros(2 * 4 * 144 * 50, np.float32)
    taps[777] = np.inf
    rc, _ = _create(taps=taps)
    assert rc == ENONFINITE


def test_create_without_gpu_reports_device_error():
    """On a machine with no GPU a VALID configuration fails with EDEVICE (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc, _ = _create()
    assert rc == EDEVICE


def test_null_arguments():
    L = bm.lib()
    h = ctypes.c_void_p()
    assert L.blade_ms_create(None, None, None, 0, 0, ctypes.byref(h)) == EINVAL
    assert L.blade_ms_create(None, None, None, 0, 0, None) == EINVAL
    assert L.blade_ms_destroy(None) == 0
    sz = ctypes.c_size_t()
    assert L.blade_ms_workspace_size(None, 1, 8, 8, ctypes.byref(sz)) == EINVAL
    assert L.blade_ms_denoise(None, None, None, 1, 8, 8, None, 0, None) == EINVAL

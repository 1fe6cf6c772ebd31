"""Per-kernel timeline of one small call in a CUDA graph (BLADE_TRACE build via BLADE_MS_LIB):
first CTA entry, last griddepcontrol.wait return, (stage: bank resident) and last warp exit of
every kernel kind, us relative to the first k_down entry."""
import ctypes
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS
from paper_1802_06130_b200.blade_ms import lib
H = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = bs.load_config("c1"); cfg.H, cfg.W, cfg.N = H, H, 1
h = BladeMS.from_config(cfg)
x = torch.from_numpy(cfg.batch()).cuda(); o = torch.empty_like(x); ws = h.workspace(1, H, H)
L = lib()
L.blade_ms_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((2, 16, 3), dtype=np.uint64)
h.denoise(x, o, ws); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    h.denoise(x, o, ws, torch.cuda.current_stream())
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for rep in range(3):
    L.blade_ms_trace(None, 1)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    L.blade_ms_trace(buf.ctypes.data, 0)
    names = {(0, 0): "k_down0", (0, 1): "k_down1", (0, 2): "fixup_multi", (1, 8): "stage (W<512: level 1)",
             (1, 10): "stage (W>=512: level 0)"}
    t0 = min(int(buf[tu, k, 0]) for (tu, k) in names if buf[tu, k, 0] != np.uint64(2**64 - 1))
    print(f"--- replay {rep} (c1 recipe {H}x{H})")
    for (tu, k), nm in names.items():
        e, w, x_ = buf[tu, k]
        if e == np.uint64(2**64 - 1):
            continue
        bank = buf[tu, k + 1, 1] if tu == 1 else 0
        print(f"{nm:26s} entry {(int(e) - t0) / 1e3:7.2f}  waited {(int(w) - t0) / 1e3:7.2f}"
              + (f"  bank {(int(bank) - t0) / 1e3:7.2f}" if bank else "") + f"  exit {(int(x_) - t0) / 1e3:7.2f} us")

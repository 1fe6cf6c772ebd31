"""k_down_tile vs k_down on single frames of growing size (c1 recipe, CUDA-graph replay, median
us of 50 steps): run twice, with BLADE_DOWN_TILE=0 and with a huge threshold, to place the default
size threshold of the small-call down pass (blade_ms.cu tile_down)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS

tag = os.environ.get("BLADE_DOWN_TILE", "default")
for H, W in [(256, 256), (512, 512), (768, 768), (1024, 1024), (1448, 1448), (2048, 2048)]:
    cfg = bs.load_config("c1")
    cfg.H, cfg.W, cfg.N = H, W, 1
    h = BladeMS.from_config(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    out = torch.empty_like(x)
    ws = h.workspace(1, H, W)
    h.denoise(x, out, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.denoise(x, out, ws, torch.cuda.current_stream())
    for _ in range(5):
        g.replay()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(51)]
    ev[0].record()
    for k in range(50):
        g.replay()
        ev[k + 1].record()
    torch.cuda.synchronize()
    t = [ev[k].elapsed_time(ev[k + 1]) * 1e3 for k in range(50)]
    print(f"BLADE_DOWN_TILE={tag} c1 {H}x{W}: launches {h.launch_count(1, H, W)}, median {np.median(t):.1f} us", flush=True)

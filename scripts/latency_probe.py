"""Latency floor of a small cascade call: the c1 recipe (L=3, 5 launches) on shrinking images,
CUDA-graph replay, back-to-back steps timed with CUDA events (median per step, us)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS

for name, shapes in (("c1", [(8, 8), (64, 64), (128, 128), (256, 256), (512, 512)]), ("c0", [(8, 8), (64, 64)])):
    for H, W in shapes:
        if len(sys.argv) > 1 and f"{H}x{W}" not in sys.argv[1:]: continue
        cfg = bs.load_config(name)
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
        print(f"{name} {H}x{W}: launches {h.launch_count(1, H, W)}, median {np.median(t):.1f} us, best {min(t):.1f} us", flush=True)

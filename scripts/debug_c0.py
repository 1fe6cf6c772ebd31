import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
cfg = bs.load_config(name)
x = torch.from_numpy(cfg.batch()).cuda()
h = BladeMS.from_config(cfg)
ws = h.workspace(cfg.N, cfg.H, cfg.W)
print("ws bytes", ws.numel())
out = torch.empty_like(x)
try:
    h.denoise(x, out, ws)
    torch.cuda.synchronize()
    print("denoise ok", h.fallback_count(cfg.N, cfg.H, cfg.W, ws))
except Exception as e:
    print("ERR", e)

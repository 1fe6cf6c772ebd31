"""One small call (profiling target): c1 recipe at HxW (default 8x8), 3 warm calls."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS
H = int(sys.argv[1]) if len(sys.argv) > 1 else 8
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = bs.load_config("c1"); cfg.H, cfg.W, cfg.N = H, W, 1
h = BladeMS.from_config(cfg)
x = torch.from_numpy(cfg.batch()).cuda(); o = torch.empty_like(x); ws = h.workspace(1, H, W)
for _ in range(3):
    h.denoise(x, o, ws)
torch.cuda.synchronize()
print("ok")

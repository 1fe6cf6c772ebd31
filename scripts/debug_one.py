"""Run one configuration through the C ABI with BLADE_SYNC_DEBUG=1 (debug helper)."""
import os, sys
os.environ.setdefault("BLADE_SYNC_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS
name, H, W, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = bs.load_config(name)
cfg.H, cfg.W, cfg.N = H, W, N
h = BladeMS.from_config(cfg)
print(name, H, W, N, h.info(), flush=True)
x = torch.from_numpy(cfg.batch()).cuda()
try:
    out = h.denoise(x)
    torch.cuda.synchronize()
    print("ok", float(out.abs().max()))
except Exception as e:
    print("FAIL", e)

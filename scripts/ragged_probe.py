"""Stage-kernel cost for ragged widths: c3 recipe at W = 1920 (TMA) vs 1918 (generic) and 1916."""
import torch
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS

for W in (1920, 1918, 1916, 1917):
    cfg = bs.load_config("c3")
    cfg.W, cfg.N = W, 8
    h = BladeMS.from_config(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    out = torch.empty_like(x)
    ws = h.workspace(8, cfg.H, W)
    for _ in range(3):
        h.denoise(x, out, ws)
    h.set_profiling(True)
    for _ in range(10):
        h.denoise(x, out, ws)
    prof = h.profile_read()
    h.set_profiling(False)
    print(W, [h.stage_kernel(8, cfg.H, W, l) for l in range(2)],
          {f"{k[0]}{k[1]}": round(t / c, 4) for k, (t, c) in sorted(prof.items())})

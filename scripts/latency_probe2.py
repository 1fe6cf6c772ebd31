"""Where the fixed per-launch time of small calls goes: c0 / c1 recipes on an 8x8 image (no work)
under knob settings, CUDA-graph replay, median per step (us); plus a graph of 3 / 5 tiny torch
kernels as the launch-overhead reference."""
import os
import subprocess
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
import blade_synth as bs
from paper_1802_06130_b200 import BladeMS
def timeg(fn, n=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        for _ in range(5): g.replay()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        ev[0].record()
        for k in range(n):
            g.replay(); ev[k + 1].record()
        torch.cuda.synchronize()
    return np.median([ev[k].elapsed_time(ev[k + 1]) * 1e3 for k in range(n)])
out = []
for name in ("c0", "c1"):
    cfg = bs.load_config(name); cfg.H, cfg.W, cfg.N = 8, 8, 1
    h = BladeMS.from_config(cfg)
    x = torch.from_numpy(cfg.batch()).cuda(); o = torch.empty_like(x); ws = h.workspace(1, 8, 8)
    out.append(f"{name}: {timeg(lambda: h.denoise(x, o, ws, torch.cuda.current_stream())):.1f}")
    out.append(f"{name} selector only: {timeg(lambda: h.selector(x, workspace=ws, stream=torch.cuda.current_stream())):.1f}")
a = torch.zeros(64, device="cuda")
out.append(f"torch x3: {timeg(lambda: [a.add_(1) for _ in range(3)]):.1f}")
out.append(f"torch x5: {timeg(lambda: [a.add_(1) for _ in range(5)]):.1f}")
print(" | ".join(out))
''' % str(ROOT)
for env in ({}, {"BLADE_PDL": "0"}, {"BLADE_CARVEOUT": "-1"}, {"BLADE_PDL": "0", "BLADE_CARVEOUT": "-1"}):
    r = subprocess.run([sys.executable, "-c", CHILD], env={**os.environ, **env}, capture_output=True, text=True)
    print(env or "default", "->", r.stdout.strip() or r.stderr[-500:], flush=True)

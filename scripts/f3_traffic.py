"""DRAM traffic of one c3-recipe call, batch schedule vs frame-chunked schedule (NEXT f3).
Run under ncu with --profile-from-start off --cache-control none: only the call between
profiler start / stop is captured, and the L2 keeps its state across kernels.
  ncu --profile-from-start off --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      python scripts/f3_traffic.py --chunk 1"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import blade_synth as bs  # noqa: E402
from paper_1802_06130_b200 import BladeMS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--frames", type=int, default=8)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--streams", type=int, default=2)
a = ap.parse_args()
cfg = bs.load_config(a.config)
cfg.N = a.frames
h = BladeMS.from_config(cfg)
x = torch.from_numpy(cfg.batch()).cuda()
out = torch.empty_like(x)


def call():
    if a.chunk:
        h.denoise_pipelined(x, out, chunk=a.chunk, n_streams=a.streams)
    else:
        h.denoise(x, out)


call()
torch.cuda.synchronize()
torch.cuda.profiler.start()
call()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", a)

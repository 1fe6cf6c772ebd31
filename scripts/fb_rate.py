"""Count pixels whose fp32 selector decision is uncertified (fallback rate) on a c3 frame:
compares the maps of two library builds (with / without the fp64 fallback)."""
import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import blade_synth as bs
cfg = bs.load_config("c3")
x = torch.from_numpy(cfg.batch(N=2)).cuda()
res = {}
for lib in sys.argv[1:]:
    os.environ["BLADE_MS_LIB"] = lib
    import importlib, paper_1802_06130_b200.blade_ms as bm
    bm._lib = None
    h = bm.BladeMS.from_config(cfg)
    res[lib] = [m.cpu().numpy() for m in h.selector(x)]
a, b = res[sys.argv[1]], res[sys.argv[2]]
for l in range(len(a)):
    d = (a[l] != b[l]).mean()
    print(f"level {l}: fraction of map entries differing {d:.3e}")

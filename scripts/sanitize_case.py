"""Small invocations of every kernel family for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python scripts/sanitize_case.py
c1 recipe at 96x136 (the smoke shape) through denoise (TMA stages, merged fix-up), selector,
a row band, halo-exchange bands, the chunked schedule; c4 recipe (phase-split 9x9 stage) and
c0 (single level), a ragged width (generic stage + row copy), c5 (4096 buckets, L2 bank)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import blade_synth as bs  # noqa: E402
from paper_1802_06130_b200 import BladeMS  # noqa: E402
from paper_1802_06130_b200.xband import denoise_bands_local  # noqa: E402


def run(name, H, W, N=1):
    cfg = bs.load_config(name)
    cfg.H, cfg.W, cfg.N = H, W, N
    h = BladeMS.from_config(cfg, device=0)
    x = torch.from_numpy(cfg.batch()).cuda()
    out = h.denoise(x)
    h.selector(x)
    if N == 1 and cfg.levels > 1:
        i0, ni = h.band_rows(H, H // 3, H // 3)
        h.denoise_rows(x[0, :, i0:i0 + ni].contiguous(), i0, H // 3, H // 3, H)
        try:
            denoise_bands_local(h, x, 2)
        except Exception as e:  # too thin for this footprint: reported, not a fault
            print(name, "xband skipped:", e)
    if N > 1:
        h.denoise_pipelined(x, chunk=1, n_streams=2)
    torch.cuda.synchronize()
    print(name, H, W, N, "ok", float(out.abs().max()))


run("c1", 96, 136)
run("c1", 96, 136, N=3)
run("c4", 160, 136)
run("c0", 64, 64)
run("c3", 70, 118)
run("c5", 64, 128)
print("sanitize case done")

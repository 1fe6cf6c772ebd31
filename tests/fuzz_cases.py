"""Random parity cases for the GPU suite and scripts/fuzz_parity.py: random shapes, pyramid depths,
footprint pairs, bucket layouts, windows and batch sizes, each checked with the GPU suite's rule
(tests/test_gpu_parity._full_parity: the CUDA path through the C ABI against the fp64 oracle)."""
from __future__ import annotations

import numpy as np


def draw(rng, big=False):
    """big: 0.4 - 1.6 MP frames (the streaming k_down, multi-tile TMA stages, merged fix-up launches)
    instead of the small-call paths."""
    levels = int(rng.choice([1, 2, 2, 3, 3, 4, 5]))
    nf = int(rng.choice([3, 5, 5, 7, 9]))
    nc = int(rng.choice([3, 5, 5, 7, 9])) if levels > 1 else 0
    if rng.random() < 0.5:  # shapes around tile and vector-width boundaries
        H = int(rng.choice([15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 257]))
        W = int(rng.choice([124, 127, 128, 129, 132, 255, 256, 257, 260, 383, 384, 388]))
    else:
        H, W = int(rng.integers(1, 300)), int(rng.integers(1, 420))
    N = int(rng.choice([1, 1, 2, 3]))
    if big:
        H = int(rng.integers(600, 1100))
        W = int(rng.choice([1024, 1280, 1284, 1000, 1002, 1337, 1536]))
        N = int(rng.choice([1, 2]))
    n_o = int(rng.choice([1, 4, 6, 8, 12, 16, 16, 16, 20]))
    n_s = int(rng.choice([1, 2, 3, 3, 4]))
    n_c = int(rng.choice([1, 2, 3, 3, 4]))
    win = int(rng.choice([1, 3, 5, 5, 5]))
    n_ph = 4 if (levels > 1 and rng.random() < 0.8) else 1
    # noise-free scenes are left out: half their pixels have an exactly zero structure tensor (every
    # feature on a quantisation boundary), so the near-boundary allowance of the rule decides them
    noise = str(rng.choice(["awgn", "signal"]))
    return dict(levels=levels, nf=nf, nc=nc, H=H, W=W, N=N, n_o=n_o, n_s=n_s, n_c=n_c, win=win,
                n_ph=n_ph, noise=noise)


def _T():
    from tests import test_gpu_parity as T
    return T


def run_case(p, seed):
    cfg = make_cfg(p, seed)
    _, _, worst = _T()._full_parity(cfg, cfg.batch(), label=str(p))
    return worst


def make_cfg(p, seed):
    """The blade_synth.Config of a drawn case (thresholds and window sigma from the case seed)."""
    rng = np.random.default_rng(seed)
    cfg = _T()._cfg_like("c1", p["H"], p["W"], p["N"], levels=p["levels"], fine_size=p["nf"],
                         coarse_size=p["nc"] if p["levels"] > 1 else 5, n_phases=p["n_ph"],
                         n_orient=p["n_o"], n_strength=p["n_s"], n_coherence=p["n_c"],
                         window_size=p["win"], window_sigma=float(rng.uniform(0.6, 2.0)), noise=p["noise"],
                         seed=int(seed))
    if p["noise"] == "signal":
        cfg.p0, cfg.p1 = 0.01, 0.0004
    nst = max(p["levels"] - 1, 1)
    cfg.strength_thresholds = [sorted(rng.uniform(0.02, 0.25, p["n_s"] - 1).tolist()) for _ in range(nst)]
    cfg.coherence_thresholds = [sorted(rng.uniform(0.02, 0.3, p["n_c"] - 1).tolist()) for _ in range(nst)]
    return cfg


def run_identity_case(p, seed, channels=1):
    """The bit-identity properties of the boundary on a drawn case, no oracle involved: per-frame
    calls, row bands (blade_ms_denoise_rows over a random partition), the chunked schedule
    (blade_ms_denoise_pipelined) and the host-buffer call all equal blade_ms_denoise bit for bit."""
    import torch
    rng = np.random.default_rng(seed + 17)
    cfg = make_cfg(p, seed)
    h = _T()._handle(cfg, cfg.taps(channels=channels) if channels != 1 else None)
    H, W, N = p["H"], p["W"], p["N"]
    xh = torch.from_numpy(cfg.batch()).pin_memory()
    x = xh.cuda()
    ref = h.denoise(x)
    n = int(rng.integers(0, N))
    assert torch.equal(h.denoise(x[n:n + 1].contiguous())[0], ref[n]), "per-frame call"
    # row bands of frame n over a random partition
    nb = int(rng.integers(1, min(5, H) + 1))
    cuts = sorted(set([0, H] + rng.integers(1, max(H, 2), nb - 1).clip(1, max(H - 1, 1)).tolist())) if H > 1 else [0, H]
    parts = []
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        i0, ni = h.band_rows(H, int(r0), int(r1 - r0))
        parts.append(h.denoise_rows(x[n, :, i0:i0 + ni].contiguous(), i0, int(r0), int(r1 - r0), H))
    assert torch.equal(torch.cat(parts, 1), ref[n]), f"row bands {cuts}"
    chunk, streams = int(rng.integers(1, N + 2)), int(rng.integers(1, 5))
    assert torch.equal(h.denoise_pipelined(x, chunk=chunk, n_streams=streams), ref), f"pipelined {chunk}/{streams}"
    outh = torch.empty_like(xh).pin_memory()
    h.denoise_host(xh, outh, torch.empty_like(ref), torch.empty_like(ref), h.workspace(N, H, W))
    assert torch.equal(outh, ref.cpu()), "host-buffer call"


def run_ycc_case(p, seed):
    """Per-channel (Y, Cb, Cr) banks (NEXT f1, with K > 256 the paper's own f1 x f2 layout) on a
    drawn case against oracle.denoise_ycc."""
    cfg = make_cfg(p, seed)
    _T()._ycc_parity(cfg, str(p))
    return True


def run_xband_case(p, seed, channels=1):
    """Halo-exchange row bands (NEXT f3 (b), the single-GPU form of the NCCL exchange) on frame 0 of
    a drawn case: G bands reproduce blade_ms_denoise bit for bit, or the layout refuses the split
    (BLADE_EUNSUPPORTED: a band would own fewer rows of some level than its neighbours need)."""
    import torch
    from paper_1802_06130_b200.blade_ms import BladeError
    from paper_1802_06130_b200.xband import denoise_bands_local
    rng = np.random.default_rng(seed + 29)
    p = dict(p, N=1)
    cfg = make_cfg(p, seed)
    h = _T()._handle(cfg, cfg.taps(channels=channels) if channels != 1 else None)
    x = torch.from_numpy(cfg.batch()).cuda()
    full = h.denoise(x)[0]
    G = int(rng.integers(2, 9))
    if G > p["H"]:  # more bands than rows: xband.band_edges refuses (ValueError)
        return False
    try:
        got = denoise_bands_local(h, x, G)
    except BladeError as e:
        assert e.status == 7, e  # refused cleanly
        return False
    torch.cuda.synchronize()
    assert torch.equal(got, full), f"xband G={G}"
    return True

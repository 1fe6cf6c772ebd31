"""GPU training (NEXT f4; Eqs. 7-8) against the numpy oracle (oracle/train.py):
the segmented fp64 SYRK accumulators, the host solve, and recovery of a known bank."""
from __future__ import annotations

import copy

import numpy as np
import pytest
import torch

import blade_synth as bs
import oracle
from oracle import train as tr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _wide_cfg():
    """K = 16 x 4 x 5 = 320 > 256 (uint16 maps, global-memory bank) with 7x7 / 5x5 pairs."""
    cfg = copy.deepcopy(bs.load_config("c5"))
    ts, tc = cfg.thresholds()
    cfg.n_strength, cfg.n_coherence = 4, 5
    cfg.strength_thresholds = ts[:, [3, 7, 11]].tolist()
    cfg.coherence_thresholds = tc[:, [2, 5, 8, 11]].tolist()
    return cfg


def _gpu_E_to_G_m(E, nt):
    """Mirror the upper 4 x 4-block triangle: G [n_seg, nt, nt], m [n_seg, nt]."""
    E = E.cpu().numpy()
    r = np.arange(nt)
    upper = (r[:, None] // 4) <= (r[None, :] // 4)
    G = np.where(upper[None], E[:, :nt, :nt], np.transpose(E[:, :nt, :nt], (0, 2, 1)))
    return G, E[:, :nt, nt]


@pytest.mark.parametrize("name,H,W,N", [("c1", 96, 128, 2), ("c0", 70, 90, 1), ("c2", 64, 96, 1),
                                        ("wide", 80, 112, 1)])
def test_train_accumulators_match_oracle(name, H, W, N):
    cfg = _wide_cfg() if name == "wide" else bs.load_config(name)
    cfg.H, cfg.W, cfg.N = H, W, N
    _train_parity(cfg)


# footprints with a Gram kernel: n_f^2 + n_c^2 <= 123 (7 + 9, 9 + 7, 9 + 9 are not built for training)
TRAIN_FOOTPRINTS = [(nf, nc) for nf in (1, 3, 5, 7, 9) for nc in (0, 1, 3, 5, 7, 9) if nf * nf + nc * nc <= 123]


def test_train_random_cases():
    """40 random cases (tests/fuzz_cases.py generator, footprints restricted to the built Gram
    kernels): accumulators, counts and the solve against oracle/train.py."""
    from tests.fuzz_cases import draw, make_cfg
    rng = np.random.default_rng(13)
    done = 0
    while done < 40:
        p = draw(rng)
        if p["H"] < 12 or p["W"] < 12:
            continue
        if p["n_o"] * p["n_s"] * p["n_c"] > 256:  # K > 256 training: 5+5, 7+5, 7+7, 7 only
            p["n_o"] = 16
        nf, nc = TRAIN_FOOTPRINTS[int(rng.integers(len(TRAIN_FOOTPRINTS)))]
        p.update(nf=nf, nc=nc, levels=1 if nc == 0 else max(p["levels"], 2))
        if nc == 0:
            p["n_ph"] = 1
        _train_parity(make_cfg(p, 13000 + done))
        done += 1


def _train_parity(cfg):
    from paper_1802_06130_b200 import BladeMS
    H, W, N = cfg.H, cfg.W, cfg.N
    z = cfg.batch()
    clean = np.stack([bs.scene(cfg.seed, i, H, W, cfg.n_grat, cfg.n_disk, "none", 0.0, 0.0)
                      for i in range(N)]).astype(np.float32)
    coarse = None
    if cfg.levels > 1:
        coarse = np.stack([oracle.pyramid(z[i], 2)[1] for i in range(N)]).astype(np.float32)
    h = BladeMS.from_config(cfg)
    nt, ntp, n_seg = h.train_layout()
    E, cnt = h.train_accumulators()
    zd = torch.from_numpy(z).cuda()
    h.train_accumulate(0, zd, torch.from_numpy(clean).cuda(),
                       None if coarse is None else torch.from_numpy(coarse).cuda(), E, cnt)
    maps = h.selector(zd)[0].cpu().numpy().astype(np.int64)
    torch.cuda.synchronize()
    G_gpu, m_gpu = _gpu_E_to_G_m(E, nt)
    Xs, ys, segs = [], [], []
    for i in range(N):
        X, y, sg = tr.samples(z[i], clean[i], None if coarse is None else coarse[i], maps[i],
                              cfg.n_phases, cfg.K, cfg.fine_size,
                              cfg.coarse_size if cfg.levels > 1 else 0)
        Xs.append(X)
        ys.append(y)
        segs.append(sg)
    G, m, c = tr.normal_equations(np.concatenate(Xs), np.concatenate(ys), np.concatenate(segs), n_seg)
    assert np.array_equal(cnt.cpu().numpy(), c // 3)  # pixels per segment (3 samples each)
    scale = np.abs(G).max()
    assert np.abs(G_gpu - G).max() <= 1e-12 * scale
    assert np.abs(m_gpu - m).max() <= 1e-12 * max(np.abs(m).max(), 1.0)
    # the host solve equals the oracle's solve
    H_gpu = h.train_solve(E, cnt, ridge=1e-3, min_count=4 * nt).reshape(n_seg, nt)
    H_ref = tr.solve(G, m, c // 3 * 0 + cnt.cpu().numpy(), cfg.fine_size, ridge=1e-3, min_count=4 * nt)
    np.testing.assert_allclose(H_gpu, H_ref, rtol=1e-4, atol=1e-5)


def test_train_recovers_a_known_bank():
    """Targets made by the oracle's stage (Eq. 9) with a known bank on white-noise inputs: the GPU
    accumulate + solve (ridge 0) returns that bank for every well-populated (phase, bucket)."""
    from paper_1802_06130_b200 import BladeMS
    cfg = bs.load_config("c1")
    rng = np.random.default_rng(3)
    H, W = 192, 256
    z = rng.uniform(0, 1, (1, 3, H, W)).astype(np.float32)
    coarse = oracle.pyramid(z[0], 2)[1].astype(np.float32)[None]
    h = BladeMS.from_config(cfg)
    zd = torch.from_numpy(z).cuda()
    maps = h.selector(zd)[0].cpu().numpy()[0].astype(np.int64)
    nt = 50
    bank = rng.normal(size=(cfg.n_phases, cfg.K, nt))
    u = oracle.stage(z[0], coarse[0], maps, bank, cfg.n_phases, 5, 5).astype(np.float32)[None]
    E, cnt = h.train_accumulators()
    h.train_accumulate(0, zd, torch.from_numpy(u).cuda(), torch.from_numpy(coarse).cuda(), E, cnt)
    taps = h.train_solve(E, cnt, ridge=0.0, min_count=3 * nt).reshape(-1, nt)
    ok = cnt.cpu().numpy() >= 3 * nt
    assert ok.sum() >= 50
    # the solved filters reproduce the targets of their segments (u was rounded to fp32, and the
    # patch Gram of a decimated noise image is ill-conditioned, so compare predictions, and the
    # coefficients only where the Gram is well-conditioned)
    X, y, seg = tr.samples(z[0], u[0], coarse[0], maps, cfg.n_phases, cfg.K, 5, 5)
    sel = ok[seg]
    pred = np.einsum("ij,ij->i", X[sel], taps[seg[sel]].astype(np.float64))
    assert np.abs(pred - y[sel]).max() < 1e-4 * np.abs(y).max()
    G, _, _ = tr.normal_equations(X, y, seg, cfg.n_phases * cfg.K)
    well = ok & np.array([np.linalg.cond(G[k]) < 1e5 if ok[k] else False for k in range(len(ok))])
    if well.any():
        np.testing.assert_allclose(taps[well], bank.reshape(-1, nt)[well], atol=1e-3)


def _psnr(a, b):
    return float(10 * np.log10(1.0 / np.mean((np.asarray(a, np.float64) - b) ** 2)))


@pytest.mark.parametrize("name,H,W,N", [("c1", 256, 256, 6), ("c0", 192, 192, 6), ("c3", 216, 384, 4)])
def test_train_multiscale_denoises_its_training_set(name, H, W, N):
    """SPEC.md:359 ("training then inference on the training images themselves -> PSNR strictly
    greater than noisy-input PSNR"): the coarse-to-fine schedule end to end."""
    from paper_1802_06130_b200 import BladeMS
    from paper_1802_06130_b200.train import train_multiscale
    cfg = copy.deepcopy(bs.load_config(name))
    cfg.H, cfg.W, cfg.N = H, W, N
    noisy = cfg.batch()
    clean = np.stack([bs.scene(cfg.seed, i, H, W, cfg.n_grat, cfg.n_disk, "none", 0.0, 0.0)
                      for i in range(N)]).astype(np.float32)
    nd, cd = torch.from_numpy(noisy).cuda(), torch.from_numpy(clean).cuda()
    taps, counts = train_multiscale(cfg, nd, cd, ridge=1e-3)
    assert np.isfinite(taps).all()
    out = BladeMS.from_config(cfg, taps=taps).denoise(nd).cpu().numpy()
    p_noisy, p_out = _psnr(noisy, clean), _psnr(out, clean)
    print(f"{name}: noisy {p_noisy:.2f} dB -> trained BLADE {p_out:.2f} dB")
    assert p_out > p_noisy + 3.0

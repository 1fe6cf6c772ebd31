"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs. Marked `gpu`; run on a B200 with `python -m pytest tests -m gpu`.

Tolerances: bucket maps bit-exact except near-boundary pixels (counted,
<= 1e-4 of a level); outputs within 1e-4 absolute outside the dependency cone of a bucket
mismatch; pyramid levels within 1e-5 (8-tap fp32 FIR with L1 gain 1.41); integer/exact cases
(delta banks, dyadic banks on constant images, band split, batch split) bit-exact.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import blade_synth as bs
import oracle
from tests.parity import OUT_ATOL, check_buckets, max_err_outside, taint_cone

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_06130_b200 import lib
    lib()  # fail loudly if the extension is missing


def _handle(cfg, taps=None, **kw):
    from paper_1802_06130_b200 import BladeMS
    return BladeMS.from_config(cfg, taps=taps, **kw)


def _cfg_like(name, H, W, N=1, **over):
    cfg = bs.load_config(name)
    cfg.H, cfg.W, cfg.N = H, W, N
    for k, v in over.items():
        setattr(cfg, k, v)
    return cfg


def _full_parity(cfg, x_np, taps=None, label="", pipelined=None, frames=None):
    """Run GPU denoise + selector on x_np [N,3,H,W]; compare with the oracle frame by frame.
    pipelined=(chunk, n_streams): the frame-chunked schedule (NEXT f3) instead of denoise().
    frames: the frames checked against the oracle (default all; the GPU runs the whole batch)."""
    taps = cfg.taps() if taps is None else taps
    h = _handle(cfg, taps)
    x = torch.from_numpy(x_np).cuda()
    out = h.denoise(x) if pipelined is None else h.denoise_pipelined(x, chunk=pipelined[0],
                                                                      n_streams=pipelined[1])
    maps = h.selector(x)
    lv = h.pyramid(x)
    torch.cuda.synchronize()
    sel = list(range(x_np.shape[0])) if frames is None else list(frames)
    pick = lambda t: np.stack([t[i].cpu().numpy() for i in sel])  # noqa: E731 (views: uint16 too)
    out = pick(out)
    maps = [pick(m) for m in maps]
    lv = [pick(t) for t in lv]
    x_np = x_np[sel]
    ts, tc = cfg.thresholds()
    stats_all = []
    worst = 0.0
    for n in range(x_np.shape[0]):
        parts = oracle.cascade_parts(cfg, x_np[n], taps)
        for l in range(1, cfg.levels):
            err = np.abs(lv[l - 1][n] - parts["levels"][l]).max()
            assert err < 1e-5, f"{label} frame {n} pyramid level {l}: {err}"
        mism = []
        for l in range(len(parts["buckets"])):
            m, st = check_buckets(maps[l][n], parts["buckets"][l], parts["features"][l],
                                  cfg.n_orient, ts[l], tc[l], f"{label} frame {n} level {l}")
            mism.append(m)
            stats_all.append(st)
        dims = [p.shape[1:] for p in parts["levels"]]
        tainted = taint_cone(mism, dims, cfg.coarse_size // 2) if cfg.levels > 1 else mism[0]
        err = max_err_outside(out[n], parts["outputs"][0], tainted)
        assert err <= OUT_ATOL, f"{label} frame {n}: max |gpu - oracle| = {err}"
        assert tainted.mean() < 0.01
        worst = max(worst, err)
    return out, stats_all, worst


# ------------------------------------------------------------------------- the five configs

def test_c0_single_level_full():
    cfg = bs.load_config("c0")
    _full_parity(cfg, cfg.batch(), label="c0")


def test_c1_full():
    cfg = bs.load_config("c1")
    _full_parity(cfg, cfg.batch(), label="c1")


def test_c3_frames_batched():
    """c3 recipe (1080p, 5x5 pairs, L=3) on 2 full frames batched in one call."""
    cfg = bs.load_config("c3")
    _full_parity(cfg, cfg.batch(N=2), label="c3")


@pytest.mark.parametrize("name,frames", [("c3", (0, 37, 63)), ("c5", (0, 7))])
def test_bench_launch_configuration_sampled_frames(name, frames):
    """The whole batch bench.py times (c3: 64 frames of 1080p in one launch; c5: 8 frames),
    the same launch configuration (band heights and grids depend on N), with sampled frames
    checked against the oracle one by one."""
    cfg = bs.load_config(name)
    _full_parity(cfg, cfg.batch(), label=f"{name} bench batch", frames=frames)


def test_c2_full_size():
    cfg = bs.load_config("c2")
    _full_parity(cfg, cfg.batch(), label="c2")


def test_c4_full_size():
    cfg = bs.load_config("c4")
    _full_parity(cfg, cfg.batch(), label="c4")


# ------------------------------------------------------------------------- ragged / edge shapes

@pytest.mark.parametrize("name,H,W,N", [("c1", 203, 333, 2), ("c1", 67, 129, 1), ("c2", 151, 97, 1),
                                        ("c4", 77, 190, 1), ("c0", 45, 131, 3), ("c3", 130, 259, 2),
                                        # widths 4 mod 16 / 8 mod 16: TMA stage with padded map rows
                                        ("c1", 96, 392, 2), ("c4", 90, 200, 1), ("c2", 70, 500, 1),
                                        ("c3", 64, 260, 2), ("c0", 40, 100, 2)])
def test_ragged_shapes(name, H, W, N):
    cfg = _cfg_like(name, H, W, N)
    _full_parity(cfg, cfg.batch(), label=f"{name}@{H}x{W}")


@pytest.mark.parametrize("name,H,W", [("c1", 1, 1), ("c1", 2, 3), ("c4", 3, 2), ("c0", 1, 5),
                                      ("c2", 5, 1), ("c4", 9, 17)])
def test_tiny_images_fold_wraps(name, H, W):
    """Tiny levels (1x1 .. 2x3) where a 9x9 footprint folds over several periods."""
    cfg = _cfg_like(name, H, W, 1)
    _full_parity(cfg, cfg.batch(), label=f"{name}@{H}x{W}")


def test_empty_batch_is_noop():
    cfg = bs.load_config("c1")
    h = _handle(cfg)
    x = torch.empty((0, 3, 16, 16), device="cuda")
    out = h.denoise(x)
    assert out.shape == x.shape


# ------------------------------------------------------------------------- exact cases

@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c4"])
def test_delta_bank_identity_bit_exact(name):
    cfg = _cfg_like(name, 97, 131, 2)
    nf = cfg.fine_size
    nt = nf * nf + (cfg.coarse_size ** 2 if cfg.levels > 1 else 0)
    taps = np.zeros((cfg.n_stages, 1, cfg.n_phases, cfg.K, nt), np.float32)
    taps[..., (nf // 2) * nf + nf // 2] = 1.0
    x = cfg.batch()
    out = _handle(cfg, taps).denoise(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(out, x)


@pytest.mark.parametrize("name", ["c0", "c1", "c4"])
def test_constant_image_dyadic_bank_exact(name, rng):
    """Filters summing to 1 leave a constant image unchanged (north star), exactly with dyadic
    taps (products and partial sums are representable in fp32)."""
    cfg = _cfg_like(name, 70, 90, 1)
    nf = cfg.fine_size
    nt = nf * nf + (cfg.coarse_size ** 2 if cfg.levels > 1 else 0)
    taps = rng.integers(-8, 9, size=(cfg.n_stages, 1, cfg.n_phases, cfg.K, nt)).astype(np.float64)
    taps[..., 0] += 64 - taps.sum(-1)
    taps = (taps / 64).astype(np.float32)
    x = np.full((1, 3, 70, 90), 0.625, np.float32)
    out = _handle(cfg, taps).denoise(torch.from_numpy(x).cuda()).cpu().numpy()
    assert (out == 0.625).all()
    assert (oracle.denoise_config(cfg, x[0], taps) == 0.625).all()


def test_batch_equals_per_frame_bit_exact():
    cfg = _cfg_like("c1", 150, 170, 3)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    full = h.denoise(x)
    for n in range(3):
        one = h.denoise(x[n:n + 1].contiguous())
        assert torch.equal(one[0], full[n])


# ------------------------------------------------------------------------- NEXT f3: chunked schedule

@pytest.mark.parametrize("name,H,W,N,chunk,streams", [("c3", 256, 384, 7, 2, 2), ("c3", 120, 200, 5, 1, 4),
                                                      ("c1", 203, 333, 3, 2, 3), ("c4", 130, 190, 2, 1, 2),
                                                      ("c0", 64, 64, 5, 3, 1), ("c2", 97, 131, 4, 8, 2)])
def test_pipelined_equals_denoise_bit_exact(name, H, W, N, chunk, streams):
    """blade_ms_denoise_pipelined: chunks of frames on internal streams give the batched output
    bit-exactly (ragged last chunk, more streams than chunks, chunk > N)."""
    cfg = _cfg_like(name, H, W, N)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    ref = h.denoise(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = h.denoise_pipelined(x, chunk=chunk, n_streams=streams, stream=s)
    s.synchronize()
    assert torch.equal(out, ref)


def test_pipelined_oracle_parity_c3_frames():
    cfg = bs.load_config("c3")
    _full_parity(cfg, cfg.batch(N=3), label="c3 pipelined", pipelined=(1, 2))


def test_pipelined_graph_capture_and_errors():
    """The fork / join are event waits: the schedule captures into a CUDA graph and replays
    bit-exactly; bad chunk / stream counts and short workspaces are rejected."""
    from paper_1802_06130_b200.blade_ms import BladeError
    cfg = _cfg_like("c3", 96, 160, 6)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    ref = h.denoise(x)
    out = torch.empty_like(x)
    ws = torch.empty(h.pipeline_workspace_size(2, 3, 96, 160), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h.denoise_pipelined(x, out, chunk=2, n_streams=3, workspace=ws, stream=s)  # warm-up
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    out.zero_()
    with torch.cuda.graph(g, stream=s):
        h.denoise_pipelined(x, out, chunk=2, n_streams=3, workspace=ws, stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    for kw, code in [(dict(chunk=0), 1), (dict(n_streams=5), 1), (dict(n_streams=0), 1)]:
        with pytest.raises(BladeError) as ei:
            h.denoise_pipelined(x, out, workspace=ws, **kw)
        assert ei.value.status == code
    with pytest.raises(BladeError) as ei:
        h.denoise_pipelined(x, out, chunk=2, n_streams=3, workspace=ws[:ws.numel() // 2])
    assert ei.value.status == 3


@pytest.mark.parametrize("name,H,W,bands", [("c4", 700, 300, 4), ("c2", 333, 260, 3),
                                            ("c1", 257, 100, 5)])
def test_row_bands_bit_identical(name, H, W, bands):
    """blade_ms_denoise_rows: concatenated band outputs equal the full-image output bit-exactly
    (BASELINE.json configs[4] split into row bands with a halo covering the pyramid)."""
    cfg = _cfg_like(name, H, W, 1)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    full = h.denoise(x)[0]
    edges = np.linspace(0, H, bands + 1).astype(int)
    parts = []
    for r0, r1 in zip(edges[:-1], edges[1:]):
        i0, ni = h.band_rows(H, int(r0), int(r1 - r0))
        band_in = x[0, :, i0:i0 + ni].contiguous()
        parts.append(h.denoise_rows(band_in, i0, int(r0), int(r1 - r0), H))
    assert torch.equal(torch.cat(parts, 1), full)


def test_denoise_host_equals_device():
    cfg = _cfg_like("c3", 120, 200, 5)
    h = _handle(cfg)
    xh = torch.from_numpy(cfg.batch()).pin_memory()
    ref = h.denoise(xh.cuda())
    outh = torch.empty_like(xh).pin_memory()
    d_in, d_out = torch.empty_like(ref), torch.empty_like(ref)
    ws = h.workspace(*cfg.batch().shape[:1], 120, 200)
    h.denoise_host(xh, outh, d_in, d_out, ws)
    assert torch.equal(outh, ref.cpu())


@pytest.mark.parametrize("name,H,W", [("c4", 2100, 2000), ("c2", 2048, 2052), ("c1", 2049, 2048), ("c3", 2050, 2046)])
def test_denoise_host_single_frame_bands_equal_device(name, H, W):
    """blade_ms_denoise_host on ONE large frame pipelines row bands (H2D of band i+1, compute of
    band i, D2H of band i-1; each band computes its rows from its input dependency cone): the
    output equals the device-resident whole-frame call bit for bit; repeated calls on the handle
    (its cached copy streams and events) too."""
    cfg = _cfg_like(name, H, W, 1)
    h = _handle(cfg)
    xh = torch.from_numpy(cfg.batch()).pin_memory()
    ref = h.denoise(xh.cuda()).cpu()
    outh = torch.empty_like(xh).pin_memory()
    d_in, d_out = torch.empty_like(xh, device="cuda"), torch.empty_like(xh, device="cuda")
    ws = h.workspace(1, H, W)
    for _ in range(2):
        outh.zero_()
        h.denoise_host(xh, outh, d_in, d_out, ws)
        assert torch.equal(outh, ref)


def test_clamp_output_flag():
    cfg = _cfg_like("c1", 64, 64, 1)
    x = torch.from_numpy(cfg.batch()).cuda()
    raw = _handle(cfg).denoise(x)
    cl = _handle(cfg, clamp_output=True).denoise(x)
    assert torch.equal(cl, raw.clamp(0, 1))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_bands_equal_full_image(world):
    """The multi-GPU band split of bench.py (paper_1802_06130_b200.shard, configs[4] recipe at a
    reduced size), run band by band on one device: bit-identical to the whole-image call."""
    from paper_1802_06130_b200.shard import shard_for
    cfg = _cfg_like("c4", 900, 260, 1)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    full = h.denoise(x)[0]
    parts = []
    for r in range(world):
        s = shard_for(cfg, r, world)
        assert s.mode == "bands"
        band_in = x[0, :, s.in_row0:s.in_row0 + s.in_rows].contiguous()
        parts.append(h.denoise_rows(band_in, s.in_row0, s.out_row0, s.out_rows, cfg.H))
    assert torch.equal(torch.cat(parts, 1), full)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_fp32_selector_fallback_is_rare(name):
    """The fp32 selector recomputes uncertified pixels in fp64 (DESIGN.md §6 H1); on the configs'
    scenes that must stay rare (it is a correctness net, not the path)."""
    cfg = bs.load_config(name)
    N = min(cfg.N, 2)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch(N=N)).cuda()
    ws = h.workspace(N, cfg.H, cfg.W)
    h.selector(x, workspace=ws)
    counts = h.fallback_count(N, cfg.H, cfg.W, ws)
    dims = h.level_dims(cfg.H, cfg.W)
    rates = [c / (N * dims[l][0] * dims[l][1]) for l, c in enumerate(counts)]
    print(f"{name}: fallback counts {counts} rates {rates}")
    assert all(r < 2e-3 for r in rates), rates


@pytest.mark.parametrize("name,H,W,N", [("c0", 64, 64, 1), ("c1", 67, 129, 2), ("c3", 130, 259, 2),
                                        ("c4", 77, 190, 1), ("c2", 5, 1, 1)])
def test_no_writes_outside_buffers(name, H, W, N):
    """Canary bytes after the output and after the workspace stay untouched (out-of-bounds writes
    into caller memory are otherwise silent)."""
    cfg = _cfg_like(name, H, W, N)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    n_out = x.numel()
    out_buf = torch.full((n_out + 4096,), 7.25, dtype=torch.float32, device="cuda")
    out = out_buf[:n_out].view_as(x)
    ws_n = h.workspace_size(N, H, W)
    ws_buf = torch.full((ws_n + 65536,), 0xA5, dtype=torch.uint8, device="cuda")
    h.denoise(x, out, ws_buf[:ws_n])
    torch.cuda.synchronize()
    assert bool((out_buf[n_out:] == 7.25).all())
    assert bool((ws_buf[ws_n:] == 0xA5).all())
    maps = h.selector(x, workspace=ws_buf[:ws_n])
    torch.cuda.synchronize()
    assert bool((ws_buf[ws_n:] == 0xA5).all())


# ------------------------------------------------------------------------- per-channel YCbCr (f1)

@pytest.mark.parametrize("name,H,W,N", [("c0", 64, 64, 1), ("c1", 203, 333, 2), ("c2", 151, 97, 1),
                                        ("c4", 77, 190, 1), ("c3", 256, 384, 1),
                                        # widths % 16 == 0: the TMA phase-split kernel (k_stage_ph)
                                        ("c1", 160, 256, 2), ("c2", 128, 192, 1), ("c4", 96, 256, 1)])
def test_ycc_channel_banks_parity(name, H, W, N):
    """NEXT f1: per-channel Y/Cb/Cr banks with the shared RGB selector against the oracle's
    denoise_ycc (same parity rule: outputs within 1e-4 outside the cone of bucket mismatches)."""
    _ycc_parity(_cfg_like(name, H, W, N), name)


def _ycc_parity(cfg, name):
    N = cfg.N
    taps = cfg.taps(channels=3)
    h = _handle(cfg, taps)
    x_np = cfg.batch()
    x = torch.from_numpy(x_np).cuda()
    out = h.denoise(x).cpu().numpy()
    maps = [m.cpu().numpy() for m in h.selector(x)]
    ts, tc = cfg.thresholds()
    for n in range(N):
        parts = oracle.cascade_parts(cfg, x_np[n], taps[:, :1])
        ref = oracle.denoise_ycc(x_np[n], cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.n_phases,
                                 cfg.n_orient, cfg.n_strength, cfg.n_coherence, ts, tc, taps,
                                 cfg.window_size, cfg.window_sigma)
        mism = [check_buckets(maps[l][n], parts["buckets"][l], parts["features"][l], cfg.n_orient,
                              ts[l], tc[l], f"{name} ycc level {l}")[0]
                for l in range(len(parts["buckets"]))]
        dims = [p.shape[1:] for p in parts["levels"]]
        tainted = taint_cone(mism, dims, cfg.coarse_size // 2) if cfg.levels > 1 else mism[0]
        err = max_err_outside(out[n], ref, tainted)
        assert err <= OUT_ATOL, f"{name} ycc frame {n}: max |gpu - oracle| = {err}"


@pytest.mark.parametrize("H,W,N", [(256, 384, 2), (130, 200, 1), (9, 17, 1)])
def test_c5_per_channel_banks_parity(H, W, N):
    """The paper's own layout: 16 x 16 x 16 buckets (uint16 maps, global-memory bank) WITH one
    bank per Y / Cb / Cr channel (f1 x f2), against oracle.denoise_ycc."""
    _ycc_parity(_cfg_like("c5", H, W, N), "c5 ycc")


def test_ycc_equal_banks_match_rgb_path():
    cfg = _cfg_like("c1", 130, 200, 2)
    t1 = cfg.taps()
    x = torch.from_numpy(cfg.batch()).cuda()
    rgb = _handle(cfg, t1).denoise(x)
    ycc = _handle(cfg, np.repeat(t1, 3, axis=1)).denoise(x)
    assert float((rgb - ycc).abs().max()) < 1e-5


def test_ycc_clamp_applies_after_conversion():
    cfg = _cfg_like("c1", 64, 64, 1)
    taps = cfg.taps(channels=3)
    x = torch.from_numpy(cfg.batch()).cuda()
    raw = _handle(cfg, taps).denoise(x)
    cl = _handle(cfg, taps, clamp_output=True).denoise(x)
    assert torch.equal(cl, raw.clamp(0, 1))


def test_runtime_argument_errors_launch_nothing():
    """Every call-time argument error is reported before any launch (ABI contract): the output
    buffer keeps its canary values."""
    from paper_1802_06130_b200 import BladeError
    cfg = _cfg_like("c1", 64, 96, 1)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    out = torch.full_like(x, 3.5)
    ws_n = h.workspace_size(1, 64, 96)
    with pytest.raises(BladeError, match="ESHAPE"):  # workspace too small
        h.denoise(x, out, torch.empty(ws_n - 256, dtype=torch.uint8, device="cuda"))
    with pytest.raises(BladeError, match="EINVAL"):  # out overlaps in
        h.denoise(x, x)
    from paper_1802_06130_b200 import lib
    xh = x.cpu()
    ws = h.workspace(1, 64, 96)
    rc = lib().blade_ms_denoise(h._h, xh.data_ptr(), out.data_ptr(), 1, 64, 96, ws.data_ptr(),
                                ws.numel(), None)
    assert rc == 4, lib().blade_ms_last_error()  # EDEVICE: host pointer
    with pytest.raises(BladeError, match="ESHAPE"):  # band that does not cover the cone
        i0, ni = h.band_rows(64, 20, 10)
        h.denoise_rows(x[0, :, i0 + 2:i0 + ni].contiguous(), i0 + 2, 20, 10, 64)
    torch.cuda.synchronize()
    assert bool((out == 3.5).all())


# ------------------------------------------------------------------------- paper-scale buckets (f2)

@pytest.mark.parametrize("H,W,N", [(1080, 1920, 1), (256, 384, 2), (130, 200, 1), (9, 17, 1)])
def test_c5_paper_bucket_layout_parity(H, W, N):
    """NEXT f2: the paper's 16 x 16 x 16 = 4096 buckets with 7x7 / 5x5 pairs:
    uint16 maps, bank read from global memory; same parity rule."""
    cfg = _cfg_like("c5", H, W, N)
    assert cfg.K == 4096
    out, stats, worst = _full_parity(cfg, cfg.batch(), label=f"c5@{H}x{W}")
    h = _handle(cfg)
    assert h.map_dtype == torch.uint16


# ------------------------------------------------------- small-call down pass (k_down_tile)

_TILE_CASES = [("c1", 512, 512, 1), ("c1", 67, 132, 2), ("c0", 64, 64, 1), ("c0", 61, 100, 3),
               ("c2", 130, 200, 1), ("c4", 203, 332, 1), ("c3", 136, 240, 2), ("c1", 9, 16, 1),
               ("c1", 1024, 1024, 1)]


def _tile_case_outputs(path):
    outs = {}
    for name, H, W, N in _TILE_CASES:
        cfg = _cfg_like(name, H, W, N)
        h = _handle(cfg)
        outs[f"{name}_{H}x{W}x{N}"] = h.denoise(torch.from_numpy(cfg.batch()).cuda()).cpu().numpy()
        outs[f"{name}_{H}x{W}x{N}_launches"] = np.array(h.launch_count(N, H, W))
    np.savez(path, **outs)


def test_down_tile_bit_identical(tmp_path):
    """Small calls run the down pass as k_down_tile (2-D tiles, fp64 fixes inline) instead of
    k_down: the same arithmetic in the same order, so the denoised outputs are bit-identical to the
    streaming kernel's (run in a child process with BLADE_DOWN_TILE=0), with no fix-up launch."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    ref = tmp_path / "stream.npz"
    code = ("import sys; sys.path.insert(0, %r); from tests.test_gpu_parity import _tile_case_outputs; "
            "_tile_case_outputs(%r)" % (str(root), str(ref)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, "BLADE_DOWN_TILE": "0"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    mine = tmp_path / "tile.npz"
    env_tile = os.environ.get("BLADE_DOWN_TILE")
    _tile_case_outputs(mine)
    a, b = np.load(ref), np.load(mine)
    for name, H, W, N in _TILE_CASES:
        k = f"{name}_{H}x{W}x{N}"
        assert np.array_equal(a[k], b[k]), (k, np.abs(a[k] - b[k]).max())
        if env_tile is None and N * H * W <= (3 << 18):  # default threshold: a small call
            L = _cfg_like(name, H, W, N).levels
            nsel = 1 if L == 1 else L - 1
            assert int(b[k + "_launches"]) == 2 * nsel + (1 if W % 4 else 0), (k, int(b[k + "_launches"]))


def test_many_tiny_frames_grid_limits():
    """65,535 frames (the ABI's per-call maximum) of 2 x 4 px: a small call whose frames fill
    k_down_tile's gridDim.z to its limit; equal bit for bit to the same frames in two calls."""
    n = 65535
    cfg = _cfg_like("c1", 2, 4, n)
    h = _handle(cfg)
    x = torch.rand(n, 3, 2, 4, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    full = h.denoise(x)
    halves = torch.cat([h.denoise(x[:n // 2].contiguous()), h.denoise(x[n // 2:].contiguous())])
    assert torch.equal(full, halves)


# ------------------------------------------------------------------------- forced kernel variants

@pytest.mark.parametrize("env", [{"BLADE_TMA_RY": "4"}, {"BLADE_TMA_RY": "2"}, {"BLADE_PDL": "0"},
                                 {"BLADE_FUSE_SEL": "1", "BLADE_TMA_RY": "4"}, {"BLADE_CARVEOUT": "100"},
                                 {"BLADE_INLINE_FIX": "0"}, {"BLADE_INLINE_FIX": "100000000"}, {"BLADE_P2": "0"},
                                 {"BLADE_DOWN_TILE": "0"}, {"BLADE_DOWN_TILE": "100000000"}])
def test_forced_variants_subprocess(env):
    """The library picks kernel variants by level size (4- vs 2-row TMA stage threads) and
    launches with programmatic dependent launch; the knobs are read once per process, so the
    ragged / exact parity cases are re-run in a child process with each choice forced."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "pytest", str(root / "tests" / "test_gpu_parity.py"), "-q", "-x",
           "-p", "no:cacheprovider", "-k",
           "(ragged_shapes or c1_full or delta_bank or c3_frames_batched or forced_selector_every_pixel or "
           "xband_bands or repeat_runs or constant_image or deep_pyramid or forced_selector_ragged) and "
           "not forced_variants"]
    r = subprocess.run(cmd, cwd=root, env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_stage_kernel_selection():
    """The variant each level runs (blade_ms_stage_kernel): the bench's c3 level 0 takes the
    4-row TMA kernel, and so does its 7.5-tile-wide level 1; a small call the 2-row one; 7x7 pairs
    the row-parity kernel (two phases per CTA), 9x9 pairs the phase-split
    kernel; every width takes TMA (levels >= 1 live in the workspace with padded rows; a level-0
    width that is not a multiple of 4 reads the 16-B-row copy of the input k_down writes)."""
    c3 = bs.load_config("c3")
    h = _handle(c3)
    assert h.stage_kernel(64, 1080, 1920, 0) == ("k_stage_tma", 4)
    assert h.stage_kernel(64, 1080, 1920, 1) == ("k_stage_tma", 4)
    assert h.stage_kernel(1, 512, 512, 0) == ("k_stage_tma", 2)
    assert h.stage_kernel(1, 130, 259, 0) == ("k_stage_tma", 2)  # reads k_down's 16-B-row input copy
    assert h.stage_kernel(1, 130, 259, 1) == ("k_stage_tma", 2)  # workspace levels are padded
    assert h.stage_kernel(1, 130, 392, 0) == ("k_stage_tma", 2)  # W % 16 == 8: padded map rows
    assert h.stage_kernel(1, 130, 260, 0) == ("k_stage_tma", 2)  # level-1 width 130, padded to 132
    assert _handle(bs.load_config("c2")).stage_kernel(1, 3000, 4000, 0)[0] == "k_stage_p2"
    assert _handle(bs.load_config("c4")).stage_kernel(1, 6000, 8000, 0)[0] == "k_stage_ph"
    from paper_1802_06130_b200.blade_ms import BladeError
    with pytest.raises(BladeError):
        h.stage_kernel(1, 64, 64, 2)


# ------------------------------------------------------------------------- selector / layout variants

_TS1, _TC1 = [0.12769653, 0.15104799], [0.06869324, 0.12480995]  # c1 stage-0 tertiles (fp32)
LAYOUTS = {
    # non-FAST bucket layouts: quadrant edges with 1 / 2 interior edges, the atan2 path (n_o % 4 != 0)
    "8x4x2": dict(n_orient=8, n_strength=4, n_coherence=2, ts=[0.06, 0.11, 0.15], tc=[0.1]),
    "12x2x3": dict(n_orient=12, n_strength=2, n_coherence=3, ts=[0.12], tc=_TC1),
    "6x3x3_atan2": dict(n_orient=6, n_strength=3, n_coherence=3, ts=_TS1, tc=_TC1),
    "1x1x1": dict(n_orient=1, n_strength=1, n_coherence=1, ts=[], tc=[]),       # one filter
    "16x4x4_K256": dict(n_orient=16, n_strength=4, n_coherence=4, ts=[0.06, 0.11, 0.15],
                        tc=[0.05, 0.09, 0.14]),                                   # largest uint8 K
    "20x4x4_K320": dict(n_orient=20, n_strength=4, n_coherence=4, ts=[0.06, 0.11, 0.15],
                        tc=[0.05, 0.09, 0.14]),                                   # uint16 maps
    "nonpos_thresholds": dict(ts=[0.0, 0.12], tc=[-0.5, 0.1]),                  # t <= 0 [R6]
    "window3": dict(window_size=3, window_sigma=0.8),
    "window1": dict(window_size=1, window_sigma=1.0),
    "one_phase": dict(n_phases=1),                                               # SPEC reading
}


@pytest.mark.parametrize("shape", [(2, 160, 256), (1, 97, 131)])
@pytest.mark.parametrize("name", list(LAYOUTS))
def test_selector_and_layout_variants(name, shape):
    """Every parameter the ABI accepts besides the configs' own: bucket layouts that take the
    generic (binary-search / quadrant-edge / atan2) selector paths, K = 1 and the uint8 / uint16
    limits, non-positive thresholds, 3x3 and 1x1 structure-tensor windows, phase-free banks; on a
    TMA-eligible and a ragged (generic stage kernel) shape, against the oracle."""
    N, H, W = shape
    over = dict(LAYOUTS[name])
    ts, tc = over.pop("ts", None), over.pop("tc", None)
    cfg = _cfg_like("c1", H, W, N, **over)
    if ts is not None:
        cfg.strength_thresholds = [list(ts)] * cfg.n_stages
        cfg.coherence_thresholds = [list(tc)] * cfg.n_stages
    _full_parity(cfg, cfg.batch(), label=f"{name}@{H}x{W}")


@pytest.mark.parametrize("shape", [(2, 130, 256), (1, 77, 190)])
@pytest.mark.parametrize("levels,nf,nc", [(2, 3, 3), (2, 5, 3), (3, 7, 5), (2, 9, 7), (1, 3, 0), (1, 5, 0),
                                          (1, 9, 0), (4, 3, 3)])
def test_footprint_variants(levels, nf, nc, shape):
    """Every built footprint pair / single-level size beyond the configs' (5+5, 7+7, 9+9, 7 and the
    wide 7+5), through the TMA (or phase-split) and generic stage kernels, against the oracle."""
    N, H, W = shape
    cfg = _cfg_like("c1", H, W, N, levels=levels, fine_size=nf, coarse_size=nc,
                    n_phases=4 if levels > 1 else 1)
    nst = max(levels - 1, 1)
    cfg.strength_thresholds = [list(_TS1)] * nst
    cfg.coherence_thresholds = [list(_TC1)] * nst
    _full_parity(cfg, cfg.batch(), label=f"L{levels} {nf}+{nc}@{H}x{W}")


_ALL_PAIRS = [(nf, nc) for nf in (1, 3, 5, 7, 9) for nc in (1, 3, 5, 7, 9)]


@pytest.mark.parametrize("nf,nc", _ALL_PAIRS)
def test_every_footprint_pair_of_the_abi_range(nf, nc):
    """Every fine / coarse pair the ABI accepts (odd sizes 1..9 each): the pairs without a
    specialised TMA kernel run the generic stage kernel; a ragged two-frame shape, L = 3."""
    cfg = _cfg_like("c1", 77, 190, 2, levels=3, fine_size=nf, coarse_size=nc)
    cfg.strength_thresholds = [list(_TS1)] * 2
    cfg.coherence_thresholds = [list(_TC1)] * 2
    _full_parity(cfg, cfg.batch(), label=f"{nf}+{nc}")


@pytest.mark.parametrize("nf,nc,H,W", [(5, 9, 129, 132), (9, 9, 64, 256), (7, 9, 33, 77)])
def test_big_bank_read_from_global_memory(nf, nc, H, W):
    """K = 256 (the uint8 limit) with footprints whose two-phase bank (219 - 333 KB) fits no CTA's
    shared memory: the stage reads the bank from global memory (uint8 maps), same parity rule."""
    over = dict(LAYOUTS["16x4x4_K256"])
    ts, tc = over.pop("ts"), over.pop("tc")
    cfg = _cfg_like("c1", H, W, 2, levels=3, fine_size=nf, coarse_size=nc, **over)
    cfg.strength_thresholds = [list(ts)] * 2
    cfg.coherence_thresholds = [list(tc)] * 2
    _full_parity(cfg, cfg.batch(), label=f"K256 {nf}+{nc}@{H}x{W}")


@pytest.mark.parametrize("nf,nc", [(5, 7), (3, 9), (9, 1)])
def test_new_footprint_pairs_ycc_and_wide(nf, nc):
    """The added pairs through the per-channel (f1) and K > 256 (f2) generic kernels."""
    cfg = _cfg_like("c1", 67, 129, 1, levels=2, fine_size=nf, coarse_size=nc)
    cfg.strength_thresholds = [list(_TS1)]
    cfg.coherence_thresholds = [list(_TC1)]
    _ycc_parity(cfg, f"{nf}+{nc}")
    over = dict(LAYOUTS["20x4x4_K320"])
    tsw, tcw = over.pop("ts"), over.pop("tc")
    cfgw = _cfg_like("c1", 67, 129, 1, levels=2, fine_size=nf, coarse_size=nc, **over)
    cfgw.strength_thresholds = [list(tsw)]
    cfgw.coherence_thresholds = [list(tcw)]
    _full_parity(cfgw, cfgw.batch(), label=f"K320 {nf}+{nc}")


def test_random_parity_cases():
    """40 random cases (tests/fuzz_cases.py: shapes around tile and vector boundaries, depths 1-5,
    every footprint pair, bucket layouts up to K = 320, windows 1 / 3 / 5, 1 or 4 phases) under the
    suite's parity rule; scripts/fuzz_parity.py runs longer sweeps of the same generator."""
    from tests.fuzz_cases import draw, run_case
    rng = np.random.default_rng(7)
    for i in range(40):
        p = draw(rng)
        run_case(p, 7000 + i)


def test_concurrent_calls_on_one_handle():
    """include/blade_ms.h "Thread safety": concurrent calls on ONE handle with distinct workspaces,
    outputs and streams are safe - four host threads mix blade_ms_denoise, _denoise_pipelined (the
    handle's shared internal streams, serialised by its mutex) and _denoise_host for several rounds
    on different inputs; every output equals the same call made alone, bit for bit."""
    import threading
    cfg = _cfg_like("c3", 120, 200, 4)
    h = _handle(cfg)
    T, R = 4, 6
    xs = [torch.from_numpy(cfg.batch(frame0=4 * t)).cuda() for t in range(T)]
    refs = [h.denoise(x).clone() for x in xs]
    torch.cuda.synchronize()
    errs = []

    def work(t):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            x, ref = xs[t], refs[t]
            xh = x.cpu().pin_memory()
            outh = torch.empty_like(xh).pin_memory()
            d_in, d_out = torch.empty_like(x), torch.empty_like(x)
            ws = h.workspace(4, 120, 200)
            out = torch.empty_like(x)
            for r in range(R):
                kind = (t + r) % 3
                out.zero_()
                if kind == 0:
                    h.denoise(x, out, workspace=ws, stream=st)
                elif kind == 1:
                    h.denoise_pipelined(x, out, chunk=1 + (r % 2), n_streams=2 + (t % 2), stream=st)
                else:
                    h.denoise_host(xh, outh, d_in, d_out, ws, stream=st)
                    out.copy_(outh)
                st.synchronize()
                torch.cuda.synchronize()
                if not torch.equal(out, ref):
                    errs.append((t, r, kind, float((out - ref).abs().max())))
        except Exception as e:  # noqa: BLE001
            errs.append((t, repr(e)))

    th = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    for q in th:
        q.start()
    for q in th:
        q.join()
    assert not errs, errs


def test_random_identity_cases():
    """25 random cases of the same generator through the bit-identity properties of the boundary
    (per-frame calls, a random row-band partition, the chunked schedule, the host-buffer call: all
    equal blade_ms_denoise bit for bit)."""
    from tests.fuzz_cases import draw, run_identity_case
    rng = np.random.default_rng(11)
    for i in range(25):
        run_identity_case(draw(rng), 11000 + i)


@pytest.mark.parametrize("name", ["c1", "c5"])
def test_fixup_list_overflow_recomputes_everything(name):
    """A frame whose top half is an exact 45-degree ramp puts every pixel there on an orientation
    bin edge, so the fp32 certificate rejects far more pixels than the fix-up list holds (1/64 of
    the level): the fix-up kernel must then recompute the WHOLE map in fp64. Check: the overflow
    happened; on the natural bottom half the map obeys the parity rule; on the ramp every bucket
    equals the oracle's or differs by one orientation bin (the decision sits exactly on an edge)."""
    cfg = _cfg_like(name, 256, 384, 1)
    x = cfg.batch()
    H, W = 256, 384
    yy, xx = np.mgrid[0:H // 2, 0:W]
    x[0, :, :H // 2] = (0.25 + (xx + yy) * 2.0 ** -10).astype(np.float32)  # exact in fp32
    h = _handle(cfg)
    xt = torch.from_numpy(x).cuda()
    ws = h.workspace(1, H, W)
    maps = h.selector(xt, workspace=ws)
    counts = h.fallback_count(1, H, W, ws)
    assert counts[0] > H * W // 64, counts  # the list overflowed at level 0
    gpu = maps[0][0].cpu().numpy().astype(np.int64)
    ts, tc = cfg.thresholds()
    ob, feats = oracle.selector(x[0].astype(np.float64), cfg.n_orient, cfg.n_strength, cfg.n_coherence,
                                ts[0], tc[0], cfg.window_size, cfg.window_sigma, features=True)
    lo = H // 2 + 4  # rows whose 5x5 window and gradients see only the natural half
    check_buckets(gpu[lo:], ob[lo:], tuple(f[lo:] for f in feats), cfg.n_orient, ts[0], tc[0],
                  f"{name} natural half after overflow")
    per_o = cfg.n_strength * cfg.n_coherence
    top = slice(2, H // 2 - 3)  # the pure ramp (away from the image border fold and the seam)
    og, oo = gpu[top] // per_o, ob[top] // per_o
    d = (og - oo) % cfg.n_orient
    assert np.isin(d, [0, 1, cfg.n_orient - 1]).all()
    assert (gpu[top] % per_o == ob[top] % per_o).all()  # strength / coherence bins agree


# ------------------------------------------------------------------ forced-selector parity mode

def _forced_parity(cfg, x_np, taps=None, label="", frames=None):
    """SURVEY.md §8(c) parity rule 2(a): the oracle's stages (Eq. 9, fp64) consume the GPU's OWN
    bucket maps, so the comparison covers every output pixel, including the dependency cones of
    near-boundary bucket mismatches that the free mode excludes. Every pixel within 1e-4."""
    taps = cfg.taps() if taps is None else taps
    t4 = taps[:, 0] if taps.ndim == 5 else taps
    h = _handle(cfg, taps)
    x = torch.from_numpy(x_np).cuda()
    out = h.denoise(x)
    maps = h.selector(x)
    torch.cuda.synchronize()
    sel = list(range(x_np.shape[0])) if frames is None else list(frames)
    L = cfg.levels
    worst = 0.0
    for n in sel:
        lv = oracle.pyramid(x_np[n], L)
        gm = [maps[l][n].cpu().numpy().astype(np.int32) for l in range(len(maps))]
        if L == 1:
            ref = oracle.stage(lv[0], None, gm[0], t4[0], cfg.n_phases, cfg.fine_size, 0)
        else:
            ref = lv[L - 1]
            for l in range(L - 2, -1, -1):
                ref = oracle.stage(lv[l], ref, gm[l], t4[l], cfg.n_phases, cfg.fine_size, cfg.coarse_size)
        err = float(np.abs(out[n].cpu().numpy().astype(np.float64) - ref).max())
        assert err <= OUT_ATOL, f"{label} frame {n}: forced-selector max |gpu - oracle| = {err}"
        worst = max(worst, err)
    return worst


@pytest.mark.parametrize("name,N,frames", [("c0", 1, None), ("c1", 1, None), ("c3", 2, None), ("c2", 1, None),
                                           ("c4", 1, None), ("c5", 2, None)])
def test_forced_selector_every_pixel(name, N, frames):
    """Forced-selector mode on every config at full size (c3 / c5: 2 frames of the recipe)."""
    cfg = bs.load_config(name)
    _forced_parity(cfg, cfg.batch(N=N), label=f"{name} forced", frames=frames)


def test_forced_selector_bench_batch_sampled_frames():
    """Forced-selector mode in the bench's launch configuration (the whole 64-frame c3 batch)."""
    cfg = bs.load_config("c3")
    _forced_parity(cfg, cfg.batch(), label="c3 bench batch forced", frames=(5, 63))


@pytest.mark.parametrize("name,H,W,N", [("c1", 67, 129, 2), ("c4", 203, 333, 1), ("c2", 9, 17, 1)])
def test_forced_selector_ragged(name, H, W, N):
    cfg = _cfg_like(name, H, W, N)
    _forced_parity(cfg, cfg.batch(), label=f"{name}@{H}x{W} forced")


# ------------------------------------------------------------------ deep pyramids (merged fix-up)

@pytest.mark.parametrize("levels,H,W", [(7, 256, 256), (6, 130, 200), (12, 300, 260)])
def test_deep_pyramid_merged_fixup(levels, H, W):
    """levels >= 6 on a small image: more than kFixMax = 4 selector levels, so the merged fp64
    fix-up runs as ceil(nsel / 4) launches; the launch count says so and every level's map and
    the output obey the parity rule (the nsel > 4 path was untested)."""
    cfg = _cfg_like("c1", H, W, 1, levels=levels)
    nst = levels - 1
    cfg.strength_thresholds = [list(_TS1)] * nst
    cfg.coherence_thresholds = [list(_TC1)] * nst
    h = _handle(cfg)
    nsel = levels - 1
    # denoise: calls of <= BLADE_INLINE_FIX px (default 16 Ki) fix uncertified pixels inside
    # k_down (no fix-up launch); larger ones run the merged fix-up, ceil(nsel / 4) launches
    import os
    inline = H * W <= int(os.environ.get("BLADE_INLINE_FIX", 16384))
    # small calls run k_down_tile (uncertified pixels fixed inline, no fix-up launch)
    inline = inline or (H * W <= int(os.environ.get("BLADE_DOWN_TILE", 3 << 18)) and W % 4 == 0)
    # forced fused level-0 selector: level 0's fix-up is the stage fix-up, one more launch
    fused = os.environ.get("BLADE_FUSE_SEL") == "1" and os.environ.get("BLADE_TMA_RY") == "4"
    fixes = 0 if inline else (nsel + 2) // 4 + 1 if fused else (nsel + 3) // 4
    assert h.launch_count(1, H, W) == 2 * nsel + fixes, h.launch_count(1, H, W)
    _full_parity(cfg, cfg.batch(), label=f"L{levels}@{H}x{W}")


def test_deep_pyramid_merged_fixup_overflow():
    """The merged fix-up with 6 selector levels where level 0's list overflows (half the frame an
    exact 45-degree ramp): the whole level-0 map is recomputed in fp64 inside the merged launch;
    the natural half obeys the parity rule at every level that sees only natural rows."""
    H, W, levels = 256, 384, 7
    cfg = _cfg_like("c1", H, W, 1, levels=levels)
    cfg.strength_thresholds = [list(_TS1)] * (levels - 1)
    cfg.coherence_thresholds = [list(_TC1)] * (levels - 1)
    x = cfg.batch()
    yy, xx = np.mgrid[0:H // 2, 0:W]
    x[0, :, :H // 2] = (0.25 + (xx + yy) * 2.0 ** -10).astype(np.float32)
    h = _handle(cfg)
    xt = torch.from_numpy(x).cuda()
    ws = h.workspace(1, H, W)
    maps = h.selector(xt, workspace=ws)
    counts = h.fallback_count(1, H, W, ws)
    assert counts[0] > H * W // 64, counts
    ts, tc = cfg.thresholds()
    ob, feats = oracle.selector(x[0].astype(np.float64), cfg.n_orient, cfg.n_strength, cfg.n_coherence,
                                ts[0], tc[0], cfg.window_size, cfg.window_sigma, features=True)
    lo = H // 2 + 4
    gpu = maps[0][0].cpu().numpy().astype(np.int64)
    check_buckets(gpu[lo:], ob[lo:], tuple(f[lo:] for f in feats), cfg.n_orient, ts[0], tc[0],
                  "L7 natural half after overflow")
    per_o = cfg.n_strength * cfg.n_coherence
    top = slice(2, H // 2 - 3)
    d = (gpu[top] // per_o - ob[top] // per_o) % cfg.n_orient
    assert np.isin(d, [0, 1, cfg.n_orient - 1]).all()
    assert (gpu[top] % per_o == ob[top] % per_o).all()


# ------------------------------------------------------------------ NEXT f3 (b): halo-exchange bands

@pytest.mark.parametrize("name,H,W,G", [("c4", 900, 260, 2), ("c4", 1200, 333, 8), ("c2", 333, 260, 3),
                                        ("c1", 257, 100, 5), ("c3", 400, 1918, 4), ("c0", 64, 64, 4),
                                        ("c5", 512, 384, 3)])
def test_xband_bands_bit_identical(name, H, W, G):
    """Bands that exchange per-level halo rows (blade_ms_xband_step + device copies between the
    bands' workspaces, the single-GPU form of the NCCL exchange) reproduce the whole-frame
    blade_ms_denoise bit-exactly, for every config recipe (c0: L = 1, nothing to exchange)."""
    from paper_1802_06130_b200.xband import denoise_bands_local
    cfg = _cfg_like(name, H, W, 1)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    full = h.denoise(x)[0]
    got = denoise_bands_local(h, x, G)
    torch.cuda.synchronize()
    assert torch.equal(got, full)


def test_xband_step_argument_errors():
    from paper_1802_06130_b200.blade_ms import BladeError
    cfg = _cfg_like("c4", 900, 260, 1)
    h = _handle(cfg)
    lay = h.xband_layout(900, 260, 300, 300)
    x = torch.from_numpy(cfg.batch()).cuda()
    ws = torch.empty(lay["ws_bytes"], dtype=torch.uint8, device="cuda")
    out = torch.empty((3, 300, 260), device="cuda")
    band = x[0, :, lay["in_row0"]:lay["in_row0"] + lay["in_rows"]].contiguous()
    with pytest.raises(BladeError):  # step out of range
        h.xband_step(lay["n_steps"], band, lay["in_row0"], out, 300, 900, ws)
    with pytest.raises(BladeError):  # input band misses needed rows
        h.xband_step(0, band[:, 2:].contiguous(), lay["in_row0"] + 2, out, 300, 900, ws)
    with pytest.raises(BladeError):  # workspace too small
        h.xband_step(0, band, lay["in_row0"], out, 300, 900, ws[: lay["ws_bytes"] // 2])


# ------------------------------------------------------- memory-safety substitutes (no sanitizer)
# compute-sanitizer is closed on this pool (profiles/r02_sanitizer.txt); these checks stand in.

@pytest.mark.parametrize("name,H,W,N", [("c3", 256, 384, 3), ("c4", 160, 520, 1), ("c5", 64, 256, 2),
                                        ("c1", 67, 129, 2), ("c0", 64, 64, 1)])
def test_repeat_runs_bit_identical(name, H, W, N):
    """A shared-memory race (a missing barrier / mbarrier phase) shows as run-to-run nondeterminism:
    the same call repeated, interleaved with an unrelated call on a second stream, must be
    bit-identical every time."""
    cfg = _cfg_like(name, H, W, N)
    h = _handle(cfg)
    other = _cfg_like("c1", 130, 200, 2)
    h2 = _handle(other)
    x = torch.from_numpy(cfg.batch()).cuda()
    x2 = torch.from_numpy(other.batch()).cuda()
    ref = h.denoise(x)
    s2 = torch.cuda.Stream()
    for _ in range(5):
        with torch.cuda.stream(s2):
            h2.denoise(x2)
        got = h.denoise(x)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)


@pytest.mark.parametrize("name,H,W", [("c4", 300, 260), ("c2", 133, 97), ("c3", 120, 1918)])
def test_band_paths_write_only_their_buffers(name, H, W):
    """Guard bands before and after the output band and the workspace of a row-band call and of
    every step of a halo-exchange band stay untouched."""
    cfg = _cfg_like(name, H, W, 1)
    h = _handle(cfg)
    x = torch.from_numpy(cfg.batch()).cuda()
    r0, rn = H // 3, H // 3
    G = 4096
    for mode in ("rows", "xband"):
        if mode == "rows":
            i0, ni = h.band_rows(H, r0, rn)
            ws_n = h.band_workspace_size(H, W, r0, rn)
        else:
            lay = h.xband_layout(H, W, r0, rn)
            i0, ni, ws_n = lay["in_row0"], lay["in_rows"], lay["ws_bytes"]
        band = x[0, :, i0:i0 + ni].contiguous()
        n_out = 3 * rn * W
        ob = torch.full((n_out + 2 * G,), -3.5, dtype=torch.float32, device="cuda")
        out = ob[G:G + n_out].view(3, rn, W)
        wb = torch.full((ws_n + 2 * G,), 0x5A, dtype=torch.uint8, device="cuda")
        ws = wb[G:G + ws_n]
        if mode == "rows":
            h.denoise_rows(band, i0, r0, rn, H, out, ws)
        else:
            for s in range(lay["n_steps"]):
                h.xband_step(s, band, i0, out, r0, H, ws)
        torch.cuda.synchronize()
        assert bool((ob[:G] == -3.5).all()) and bool((ob[G + n_out:] == -3.5).all()), mode
        assert bool((wb[:G] == 0x5A).all()) and bool((wb[G + ws_n:] == 0x5A).all()), mode

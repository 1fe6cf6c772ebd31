"""Host logic of the halo-exchange row bands (NEXT f3 (b)), on CPU:

  * the plan (blade_ms_xband_layout, host-only C ABI): own rows partition every level, halos and
    input rows cover what the kernels read, and each band's send regions match its neighbours'
    recv regions row for row;
  * the transport: a world_size-3 gloo process group runs the exchange of bench.py's
    multi-GPU path (paper_1802_06130_b200.xband.exchange_dist) on CPU workspaces whose own rows
    carry (step, plane, global row, column) codes, and every halo row must arrive with the code
    of the same global row from the right neighbour.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import blade_synth as bs
from paper_1802_06130_b200.blade_ms import BladeError, region_view, xband_layout
from paper_1802_06130_b200.xband import band_edges


def _layouts(name, H, W, G):
    cfg = bs.load_config(name)
    return cfg, [xband_layout(cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.window_size, cfg.K, H, W,
                              r0, r1 - r0) for r0, r1 in band_edges(H, G)]


@pytest.mark.parametrize("name,H,W,G", [("c4", 6000, 8000, 8), ("c4", 6000, 8000, 2), ("c2", 3000, 4000, 4),
                                        ("c1", 512, 512, 3), ("c3", 1080, 1920, 5)])
def test_xband_plan_partitions_and_matches_neighbours(name, H, W, G):
    cfg, lays = _layouts(name, H, W, G)
    L = cfg.levels
    dims = [H]
    for _ in range(L - 1):
        dims.append((dims[-1] + 1) // 2)
    rf, rc = cfg.fine_size // 2, cfg.coarse_size // 2
    for l in range(L):  # own rows partition every level
        owns = [lay["own"][l] for lay in lays]
        assert owns[0][0] == 0 and owns[-1][1] == dims[l]
        assert all(a[1] == b[0] for a, b in zip(owns, owns[1:]))
    for b, lay in enumerate(lays):
        hz, hu = lay["halo_z"], lay["halo_u"]
        # the halo covers the selector (ws/2 + 1), decimation (4), fine taps and coarse taps + 1
        assert hz >= max(cfg.window_size // 2 + 1, 4, rf, rc + 1) and hu >= rc + 1
        o0, o1 = lay["own"][0]
        assert lay["in_row0"] == max(0, o0 - hz) and lay["in_row0"] + lay["in_rows"] == min(H, o1 + hz)
        for s in range(lay["n_steps"]):
            for side in (0, 1):
                snd, rcv = lay["send"][s][side], lay["recv"][s][side]
                nb = b - 1 if side == 0 else b + 1
                if not 0 <= nb < G:
                    assert rcv["rows"] == 0 and snd["rows"] == 0
                    continue
                other = lays[nb]
                o_snd, o_rcv = other["send"][s][1 - side], other["recv"][s][1 - side]
                assert (snd["row0"], snd["rows"], snd["planes"]) == (o_rcv["row0"], o_rcv["rows"], o_rcv["planes"])
                assert (rcv["row0"], rcv["rows"], rcv["planes"]) == (o_snd["row0"], o_snd["rows"], o_snd["planes"])
                assert snd["offset"] + snd["plane_stride"] * (snd["planes"] - 1) + 4 * snd["rows"] * snd["pitch"] \
                    <= lay["ws_bytes"]
        # exchanges: after every down step (z^{l+1}), after up steps of levels >= 1 (u^l)
        n = lay["n_steps"] // 2
        ex = [s for s in range(lay["n_steps"]) if any(lay["recv"][s][d]["rows"] or lay["send"][s][d]["rows"]
                                                     for d in (0, 1))]
        assert ex == (list(range(n)) + list(range(n, 2 * n - 1)) if L > 1 else [])
        # six planes (hi + lo) for levels that feed a selector, three otherwise
        for s in range(n):
            planes = {lay["send"][s][d]["planes"] for d in (0, 1) if lay["send"][s][d]["rows"]}
            assert planes <= {6 if s + 1 < L - 1 else 3}


def test_xband_plan_halo_far_smaller_than_recomputed_cone():
    """c4 at 8 bands: an interior band reads own +- 5 level-0 rows instead of the ~165-row cone
    of blade_ms_denoise_rows."""
    from paper_1802_06130_b200.shard import shard_for
    cfg, lays = _layouts("c4", 6000, 8000, 8)
    rec = shard_for(cfg, 3, 8)
    assert lays[3]["in_rows"] == 750 + 2 * 5
    assert rec.in_rows > 750 + 2 * 150


def test_xband_plan_rejects_too_thin_bands():
    cfg = bs.load_config("c4")
    with pytest.raises(BladeError) as ei:
        xband_layout(cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.window_size, cfg.K, 300, 64, 100, 40)
    assert ei.value.status == 7  # BLADE_EUNSUPPORTED: level 4 would own 3 < 5 rows
    whole = xband_layout(cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.window_size, cfg.K, 9, 17, 0, 9)
    assert whole["in_rows"] == 9 and all(r["rows"] == 0 for s in whole["recv"] for r in s)


def _code(step, plane, rows, cols):
    return ((step * 8 + plane) * 2048 + rows)[:, None] + cols[None, :] / 64.0  # exact in fp32


def _fill_own(ws, lay, s):
    for side in (0, 1):
        r = lay["send"][s][side]
        if r["rows"]:
            v = region_view(ws, r)
            for p in range(r["planes"]):
                rows = np.arange(r["row0"], r["row0"] + r["rows"], dtype=np.float64)
                v[p] = torch.from_numpy(_code(s, p, rows, np.arange(r["pitch"], dtype=np.float64)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_06130_b200.xband import exchange_dist
        cfg = bs.load_config("c4")
        H, W = 1200, 64
        r0, r1 = band_edges(H, world)[rank]
        lay = xband_layout(cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.window_size, cfg.K, H, W, r0, r1 - r0)
        ws = torch.full((lay["ws_bytes"],), 255, dtype=torch.uint8)
        bad = 0
        for s in range(lay["n_steps"]):
            _fill_own(ws, lay, s)
            exchange_dist(ws, lay, s, rank, world)
            for side in (0, 1):
                r = lay["recv"][s][side]
                if not r["rows"]:
                    continue
                v = region_view(ws, r).numpy()
                rows = np.arange(r["row0"], r["row0"] + r["rows"], dtype=np.float64)
                for p in range(r["planes"]):
                    bad += int((v[p] != _code(s, p, rows, np.arange(r["pitch"], dtype=np.float64))).sum())
        dist.barrier()
        q.put((rank, bad, lay["n_steps"]))
    finally:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_gloo_world3_halo_exchange_delivers_neighbour_rows():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [0] * world, res
    assert all(r[2] == 8 for r in res)

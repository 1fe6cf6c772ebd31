"""Multi-GPU host logic on CPU: the frame / row-band split of BASELINE.json
configs[3] / configs[4], the halo of a band checked against an independent brute-force dependency
cone written from the paper's definitions, and a world_size-2 gloo process group running the
bench's max-over-ranks reduction and shard planning (the data path itself has no collective)."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import blade_synth as bs
from paper_1802_06130_b200.shard import max_over_ranks, shard_for, split_even, units

ROOT = Path(__file__).resolve().parents[1]


def _fold(i: int, n: int) -> int:
    p = 2 * n
    m = i % p
    return m if m < n else p - 1 - m


def cone_rows(levels: int, nf: int, nc: int, ws: int, H: int, o0: int, on: int) -> set[int]:
    """Level-0 input rows the output rows [o0, o0+on) depend on, by brute-force propagation of
    row sets through the cascade (PAPER.md:265-284 Eq. 9, :260-263 decimation rows 2y-3..2y+4,
    :131-137 selector = gradient (+-1) and window (+-ws/2)); folds at every level's border."""
    dims = [H]
    for _ in range(levels - 1):
        dims.append((dims[-1] + 1) // 2)
    rf, rc, R = nf // 2, nc // 2, max(nf // 2, ws // 2 + 1)
    need_z = [set() for _ in range(levels)]
    need_u = [set() for _ in range(levels)]
    need_u[0] = set(range(o0, o0 + on))
    if levels == 1:
        return {_fold(y + d, H) for y in need_u[0] for d in range(-R, R + 1)}
    for l in range(levels - 1):
        for y in need_u[l]:
            need_z[l] |= {_fold(y + d, dims[l]) for d in range(-R, R + 1)}
            need_u[l + 1] |= {_fold(y // 2 + d, dims[l + 1]) for d in range(-rc, rc + 1)}
    need_z[levels - 1] |= need_u[levels - 1]
    for l in range(levels - 1, 0, -1):
        for y in need_z[l]:
            need_z[l - 1] |= {_fold(2 * y - 3 + a, dims[l - 1]) for a in range(8)}
    return need_z[0]


def test_split_even_partitions():
    for n in (1, 7, 64, 6000):
        for world in (1, 2, 3, 4, 8):
            parts = [split_even(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_frame_shards_cover_batch(world):
    cfg = bs.load_config("c3")
    shards = [shard_for(cfg, r, world) for r in range(world)]
    assert all(s.mode == "frames" for s in shards)
    frames = [f for s in shards for f in range(s.frame0, s.frame0 + s.frames)]
    assert frames == list(range(cfg.N))
    assert sum(units(cfg, s) for s in shards) == cfg.N * cfg.H * cfg.W


@pytest.mark.parametrize("name,world", [("c4", 2), ("c4", 4), ("c4", 8), ("c2", 3), ("c1", 5)])
def test_band_shards_cover_image_and_halo_covers_cone(name, world):
    cfg = bs.load_config(name)
    cfg.N = 1
    shards = [shard_for(cfg, r, world) for r in range(world)]
    assert all(s.mode == "bands" for s in shards) or world == 1
    rows = [y for s in shards for y in range(s.out_row0, s.out_row0 + s.out_rows)]
    assert rows == list(range(cfg.H))
    assert sum(units(cfg, s) for s in shards) == cfg.H * cfg.W
    for s in shards:
        cone = cone_rows(cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.window_size, cfg.H,
                         s.out_row0, s.out_rows)
        assert min(cone) >= s.in_row0 and max(cone) < s.in_row0 + s.in_rows, (s, min(cone), max(cone))
        assert s.in_rows <= max(cone) - min(cone) + 1 + 8  # not looser than the cone's span


def test_band_halo_c4_magnitude():
    """c4 (9x9, L=5): the halo of an interior band is ~165 rows each side."""
    cfg = bs.load_config("c4")
    s = shard_for(cfg, 3, 8)
    assert 150 <= s.out_row0 - s.in_row0 <= 180
    assert 150 <= (s.in_row0 + s.in_rows) - (s.out_row0 + s.out_rows) <= 180


def _free_port() -> int:
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c3, c4 = bs.load_config("c3"), bs.load_config("c4")
        mine = (shard_for(c3, rank, world), shard_for(c4, rank, world))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        t = max_over_ranks(10.0 + rank)  # the bench's step-time reduction
        dist.barrier()
        if rank == 0:
            q.put((gathered, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_and_max_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 11.0
    c3, c4 = bs.load_config("c3"), bs.load_config("c4")
    f = [s[0] for s in gathered]
    assert [(s.frame0, s.frames) for s in f] == [(0, 32), (32, 32)]
    b = [s[1] for s in gathered]
    assert b[0].out_row0 == 0 and b[0].out_rows + b[1].out_rows == c4.H
    assert b[1].out_row0 == b[0].out_rows
    # the two bands' input halos overlap (recomputed, not exchanged)
    assert b[1].in_row0 < b[0].out_rows < b[0].in_row0 + b[0].in_rows
    assert sum(units(c3, s) for s in f) == c3.N * c3.H * c3.W


def _bench_json(stdout: str) -> dict:
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{")]
    assert lines, stdout
    return json.loads(lines[-1])


def test_bench_self_launches_world2_dry_run():
    """bench.py --gpus 2 with no WORLD_SIZE launches its own 2 ranks (torch.distributed.run,
    127.0.0.1) and the world-2 path (gloo here: barrier, max-over-ranks time, rank-0 line)
    prints n_gpus: 2 (--gpus was parsed and ignored)."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _bench_json(r.stdout)
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    c3 = bs.load_config("c3")
    assert d["config"]["units_all_ranks"] == c3.N * c3.H * c3.W
    assert d["config"]["rank0_shard"]["frames"] == c3.N // 2


def test_bench_rejects_gpus_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2 and "disagrees" in r.stderr


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the tier's reference arm: the fp64 oracle on the host cores) prints
    one JSON line with impl, the metric / unit / higher_is_better of the blade arm, a cpu_baseline
    describing the run and an e2e with zero host<->device bytes; it runs on CPU (no GPU needed)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _bench_json(r.stdout)
    assert d["impl"] == "reference" and d["unit"] == "MP/s" and d["higher_is_better"] is True
    assert d["metric"] == "megapixels/sec full multiscale denoise" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "c1"

#!/usr/bin/env python
"""Benchmark: megapixels/s of the full multiscale BLADE denoise (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl blade|reference]

Default workload: configs/c3.json = BASELINE.json configs[3] (64 frames of 1920x1080 RGB fp32,
3-level pyramid, 144 buckets, 5x5 fine + 5x5 coarse phase-indexed pairs, AWGN 15/255). The
batch is split evenly over the GPUs (no collective on the data path; NCCL only for the start
barrier and the max-over-ranks time). One step = one blade_ms_denoise call over this rank's
frames: K1 decimation, K2 selector and K3 stage kernels for every level (all of SURVEY.md §8(a)).

Timing: W untimed warm-up steps, then K steps bracketed by barrier + cuda synchronize, CUDA
events on the launching stream, max over ranks. Inputs (1.59 GB at N=1) exceed the 126 MB L2,
so no flush is needed between steps. nvidia-smi clocks are sampled during the timed region.

`--impl reference` times the fp64 CPU oracle (oracle/) on the host cores, on bounded samples
of the same workload (the tier's reference arm); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import blade_synth as bs  # noqa: E402

FP32_LANES_PER_SM = 128  # B200: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md / guide unit counts)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks) of the run; without WORLD_SIZE in the environment and N > 1 "
                         "the bench launches its own N ranks (torch.distributed.run, one per GPU)")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--frames", type=int, default=None,
                    help="override the frame count (profiling only; not a bench line)")
    ap.add_argument("--impl", default="blade", choices=["blade", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--train", action="store_true",
                    help="NEXT f4: time the training accumulation (normal equations) of stage 0 "
                         "over this rank's frames instead of the denoise (not the headline)")
    ap.add_argument("--ycc", action="store_true",
                    help="per-channel Y/Cb/Cr banks (NEXT row f1) instead of one bank for R,G,B")
    ap.add_argument("--chunk", type=int, default=0,
                    help="NEXT f3: frame-chunked schedule, chunks of this many frames (0 = off)")
    ap.add_argument("--streams", type=int, default=2, help="internal streams of the chunked schedule")
    ap.add_argument("--halo", default="recompute", choices=["recompute", "exchange"],
                    help="row-band configs (c4) at N > 1: recompute each band's dependency cone, or "
                         "exchange per-level halo rows with the neighbour ranks (NEXT f3)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph (auto: when the call is small enough to be "
                         "launch-bound, <= 4 MP per rank)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU plumbing check of the multi-rank path (gloo, no GPU work, no kernels): "
                         "self-launch, barrier, max-over-ranks timing and the rank-0 JSON line, "
                         "marked dry_run; never a bench result")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time of the oracle sample (cpu_baseline)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def self_launch(args):
    """--gpus N: under torchrun (WORLD_SIZE set) N must equal WORLD_SIZE; otherwise, for N > 1,
    launch N ranks on this node with torch.distributed.run (127.0.0.1 rendezvous) running this
    same command line, and return its exit code. None = run in this process."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if args.gpus is not None and args.gpus != int(ws):
            print(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={ws}", file=sys.stderr)
            return 2
        return None
    if args.gpus is None or args.gpus <= 1:
        return None
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_dist(backend: str, local: int, world: int):
    """Process group for world > 1. NCCL logs its communicator set-up (NCCL_DEBUG=INFO, INIT
    subsystem) unless the caller chose otherwise, so the rank count is visible in the log."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampled every 50 ms in the background; keeps (t, fields) per line."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [s.strip() for s in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0: float, t1: float) -> dict:
        win = [f for t, f in self.samples if t0 <= t <= t1 + 0.05]
        if not win:  # region shorter than one period: take the nearest samples
            win = [f for t, f in self.samples if t0 - 0.2 <= t <= t1 + 0.2]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"],
                    "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return float("nan")
        sm = [num(f[0]) for f in win]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for f in win:
            for name, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.nanmedian(sm)), "sm_max_mhz": num(win[0][1]),
                "power_w_max": float(np.nanmax([num(f[2]) for f in win])),
                "reasons": sorted(reasons), "samples": len(win)}


# ----------------------------------------------------------------------------- work model

def level_dims(H, W, L):
    d = [(H, W)]
    for _ in range(L - 1):
        d.append(((d[-1][0] + 1) // 2, (d[-1][1] + 1) // 2))
    return d


def algorithmic_work(cfg, N):
    """Algorithmic HBM bytes / FP32 FLOPs per kernel launch for N frames.

    k_down(l) ("selector" in the profile): reads z^l (12 B/px at l = 0, fp32; 24 B/px hi + lo
    fp32 pair at l >= 1), writes s^l (1 B/px) and z^{l+1} as hi (+ lo unless l+1 is the
    coarsest level), 12 (+12) B per level-(l+1) px.
    k_stage(l): reads z^l fp32 (12 B/px), u^{l+1} fp32 (12 B per coarse px), s^l (1 B/px), writes
    u^l fp32 (12 B/px); FLOPs = 2 * 3 * (nf^2 + nc^2) per output pixel (one FMA = 2 FLOPs).
    """
    d = level_dims(cfg.H, cfg.W, cfg.levels)
    L = cfg.levels
    nf2 = cfg.fine_size ** 2
    nc2 = cfg.coarse_size ** 2 if L > 1 else 0
    out = {}
    nsel = 1 if L == 1 else L - 1
    for l in range(nsel):
        px = d[l][0] * d[l][1]
        px1 = d[l + 1][0] * d[l + 1][1] if L > 1 else 0
        rd = (12 if l == 0 else 24) * px
        wr = px + (px1 * (12 + (12 if l + 1 < L - 1 else 0)) if L > 1 else 0)
        out[("selector", l)] = dict(bytes=N * (rd + wr), flops=None)
        out[("stage", l)] = dict(bytes=N * (12 * px + 12 * px1 + px + 12 * px),
                                 flops=N * px * 3 * 2 * (nf2 + nc2))
    return out


def stage_smem_bytes_per_px(cfg, kind="k_stage_tma", ry=2):
    """Algorithmic (conflict-free) shared-memory bytes per output pixel of the stage kernel:
    every tap of the pixel's filter once (4 B), plus the window values a thread reads per pixel
    (k_stage_tma: ry x 4 pixels per thread share window rows; k_stage_ph: 2 x 2 sub-lattice;
    k_stage_p2: 2 rows 2 apart x 4 consecutive pixels)."""
    nf = cfg.fine_size
    nc = cfg.coarse_size if cfg.levels > 1 else 0
    taps = 4 * (nf * nf + nc * nc)
    if kind == "k_stage_ph":  # phase-split kernel, 2 x 2 sub-lattice pixels per thread
        vals = (nf + 2) * (nf + 2) * 12 / 4 + (nc + 1) * (nc + 1) * 12 / 4
    elif kind == "k_stage_p2":  # row-parity kernel: 2 rows (2 apart) x 4 consecutive pixels
        vals = (nf + 2) * (nf + 3) * 12 / 8 + (nc + 1) * (nc + 1) * 12 / 8
    else:                     # ry x 4 pixels per thread
        vals = (nf + ry - 1) * (nf + 3) * 12 / (4 * ry) + \
            ((nc + ry // 2 - 1) * (nc + 1) * 12 / (4 * ry) if nc else 0)
    return taps + vals


# ----------------------------------------------------------------------------- reference arm

def oracle_sample_rate(cfg, target_s: float):
    """Time the fp64 oracle (all host cores) on a bounded sample of the workload: whole frames of
    the config (frame 0, 1, ...) until about target_s seconds have been spent (at least one
    frame; if one frame would take longer than target_s, a full-width band of frame 0 treated
    as an image)."""
    import oracle
    oracle.build()
    taps = cfg.taps()
    W = cfg.W
    rows = min(cfg.H, 64)
    sub = bs.Config(**{**cfg.__dict__, "H": rows})
    z = cfg.frame(0, row0=0, rows=rows)
    t = time.perf_counter()
    oracle.denoise_config(sub, z, taps)
    per_px = (time.perf_counter() - t) / (rows * W)
    if per_px * cfg.H * W > target_s:  # one frame is already too long: a band of frame 0
        rows = int(min(cfg.H, max(16, target_s / per_px / W)))
        sub = bs.Config(**{**cfg.__dict__, "H": rows})
        z = cfg.frame(0, row0=0, rows=rows)
        t = time.perf_counter()
        oracle.denoise_config(sub, z, taps)
        dt = time.perf_counter() - t
        return rows * W / 1e6 / dt, dt, f"one {rows}x{W} full-width band of frame 0", oracle.max_threads()
    n, dt = 0, 0.0
    while dt < target_s and n < max(cfg.N, 1) * 4:
        z = cfg.frame(n % max(cfg.N, 1))
        t = time.perf_counter()
        oracle.denoise_config(cfg, z, taps)
        dt += time.perf_counter() - t
        n += 1
    return n * cfg.H * W / 1e6 / dt, dt, f"{n} full {cfg.H}x{W} frame(s)", oracle.max_threads()


def oracle_single_thread_rate(cfg, target_s: float = 3.0):
    """The same oracle on ONE host thread (the single-core figure), on a
    full-width band of frame 0 sized to about target_s seconds; MP/s and what was timed."""
    import oracle
    oracle.build()
    taps = cfg.taps()
    W = cfg.W
    nthreads = oracle.max_threads()
    oracle.set_threads(1)
    try:
        rows = min(cfg.H, 16)
        sub = bs.Config(**{**cfg.__dict__, "H": rows})
        z = cfg.frame(0, row0=0, rows=rows)
        t = time.perf_counter()
        oracle.denoise_config(sub, z, taps)
        per_px = (time.perf_counter() - t) / (rows * W)
        rows = int(min(cfg.H, max(16, target_s / per_px / W)))
        sub = bs.Config(**{**cfg.__dict__, "H": rows})
        z = cfg.frame(0, row0=0, rows=rows)
        t = time.perf_counter()
        oracle.denoise_config(sub, z, taps)
        dt = time.perf_counter() - t
    finally:
        oracle.set_threads(nthreads)
    return rows * W / 1e6 / dt, f"one {rows}x{W} full-width band of frame 0 (treated as an image), 1 thread, {dt:.1f} s"


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    cfg = bs.load_config(args.config)
    import oracle
    oracle.build()
    # one step = one bounded sample (a full-width band of one frame, ~0.25 MP)
    rows = int(min(cfg.H, max(16, 250_000 // cfg.W)))
    sub = bs.Config(**{**cfg.__dict__, "H": rows})
    taps = cfg.taps()
    frames = [cfg.frame(i % max(cfg.N, 1), row0=0, rows=rows) for i in range(min(4, args.steps + args.warmup))]
    for i in range(args.warmup):
        oracle.denoise_config(sub, frames[i % len(frames)], taps)
    t = time.perf_counter()
    for i in range(args.steps):
        oracle.denoise_config(sub, frames[i % len(frames)], taps)
    dt = (time.perf_counter() - t) / max(args.steps, 1)
    mp = rows * cfg.W / 1e6
    val = mp / dt
    sample = (f"one {rows}x{cfg.W} full-width band of a {cfg.name} frame per step "
              f"(treated as an image), fp64 oracle, OpenMP over rows")
    line = {"impl": "reference", "metric": "megapixels/sec full multiscale denoise",
            "value": val, "unit": "MP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "desc": cfg.description, "frames": cfg.N,
                       "H": cfg.H, "W": cfg.W, "levels": cfg.levels},
            "cpu_baseline": {"value": val, "unit": "MP/s", "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "MP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- dry run (CPU)

def run_dry(args):
    """The multi-rank plumbing of the blade arm on CPU (gloo): the same shard split, barrier,
    max-over-ranks reduction and rank-0 line; the step is a 1 ms host sleep, not the hot path."""
    import torch.distributed as dist
    from paper_1802_06130_b200.shard import max_over_ranks, shard_for, units
    rank, local, world = dist_env()
    init_dist("gloo", local, world)
    cfg = bs.load_config(args.config)
    shard = shard_for(cfg, rank, world)
    def barrier():
        if world > 1:
            dist.barrier()
    for _ in range(args.warmup):
        time.sleep(0.001)
    barrier()
    t = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.001)
    ms = (time.perf_counter() - t) * 1e3
    barrier()
    ms_max = max_over_ranks(ms)
    total = sum(units(cfg, shard_for(cfg, r, world)) for r in range(world))
    if rank == 0:
        print(json.dumps({"metric": "megapixels/sec full multiscale denoise", "dry_run": True,
                          "value": None, "unit": "MP/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms_max / max(args.steps, 1),
                          "config": {"workload": cfg.name, "units_all_ranks": total,
                                     "rank0_shard": shard.__dict__}}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- blade arm

def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:
        return rc
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    rank, local, world = dist_env()
    init_dist("nccl", local, world)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1802_06130_b200 import BladeMS
    from paper_1802_06130_b200.shard import max_over_ranks, shard_for, units
    cfg = bs.load_config(args.config)
    if args.frames:
        cfg.N = args.frames
    shard = shard_for(cfg, rank, world)
    H, W = cfg.H, cfg.W
    h = BladeMS.from_config(cfg, taps=cfg.taps(channels=3 if args.ycc else 1), device=local)
    stream = torch.cuda.current_stream(dev)

    def cur():  # the stream a step launches on (the capture stream while a graph is recorded)
        return torch.cuda.current_stream(dev)
    if shard.mode == "frames":
        # ---- this rank's frames, generated on the host (seeded), copied once to HBM
        n_local, f0 = shard.frames, shard.frame0
        x_host = torch.empty((n_local, 3, H, W), dtype=torch.float32).pin_memory()
        xn = x_host.numpy()
        for i in range(n_local):
            bs.scene(cfg.seed, f0 + i, H, W, cfg.n_grat, cfg.n_disk, cfg.noise, cfg.p0, cfg.p1,
                     out=xn[i])
        x = x_host.to(dev, non_blocking=False)
        out = torch.empty_like(x)
        if args.chunk:
            ws = torch.empty(h.pipeline_workspace_size(args.chunk, args.streams, H, W),
                             dtype=torch.uint8, device=dev)

            def step():
                h.denoise_pipelined(x, out, args.chunk, args.streams, ws, cur())
        else:
            ws = h.workspace(n_local, H, W)

            def step():
                h.denoise(x, out, ws, cur())

        def e2e_step():
            h.denoise_host(x_host, out_host, d_in, out, ws, stream)
        out_host = torch.empty_like(x_host).pin_memory()
        d_in = torch.empty_like(x)
        if args.chunk:
            ws_e2e = h.workspace(n_local, H, W)

            def e2e_step():  # noqa: F811 - the host path keeps its own frame pipeline
                h.denoise_host(x_host, out_host, d_in, out, ws_e2e, stream)
        io_in = io_out = n_local * 3 * H * W * 4
    else:
        # ---- this rank's row band of the one image: input rows of its dependency cone
        #      (--halo recompute), or own rows +- a small halo with per-level halo exchange
        #      between neighbour ranks (--halo exchange, NEXT f3; NCCL P2P)
        n_local = 1
        if args.halo == "exchange":
            from paper_1802_06130_b200.xband import denoise_band_dist
            lay = h.xband_layout(H, W, shard.out_row0, shard.out_rows)
            in_row0, in_rows = lay["in_row0"], lay["in_rows"]
            ws = torch.empty(lay["ws_bytes"], dtype=torch.uint8, device=dev)

            def run_band(src):
                denoise_band_dist(h, src, lay, out, ws, shard.out_row0, H, rank, world, cur())
        else:
            in_row0, in_rows = shard.in_row0, shard.in_rows
            ws = torch.empty(h.band_workspace_size(H, W, shard.out_row0, shard.out_rows),
                             dtype=torch.uint8, device=dev)

            def run_band(src):
                h.denoise_rows(src, in_row0, shard.out_row0, shard.out_rows, H, out, ws, cur())
        x_host = torch.from_numpy(np.ascontiguousarray(
            cfg.frame(0, row0=in_row0, rows=in_rows))).pin_memory()
        x = x_host.to(dev)
        out = torch.empty((3, shard.out_rows, W), dtype=torch.float32, device=dev)

        def step():
            run_band(x)

        out_host = torch.empty((3, shard.out_rows, W), dtype=torch.float32).pin_memory()
        d_in = torch.empty_like(x)

        def e2e_step():
            d_in.copy_(x_host, non_blocking=True)
            run_band(d_in)
            out_host.copy_(out, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
        io_in = 3 * in_rows * W * 4
        io_out = 3 * shard.out_rows * W * 4

    if args.train:
        if shard.mode != "frames":
            raise SystemExit("--train needs a frame-split config")
        clean_host = torch.empty_like(x_host)
        for i in range(n_local):
            bs.scene(cfg.seed, f0 + i, H, W, cfg.n_grat, cfg.n_disk, "none", 0.0, 0.0,
                     out=clean_host[i].numpy())
        clean = clean_host.to(dev)
        coarse = h.pyramid(x)[0] if cfg.levels > 1 else None
        E, cnt = h.train_accumulators()
        tws = torch.empty(1, dtype=torch.uint8, device=dev)
        import ctypes as _ct
        from paper_1802_06130_b200.blade_ms import lib as _lib
        b = _ct.c_size_t()
        _lib().blade_ms_train_workspace_size(h._h, n_local, H, W, _ct.byref(b))
        tws = torch.empty(b.value, dtype=torch.uint8, device=dev)

        def step():  # noqa: F811 - the timed step is one accumulation pass over the frames
            h.train_accumulate(0, x, clean, coarse, E, cnt, tws, stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- what one step touches, against the L2: small working sets are timed after an L2
    #      flush, large ones back to back (their inputs exceed the L2)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    footprint = int(x.numel() * 4 + out.numel() * 4 + ws.numel())
    small = footprint < 2 * l2
    use_graph = (args.graph == "on" or (args.graph == "auto" and n_local * H * W <= (4 << 20))) \
        and not args.train and not (args.halo == "exchange" and world > 1)
    run = step
    if use_graph:  # the whole cascade as one CUDA graph (launch-bound small calls)
        step()
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        run = graph.replay

    for _ in range(args.warmup):
        run()
    barrier()

    sampler = ClockSampler(local)
    time.sleep(0.4)  # nvidia-smi start-up
    barrier()
    # an event after every step (markers only): the timed region is e[0] .. e[K]; the per-step
    # spans give the median and best step beside the mean (SURVEY.md §8(d) timing protocol)
    evts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    t0 = time.time()
    evts[0].record(stream)
    for k in range(args.steps):
        run()
        evts[k + 1].record(stream)
    torch.cuda.synchronize(dev)
    t1 = time.time()
    barrier()
    warm_ms = evts[0].elapsed_time(evts[-1])
    step_spans = [evts[k].elapsed_time(evts[k + 1]) for k in range(args.steps)]
    flushed_ms = None
    if small:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        evs = []
        for _ in range(args.steps):
            flush.fill_(1)  # not timed: a 256 MB write evicts the previous step's lines
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize(dev)
        t1 = time.time()
        flushed_ms = sum(a.elapsed_time(b) for a, b in evs)
        barrier()
    time.sleep(0.1)
    sampler.stop()
    clocks = sampler.summary(t0, t1)
    ms = flushed_ms if small else warm_ms
    ms_max = max_over_ranks(ms, dev)
    ms_per_step = ms_max / args.steps
    total_px = cfg.N * H * W  # all ranks together (frames: the batch; bands: the whole image)
    assert world > 1 or units(cfg, shard) == total_px
    value = total_px / 1e6 / (ms_per_step / 1e3)
    warm_step = max_over_ranks(warm_ms, dev) / args.steps
    if small:
        l2_note = (f"working set {footprint / 1e6:.1f} MB < 2 x L2 ({l2 / 1e6:.0f} MB): L2 flushed by a "
                   f"256 MB write before every timed step (value); back-to-back rate in 'warm'")
    else:
        l2_note = f"working set {footprint / 1e9:.2f} GB per step > L2 ({l2 / 1e6:.0f} MB): no flush"

    if args.train:
        nt = cfg.fine_size ** 2 + (cfg.coarse_size ** 2 if cfg.levels > 1 else 0)
        dfma_px = 3 * (((nt + 1 + 3) // 4) * (((nt + 1 + 3) // 4) + 1) // 2) * 16
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
            if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        fp64_peak = n_sm * 64 * 2 * sm_max * 1e6 / 1e12
        line = {"metric": "megapixels/sec of training data (stage-0 normal equations, f4)",
                "value": value, "unit": "MP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64 accumulation",
                "data": "synthetic", "config": {"workload": cfg.name, "frames": cfg.N, "H": H, "W": W,
                                                 "taps": nt, "segments": cfg.n_phases * cfg.K},
                "dfma_per_px": dfma_px,
                "roofline": {"bound": "alu", "kernel": "k_train_gram (+ selector, sort)",
                             "achieved": value * 1e6 * dfma_px * 2 / 1e12, "peak": fp64_peak,
                             "unit": "TFLOP/s", "frac": value * 1e6 * dfma_px * 2 / 1e12 / fp64_peak,
                             "traffic": None,
                             "peak_source": f"derived: {n_sm} SMs x 64 FP64 lanes x 2 x {sm_max:.0f} MHz",
                             "note": "whole training step time (all kernels) against the FP64 pipe; "
                                     "algorithmic DFMA = 3 channels x 16 per 4x4 block of the upper "
                                     "block triangle of the (nt+1)-padded Gram"},
                "clocks": clocks}
        if rank == 0:
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- per-kernel breakdown: same steps again with events around every launch
    h.set_profiling(True)
    for _ in range(args.steps):
        step()
    prof = h.profile_read()
    h.set_profiling(False)
    torch.cuda.synchronize(dev)

    # ---- end to end through the C ABI with host buffers (H2D + compute + D2H per step)
    e2e_ms = []
    e2e_step()  # warm
    for _ in range(max(args.e2e_steps, 1)):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms.append(a.elapsed_time(b))
    e2e_t = max_over_ranks(float(np.median(e2e_ms)), dev)
    e2e_val = total_px / 1e6 / (e2e_t / 1e3)

    # ---- roofline of the dominant kernel
    if shard.mode == "frames":  # per launch: a chunk of frames under the chunked schedule
        work = algorithmic_work(cfg, min(args.chunk, n_local) if args.chunk else n_local)
    else:  # a band: the work model of an out_rows-row image (the halo rows are not counted)
        work = algorithmic_work(bs.Config(**{**cfg.__dict__, "H": shard.out_rows}), 1)
    kern = {k: (t / c, c) for k, (t, c) in prof.items()}
    step_kernel_ms = sum(t for t, _ in prof.values()) / args.steps
    dom = max(prof, key=lambda k: prof[k][0])
    dom_ms = kern[dom][0]
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = n_sm * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12  # TFLOP/s
    w = work[dom]
    traffic = None
    ent = None
    ncu_path = ROOT / "profiles" / "ncu_summary.json"
    if ncu_path.exists():
        try:
            nsum = json.loads(ncu_path.read_text())
            ent = nsum.get("kernels", {}).get(f"{cfg.name}:{dom[0]}:{dom[1]}")
            if ent:
                traffic = ent.get("dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    if w["flops"]:
        ach = w["flops"] / (dom_ms / 1e3) / 1e12
        roof = {"bound": "alu", "kernel": f"k_stage level {dom[1]}" if dom[0] == "stage" else dom[0],
                "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                "traffic": traffic,
                "peak_source": f"derived: {n_sm} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz",
                "algorithmic_flops_per_launch": w["flops"],
                "algorithmic_bytes_per_launch": w["bytes"], "ms_per_launch": dom_ms,
                "hbm_frac_of_measured": w["bytes"] / (dom_ms / 1e3) / 1e9 / hbm_peak}
        if dom[0] == "stage":
            # the unit that binds this kernel: shared memory. Conflict-free
            # algorithmic smem bytes / launch time vs 128 B/clk/SM; bank conflicts are the rest.
            px = w["flops"] / (6 * (cfg.fine_size ** 2 + (cfg.coarse_size ** 2 if cfg.levels > 1 else 0)))
            n_launch = (min(args.chunk, n_local) if args.chunk else n_local) if shard.mode == "frames" else 1
            skind, sry = h.stage_kernel(n_launch, H if shard.mode == "frames" else shard.out_rows, W, dom[1])
            roof["kernel"] = f"{skind} level {dom[1]} ({sry} rows/thread)" if skind == "k_stage_tma" \
                else f"{skind} level {dom[1]}"
            sb = px * stage_smem_bytes_per_px(cfg, skind, sry)
            sp = n_sm * 128 * sm_max * 1e6 / 1e12  # TB/s
            roof["sram"] = {"achieved": sb / (dom_ms / 1e3) / 1e12, "peak": sp, "unit": "TB/s",
                            "frac": sb / (dom_ms / 1e3) / 1e12 / sp,
                            "bytes_per_px": stage_smem_bytes_per_px(cfg, skind, sry),
                            "note": "conflict-free model (taps 4 B each + window values); the ncu "
                                    "capture of this launch (profiles/ncu_summary.json) gives the "
                                    "measured wavefronts below: the binding unit"}
            if ent and ent.get("smem_wavefronts"):
                roof["sram"]["measured"] = {
                    "wavefronts_per_launch": ent["smem_wavefronts"],
                    "bank_conflict_wavefronts": ent.get("smem_bank_conflicts"),
                    "frac_of_wavefront_slots": ent.get("smem_wavefront_frac"),
                    "source": "ncu --set full, l1tex__data_pipe_lsu_wavefronts_mem_shared (one launch)"}
    else:
        ach = w["bytes"] / (dom_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": f"k_down level {dom[1]}", "achieved": ach, "peak": hbm_peak,
                "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic,
                "ms_per_launch": dom_ms}
    step_work = algorithmic_work(cfg, n_local) if shard.mode == "frames" else work
    step_bytes = sum(v["bytes"] for v in step_work.values())
    hbm_ach = step_bytes / (ms_per_step / 1e3) / 1e9  # per GPU
    names = {"selector": "k_down", "stage": "k_stage", "decimate": "k_decimate", "fixup": "k_down_fixup"}
    breakdown = {f"{names.get(k[0], k[0])}{k[1]}": round(t, 4) for k, (t, c) in sorted(kern.items())}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            mps, dt, what, cores = oracle_sample_rate(cfg, args.cpu_seconds)
            cpu = {"value": mps, "unit": "MP/s", "cores": cores, "kind": "oracle",
                   "sample": f"{what} of {cfg.name}, fp64 C oracle, OpenMP over rows "
                             f"({dt:.1f} s of CPU time)"}
            v1, what1 = oracle_single_thread_rate(cfg)
            cpu["single_thread"] = {"value": v1, "unit": "MP/s", "cores": 1, "sample": what1}
        except Exception as e:  # the baseline must never break the GPU line
            cpu = {"value": None, "unit": "MP/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": "megapixels/sec full multiscale denoise",
            "value": value, "unit": "MP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "desc": cfg.description, "frames": cfg.N,
                       "frames_per_gpu": n_local, "H": H, "W": W, "levels": cfg.levels,
                       "fine": cfg.fine_size, "coarse": cfg.coarse_size, "buckets": cfg.K,
                       "filter_channels": "Y,Cb,Cr (f1)" if args.ycc else "shared R,G,B",
                       "parallelism": (f"frames split over {world} GPU(s), no collective"
                                       if shard.mode == "frames" else
                                       (f"row bands over {world} GPU(s) with recomputed halo "
                                        f"(rank 0: out rows {shard.out_row0}+{shard.out_rows}, "
                                        f"in rows {shard.in_row0}+{shard.in_rows}), no collective"
                                        if args.halo == "recompute" else
                                        f"row bands over {world} GPU(s), per-level halo rows "
                                        f"exchanged with the neighbour ranks (NCCL P2P)")),
                       "l2": l2_note,
                       "cuda_graph": bool(use_graph),
                       "schedule": (f"frame chunks of {args.chunk} on {args.streams} streams (f3)"
                                    if args.chunk and shard.mode == "frames" else "whole batch per launch")},
            "warm": {"value": total_px / 1e6 / (warm_step / 1e3), "ms_per_step": warm_step,
                     "note": "back-to-back steps, no flush" + (" (L2-resident working set)" if small else "")},
            "roofline": roof,
            "hbm": {"achieved": hbm_ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm_ach / hbm_peak,
                    "bytes_per_step_per_gpu": step_bytes,
                    "floor_frac": 24.0 * units(cfg, shard) / (ms_per_step / 1e3) / 1e9 / hbm_peak,
                    "note": "level-materialised algorithmic bytes of all kernels / step time; "
                            "floor_frac: 24 B/px (read the RGB input once, write the output once)"},
            "step_ms_stats": {"mean": warm_step, "median": float(np.median(step_spans)),
                              "best": float(np.min(step_spans)),
                              "note": "back-to-back timed steps of this rank (events between steps)"},
            "kernel_ms_per_step": breakdown,
            "kernel_sum_ms_per_step": step_kernel_ms,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "MP/s", "h2d_bytes_per_step": io_in,
                    "d2h_bytes_per_step": io_out, "ms_per_step": e2e_t},
            "gpu_launches": args.steps * world * (
                h.launch_count(n_local, H, W) if not (args.chunk and shard.mode == "frames") else
                h.launch_count(args.chunk, H, W) * -(-n_local // args.chunk)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Multi-GPU work split of the hot path. Host logic only.

The path shards with no collective on the data path (BASELINE.json north_star):
  * frames  (configs[3]): rank r of G takes frames [r*N/G, (r+1)*N/G) -- a batch is a set of
    independent problems;
  * bands   (configs[4]): rank r of G takes output rows [r*H/G, (r+1)*H/G) of ONE image and reads
    the input rows of that band's whole-pyramid dependency cone (blade_ms_band_plan); every index
    is global, so the concatenated band outputs equal the 1-GPU output bit-exactly.
NCCL (or gloo on CPU) carries only the start barrier and the max-over-ranks step time.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    mode: str          # "frames" or "bands"
    frame0: int        # frames mode: first frame; bands mode: 0
    frames: int        # frames mode: frame count; bands mode: 1
    out_row0: int = 0  # bands mode: output rows [out_row0, out_row0 + out_rows)
    out_rows: int = 0
    in_row0: int = 0   # bands mode: input rows needed [in_row0, in_row0 + in_rows)
    in_rows: int = 0


def split_even(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's share of n items, shares differing by at most one."""
    lo = rank * n // world
    hi = (rank + 1) * n // world
    return lo, hi


def shard_for(cfg, rank: int, world: int) -> Shard:
    """The work of `rank` out of `world` for a config (blade_synth.Config-like)."""
    if cfg.N > 1 or world == 1:
        if cfg.N % world:
            raise ValueError(f"{cfg.name}: {cfg.N} frames do not split evenly over {world} ranks")
        f0, f1 = split_even(cfg.N, world, rank)
        return Shard("frames", f0, f1 - f0, 0, cfg.H, 0, cfg.H)
    from .blade_ms import band_plan
    r0, r1 = split_even(cfg.H, world, rank)
    i0, ni = band_plan(cfg.levels, cfg.fine_size, cfg.coarse_size, cfg.window_size, cfg.H,
                       r0, r1 - r0)
    return Shard("bands", 0, 1, r0, r1 - r0, i0, ni)


def units(cfg, shard: Shard) -> int:
    """Output pixels (megapixel numerator) a shard produces."""
    if shard.mode == "frames":
        return shard.frames * cfg.H * cfg.W
    return shard.out_rows * cfg.W


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (step time) over the process group; identity without one."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

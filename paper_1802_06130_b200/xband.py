"""Row bands with a per-level halo EXCHANGE (NEXT f3). Host orchestration only.

SURVEY.md §8 f3 asks for "NVLink P2P per-level halo exchange for bands" in place of the recomputed
dependency cone of `blade_ms_denoise_rows` (§5: time linear in the pixels). A band
owns rows own^l of every level (own^{l+1} = [ceil(lo/2), ceil(hi/2)), a partition of each level
when the bands partition the image) and computes only those, step by step through the C ABI
(`blade_ms_xband_step`: the down pass level by level, then the up pass); after each step the
halo_z rows of z^{l+1} (hi + lo planes) or halo_u rows of u^l around its own rows are received
from the neighbour bands (`blade_ms_xband_layout` names the workspace regions):

  * `denoise_bands_local`: every band in this process (one GPU, or bands on several devices of
    one process); the exchange is a device copy between the bands' workspaces;
  * `denoise_band_dist`: one band per rank of a process group; the exchange is a
    `batch_isend_irecv` with ranks r - 1 and r + 1 (NCCL over NVLink between B200s; gloo on CPU
    for the host-logic tests). This is the path's only collective: a real exchange step.

The concatenated band outputs equal `blade_ms_denoise` of the whole frame bit-exactly.
"""
from __future__ import annotations

import torch

from .blade_ms import region_view


def exchange_local(workspaces, layouts, step: int) -> None:
    """Copy every band's send regions of `step` into its neighbours' recv regions."""
    G = len(layouts)
    for b in range(G):
        for side, nb in ((0, b - 1), (1, b + 1)):
            r = layouts[b]["recv"][step][side]
            if r["rows"] == 0:
                continue
            if not 0 <= nb < G:
                raise RuntimeError(f"band {b} expects halo rows from a missing band {nb}")
            s = layouts[nb]["send"][step][1 - side]
            if (s["row0"], s["rows"], s["planes"]) != (r["row0"], r["rows"], r["planes"]):
                raise RuntimeError(f"step {step}: band {nb} sends {s}, band {b} expects {r}")
            region_view(workspaces[b], r).copy_(region_view(workspaces[nb], s), non_blocking=True)


def band_edges(H: int, G: int) -> list[tuple[int, int]]:
    """Output rows [r0, r1) of G bands partitioning H rows (shares differ by at most one)."""
    if not 1 <= G <= H:
        raise ValueError(f"cannot split {H} rows into {G} non-empty bands")
    return [(g * H // G, (g + 1) * H // G) for g in range(G)]


def denoise_bands_local(h, x: torch.Tensor, G: int, stream=None) -> torch.Tensor:
    """All G bands of one frame x [1, 3, H, W] (CUDA) in this process, on x's device, step by
    step with device-copy halo exchanges; returns the denoised frame [3, H, W]."""
    _, _, H, W = x.shape
    bands = band_edges(H, G)
    lays = [h.xband_layout(H, W, r0, r1 - r0) for r0, r1 in bands]
    wss = [torch.empty(lay["ws_bytes"], dtype=torch.uint8, device=x.device) for lay in lays]
    ins = [x[0, :, lay["in_row0"]:lay["in_row0"] + lay["in_rows"]].contiguous() for lay in lays]
    outs = [torch.empty((3, r1 - r0, W), dtype=torch.float32, device=x.device) for r0, r1 in bands]
    for s in range(lays[0]["n_steps"]):
        for b, lay in enumerate(lays):
            h.xband_step(s, ins[b], lay["in_row0"], outs[b], bands[b][0], H, wss[b], stream)
        exchange_local(wss, lays, s)
    return torch.cat(outs, 1)


def exchange_dist(ws: torch.Tensor, layout: dict, step: int, rank: int, world: int) -> None:
    """One band per rank: send this band's boundary rows of `step` to ranks rank -/+ 1 and
    receive its halo rows from them (torch.distributed P2P, one batch)."""
    import torch.distributed as dist
    ops, recvs = [], []
    for side, peer in ((0, rank - 1), (1, rank + 1)):
        snd, rcv = layout["send"][step][side], layout["recv"][step][side]
        if not 0 <= peer < world:
            if rcv["rows"]:
                raise RuntimeError(f"rank {rank} expects halo rows from a missing rank {peer}")
            continue
        if snd["rows"]:
            ops.append(dist.P2POp(dist.isend, region_view(ws, snd).contiguous(), peer))
        if rcv["rows"]:
            buf = torch.empty((rcv["planes"], rcv["rows"], rcv["pitch"]), dtype=torch.float32,
                              device=ws.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer))
            recvs.append((rcv, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for rcv, buf in recvs:
        region_view(ws, rcv).copy_(buf)


def denoise_band_dist(h, in_band: torch.Tensor, layout: dict, out_band: torch.Tensor, ws: torch.Tensor,
                      out_row0: int, H: int, rank: int, world: int, stream=None) -> torch.Tensor:
    """This rank's band (layout of h.xband_layout for out rows [out_row0, +out_band.shape[1])):
    every step through the C ABI, halos exchanged with the neighbour ranks in between."""
    for s in range(layout["n_steps"]):
        h.xband_step(s, in_band, layout["in_row0"], out_band, out_row0, H, ws, stream)
        exchange_dist(ws, layout, s, rank, world)
    return out_band

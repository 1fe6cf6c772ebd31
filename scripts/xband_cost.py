"""NEXT f3 (b) evidence on ONE B200: the per-band cost of the c4 row-band split with a recomputed
dependency cone (blade_ms_denoise_rows) against per-level halo exchange (blade_ms_xband_step),
for G = 2, 4, 8 bands of the 48 MP image. Each band is timed alone (CUDA events, 5 repeats,
median); the G-GPU step would be the slowest band plus, for the exchange, the 2(L-1)-1 neighbour
transfers (measured here as device copies between the bands' workspaces, an upper bound on the
bytes and a lower bound on the NVLink latency). Prints one JSON line per G.

    python scripts/xband_cost.py [--config c4] [--bands 2,4,8]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import blade_synth as bs  # noqa: E402
from paper_1802_06130_b200 import BladeMS  # noqa: E402
from paper_1802_06130_b200.blade_ms import region_view  # noqa: E402
from paper_1802_06130_b200.xband import band_edges  # noqa: E402


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[1:]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--bands", default="2,4,8")
    args = ap.parse_args()
    cfg = bs.load_config(args.config)
    H, W = cfg.H, cfg.W
    h = BladeMS.from_config(cfg, device=0)
    x = torch.from_numpy(cfg.frame(0)).cuda()
    full = h.denoise(x[None])
    t_full = timed(lambda: h.denoise(x[None], full))
    for G in [int(g) for g in args.bands.split(",")]:
        bands = band_edges(H, G)
        rec, exc, xfer, rows_rec, rows_exc = [], [], [], [], []
        lays = [h.xband_layout(H, W, r0, r1 - r0) for r0, r1 in bands]
        wss = [torch.empty(l["ws_bytes"], dtype=torch.uint8, device="cuda") for l in lays]
        outs = [torch.empty((3, r1 - r0, W), device="cuda") for r0, r1 in bands]
        for g, (r0, r1) in enumerate(bands):
            i0, ni = h.band_rows(H, r0, r1 - r0)
            band = x[:, i0:i0 + ni].contiguous()
            ws = torch.empty(h.band_workspace_size(H, W, r0, r1 - r0), dtype=torch.uint8, device="cuda")
            o = torch.empty((3, r1 - r0, W), device="cuda")
            rec.append(timed(lambda: h.denoise_rows(band, i0, r0, r1 - r0, H, o, ws)))
            rows_rec.append(ni)
            lay = lays[g]
            xb = x[:, lay["in_row0"]:lay["in_row0"] + lay["in_rows"]].contiguous()
            rows_exc.append(lay["in_rows"])

            def run_steps(lay=lay, xb=xb, g=g, r0=r0):
                for s in range(lay["n_steps"]):
                    h.xband_step(s, xb, lay["in_row0"], outs[g], r0, H, wss[g])
            exc.append(timed(run_steps))
        # the transfers of every exchange, as device copies (both directions of every boundary)
        def copies():
            for s in range(lays[0]["n_steps"]):
                for b in range(G):
                    for side, nb in ((0, b - 1), (1, b + 1)):
                        r = lays[b]["recv"][s][side]
                        if r["rows"] and 0 <= nb < G:
                            region_view(wss[b], r).copy_(region_view(wss[nb], lays[nb]["send"][s][1 - side]))
        t_copy = timed(copies)
        xbytes = sum(4 * r["planes"] * r["rows"] * r["pitch"] for lay in lays for s in lay["recv"] for r in s)
        print(json.dumps({"config": cfg.name, "bands": G, "full_image_ms": t_full,
                          "recompute": {"max_band_ms": max(rec), "sum_ms": sum(rec),
                                        "max_in_rows": max(rows_rec)},
                          "exchange": {"max_band_ms": max(exc), "sum_ms": sum(exc),
                                       "max_in_rows": max(rows_exc), "n_exchanges": 2 * (cfg.levels - 1) - 1,
                                       "halo_bytes_all_bands": xbytes,
                                       "all_copies_one_gpu_ms": t_copy}}), flush=True)


if __name__ == "__main__":
    main()

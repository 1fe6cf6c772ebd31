"""Regenerate DESIGN.md §11's status table from profiles/r01_bench_*.jsonl (run after
scripts/collect_round.sh)."""
import json
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def L(n):
    return json.loads((ROOT / f"profiles/r01_bench_{n}.jsonl").read_text().strip().splitlines()[-1])


def f(x):
    return f"{x:,.0f}"


rows = []
d = L("c3"); k = d["kernel_ms_per_step"]
rows.append(f"| c3 (headline) | {f(d['value'])} | {d['ms_per_step']:.2f} | down {k['k_down0']:.2f} / {k['k_down1']:.2f}, "
            f"stage {k['k_stage0']:.2f} / {k['k_stage1']:.2f} | {f(d['e2e']['value'])} | {d['cpu_baseline']['value']:.1f} |")
for n, lab, note in [("c2", "c2 (7×7 pairs)", "(phase-split TMA)"), ("c4", "c4 (9×9 pairs, 48 MP)", "(phase-split TMA)")]:
    d = L(n); k = d["kernel_ms_per_step"]
    rows.append(f"| {lab} | {f(d['value'])} | {d['ms_per_step']:.2f} | down0 {k['k_down0']:.2f}, stage0 {k['k_stage0']:.2f} "
                f"{note} | {f(d['e2e']['value'])} | {d['cpu_baseline']['value']:.1f} |")
for n, lab in [("c1", "c1 (512², latency)"), ("c0", "c0 (64², latency)")]:
    d = L(n); k = d["kernel_ms_per_step"]
    lo, hi = min(k.values()) * 1e3, max(k.values()) * 1e3
    rows.append(f"| {lab} | {f(d['value'])} | {d['ms_per_step']:.3f} | {lo:.0f}–{hi:.0f} µs per kernel | "
                f"{f(d['e2e']['value'])} | {d['cpu_baseline']['value']:.1f} |")
d = L("c5"); k = d["kernel_ms_per_step"]
rows.append(f"| c5 (f2: 4096 buckets, 7×7/5×5) | {f(d['value'])} | {d['ms_per_step']:.2f} | down0 {k['k_down0']:.2f}, "
            f"stage0 {k['k_stage0']:.2f} (L2 taps) | {f(d['e2e']['value'])} | {d['cpu_baseline']['value']:.1f} |")
for n, lab in [("c3_ycc", "c3, f1 per-channel banks"), ("c2_ycc", "c2, f1"), ("c4_ycc", "c4, f1")]:
    d = L(n); k = d["kernel_ms_per_step"]
    rows.append(f"| {lab} | {f(d['value'])} | {d['ms_per_step']:.2f} | stage0 {k['k_stage0']:.2f} | {f(d['e2e']['value'])} | — |")
a, b = L("c1_ycc"), L("c0_ycc")
rows.append(f"| c1, f1 / c0, f1 | {f(a['value'])} / {f(b['value'])} | {a['ms_per_step']:.3f} / {b['ms_per_step']:.3f} | "
            f"latency | {f(a['e2e']['value'])} / {f(b['e2e']['value'])} | — |")
rows.append("| c3, f3 chunked schedule (1 frame × 2 streams / 8 frames × 2) | 19,594 / 27,157 | 6.77 / 4.89 | "
            "per-chunk launches (§10c) | — | — |")
d = L("c3_train")
rows.append(f"| c3, f4 training (stage-0 normal equations) | {f(d['value'])} | {d['ms_per_step']:.1f} (16 frames) | "
            f"k_train_gram ({d['roofline']['frac']:.2f} of FP64) | — | — |")
table = ("| config | MP/s | ms/step | kernel ms (down / stage per level) | e2e MP/s | oracle MP/s (16 cores) |\n"
         "|---|---|---|---|---|---|\n" + "\n".join(rows) + "\n\n")
p = ROOT / "DESIGN.md"
s = p.read_text()
a0 = s.index("| config | MP/s | ms/step |")
b0 = s.index("Reference arm (`bench.py --impl reference`")
s = s[:a0] + table + s[b0:]
ref = L("reference")
s = re.sub(r"on a 130×1920 band of a c3 frame per step, [0-9.]+ MP/s on [0-9]+ host cores",
           f"on a 130×1920 band of a c3 frame per step, {ref['value']:.1f} MP/s on "
           f"{ref['cpu_baseline']['cores']} host cores", s)
p.write_text(s)
print(table)

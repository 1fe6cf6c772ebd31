"""Summarise an `ncu --page source --csv --print-source cuda,sass` export per CUDA source line:
warp-stall samples and executed instructions (reads the CSV on stdin)."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hi = next(i for i, r in enumerate(rows[:10]) if "Source" in r)
hdr = rows[hi]
ci = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
agg = []
for r in rows[hi + 1:]:
    if r and r[0] and len(r) == len(hdr):  # a CUDA source line (SASS lines have an empty line number)
        try:
            agg.append((int(r[ci["Warp Stall Sampling (All Samples)"]] or 0),
                        int(r[ci["Instructions Executed"]] or 0), r[0], r[1][:90]))
        except (ValueError, KeyError):
            pass
tot_s = sum(a[0] for a in agg) or 1
tot_i = sum(a[1] for a in agg) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, n, ln, src in sorted(agg, reverse=True)[: int(sys.argv[1]) if len(sys.argv) > 1 else 25]:
    print(f"{100*s/tot_s:5.1f}% stall {100*n/tot_i:5.1f}% inst  L{ln:>4} {src}")

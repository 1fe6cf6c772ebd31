"""Per-CUDA-source-line summary of an ncu report: warp-stall samples and executed warp
instructions (from `ncu -i X --page source --csv --print-source cuda,sass`).

    python scripts/ncu_lines.py gpurun_out/X.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
cur_file = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        hdr = r if r[0] == "Line No" else None
        if hdr:
            H = hdr
        continue
    if len(r) < 8 or not r[0].isdigit():
        continue
    d = dict(zip(H, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        n = int(d.get("Instructions Executed") or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1][:90]])
    a[0] += s
    a[1] += n
tot_s = sum(a[0] for a in agg.values()) or 1
tot_i = sum(a[1] for a in agg.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for (f, ln), (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*s/tot_s:5.1f}% stall {100*n/tot_i:5.1f}% inst  {f}:{ln:<4} {src}")

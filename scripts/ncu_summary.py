"""Compact text summary of an ncu report (`ncu -i X.ncu-rep --page details --csv`) plus the
DRAM bytes per launch (`--page raw`: dram__bytes_read.sum + dram__bytes_write.sum).

    python scripts/ncu_summary.py gpurun_out/X.ncu-rep > profiles/rNN_X.txt
"""
import csv
import subprocess
import sys

KEEP = {"GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
        "Occupancy", "Launch Statistics", "Warp State Statistics", "Scheduler Statistics",
        "Instruction Statistics", "Source Counters"}


def run(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(out.splitlines()))


def main(rep):
    rows = run(rep, "details")
    hdr = rows[0]
    cur = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = f"[{d['ID']}] {d['Kernel Name'][:90]} grid {d['Grid Size']} block {d['Block Size']}"
        if k != cur:
            cur = k
            print("=" * 100)
            print(k)
        if d["Section Name"] not in KEEP and not d.get("Rule Name"):
            continue
        if d["Metric Name"]:
            print(f"  {d['Section Name'][:28]:28s} {d['Metric Name'][:44]:44s} "
                  f"{d['Metric Value']:>14s} {d['Metric Unit']}")
        elif d.get("Rule Description"):
            print(f"  ! {d['Rule Name']}: {d['Rule Description'][:300]}")
    raw = run(rep, "raw")
    h = raw[0]
    idx = {n: i for i, n in enumerate(h)}
    for r in raw[2:]:
        try:
            rd = float(r[idx["dram__bytes_read.sum"]].replace(",", ""))
            wr = float(r[idx["dram__bytes_write.sum"]].replace(",", ""))
        except (KeyError, ValueError):
            continue
        print(f"DRAM [{r[idx['ID']]}] {r[idx['Kernel Name']][:60]}: read {rd} "
              f"{raw[1][idx['dram__bytes_read.sum']]}, write {wr} "
              f"{raw[1][idx['dram__bytes_write.sum']]}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Write profiles/ncu_summary.json (the `traffic` source of bench.py's roofline) from full ncu
captures: per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and duration.

    python scripts/ncu_json.py c3:stage:0=gpurun_out/k_stage_full.ncu-rep \
                               c3:selector:0=gpurun_out/k_down_full.ncu-rep > profiles/ncu_summary.json
"""
import csv
import json
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def first_launch(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, r = rows[0], rows[1], rows[2]
    idx = {n: i for i, n in enumerate(h)}

    def val(name):
        return float(r[idx[name]].replace(",", "")) * UNIT.get(units[idx[name]], 1.0)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    d = {"kernel": r[idx["Kernel Name"]][:60], "dram_read_bytes": rd, "dram_write_bytes": wr,
         "dram_bytes_per_launch": rd + wr,
         "duration": f"{r[idx['gpu__time_duration.sum']]} {units[idx['gpu__time_duration.sum']]}"}
    # the shared-memory pipe (the stage's binding unit): wavefronts, their share of the launch's
    # wavefront slots, and the bank-conflict excess
    for k, name in (("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                    ("smem_wavefront_frac", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")):
        if name in idx:
            v = float(r[idx[name]].replace(",", ""))
            d[k] = v / 100.0 if k.endswith("frac") else v
    return d


out = {"note": "per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) from one "
               "`ncu --set full --clock-control none` capture of the timed-step launch of each kernel "
               "(bench.py default c3, 64 frames); writes still resident in L2 at kernel end are not "
               "counted", "kernels": {}}
for arg in sys.argv[1:]:
    key, rep = arg.split("=", 1)
    out["kernels"][key] = first_launch(rep)
print(json.dumps(out, indent=1))

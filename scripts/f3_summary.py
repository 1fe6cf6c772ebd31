"""Summarise the f3 runs (scripts/f3_run.sh outputs in gpurun_out/) into profiles/r01_f3_summary.txt."""
import csv
import glob
import json

MULT = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1, 'nsecond': 1, 'ns': 1, 'usecond': 1e3,
        'us': 1e3, 'msecond': 1e6, 'ms': 1e6}
print("NEXT f3: frame-chunked schedule (blade_ms_denoise_pipelined) vs the batch schedule, c3 recipe, 1 B200")
print()
print("DRAM bytes per level-0 pixel of one call on 8 frames (ncu --cache-control none, kernels serialised;")
print("scripts/f3_traffic.py; floor = 24 B/px: read the RGB fp32 input once, write the output once)")
for f in sorted(glob.glob('gpurun_out/f3_ncu_*.csv')):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    iv, iu, ival = hdr.index('Metric Name'), hdr.index('Metric Unit'), hdr.index('Metric Value')
    tot = {}
    for r in rows[1:]:
        tot[r[iv]] = tot.get(r[iv], 0) + float(r[ival].replace(',', '')) * MULT[r[iu]]
    px = 8 * 1920 * 1080
    name = f.split('f3_ncu_')[1][:-4]
    rd, wr = tot['dram__bytes_read.sum'] / px, tot['dram__bytes_write.sum'] / px
    print(f"  {name:18s} read {rd:6.2f} B/px  write {wr:6.2f} B/px  total {rd + wr:6.2f} B/px  "
          f"launches {(len(rows) - 1) // 3:4d}  kernel time (serialised) {tot['gpu__time_duration.sum'] / 1e6:.3f} ms")
print()
print("Throughput, bench.py --steps 10 --warmup 3 (64 x 1080p, inputs resident); kernel ms summed over the step")
for l in open('gpurun_out/f3_bench.log'):
    if l.startswith('{'):
        d = json.loads(l)
        print(f"  {d['config']['schedule']:42s} {d['value']:8.0f} MP/s  {d['ms_per_step']:.3f} ms/step  "
              f"kernels {d['kernel_ms_per_step']}")

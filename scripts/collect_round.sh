#!/bin/bash
# Copy the refresh outputs (scripts/refresh_round.sh) into profiles/ as round R (default r01).
R=${R:-r02}; O=gpurun_out/r; P=profiles
cp $O/pytest_gpu.txt $P/${R}_pytest_gpu.txt
cp $O/smoke.txt $P/${R}_smoke.txt
for f in $O/bench_*.jsonl; do b=$(basename $f); cp $f $P/${R}_$b; done
python scripts/ncu_launches.py $O/launches.csv > $P/${R}_launches.txt
python scripts/ncu_summary.py $O/k_stage_full.ncu-rep > $P/${R}_k_stage_tma_full.txt
python scripts/ncu_summary.py $O/k_down_full.ncu-rep > $P/${R}_k_down_full.txt
python scripts/ncu_lines.py $O/k_stage_full.ncu-rep 40 > $P/${R}_k_stage_tma_lines.txt
python scripts/ncu_lines.py $O/k_down_full.ncu-rep 40 > $P/${R}_k_down_lines.txt
python scripts/ncu_json.py c3:stage:0=$O/k_stage_full.ncu-rep c3:selector:0=$O/k_down_full.ncu-rep > $P/ncu_summary.json
cp $O/xband_cost.jsonl $P/${R}_xband_cost.jsonl 2>/dev/null; python scripts/sass_census.py > $P/${R}_sass_census.txt

( for f in $O/fuzz_*.log; do echo "$(basename $f): $(tail -1 $f | cut -c1-400)"; done ) > $P/${R}_fuzz_last_refresh.txt 2>/dev/null

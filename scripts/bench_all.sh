#!/bin/bash
# Bench lines of every config on one B200 (the refresh's bench part only) into gpurun_out/r/.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r; mkdir -p $O
for c in c3 c0 c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c > $O/bench_$c.jsonl 2> $O/bench_$c.err
done
for c in c3 c1; do
  timeout 600 python bench.py --config $c --ycc --no-cpu-baseline > $O/bench_${c}_ycc.jsonl 2> $O/bench_${c}_ycc.err
done

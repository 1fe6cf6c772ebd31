#!/bin/bash
# Single-GPU proxy of the c3 frame split: per-GPU work of an N-GPU run is 64/N frames.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for f in 8 16 32 64; do
  timeout 300 python bench.py --frames $f --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/frames_$f.json 2> gpurun_out/frames_$f.err
done

#!/bin/bash
# k_down band-height cap (BLADE_DOWN_RBMAX) at the per-GPU batches of the frame split
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for fr in 8 64; do for rb in 128 96 64 48 32 24 16; do
  echo "frames=$fr rbmax=$rb $(BLADE_DOWN_RBMAX=$rb timeout 120 python bench.py --frames $fr --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(round(d["value"]), round(d["ms_per_step"],4), d["kernel_ms_per_step"])')"
done; done > gpurun_out/rb_sweep.txt 2>&1

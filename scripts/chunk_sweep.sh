cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for fr in 8 16; do for ch in 1 2 4; do for s in 2 3; do
  echo "frames=$fr chunk=$ch streams=$s $(timeout 120 python bench.py --frames $fr --chunk $ch --streams $s --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(round(d["value"]), d["ms_per_step"])')"
done; done; done > gpurun_out/chunk_sweep.txt 2>&1

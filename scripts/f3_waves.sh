# Historical (round 1): swept the old wave-target band-height heuristic (BLADE_DOWN_WAVES), since
# replaced by the cost model in blade_ms.cu; kept as the record of profiles/r01_f3_summary.txt context.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for w in 1 2 4; do
for a in "--config c1" "--config c2" "--config c4" "--config c5" "--config c3" "--config c3 --chunk 1 --streams 2" "--config c3 --chunk 1 --streams 1"; do
  echo "WAVES $w ARGS $a" >> gpurun_out/waves.log
  BLADE_DOWN_WAVES=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 $a 2>&1 | tail -1 >> gpurun_out/waves.log
done; done

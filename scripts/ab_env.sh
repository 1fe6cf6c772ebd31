# A/B an environment knob over configs: VAR=BLADE_PDL VALS="0 1" CONFIGS="c1 c3" bash scripts/ab_env.sh
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in ${VALS}; do for c in ${CONFIGS}; do
  echo "$VAR=$v $c $(env $VAR=$v timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 ${EXTRA} 2>&1 | tail -1)" >> gpurun_out/ab.log
done; done

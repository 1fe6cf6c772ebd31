#!/bin/bash
# Compare alternative builds of libblade_ms.so on the default bench (kernel breakdown).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in main ${LIBS}; do
  if [ $v = main ]; then unset BLADE_MS_LIB; else export BLADE_MS_LIB=$PWD/$v; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/exp_$(basename $v).log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/exp_$(basename $v).log').readline());print('$v', round(d['value']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/exp_$(basename $v).log
done

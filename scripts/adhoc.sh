cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for ry in 0 4 0 4; do
if [ $ry = 0 ]; then unset BLADE_TMA_RY; else export BLADE_TMA_RY=$ry; fi
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ry.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/ry.log') if l.startswith('{')][-1]);print('ry=$ry', round(d['value']), d['kernel_ms_per_step'])" || tail -3 gpurun_out/ry.log
done

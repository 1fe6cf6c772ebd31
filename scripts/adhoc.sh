cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for k in 1 2; do
timeout 120 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c5.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/c5.log') if l.startswith('{')][-1]);print('c5', round(d['value']), d['kernel_ms_per_step'])" || tail -3 gpurun_out/c5.log
done
timeout 600 python -m pytest tests -m gpu -x -q -k "c5 or 320 or wide or selector_and_layout or train or forced_selector" > gpurun_out/pt_c5.log 2>&1; tail -3 gpurun_out/pt_c5.log

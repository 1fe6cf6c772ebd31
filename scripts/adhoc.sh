cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for tr in 16 0; do for c in c1 c0; do
BLADE_TMA_TR=$tr timeout 120 python bench.py --config $c --steps 50 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sm.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/sm.log') if l.startswith('{')][-1]);print('tr=$tr $c', round(d['value']), round(d['ms_per_step']*1e3,1), 'warm', round(d['warm']['ms_per_step']*1e3,1), d['kernel_ms_per_step'])" || tail -3 gpurun_out/sm.log
done; done
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sm3.log 2>&1; python -c "import json;d=json.loads([l for l in open('gpurun_out/sm3.log') if l.startswith('{')][-1]);print('c3', round(d['value']), d['kernel_ms_per_step'])"
timeout 600 python -m pytest tests -m gpu -x -q -k "c1 or c0 or ragged or tiny or delta or constant or footprint or forced_selector or band or repeat or variants" > gpurun_out/pt_sm.log 2>&1; tail -3 gpurun_out/pt_sm.log

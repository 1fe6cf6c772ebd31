cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for tr in 16 20 16 20; do
BLADE_TMA_TR=$tr timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tr.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/tr.log') if l.startswith('{')][-1]);print('tr=$tr', round(d['value']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/tr.log
done
BLADE_TMA_TR=20 timeout 600 python -m pytest tests -m gpu -x -q -k "c3 or c1_full or bench_launch or forced_selector_every or ragged or delta or constant or band or repeat" > gpurun_out/pt_tr.log 2>&1; tail -3 gpurun_out/pt_tr.log

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for d in 1 0 1 0; do
BLADE_DOWN4=$d timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/d4.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/d4.log') if l.startswith('{')][-1]);print('down4=$d', round(d['value']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/d4.log
done
timeout 600 python -m pytest tests -m gpu -x -q -k "c3 or c1 or c0 or c2 or bench_launch or forced_selector or ragged or tiny or band or repeat or selector_and_layout or fallback or overflow or batch or pipelined" > gpurun_out/pt_d4.log 2>&1; tail -3 gpurun_out/pt_d4.log

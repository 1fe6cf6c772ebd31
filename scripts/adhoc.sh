cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for f in 1 0; do
BLADE_FUSE_SEL=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fs.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/fs.log') if l.startswith('{')][-1]);print('fuse=$f', round(d['value']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/fs.log
done
timeout 900 python -m pytest tests -m gpu -x -q -k "c3 or bench_launch or forced or fallback or repeat or band or xband or delta or constant or batch or pipelined or no_writes or ragged or c4 or clamp" > gpurun_out/pt_fs.log 2>&1; tail -15 gpurun_out/pt_fs.log

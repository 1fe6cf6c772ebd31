cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for lib in pk0 pk1 pk0 pk1; do
export BLADE_MS_LIB=$PWD/paper_1802_06130_b200/libblade_ms_$lib.so
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_$lib.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/b_$lib.log') if l.startswith('{')][-1]);print('$lib', round(d['value']), d['kernel_ms_per_step'])"
done

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for lib in main t24 main t24; do
if [ $lib = main ]; then unset BLADE_MS_LIB; else export BLADE_MS_LIB=$PWD/paper_1802_06130_b200/libblade_ms_$lib.so; fi
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/t24.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/t24.log') if l.startswith('{')][-1]);print('$lib', round(d['value']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/t24.log
done
export BLADE_MS_LIB=$PWD/paper_1802_06130_b200/libblade_ms_t24.so
timeout 900 python -m pytest tests -m gpu -x -q -k "c3 or c1 or bench_launch or forced_selector or delta or constant or ragged or band or repeat" > gpurun_out/pt_t24.log 2>&1; tail -5 gpurun_out/pt_t24.log

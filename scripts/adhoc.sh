cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
rm -f gpurun_out/fixup_ab.txt
run() { tag=$1; shift; for m in 0 1; do
BLADE_FIXUP_MERGE=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 --graph off "$@" > gpurun_out/fx.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/fx.log') if l.startswith('{')][-1]);print('$tag merge=$m', round(d['config']['frames_per_gpu']*d['config']['H']*d['config']['W']/1e6,2), 'MP', round(d['warm']['ms_per_step']*1e3,1), 'us warm', round(d['ms_per_step']*1e3,1), 'us value')" >> gpurun_out/fixup_ab.txt; done; }
run c1 --config c1
run c1x4 --config c1 --frames 4
run c3f1 --frames 1
run c3f2 --frames 2
run c3f4 --frames 4
run c3f8 --frames 8
run c3f16 --frames 16
cat gpurun_out/fixup_ab.txt

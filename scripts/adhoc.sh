cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/pt_train.log 2>&1; tail -2 gpurun_out/pt_train.log
for k in 1 2; do
timeout 300 python bench.py --train --frames 16 --steps 5 --warmup 3 > gpurun_out/tr.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/tr.log') if l.startswith('{')][-1]);print('train', round(d['value']), d['roofline']['frac'])" || tail -3 gpurun_out/tr.log
done

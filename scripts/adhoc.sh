cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/pt_train.log 2>&1; tail -2 gpurun_out/pt_train.log
for g in -1 -1; do
timeout 300 python bench.py --train --frames 16 --steps 5 --warmup 3 > gpurun_out/tr.log 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/tr.log') if l.startswith('{')][-1]);print('group=$g', round(d['value']), d['roofline']['frac'])" || tail -3 gpurun_out/tr.log
done
timeout 300 python bench.py --train --frames 16 --steps 2 --warmup 3 > gpurun_out/tr_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 70 -c 70 --csv --log-file gpurun_out/tr_launches.csv python bench.py --train --frames 16 --steps 2 --warmup 3 > gpurun_out/tr_ncu.log 2>&1

#!/bin/bash
# Full evidence refresh on one B200 (one gpurun call): GPU tests, smoke, bench lines for every
# config (+ per-channel banks, training, reference arm), the halo-exchange band cost, the c3 ncu
# launch list and full captures of the two dominant kernels. Outputs under gpurun_out/r/;
# scripts/collect_round.sh copies the summaries into profiles/.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
for c in c3 c0 c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c > $O/bench_$c.jsonl 2> $O/bench_$c.err
done
for c in c3 c1 c5; do  # c5 --ycc: the paper's own layout (4096 buckets x per-channel banks)
  timeout 600 python bench.py --config $c --ycc --no-cpu-baseline > $O/bench_${c}_ycc.jsonl 2> $O/bench_${c}_ycc.err
done
# random sweeps (tests/fuzz_cases.py): parity, bit-identity, per-channel banks, halo-exchange bands
for m in "" identity ycc xband; do
  timeout 600 python scripts/fuzz_parity.py 200 41 $m > $O/fuzz_${m:-parity}.log 2>&1
done
timeout 600 python scripts/fuzz_parity.py 40 42 big > $O/fuzz_big.log 2>&1
timeout 600 python bench.py --train --frames 16 --steps 5 --warmup 3 > $O/bench_c3_train.jsonl 2> $O/bench_c3_train.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.jsonl 2> $O/bench_reference.err
timeout 600 python scripts/xband_cost.py > $O/xband_cost.jsonl 2> $O/xband_cost.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 7 -c 1 -o $O/k_stage_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_stage.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_down -s 12 -c 1 -o $O/k_down_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_down.log 2>&1
echo done > $O/DONE

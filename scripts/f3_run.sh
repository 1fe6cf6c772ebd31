set -x
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined or batch_equals or host_equals" > gpurun_out/f3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f3_pytest.log
for a in "" "--chunk 1 --streams 1" "--chunk 1 --streams 2" "--chunk 2 --streams 2" "--chunk 1 --streams 3" "--chunk 4 --streams 2"; do
  echo "ARGS $a" >> gpurun_out/f3_bench.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 $a >> gpurun_out/f3_bench.log 2>&1
done
for a in "" "--chunk 1 --streams 1" "--chunk 1 --streams 2" "--chunk 2 --streams 2"; do
  n=$(echo "$a" | tr -d ' -'); n=${n:-batch}
  timeout 300 ncu --profile-from-start off --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/f3_ncu_$n.csv python scripts/f3_traffic.py --frames 8 $a > gpurun_out/f3_ncu_$n.log 2>&1
done

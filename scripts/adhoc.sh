cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "xband or forced or deep or row_bands or shard" > gpurun_out/pt_new.log 2>&1; echo "rc=$?" >> gpurun_out/pt_new.log
timeout 300 python bench.py --config c4 --halo exchange --no-cpu-baseline --e2e-steps 1 --steps 10 > gpurun_out/b_c4x.log 2>&1
timeout 300 python bench.py --config c4 --no-cpu-baseline --e2e-steps 1 --steps 10 > gpurun_out/b_c4.log 2>&1

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "forced_variants" > gpurun_out/pt_ifix.log 2>&1; tail -3 gpurun_out/pt_ifix.log

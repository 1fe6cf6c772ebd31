cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_ph -s 3 -c 1 -o gpurun_out/ph_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ph_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_ph -s 2 -c 1 -o gpurun_out/ph_c2 -f python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ph_c2.log 2>&1

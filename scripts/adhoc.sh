cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/st_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_tma -s 7 -c 1 -o gpurun_out/st_r4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/st_ncu.log 2>&1; echo rc=$?

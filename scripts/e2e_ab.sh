# e2e (host buffers) A/B over the number of pipeline chunks of blade_ms_denoise_host
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/pcie_bw.py > gpurun_out/e2e_ab.log 2>&1
for c in 16 32 64 32; do
  echo "CH=$c $(BLADE_E2E_CHUNKS=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 2>&1 | tail -1)" >> gpurun_out/e2e_ab.log
done

cd $GRAFT_REPO_ROOT
./scripts/fp64_peak > gpurun_out/r2b_fp64.json 2>&1; cat gpurun_out/r2b_fp64.json
timeout 60 ./scripts/tmem_probe > gpurun_out/r2b_tmem.json 2>&1; cat gpurun_out/r2b_tmem.json
timeout 1500 python -m pytest tests -m gpu -q -s -k "192 or polynomial or generic or 64 or monitor" > gpurun_out/r2b_gpu_new.log 2>&1; echo "new rc=$?"; grep -E "192\^3|passed|failed" gpurun_out/r2b_gpu_new.log | tail -5
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2b_gpu.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/r2b_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2b_bench_wave.log 2>&1; tail -1 gpurun_out/r2b_bench_wave.log | cut -c1-300
timeout 600 python bench.py --config bssn192 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2b_bench_bssn.log 2>&1; tail -1 gpurun_out/r2b_bench_bssn.log | cut -c1-300

# fused-pair kernel iteration: parity tests, then bench (no ncu)
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_wave.py -x -q > gpurun_out/f3_pytest.log 2>&1; tail -3 gpurun_out/f3_pytest.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/f3_bench.log 2>&1; tail -1 gpurun_out/f3_bench.log | cut -c1-400
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/f3_bench2.log 2>&1; tail -1 gpurun_out/f3_bench2.log | cut -c1-400

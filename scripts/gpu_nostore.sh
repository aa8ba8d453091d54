timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_wave.py -x -q > gpurun_out/ts_pytest.log 2>&1; tail -1 gpurun_out/ts_pytest.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ns_0.log 2>&1; echo "tmastore $(tail -1 gpurun_out/ns_0.log | cut -c100-175)"

timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/f7_pytest.log 2>&1; tail -3 gpurun_out/f7_pytest.log
for v in 6 7; do
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant $v > gpurun_out/f7_b$v.log 2>&1; echo "v=$v $(tail -1 gpurun_out/f7_b$v.log | cut -c100-175)"
done

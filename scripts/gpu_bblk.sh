for b in 32x4x1 16x4x2 8x4x4 8x8x2 16x8x1 4x4x8 32x2x2; do
CHEMORA_BSSN_BLOCK=$b python bench.py --config bssn192 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bb_$b.log 2>&1
done
python -m pytest tests/test_gpu_bssn.py -x -q > gpurun_out/bb_pytest.log 2>&1; tail -1 gpurun_out/bb_pytest.log

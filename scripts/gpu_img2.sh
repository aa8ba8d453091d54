timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_wave.py tests/test_gpu_next.py -x -q 2>&1 | tail -1
for v in 6 0 4; do
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant $v > gpurun_out/im_$v.log 2>&1; echo "v=$v $(tail -1 gpurun_out/im_$v.log | cut -c100-180)"
done

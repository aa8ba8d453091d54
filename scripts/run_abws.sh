# A/B of an alternative wave pair kernel build (ab/lib$1.so): GPU wave tests, then timing
mkdir -p ab
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig0.so
cp ab/lib$1.so $L
timeout 120 python -m pytest -x -q -m gpu tests/test_gpu_wave.py tests/test_gpu_fused.py tests/test_gpu_next.py > gpurun_out/pt_$1.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_$1.log
cp ab/orig0.so $L
bash scripts/ab_swap.sh "--steps 20 --warmup 5 --no-secondary" cur $1 > gpurun_out/ab_$1.log 2>&1

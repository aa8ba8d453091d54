# order-2 pair kernels: tests (wave) + timing of variant 0 vs 8 at order 2, and order 4 A/B vs cur
mkdir -p ab
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig0.so
cp ab/lib$1.so $L
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_wave.py tests/test_gpu_fused.py tests/test_gpu_next.py > gpurun_out/pt_$1.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_$1.log
for v in 0 8 0 8; do timeout 300 python bench.py --fd-order 2 --variant $v --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-secondary | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('order2 variant', $v, d['ms_per_step'])"; done >> gpurun_out/o2_$1.log 2>&1
cp ab/orig0.so $L
bash scripts/ab_swap.sh "--steps 20 --warmup 5 --no-secondary" cur $1 >> gpurun_out/o2_$1.log 2>&1

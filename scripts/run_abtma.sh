# A/B of the persistent TMA z-march (wave variant 4, default for FD orders 6/8): tests, timing
mkdir -p ab
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig0.so
cp ab/lib$1.so $L
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_wave.py > gpurun_out/pt_$1.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_$1.log
cp ab/orig0.so $L
for o in 6 8; do
  echo "order $o" >> gpurun_out/ab_$1.log
  bash scripts/ab_swap.sh "--steps 10 --warmup 3 --no-secondary --fd-order $o" cur $1 >> gpurun_out/ab_$1.log 2>&1
done

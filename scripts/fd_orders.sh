# NEXT-1: the wave step at every run-time FD order (512^3, default tiling per order)
for o in 2 4 6 8; do
  timeout 300 python bench.py --fd-order $o --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-secondary | tail -1 >> gpurun_out/fd_orders.jsonl
done

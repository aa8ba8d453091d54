for p in 0 1 2; do for v in 3 4; do
CHEMORA_TMA_PROMO=$p python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant $v > gpurun_out/p_${p}_v$v.log 2>&1
done; done
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 0 > gpurun_out/p_v0.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 4"
$B > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches.csv $B > gpurun_out/p_ncu1.log 2>&1

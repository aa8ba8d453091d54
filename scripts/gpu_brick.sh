python -m pytest tests/test_gpu_wave.py -x -q -k "variants or fd_order" > gpurun_out/br_pytest.log 2>&1; tail -1 gpurun_out/br_pytest.log
for v in 0 5 1; do
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant $v > gpurun_out/br_v$v.log 2>&1
done
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 5"
$B > gpurun_out/br_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv --log-file gpurun_out/br_launches.csv $B > gpurun_out/br_ncu1.log 2>&1

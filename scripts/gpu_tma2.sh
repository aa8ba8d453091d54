python -m pytest tests/test_gpu_wave.py -x -q > gpurun_out/t2_pytest.log 2>&1
tail -1 gpurun_out/t2_pytest.log
for v in 0 3 4; do
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant $v > gpurun_out/t2_v$v.log 2>&1
done
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 4"
$B > gpurun_out/t2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/t2_launches.csv $B > gpurun_out/t2_ncu1.log 2>&1

timeout 900 python -m pytest tests/test_gpu_bssn.py tests/test_gpu_bssn_variants.py tests/test_gpu_next.py -x -q > gpurun_out/bt_pytest.log 2>&1; tail -3 gpurun_out/bt_pytest.log
for v in 0 2; do
python bench.py --config bssn192 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 --variant $v > gpurun_out/bt_v$v.log 2>&1
done
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 0"
$B > gpurun_out/bt_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -c 12 --csv --log-file gpurun_out/bt_launches.csv $B > gpurun_out/bt_ncu.log 2>&1

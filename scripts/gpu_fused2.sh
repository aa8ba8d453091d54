timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/fu2_pytest.log 2>&1; tail -3 gpurun_out/fu2_pytest.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 6 > gpurun_out/fu2_v6.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 6"
$B > gpurun_out/fu2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active --clock-control none -c 40 --csv --log-file gpurun_out/fu2_launches.csv $B > gpurun_out/fu2_ncu1.log 2>&1

python -m pytest tests/test_gpu_bssn.py -x -q > gpurun_out/b_pytest.log 2>&1
python bench.py --config bssn192 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_bench0.log 2>&1
python bench.py --config bssn192 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 1 > gpurun_out/b_bench1.log 2>&1
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none -c 40 --csv --log-file gpurun_out/b_launches.csv $B > gpurun_out/b_ncu.log 2>&1
tail -3 gpurun_out/b_pytest.log

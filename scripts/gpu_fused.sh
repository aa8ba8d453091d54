timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/fu_pytest.log 2>&1; tail -15 gpurun_out/fu_pytest.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 6 > gpurun_out/fu_v6.log 2>&1
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 0 > gpurun_out/fu_v0.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 6"
$B > gpurun_out/fu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/fu_launches.csv $B > gpurun_out/fu_ncu1.log 2>&1

set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 1 > gpurun_out/r2_bench_v1.log 2>&1
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 0 > gpurun_out/r2_bench_v0.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/r2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv $B > gpurun_out/r2_ncu1.log 2>&1
$B --variant 1 > gpurun_out/r2_plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_v1.csv $B --variant 1 > gpurun_out/r2_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wave_zmarch -s 4 -c 4 -o gpurun_out/r2_prof $B > gpurun_out/r2_ncu3.log 2>&1
tail -2 gpurun_out/r2_pytest.log

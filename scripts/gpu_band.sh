python -m pytest tests/test_gpu_wave.py -x -q > gpurun_out/bd_pytest.log 2>&1
tail -1 gpurun_out/bd_pytest.log
for b in 0 2 4 8 16 32 64; do
  CHEMORA_WAVE_BAND=$b python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bd_$b.log 2>&1
done
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bd_auto.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/bd_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/bd_launches.csv $B > gpurun_out/bd_ncu1.log 2>&1

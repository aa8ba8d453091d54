python bench.py --config bssn192 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bm.log 2>&1
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/bm_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 16 --csv --log-file gpurun_out/bm_launches.csv $B > gpurun_out/bm_ncu.log 2>&1

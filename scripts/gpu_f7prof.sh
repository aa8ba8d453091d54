B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 7"
$B > gpurun_out/f7p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wave_fused2 -s 2 -c 2 -o gpurun_out/f7_prof $B > gpurun_out/f7p_ncu.log 2>&1
tail -1 gpurun_out/f7p_ncu.log

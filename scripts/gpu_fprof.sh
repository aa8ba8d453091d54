B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 6"
$B > gpurun_out/fp3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wave_fused -s 2 -c 2 -o gpurun_out/fp3_prof $B > gpurun_out/fp3_ncu.log 2>&1

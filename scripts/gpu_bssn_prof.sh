B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/bp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bssn_simple -s 3 -c 3 -o gpurun_out/bp_prof $B > gpurun_out/bp_ncu.log 2>&1

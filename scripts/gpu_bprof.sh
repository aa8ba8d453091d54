B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/bp2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bssn_deriv|bssn_alg" -s 3 -c 3 -o gpurun_out/bp2_prof $B > gpurun_out/bp2_ncu.log 2>&1
tail -2 gpurun_out/bp2_ncu.log

cd $GRAFT_REPO_ROOT
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary"
$B > gpurun_out/p4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/p4_launches.csv $B > gpurun_out/p4_ncu.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:bssn_fused -s 4 -c 1 -o gpurun_out/p4_stage4 $B > gpurun_out/p4_full.log 2>&1; echo "full rc=$?"

timeout 900 python -m pytest tests/test_gpu_bssn_variants.py -x -q > gpurun_out/bh_pytest.log 2>&1; tail -3 gpurun_out/bh_pytest.log
for mb in 3; do
CHEMORA_BSSN_ALG_MB=$mb python bench.py --config bssn192 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 3 > gpurun_out/bh_mb$mb.log 2>&1; echo mb=$mb; tail -1 gpurun_out/bh_mb$mb.log | cut -c100-200
done
B="env CHEMORA_BSSN_ALG_MB=3 python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 3"
$B > gpurun_out/bh_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 12 --csv --log-file gpurun_out/bh_launches.csv $B > gpurun_out/bh_ncu1.log 2>&1

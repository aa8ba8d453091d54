cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config bssn192 --variant 4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2e_b4.log 2>&1; echo "b4 rc=$?"; tail -1 gpurun_out/r2e_b4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('v4', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms frac', round(r['frac'],3), r.get('frac_of_measured_sustained'), d['clocks'])"
timeout 300 python bench.py --config bssn192 --variant 3 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2e_b3.log 2>&1; echo "b3 rc=$?"; tail -1 gpurun_out/r2e_b3.log | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_bssn_variants.py -q > gpurun_out/r2e_var.log 2>&1; echo "var rc=$?"; tail -3 gpurun_out/r2e_var.log
B="python bench.py --config bssn192 --variant 4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-secondary"
$B > gpurun_out/r2e_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:bssn_fused -s 2 -c 1 -o gpurun_out/r2e_bssn4 $B > gpurun_out/r2e_ncu.log 2>&1; echo "ncu rc=$?"

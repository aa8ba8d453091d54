cd $GRAFT_REPO_ROOT
timeout 300 python scripts/dbg_bssn4.py 2>&1 | grep "rel diff"
timeout 300 python bench.py --config bssn192 --variant 4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2f_b4.log 2>&1; echo "b4 rc=$?"; tail -1 gpurun_out/r2f_b4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('v4', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms frac', round(r['frac'],3), r.get('frac_of_measured_sustained'), d['launch_timing'], d['clocks'])"

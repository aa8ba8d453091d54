cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r2c_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2c_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('wave', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms', r['kernel'], 'frac', round(r['frac'],3), 'share', round(r['launch_share_of_step'],3), 'step432', round(r['step_frac_at_432_bytes'],3), 'launches', d['gpu_launches'])
s=d['secondary']['bssn192']; r=s['roofline']; print('bssn', round(s['value']/1e9,3), 'G/s', round(s['ms_per_step'],3), 'ms frac', round(r['frac'],3), r.get('frac_of_measured_sustained'))
print('config0', d['config0']); print('e2e', d['e2e']['value']/1e9, 'cpu', d['cpu_baseline']['value']/1e6, d['clocks'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 2 --e2e-steps 0 --no-secondary > gpurun_out/r2c_bench2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/r2c_bench2.log | cut -c1-300

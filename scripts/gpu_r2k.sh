cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2k_gpu.log 2>&1; echo "gpu rc=$?"; tail -4 gpurun_out/r2k_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2k_smoke.log
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2k_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('wave', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms', r['kernel'], 'frac', round(r['frac'],3), 'step432', round(r['step_frac_at_432_bytes'],3), 'launches', d['gpu_launches'], d['clocks'])
s=d['secondary']['bssn192']; r=s['roofline']; print('bssn', round(s['value']/1e9,3), 'G/s', round(s['ms_per_step'],3), 'ms frac', round(r['frac'],3), r.get('frac_of_measured_sustained'), s['gpu_launches'])
print('e2e', d['e2e']['value']/1e9, 'cpu', d['cpu_baseline']['value']/1e6)"
F="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary"
$F > gpurun_out/r2k_wplain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wave_fused3 -s 2 -c 2 -o gpurun_out/r2k_wave $F > gpurun_out/r2k_wncu.log 2>&1; echo "ncu rc=$?"

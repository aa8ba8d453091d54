# NEXT-1: the wave step at 512^3 for every run-time accuracy order (one bench line each)
for o in 2 4 6 8; do
  timeout 300 python bench.py --fd-order $o --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fdo_$o.log 2>&1
  echo -n "order $o: "; tail -1 gpurun_out/fdo_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms  variant', r['variant'], 'frac', round(r['frac'],3), d['clocks']['reasons'])"
done

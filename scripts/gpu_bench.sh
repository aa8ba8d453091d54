python bench.py > gpurun_out/b3_wave.log 2>&1
python bench.py --config bssn192 --steps 5 --warmup 3 > gpurun_out/b3_bssn.log 2>&1
python bench.py --variant 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b3_wave_v0.log 2>&1

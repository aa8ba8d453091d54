python -m pytest tests/test_gpu_wave.py -x -q -k "fd_order or variants" > gpurun_out/tp_pytest.log 2>&1
tail -1 gpurun_out/tp_pytest.log
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 4"
$B > gpurun_out/tp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wave_tma2 -s 4 -c 2 -o gpurun_out/tp_prof $B > gpurun_out/tp_ncu.log 2>&1

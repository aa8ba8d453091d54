python -m pytest tests/test_gpu_wave.py -x -q > gpurun_out/bz_pytest.log 2>&1; tail -1 gpurun_out/bz_pytest.log
for bz in 1 2 4 8; do for b in -1 0; do
CHEMORA_WAVE_BZ=$bz CHEMORA_WAVE_BAND=$b python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bz_${bz}_${b}.log 2>&1
done; done
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
CHEMORA_WAVE_BZ=4 $B > gpurun_out/bz_plain.log 2>&1 && \
CHEMORA_WAVE_BZ=4 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/bz_launches4.csv $B > gpurun_out/bz_ncu1.log 2>&1

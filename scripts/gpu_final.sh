# round-end evidence: tests, smoke, bench lines, ncu launch lists and one full capture
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; tail -2 gpurun_out/fin_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
python bench.py > gpurun_out/fin_bench_wave.log 2>&1; tail -1 gpurun_out/fin_bench_wave.log | cut -c1-200
python bench.py --config bssn192 > gpurun_out/fin_bench_bssn.log 2>&1; tail -1 gpurun_out/fin_bench_bssn.log | cut -c1-200
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_bench_ref.log 2>&1; tail -1 gpurun_out/fin_bench_ref.log | cut -c1-200
W="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$W > gpurun_out/fin_wplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_wave_launches.csv $W > gpurun_out/fin_wncu.log 2>&1
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/fin_bplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum --clock-control none -c 40 --csv --log-file gpurun_out/fin_bssn_launches.csv $B > gpurun_out/fin_bncu.log 2>&1
F="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
ncu --set full --clock-control none --import-source on -k regex:wave_fused -s 2 -c 2 -o gpurun_out/fin_wave_full $F > gpurun_out/fin_wfull.log 2>&1
echo done

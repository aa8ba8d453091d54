# full GPU check: tests, smoke, benches, BSSN launch list with fp64 counts
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/rd_pytest.log 2>&1; tail -3 gpurun_out/rd_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rd_smoke.log 2>&1; tail -1 gpurun_out/rd_smoke.log
python bench.py > gpurun_out/rd_bench.log 2>&1; tail -1 gpurun_out/rd_bench.log | cut -c1-300
python bench.py --config bssn192 --steps 5 --warmup 3 > gpurun_out/rd_bench_bssn.log 2>&1; tail -1 gpurun_out/rd_bench_bssn.log | cut -c1-300
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$B > gpurun_out/rd_bplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum --clock-control none -c 20 --csv --log-file gpurun_out/rd_bssn_launches.csv $B > gpurun_out/rd_bncu.log 2>&1
echo done

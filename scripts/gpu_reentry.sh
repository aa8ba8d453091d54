# re-entry check of the restored tree: tests, smoke, default bench lines
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/re_pytest.log 2>&1; tail -2 gpurun_out/re_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re_smoke.log 2>&1; tail -1 gpurun_out/re_smoke.log
python bench.py > gpurun_out/re_bench_wave.log 2>&1; tail -1 gpurun_out/re_bench_wave.log | cut -c1-300
python bench.py --config bssn192 > gpurun_out/re_bench_bssn.log 2>&1; tail -1 gpurun_out/re_bench_bssn.log | cut -c1-300
echo done

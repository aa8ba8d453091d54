cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_bssn_variants.py tests/test_gpu_ipc_procs.py tests/test_gpu_bssn.py -q > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2j_tests.log
B="python bench.py --config bssn192 --variant 4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-secondary"
$B > gpurun_out/r2j_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:bssn_fused -s 2 -c 1 -o gpurun_out/r2j_bssn4 $B > gpurun_out/r2j_ncu.log 2>&1; echo "ncu rc=$?"

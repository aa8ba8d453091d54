cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_bssn_variants.py -x -q > gpurun_out/r2d_var.log 2>&1; echo "var rc=$?"; tail -30 gpurun_out/r2d_var.log
timeout 300 python bench.py --config bssn192 --variant 4 --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2d_b4.log 2>&1; echo "b4 rc=$?"; tail -3 gpurun_out/r2d_b4.log | cut -c1-400

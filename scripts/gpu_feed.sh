cd $GRAFT_REPO_ROOT
timeout 300 python scripts/check_bssn_designs.py 2>&1 | grep "rel diff"
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_bssn_variants.py tests/test_gpu_ipc_procs.py -q -x > gpurun_out/feed_t.log 2>&1; echo "t rc=$?"; tail -2 gpurun_out/feed_t.log
bash scripts/ab_swap.sh "--config bssn192 --steps 10 --warmup 3" mon feed

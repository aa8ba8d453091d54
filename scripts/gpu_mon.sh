cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_bssn_variants.py -q -x > gpurun_out/mon_t.log 2>&1; echo "t rc=$?"; tail -2 gpurun_out/mon_t.log
bash scripts/ab_swap.sh "--config bssn192 --steps 10 --warmup 3" nan mon

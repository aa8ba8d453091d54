cd $GRAFT_REPO_ROOT
timeout 300 python scripts/dbg_bssn4.py 2>&1 | grep "rel diff"
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_bssn_variants.py tests/test_gpu_ipc_procs.py tests/test_gpu_bssn.py -q -x > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2i_tests.log
cp paper_1410_1764_b200/libchemora.so ab/libcur.so
bash scripts/ab_swap.sh "--config bssn192 --variant 4 --steps 10 --warmup 3" cur 2gi

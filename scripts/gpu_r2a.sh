cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ipc_procs.py -x -q > gpurun_out/r2a_ipc.log 2>&1; echo "ipc rc=$?"; tail -30 gpurun_out/r2a_ipc.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2a_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/r2a_gpu.log

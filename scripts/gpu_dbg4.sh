cd $GRAFT_REPO_ROOT
cp scripts/libchemora_dbg.so paper_1410_1764_b200/libchemora.so
CUDA_MODULE_LOADING=LAZY timeout 120 python -X faulthandler scripts/dbg_bssn4b.py > gpurun_out/dbg4d.log 2>&1; echo rc=$?; tail -20 gpurun_out/dbg4d.log


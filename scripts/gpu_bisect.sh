cd $GRAFT_REPO_ROOT/scripts
timeout 60 ./capi_bssn4_probe 2>&1 | tail -4
cd ..; timeout 300 python scripts/dbg_bssn4.py 2>&1 | tail -12

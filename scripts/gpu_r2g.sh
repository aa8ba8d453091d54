cd $GRAFT_REPO_ROOT
timeout 300 python scripts/dbg_bssn4.py 2>&1 | grep "rel diff"
bash scripts/ab_swap.sh "--config bssn192 --variant 4 --steps 10 --warmup 3" 2g 3g

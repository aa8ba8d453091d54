cd $GRAFT_REPO_ROOT
cp ab/libprod2.so paper_1410_1764_b200/libchemora.so
timeout 300 python scripts/check_bssn_designs.py 2>&1 | grep "rel diff"
bash scripts/ab_swap.sh "--config bssn192 --steps 10 --warmup 3" nan prod2

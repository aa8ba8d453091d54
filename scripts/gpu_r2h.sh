cd $GRAFT_REPO_ROOT
cp ab/lib2gi.so paper_1410_1764_b200/libchemora.so
timeout 300 python scripts/dbg_bssn4.py 2>&1 | grep "rel diff"
bash scripts/ab_swap.sh "--config bssn192 --variant 4 --steps 10 --warmup 3" 2g 2gi
bash scripts/ab_swap.sh "--config bssn192 --variant 3 --steps 10 --warmup 3" 2gi
B="python bench.py --config bssn192 --variant 4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-secondary"
cp ab/lib2gi.so paper_1410_1764_b200/libchemora.so
$B > gpurun_out/r2h_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:bssn_fused -s 2 -c 1 -o gpurun_out/r2h_bssn4 $B > gpurun_out/r2h_ncu.log 2>&1; echo "ncu rc=$?"

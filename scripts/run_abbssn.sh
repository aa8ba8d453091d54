# A/B of an alternative BSSN build (ab/lib$1.so): design check + BSSN GPU tests, then timing
mkdir -p ab
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig0.so
cp ab/lib$1.so $L
timeout 300 python scripts/check_bssn_designs.py > gpurun_out/chk_$1.log 2>&1; echo "chk rc $?" >> gpurun_out/chk_$1.log
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_bssn.py tests/test_gpu_bssn_variants.py tests/test_gpu_next.py tests/test_gpu_constraints.py > gpurun_out/pt_$1.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_$1.log
cp ab/orig0.so $L
bash scripts/ab_swap.sh "--config bssn192 --steps 10 --warmup 3" cur $1 > gpurun_out/ab_$1.log 2>&1

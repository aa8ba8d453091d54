# ncu --set full of one BSSN fused stage kernel with an alternative build ab/lib$1.so
mkdir -p ab
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig0.so
cp ab/lib$1.so $L
B="python bench.py --config bssn192 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/ncub_$1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bssn_fused -s 6 -c 1 -o gpurun_out/ncub_$1 $B > gpurun_out/ncub_$1.log 2>&1; echo "rc=$?" >> gpurun_out/ncub_$1.log
cp ab/orig0.so $L

# ncu --set full of the wave pair kernels with an alternative build ab/lib$1.so
mkdir -p ab
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig0.so
cp ab/lib$1.so $L
W="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-secondary"
timeout 300 $W > gpurun_out/ncuab_$1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wave_fused3 -s 2 -c 2 -o gpurun_out/ncuab_$1 $W > gpurun_out/ncuab_$1.log 2>&1; echo "rc=$?" >> gpurun_out/ncuab_$1.log
cp ab/orig0.so $L

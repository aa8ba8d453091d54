for v in 0 2 3 4; do for o in 2 4; do timeout 60 python scripts/dbg_order.py $v $o 2>&1 | tail -1; done; done > gpurun_out/ch_dbg.log
for c in 4 8 16 32 64 128; do
CHEMORA_TMA_CHUNK=$c python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --variant 4 > gpurun_out/ch_$c.log 2>&1
done
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --variant 4"
CHEMORA_TMA_CHUNK=8 $B > gpurun_out/ch_plain.log 2>&1 && \
CHEMORA_TMA_CHUNK=8 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/ch_launches8.csv $B > gpurun_out/ch_ncu1.log 2>&1

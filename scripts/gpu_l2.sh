for v in 0 4 6; do for N in 64 256; do
python scripts/l2_probe.py $v $N > gpurun_out/l2_plain_${v}_$N.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -s 12 -c 8 --csv --log-file gpurun_out/l2_${v}_$N.csv python scripts/l2_probe.py $v $N > /dev/null 2>&1
done; done

for v in 0 1 2 3 4; do for o in 2 4 6 8; do timeout 60 python scripts/dbg_order.py $v $o 2>&1 | tail -1; done; done > gpurun_out/dbg.log

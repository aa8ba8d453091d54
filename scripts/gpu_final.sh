# Round-end evidence on one B200 (outputs in gpurun_out/<prefix>_*, summarised in profiles/r2_*):
# tests, smoke, the default bench line (wave 512^3 + BSSN 192^3 secondary + configs[0]), the
# BSSN bench per design, the reference arm, the 2-ranks-on-one-GPU bench, ncu launch lists of
# the bench commands and one ncu --set full capture per dominant kernel.
cd ${GRAFT_REPO_ROOT:-.}
P=${1:-fin2}   # output prefix
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${P}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.log 2>&1; echo "bench rc=$?"
for v in 4 3; do
  timeout 600 python bench.py --config bssn192 --variant $v --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${P}_bssn_v$v.log 2>&1; echo "bssn v$v rc=$?"
done
timeout 900 python bench.py --config bssn384 --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${P}_bssn384.log 2>&1; echo "bssn384 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${P}_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 2 --e2e-steps 0 --no-secondary > gpurun_out/${P}_bench2.log 2>&1; echo "bench2 rc=$?"
W="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary"
$W > gpurun_out/${P}_wplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_wave_launches.csv $W > gpurun_out/${P}_wncu.log 2>&1; echo "wave launches rc=$?"
B="python bench.py --config bssn192 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary"
$B > gpurun_out/${P}_bplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum --clock-control none -c 40 --csv --log-file gpurun_out/${P}_bssn_launches.csv $B > gpurun_out/${P}_bncu.log 2>&1; echo "bssn launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:wave_fused3 -s 2 -c 2 -o gpurun_out/${P}_wave_full $W > gpurun_out/${P}_wfull.log 2>&1; echo "wave full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:bssn_fused -s 2 -c 1 -o gpurun_out/${P}_bssn_full $B > gpurun_out/${P}_bfull.log 2>&1; echo "bssn full rc=$?"
echo done

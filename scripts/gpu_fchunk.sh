for c in 32 64 128 256 512; do
CHEMORA_FUSED_CHUNK=$c python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fc_$c.log 2>&1; echo "chunk=$c $(tail -1 gpurun_out/fc_$c.log | cut -c100-160)"
done

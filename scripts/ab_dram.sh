# Same-box A/B of alternative builds with their DRAM traffic: timing (two interleaved rounds,
# scripts/ab_swap.sh) then one ncu launch list (time + DRAM bytes) per build.
# usage: bash scripts/ab_dram.sh "<bench args>" A B ...
mkdir -p ab
ARGS="$1"; shift
bash scripts/ab_swap.sh "$ARGS" "$@"
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig1.so
for v in "$@"; do
  cp ab/lib$v.so $L
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/abd_$v.csv python bench.py $ARGS --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  python - "$v" <<'PY'
import sys; sys.path.insert(0, "scripts")
from traffic_from_ncu import launches, dram
v = sys.argv[1]
for _, n, m in launches(f"gpurun_out/abd_{v}.csv")[-8:]:
    if "init" in n: continue
    print(v, n.split("(")[0][-24:], "%.2f GB %.3f ms" % (dram(m) / 1e9, m.get("gpu__time_duration.sum", 0) / 1e6))
PY
done
cp ab/orig1.so $L

# Same-box A/B of alternative builds of libchemora.so (box-to-box spread is ~3 %, so
# variants are compared inside one gpurun call, interleaved, two rounds).
# Usage (on the GPU box):  bash scripts/ab_swap.sh "<bench args>" A B C ...
#   each name X refers to ab/libX.so (build it here: edit, build, cp the .so to ab/libX.so;
#   ab/ is git-ignored but travels with the gpurun snapshot).
mkdir -p ab
ARGS="$1"; shift
L=paper_1410_1764_b200/libchemora.so
cp $L ab/orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp ab/lib$v.so $L
    echo -n "$v "
    timeout 120 python bench.py $ARGS --no-cpu-baseline --e2e-steps 0 | \
      python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms_per_step'])"
  done
done
cp ab/orig.so $L

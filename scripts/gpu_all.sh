timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/all2_pytest.log 2>&1; tail -3 gpurun_out/all2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/all2_smoke.log 2>&1; tail -1 gpurun_out/all2_smoke.log
python bench.py > gpurun_out/all2_bench.log 2>&1
python bench.py --config bssn192 --steps 5 --warmup 3 > gpurun_out/all2_bench_bssn.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/all2_ref.log 2>&1
python -c "
import math, paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C
n=(512,512,512); h=tuple(2*math.pi/v for v in n)
g=P.Grid(C.SYS_WAVE,n,h); g.set_initial(C.INIT_PLANE_WAVES)
print(g.autotune(trials=2))
" > gpurun_out/all2_autotune.log 2>&1

"""Host<->device copy rates for the e2e path: contiguous pinned copies vs the library's
strided (padded-layout) upload/download of a 512^3 wave state."""
import torch, time, sys
sys.path.insert(0, ".")
import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C

def t(fn, s, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

n = 512
nb = 5 * n ** 3 * 8
h = torch.empty(5, n, n, n, dtype=torch.float64).pin_memory()
h2 = torch.empty(5, n, n, n, dtype=torch.float64).pin_memory()
d = torch.empty(5, n, n, n, dtype=torch.float64, device="cuda")
d2 = torch.empty(5, n, n, n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
s2 = torch.cuda.Stream()
ms = t(lambda: d.copy_(h, non_blocking=True), s); print(f"H2D contiguous {nb/ms/1e6:.1f} GB/s ({ms:.1f} ms)")
ms = t(lambda: h.copy_(d, non_blocking=True), s); print(f"D2H contiguous {nb/ms/1e6:.1f} GB/s ({ms:.1f} ms)")
def both():
    ev = torch.cuda.Event(); ev.record(s)
    s2.wait_event(ev)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    d.copy_(h, non_blocking=True)
    ev2 = torch.cuda.Event(); ev2.record(s2); s.wait_event(ev2)
ms = t(both, s); print(f"H2D || D2H contiguous {2*nb/ms/1e6:.1f} GB/s total ({ms:.1f} ms)")
del d2
L = 2 * 3.141592653589793
g = P.Grid(C.SYS_WAVE, (n, n, n), (L / n,) * 3)
g.set_initial(C.INIT_PLANE_WAVES, seed=1)
ms = t(lambda: g.upload_state(h), s); print(f"upload_state (strided + halo) {nb/ms/1e6:.1f} GB/s ({ms:.1f} ms)")
ms = t(lambda: g.download_state(h), s); print(f"download_state (strided) {nb/ms/1e6:.1f} GB/s ({ms:.1f} ms)")

"""Where the host-buffer ktruss time goes (R-MAT s20, a K sample): wall time
of kt.ktruss vs the engine path split into load / fixpoint / extract."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
n, slots = g.num_vertices, g.total_slots()
keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32, pin_memory=True))
keep[0].numpy().view(np.uint32)[:] = g.row_ptr; keep[1].numpy().view(np.uint32)[:] = g.col_idx
hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
ks = list(range(3, 305, 15))
kt.ktruss(hg, 3)
tot = 0.0
for k in ks:
    torch.cuda.synchronize(); t = time.perf_counter(); r = kt.ktruss(hg, k); torch.cuda.synchronize()
    tot += time.perf_counter() - t
print(f"ktruss wall per K {1e3 * tot / len(ks):.2f} ms")
e = kt.Engine()
lt = rt = dt = xt = 0.0
for k in ks:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e.load(hg); torch.cuda.synchronize(); t1 = time.perf_counter()
    e.run(k); t2 = time.perf_counter(); dt += e.info()["device_ms"]
    x = e.extract(); t3 = time.perf_counter()
    lt += t1 - t0; rt += t2 - t1; xt += t3 - t2
m = len(ks)
print(f"engine: load {1e3*lt/m:.2f}  run {1e3*rt/m:.2f} (device {dt/m:.2f})  extract {1e3*xt/m:.2f} ms per K")
t = time.perf_counter()
for _ in range(20):
    a = [torch.empty(slots, dtype=torch.int32, pin_memory=True) for _ in range(3)]
print(f"3x pinned alloc {1e3*(time.perf_counter()-t)/20:.3f} ms")

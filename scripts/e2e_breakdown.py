import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
n, slots = g.num_vertices, g.total_slots()
keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32, pin_memory=True))
keep[0].numpy().view(np.uint32)[:] = g.row_ptr; keep[1].numpy().view(np.uint32)[:] = g.col_idx
hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
for k in (3, 18, 304):
    kt.ktruss(hg, k)
    t = time.perf_counter(); r = kt.ktruss(hg, k); t1 = time.perf_counter()
    e = kt.Engine()
    t2 = time.perf_counter(); e.load(hg); torch.cuda.synchronize(); t3 = time.perf_counter()
    e.run(k); t4 = time.perf_counter(); x = e.extract(); t5 = time.perf_counter()
    print(f"k={k} ktruss_total={1e3*(t1-t):.1f}ms | engine load={1e3*(t3-t2):.1f} run={1e3*(t4-t3):.1f} (dev {e.info()['device_ms']:.1f}) extract={1e3*(t5-t4):.1f} edges={len(x)}", flush=True)
    e.close()

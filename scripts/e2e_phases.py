"""Per-phase wall times of kt.ktruss (KTG_LOAD_TIMING=1 prints the engine's
phases; this adds the Python wall time around each call).
  python scripts/e2e_phases.py [scale] [k ...]"""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2009_07929_b200 as kt
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ks = [int(x) for x in sys.argv[2:]] or [3, 18, 100, 304]
cache = f"/tmp/ktg_s{scale}.ztcsr"
g = kt.graph.read_csr_cache(cache) if os.path.exists(cache) else kt.rmat(scale)
n, slots = g.num_vertices, g.total_slots()
keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32, pin_memory=True))
keep[0].numpy().view(np.uint32)[:] = g.row_ptr; keep[1].numpy().view(np.uint32)[:] = g.col_idx
hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
r = kt.ktruss(hg, 3)
for k in ks:
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); r = None; r = kt.ktruss(hg, k); torch.cuda.synchronize()
        print(f"k={k} ktruss wall {1e3 * (time.perf_counter() - t):.2f} ms, {len(r)} edges", file=sys.stderr, flush=True)

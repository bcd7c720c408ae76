"""Two host-buffer loads of R-MAT s20 into one engine (the second reuses every
buffer, as the cached host-API engine does); run under an ncu launch list to
see the load path's kernels."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2009_07929_b200 as kt
g = kt.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
n, slots = g.num_vertices, g.total_slots()
keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32, pin_memory=True))
keep[0].numpy().view(np.uint32)[:] = g.row_ptr; keep[1].numpy().view(np.uint32)[:] = g.col_idx
hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
e = kt.Engine()
for _ in range(2):
    e.load(hg)
    torch.cuda.synchronize()
print("loaded")

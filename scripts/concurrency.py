"""Device-resident sweep (every K from pristine) with P engines on P streams
running K values concurrently; also the host-buffer sweep from P threads."""
import sys, threading, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
ks = list(range(3, 305))
PS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4]
for P in PS:
    streams = [torch.cuda.Stream() for _ in range(P)]
    engs = [kt.Engine(g, stream=s.cuda_stream) for s in streams]
    def sweep():
        for i, k in enumerate(ks):
            e = engs[i % P]
            e.reset(); e.run(k, sync=False)
    sweep(); torch.cuda.synchronize()
    t = time.perf_counter(); sweep(); torch.cuda.synchronize(); ms = (time.perf_counter() - t) * 1e3
    print(f"device sweep P={P}: {ms:.1f} ms ({len(ks) * g.num_edges / ms / 1e6:.3e} edges/s)", flush=True)
    for e in engs: e.close()
n, slots = g.num_vertices, g.total_slots()
keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32, pin_memory=True))
keep[0].numpy().view(np.uint32)[:] = g.row_ptr; keep[1].numpy().view(np.uint32)[:] = g.col_idx
hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
for T in ((1, 2, 4) if len(sys.argv) <= 2 else [int(x) for x in sys.argv[2].split(",") if x]):
    def work(part):
        for k in part:
            r = kt.ktruss(hg, k)
    parts = [ks[i::T] for i in range(T)]
    th = [threading.Thread(target=work, args=([p[0]],)) for p in parts]  # warm per-thread engines
    for x in th: x.start()
    for x in th: x.join()
    t = time.perf_counter()
    th = [threading.Thread(target=work, args=(p,)) for p in parts]
    for x in th: x.start()
    for x in th: x.join()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3
    print(f"e2e sweep T={T}: {ms:.1f} ms ({len(ks) * g.num_edges / ms / 1e6:.3e} edges/s)", flush=True)

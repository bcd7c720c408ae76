"""Host-buffer sweep from T threads: per-call wall time per thread, to see
what serialises (per-thread cached engines, pooled pinned results)."""
import sys, threading, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
n, slots = g.num_vertices, g.total_slots()
keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32, pin_memory=True))
keep[0].numpy().view(np.uint32)[:] = g.row_ptr; keep[1].numpy().view(np.uint32)[:] = g.col_idx
hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
ks = list(range(3, 305, 3))
for T in (1, 2, 3):
    stats = [[] for _ in range(T)]
    parts = [ks[i::T] for i in range(T)]
    bar = threading.Barrier(T + 1)
    def work(i):
        for k in parts[i][:2]:  # warm this thread's cached engine and the result pool
            kt.ktruss(hg, k)
        torch.cuda.synchronize()
        bar.wait(); bar.wait()
        for k in parts[i]:
            t = time.perf_counter(); r = kt.ktruss(hg, k); stats[i].append((time.perf_counter() - t) * 1e3)
    th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
    for x in th: x.start()
    bar.wait()
    t = time.perf_counter()
    bar.wait()
    for x in th: x.join()
    ms = (time.perf_counter() - t) * 1e3
    print(f"T={T}: total {ms:.0f} ms; per-call mean by thread: " +
          ", ".join(f"{np.mean(s):.2f}" for s in stats) + f"; sum of calls {sum(map(sum, stats)):.0f}", flush=True)

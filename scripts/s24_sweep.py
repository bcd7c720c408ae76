"""North-star workload: R-MAT s24 K sweep 3..K_max on one B200, every K from
the pristine graph (4 resident engines on their own streams, as bench.py),
plus the incremental sweep; survivors per K are recorded and the sweep's
K_max+1 truss must be empty."""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2009_07929_b200 as kt
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = kt.rmat(scale)
streams = [torch.cuda.Stream() for _ in range(4)]
engs = [kt.Engine(g, stream=s.cuda_stream) for s in streams]
kmax = engs[0].kmax()
ks = list(range(3, kmax + 1))
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(streams[0])
for s in streams[1:]:
    s.wait_event(e0)
for i, k in enumerate(ks):
    e = engs[i % 4]
    e.reset(); e.run(k, sync=False)
for s in streams[1:]:
    d = torch.cuda.Event(); d.record(s); streams[0].wait_event(d)
e1.record(streams[0]); e1.synchronize()
ms = e0.elapsed_time(e1)
m = g.num_edges
print(f"s{scale} pristine sweep K=3..{kmax}: {ms/1e3:.2f} s, {len(ks)*m/(ms/1e3):.3e} edges/s", flush=True)
e = engs[0]
e.reset()
t = time.perf_counter()
live = {}
for k in ks + [kmax + 1]:
    e.run(k)
    live[k] = e.info()["live_edges"]
torch.cuda.synchronize()
inc_s = time.perf_counter() - t
print(f"s{scale} incremental sweep: {inc_s:.2f} s; live[3]={live[3]} live[kmax]={live[kmax]} live[kmax+1]={live[kmax+1]}",
      flush=True)
json.dump({"scale": scale, "kmax": kmax, "pristine_sweep_s": ms / 1e3, "edges_per_s": len(ks) * m / (ms / 1e3),
           "incremental_sweep_s": inc_s, "live_kmax": live[kmax], "live_kmax_plus_1": live[kmax + 1],
           "live_per_k": live}, open(f"gpurun_out/s{scale}_sweep.json", "w"))

"""Scratch timing: device-resident fixpoint at a few scales (CUDA events)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt

for scale in [int(x) for x in (sys.argv[1:] or ["16", "18", "20"])]:
    t = time.time()
    g = kt.rmat(scale)
    tg = time.time() - t
    e = kt.Engine(g)
    for k in (3,):
        e.reset(); h = e.run(k)
        ts = []
        for _ in range(3):
            e.reset(); h = e.run(k); ts.append(e.info()["device_ms"])
        info = e.info()
        print(f"s{scale} gen {tg:.1f}s m={g.num_edges} k={k} iters={len(h)} hist={h[:4]} "
              f"ms={min(ts):.3f} ME/s={g.num_edges/min(ts)/1e3:.1f} tri={info['triangles']} live={info['live_edges']}", flush=True)
    e.reset(); tri = e.support_pass(); 
    print(f"  support_pass tri={tri} maxS={e.info()['max_support']}", flush=True)

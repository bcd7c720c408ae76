"""Per-round live edges, L_r, triangles and support time for a few K (s20)."""
import os, sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(int(os.environ.get("SCALE", "20")))
ew = kt.Engine(g, collect_work=True)
et = kt.Engine(g, time_support=True)
for k in [int(x) for x in sys.argv[1:]] or [18, 304]:
    ew.reset(); ew.run(k); w = ew.round_work()
    et.reset(); et.run(k); t = et.round_work()
    print(f"k={k}")
    for i, (a, b) in enumerate(zip(w, t)):
        print(f"  r{i:2d} live={a['live_edges']:9d} L={a['L']:12d} tri={a['triangles']:11d} removed={a['removed']:9d} sup_ms={b['support_ms']:.3f}")

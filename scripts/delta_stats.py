"""Per-round carried-support statistics (s20): removed, full pass or not,
delta cost, keep cost, queued long-intersection pieces, support time."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
e = kt.Engine(g, time_support=True)
for k in [int(x) for x in sys.argv[1:]] or [10, 60, 150, 304]:
    e.reset(); e.run(k); w = e.round_work()
    print(f"k={k}")
    for i, r in enumerate(w):
        print(f"  r{i:2d} live={r['live_edges']:9d} removed={r['removed']:9d} full={r['full_pass']} carried={r['carried']} "
              f"dcost={r['delta_cost']:11d} kcost={r['keep_cost']:11d} pieces={r['delta_pieces']:7d} sup_ms={r['support_ms']:.3f}")

"""R-MAT s24 fixpoint device times at a few K (KTG_LIB_DIR selects the build)."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
e = kt.Engine(g)
tot = 0.0
for k in (3, 10, 30, 100, 300, 935):
    ts = []
    for _ in range(2):
        e.reset(); h = e.run(k); ts.append(e.info()["device_ms"])
    tot += min(ts)
    print(f"s24 k={k} rounds={len(h)} ms={min(ts):.1f} live={e.info()['live_edges']}", flush=True)
print(f"s24 sum ms={tot:.1f}")

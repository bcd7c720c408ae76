"""A/B timing of the headline path (KTG_LIB_DIR selects the build): best-of-5
full-pass k_support_a22 time (no degree bound, host loop + CUDA events) and
the device-resident fixpoint time at a few K, R-MAT s20."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
e = kt.Engine(g, kt.TrussOptions(no_degree_bound=True), time_support=True)
for k in (3, 60, 304):
    best = [1e9] * 2
    for _ in range(5):
        e.reset(); e.run(k); w = e.round_work()
        for i in range(min(2, len(w))):
            if w[i]["full_pass"]:
                best[i] = min(best[i], w[i]["support_ms"])
    print(f"a22 k={k} full-pass ms rounds 0-1: " + " ".join(f"{b:.3f}" for b in best), flush=True)
e.close()
e = kt.Engine(g)
tot = 0.0
for k in (3, 10, 30, 60, 100, 200, 304):
    ts = []
    for _ in range(3):
        e.reset(); e.run(k); ts.append(e.info()["device_ms"])
    tot += min(ts)
    print(f"fixpoint k={k} ms={min(ts):.3f}", flush=True)
print(f"fixpoint sum ms={tot:.3f}")

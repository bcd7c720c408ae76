"""Round-0 support kernel time (s20, host loop + CUDA events), best of 5."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
e = kt.Engine(g, kt.TrussOptions(recompute=True), time_support=True)
for k in (3, 60, 304):
    best = [1e9] * 3
    for _ in range(5):
        e.reset(); e.run(k); w = e.round_work()
        for i in range(min(3, len(w))):
            best[i] = min(best[i], w[i]["support_ms"])
    print(f"k={k} support ms rounds 0-2: " + " ".join(f"{b:.3f}" for b in best), flush=True)

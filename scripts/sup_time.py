"""Round-0 support kernel time (s20, host loop + CUDA events), best of 5:
A22-staged pass (carried-support engine) vs k_support_chunked (recompute)."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
for name, opts in (("a22", kt.TrussOptions(no_degree_bound=True)), ("chunked", kt.TrussOptions(recompute=True))):
    e = kt.Engine(g, opts, time_support=True)
    for k in (3, 60, 304):
        best = [1e9] * 3
        for _ in range(5):
            e.reset(); e.run(k); w = e.round_work()
            for i in range(min(3, len(w))):
                if w[i]["full_pass"]:
                    best[i] = min(best[i], w[i]["support_ms"])
        print(f"{name} k={k} support ms rounds 0-2 (full passes): " + " ".join(f"{b:.3f}" for b in best), flush=True)
    e.close()

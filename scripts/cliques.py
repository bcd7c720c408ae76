"""BASELINE configs[4]: R-MAT + planted cliques (128, 256, 512, 1024), deep
K_max, on one B200 (the config names 8 GPUs; the graph is replicated per GPU
anyway, so one GPU shows the per-GPU working set).

  python scripts/cliques.py 26 32      # the full s26/ef32 config

Generation, K_max by kmax_search (binary search from pristine), K=3 and the
K_max fixpoint timed, K_max + 1 empty, and a CPU soundness check of the K_max
truss: its edges rebuilt into a CSR and the oracle's compute_supports over
that subgraph must give every edge S >= K_max - 2 (the truss property) and
exactly the engine's supports."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2009_07929_b200 as kt
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 32
t = time.time()
g = kt.rmat_cliques(scale, ef, 42)
gen = time.time() - t
print(f"gen s{scale}/ef{ef}+cliques: {gen:.1f}s n={g.num_vertices} m={g.num_edges} slots={g.total_slots()}", flush=True)
t = time.time()
e = kt.Engine(g)
load = time.time() - t
e.reset()
tri = e.support_pass()
info = e.info()
print(f"load {load:.1f}s carried={info['carried']} T={tri} maxS={info['max_support']}", flush=True)
t = time.time()
km = e.kmax()
print(f"kmax={km} ({time.time()-t:.1f}s, binary search from pristine)", flush=True)
out = {"scale": scale, "ef": ef, "n": g.num_vertices, "m": g.num_edges, "slots": g.total_slots(), "kmax": km,
       "gen_s": gen, "load_s": load, "carried_mode": bool(info["carried"]), "triangles": tri,
       "max_support": info["max_support"]}
for k in (3, km, km + 1):
    ts = []
    for _ in range(2):
        e.reset(); h = e.run(k); ts.append(e.info()["device_ms"])
    print(f"K={k}: rounds={len(h)} ms={min(ts):.1f} survivors={e.info()['live_edges']} "
          f"edges/s={g.num_edges / (min(ts) / 1e3):.3e}", flush=True)
    out[f"k{k}"] = {"rounds": len(h), "ms": min(ts), "survivors": e.info()["live_edges"], "hist_head": h[:8]}
assert out[f"k{km + 1}"]["survivors"] == 0 and out[f"k{km}"]["survivors"] > 0
# soundness of the K_max truss on the CPU oracle
e.reset(); e.run(km)
r = e.extract()
edges = r.edges
sub = oracle.ref().canonicalize(edges[:, :2].astype(np.uint64))
S = np.zeros(sub.total_slots(), np.uint32)
tri_sub, S = oracle.port().compute_supports(sub, S, threads=16)
live = sub.col_idx != 0
ok_truss = bool(S[live].min() >= km - 2)
# canonicalize relabels; the multiset of supports must match the engine's
ok_sup = bool(np.array_equal(np.sort(S[live]), np.sort(edges[:, 2])))
out["kmax_truss_soundness"] = {"edges": int(len(edges)), "min_support_cpu": int(S[live].min()),
                               "truss_property": ok_truss, "supports_match_cpu": ok_sup}
print("soundness", out["kmax_truss_soundness"], flush=True)
json.dump(out, open(f"gpurun_out/cliques_s{scale}_ef{ef}.json", "w"), indent=1)

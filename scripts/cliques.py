"""BASELINE configs[4] at a single-GPU scale: R-MAT + planted cliques
(128, 256, 512, 1024), deep K_max. Generation, known-answer K_max >= 1024,
the K_max fixpoint and K=3 on one B200 (the full s26/ef32 config is an
8-GPU workload)."""
import json, sys, time
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 32
t = time.time()
g = kt.rmat_cliques(scale, ef, 42)
gen = time.time() - t
print(f"gen s{scale}/ef{ef}+cliques: {gen:.1f}s n={g.num_vertices} m={g.num_edges} slots={g.total_slots()}", flush=True)
e = kt.Engine(g)
t = time.time()
km = e.kmax()
print(f"kmax={km} ({time.time()-t:.1f}s, binary search from pristine)", flush=True)
out = {"scale": scale, "ef": ef, "n": g.num_vertices, "m": g.num_edges, "slots": g.total_slots(), "kmax": km,
       "gen_s": gen}
for k in (3, 100, 512, km):
    ts = []
    for _ in range(2):
        e.reset(); h = e.run(k); ts.append(e.info()["device_ms"])
    print(f"K={k}: rounds={len(h)} ms={min(ts):.1f} survivors={e.info()['live_edges']} "
          f"edges/s={g.num_edges / (min(ts) / 1e3):.3e}", flush=True)
    out[f"k{k}"] = {"rounds": len(h), "ms": min(ts), "survivors": e.info()["live_edges"]}
json.dump(out, open(f"gpurun_out/cliques_s{scale}_ef{ef}.json", "w"), indent=1)

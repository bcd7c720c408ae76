"""A/B of engine builds at the north-star size (KTG_LIB_DIR selects the
build): full-pass k_support_a22 time (K=3 round 0, no degree bound, CUDA
events) and device-resident fixpoint times at K=3 / K=935, best of 3.
The graph is cached (ZTCSR1) at --cache so several builds share one
generation."""
import argparse, json, os, sys, time
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--graph", default="rmat", choices=["rmat", "er"])
ap.add_argument("--cache", default="/tmp/ktg_s24.ztcsr")
ap.add_argument("--ks", default="3,935")
ap.add_argument("--tag", default=os.environ.get("KTG_LIB_DIR", "lib"))
ap.add_argument("--recompute", action="store_true", help="KTG_FLAG_RECOMPUTE engines (k_support_chunked)")
a = ap.parse_args()
if not os.path.exists(a.cache):
    g = kt.rmat(a.scale) if a.graph == "rmat" else kt.erdos_renyi(a.scale, 16 << a.scale)
    kt.graph.write_csr_cache(g, a.cache)
g = kt.graph.read_csr_cache(a.cache)
out = {"tag": a.tag, "graph": f"{a.graph}{a.scale}"}
e = kt.Engine(g, kt.TrussOptions(recompute=True) if a.recompute else kt.TrussOptions(no_degree_bound=True),
              time_support=True)
best = 1e9
for _ in range(3):
    e.reset(); e.run(3)
    w = e.round_work()
    best = min(best, w[0]["support_ms"])
out["a22_full_pass_ms" if not a.recompute else "chunked_pass_ms"] = round(best, 3)
e.close()
e = kt.Engine(g, kt.TrussOptions(recompute=True) if a.recompute else None)
for k in map(int, a.ks.split(",")):
    ts = []
    for _ in range(3):
        e.reset(); h = e.run(k); ts.append(e.info()["device_ms"])
    out[f"k{k}_ms"] = round(min(ts), 3)
    out[f"k{k}_rounds"] = len(h)
    out[f"k{k}_live"] = int(e.info()["live_edges"])
print(json.dumps(out), flush=True)

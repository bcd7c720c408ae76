"""North-star config: R-MAT scale-24 ef16 on one B200.
Checks the survey's known answers, times K=3 and the K_max fixpoint, and
the per-round support work/time for the roofline."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2009_07929_b200 as kt

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
t = time.time()
g = kt.rmat(scale)
print(f"gen s{scale}: {time.time()-t:.1f}s n={g.num_vertices} m={g.num_edges} slots={g.total_slots()}", flush=True)
if "--a22" in sys.argv:
    # the default path's support kernel (k_support_a22, carried supports) on
    # its full passes, without the round-0 degree bound so round 0 is a
    # whole pass; one engine records both the work and the kernel times
    ea = kt.Engine(g, kt.TrussOptions(no_degree_bound=True), collect_work=True, time_support=True)
    res = {}
    for k in (3, 10, 100, 935):
        ea.reset(); ea.run(k); w = ea.round_work()
        full = [x for x in w if x["full_pass"]]
        B = sum(4*x["L"] + 4*g.total_slots() + 4*(g.num_vertices+2) + 12*x["triangles"] for x in full)
        X = sum(4*x["L_tail"] + 4*g.total_slots() + 8*x["live_edges"] + 8*(g.num_vertices+2) + 12*x["triangles"]
                for x in full)
        T = sum(x["support_ms"] for x in full)
        print(f"K={k} a22 full passes: {len(full)} ms={T:.1f} algorithmic={B/1e9:.0f}GB -> {B/T/1e6:.0f} GB/s; "
              f"executed={X/1e9:.0f}GB -> {X/T/1e6:.0f} GB/s", flush=True)
        res[k] = {"full_passes": len(full), "ms": T, "alg_GBps": B / T / 1e6, "exec_GBps": X / T / 1e6}
    json.dump(res, open(f"gpurun_out/s{scale}_a22.json", "w"), indent=1)
    sys.exit(0)
t = time.time()
e = kt.Engine(g)
print(f"load+reorient: {time.time()-t:.1f}s", flush=True)
e.reset()
tri = e.support_pass()
print(f"support pass: T={tri} maxS={e.info()['max_support']}", flush=True)
out = {"scale": scale, "n": g.num_vertices, "m": g.num_edges, "triangles": tri, "max_support": e.info()["max_support"]}
for k in (3, 10, 100, 935):
    e.reset(); h = e.run(k)
    ms = []
    for _ in range(2):
        e.reset(); h = e.run(k); ms.append(e.info()["device_ms"])
    print(f"K={k}: rounds={len(h)} hist={h[:3]} ms={min(ms):.1f} survivors={e.info()['live_edges']} T={e.info()['triangles']}", flush=True)
    out[f"k{k}_ms"] = min(ms); out[f"k{k}_hist"] = h; out[f"k{k}_survivors"] = e.info()["live_edges"]
er = kt.Engine(g, kt.TrussOptions(recompute=True))
for k in (3, 935):
    er.reset(); hr = er.run(k)
    print(f"recompute K={k}: rounds={len(hr)} ms={er.info()['device_ms']:.1f} survivors={er.info()['live_edges']}", flush=True)
    out[f"k{k}_recompute_ms"] = er.info()["device_ms"]
er.close()
t = time.time()
km = e.kmax()
print(f"kmax={km} ({time.time()-t:.1f}s) survivors={e.info()['live_edges']}", flush=True)
e.reset(); h = e.run(km)
print(f"K_max fixpoint: rounds={len(h)} ms={e.info()['device_ms']:.1f}", flush=True)
out.update({"kmax": km, "kmax_rounds": len(h), "kmax_ms": e.info()["device_ms"], "kmax_survivors": e.info()["live_edges"]})
e.close()
ew = kt.Engine(g, kt.TrussOptions(recompute=True), collect_work=True)
et = kt.Engine(g, kt.TrussOptions(recompute=True), time_support=True)
for k in (3, km):
    ew.reset(); ew.run(k); w = ew.round_work(); et.reset(); et.run(k); tw = et.round_work()
    B = sum(4*x["L"] + 4*g.total_slots() + 4*(g.num_vertices+2) + 12*x["triangles"] for x in w)
    T = sum(x["support_ms"] for x in tw)
    print(f"K={k} support: rounds={len(w)} L={[x['L'] for x in w][:3]} bytes={B/1e9:.1f}GB ms={T:.1f} -> {B/T/1e6:.0f} GB/s", flush=True)
    out[f"k{k}_support_GBps"] = B / T / 1e6
json.dump(out, open(f"gpurun_out/s{scale}.json", "w"), indent=1)

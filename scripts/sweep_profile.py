"""Per-K fixpoint time over the s20 sweep + per-round (live, removed, support ms)
for a few K: where the sweep's time goes."""
import os, sys, json
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
scale = int(os.environ.get("SCALE", "20"))
g = kt.rmat(scale)
eng = kt.Engine(g)
kmax = eng.kmax()
out = {"per_k": []}
for k in range(3, kmax + 1):
    eng.reset(); h = eng.run(k)
    inf = eng.info()
    out["per_k"].append((k, len(h), round(inf["device_ms"], 3)))
tot = sum(x[2] for x in out["per_k"])
print("kmax", kmax, "total ms", tot)
buckets = {}
for k, r, ms in out["per_k"]:
    b = min(k // 20 * 20, 300)
    buckets.setdefault(b, [0, 0, 0.0]); buckets[b][0] += 1; buckets[b][1] += r; buckets[b][2] += ms
for b, (n, r, ms) in sorted(buckets.items()):
    print(f"K {b:3d}-{b+19:3d}: nK={n:3d} rounds={r:5d} ms={ms:9.1f} ({100*ms/tot:4.1f}%)")
et = kt.Engine(g, time_support=True, collect_work=True)
for k in [int(x) for x in sys.argv[1:]] or [3, 10, 30, 60, 120, 304]:
    et.reset(); et.run(k); t = et.round_work()
    print(f"k={k}")
    for i, a in enumerate(t):
        print(f"  r{i:2d} live={a['live_edges']:9d} L={a['L']:12d} tri={a['triangles']:11d} removed={a['removed']:9d} sup_ms={a['support_ms']:.3f}")
json.dump(out, open("gpurun_out/sweep_profile.json", "w"))

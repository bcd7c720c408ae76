"""Profiling driver: host-driven loop (kernels launched individually so ncu can
see them; conditional-graph kernel nodes are not profilable)."""
import argparse, sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--k", type=int, nargs="+", default=[3])
ap.add_argument("--naive", action="store_true")
a = ap.parse_args()
g = kt.rmat(a.scale)
e = kt.Engine(g, kt.TrussOptions(host_loop=True, naive_support=a.naive))
for k in a.k:
    e.reset()
    h = e.run(k)
    print(f"s{a.scale} k={k} rounds={len(h)} live={e.info()['live_edges']} ms={e.info()['device_ms']:.2f}", flush=True)

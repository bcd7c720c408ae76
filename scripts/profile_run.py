"""Profiling driver: host-driven loop (kernels launched individually so ncu can
see them; conditional-graph kernel nodes are not profilable).

  python scripts/profile_run.py --graph rmat --scale 24 --k 3
  python scripts/profile_run.py --graph er --scale 22 --k 3
"""
import argparse, sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt

ap = argparse.ArgumentParser()
ap.add_argument("--graph", default="rmat", choices=["rmat", "er"])
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--k", type=int, nargs="+", default=[3])
ap.add_argument("--naive", action="store_true")
ap.add_argument("--no-degree-bound", action="store_true")
a = ap.parse_args()
g = kt.erdos_renyi(a.scale, a.ef << a.scale) if a.graph == "er" else kt.rmat(a.scale, a.ef)
e = kt.Engine(g, kt.TrussOptions(host_loop=True, naive_support=a.naive, no_degree_bound=a.no_degree_bound))
for k in a.k:
    e.reset()
    h = e.run(k)
    print(f"{a.graph} s{a.scale} k={k} rounds={len(h)} live={e.info()['live_edges']} ms={e.info()['device_ms']:.2f}",
          flush=True)

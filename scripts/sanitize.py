"""Driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
small R-MAT graphs through every engine mode, checked against the oracle so
a sanitizer run is also a parity run. Host loop (kernels launched one by one:
the sanitizers do not instrument conditional-graph bodies as reliably).

  compute-sanitizer --tool racecheck python scripts/sanitize.py --mode all
"""
import argparse, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2009_07929_b200 as kt

MODES = {
    "inc": dict(host_loop=True),
    "inc_graph": dict(),
    "recompute": dict(recompute=True, host_loop=True),
    "recompute_graph": dict(recompute=True),
    "label": dict(label_order=True, host_loop=True),
    "naive": dict(label_order=True, naive_support=True, host_loop=True),
}

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="all")
ap.add_argument("--scale", type=int, default=11)
ap.add_argument("--ks", default="3,5,9,20")
ap.add_argument("--no-api", action="store_true", help="skip the host-buffer ktruss / kmax_search calls")
a = ap.parse_args()
port = oracle.port()
modes = list(MODES) if a.mode == "all" else a.mode.split(",")
ks = [int(x) for x in a.ks.split(",")]
bad = 0
for seed in (1, 2):
    g = kt.rmat(a.scale, 16, seed=seed)
    for mode in modes:
        e = kt.Engine(g, kt.TrussOptions(**MODES[mode]))
        for k in ks:
            e.reset()
            hist = e.run(k)
            col, S = e.read()
            ce, Se, he = port.run_fixpoint(g, k, threads=4)
            ok = hist == he and np.array_equal(col, ce) and np.array_equal(S, Se)
            bad += not ok
            print(f"seed={seed} mode={mode} k={k} rounds={len(hist)} parity={'ok' if ok else 'FAIL'}", flush=True)
        e.close()
    if not a.no_api:
        r = kt.ktruss(g, 4)
        km = kt.kmax_search(g)
        print(f"seed={seed} ktruss(4)={len(r)} kmax={km.k_max}", flush=True)
print("PARITY", "FAIL" if bad else "OK")
sys.exit(1 if bad else 0)

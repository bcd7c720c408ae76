"""Fixpoint time per K under different carry/recompute cost ratios
(KTG_DELTA_RATIO), to calibrate delta_round's cost model."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
cache = os.environ.get("CACHE")
if cache and os.path.exists(cache):
    g = kt.graph.read_csr_cache(cache)
else:
    g = kt.rmat(int(os.environ.get("SCALE", "20")))
    if cache:
        kt.graph.write_csr_cache(g, cache)
ks = [3, 5, 10, 20, 30, 45, 60, 80, 100, 110, 120, 135, 150, 165, 180, 200, 215, 230, 260, 304]
if os.environ.get("KS"):
    ks = [int(x) for x in os.environ["KS"].split(",")]
# RATIO_VAR=KTG_DELTA_RATIO0 scans round 0 from pristine only
var = os.environ.get("RATIO_VAR", "KTG_DELTA_RATIO")
ratios = sys.argv[1:] or ["0", "0.05", "0.1", "0.2", "0.5", "1", "1e9"]
res = {}
for r in ratios:
    os.environ[var] = r
    if var == "KTG_DELTA_RATIO" and os.environ.get("FIX0"):  # scan later rounds only
        os.environ["KTG_DELTA_RATIO0"] = os.environ["FIX0"]
    eng = kt.Engine(g)
    row = []
    for k in ks:
        best = 1e9
        for _ in range(2):
            eng.reset(); eng.run(k)
            best = min(best, eng.info()["device_ms"])
        row.append(best)
    res[r] = row
    eng.close()
print("K      " + " ".join(f"{r:>8s}" for r in ratios))
for i, k in enumerate(ks):
    print(f"{k:5d}  " + " ".join(f"{res[r][i]:8.2f}" for r in ratios))
print("sum    " + " ".join(f"{sum(res[r]):8.1f}" for r in ratios))

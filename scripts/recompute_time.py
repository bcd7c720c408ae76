"""Recompute-mode and label-order fixpoint time sums at s20 (KTG_LIB_DIR selects the build)."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
for name, o in (("recompute", kt.TrussOptions(recompute=True)), ("label", kt.TrussOptions(label_order=True))):
    e = kt.Engine(g, o)
    tot = 0
    for k in (3, 10, 100, 304):
        ts = []
        for _ in range(3):
            e.reset(); e.run(k); ts.append(e.info()["device_ms"])
        tot += min(ts)
    print(f"{name} sum ms={tot:.2f}", flush=True)
    e.close()

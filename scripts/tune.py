"""Scratch: per-round support time (host loop + events) and graph-mode
fixpoint time at s20 for a few K; run with KTG_SCAN_RATIO=... to tune."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
scale = int(os.environ.get("SCALE", "20"))
g = kt.rmat(scale)
et = kt.Engine(g, time_support=True)
eg = kt.Engine(g)
tot = 0.0
for k in (3, 18, 60, 150, 304):
    et.reset(); et.run(k); w = et.round_work()
    sup = [x["support_ms"] for x in w]
    eg.reset(); eg.run(k)
    ts = []
    for _ in range(2):
        eg.reset(); eg.run(k); ts.append(eg.info()["device_ms"])
    tot += min(ts)
    print(f"ratio={os.environ.get('KTG_SCAN_RATIO','def')} k={k} rounds={len(sup)} sup_ms[0:3]={[round(x,2) for x in sup[:3]]} sup_total={sum(sup):.2f} fixpoint_ms={min(ts):.2f}", flush=True)
print(f"ratio={os.environ.get('KTG_SCAN_RATIO','def')} TOTAL5 {tot:.2f} ms")

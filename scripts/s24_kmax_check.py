"""s24: the GPU's K_max is consistent (K_max-truss non-empty, (K_max+1)-truss empty)."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(24)
e = kt.Engine(g)
for k in (935, 936):
    e.reset(); h = e.run(k); print(f"s24 K={k}: rounds={len(h)} survivors={e.info()['live_edges']}", flush=True)

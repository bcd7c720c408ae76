"""ER 2^22 K=3 fixpoint device time (KTG_LIB_DIR selects the build)."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
ln = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = kt.erdos_renyi(ln, 16 << ln)
e = kt.Engine(g)
ts = []
for _ in range(4):
    e.reset(); h = e.run(3); ts.append(e.info()["device_ms"])
print(f"er K=3 rounds={len(h)} ms={min(ts):.3f} live={e.info()['live_edges']}", flush=True)

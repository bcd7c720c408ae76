"""Host-loop run of the whole s20 K sweep (every K from pristine), for an ncu
launch list: the per-kernel share of the headline workload."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
e = kt.Engine(g, kt.TrussOptions(host_loop=True))
km = e.kmax()
stride = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for k in range(3, km + 1, stride):
    e.reset()
    e.run(k)
print("done", km)

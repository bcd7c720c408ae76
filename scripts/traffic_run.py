"""Driver for the ncu DRAM-traffic capture of the headline support kernel
(k_support_a22) over the bench's roofline sample: the same engines as the
bench's roofline leg (carried supports, no round-0 degree bound), host loop
so kernels are profilable. Launches of carried rounds exit at once and are
filtered out by duration in scripts/traffic_summary.py."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
e = kt.Engine(g, kt.TrussOptions(host_loop=True, no_degree_bound=True))
for k in (3, 78, 153, 228, 303, 304):
    e.reset(); e.run(k)

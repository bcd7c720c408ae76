"""Driver for the ncu DRAM-traffic capture of k_support_chunked over the
bench's roofline sample (host loop so kernels are profilable)."""
import sys
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
g = kt.rmat(20)
e = kt.Engine(g, kt.TrussOptions(host_loop=True))
for k in (3, 78, 153, 228, 303, 304):
    e.reset(); e.run(k)

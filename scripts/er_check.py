"""BASELINE configs[2]: Erdős–Rényi 2^22 vertices, 64M draws -- known answers
 and K_max on one B200."""
import sys, time
sys.path.insert(0, ".")
import paper_2009_07929_b200 as kt
t = time.time(); g = kt.erdos_renyi(22, 16 << 22, 42); print(f"gen {time.time()-t:.1f}s n={g.num_vertices} m={g.num_edges}", flush=True)
e = kt.Engine(g); e.reset(); tri = e.support_pass(); print(f"T={tri} maxS={e.info()['max_support']}", flush=True)
km = e.kmax(); print(f"kmax={km} survivors={e.info()['live_edges']}", flush=True)
e.reset(); h = e.run(km + 1); print(f"K={km+1}: survivors={e.info()['live_edges']} hist={h}", flush=True)

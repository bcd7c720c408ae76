"""Reference digests at the headline / north-star sizes (VERDICT r1 "next" #1).

Runs the UNMODIFIED reference (oracle/_ref/libktruss_ref.so: the reference
canonicalize + build_csr, then detail::run_fixpoint with Strategy::Fine on all
host threads, truss.cpp:41-53) and records, per (graph, K), SHA-256 of the
converged col_idx and S plus removed_per_iteration -- exactly the triple the
reference's ktruss() derives its result from (truss.cpp:57-71).

    nohup python tests/golden/make_golden_large.py > /tmp/golden.log 2>&1 &

It is resumable: every finished (graph, K) is written to
tests/golden/large_ref.json immediately and skipped on the next run. The GPU
box never runs this; tests/test_gpu_golden_large.py compares the engine's
digests with the committed JSON.

Graphs (SURVEY §8(d) generators, seed 42; the CSR itself is built by the
reference's own canonicalize -- `fast=False` -- and the digest of the parallel
restatement used by bench.py's reference arm is checked equal):
  s24    R-MAT scale 24 ef16: K in {936 (empty => K_max 935), 935, 3, 10, 30, 100, 300}
  er22   Erdos-Renyi 2^22 / 2^26 draws: K in {3, 4}
  cl22   R-MAT scale 22 ef32 + cliques {128,256,512,1024}: K in {K_max, K_max+1}
  s20    R-MAT scale 20 ef16: every K in 3..305
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(HERE, "large_ref.json")
CLIQUES = (128, 256, 512, 1024)
# K_max claims under test (the engine's own results, profiles/): the
# reference must give a non-empty truss at the claim and an empty one above.
KMAX_CLAIM = {"s24": 935, "cl22": 1057}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def load():
    return json.load(open(OUT)) if os.path.exists(OUT) else {}


def save(d):
    tmp = OUT + ".tmp"
    json.dump(d, open(tmp, "w"), indent=1, sort_keys=True)
    os.replace(tmp, OUT)


FAST_BUILD = False  # --fast-build: parallel canonicalize restatement, digest-checked against the stored reference one


def build(R, name):
    if FAST_BUILD:
        g = {"s24": lambda: R.rmat(24, 16, 42, fast=True), "s20": lambda: R.rmat(20, 16, 42, fast=True),
             "er22": lambda: R.erdos_renyi(22, 16 << 22, 42, fast=True),
             "cl22": lambda: R.rmat(22, 32, 42, extra_pairs=oracle.clique_pairs(1 << 22, CLIQUES, 42),
                                    fast=True)}[name]()
        ent = load().get(name, {})
        assert ent.get("col_sha256") == sha(g.col_idx) and ent.get("row_ptr_sha256") == sha(g.row_ptr), \
            "fast build differs from the reference canonicalize digest"
        return g
    if name == "s24":
        return R.rmat(24, 16, 42, fast=False)
    if name == "s20":
        return R.rmat(20, 16, 42, fast=False)
    if name == "er22":
        return R.erdos_renyi(22, 16 << 22, 42, fast=False)
    if name == "cl22":
        return R.rmat(22, 32, 42, extra_pairs=oracle.clique_pairs(1 << 22, CLIQUES, 42), fast=False)
    raise KeyError(name)


def fast_equal(R, name, g):
    if name == "s24":
        f = R.rmat(24, 16, 42, fast=True)
    elif name == "s20":
        f = R.rmat(20, 16, 42, fast=True)
    elif name == "er22":
        f = R.erdos_renyi(22, 16 << 22, 42, fast=True)
    else:
        f = R.rmat(22, 32, 42, extra_pairs=oracle.clique_pairs(1 << 22, CLIQUES, 42), fast=True)
    return bool(np.array_equal(f.row_ptr, g.row_ptr) and np.array_equal(f.col_idx, g.col_idx))


def plan(d):
    jobs = [("s24", k) for k in (936, 935, 3)] + [("er22", 3), ("er22", 4)]
    jobs += [("cl22", "kmax"), ("cl22", "kmax+1")]
    jobs += [("s20", k) for k in range(3, 306)]
    jobs += [("s24", k) for k in (300, 100, 30, 10)]
    return jobs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--only", default=None, help="comma list of graph names")
    ap.add_argument("--kmin", type=int, default=0, help="only K >= kmin (split a sweep across machines)")
    ap.add_argument("--kmax", type=int, default=1 << 30, help="only K <= kmax")
    ap.add_argument("--out", default=None, help="write here instead of tests/golden/large_ref.json")
    ap.add_argument("--fast-build", action="store_true",
                    help="build the CSR with the parallel canonicalize (must match the stored reference digest)")
    ap.add_argument("--ks", default=None, help="comma list of K (restricts the plan)")
    args = ap.parse_args()
    global OUT, FAST_BUILD
    FAST_BUILD = args.fast_build
    if args.out:
        OUT = args.out
    R = oracle.ref()
    d = load()
    graphs = {}
    for name, k in plan(d):
        if args.only and name not in args.only.split(","):
            continue
        if isinstance(k, int) and not args.kmin <= k <= args.kmax:
            continue
        if args.ks and isinstance(k, int) and k not in [int(x) for x in args.ks.split(",")]:
            continue
        ent = d.setdefault(name, {"fixpoints": {}})
        kk = KMAX_CLAIM[name] + (k == "kmax+1") if k in ("kmax", "kmax+1") else k
        if str(kk) in ent["fixpoints"] and "row_ptr_sha256" in ent:
            continue  # done: no need to rebuild the graph
        if name not in graphs:
            t0 = time.time()
            g = build(R, name)
            graphs = {name: g}  # keep one graph resident
            if "row_ptr_sha256" not in ent:
                ent.update(n=g.num_vertices, m=g.num_edges, slots=g.total_slots(), row_ptr_sha256=sha(g.row_ptr),
                           col_sha256=sha(g.col_idx), build_s=round(time.time() - t0, 1),
                           fast_canonicalize_equal=fast_equal(R, name, g))
                rc, tri, S = R.compute_supports(g, 2, args.threads)
                ent.update(triangles=tri, max_support=int(S.max()), supports_sha256=sha(S))
                del S
                save(d)
                print(name, "graph", {k_: v for k_, v in ent.items() if k_ != "fixpoints"}, flush=True)
        g = graphs[name]
        if k in ("kmax", "kmax+1"):
            # K_max is confirmed by a non-empty truss at the claim and an
            # empty one at claim+1 (trusses nest, kmax_search truss.cpp:73-103)
            k = KMAX_CLAIM[name] + (k == "kmax+1")
        key = str(k)
        if key in ent["fixpoints"]:
            continue
        col, S, hist, ms = R.run_fixpoint(g, k, 2, args.threads)
        live = int(np.count_nonzero(col))
        ent["fixpoints"][key] = {"col_sha256": sha(col), "supports_sha256": sha(S), "removed": hist,
                                 "survivors": live, "iterations": len(hist), "ms": round(ms, 1),
                                 "threads": args.threads}
        save(d)
        print(name, k, "survivors", live, "iters", len(hist), f"{ms / 1e3:.1f}s", flush=True)


if __name__ == "__main__":
    main()

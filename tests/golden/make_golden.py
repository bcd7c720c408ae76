"""Generates tests/golden/*.json from the UNMODIFIED reference library.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
The fixtures travel with the repo; the GPU box never reads /root/reference.

Contents:
  kat.json   -- the reference's own fixed graphs (test_helpers.hpp:14-43,
                proj/data/*.txt, test_support.cpp book graph) with the
                reference's compute_supports / ktruss(k) / kmax_search output.
  rmat.json  -- R-MAT s10/s12 (SURVEY §8(d) spec) stats, K=3 truss digest and
                K_max from the reference, and s14 known-answer stats.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2009_07929_b200 import graph  # noqa: E402


def complete(n, pendant=False):
    raw = [(u, v) for u in range(1, n + 1) for v in range(u + 1, n + 1)]
    if pendant:
        raw.append((n, n + 1))
    return raw


def parse_txt(path):
    raw = []
    for line in open(path):
        line = line.strip()
        if not line or line[0] in "#%":
            continue
        a, b = line.split()
        raw.append((int(a), int(b)))
    return raw


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def main():
    R = oracle.ref()
    cases = {
        "triangle": [(1, 2), (1, 3), (2, 3)],
        "path3": [(1, 2), (2, 3)],
        "single_edge": [(1, 2)],
        "bowtie": [(1, 2), (1, 3), (2, 3), (1, 4), (1, 5), (4, 5)],
        "k4": complete(4),
        "k5": complete(5),
        "k4_pendant": complete(4, True),
        "k5_pendant": complete(5, True),
        "two_triangles": [(1, 2), (1, 3), (2, 3), (4, 5), (4, 6), (5, 6)],
    }
    ref_data = "/root/reference/proj/data"
    for f in ("bowtie.txt", "k4_pendant.txt"):
        cases["data_" + f[:-4]] = parse_txt(os.path.join(ref_data, f))
    out = {}
    for name, raw in cases.items():
        g = R.canonicalize(raw)
        rc, tri, S = R.compute_supports(g, 2, 1)
        assert rc == 0
        ent = {"raw": raw, "n": g.num_vertices, "row_ptr": g.row_ptr.tolist(), "col_idx": g.col_idx.tolist(),
               "supports": S.tolist(), "triangles": tri, "truss": {}}
        km = R.kmax_search(g)
        ent["kmax"] = km["k_max"]
        for k in range(2, km["k_max"] + 2):
            t = R.ktruss(g, k)
            ent["truss"][str(k)] = {"edges": t["edges"].tolist(), "iterations": t["iterations"],
                                    "removed": t["removed"]}
        out[name] = ent
    # book graph (test_support.cpp:108-137): edge (1,2) with 70000 common neighbours
    raw = [(1, 2)] + [p for w in range(3, 70003) for p in ((1, w), (2, w))]
    g = R.canonicalize(raw)
    rc, tri, S = R.compute_supports(g, 2, 4)
    rc16, _, _ = R.compute_supports(g, 2, 4, width16=True)
    out["book70000"] = {"n": g.num_vertices, "slots": g.total_slots(), "triangles": tri, "S0": int(S[0]),
                        "supports_sha256": digest(S), "bits16_rc": rc16,
                        "bits16_slot": int(R.L.ref_last_error_slot()),
                        "bits16_msg": R.L.ref_last_error().decode()}
    json.dump(out, open(os.path.join(HERE, "kat.json"), "w"))

    rm = {}
    for scale in (10, 12):
        g = graph.rmat(scale, 16, 42)
        rc, tri, S = R.compute_supports(g, 2, 8)
        km = R.kmax_search(g, 2, 8)
        t3 = R.ktruss(g, 3, 2, 8)
        rm[f"s{scale}"] = {"n": g.num_vertices, "m": g.num_edges, "slots": g.total_slots(),
                           "col_sha256": digest(g.col_idx), "row_ptr_sha256": digest(g.row_ptr),
                           "triangles": tri, "max_support": int(S.max()), "supports_sha256": digest(S),
                           "kmax": km["k_max"], "kmax_edges": len(km["edges"]),
                           "kmax_edges_sha256": digest(km["edges"]),
                           "k3_edges_sha256": digest(t3["edges"]), "k3_removed": t3["removed"]}
    # s14 / s20 stats quoted in SURVEY §8(d) (reference-measured)
    rm["s14_known"] = {"n": 12527, "m": 213172, "slots": 225699, "triangles": 2840532, "max_support": 1287,
                       "kmax": 79, "k3_survivors": 199549, "kmax_survivors": 5067, "L_round1": 46086818,
                       "max_out_degree": 1755}
    rm["s20_known"] = {"n": 646609, "m": 15701434, "triangles": 423303124, "max_support": 15111, "kmax": 304,
                       "kmax_survivors": 481036, "k3_survivors": 13693463}
    json.dump(rm, open(os.path.join(HERE, "rmat.json"), "w"), indent=1)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()

"""The CPU oracle (oracle/ktruss_oracle.c) pinned against the reference's
known-answer vectors and against the unmodified reference library."""
import numpy as np
import pytest

from _util import corpus, digest, golden, kat_graph
from paper_2009_07929_b200 import graph


# --- literal KATs from the reference unit tests ------------------------------

def test_triangle_intersect_tails(port):
    """test_support.cpp:22-46."""
    g = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    S = np.zeros(g.total_slots(), np.uint32)
    assert port.intersect_tails(g, 0, 2, S) == 1
    S[0] += 1
    assert S.tolist() == [1, 1, 0, 1, 0, 0]
    S = np.zeros(g.total_slots(), np.uint32)
    assert port.intersect_tails(g, 1, 3, S) == 0 and S.sum() == 0


def test_supports_kats(port):
    """test_support.cpp:48-69."""
    tri = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    t, S = port.compute_supports(tri)
    assert t == 1 and S.tolist() == [1, 1, 0, 1, 0, 0]
    k4 = graph.csr_from_pairs([(u, v) for u in range(1, 5) for v in range(u + 1, 5)])
    t, S = port.compute_supports(k4)
    assert t == 4 and S.tolist() == [2, 2, 2, 0, 2, 2, 0, 2, 0, 0]
    path = graph.csr_from_pairs([(1, 2), (2, 3)])
    t, S = port.compute_supports(path)
    assert t == 0 and S.sum() == 0


def test_prune_kats(port):
    """test_truss.cpp:30-74."""
    tri = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    S = np.array([1, 1, 0, 1, 0, 0], np.uint32)
    for k, removed, col in [(3, 0, [2, 3, 0, 3, 0, 0]), (4, 3, [0] * 6), (2, 0, [2, 3, 0, 3, 0, 0])]:
        g = tri.copy()
        assert port.prune_edges(g, S, k) == removed
        assert g.col_idx.tolist() == col
    bow = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3), (1, 4), (1, 5), (4, 5)])
    _, S = port.compute_supports(bow)
    g = bow.copy()
    assert port.prune_edges(g, S, 4) == 6 and not g.col_idx.any()


def test_fixpoint_kats(port):
    """test_truss.cpp:76-104."""
    tri = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    e, hist = port.truss_edges(tri, 3)
    assert e.tolist() == [[1, 2, 1], [1, 3, 1], [2, 3, 1]] and hist == [0]
    k4p = graph.csr_from_pairs([(u, v) for u in range(1, 5) for v in range(u + 1, 5)] + [(4, 5)])
    e, hist = port.truss_edges(k4p, 3)
    assert hist == [1, 0] and (e[:, 2] == 2).all() and len(e) == 6


def test_kmax_kats(port):
    """test_truss.cpp:193-233 / acceptance.cpp:231-253."""
    def complete(n):
        return [(u, v) for u in range(1, n + 1) for v in range(u + 1, n + 1)]
    assert port.kmax(graph.csr_from_pairs(complete(4))) == 4
    assert port.kmax(graph.csr_from_pairs(complete(5))) == 5
    assert port.kmax(graph.csr_from_pairs(complete(5) + [(5, 6)])) == 5
    assert port.kmax(graph.csr_from_pairs([(1, 2), (2, 3)])) == 2
    assert port.kmax(graph.csr_from_pairs([(1, 2), (1, 3), (2, 3), (4, 5), (4, 6), (5, 6)])) == 3


# --- golden fixtures generated from the reference library ---------------------

def test_port_matches_golden_kat(port):
    for name, ent in golden("kat.json").items():
        if name == "book70000":
            continue
        g = kat_graph(ent)
        t, S = port.compute_supports(g)
        assert t == ent["triangles"] and S.tolist() == ent["supports"], name
        assert port.kmax(g) == ent["kmax"], name
        for k, tr in ent["truss"].items():
            e, hist = port.truss_edges(g, int(k))
            assert e.tolist() == tr["edges"] and hist == tr["removed"], (name, k)


def test_port_book_graph_bits16(port):
    ent = golden("kat.json")["book70000"]
    raw = [(1, 2)] + [p for w in range(3, 70003) for p in ((1, w), (2, w))]
    g = graph.csr_from_pairs(raw)
    t, S = port.compute_supports(g, threads=4)
    assert t == ent["triangles"] and int(S[0]) == ent["S0"] == 70000
    assert digest(S) == ent["supports_sha256"]
    assert port.first_overflow_16(S) == ent["bits16_slot"] == 0


@pytest.mark.parametrize("scale", [10, 12])
def test_port_matches_golden_rmat(port, scale):
    ent = golden("rmat.json")[f"s{scale}"]
    g = graph.rmat(scale, 16, 42)
    assert digest(g.col_idx) == ent["col_sha256"] and digest(g.row_ptr) == ent["row_ptr_sha256"]
    t, S = port.compute_supports(g, threads=4)
    assert t == ent["triangles"] and digest(S) == ent["supports_sha256"]
    e, hist = port.truss_edges(g, 3, threads=4)
    assert digest(e) == ent["k3_edges_sha256"] and hist == ent["k3_removed"]
    assert port.kmax(g, threads=4) == ent["kmax"]


def test_port_s14_known_answers(port):
    ent = golden("rmat.json")["s14_known"]
    g = graph.rmat(14, 16, 42)
    assert (g.num_vertices, g.num_edges, g.total_slots()) == (ent["n"], ent["m"], ent["slots"])
    t, S = port.compute_supports(g, threads=8)
    assert t == ent["triangles"] and int(S.max()) == ent["max_support"]
    w = port.round_work(g)
    assert w["L"] == ent["L_round1"] and w["max_out_degree"] == ent["max_out_degree"]
    e, _ = port.truss_edges(g, 3, threads=8)
    assert len(e) == ent["k3_survivors"]


# --- port vs the unmodified reference library ---------------------------------

def test_port_matches_reference_on_corpus(port, ref):
    for i, g in enumerate(corpus(60)):
        rc, t_r, S_r = ref.compute_supports(g, 2, 2)
        t_p, S_p = port.compute_supports(g, threads=2)
        assert rc == 0 and t_r == t_p and np.array_equal(S_r, S_p), i
        km = ref.oracle_kmax(g)
        assert port.kmax(g) == km, i
        for k in range(2, km + 2):
            c_r, s_r, h_r, _ = ref.run_fixpoint(g, k)
            c_p, s_p, h_p = port.run_fixpoint(g, k)
            assert h_r == h_p and np.array_equal(c_r, c_p) and np.array_equal(s_r, s_p), (i, k)


def test_planted_cliques_config(port):
    """BASELINE configs[4] generator (graph.rmat_cliques): deterministic,
    every clique pair present, K_max = the largest planted clique when it
    dominates the R-MAT part."""
    from paper_2009_07929_b200.graph import clique_members
    g1 = graph.rmat_cliques(10, 8, 42, sizes=(16, 40))
    g2 = graph.rmat_cliques(10, 8, 42, sizes=(16, 40))
    assert np.array_equal(g1.col_idx, g2.col_idx) and np.array_equal(g1.row_ptr, g2.row_ptr)
    m = clique_members(1 << 10, 40, 43)
    assert len(set(m.tolist())) == 40
    assert port.kmax(g1, threads=4) == 40


@pytest.mark.parametrize("scale,ef", [(10, 16), (13, 8), (12, 32)])
def test_reference_side_generator_and_fast_canonicalize(ref, scale, ef):
    """bench.py's reference arm builds its input on the reference side only:
    the §8(d) generator restated in oracle/ref_capi.cpp, then either the
    reference canonicalize or its parallel restatement -- byte-identical, and
    identical to the product's generator (the large digests pin s20/s24)."""
    import oracle
    from paper_2009_07929_b200 import graph
    extra = oracle.clique_pairs(1 << scale, (8, 20), 42) if ef == 32 else None
    a = ref.rmat(scale, ef, 42, extra_pairs=extra, fast=True)
    b = ref.rmat(scale, ef, 42, extra_pairs=extra, fast=False)
    c = graph.rmat_cliques(scale, ef, 42, sizes=(8, 20)) if ef == 32 else graph.rmat(scale, ef, 42)
    for x in (b, c):
        assert np.array_equal(a.row_ptr, x.row_ptr) and np.array_equal(a.col_idx, x.col_idx)
    e1 = ref.erdos_renyi(scale, ef << scale, 7, fast=True)
    e2 = ref.erdos_renyi(scale, ef << scale, 7, fast=False)
    assert np.array_equal(e1.col_idx, e2.col_idx) and np.array_equal(e1.row_ptr, e2.row_ptr)


def test_reference_fine_sample_partitions_a_pass(ref):
    """The cpu_baseline sample (support.cpp:115-127 over a chunk subset):
    the stride phases together are exactly one compute_supports pass."""
    g = ref.rmat(12, 16, 42)
    _, tri, S = ref.compute_supports(g, 2, 2)
    acc = np.zeros(g.total_slots(), np.uint32)
    tot = 0
    for ph in range(5):
        t, acc, _ = ref.fine_sample(g, 5, ph, 2, acc)
        tot += t
    assert tot == tri and np.array_equal(acc, S)


def test_large_golden_file_is_consistent():
    """tests/golden/large_ref.json (reference digests at s20/s24/ER/cliques):
    every fixpoint record ends in a zero-removal round, survivors fit the
    graph, and s24's K_max claim is bracketed when both probes exist."""
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "large_ref.json")
    if not os.path.exists(p):
        pytest.skip("large_ref.json not generated yet")
    d = json.load(open(p))
    for name, ent in d.items():
        for k, fp in ent.get("fixpoints", {}).items():
            assert fp["removed"][-1] == 0 and fp["iterations"] == len(fp["removed"])
            assert 0 <= fp["survivors"] <= ent["m"]
            assert ent["m"] - sum(fp["removed"]) == fp["survivors"], (name, k)
    s24 = d.get("s24", {}).get("fixpoints", {})
    if "935" in s24 and "936" in s24:
        assert s24["935"]["survivors"] > 0 and s24["936"]["survivors"] == 0

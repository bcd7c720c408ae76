"""Reference unit-test KATs (test_support.cpp, test_truss.cpp) through the
product API on the B200, plus the golden fixtures from the reference."""
import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from _util import digest, golden, kat_graph
from paper_2009_07929_b200 import errors

pytestmark = pytest.mark.gpu
ALL = [kt.Strategy.Serial, kt.Strategy.Coarse, kt.Strategy.Fine]


def complete(n, pendant=False):
    raw = [(u, v) for u in range(1, n + 1) for v in range(u + 1, n + 1)]
    return kt.csr_from_pairs(raw + ([(n, n + 1)] if pendant else []))


def test_intersect_tails():
    tri = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    S = kt.SupportArray.zeros(tri.total_slots())
    assert kt.intersect_tails(tri, 0, 2, S) == 1
    S.counts[0] += 1
    assert S.counts.tolist() == [1, 1, 0, 1, 0, 0]
    S = kt.SupportArray.zeros(tri.total_slots())
    assert kt.intersect_tails(tri, 1, 3, S) == 0 and S.counts.sum() == 0
    path = kt.csr_from_pairs([(1, 2), (2, 3)])
    S = kt.SupportArray.zeros(path.total_slots())
    assert kt.intersect_tails(path, 0, 2, S) == 0


@pytest.mark.parametrize("strategy", ALL)
def test_compute_supports_kats(strategy):
    tri = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    S = kt.SupportArray.zeros(tri.total_slots())
    assert kt.compute_supports(tri, S, strategy, 2) == 1
    assert S.counts.tolist() == [1, 1, 0, 1, 0, 0]
    k4 = complete(4)
    S = kt.SupportArray.zeros(k4.total_slots())
    assert kt.compute_supports(k4, S, strategy, 2) == 4
    assert S.counts.tolist() == [2, 2, 2, 0, 2, 2, 0, 2, 0, 0]
    path = kt.csr_from_pairs([(1, 2), (2, 3)])
    S = kt.SupportArray.zeros(path.total_slots())
    assert kt.compute_supports(path, S, strategy, 2) == 0 and S.counts.sum() == 0


def test_compute_supports_accumulates_like_reference():
    """compute_supports adds into S (it does not reset, support.hpp:48-51)."""
    tri = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    S = kt.SupportArray(np.array([5, 0, 7, 0, 0, 0], np.uint32))
    kt.compute_supports(tri, S)
    assert S.counts.tolist() == [6, 1, 7, 1, 0, 0]


def test_golden_kat_graphs():
    for name, ent in golden("kat.json").items():
        if name == "book70000":
            continue
        g = kat_graph(ent)
        S = kt.SupportArray.zeros(g.total_slots())
        assert kt.compute_supports(g, S) == ent["triangles"], name
        assert S.counts.tolist() == ent["supports"], name
        km = kt.kmax_search(g)
        assert km.k_max == ent["kmax"], name
        assert km.truss.edges.tolist() == ent["truss"][str(ent["kmax"])]["edges"], name
        for k, tr in ent["truss"].items():
            for host_loop in (False, True):
                r = kt.ktruss(g, int(k), kt.TrussOptions(host_loop=host_loop))
                assert r.edges.tolist() == tr["edges"], (name, k)
                assert r.iterations == tr["iterations"] and r.removed_per_iteration == tr["removed"], (name, k)


def test_book_graph_bits16():
    ent = golden("kat.json")["book70000"]
    raw = [(1, 2)] + [p for w in range(3, 70003) for p in ((1, w), (2, w))]
    g = kt.csr_from_pairs(raw)
    S = kt.SupportArray.zeros(g.total_slots())
    assert kt.compute_supports(g, S, kt.Strategy.Fine, 2, kt.SupportWidth.Bits32) == 70000
    assert S.counts[0] == 70000 and digest(S.counts) == ent["supports_sha256"]
    S = kt.SupportArray.zeros(g.total_slots())
    with pytest.raises(errors.SupportOverflowError) as ex:
        kt.compute_supports(g, S, kt.Strategy.Fine, 2, kt.SupportWidth.Bits16)
    assert ex.value.slot == ent["bits16_slot"] == 0
    assert str(ex.value) == ent["bits16_msg"]
    # the fixpoint surfaces the same error
    with pytest.raises(errors.SupportOverflowError):
        kt.ktruss(g, 3, kt.TrussOptions(width=kt.SupportWidth.Bits16))
    # within range both widths agree (test_support.cpp:130-136)
    k5 = complete(5)
    a, b = kt.SupportArray.zeros(k5.total_slots()), kt.SupportArray.zeros(k5.total_slots())
    kt.compute_supports(k5, a, kt.Strategy.Serial, 1, kt.SupportWidth.Bits32)
    kt.compute_supports(k5, b, kt.Strategy.Serial, 1, kt.SupportWidth.Bits16)
    assert np.array_equal(a.counts, b.counts)


def test_book_graph_truss_long_rows(port):
    """Rows far longer than a staged chunk (1024) and the CTA-prune threshold."""
    raw = [(1, 2)] + [p for w in range(3, 70003) for p in ((1, w), (2, w))]
    g = kt.csr_from_pairs(raw)
    for k in (3, 4, 5):
        r = kt.ktruss(g, k)
        e, hist = port.truss_edges(g, k, threads=4)
        assert np.array_equal(r.edges, e) and r.removed_per_iteration == hist, k


def test_prune_kats():
    tri = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    S = kt.SupportArray(np.array([1, 1, 0, 1, 0, 0], np.uint32))
    for k, removed, col in [(3, 0, [2, 3, 0, 3, 0, 0]), (4, 3, [0] * 6), (2, 0, [2, 3, 0, 3, 0, 0])]:
        g = tri.copy()
        assert kt.prune_edges(g, S, k) == removed
        assert g.col_idx.tolist() == col
        kt.validate_csr(g)
    with pytest.raises(errors.InvalidParameterError):
        kt.prune_edges(tri.copy(), S, 1)
    bow = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3), (1, 4), (1, 5), (4, 5)])
    S = kt.SupportArray.zeros(bow.total_slots())
    kt.compute_supports(bow, S, kt.Strategy.Serial, 1)
    g = bow.copy()
    assert kt.prune_edges(g, S, 4) == 6 and g.live_edges() == 0
    k4p = complete(4, True)
    S = kt.SupportArray.zeros(k4p.total_slots())
    kt.compute_supports(k4p, S)
    g = k4p.copy()
    assert kt.prune_edges(g, S, 3) == 1
    kt.validate_csr(g)
    u, v = kt.extract_edges(g)
    assert list(zip(u.tolist(), v.tolist())) == [(a, b) for a in range(1, 5) for b in range(a + 1, 5)]


def test_fixpoint_kats():
    r = kt.ktruss(kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)]), 3)
    assert r.edges.tolist() == [[1, 2, 1], [1, 3, 1], [2, 3, 1]]
    assert r.iterations == 1 and r.removed_per_iteration == [0]
    r = kt.ktruss(kt.csr_from_pairs([(1, 2), (1, 3), (2, 3), (1, 4), (1, 5), (4, 5)]), 3)
    assert len(r.edges) == 6 and (r.edges[:, 2] == 1).all()
    r = kt.ktruss(complete(4, True), 3)
    assert r.iterations == 2 and r.removed_per_iteration == [1, 0] and (r.edges[:, 2] == 2).all()
    r = kt.ktruss(kt.csr_from_pairs([(1, 2), (2, 3)]), 2)
    assert r.iterations == 1 and len(r.edges) == 2
    with pytest.raises(errors.InvalidParameterError):
        kt.ktruss(complete(3), 1)


def test_ktruss_leaves_input_untouched():
    g = complete(4, True)
    before = g.col_idx.copy()
    kt.ktruss(g, 5)
    assert np.array_equal(g.col_idx, before)


def test_observer_sees_every_round():
    g = complete(4, True)
    seen = []

    def obs(graph, S, removed):
        kt.validate_csr(graph)
        assert S.size() == graph.total_slots()
        seen.append(removed)

    r = kt.ktruss(g, 3, kt.TrussOptions(observer=obs))
    assert seen == r.removed_per_iteration == [1, 0]


def test_observer_supports_match_reference(ref):
    """Observer gets the round's supports exactly as the reference passes them."""
    g = kt.rmat(9, 16, seed=3)
    for k in (4, 7):
        mine, theirs = [], []
        kt.ktruss(g, k, kt.TrussOptions(observer=lambda gg, S, r: mine.append((gg.col_idx.copy(), S.counts.copy(), r))))
        col = g.col_idx.copy()
        S = np.zeros(g.total_slots(), np.uint32)
        # replay the reference loop round by round
        work = g.copy()
        while True:
            rc, _, S = ref.compute_supports(work, 2, 1)
            rc, removed, newcol = ref.prune_edges(work, S, k)
            work.col_idx = newcol
            theirs.append((newcol.copy(), S.copy(), removed))
            if removed == 0:
                break
        assert len(mine) == len(theirs)
        for (c1, s1, r1), (c2, s2, r2) in zip(mine, theirs):
            assert r1 == r2 and np.array_equal(c1, c2) and np.array_equal(s1, s2)


def test_kmax_kats():
    k4 = kt.kmax_search(complete(4))
    assert k4.k_max == 4 and len(k4.truss.edges) == 6 and (k4.truss.edges[:, 2] == 2).all()
    path = kt.kmax_search(kt.csr_from_pairs([(1, 2), (2, 3)]))
    assert path.k_max == 2 and len(path.truss.edges) == 2 and (path.truss.edges[:, 2] == 0).all()
    k5p = kt.kmax_search(complete(5, True))
    assert k5p.k_max == 5 and [tuple(e[:2]) for e in k5p.truss.edges] == [
        (a, b) for a in range(1, 6) for b in range(a + 1, 6)]
    two = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3), (4, 5), (4, 6), (5, 6)])
    assert kt.kmax_search(two).k_max == 3
    empty = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    empty.col_idx[:] = 0
    with pytest.raises(errors.InvalidParameterError, match="kmax_search needs a non-empty graph"):
        kt.kmax_search(empty)


def test_all_zero_graph_fixpoint():
    g = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    g.col_idx[:] = 0
    r = kt.ktruss(g, 3)
    assert r.iterations == 1 and r.removed_per_iteration == [0] and len(r.edges) == 0


def test_thread_counts_are_deterministic():
    g = kt.rmat(9, 16, seed=99)
    base = kt.ktruss(g, 4, kt.TrussOptions(threads=1))
    for t in (2, 4, 8):
        r = kt.ktruss(g, 4, kt.TrussOptions(strategy=kt.Strategy.Fine, threads=t))
        assert np.array_equal(r.edges, base.edges) and r.removed_per_iteration == base.removed_per_iteration

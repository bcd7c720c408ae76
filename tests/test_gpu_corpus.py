"""Acceptance criteria c1/c2/c3/c5/c6 (acceptance.cpp:127-256) on the B200."""
import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from _util import corpus

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def graphs():
    return corpus(200)


def test_c1_c6_oracle_equivalence(graphs, ref):
    """Every k in 2..kmax+1: survivors and supports equal the brute-force
    oracle (ktruss_edges + edge_supports); CSR valid after every round."""
    runs = 0
    for i, g in enumerate(graphs):
        km = ref.oracle_kmax(g)
        for k in range(2, km + 2):
            expected = ref.oracle_truss(g, k)
            r = kt.ktruss(g, k)
            assert np.array_equal(r.edges, expected), (i, k)
            runs += 1
            if i % 10 == 0:
                slots = g.total_slots()

                def obs(gg, S, removed):
                    kt.validate_csr(gg)
                    assert gg.total_slots() == slots
                r2 = kt.ktruss(g, k, kt.TrussOptions(observer=obs))
                assert np.array_equal(r2.edges, expected)
    assert runs > 1000


def test_c2_strategy_and_kernel_equivalence(ref):
    for i in range(50):
        n = [64, 96, 128, 192, 256, 384, 512][i % 7]
        p = min(0.3, 12.0 / n)
        g = ref.random_graph(n, p, 2000 + i)
        _, _, S_ser = ref.compute_supports(g, 0, 1)
        for strategy in kt.Strategy:
            S = kt.SupportArray.zeros(g.total_slots())
            kt.compute_supports(g, S, strategy, 4)
            assert np.array_equal(S.counts, S_ser), i
        e = kt.Engine(g, kt.TrussOptions(naive_support=True))
        e.support_pass()
        assert np.array_equal(e.read()[1], S_ser)


def test_c3_triple_count_identity(graphs, ref):
    for g in graphs:
        S = kt.SupportArray.zeros(g.total_slots())
        t = kt.compute_supports(g, S)
        assert int(S.counts.sum(dtype=np.uint64)) == 3 * t
        assert t == ref.oracle_triangles(g)


def test_c5_kmax(graphs, ref):
    for g in graphs[::2]:
        assert kt.kmax_search(g).k_max == ref.oracle_kmax(g)

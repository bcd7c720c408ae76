"""Fast GPU parity: engine vs CPU oracle on small graphs (byte-exact)."""
import numpy as np
import pytest

import paper_2009_07929_b200 as kt

pytestmark = pytest.mark.gpu


def _graphs():
    yield "triangle", kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    yield "k4p", kt.csr_from_pairs([(1, 2), (1, 3), (1, 4), (2, 3), (2, 4), (3, 4), (4, 5)])
    yield "rmat10", kt.rmat(10, 16, seed=7)
    yield "rmat12", kt.rmat(12, 16, seed=42)


@pytest.mark.parametrize("naive", [False, True])
@pytest.mark.parametrize("label", [False, True])
def test_supports_match_oracle(port, naive, label):
    for name, g in _graphs():
        t_exp, S_exp = port.compute_supports(g, threads=4)
        if naive or label:
            eng = kt.Engine(g, kt.TrussOptions(naive_support=naive, label_order=label))
            eng.reset()
            t = eng.support_pass()
            _, S = eng.read()
        else:
            S = kt.SupportArray.zeros(g.total_slots())
            t = kt.compute_supports(g, S)
            S = S.counts
        assert t == t_exp, name
        assert np.array_equal(S, S_exp), name


@pytest.mark.parametrize("host_loop", [False, True])
@pytest.mark.parametrize("label", [False, True])
def test_fixpoint_matches_oracle(port, host_loop, label):
    for name, g in _graphs():
        for k in (2, 3, 4, 5, 8):
            col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=4)
            work = g.copy()
            S = kt.SupportArray.zeros(g.total_slots())
            hist = kt.run_fixpoint(work, S, k, kt.TrussOptions(host_loop=host_loop, label_order=label))
            assert hist == hist_e, (name, k)
            assert np.array_equal(work.col_idx, col_e), (name, k)
            assert np.array_equal(S.counts, S_e), (name, k)

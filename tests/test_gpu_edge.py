"""Edge cases: degenerate and ragged inputs, extreme k, buffer reuse across
graphs of different sizes -- all against the oracle, byte-exact."""
import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from paper_2009_07929_b200 import errors

pytestmark = pytest.mark.gpu


def _check_fixpoint(port, g, k, **opt):
    work = g.copy()
    S = kt.SupportArray.zeros(g.total_slots())
    hist = kt.run_fixpoint(work, S, k, kt.TrussOptions(**opt))
    col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=4)
    assert hist == hist_e
    assert np.array_equal(work.col_idx, col_e) and np.array_equal(S.counts, S_e)


def test_single_vertex_graph(port):
    g = kt.ZeroTerminatedCsr(1, np.array([0, 0, 1], np.uint32), np.array([0], np.uint32))
    r = kt.ktruss(g, 3)
    assert r.iterations == 1 and r.removed_per_iteration == [0] and len(r) == 0
    with pytest.raises(errors.InvalidParameterError):
        kt.kmax_search(g)


@pytest.mark.parametrize("label", [False, True])
def test_pruned_ragged_input(port, label):
    """Input that is itself a pruned CSR: rows with zero tails and empty rows."""
    g = kt.rmat(11, 16, seed=8)
    col, _, _ = port.run_fixpoint(g, 6, threads=4)
    pruned = kt.ZeroTerminatedCsr(g.num_vertices, g.row_ptr, col)
    kt.validate_csr(pruned)
    assert pruned.live_edges() < g.live_edges()
    for k in (2, 3, 7, 9):
        _check_fixpoint(port, pruned, k, label_order=label)
    km = kt.kmax_search(pruned)
    assert km.k_max == port.kmax(pruned, threads=4)


def test_extreme_k(port):
    g = kt.rmat(10, 16, seed=2)
    for k in (2, 10**6):
        _check_fixpoint(port, g, k)
    r = kt.ktruss(g, 10**6)
    assert len(r) == 0 and r.removed_per_iteration == [g.live_edges(), 0]


def test_engine_reload_sizes(port):
    e = kt.Engine()
    for scale in (12, 9, 13, 10):
        g = kt.rmat(scale, 16, seed=scale)
        e.load(g)
        for k in (3, 5):
            e.reset()
            hist = e.run(k)
            col, S = e.read()
            col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=4)
            assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e), (scale, k)


def test_results_survive_later_calls(port):
    """ktruss results live in pooled page-locked buffers: a result kept by the
    caller must not be overwritten by later calls (large results stay views
    of their buffer, small ones are copied out)."""
    g = kt.rmat(16, 16, seed=42)  # K=3/4 results exceed the copy-out size
    kept = {k: kt.ktruss(g, k) for k in (3, 4, 60)}
    assert kept[3].u.base is not None  # a view of a pooled buffer
    for _ in range(3):  # churn the pool with other K values
        for k in (5, 30, 3):
            kt.ktruss(g, k)
    for k, r in kept.items():
        e, hist = port.truss_edges(g, k, threads=4)
        assert np.array_equal(r.edges, e) and r.removed_per_iteration == hist, k
    del kept
    r = kt.ktruss(g, 3)  # buffers released above are reused
    e, _ = port.truss_edges(g, 3, threads=4)
    assert np.array_equal(r.edges, e)


def test_engine_reports_carried_mode():
    """ktg_run_info.carried: 1 when the carried-support structures are
    resident (default), 0 for recompute-only engines (KTG_FLAG_RECOMPUTE,
    label order; also a load whose structures do not fit in HBM)."""
    g = kt.rmat(10, 16, seed=3)
    e = kt.Engine(g)
    e.reset()
    e.run(4)
    assert e.info()["carried"] == 1
    e.close()
    for o in (kt.TrussOptions(recompute=True), kt.TrussOptions(label_order=True)):
        e = kt.Engine(g, o)
        e.reset()
        e.run(4)
        assert e.info()["carried"] == 0
        e.close()

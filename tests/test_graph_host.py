"""Host graph preparation (libktg_graph.so) vs the reference's canonicalize +
build_csr (edge_list.cpp:62-103, csr.cpp:10-32), and validate_csr."""
import numpy as np
import pytest

from _util import golden
from paper_2009_07929_b200 import errors, graph


def test_layout_kats():
    """test_graph_io.cpp:93-109."""
    g = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    assert g.row_ptr.tolist() == [0, 0, 3, 5, 6] and g.col_idx.tolist() == [2, 3, 0, 3, 0, 0]
    g = graph.csr_from_pairs([(1, 2)])
    assert g.row_ptr.tolist() == [0, 0, 2, 3] and g.col_idx.tolist() == [2, 0, 0]
    g = graph.csr_from_pairs([(1, 2), (2, 3)])
    assert g.row_ptr.tolist() == [0, 0, 2, 4, 5] and g.col_idx.tolist() == [2, 0, 3, 0, 0]


def test_canonicalize_drops_loops_dupes_and_relabels():
    g = graph.csr_from_pairs([(10, 20), (20, 10), (7, 7), (20, 30), (30, 30), (99, 10)])
    assert g.num_vertices == 4  # labels 10,20,30,99 (7 only in a self-loop)
    assert g.original_ids.tolist() == [0, 10, 20, 30, 99]
    u, v = graph.extract_edges(g)
    assert list(zip(u.tolist(), v.tolist())) == [(1, 2), (1, 4), (2, 3)]


def test_empty_graph_raises():
    with pytest.raises(errors.EmptyGraphError):
        graph.csr_from_pairs([(3, 3), (4, 4)])


@pytest.mark.parametrize("seed", range(6))
def test_matches_reference_canonicalize(ref, seed):
    rng = np.random.default_rng(seed)
    sparse = seed % 2 == 0
    hi = 2**40 if sparse else 300
    raw = rng.integers(0, hi, size=(2000, 2), dtype=np.uint64)
    raw[::7, 1] = raw[::7, 0]  # self loops
    raw = np.concatenate([raw, raw[::5, ::-1]])  # reversed duplicates
    mine = graph.csr_from_pairs(raw)
    theirs = ref.canonicalize(raw)
    assert mine.num_vertices == theirs.num_vertices
    assert np.array_equal(mine.row_ptr, theirs.row_ptr) and np.array_equal(mine.col_idx, theirs.col_idx)


def test_rmat_raw_matches_reference_canonicalize(ref):
    """The full s12 generator output canonicalized by the reference itself."""
    import ctypes
    g = graph._g()
    h = ctypes.c_void_p()
    assert g.ktgg_rmat_raw(12, 16, 42, 0.57, 0.19, 0.19, ctypes.byref(h)) == 0
    m = g.ktgg_raw_count(h)
    pairs = np.ctypeslib.as_array(g.ktgg_raw_pairs(h), shape=(2 * m,)).copy()
    g.ktgg_raw_free(h)
    theirs = ref.canonicalize(pairs.reshape(-1, 2).astype(np.uint64))
    mine = graph.rmat(12, 16, 42)
    assert np.array_equal(mine.col_idx, theirs.col_idx) and np.array_equal(mine.row_ptr, theirs.row_ptr)


def test_rmat_s14_known_stats():
    ent = golden("rmat.json")["s14_known"]
    g = graph.rmat(14)
    w = graph.round_work(g)
    assert (g.num_vertices, g.num_edges) == (ent["n"], ent["m"])
    assert w["L"] == ent["L_round1"] and w["max_out_degree"] == ent["max_out_degree"]
    graph.validate_csr(g)


def test_er_small_matches_reference(ref):
    import ctypes
    L = graph._g()
    h = ctypes.c_void_p()
    assert L.ktgg_er_raw(10, 4000, 42, ctypes.byref(h)) == 0
    m = L.ktgg_raw_count(h)
    pairs = np.ctypeslib.as_array(L.ktgg_raw_pairs(h), shape=(2 * m,)).copy()
    L.ktgg_raw_free(h)
    theirs = ref.canonicalize(pairs.reshape(-1, 2).astype(np.uint64))
    mine = graph.erdos_renyi(10, 4000, 42)
    assert np.array_equal(mine.col_idx, theirs.col_idx)


def _bad(g, **kw):
    g = g.copy()
    for k, v in kw.items():
        getattr(g, k)[:] = v
    return g


def test_validate_csr_agrees_with_reference(ref):
    base = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    cases = [
        base,
        graph.ZeroTerminatedCsr(3, base.row_ptr, np.array([2, 3, 0, 3, 0, 1], np.uint32)),  # no end zero
        graph.ZeroTerminatedCsr(3, base.row_ptr, np.array([0, 3, 0, 3, 0, 0], np.uint32)),  # nonzero after zero
        graph.ZeroTerminatedCsr(3, base.row_ptr, np.array([3, 2, 0, 3, 0, 0], np.uint32)),  # not ascending
        graph.ZeroTerminatedCsr(3, base.row_ptr, np.array([2, 4, 0, 3, 0, 0], np.uint32)),  # beyond n
        graph.ZeroTerminatedCsr(3, base.row_ptr, np.array([1, 3, 0, 3, 0, 0], np.uint32)),  # w <= v
        graph.ZeroTerminatedCsr(3, np.array([0, 1, 3, 5, 6], np.uint32), base.col_idx),  # phantom owns slot
    ]
    for g in cases:
        expected = ref.validate(g)
        try:
            graph.validate_csr(g)
            got = None
        except errors.InvalidInputError as e:
            got = str(e)
        assert got == expected

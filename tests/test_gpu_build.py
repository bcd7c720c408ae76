"""canonicalize + build_csr on the device equals the
reference's (edge_list.cpp:62-103, csr.cpp:10-32) byte for byte."""
import ctypes

import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from paper_2009_07929_b200 import errors, graph

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.num_vertices == b.num_vertices
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)


@pytest.mark.parametrize("seed", range(4))
def test_random_labels_match_reference(ref, seed):
    rng = np.random.default_rng(seed)
    hi = 2**40 if seed % 2 == 0 else 500
    raw = rng.integers(0, hi, size=(5000, 2), dtype=np.uint64)
    raw[::9, 1] = raw[::9, 0]                      # self-loops
    raw = np.concatenate([raw, raw[::4, ::-1]])    # reversed duplicates
    g = kt.Engine().build_csr(raw)
    _same(g, ref.canonicalize(raw))
    host = graph.csr_from_pairs(raw)
    assert np.array_equal(g.original_ids, host.original_ids)


def test_rmat_raw_matches_host_build():
    L = graph._g()
    h = ctypes.c_void_p()
    assert L.ktgg_rmat_raw(16, 16, 42, 0.57, 0.19, 0.19, ctypes.byref(h)) == 0
    m = L.ktgg_raw_count(h)
    pairs = np.ctypeslib.as_array(L.ktgg_raw_pairs(h), shape=(2 * m,)).astype(np.uint64)
    L.ktgg_raw_free(h)
    e = kt.Engine()
    g = e.build_csr(pairs)
    _same(g, graph.rmat(16))
    e.reset()
    assert e.run(3)[-1] == 0


def test_empty_after_loops_raises():
    with pytest.raises(errors.EmptyGraphError):
        kt.Engine().build_csr(np.array([[5, 5], [7, 7]], np.uint64))


def test_built_graph_fixpoint(port):
    rng = np.random.default_rng(11)
    raw = rng.integers(1, 3000, size=(40000, 2), dtype=np.uint64)
    e = kt.Engine()
    g = e.build_csr(raw)
    for k in (3, 4):
        e.reset()
        hist = e.run(k)
        col, S = e.read()
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e)

"""ZTCSR1 cache: byte layout and corruption handling match
the reference (csr_cache.cpp, test_graph_io.cpp:185-235); the device loader
streams it into HBM and validates it there."""
import os

import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from paper_2009_07929_b200 import errors, graph


def test_layout_pinned_byte_for_byte(tmp_path):
    """test_graph_io.cpp:189-203."""
    g = graph.csr_from_pairs([(1, 2)])
    p = str(tmp_path / "e.ztcsr")
    graph.write_csr_cache(g, p)
    expected = bytes([ord(c) for c in "ZTCSR1"] + [0, 0, 2, 0, 0, 0, 3, 0, 0, 0, 0, 0, 0, 0] +
                     [0] * 8 + [2, 0, 0, 0, 3, 0, 0, 0] + [2, 0, 0, 0] + [0] * 8)
    assert open(p, "rb").read() == expected


def test_round_trip_and_identity_with_reference(tmp_path, ref):
    g = graph.rmat(11, 16, seed=3)
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    graph.write_csr_cache(g, a)
    ref.write_cache(g, b)
    assert open(a, "rb").read() == open(b, "rb").read()
    back = graph.read_csr_cache(b)
    assert back.num_vertices == g.num_vertices
    assert np.array_equal(back.row_ptr, g.row_ptr) and np.array_equal(back.col_idx, g.col_idx)


def _corruptions(good):
    yield "short file", good[:4]
    bad = bytearray(good)
    bad[0] = ord("X")
    yield "bad magic", bytes(bad)
    yield "truncated payload", good[:-3]
    yield "trailing bytes", good + b"x"
    bad = bytearray(good)
    bad[-4] = 9  # last col entry (row 3's sentinel)
    yield "row without a sentinel", bytes(bad)
    bad = bytearray(good)
    bad[8] = 0  # n = 0
    yield "implausible dims", bytes(bad)


def test_corruption_matches_reference(tmp_path, ref):
    """test_graph_io.cpp:205-235: every corruption raises CorruptCacheError
    with the reference's message."""
    g = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    p = str(tmp_path / "t")
    graph.write_csr_cache(g, p)
    good = open(p, "rb").read()
    for name, data in _corruptions(good):
        q = str(tmp_path / name.replace(" ", "_"))
        open(q, "wb").write(data)
        _, ref_msg = ref.read_cache(q)
        assert ref_msg is not None, name
        with pytest.raises(errors.CorruptCacheError) as ex:
            graph.read_csr_cache(q)
        assert str(ex.value) == ref_msg, name


@pytest.mark.gpu
def test_device_cache_load(tmp_path, port):
    g = graph.rmat(12, 16, seed=42)
    p = str(tmp_path / "s12.ztcsr")
    graph.write_csr_cache(g, p)
    e = kt.Engine()
    e.load_cache(p)
    for k in (3, 9):
        e.reset()
        hist = e.run(k)
        col, S = e.read()
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e)


@pytest.mark.gpu
def test_device_cache_corruption(tmp_path, ref):
    g = graph.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    p = str(tmp_path / "t")
    graph.write_csr_cache(g, p)
    good = open(p, "rb").read()
    cases = list(_corruptions(good))
    # interior invariant violations the device validator must name
    # header 20 B + row_ptr 5 x 4 B: col starts at byte 40
    for pos, val in ((40, 3), (44, 7), (32, 7)):  # col[0]=3 (not ascending), col[1]=7 (> n), row_ptr[3]=7
        bad = bytearray(good)
        bad[pos] = val
        cases.append((f"interior {pos}", bytes(bad)))
    bad = []
    for name, data in cases:
        q = str(tmp_path / name.replace(" ", "_"))
        open(q, "wb").write(data)
        _, ref_msg = ref.read_cache(q)
        assert ref_msg is not None, name
        e = kt.Engine()
        try:
            e.load_cache(q)
            bad.append((name, "no error", ref_msg))
        except errors.CorruptCacheError as ex:
            if str(ex) != ref_msg:
                bad.append((name, str(ex), ref_msg))
    assert not bad, bad

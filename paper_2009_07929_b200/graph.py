"""Zero-terminated upper-triangular CSR and its host-side preparation.

`ZeroTerminatedCsr` mirrors /root/reference/proj/include/ktruss/csr.hpp:17-23:
vertex ids 1..n (0 is the sentinel / phantom vertex), row_ptr has n+2 entries
with row_ptr[0] == row_ptr[1] == 0, every row is strictly ascending w > v
followed by at least one zero slot.

Generators and canonicalize/build_csr run natively (libktg_graph.so, see
include/ktg_graph.h); they are the input side of the boundary, not the hot
path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import errors
from ._lib import graph_lib

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


class _Work(ctypes.Structure):
    _fields_ = [
        ("live_edges", ctypes.c_uint64),
        ("max_out_degree", ctypes.c_uint32),
        ("tail_elements", ctypes.c_uint64),
        ("cross_elements", ctypes.c_uint64),
        ("L", ctypes.c_uint64),
        ("sum_dout_sq", ctypes.c_uint64),
    ]


_configured = False


def _g():
    global _configured
    lib = graph_lib()
    if not _configured:
        vp = ctypes.c_void_p
        lib.ktgg_last_error.restype = ctypes.c_char_p
        lib.ktgg_rmat_raw.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.POINTER(vp)]
        lib.ktgg_er_raw.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.POINTER(vp)]
        lib.ktgg_raw_count.argtypes = [vp]
        lib.ktgg_raw_count.restype = ctypes.c_uint64
        lib.ktgg_raw_pairs.argtypes = [vp]
        lib.ktgg_raw_pairs.restype = _u32p
        lib.ktgg_raw_free.argtypes = [vp]
        lib.ktgg_csr_from_raw.argtypes = [vp, ctypes.POINTER(vp)]
        lib.ktgg_csr_from_pairs_u32.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(vp)]
        lib.ktgg_csr_from_pairs_u64.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(vp)]
        lib.ktgg_csr_n.argtypes = [vp]
        lib.ktgg_csr_n.restype = ctypes.c_uint32
        lib.ktgg_csr_slots.argtypes = [vp]
        lib.ktgg_csr_slots.restype = ctypes.c_uint64
        lib.ktgg_csr_copy.argtypes = [vp, vp, vp, vp]
        lib.ktgg_csr_free.argtypes = [vp]
        lib.ktgg_round_work.argtypes = [vp, ctypes.c_uint32, vp, ctypes.POINTER(_Work)]
        lib.ktgg_write_csr_cache.argtypes = [ctypes.c_char_p, vp, ctypes.c_uint32, vp, ctypes.c_uint64]
        lib.ktgg_read_csr_cache.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
        _configured = True
    return lib


def _raise(rc: int):
    msg = _g().ktgg_last_error().decode()
    if rc == 1:
        raise errors.InvalidParameterError(msg)
    if rc == 3:
        raise errors.InvalidInputError(msg)
    if rc == 4:
        raise errors.EmptyGraphError(msg)
    if rc == 5:
        raise errors.CorruptCacheError(msg)
    if rc == 7:
        raise MemoryError(msg)
    raise errors.Error(msg)


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class ZeroTerminatedCsr:
    """ktruss::ZeroTerminatedCsr (csr.hpp:17-23). Arrays are u32, C-contiguous."""

    num_vertices: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    original_ids: Optional[np.ndarray] = field(default=None, repr=False)

    def total_slots(self) -> int:
        return int(self.col_idx.shape[0])

    @property
    def num_edges(self) -> int:
        """Original canonical edge count, slots - n (bench.cpp:45)."""
        return self.total_slots() - self.num_vertices

    def copy(self) -> "ZeroTerminatedCsr":
        return ZeroTerminatedCsr(self.num_vertices, self.row_ptr.copy(), self.col_idx.copy(),
                                 self.original_ids)

    def live_edges(self) -> int:
        """count_live_edges (csr.cpp:108-114): nonzero slots."""
        return int(np.count_nonzero(self.col_idx))


def _csr_from_handle(h: ctypes.c_void_p) -> ZeroTerminatedCsr:
    lib = _g()
    try:
        n = lib.ktgg_csr_n(h)
        slots = lib.ktgg_csr_slots(h)
        row_ptr = np.empty(n + 2, dtype=np.uint32)
        col = np.empty(slots, dtype=np.uint32)
        ids = np.empty(n + 1, dtype=np.uint64)
        lib.ktgg_csr_copy(h, _ptr(row_ptr), _ptr(col), _ptr(ids))
    finally:
        lib.ktgg_csr_free(h)
    return ZeroTerminatedCsr(int(n), row_ptr, col, ids)


def csr_from_pairs(pairs) -> ZeroTerminatedCsr:
    """canonicalize (edge_list.cpp:62-103) + build_csr (csr.cpp:10-32) of raw
    (label, label) pairs. Raises EmptyGraphError when no non-loop pair exists."""
    a = np.ascontiguousarray(np.asarray(pairs))
    if a.size == 0:
        raise errors.EmptyGraphError("no edges survive canonicalization")
    a = a.reshape(-1, 2)
    lib = _g()
    h = ctypes.c_void_p()
    if a.dtype != np.uint64 and a.max() < 2**32 and a.min() >= 0:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        rc = lib.ktgg_csr_from_pairs_u32(_ptr(a), a.shape[0], ctypes.byref(h))
    else:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        rc = lib.ktgg_csr_from_pairs_u64(_ptr(a), a.shape[0], ctypes.byref(h))
    if rc:
        _raise(rc)
    return _csr_from_handle(h)


def _raw_to_csr(h: ctypes.c_void_p) -> ZeroTerminatedCsr:
    lib = _g()
    c = ctypes.c_void_p()
    try:
        rc = lib.ktgg_csr_from_raw(h, ctypes.byref(c))
    finally:
        lib.ktgg_raw_free(h)
    if rc:
        _raise(rc)
    return _csr_from_handle(c)


def rmat(scale: int, edgefactor: int = 16, seed: int = 42,
         a: float = 0.57, b: float = 0.19, c: float = 0.19) -> ZeroTerminatedCsr:
    """R-MAT per SURVEY.md §8(d) (Graph500 parameters), canonicalized."""
    lib = _g()
    h = ctypes.c_void_p()
    rc = lib.ktgg_rmat_raw(scale, edgefactor, seed, a, b, c, ctypes.byref(h))
    if rc:
        _raise(rc)
    return _raw_to_csr(h)


def clique_members(n_labels: int, c: int, seed: int) -> np.ndarray:
    """c distinct labels in [0, n_labels): the first c positions of a
    partial Fisher-Yates shuffle driven by numpy's MT19937(seed)."""
    if c > n_labels:
        raise errors.InvalidParameterError("clique larger than the vertex set")
    rng = np.random.Generator(np.random.MT19937(seed))
    draws = rng.integers(0, np.arange(n_labels, n_labels - c, -1, dtype=np.int64), dtype=np.int64)
    chosen = {}
    out = np.empty(c, np.int64)
    for i in range(c):  # swap position i with i + draws[i] (sparse permutation)
        j = i + int(draws[i])
        out[i] = chosen.get(j, j)
        chosen[j] = chosen.get(i, i)
    return out.astype(np.uint64)


def rmat_cliques(scale: int, edgefactor: int = 32, seed: int = 42, sizes=(128, 256, 512, 1024),
                 a: float = 0.57, b: float = 0.19, c: float = 0.19) -> ZeroTerminatedCsr:
    """BASELINE.json configs[4] (SURVEY.md §8(d) "planted cliques"): the
    R-MAT raw pairs plus, before canonicalize, every pair of each planted
    clique; clique of size c_i uses clique_members(2^scale, c_i, seed + i).
    K_max >= max(sizes), with many prune rounds."""
    lib = _g()
    h = ctypes.c_void_p()
    rc = lib.ktgg_rmat_raw(scale, edgefactor, seed, a, b, c, ctypes.byref(h))
    if rc:
        _raise(rc)
    try:
        m = int(lib.ktgg_raw_count(h))
        raw = np.ctypeslib.as_array(lib.ktgg_raw_pairs(h), shape=(2 * m,)).reshape(m, 2).astype(np.uint64)
    finally:
        lib.ktgg_raw_free(h)
    parts = [raw]
    for i, cs in enumerate(sizes):
        mem = clique_members(1 << scale, int(cs), seed + i)
        iu, ju = np.triu_indices(len(mem), 1)
        parts.append(np.stack([mem[iu], mem[ju]], axis=1))
    return csr_from_pairs(np.concatenate(parts))


def erdos_renyi(log_n: int, m: int, seed: int = 42) -> ZeroTerminatedCsr:
    """Erdős–Rényi per SURVEY.md §8(d): m uniform endpoint draws, canonicalized."""
    lib = _g()
    h = ctypes.c_void_p()
    rc = lib.ktgg_er_raw(log_n, m, seed, ctypes.byref(h))
    if rc:
        _raise(rc)
    return _raw_to_csr(h)


def write_csr_cache(g: ZeroTerminatedCsr, path: str) -> None:
    """write_csr_cache (csr_cache.cpp:71-78): the ZTCSR1 binary layout."""
    rc = _g().ktgg_write_csr_cache(path.encode(), _ptr(np.ascontiguousarray(g.row_ptr, np.uint32)), g.num_vertices,
                                   _ptr(np.ascontiguousarray(g.col_idx, np.uint32)), g.total_slots())
    if rc:
        _raise(rc)


def read_csr_cache(path: str) -> ZeroTerminatedCsr:
    """read_csr_cache (csr_cache.cpp:80-111): raises CorruptCacheError with
    the reference's messages."""
    h = ctypes.c_void_p()
    rc = _g().ktgg_read_csr_cache(path.encode(), ctypes.byref(h))
    if rc:
        _raise(rc)
    return _csr_from_handle(h)


def round_work(g: ZeroTerminatedCsr) -> dict:
    """Closed-form merge work of one support pass over g's live edges
    (SURVEY.md §8(d)): L = sum_v d+(d+-1)/2 + d+ d-."""
    w = _Work()
    _g().ktgg_round_work(_ptr(g.row_ptr), g.num_vertices, _ptr(g.col_idx), ctypes.byref(w))
    return {k: getattr(w, k) for k, _ in _Work._fields_}


def validate_csr(g: ZeroTerminatedCsr) -> None:
    """validate_csr (csr.cpp:34-80): raises InvalidInputError naming the first
    violated invariant. Vectorised restatement."""
    n = g.num_vertices
    rp = np.asarray(g.row_ptr, dtype=np.int64)
    col = np.asarray(g.col_idx, dtype=np.int64)
    if n == 0:
        raise errors.InvalidInputError("csr has no vertices")
    if rp.shape[0] != n + 2:
        raise errors.InvalidInputError("row_ptr must have num_vertices + 2 entries")
    if rp[0] != 0 or rp[1] != 0:
        raise errors.InvalidInputError("phantom vertex 0 must own no slots")
    if col.shape[0] > 0xFFFFFFFF:
        raise errors.InvalidInputError("slot count exceeds 32-bit offsets")
    if rp[n + 1] != col.shape[0]:
        raise errors.InvalidInputError("row_ptr end does not match slot count")
    begin, end = rp[1:n + 1], rp[2:n + 2]
    bad = np.nonzero(begin >= end)[0]
    if bad.size:
        raise errors.InvalidInputError(f"row {bad[0] + 1} owns no sentinel slot")
    bad = np.nonzero(col[end - 1] != 0)[0]
    if bad.size:
        raise errors.InvalidInputError(f"row {bad[0] + 1} does not end in a zero slot")
    row_of = np.repeat(np.arange(1, n + 1), end - begin)
    first = np.zeros(col.shape[0], dtype=bool)
    first[begin] = True
    prev = np.where(first, 0, np.concatenate(([0], col[:-1])))
    zero = col == 0
    prev_zero = np.where(first, False, np.concatenate(([False], zero[:-1])))
    v = np.nonzero((~zero) & prev_zero)[0]
    if v.size:
        raise errors.InvalidInputError(f"row {row_of[v[0]]} has a nonzero after a zero slot")
    bound = np.where(first, row_of, prev)
    v = np.nonzero((~zero) & (col <= bound))[0]
    if v.size:
        raise errors.InvalidInputError(
            f"row {row_of[v[0]]} entries are not strictly ascending above the vertex")
    v = np.nonzero(col > n)[0]
    if v.size:
        raise errors.InvalidInputError(f"row {row_of[v[0]]} references vertex beyond n")


def extract_edges(g: ZeroTerminatedCsr, supports: Optional[np.ndarray] = None):
    """extract_edges (csr.cpp:82-106): live (u, v[, support]) in row-major,
    i.e. lexicographic, order. Returns (u, v) or (u, v, s) u32 arrays."""
    n = g.num_vertices
    rp = g.row_ptr.astype(np.int64)
    if supports is not None and supports.shape[0] != g.total_slots():
        raise errors.InvalidParameterError("support array does not match slot count")
    row_of = np.repeat(np.arange(1, n + 1, dtype=np.uint32), np.diff(rp[1:n + 2]))
    live = g.col_idx != 0
    u = row_of[live]
    v = g.col_idx[live]
    if supports is None:
        return u, v
    return u, v, supports[live]

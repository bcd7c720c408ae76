"""CPU oracle for the K-truss hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker / the timed CPU
baseline; the product (paper_2009_07929_b200/) never touches it.

Two layers:
  * `port`: our plain-C restatement (oracle/ktruss_oracle.c -> liboracle.so),
    each function citing the reference lines it follows;
  * `ref`:  the UNMODIFIED reference library compiled from
    /root/reference/proj/src by oracle/Makefile into oracle/_ref/ (C shim
    oracle/ref_capi.cpp). Parity of `port` is pinned against `ref` and
    against the reference's own known-answer vectors (tests/golden/).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_vp = ctypes.c_void_p
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_P = ctypes.POINTER


def _p(a):
    return _vp(a.ctypes.data)


def _u32a(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class _Port:
    def __init__(self):
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run make -C oracle")
        L = ctypes.CDLL(path)
        L.orc_compute_supports.argtypes = [_vp, _u32, _vp, _u64, _vp, ctypes.c_int]
        L.orc_compute_supports.restype = _u64
        L.orc_intersect_tails.argtypes = [_vp, _vp, _u32, _u32, _vp]
        L.orc_intersect_tails.restype = _u32
        L.orc_prune_edges.argtypes = [_vp, _u32, _vp, _vp, _u32, ctypes.c_int]
        L.orc_prune_edges.restype = _u64
        L.orc_run_fixpoint.argtypes = [_vp, _u32, _vp, _u64, _vp, _u32, ctypes.c_int, _vp, _u32]
        L.orc_run_fixpoint.restype = _u32
        L.orc_kmax.argtypes = [_vp, _u32, _vp, _u64, ctypes.c_int]
        L.orc_kmax.restype = _u32
        L.orc_first_overflow_16.argtypes = [_vp, _u64]
        L.orc_first_overflow_16.restype = _u64
        L.orc_round_work.argtypes = [_vp, _u32, _vp, _P(_u64), _P(_u64), _P(_u32)]
        L.orc_brute_supports.argtypes = [_u32, _vp, _u64, _vp]
        L.orc_random_graph_raw.argtypes = [_u32, ctypes.c_double, _u64, _vp]
        L.orc_random_graph_raw.restype = _u64
        L.orc_support_tasks.argtypes = [_vp, _u32, _vp, _u64, _u32, _u32, _u32, _vp]
        L.orc_support_tasks.restype = _u64
        L.orc_task_cost.argtypes = [_vp, _u32, _vp, _u64, _u32, _u64]
        L.orc_task_cost.restype = _u64
        self.L = L

    def compute_supports(self, g, supports=None, threads=1):
        S = np.zeros(g.total_slots(), np.uint32) if supports is None else supports
        col = _u32a(g.col_idx)
        t = self.L.orc_compute_supports(_p(_u32a(g.row_ptr)), g.num_vertices, _p(col), col.shape[0], _p(S),
                                        threads)
        return int(t), S

    def support_tasks(self, g, rank, world, chunk=512):
        """One rank's partial supports under the engine's task partition
        (mirror of the device planner; see ktruss_oracle.c). `chunk` must be
        the engine's (ktg_task_chunk())."""
        S = np.zeros(g.total_slots(), np.uint32)
        t = self.L.orc_support_tasks(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                     g.total_slots(), chunk, rank, world, _p(S))
        return int(t), S

    def task_costs(self, g, chunk=512):
        """Work estimate of every diagonal support task (the multi-GPU split's
        weights, mirror of the engine's k_task_cost)."""
        rp, col = _u32a(g.row_ptr), _u32a(g.col_idx)
        Q = (g.total_slots() + chunk - 1) // chunk
        return np.array([self.L.orc_task_cost(_p(rp), g.num_vertices, _p(col), g.total_slots(), chunk, q)
                         for q in range(Q)], dtype=np.uint64)

    def intersect_tails(self, g, pivot, pred, S):
        return int(self.L.orc_intersect_tails(_p(_u32a(g.row_ptr)), _p(_u32a(g.col_idx)), pivot, pred, _p(S)))

    def prune_edges(self, g, S, k, threads=1):
        """Mutates g.col_idx (must be a u32 array)."""
        return int(self.L.orc_prune_edges(_p(_u32a(g.row_ptr)), g.num_vertices, _p(g.col_idx), _p(_u32a(S)),
                                          k, threads))

    def run_fixpoint(self, g, k, threads=1):
        """Returns (col, S, removed_per_iteration) on a copy."""
        col = _u32a(g.col_idx).copy()
        S = np.zeros(col.shape[0], np.uint32)
        cap = 1 << 16
        hist = np.zeros(cap, np.uint64)
        it = self.L.orc_run_fixpoint(_p(_u32a(g.row_ptr)), g.num_vertices, _p(col), col.shape[0], _p(S), k,
                                     threads, _p(hist), cap)
        return col, S, [int(x) for x in hist[:min(it, cap)]]

    def kmax(self, g, threads=1):
        return int(self.L.orc_kmax(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                   g.total_slots(), threads))

    def first_overflow_16(self, S):
        r = int(self.L.orc_first_overflow_16(_p(_u32a(S)), S.shape[0]))
        return None if r == 2**64 - 1 else r

    def round_work(self, g):
        L, live, md = _u64(), _u64(), _u32()
        self.L.orc_round_work(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)), ctypes.byref(L),
                              ctypes.byref(live), ctypes.byref(md))
        return {"L": L.value, "live_edges": live.value, "max_out_degree": md.value}

    def brute_supports(self, n, edges):
        e = _u32a(np.asarray(edges).reshape(-1, 2))
        out = np.zeros(e.shape[0], np.uint32)
        self.L.orc_brute_supports(n, _p(e), e.shape[0], _p(out))
        return out

    def random_graph_raw(self, n, p, seed):
        buf = np.zeros(max(1, n * (n - 1)), np.uint64)
        m = self.L.orc_random_graph_raw(n, p, seed, _p(buf))
        return buf[:2 * m].reshape(-1, 2)

    def truss_edges(self, g, k, threads=1):
        """(u, v, S) survivors of run_fixpoint at k, lexicographic -- what
        ktruss() returns (truss.cpp:57-71, csr.cpp:93-106)."""
        col, S, hist = self.run_fixpoint(g, k, threads)
        n = g.num_vertices
        rp = g.row_ptr.astype(np.int64)
        row_of = np.repeat(np.arange(1, n + 1, dtype=np.uint32), np.diff(rp[1:n + 2]))
        live = col != 0
        return np.stack([row_of[live], col[live], S[live]], axis=1).astype(np.uint32), hist


class _Ref:
    """The unmodified reference library (oracle/_ref/libktruss_ref.so)."""

    def __init__(self):
        path = os.path.join(HERE, "_ref", "libktruss_ref.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run make -C oracle (needs /root/reference at build time)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_last_error_slot.restype = _u64
        L.ref_compute_supports.argtypes = [_vp, _u32, _vp, _u64, _vp, _u64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _P(_u64)]
        L.ref_prune_edges.argtypes = [_vp, _u32, _vp, _u64, _vp, _u64, _u32, ctypes.c_int, _P(_u64)]
        L.ref_run_fixpoint.argtypes = [_vp, _u32, _vp, _u64, _vp, _u32, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, _vp, _u32, _P(_u32), _P(ctypes.c_double)]
        L.ref_ktruss.argtypes = [_vp, _u32, _vp, _u64, _u32, ctypes.c_int, ctypes.c_int, _P(_vp)]
        L.ref_kmax_search.argtypes = [_vp, _u32, _vp, _u64, ctypes.c_int, ctypes.c_int, _P(_vp)]
        for f in ("ref_truss_kmax", "ref_truss_k", "ref_truss_iterations"):
            getattr(L, f).argtypes = [_vp]
            getattr(L, f).restype = _u32
        L.ref_truss_num_edges.argtypes = [_vp]
        L.ref_truss_num_edges.restype = _u64
        L.ref_truss_removed.argtypes = [_vp, _vp]
        L.ref_truss_edges.argtypes = [_vp, _vp, _vp, _vp]
        L.ref_truss_free.argtypes = [_vp]
        L.ref_canonicalize_csr.argtypes = [_vp, _u64, _P(_vp)]
        L.ref_random_graph_csr.argtypes = [_u32, ctypes.c_double, _u64, _P(_vp)]
        L.ref_csr_n.argtypes = [_vp]
        L.ref_csr_n.restype = _u32
        L.ref_csr_slots.argtypes = [_vp]
        L.ref_csr_slots.restype = _u64
        L.ref_csr_copy.argtypes = [_vp, _vp, _vp]
        L.ref_csr_free.argtypes = [_vp]
        L.ref_validate_csr.argtypes = [_vp, _u32, _vp, _u64]
        L.ref_oracle_kmax.argtypes = [_vp, _u32, _vp, _u64]
        L.ref_oracle_kmax.restype = _u32
        L.ref_oracle_triangle_count.argtypes = [_vp, _u32, _vp, _u64]
        L.ref_oracle_triangle_count.restype = _u64
        L.ref_oracle_truss.argtypes = [_vp, _u32, _vp, _u64, _u32, _vp, _vp, _vp]
        L.ref_oracle_truss.restype = _u64
        L.ref_hardware_threads.restype = ctypes.c_int
        L.ref_write_csr_cache.argtypes = [ctypes.c_char_p, _vp, _u32, _vp, _u64]
        L.ref_read_csr_cache.argtypes = [ctypes.c_char_p, _P(_vp)]
        L.ref_rmat_csr.argtypes = [_u32, _u32, _u64, ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp, _u64,
                                   ctypes.c_int, _P(_vp)]
        L.ref_er_csr.argtypes = [_u32, _u64, _u64, ctypes.c_int, _P(_vp)]
        L.ref_fine_sample.argtypes = [_vp, _u32, _vp, _u64, _vp, _u32, _u32, ctypes.c_int, _P(_u64),
                                      _P(ctypes.c_double)]
        self.L = L

    def _err(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def _csr(self, h):
        from paper_2009_07929_b200.graph import ZeroTerminatedCsr
        n = self.L.ref_csr_n(h)
        slots = self.L.ref_csr_slots(h)
        rp = np.empty(n + 2, np.uint32)
        col = np.empty(slots, np.uint32)
        self.L.ref_csr_copy(h, _p(rp), _p(col))
        self.L.ref_csr_free(h)
        return ZeroTerminatedCsr(int(n), rp, col)

    def random_graph(self, n, p, seed):
        h = _vp()
        self._err(self.L.ref_random_graph_csr(n, p, seed, ctypes.byref(h)))
        return self._csr(h)

    def canonicalize(self, pairs):
        a = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1, 2))
        h = _vp()
        self._err(self.L.ref_canonicalize_csr(_p(a), a.shape[0], ctypes.byref(h)))
        return self._csr(h)

    def rmat(self, scale, edgefactor=16, seed=42, extra_pairs=None, fast=True, a=0.57, b=0.19, c=0.19):
        """SURVEY §8(d) R-MAT (+ optional extra label pairs, e.g. planted
        cliques), canonicalized by the reference canonicalize (fast=False) or
        its parallel restatement (fast=True), built by the reference build_csr."""
        ex = np.zeros((0, 2), np.uint64) if extra_pairs is None else np.ascontiguousarray(extra_pairs, np.uint64)
        h = _vp()
        self._err(self.L.ref_rmat_csr(scale, edgefactor, seed, a, b, c, _p(ex), ex.shape[0], int(fast),
                                      ctypes.byref(h)))
        return self._csr(h)

    def erdos_renyi(self, log_n, m, seed=42, fast=True):
        h = _vp()
        self._err(self.L.ref_er_csr(log_n, m, seed, int(fast), ctypes.byref(h)))
        return self._csr(h)

    def fine_sample(self, g, stride, phase, threads, supports=None):
        """support.cpp:115-127 (reference intersect_tails per slot) over the
        256-slot chunks c % stride == phase. Returns (triangles, S, ms)."""
        S = np.zeros(g.total_slots(), np.uint32) if supports is None else supports
        t, ms = _u64(), ctypes.c_double()
        self._err(self.L.ref_fine_sample(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                         g.total_slots(), _p(S), stride, phase, threads, ctypes.byref(t),
                                         ctypes.byref(ms)))
        return int(t.value), S, ms.value

    def compute_supports(self, g, strategy=2, threads=1, width16=False, supports=None):
        S = np.zeros(g.total_slots(), np.uint32) if supports is None else supports
        t = _u64()
        rc = self.L.ref_compute_supports(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                         g.total_slots(), _p(S), S.shape[0], strategy, threads, int(width16),
                                         ctypes.byref(t))
        return rc, int(t.value), S

    def prune_edges(self, g, S, k, threads=1):
        col = _u32a(g.col_idx).copy()
        r = _u64()
        rc = self.L.ref_prune_edges(_p(_u32a(g.row_ptr)), g.num_vertices, _p(col), col.shape[0], _p(_u32a(S)),
                                    S.shape[0], k, threads, ctypes.byref(r))
        return rc, int(r.value), col

    def run_fixpoint(self, g, k, strategy=2, threads=1):
        """Returns (col, S, removed_per_iteration, elapsed_ms) on a copy."""
        col = _u32a(g.col_idx).copy()
        S = np.zeros(col.shape[0], np.uint32)
        cap = 1 << 16
        hist = np.zeros(cap, np.uint64)
        it = _u32()
        ms = ctypes.c_double()
        self._err(self.L.ref_run_fixpoint(_p(_u32a(g.row_ptr)), g.num_vertices, _p(col), col.shape[0], _p(S),
                                          k, strategy, threads, 0, _p(hist), cap, ctypes.byref(it),
                                          ctypes.byref(ms)))
        return col, S, [int(x) for x in hist[:min(it.value, cap)]], ms.value

    def _truss(self, h):
        m = self.L.ref_truss_num_edges(h)
        u = np.empty(m, np.uint32)
        v = np.empty(m, np.uint32)
        s = np.empty(m, np.uint32)
        self.L.ref_truss_edges(h, _p(u), _p(v), _p(s))
        it = self.L.ref_truss_iterations(h)
        rem = np.empty(it, np.uint64)
        self.L.ref_truss_removed(h, _p(rem))
        kmax = self.L.ref_truss_kmax(h)
        k = self.L.ref_truss_k(h)
        self.L.ref_truss_free(h)
        return {"k": int(k), "k_max": int(kmax), "edges": np.stack([u, v, s], axis=1),
                "iterations": int(it), "removed": [int(x) for x in rem]}

    def ktruss(self, g, k, strategy=2, threads=1):
        h = _vp()
        self._err(self.L.ref_ktruss(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)), g.total_slots(),
                                    k, strategy, threads, ctypes.byref(h)))
        return self._truss(h)

    def kmax_search(self, g, strategy=2, threads=1):
        h = _vp()
        self._err(self.L.ref_kmax_search(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                         g.total_slots(), strategy, threads, ctypes.byref(h)))
        return self._truss(h)

    def write_cache(self, g, path):
        self._err(self.L.ref_write_csr_cache(path.encode(), _p(_u32a(g.row_ptr)), g.num_vertices,
                                             _p(_u32a(g.col_idx)), g.total_slots()))

    def read_cache(self, path):
        """(graph, None) or (None, CorruptCacheError message)."""
        h = _vp()
        rc = self.L.ref_read_csr_cache(path.encode(), ctypes.byref(h))
        if rc:
            return None, self.L.ref_last_error().decode()
        return self._csr(h), None

    def validate(self, g):
        rc = self.L.ref_validate_csr(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)), g.total_slots())
        return None if rc == 0 else self.L.ref_last_error().decode()

    def oracle_kmax(self, g):
        return int(self.L.ref_oracle_kmax(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                          g.total_slots()))

    def oracle_triangles(self, g):
        return int(self.L.ref_oracle_triangle_count(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)),
                                                    g.total_slots()))

    def oracle_truss(self, g, k):
        m = int(np.count_nonzero(g.col_idx))
        u = np.empty(max(m, 1), np.uint32)
        v = np.empty(max(m, 1), np.uint32)
        s = np.empty(max(m, 1), np.uint32)
        c = self.L.ref_oracle_truss(_p(_u32a(g.row_ptr)), g.num_vertices, _p(_u32a(g.col_idx)), g.total_slots(),
                                    k, _p(u), _p(v), _p(s))
        return np.stack([u[:c], v[:c], s[:c]], axis=1)


_port = None
_ref = None


def clique_members(n_labels, c, seed):
    """c distinct labels of [0, n_labels): the first c positions of a partial
    Fisher-Yates shuffle driven by numpy's MT19937(seed) (the planted-clique
    spec of BASELINE configs[4], restated independently of the product)."""
    rng = np.random.Generator(np.random.MT19937(seed))
    draws = rng.integers(0, np.arange(n_labels, n_labels - c, -1, dtype=np.int64), dtype=np.int64)
    swapped = {}
    out = np.empty(c, np.uint64)
    for i in range(c):
        j = i + int(draws[i])
        out[i] = swapped.get(j, j)
        swapped[j] = swapped.get(i, i)
    return out


def clique_pairs(n_labels, sizes, seed):
    """Every pair of each planted clique; clique i uses seed + i."""
    parts = []
    for i, c in enumerate(sizes):
        mem = clique_members(n_labels, int(c), seed + i)
        iu, ju = np.triu_indices(len(mem), 1)
        parts.append(np.stack([mem[iu], mem[ju]], axis=1))
    return np.concatenate(parts).astype(np.uint64)


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libktruss_ref.so"))

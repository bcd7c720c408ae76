"""Host-side mirror of the reference K-truss API over the sm_100a engine.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/ktruss/support.hpp and truss.hpp); every call
goes through the C ABI of libktg.so (include/ktg.h). There is no CPU path:
without the engine library or a B200 these functions raise.

    compute_supports  support.hpp:52-54   support.cpp:93-132
    reset_supports    support.hpp:56      support.cpp:134-136
    intersect_tails   support.hpp:44-45   support.cpp:64-91
    prune_edges       truss.hpp:38-39     truss.cpp:9-37
    run_fixpoint      truss.hpp:62-63     truss.cpp:41-53
    ktruss            truss.hpp:44-45     truss.cpp:57-71
    kmax_search       truss.hpp:56        truss.cpp:73-103
"""
from __future__ import annotations

import ctypes
import enum
import os
import sys
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import errors
from ._lib import engine_lib
from .graph import ZeroTerminatedCsr

_vp = ctypes.c_void_p
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64


class Strategy(enum.IntEnum):
    """support.hpp:12-16. All three run the same device path (identical
    results are the reference's own contract)."""
    Serial = 0
    Coarse = 1
    Fine = 2


class SupportWidth(enum.IntEnum):
    """support.hpp:21-24."""
    Bits32 = 32
    Bits16 = 16


def to_string(s: Strategy) -> str:
    """support.cpp:13-20."""
    return {Strategy.Serial: "serial", Strategy.Coarse: "coarse", Strategy.Fine: "fine"}.get(s, "?")


def strategy_from_string(name: str) -> Optional[Strategy]:
    """support.cpp:22-27."""
    return {"serial": Strategy.Serial, "coarse": Strategy.Coarse, "fine": Strategy.Fine}.get(name)


def hardware_threads() -> int:
    """support.cpp:29-32."""
    return os.cpu_count() or 1


@dataclass
class SupportArray:
    """support.hpp:28-35: one u32 counter per CSR slot."""
    counts: np.ndarray

    @classmethod
    def zeros(cls, slot_count: int) -> "SupportArray":
        return cls(np.zeros(slot_count, dtype=np.uint32))

    def size(self) -> int:
        return int(self.counts.shape[0])


RoundObserver = Callable[[ZeroTerminatedCsr, SupportArray, int], None]


@dataclass
class TrussOptions:
    """truss.hpp:28-33, plus engine flags (host_loop, naive_support) used by
    tests to cross-check the device-resident loop and the optimised kernel."""
    strategy: Strategy = Strategy.Fine
    threads: int = 1
    width: SupportWidth = SupportWidth.Bits32
    observer: Optional[RoundObserver] = None
    host_loop: bool = False
    naive_support: bool = False
    label_order: bool = False   # run on the caller's CSR, not the degree-ordered copy
    recompute: bool = False     # full support pass every round (no carried supports)
    no_degree_bound: bool = False  # round 0 counts every pivot (no min-degree skip)
    device: int = -1


class TrussResult:
    """truss.hpp:12-21. The surviving edges in lexicographic order (the
    reference's vector<SupportedEdge>) as three u32 columns `u`, `v`,
    `support`; `edges` stacks them into an (m, 3) array on first use."""

    def __init__(self, k: int, u: np.ndarray, v: np.ndarray, support: np.ndarray, iterations: int,
                 removed_per_iteration: List[int]):
        self.k = k
        self.u, self.v, self.support = u, v, support
        self.iterations = iterations
        self.removed_per_iteration = removed_per_iteration
        self._edges = None

    @property
    def edges(self) -> np.ndarray:
        if self._edges is None:
            self._edges = np.stack([self.u, self.v, self.support], axis=1)
        return self._edges

    def __len__(self) -> int:
        return int(self.u.shape[0])

    @property
    def nbytes(self) -> int:
        return int(self.u.nbytes + self.v.nbytes + self.support.nbytes)

    def edge_tuples(self):
        return [tuple(int(x) for x in r) for r in self.edges]


@dataclass
class KmaxResult:
    """truss.hpp:47-50."""
    k_max: int
    truss: TrussResult


# ---------------------------------------------------------------------------
# ctypes plumbing
# ---------------------------------------------------------------------------
ROUND_CB = ctypes.CFUNCTYPE(None, ctypes.POINTER(_u32), ctypes.POINTER(_u32), _u64, _u64, _vp)
ALLREDUCE_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(_u32), _u64, _vp, _vp)
# ktg_peer_cb(phase, d_supports, slots, span, d_triangles, stream, user)
PEER_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, _vp, _u64, _u64, _vp, _vp, _vp)


class _Options(ctypes.Structure):
    _fields_ = [("struct_size", _u32), ("device", ctypes.c_int32), ("strategy", _u32),
                ("width_bits", _u32), ("flags", _u32), ("stream", _vp),
                ("observer", ROUND_CB), ("observer_user", _vp)]


class _RunInfo(ctypes.Structure):
    _fields_ = [("iterations", _u32), ("live_edges", _u64), ("triangles", _u64),
                ("max_support", _u32), ("device_ms", ctypes.c_double), ("carried", _u32)]


class _RoundWork(ctypes.Structure):
    _fields_ = [("live_edges", _u64), ("L", _u64), ("triangles", _u64), ("removed", _u64),
                ("support_ms", ctypes.c_double), ("full_pass", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("L_tail", _u64), ("delta_cost", _u64), ("keep_cost", _u64),
                ("delta_pieces", ctypes.c_uint32), ("carried", ctypes.c_uint32)]


FLAG_HOST_LOOP = 1
FLAG_NAIVE_SUPPORT = 2
FLAG_COLLECT_WORK = 4
FLAG_TIME_SUPPORT = 8
FLAG_LABEL_ORDER = 16
FLAG_RECOMPUTE = 32
FLAG_NO_DEGREE_BOUND = 64

_configured = False


def lib():
    global _configured
    L = engine_lib()
    if not _configured:
        P = ctypes.POINTER
        L.ktg_last_error.restype = ctypes.c_char_p
        L.ktg_last_error_slot.restype = _u64
        L.ktg_version.restype = ctypes.c_char_p
        L.ktg_device_available.restype = ctypes.c_int
        L.ktg_task_chunk.restype = _u32
        L.ktg_options_init.argtypes = [P(_Options)]
        L.ktg_compute_supports.argtypes = [_vp, _u32, _vp, _u64, _vp, _u64, P(_Options), P(_u64)]
        L.ktg_reset_supports.argtypes = [_vp, _u64]
        L.ktg_intersect_tails.argtypes = [_vp, _u32, _vp, _u64, _u32, _u32, _vp, P(_u32)]
        L.ktg_prune_edges.argtypes = [_vp, _u32, _vp, _u64, _vp, _u64, _u32, P(_Options), P(_u64)]
        L.ktg_run_fixpoint.argtypes = [_vp, _u32, _vp, _u64, _vp, _u64, _u32, P(_Options), _vp, _u32,
                                       P(_u32)]
        L.ktg_ktruss.argtypes = [_vp, _u32, _vp, _u64, _u32, P(_Options), _vp, _vp, _vp, _u64, P(_u64),
                                 _vp, _u32, P(_u32)]
        L.ktg_kmax_search.argtypes = [_vp, _u32, _vp, _u64, P(_Options), P(_u32), _vp, _vp, _vp, _u64,
                                      P(_u64), _vp, _u32, P(_u32)]
        L.ktg_engine_create.argtypes = [P(_Options), P(_vp)]
        L.ktg_engine_destroy.argtypes = [_vp]
        L.ktg_engine_load.argtypes = [_vp, _vp, _u32, _vp, _u64]
        L.ktg_engine_load_device.argtypes = [_vp, _vp, _u32, _vp, _u64]
        L.ktg_engine_load_cache.argtypes = [_vp, ctypes.c_char_p]
        L.ktg_engine_build_csr.argtypes = [_vp, _vp, _u64, ctypes.c_int]
        L.ktg_engine_csr_info.argtypes = [_vp, P(_u32), P(_u64)]
        L.ktg_engine_read_csr.argtypes = [_vp, _vp, _vp, _vp]
        L.ktg_engine_reset.argtypes = [_vp]
        L.ktg_engine_run.argtypes = [_vp, _u32, _vp, _u32, P(_u32)]
        L.ktg_engine_support_pass.argtypes = [_vp, P(_u64)]
        L.ktg_engine_sync.argtypes = [_vp]
        L.ktg_engine_info.argtypes = [_vp, P(_RunInfo)]
        L.ktg_engine_round_work.argtypes = [_vp, P(_RoundWork), _u32]
        L.ktg_engine_round_work.restype = _u32
        L.ktg_engine_read.argtypes = [_vp, _vp, _vp]
        L.ktg_engine_device_state.argtypes = [_vp, P(_vp), P(_vp), P(_vp)]
        L.ktg_engine_extract.argtypes = [_vp, _vp, _vp, _vp, _u64, P(_u64)]
        L.ktg_engine_set_partition.argtypes = [_vp, _u32, _u32, ALLREDUCE_CB, _vp]
        L.ktg_engine_support_buffers.argtypes = [_vp, P(_vp), P(_vp), P(_u64)]
        L.ktg_engine_set_peers.argtypes = [_vp, _u32, _u32, _vp, _vp, PEER_CB, _vp]
        L.ktg_device_copy.argtypes = [_vp, _vp, _u64, _vp]
        L.ktg_ipc_handle.argtypes = [_vp, _vp]
        L.ktg_ipc_open.argtypes = [_vp, P(_vp)]
        L.ktg_ipc_close.argtypes = [_vp]
        L.ktg_nccl_unique_id.argtypes = [_vp]
        L.ktg_engine_set_nccl.argtypes = [_vp, _u32, _u32, _vp]
        try:  # (older builds used for A/B timing lack the peer group)
            L.ktg_engine_group_area.argtypes = [_vp, P(_vp), P(_u64)]
            L.ktg_engine_set_group.argtypes = [_vp, _u32, _u32, _vp, _vp, _vp]
        except AttributeError:
            pass
        _configured = True
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    L = lib()
    msg = L.ktg_last_error().decode()
    if rc == 1:
        raise errors.InvalidParameterError(msg)
    if rc == 2:
        raise errors.SupportOverflowError(int(L.ktg_last_error_slot()), msg)
    if rc == 3:
        raise errors.InvalidInputError(msg)
    if rc == 4:
        raise errors.CorruptCacheError(msg)
    if rc == 8:
        raise errors.EmptyGraphError(msg)
    if rc == 7:
        raise MemoryError(msg)
    raise errors.DeviceError(msg)


def _p(a: np.ndarray) -> _vp:
    return _vp(a.ctypes.data)


def _u32arr(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a


def _options(o: Optional[TrussOptions], keep=None) -> _Options:
    c = _Options()
    lib().ktg_options_init(ctypes.byref(c))
    if o is None:
        return c
    c.strategy = int(o.strategy)
    c.width_bits = int(o.width)
    c.device = o.device
    flags = 0
    if o.host_loop:
        flags |= FLAG_HOST_LOOP
    if o.naive_support:
        flags |= FLAG_NAIVE_SUPPORT
    if o.label_order:
        flags |= FLAG_LABEL_ORDER
    if o.recompute:
        flags |= FLAG_RECOMPUTE
    if o.no_degree_bound:
        flags |= FLAG_NO_DEGREE_BOUND
    c.flags = flags
    if o.observer is not None and keep is not None:
        obs = o.observer
        n_state = keep["graph"]

        def tramp(col_p, s_p, slots, removed, _user):
            col = np.ctypeslib.as_array(col_p, shape=(slots,)).copy()
            sup = np.ctypeslib.as_array(s_p, shape=(slots,)).copy()
            g = ZeroTerminatedCsr(n_state.num_vertices, n_state.row_ptr, col)
            obs(g, SupportArray(sup), int(removed))

        cb = ROUND_CB(tramp)
        keep["cb"] = cb
        c.observer = cb
    return c


class _ResultPool:
    """Page-locked (u, v, support) result columns reused across calls.

    Pinning fresh host memory per call costs more than the fixpoint itself
    (cudaHostAlloc of ~190 MB at R-MAT s20 is ~7 ms), so each call borrows a
    pooled buffer. A buffer is free again once no array viewing it is alive
    (the refcount of the ndarray that owns the pinned pages). Results much
    smaller than the buffer are copied out so a kept result does not pin a
    whole buffer."""

    MAX_POOLED = 4
    COPY_OUT_BYTES = 4 << 20

    def __init__(self):
        import threading
        self._owners = []
        # the C engines are per thread, so calls may run concurrently: the
        # free check and the caller's reference must not interleave
        self._lock = threading.Lock()

    def take(self, cap: int):
        with self._lock:
            return self._take(cap)

    def _take(self, cap: int):
        words = 3 * max(cap, 1)
        for owner in self._owners:
            # refs: the pool list, this loop variable, getrefcount's argument
            if owner.shape[0] >= words and sys.getrefcount(owner) <= 3:
                return owner
        owner = self._alloc(1 << max(20, (words - 1).bit_length()))  # power-of-two classes
        if owner is None:
            return np.empty(words, np.int32)
        if len(self._owners) >= self.MAX_POOLED:  # drop the smallest free buffer
            free = [i for i in range(len(self._owners)) if sys.getrefcount(self._owners[i]) <= 2]
            if free:
                del self._owners[min(free, key=lambda i: self._owners[i].shape[0])]
        if len(self._owners) < self.MAX_POOLED:
            self._owners.append(owner)
        return owner

    @staticmethod
    def _alloc(size: int):
        try:
            import torch
            if torch.cuda.is_available():
                return torch.empty(size, dtype=torch.int32, pin_memory=True).numpy()
        except Exception:
            pass
        return None

    @staticmethod
    def columns(owner, cap: int):
        buf = owner.view(np.uint32)
        cap = max(cap, 1)
        return buf[:cap], buf[cap:2 * cap], buf[2 * cap:3 * cap]

    @classmethod
    def finish(cls, u, v, sup, m: int):
        if 12 * m <= cls.COPY_OUT_BYTES:
            return u[:m].copy(), v[:m].copy(), sup[:m].copy()
        return u[:m], v[:m], sup[:m]


_result_pool = _ResultPool()


def _check_threads(threads: int) -> None:
    if threads < 1:
        raise errors.InvalidParameterError("thread count must be >= 1")


# ---------------------------------------------------------------------------
# Reference API
# ---------------------------------------------------------------------------

def intersect_tails(graph: ZeroTerminatedCsr, pivot_slot: int, predecessor: int,
                    supports: SupportArray) -> int:
    """support.cpp:64-91. Mutates supports; returns the match count (the
    caller owns the pivot add)."""
    found = _u32()
    col = _u32arr(graph.col_idx)
    _check(lib().ktg_intersect_tails(_p(_u32arr(graph.row_ptr)), graph.num_vertices, _p(col),
                                     col.shape[0], pivot_slot, predecessor, _p(supports.counts),
                                     ctypes.byref(found)))
    return int(found.value)


def compute_supports(graph: ZeroTerminatedCsr, supports: SupportArray,
                     strategy: Strategy = Strategy.Fine, threads: int = 1,
                     width: SupportWidth = SupportWidth.Bits32) -> int:
    """support.cpp:93-132: adds per-slot triangle counts into `supports`
    (required zero on entry), returns the triangle total."""
    _check_threads(threads)
    if supports.counts.dtype != np.uint32 or not supports.counts.flags.c_contiguous:
        supports.counts = _u32arr(supports.counts)
    o = _options(TrussOptions(strategy=strategy, threads=threads, width=width))
    tri = _u64()
    col = _u32arr(graph.col_idx)
    _check(lib().ktg_compute_supports(_p(_u32arr(graph.row_ptr)), graph.num_vertices, _p(col),
                                      col.shape[0], _p(supports.counts), supports.size(),
                                      ctypes.byref(o), ctypes.byref(tri)))
    return int(tri.value)


def reset_supports(supports: SupportArray) -> None:
    """support.cpp:134-136."""
    supports.counts[:] = 0


def prune_edges(graph: ZeroTerminatedCsr, supports: SupportArray, k: int, threads: int = 1) -> int:
    """truss.cpp:9-37: in-place stable compaction of graph.col_idx; returns
    the removed count. supports is read only."""
    if k < 2:
        raise errors.InvalidParameterError("k must be >= 2")
    _check_threads(threads)
    if supports.size() != graph.total_slots():
        raise errors.InvalidParameterError("support array does not match slot count")
    graph.col_idx = _u32arr(graph.col_idx)
    removed = _u64()
    o = _options(None)
    _check(lib().ktg_prune_edges(_p(_u32arr(graph.row_ptr)), graph.num_vertices, _p(graph.col_idx),
                                 graph.total_slots(), _p(_u32arr(supports.counts)), supports.size(), k,
                                 ctypes.byref(o), ctypes.byref(removed)))
    return int(removed.value)


def run_fixpoint(graph: ZeroTerminatedCsr, supports: SupportArray, k: int,
                 options: Optional[TrussOptions] = None) -> List[int]:
    """detail::run_fixpoint (truss.cpp:41-53): mutates graph.col_idx and
    supports in place; returns the per-round removal counts (last is 0)."""
    options = options or TrussOptions()
    _check_threads(options.threads)
    if supports.size() != graph.total_slots():
        raise errors.InvalidParameterError("support array does not match slot count")
    if k < 2:
        raise errors.InvalidParameterError("k must be >= 2")
    graph.col_idx = _u32arr(graph.col_idx)
    supports.counts = _u32arr(supports.counts)
    keep = {"graph": graph}
    o = _options(options, keep)
    cap = 1 << 16
    hist = np.zeros(cap, dtype=np.uint64)
    it = _u32()
    _check(lib().ktg_run_fixpoint(_p(_u32arr(graph.row_ptr)), graph.num_vertices, _p(graph.col_idx),
                                  graph.total_slots(), _p(supports.counts), supports.size(), k,
                                  ctypes.byref(o), _p(hist), cap, ctypes.byref(it)))
    return [int(x) for x in hist[:min(it.value, cap)]]


def ktruss(graph: ZeroTerminatedCsr, k: int, options: Optional[TrussOptions] = None) -> TrussResult:
    """truss.cpp:57-71: fixpoint on a private copy; survivors with their
    converged supports."""
    if k < 2:
        raise errors.InvalidParameterError("k must be >= 2")
    options = options or TrussOptions()
    _check_threads(options.threads)
    col = _u32arr(graph.col_idx)
    cap_e = max(col.shape[0] - graph.num_vertices, 1)  # >= live edges
    owner = _result_pool.take(cap_e)
    u, v, sup = _ResultPool.columns(owner, cap_e)
    num = _u64()
    hcap = 1 << 16
    hist = np.zeros(hcap, dtype=np.uint64)
    it = _u32()
    keep = {"graph": graph}
    o = _options(options, keep)
    _check(lib().ktg_ktruss(_p(_u32arr(graph.row_ptr)), graph.num_vertices, _p(col), col.shape[0], k,
                            ctypes.byref(o), _p(u), _p(v), _p(sup), cap_e,
                            ctypes.byref(num), _p(hist), hcap, ctypes.byref(it)))
    m = int(num.value)
    u, v, sup = _ResultPool.finish(u, v, sup, m)
    del owner
    return TrussResult(k, u, v, sup, int(it.value), [int(x) for x in hist[:min(it.value, hcap)]])


def kmax_search(graph: ZeroTerminatedCsr, options: Optional[TrussOptions] = None) -> KmaxResult:
    """truss.cpp:73-103: largest k with a non-empty k-truss, and that truss."""
    options = options or TrussOptions()
    _check_threads(options.threads)
    col = _u32arr(graph.col_idx)
    cap_e = max(col.shape[0] - graph.num_vertices, 1)
    owner = _result_pool.take(cap_e)
    u, v, sup = _ResultPool.columns(owner, cap_e)
    num = _u64()
    hcap = 1 << 16
    hist = np.zeros(hcap, dtype=np.uint64)
    it = _u32()
    kmax = _u32()
    keep = {"graph": graph}
    o = _options(options, keep)
    _check(lib().ktg_kmax_search(_p(_u32arr(graph.row_ptr)), graph.num_vertices, _p(col), col.shape[0],
                                 ctypes.byref(o), ctypes.byref(kmax), _p(u), _p(v), _p(sup),
                                 cap_e, ctypes.byref(num), _p(hist), hcap, ctypes.byref(it)))
    m = int(num.value)
    u, v, sup = _ResultPool.finish(u, v, sup, m)
    del owner
    tr = TrussResult(int(kmax.value), u, v, sup, int(it.value),
                     [int(x) for x in hist[:min(it.value, hcap)]])
    return KmaxResult(int(kmax.value), tr)


class detail:  # namespace ktruss::detail (truss.hpp:58-63)
    run_fixpoint = staticmethod(run_fixpoint)


# ---------------------------------------------------------------------------
# Device-resident engine (what the benchmark times)
# ---------------------------------------------------------------------------

def device_copy(dst: int, src: int, nbytes: int, stream: Optional[int] = None) -> None:
    """cudaMemcpyAsync(cudaMemcpyDefault) + synchronize (device or host
    pointers), for peer-exchange callbacks."""
    _check(lib().ktg_device_copy(dst, src, nbytes, stream))


def ipc_handle(d_ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (a support buffer)."""
    buf = (ctypes.c_uint8 * 64)()
    _check(lib().ktg_ipc_handle(d_ptr, buf))
    return bytes(buf)


def ipc_open(handle: bytes) -> int:
    """Maps a peer process's allocation into this one; returns the pointer."""
    buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = _vp()
    _check(lib().ktg_ipc_open(buf, ctypes.byref(p)))
    return p.value


def ipc_close(d_ptr: int) -> None:
    _check(lib().ktg_ipc_close(d_ptr))


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) for Engine.set_nccl."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().ktg_nccl_unique_id(buf))
    return bytes(buf)


class Engine:
    """A graph resident in HBM with its pristine copy; ktg_engine_* calls."""

    def __init__(self, graph: Optional[ZeroTerminatedCsr] = None, options: Optional[TrussOptions] = None,
                 collect_work: bool = False, time_support: bool = False, stream: Optional[int] = None):
        L = lib()
        self._keep = {"graph": graph}
        o = _options(options, self._keep)
        if collect_work:
            o.flags |= FLAG_COLLECT_WORK
        if time_support:
            o.flags |= FLAG_TIME_SUPPORT
        if stream is not None:
            o.stream = _vp(stream)
        self._h = _vp()
        _check(L.ktg_engine_create(ctypes.byref(o), ctypes.byref(self._h)))
        self.graph = None
        if graph is not None:
            self.load(graph)

    def close(self):
        if self._h:
            lib().ktg_engine_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, graph: ZeroTerminatedCsr) -> None:
        self.graph = graph
        self._keep["graph"] = graph
        rp, col = _u32arr(graph.row_ptr), _u32arr(graph.col_idx)
        _check(lib().ktg_engine_load(self._h, _p(rp), graph.num_vertices, _p(col), col.shape[0]))

    def build_csr(self, pairs) -> ZeroTerminatedCsr:
        """canonicalize + build_csr on the device from raw (label, label)
        pairs; the result is loaded and also returned
        (host copy with original_ids)."""
        a = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1, 2))
        _check(lib().ktg_engine_build_csr(self._h, _p(a), a.shape[0], 0))
        g = self.csr()
        self.graph = g
        self._keep["graph"] = g
        return g

    def csr(self) -> ZeroTerminatedCsr:
        """The loaded (pristine) graph copied to the host."""
        n, slots = _u32(), _u64()
        _check(lib().ktg_engine_csr_info(self._h, ctypes.byref(n), ctypes.byref(slots)))
        rp = np.empty(n.value + 2, np.uint32)
        col = np.empty(slots.value, np.uint32)
        ids = np.empty(n.value + 1, np.uint64)
        rc = lib().ktg_engine_read_csr(self._h, _p(rp), _p(col), _p(ids))
        if rc == 1:  # not built on device: no original ids
            _check(lib().ktg_engine_read_csr(self._h, _p(rp), _p(col), None))
            ids = None
        else:
            _check(rc)
        return ZeroTerminatedCsr(int(n.value), rp, col, ids)

    def load_cache(self, path: str) -> None:
        """ZTCSR1 file straight into HBM (validated on the device)."""
        _check(lib().ktg_engine_load_cache(self._h, path.encode()))
        import numpy as _np  # shape info for extract / read
        with open(path, "rb") as f:
            head = f.read(20)
        n = int(_np.frombuffer(head[8:12], _np.uint32)[0])
        slots = int(_np.frombuffer(head[12:20], _np.uint64)[0])
        self.graph = ZeroTerminatedCsr(n, _np.zeros(0, _np.uint32), _np.zeros(slots, _np.uint32))

    def load_device(self, d_row_ptr: int, n: int, d_col: int, slots: int) -> None:
        _check(lib().ktg_engine_load_device(self._h, _vp(d_row_ptr), n, _vp(d_col), slots))

    def reset(self) -> None:
        _check(lib().ktg_engine_reset(self._h))

    def run(self, k: int, sync: bool = True) -> Optional[List[int]]:
        if not sync:
            _check(lib().ktg_engine_run(self._h, k, None, 0, None))
            return None
        cap = 1 << 16
        hist = np.zeros(cap, dtype=np.uint64)
        it = _u32()
        _check(lib().ktg_engine_run(self._h, k, _p(hist), cap, ctypes.byref(it)))
        return [int(x) for x in hist[:min(it.value, cap)]]

    def kmax(self) -> int:
        """kmax_search's search (truss.cpp:73-103) on the resident graph: bound
        by one support pass, binary search with every probe from pristine.
        Leaves the engine holding the k_max truss."""
        self.reset()
        self.support_pass()
        max_support = int(self.info()["max_support"])
        lo = 2
        if max_support > 0:
            lo, hi = 3, max_support + 2
            while lo < hi:
                mid = lo + (hi - lo + 1) // 2
                self.reset()
                self.run(mid)
                if self.info()["live_edges"] == 0:
                    hi = mid - 1
                else:
                    lo = mid
        self.reset()
        self.run(lo)
        return lo

    def sweep(self, k_lo: int = 3, k_hi: Optional[int] = None, extract: bool = False):
        """Incremental K sweep: K = k_lo, k_lo+1, ... each
        fixpoint starting from the previous K's truss instead of the pristine
        graph. The k-truss is unique and trusses are nested, so every K's
        survivors and supports equal ktruss(graph, K) from pristine (tested);
        only `iterations` differ. Stops after k_hi or at the first empty
        truss (that K is K_max + 1 and is included). Returns a list of dicts
        (k, live_edges, iterations[, truss])."""
        self.reset()
        out = []
        k = k_lo
        while k_hi is None or k <= k_hi:
            hist = self.run(k)
            rec = {"k": k, "live_edges": int(self.info()["live_edges"]), "iterations": len(hist)}
            if extract:
                rec["truss"] = self.extract()
            out.append(rec)
            if rec["live_edges"] == 0:
                break
            k += 1
        return out

    def support_pass(self) -> int:
        tri = _u64()
        _check(lib().ktg_engine_support_pass(self._h, ctypes.byref(tri)))
        return int(tri.value)

    def sync(self) -> None:
        _check(lib().ktg_engine_sync(self._h))

    def info(self) -> dict:
        i = _RunInfo()
        _check(lib().ktg_engine_info(self._h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _RunInfo._fields_}

    def round_work(self) -> List[dict]:
        buf = (_RoundWork * (1 << 16))()
        m = lib().ktg_engine_round_work(self._h, buf, 1 << 16)
        return [{k: getattr(buf[i], k) for k, _ in _RoundWork._fields_} for i in range(m)]

    def read(self):
        slots = self.graph.total_slots()
        col = np.empty(slots, dtype=np.uint32)
        sup = np.empty(slots, dtype=np.uint32)
        _check(lib().ktg_engine_read(self._h, _p(col), _p(sup)))
        return col, sup

    def device_state(self):
        c, s, st = _vp(), _vp(), _vp()
        _check(lib().ktg_engine_device_state(self._h, ctypes.byref(c), ctypes.byref(s), ctypes.byref(st)))
        return c.value, s.value, st.value

    def extract(self, cap: Optional[int] = None):
        """Survivors as a TrussResult-like (u, v, support) triple of u32
        columns (pinned host memory); .edges stacks them."""
        if cap is None:  # exact survivor count (synchronises)
            self.sync()
            cap = max(1, int(self.info()["live_edges"]))
        owner = _result_pool.take(cap)
        u, v, sup = _ResultPool.columns(owner, cap)
        num = _u64()
        _check(lib().ktg_engine_extract(self._h, _p(u), _p(v), _p(sup), cap, ctypes.byref(num)))
        m = int(num.value)
        u, v, sup = _ResultPool.finish(u, v, sup, m)
        del owner
        return TrussResult(0, u, v, sup, 0, [])

    def set_nccl(self, rank: int, world: int, unique_id: bytes) -> None:
        """Edge-partitioned fixpoint over NCCL (collective across ranks)."""
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().ktg_engine_set_nccl(self._h, rank, world, buf))

    def support_buffers(self):
        """Device pointers of the active layout's two support buffers and
        the slot count (what peers add into under set_peers)."""
        a, b, n = _vp(), _vp(), _u64()
        _check(lib().ktg_engine_support_buffers(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, int(n.value)

    def set_peers(self, rank: int, world: int, s0, s1, exchange) -> None:
        """Fused multi-GPU support pass: increments go straight to the owner
        rank's buffer (peer pointers s0/s1, one per rank, this engine's own at
        `rank`); `exchange(phase, d_supports, slots, span, d_triangles,
        stream)` is the ktg_peer_cb contract of include/ktg.h."""
        t0 = (ctypes.c_void_p * world)(*s0)
        t1 = (ctypes.c_void_p * world)(*s1)

        def tramp(phase, d_s, slots, span, d_tri, stream, user):
            try:
                exchange(int(phase), d_s, int(slots), int(span), d_tri, stream)
                return 0
            except Exception:  # surfaces as KTG_ERR_CUDA
                import traceback
                traceback.print_exc()
                return 1

        cb = PEER_CB(tramp)
        self._keep["peers"] = (t0, t1, cb)
        _check(lib().ktg_engine_set_peers(self._h, rank, world, t0, t1, cb, None))

    def group_area(self):
        """(device pointer, bytes) of this engine's peer-group exchange area
        (ktg_engine_group_area); share it with the peers (ipc_handle)."""
        a, b = _vp(), _u64()
        _check(lib().ktg_engine_group_area(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, int(b.value)

    def set_group(self, rank: int, world: int, areas, s0, s1) -> None:
        """Device-resident partitioned fixpoint (ktg_engine_set_group): every
        rank's exchange area and support buffers, mapped into this process,
        own entries at `rank`. Collective; meet in a host barrier before the
        first run."""
        ta = (ctypes.c_void_p * world)(*areas)
        t0 = (ctypes.c_void_p * world)(*s0)
        t1 = (ctypes.c_void_p * world)(*s1)
        self._keep["group"] = (ta, t0, t1)
        _check(lib().ktg_engine_set_group(self._h, rank, world, ta, t0, t1))

    def set_partition(self, rank: int, world: int, allreduce=None) -> None:
        cb = ALLREDUCE_CB(allreduce) if allreduce is not None else ALLREDUCE_CB()
        self._keep["allreduce"] = cb
        _check(lib().ktg_engine_set_partition(self._h, rank, world, cb, None))

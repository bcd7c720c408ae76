"""Fused reduce-scatter (ktg_engine_set_peers): each rank's support kernel
sends every increment straight to the owner rank's buffer over peer memory;
the exchange callback only all-gathers the owned spans. Two "virtual ranks"
(two engines driven from two threads, one device) against the oracle,
byte-exact -- the multi-GPU path's arithmetic and synchronisation protocol
on the one GPU available to the tests."""
import ctypes
import threading

import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from paper_2009_07929_b200 import truss

pytestmark = pytest.mark.gpu


def _run_ranks(g, world, ks):
    engines = [kt.Engine(g) for _ in range(world)]
    bufs = [e.support_buffers() for e in engines]
    s0 = [b[0] for b in bufs]
    s1 = [b[1] for b in bufs]
    bar = threading.Barrier(world, timeout=120)
    parts = [0] * world

    def exchange_for(r):
        def ex(phase, d_s, slots, span, d_tri, stream):
            v = ctypes.c_uint64()
            truss.device_copy(ctypes.addressof(v), ctypes.addressof(v), 0, stream)  # waits for the stream
            bar.wait()
            if phase == 0:  # every rank's previous prune is done
                return
            truss.device_copy(ctypes.addressof(v), d_tri, 8, stream)
            parts[r] = v.value
            bar.wait()
            v.value = sum(parts)
            truss.device_copy(d_tri, ctypes.addressof(v), 8, stream)
            src = s0 if d_s == s0[r] else s1
            for q in range(world):
                lo = q * span
                cnt = min(span, slots - lo)
                if q != r and cnt > 0:
                    truss.device_copy(d_s + 4 * lo, src[q] + 4 * lo, 4 * cnt, stream)
            bar.wait()  # nobody prunes (zeroes) or adds again before all copies
        return ex

    for r, e in enumerate(engines):
        e.set_peers(r, world, s0, s1, exchange_for(r))
    out = [dict() for _ in range(world)]
    errs = []

    def body(r):
        try:
            for k in ks:
                engines[r].reset()
                hist = engines[r].run(k)
                col, S = engines[r].read()
                out[r][k] = (hist, col.copy(), S.copy(), engines[r].info()["triangles"])
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)
            bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in engines:
        e.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_fused_reduce_scatter_virtual_ranks(port, world):
    g = kt.rmat(13, 16, seed=4)
    ks = (3, 5, 9)
    out = _run_ranks(g, world, ks)
    for k in ks:
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        tri_e, _ = port.compute_supports(kt.ZeroTerminatedCsr(g.num_vertices, g.row_ptr, col_e), threads=8)
        for r in range(world):
            hist, col, S, tri = out[r][k]
            assert hist == hist_e, (world, r, k)
            assert np.array_equal(col, col_e) and np.array_equal(S, S_e), (world, r, k)
            assert tri == tri_e, (world, r, k)


def _proc(rank, world, port, ks, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2009_07929_b200 as kt2
    from paper_2009_07929_b200 import dist as kd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = kt2.rmat(13, 16, seed=4)
        e = kt2.Engine(g)
        mapped = kd.engine_join_fused(e)
        res = {}
        for k in ks:
            e.reset()
            hist = e.run(k)
            col, S = e.read()
            res[k] = (hist, col.copy(), S.copy())
        dist.barrier()
        e.close()
        for p in mapped:
            kt2.truss.ipc_close(p)
        q.put((rank, res))
    except Exception as ex:  # surfaced by the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def test_fused_reduce_scatter_two_processes_ipc(port):
    """The multi-process wiring (dist.engine_join_fused): CUDA IPC handles of
    the support buffers exchanged over torch.distributed, peer atomics into
    the other process's buffers, gloo barriers -- two rank processes sharing
    the one device, byte-exact against the oracle."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    ks = (3, 6)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc, args=(r, 2, p, ks, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    g = kt.rmat(13, 16, seed=4)
    for r in range(2):
        assert not isinstance(out[r], str), out[r]
        for k in ks:
            col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
            hist, col, S = out[r][k]
            assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e), (r, k)


def test_carried_run_partitioned_virtual_ranks(port):
    """Multi-rank carried-support run (set_partition): each rank's full
    passes cover its share of the A22 tasks, the callback sums the partial
    supports, and every rank runs the same mark / delta / compaction --
    two engines in two threads on one device, byte-exact against the oracle."""
    world = 2
    g = kt.rmat(13, 16, seed=4)
    # collect_work: per-round records prove the carried path ran (rounds with
    # full_pass == 0), not a silent fallback to recompute mode
    engines = [kt.Engine(g, collect_work=True) for _ in range(world)]
    bar = threading.Barrier(world, timeout=120)
    parts = [None] * world
    slots = g.total_slots()

    def reducer(r):
        def cb(d_buf, count, stream, user):
            try:
                addr = ctypes.cast(d_buf, ctypes.c_void_p).value
                host = np.empty(count, np.uint32)
                truss.device_copy(host.ctypes.data, addr, 4 * count, stream)  # waits for the stream
                parts[r] = host
                bar.wait()
                total = parts[0] + parts[1]
                bar.wait()
                truss.device_copy(addr, total.ctypes.data, 4 * count, stream)
                return 0
            except Exception:  # pragma: no cover
                bar.abort()
                return 1
        return cb

    for r, e in enumerate(engines):
        e.set_partition(r, world, allreduce=reducer(r))
    ks = (3, 6, 10)
    out = [dict() for _ in range(world)]
    errs = []

    def body(r):
        try:
            for k in ks:
                engines[r].reset()
                hist = engines[r].run(k)
                col, S = engines[r].read()
                out[r][k] = (hist, col.copy(), S.copy(), engines[r].round_work())
        except Exception as ex:  # pragma: no cover
            errs.append(ex)
            bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in engines:
        e.close()
    if errs:
        raise errs[0]
    assert slots > 0
    carried = 0
    for k in ks:
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        for r in range(world):
            hist, col, S, work = out[r][k]
            assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e), (r, k)
            carried += sum(1 for w in work if not w["full_pass"])
    assert carried > 0, "no carried round ran: the partitioned carried path was not exercised"

"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: the K split,
the NCCL-id broadcast, and the edge-partitioned fixpoint (partial supports
of each rank's task share -> all-reduce -> replicated prune) with the
oracle's mirror of the engine's task partition standing in for the kernel."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as ex:  # surface to the parent
        q.put((rank, ex))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


def _k_split(rank, world):
    from paper_2009_07929_b200 import dist as kd
    ks = list(range(3, 305))
    mine = kd.split_k_values(ks, rank, world)
    got = [None] * world
    dist.all_gather_object(got, mine)
    return got, kd.max_over_ranks(rank + 1.0), kd.sum_over_ranks(1.0)


def test_k_split_covers_every_k_once():
    res = _spawn(_k_split)
    got, mx, sm = res[0]
    flat = sorted(k for part in got for k in part)
    assert flat == list(range(3, 305))
    assert abs(len(got[0]) - len(got[1])) <= 1
    assert mx == 2.0 and sm == 2.0


def _nccl_id(rank, world):
    from paper_2009_07929_b200 import dist as kd
    from paper_2009_07929_b200 import truss
    try:
        truss.lib()
    except ImportError:
        return "skip"
    try:
        uid = kd.broadcast_nccl_id()
    except Exception as ex:  # libnccl absent on this host
        return f"skip:{ex}"
    return uid


def test_nccl_id_broadcast():
    a, b = _spawn(_nccl_id)
    if isinstance(a, str) and a.startswith("skip"):
        pytest.skip(a)
    assert isinstance(a, bytes) and len(a) == 128 and a == b


def _partitioned_fixpoint(rank, world):
    import torch

    import oracle
    from paper_2009_07929_b200 import graph
    P = oracle.port()
    g = graph.rmat(11, 16, seed=5)
    out = {}
    for k in (3, 6, 10):
        work = g.copy()
        hist = []
        while True:
            _, S = P.support_tasks(work, rank, world)          # this rank's tasks (engine chunking)
            t = torch.from_numpy(S.view(np.int32).copy())
            dist.all_reduce(t)                                  # exact integer sum
            S = t.numpy().view(np.uint32)
            removed = P.prune_edges(work, S, k)                 # replicated prune
            hist.append(removed)
            if removed == 0:
                break
        out[k] = (work.col_idx.copy(), S.copy(), hist)
    return out


def test_partitioned_fixpoint_equals_single_process():
    import oracle
    from paper_2009_07929_b200 import graph
    r0, r1 = _spawn(_partitioned_fixpoint)
    g = graph.rmat(11, 16, seed=5)
    for k in (3, 6, 10):
        col, S, hist = oracle.port().run_fixpoint(g, k)
        for r in (r0, r1):
            assert r[k][2] == hist
            assert np.array_equal(r[k][0], col) and np.array_equal(r[k][1], S)


def test_task_split_is_work_balanced():
    """the diagonal support tasks are split into contiguous
    chunk ranges of equal estimated work (prefix sum of the per-chunk work,
    mirror of k_task_cost / k_rank_range); equal slot counts are not."""
    import oracle
    from paper_2009_07929_b200 import graph
    g = graph.rmat(14, 16, 42)
    c = oracle.port().task_costs(g).astype(np.float64)
    T, Q = c.sum(), len(c)
    pre = np.concatenate([[0.0], np.cumsum(c)])
    for w in (2, 4, 8):
        own = np.minimum(w - 1, (pre[:-1] * w // T)).astype(int)
        assert np.all(np.diff(own) >= 0)  # contiguous ranges
        tot = np.bincount(own, weights=c, minlength=w)
        assert tot.max() / tot.mean() < 1.02, w
        eq = np.bincount(np.minimum(w - 1, np.arange(Q) * w // Q), weights=c, minlength=w)
        assert eq.max() / eq.mean() > 1.2, w


def owner_of(eid, world):
    """Mirror of ktg_kernels.cuh owner_of: the rank sharding removed edge
    `eid` in a carried round of the peer group."""
    return ((eid * 2654435761) & 0xFFFFFFFF) * world >> 32


def _support_all(edges, live):
    adj = {}
    for i in np.flatnonzero(live):
        u, v = edges[i]
        adj.setdefault(u, set()).add(v)
        adj.setdefault(v, set()).add(u)
    S = np.zeros(len(edges), np.int64)
    for i in np.flatnonzero(live):
        u, v = edges[i]
        S[i] = len(adj[u] & adj[v])
    return S, adj


def _sharded_carried_fixpoint(rank, world):
    """The peer group's carried rounds on CPU ranks: each rank finds the lost
    triangles of its share of the removed edges (owner_of), a triangle is
    handled by its removed edge of smallest id, the decrement lists are
    all-gathered and every rank applies all of them. Every round's supports
    must equal a from-scratch recount, and the fixpoint the reference loop's
    (truss.cpp:41-53: reset + recount + prune every round)."""
    import oracle
    from paper_2009_07929_b200 import graph
    g = graph.rmat(9, 16, seed=5)
    rp, col = g.row_ptr.astype(np.int64), g.col_idx
    rows = np.repeat(np.arange(g.num_vertices + 1), np.diff(rp[:g.num_vertices + 2]))
    sl = np.flatnonzero(col != 0)
    edges = np.stack([rows[sl], col[sl].astype(np.int64)], axis=1)
    eid = {(int(u), int(v)): i for i, (u, v) in enumerate(edges)}
    out = {}
    for k in (4, 6, 9):
        thr = k - 2
        live = np.ones(len(edges), bool)
        S, adj = _support_all(edges, live)
        hist = []
        while True:
            rem = live & (S < thr)
            hist.append(int(rem.sum()))
            if not rem.any():
                break
            dec = []
            for e in np.flatnonzero(rem):
                if owner_of(int(e), world) != rank:
                    continue
                u, v = edges[e]
                for w in adj[u] & adj[v]:
                    a = eid[(min(u, w), max(u, w))]
                    b = eid[(min(v, w), max(v, w))]
                    if (rem[a] and a < e) or (rem[b] and b < e):
                        continue  # a smaller removed id handles this triangle
                    dec += [x for x in (a, b) if not rem[x]]
            lists = [None] * world
            dist.all_gather_object(lists, dec)
            live &= ~rem
            for lst in lists:
                for x in lst:
                    S[x] -= 1
            S[~live] = 0
            fresh, adj = _support_all(edges, live)
            assert np.array_equal(S, fresh), (k, len(hist))
        col_e, S_e, hist_e = oracle.port().run_fixpoint(g, k, threads=1)
        assert hist == hist_e, (k, hist, hist_e)
        assert int(live.sum()) == int(np.count_nonzero(col_e))
        out[k] = (hist, int(live.sum()))
    return out


def test_sharded_carried_rounds_match_recount():
    res = _spawn(_sharded_carried_fixpoint)
    assert res[0] == res[1]

"""Device-resident partitioned fixpoint (ktg_engine_set_group):
the exchange runs as kernels over peer memory inside each rank's fixpoint
graph -- work-balanced split of every full pass with an in-kernel
all-reduce of S, carried rounds' removals sharded by edge id with the
decrements exchanged through per-rank lists. "Virtual ranks" (engines on
one device, one thread each) and two rank processes over CUDA IPC, byte-exact
against the oracle (the reference loop truss.cpp:41-53 restated)."""
import json
import os
import threading

import numpy as np
import pytest

import paper_2009_07929_b200 as kt

pytestmark = pytest.mark.gpu

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def _group_ranks(g, world, ks, opts=None, reload=False, **kw):
    engines = [kt.Engine(g, opts, **kw) for _ in range(world)]
    areas = [e.group_area()[0] for e in engines]
    bufs = [e.support_buffers() for e in engines]
    for r, e in enumerate(engines):
        e.set_group(r, world, areas, [b[0] for b in bufs], [b[1] for b in bufs])
    for e in engines:
        e.sync()
    out = [dict() for _ in range(world)]
    errs = []
    bar = threading.Barrier(world, timeout=300)

    def body(r):
        try:
            for k in ks:
                bar.wait()  # every rank runs the same fixpoint sequence
                if reload:  # same graph again: the group survives the load
                    engines[r].load(g)
                engines[r].reset()
                hist = engines[r].run(k)
                info = engines[r].info()
                col, S = engines[r].read()
                work = engines[r].round_work() if kw.get("collect_work") else None
                out[r][k] = (hist, col.copy(), S.copy(), info["triangles"], info["device_ms"], work)
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


def _check(port, g, out, ks):
    for k in ks:
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        tri_e, _ = port.compute_supports(kt.ZeroTerminatedCsr(g.num_vertices, g.row_ptr, col_e), threads=8)
        for r, o in enumerate(out):
            hist, col, S, tri = o[k][:4]
            assert hist == hist_e, (r, k, hist[:5], hist_e[:5])
            assert np.array_equal(col, col_e) and np.array_equal(S, S_e), (r, k)
            assert tri == tri_e, (r, k)


@pytest.mark.parametrize("world", [2, 3])
def test_group_virtual_ranks_device_resident(port, world):
    """Default (carried-support) runs, graph mode: one graph launch per
    fixpoint per rank, every exchange on the device."""
    g = kt.rmat(13, 16, seed=4)
    ks = (3, 4, 6, 9, 14)
    out = _group_ranks(g, world, ks)
    _check(port, g, out, ks)
    # per-round overhead of the device-side exchange against one engine
    e = kt.Engine(g)
    rec = {"world": world, "graph": "rmat-s13-ef16-seed4", "k": {}}
    for k in ks:
        e.reset()
        h = e.run(k)
        solo = e.info()["device_ms"]
        grp = max(o[k][4] for o in out)
        rec["k"][k] = {"rounds": len(h), "single_ms": round(solo, 3), "group_ms": round(grp, 3),
                       "overhead_us_per_round": round(1e3 * (grp - solo) / max(1, len(h)), 1)}
    e.close()
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"group_overhead_w{world}.json"), "w") as f:
        json.dump(rec, f, indent=1)


def test_group_survives_reload(port):
    """Reloading the same graph keeps the group (same buffers) and the
    barrier epochs (the loop state is reset, the peers' flags are not): a
    multi-rank end-to-end run reloads before every fixpoint."""
    g = kt.rmat(12, 16, seed=9)
    ks = (3, 5, 8)
    out = _group_ranks(g, 2, ks, reload=True)
    _check(port, g, out, ks)


def test_group_carried_rounds_are_sharded(port):
    """Host-recorded run of the same group path: some rounds carry supports
    (full_pass == 0), i.e. the sharded delta + decrement exchange ran, and
    the results are still byte-exact."""
    g = kt.rmat(13, 16, seed=4)
    ks = (5, 9)
    out = _group_ranks(g, 2, ks, collect_work=True)
    _check(port, g, out, ks)
    carried = [w for o in out for k in ks for w in o[k][5] if w["carried"]]
    assert carried, "no carried round ran: the sharded delta path was not exercised"


def test_group_recompute_virtual_ranks(port):
    """KTG_FLAG_RECOMPUTE runs: chunk tasks split by work, the in-kernel
    all-reduce every round."""
    g = kt.rmat(12, 16, seed=9)
    ks = (3, 7, 11)
    out = _group_ranks(g, 2, ks, kt.TrussOptions(recompute=True))
    _check(port, g, out, ks)


def test_group_support_pass_and_kmax_are_whole_graph(port):
    """A partitioned engine's standalone support pass is never split (ADVICE
    r1): every rank gets the whole-graph T and max S, so kmax agrees."""
    g = kt.rmat(12, 16, seed=9)
    engines = [kt.Engine(g) for _ in range(2)]
    areas = [e.group_area()[0] for e in engines]
    bufs = [e.support_buffers() for e in engines]
    for r, e in enumerate(engines):
        e.set_group(r, 2, areas, [b[0] for b in bufs], [b[1] for b in bufs])
    tri_e, _ = port.compute_supports(g, threads=8)
    for e in engines:
        e.reset()
        assert e.support_pass() == tri_e
    for e in engines:
        e.close()


def _proc(rank, world, port, ks, q):
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
        mapped = kd.engine_join_group(e)
        res = {}
        for k in ks:
            dist.barrier()
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


def test_group_two_processes_ipc(port):
    """dist.engine_join_group across two rank processes (IPC handles over
    torch.distributed, barriers and all-reduce as kernels on peer memory),
    sharing the one device: byte-exact against the oracle."""
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
    out = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    g = kt.rmat(13, 16, seed=4)
    for r in range(2):
        assert not isinstance(out[r], str), out[r]
        for k in ks:
            col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
            hist, col, S = out[r][k]
            assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e), (r, k)

"""Large-graph parity: byte-exact (col_idx, S, removed history) against the
oracle at s14 for every K, s20 at K=3 / K_max, plus size-independent
properties and the pinned known answers of SURVEY §8(d)."""
import numpy as np
import pytest

import paper_2009_07929_b200 as kt
from _util import digest, golden, skew_graph

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [10, 12])
def test_golden_rmat(scale):
    ent = golden("rmat.json")[f"s{scale}"]
    g = kt.rmat(scale)
    S = kt.SupportArray.zeros(g.total_slots())
    assert kt.compute_supports(g, S) == ent["triangles"] and digest(S.counts) == ent["supports_sha256"]
    r = kt.ktruss(g, 3)
    assert digest(r.edges) == ent["k3_edges_sha256"] and r.removed_per_iteration == ent["k3_removed"]
    km = kt.kmax_search(g)
    assert km.k_max == ent["kmax"] and digest(km.truss.edges) == ent["kmax_edges_sha256"]


@pytest.fixture(scope="module")
def s14():
    return kt.rmat(14)


# label: caller layout, full pass per round. recompute: working layout, full
# pass per round. inc: carried supports where cheaper (default). delta /
# delta_host: carried supports every round after the first (forced by the
# cost ratio), device loop / host loop.
MODES = {
    "label": (dict(label_order=True), None, {}),
    "recompute": (dict(recompute=True), None, {}),
    "inc": ({}, None, {}),
    "inc_nobound": (dict(no_degree_bound=True), None, {}),
    "delta": ({}, "1e9", {}),
    "delta_host": (dict(host_loop=True), "1e9", dict(time_support=True)),
}


def mode_engine(g, mode, monkeypatch):
    opts, ratio, extra = MODES[mode]
    if ratio is not None:
        monkeypatch.setenv("KTG_DELTA_RATIO", ratio)
    else:
        monkeypatch.delenv("KTG_DELTA_RATIO", raising=False)
    eng = kt.Engine(g, kt.TrussOptions(**opts), **extra)
    monkeypatch.delenv("KTG_DELTA_RATIO", raising=False)
    return eng


@pytest.mark.parametrize("mode", list(MODES))
def test_s14_every_k_byte_exact(s14, port, mode, monkeypatch):
    ent = golden("rmat.json")["s14_known"]
    eng = mode_engine(s14, mode, monkeypatch)
    for k in range(3, ent["kmax"] + 2):
        eng.reset()
        hist = eng.run(k)
        col, S = eng.read()
        col_e, S_e, hist_e = port.run_fixpoint(s14, k, threads=8)
        assert hist == hist_e, k
        assert np.array_equal(col, col_e) and np.array_equal(S, S_e), k
        assert eng.info()["triangles"] * 3 == int(S_e.sum(dtype=np.uint64)), k
        if k == 3:
            assert eng.info()["live_edges"] == ent["k3_survivors"]
        if k == ent["kmax"]:
            assert eng.info()["live_edges"] == ent["kmax_survivors"]
        if k == ent["kmax"] + 1:
            assert eng.info()["live_edges"] == 0
    assert eng.kmax() == ent["kmax"]


def test_s14_naive_and_host_loop_agree(s14):
    base = kt.ktruss(s14, 5)
    for o in (kt.TrussOptions(naive_support=True), kt.TrussOptions(host_loop=True),
              kt.TrussOptions(label_order=True), kt.TrussOptions(label_order=True, naive_support=True)):
        r = kt.ktruss(s14, 5, o)
        assert np.array_equal(r.edges, base.edges) and r.removed_per_iteration == base.removed_per_iteration


def test_incremental_runs_equal_pristine(s14):
    """Running K+1 on the K-truss (no reset) gives the pristine (K+1)-truss:
    exercises the device-side buffer parity across runs."""
    eng = kt.Engine(s14)
    ref_eng = kt.Engine(s14)
    eng.reset()
    for k in range(3, 40, 3):
        eng.run(k)
        ref_eng.reset()
        ref_eng.run(k)
        a, b = eng.read(), ref_eng.read()
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), k


def test_partitioned_engine_support_pass_is_whole_graph(s14):
    """A standalone support pass (compute_supports / the kmax_search bound,
    support.cpp:93-132) on an engine partitioned over P ranks is never split
    (ADVICE r1): every rank returns the whole-graph T and S, so a partitioned
    kmax cannot bisect under a partial max S. The split itself (partial
    supports summing to the full ones) is exercised by the multi-rank
    fixpoint tests (test_gpu_peers.py, test_gpu_group.py)."""
    full = kt.Engine(s14)
    full.reset()
    t_full = full.support_pass()
    S_full = full.read()[1]
    for P in (2, 3, 8):
        for r in range(P):
            e = kt.Engine(s14)
            e.set_partition(r, P, allreduce=lambda *a: 0)
            e.reset()
            assert e.support_pass() == t_full, (P, r)
            assert np.array_equal(e.read()[1], S_full), (P, r)
            e.close()


def test_skew_graph(port):
    g = skew_graph()
    for k in (3, 4):
        r = kt.ktruss(g, k)
        e, hist = port.truss_edges(g, k, threads=8)
        assert np.array_equal(r.edges, e) and r.removed_per_iteration == hist


def test_er_small(port):
    g = kt.erdos_renyi(16, 16 << 16, 42)
    for k in (3, 4):
        r = kt.ktruss(g, k)
        e, hist = port.truss_edges(g, k, threads=8)
        assert np.array_equal(r.edges, e) and r.removed_per_iteration == hist
    assert kt.kmax_search(g).k_max == port.kmax(g, threads=8)


@pytest.fixture(scope="module")
def s20():
    return kt.rmat(20)


def test_s20_known_answers_and_properties(s20):
    ent = golden("rmat.json")["s20_known"]
    assert (s20.num_vertices, s20.num_edges) == (ent["n"], ent["m"])
    eng = kt.Engine(s20)
    eng.reset()
    t = eng.support_pass()
    col, S = eng.read()
    assert t == ent["triangles"] and int(S.max()) == ent["max_support"]
    assert int(S.sum(dtype=np.uint64)) == 3 * t  # triple-count identity
    eng.reset()
    eng.run(3)
    assert eng.info()["live_edges"] == ent["k3_survivors"]
    # idempotence: the truss is a fixpoint of its own k
    hist = eng.run(3)
    assert hist == [0]
    assert eng.kmax() == ent["kmax"]
    assert eng.info()["live_edges"] == ent["kmax_survivors"]


@pytest.mark.parametrize("k,mode", [(3, "inc"), (304, "inc"), (3, "label"), (30, "delta"), (120, "recompute")])
def test_s20_byte_exact(s20, port, k, mode, monkeypatch):
    eng = mode_engine(s20, mode, monkeypatch)
    eng.reset()
    hist = eng.run(k)
    col, S = eng.read()
    col_e, S_e, hist_e = port.run_fixpoint(s20, k, threads=16)
    assert hist == hist_e
    assert np.array_equal(col, col_e) and np.array_equal(S, S_e)


def test_rank_partials_match_oracle_task_partition(port):
    """Each rank's partial supports of a partitioned fixpoint's first round
    (recompute path: work-balanced chunk range + off-diagonal share) equal
    the oracle's mirror of the device planner, rank by rank. The partial
    buffer is captured inside the allreduce callback, before any exchange."""
    import ctypes
    g = kt.rmat(12, 16, seed=9)
    for world in (2, 3):
        for r in range(world):
            got = []

            def cb(d_buf, count, stream, user):
                if not got:
                    host = np.empty(count, np.uint32)
                    kt.truss.device_copy(host.ctypes.data, ctypes.cast(d_buf, ctypes.c_void_p).value, 4 * count,
                                         stream)
                    got.append(host)
                return 0

            e = kt.Engine(g, kt.TrussOptions(label_order=True))
            e.set_partition(r, world, allreduce=cb)
            e.reset()
            e.run(3)
            e.close()
            t_o, S_o = port.support_tasks(g, r, world, chunk=kt.truss.lib().ktg_task_chunk())
            assert np.array_equal(got[0], S_o), (world, r)


def test_nccl_single_rank_fixpoint(port):
    """The native ncclAllReduce path (world of 1 on this box) runs the
    host-driven partitioned loop byte-exactly."""
    g = kt.rmat(13, 16, seed=4)
    e = kt.Engine(g)
    e.set_nccl(0, 1, kt.truss.nccl_unique_id())
    for k in (3, 7):
        e.reset()
        hist = e.run(k)
        col, S = e.read()
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e)


def test_incremental_sweep_equals_pristine(s14, port):
    """Engine.sweep: every K's truss (edges + supports) equals the pristine
    ktruss(K); the sweep ends at K_max + 1 (empty)."""
    ent = golden("rmat.json")["s14_known"]
    eng = kt.Engine(s14)
    recs = eng.sweep(3, extract=True)
    assert recs[-1]["live_edges"] == 0 and recs[-1]["k"] == ent["kmax"] + 1
    for rec in recs[::7] + [recs[-2]]:
        e, _ = port.truss_edges(s14, rec["k"], threads=8)
        assert np.array_equal(rec["truss"].edges, e), rec["k"]


def test_planted_cliques_deep_kmax(port):
    """configs[4] semantics at a small scale (deep K_max, many prune rounds):
    byte-exact fixpoints and K_max."""
    g = kt.rmat_cliques(12, 16, 42, sizes=(24, 64))
    km = kt.kmax_search(g)
    assert km.k_max == port.kmax(g, threads=8) == 64
    eng = kt.Engine(g)
    for k in (3, 30, 64, 65):
        eng.reset()
        hist = eng.run(k)
        col, S = eng.read()
        col_e, S_e, hist_e = port.run_fixpoint(g, k, threads=8)
        assert hist == hist_e and np.array_equal(col, col_e) and np.array_equal(S, S_e), k
    eng.close()

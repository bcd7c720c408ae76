"""CPU model of the engine's carried-support rounds, checked against the
oracle's reset + computeSupports (truss.cpp:44-46) round by round.

The device (k_mark / k_delta, ktg_kernels.cuh) never recomputes a round's
supports when carrying is cheaper: every triangle of G_r that loses an edge
is handled once, from its removed edge with the smallest id, and each
surviving edge of it loses 1. This file restates that rule in plain Python
on small graphs and asserts:
  * carried S_{r+1} == the oracle's full pass on G_{r+1}, every round;
  * the next round's removals are exactly the edges whose carried support
    crossed below k-2 during the decrement (the frontier queue);
  * the round-0 degree bound: S(u,v) <= min(du, dv) - 1, so every edge with
    min(du, dv) < k - 1 is in the round-0 removal set (k_heavy_rank).
"""
import numpy as np
import pytest

from paper_2009_07929_b200 import graph


def _edges(g):
    """{(u, v): slot} of the live edges of a zero-terminated CSR."""
    rp, col = np.asarray(g.row_ptr), np.asarray(g.col_idx)
    out = {}
    for u in range(1, g.num_vertices + 1):
        for s in range(int(rp[u]), int(rp[u + 1])):
            if col[s] == 0:
                break
            out[(u, int(col[s]))] = s
    return out


def _carry(edges, S, removed, thr):
    """One carried round: S over `edges` (dict edge -> support, exact for
    G_r), `removed` the round's removal set (ids = slots). Returns the
    supports of G_{r+1} and the frontier (edges crossing below thr)."""
    nbr = {}
    for (u, v) in edges:
        nbr.setdefault(u, {})[v] = edges[(u, v)]
        nbr.setdefault(v, {})[u] = edges[(u, v)]
    rem_ids = {edges[e] for e in removed}
    S2 = {e: s for e, s in S.items() if e not in removed}
    frontier = set()
    for (u, v) in removed:
        e = edges[(u, v)]
        for w in set(nbr[u]) & set(nbr[v]):
            ea, eb = nbr[u][w], nbr[v][w]
            da, db = ea in rem_ids, eb in rem_ids
            if (da and ea < e) or (db and eb < e):
                continue  # another removed edge of this triangle has a smaller id
            for (x, y), dead in (((min(u, w), max(u, w)), da), ((min(v, w), max(v, w)), db)):
                if not dead:
                    if S2[(x, y)] == thr:
                        frontier.add((x, y))
                    S2[(x, y)] -= 1
    return S2, frontier


@pytest.mark.parametrize("scale,seed", [(8, 1), (9, 7), (10, 42)])
def test_carried_supports_equal_recompute(port, scale, seed):
    g0 = graph.rmat(scale, 16, seed=seed)
    for k in (3, 4, 6, 9, 14):
        thr = k - 2
        g = g0.copy()
        _, S_arr = port.compute_supports(g)
        edges = _edges(g)
        S = {e: int(S_arr[s]) for e, s in edges.items()}
        # round-0 degree bound
        deg = {}
        for (u, v) in edges:
            deg[u] = deg.get(u, 0) + 1
            deg[v] = deg.get(v, 0) + 1
        for (u, v), s in S.items():
            assert s <= min(deg[u], deg[v]) - 1
            if min(deg[u], deg[v]) < k - 1:
                assert s < thr
        removed = {e for e, s in S.items() if s < thr}
        rounds = 0
        while removed:
            S_next, frontier = _carry(edges, S, removed, thr)
            # the reference's next round: prune, reset, full pass
            S_prune = np.zeros(g.total_slots(), np.uint32)
            for e, s in S.items():
                S_prune[edges[e]] = s
            port.prune_edges(g, S_prune, k)
            _, S_full = port.compute_supports(g)
            edges = _edges(g)
            assert set(edges) == set(S_next), (k, rounds)
            for e, s in edges.items():
                assert S_next[e] == int(S_full[s]), (k, rounds, e)
            S = S_next
            removed = {e for e, s in S.items() if s < thr}
            assert removed == frontier, (k, rounds)
            rounds += 1
        col_e, S_e, hist = port.run_fixpoint(g0, k)
        assert rounds + 1 == len(hist), k
        assert np.array_equal(g.col_idx, col_e), k

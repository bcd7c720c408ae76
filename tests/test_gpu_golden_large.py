"""Reference-pinned parity at the headline / north-star sizes.

tests/golden/large_ref.json holds, per (graph, K), SHA-256 of the converged
(col_idx, S) and removed_per_iteration produced by the UNMODIFIED reference
(detail::run_fixpoint, Strategy::Fine, truss.cpp:41-53) on CSRs built by the
reference's own canonicalize + build_csr (tests/golden/make_golden_large.py,
run in the build container). Here the engine's results through the product
API are hashed and compared byte for byte -- no C port in the chain.

  s24   R-MAT scale 24 ef16 (the north-star config), K in {3, 10, 30, 100,
        300, 935, 936}: 935 non-empty and 936 empty pins K_max = 935
  s20   R-MAT scale 20 ef16, every K in 3..305 (the K-sweep config)
  er22  Erdos-Renyi 2^22 / 2^26 draws, K in {3, 4}
  cl22  R-MAT scale 22 ef32 + planted cliques {128,256,512,1024}, K_max
        (1057) and K_max + 1
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2009_07929_b200 as kt

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "large_ref.json")
CLIQUES = (128, 256, 512, 1024)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def golden():
    return json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else {}


def build(name):
    if name == "s24":
        return kt.rmat(24, 16, 42)
    if name == "s20":
        return kt.rmat(20, 16, 42)
    if name == "er22":
        return kt.erdos_renyi(22, 16 << 22, 42)
    return kt.rmat_cliques(22, 32, 42, sizes=CLIQUES)


def ks_of(name):
    return sorted(int(k) for k in golden().get(name, {}).get("fixpoints", {}))


@pytest.fixture(scope="module", params=["s24", "s20", "er22", "cl22"])
def case(request):
    name = request.param
    ent = golden().get(name)
    if not ent or "col_sha256" not in ent:
        pytest.skip(f"no reference digests for {name} yet")
    g = build(name)
    yield name, ent, g


def test_graph_matches_reference_canonicalize(case):
    """The product generator + canonicalize give the reference's CSR."""
    name, ent, g = case
    assert (g.num_vertices, g.num_edges, g.total_slots()) == (ent["n"], ent["m"], ent["slots"])
    assert sha(g.row_ptr) == ent["row_ptr_sha256"] and sha(g.col_idx) == ent["col_sha256"]


def test_support_pass_matches_reference(case):
    """compute_supports (support.cpp:93-132) on the pristine graph: T, max S
    and the whole S array (the kmax_search bound pass, truss.cpp:77-78)."""
    name, ent, g = case
    S = kt.SupportArray.zeros(g.total_slots())
    assert kt.compute_supports(g, S) == ent["triangles"]
    assert int(S.counts.max()) == ent["max_support"]
    assert sha(S.counts) == ent["supports_sha256"]


def test_fixpoints_match_reference(case):
    """run_fixpoint at every referenced K from pristine: converged col_idx, S
    and removed_per_iteration byte-equal to the reference's."""
    name, ent, g = case
    eng = kt.Engine(g)
    bad = []
    try:
        for key, ref in sorted(ent["fixpoints"].items(), key=lambda kv: int(kv[0])):
            k = int(key)
            eng.reset()
            hist = eng.run(k)
            col, S = eng.read()
            got = (sha(col), sha(S), hist, int(np.count_nonzero(col)))
            exp = (ref["col_sha256"], ref["supports_sha256"], ref["removed"], ref["survivors"])
            if got != exp:
                bad.append((k, got[3], exp[3], hist[:4], ref["removed"][:4]))
    finally:
        eng.close()
    assert not bad, bad[:5]


def test_kmax_confirmed_by_reference(case):
    """Where the reference ran K_max and K_max+1: the engine's kmax_search
    returns the K whose truss the reference found non-empty while K+1 is
    empty (trusses nest; kmax_search truss.cpp:73-103)."""
    name, ent, g = case
    fp = ent["fixpoints"]
    cand = [int(k) for k in fp if fp[k]["survivors"] > 0 and str(int(k) + 1) in fp
            and fp[str(int(k) + 1)]["survivors"] == 0]
    if not cand:
        pytest.skip("reference has no (K_max, K_max+1) pair for this graph")
    eng = kt.Engine(g)
    try:
        assert eng.kmax() == cand[0]
    finally:
        eng.close()

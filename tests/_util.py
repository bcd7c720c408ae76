import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return json.load(open(os.path.join(GOLDEN, name)))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def kat_graph(entry):
    from paper_2009_07929_b200.graph import ZeroTerminatedCsr
    return ZeroTerminatedCsr(entry["n"], np.array(entry["row_ptr"], np.uint32), np.array(entry["col_idx"], np.uint32))


def corpus(count=200):
    """Acceptance corpus (acceptance.cpp:114-125): G(n,p) with the
    reference's seeded generator, n in {8..64}, p in {.05,.1,.3,.6,1}."""
    import oracle
    from paper_2009_07929_b200 import graph
    probs = [0.05, 0.1, 0.3, 0.6, 1.0]
    sizes = [8, 12, 16, 24, 32, 48, 64]
    P = oracle.port()
    out = []
    for i in range(count):
        raw = P.random_graph_raw(sizes[i % 7], probs[i % 5], 1000 + i)
        out.append(graph.csr_from_pairs(raw))
    return out


def skew_graph():
    """acceptance.cpp:83-101 shape (hub of degree 4097 + fan ring + far vertex
    + 105k random edges); random part from numpy (shape, not bytes, matters)."""
    from paper_2009_07929_b200 import graph
    n, fan_end, far = 30000, 4098, 4100
    raw = [(1, w) for w in range(2, fan_end + 1)]
    raw += [(w, w + 1) for w in range(2, fan_end)]
    raw += [(w, far) for w in range(2, fan_end + 1)]
    rng = np.random.default_rng(20240707)
    r = rng.integers(1, n + 1, size=(105000, 2))
    r = r[r[:, 0] != r[:, 1]]
    return graph.csr_from_pairs(np.concatenate([np.array(raw), r]))

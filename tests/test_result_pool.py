"""Host-side result buffer pool of the Python API (no GPU needed): a pinned
buffer is reused only when no result views it; small results are copied out."""
import numpy as np

from paper_2009_07929_b200 import truss


class _Pool(truss._ResultPool):
    allocs = 0

    @staticmethod
    def _alloc(size):
        _Pool.allocs += 1
        return np.zeros(size, np.int32)


def test_reuse_only_when_free():
    _Pool.allocs = 0
    pool = _Pool()
    cap = 1 << 20
    owner = pool.take(cap)
    u, v, s = pool.columns(owner, cap)
    u[:] = 1
    res = pool.finish(u, v, s, cap)  # large: stays a view of the pooled buffer
    del owner, u, v, s
    assert res[0].base is not None
    o2 = pool.take(cap)  # first buffer is still referenced by res
    assert _Pool.allocs == 2
    del o2
    del res
    o3 = pool.take(cap)  # both free now: no new allocation
    assert _Pool.allocs == 2
    del o3


def test_small_results_copied_out():
    pool = _Pool()
    owner = pool.take(1000)
    u, v, s = pool.columns(owner, 1000)
    u[:10] = np.arange(10)
    ru, rv, rs = pool.finish(u, v, s, 10)
    del u, v, s
    assert ru.base is None and list(ru) == list(range(10))
    assert len(rv) == 10 and len(rs) == 10
    import sys
    assert sys.getrefcount(owner) == 3  # pool list + local + argument: free again

"""The C-ABI libraries load, export every symbol their headers declare, and
the engine refuses to run without a B200 (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ktgg?_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("ktg.h", "libktg.so"), ("ktg_graph.h", "libktg_graph.so")])
def test_exports(header, lib):
    L = ctypes.CDLL(os.path.join(ROOT, "paper_2009_07929_b200", "lib", lib))
    names = _declared(header)
    assert len(names) > 5
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    from paper_2009_07929_b200 import errors, truss
    if truss.lib().ktg_device_available():
        pytest.skip("a device is present")
    import paper_2009_07929_b200 as kt
    g = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    with pytest.raises(errors.DeviceError):
        kt.ktruss(g, 3)
    with pytest.raises(errors.DeviceError):
        kt.compute_supports(g, kt.SupportArray.zeros(g.total_slots()))


def test_parameter_errors_before_device():
    """Validation mirrors the reference and fires before any device work."""
    import paper_2009_07929_b200 as kt
    from paper_2009_07929_b200 import errors
    g = kt.csr_from_pairs([(1, 2), (1, 3), (2, 3)])
    with pytest.raises(errors.InvalidParameterError, match="thread count must be >= 1"):
        kt.compute_supports(g, kt.SupportArray.zeros(g.total_slots()), kt.Strategy.Fine, 0)
    with pytest.raises(errors.InvalidParameterError, match="k must be >= 2"):
        kt.ktruss(g, 1)
    with pytest.raises(errors.InvalidParameterError, match="k must be >= 2"):
        kt.prune_edges(g, kt.SupportArray.zeros(g.total_slots()), 1)
    with pytest.raises(errors.InvalidParameterError, match="support array does not match slot count"):
        kt.prune_edges(g, kt.SupportArray.zeros(2), 3)


def test_strategy_strings():
    import paper_2009_07929_b200 as kt
    for s in kt.Strategy:
        assert kt.strategy_from_string(kt.to_string(s)) == s
    assert kt.strategy_from_string("bogus") is None

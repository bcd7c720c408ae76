"""Locates and loads the in-tree native libraries.

The product path has no fallback: if libktg.so (the sm_100a engine) is
missing, every entry point raises. Build with `python __graft_entry__.py build`
or `make -C paper_2009_07929_b200`.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.environ.get("KTG_LIB_DIR", os.path.join(_HERE, "lib"))

_cache = {}


def _load(name: str) -> ctypes.CDLL:
    if name in _cache:
        return _cache[name]
    path = os.path.join(LIB_DIR, name)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the native engine first "
            "(python __graft_entry__.py build); there is no CPU fallback")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    _cache[name] = lib
    return lib


def graph_lib() -> ctypes.CDLL:
    return _load("libktg_graph.so")


def engine_lib() -> ctypes.CDLL:
    return _load("libktg.so")

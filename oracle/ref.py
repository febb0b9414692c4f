"""TEST INFRASTRUCTURE ONLY: ctypes access to the unmodified reference.

`oracle/_ref/libtrs_ref.so` is the reference library compiled from its own
sources under /root/reference (see oracle/Makefile) plus `ref_driver.cpp`.
Only tests/, __graft_entry__.smoke() and bench.py's reference arm may use it.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtrs_ref.so")


class _RefResult(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int),
        ("message", ctypes.c_char * 512),
        ("rewrites", ctypes.c_uint64),
        ("sweeps", ctypes.c_uint32),
        ("micros", ctypes.c_uint64),
        ("max_width", ctypes.c_uint64),
        ("median_width", ctypes.c_uint64),
        ("widths", ctypes.POINTER(ctypes.c_uint64)),
        ("live", ctypes.POINTER(ctypes.c_uint32)),
        ("n_widths", ctypes.c_uint32),
        ("words", ctypes.POINTER(ctypes.c_uint32)),
        ("n_words", ctypes.c_uint64),
        ("n_nodes", ctypes.c_uint32),
        ("num_symbols", ctypes.c_uint32),
        ("peak_depth", ctypes.c_uint64),
    ]


@dataclass
class RefRun:
    status: int
    message: str
    rewrites: int
    sweeps: int
    micros: int
    widths: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    live: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    words: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    n_nodes: int = 0
    max_width: int = 0
    median_width: int = 0


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (run `make -C oracle ref` where /root/reference exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint, ctypes.c_uint,
                              ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                              ctypes.POINTER(_RefResult)]
        L.ref_run.restype = ctypes.c_int
        L.ref_result_free.argtypes = [ctypes.POINTER(_RefResult)]
        L.ref_run_many.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.c_char_p,
                                   ctypes.c_uint, ctypes.POINTER(ctypes.c_uint64),
                                   ctypes.POINTER(ctypes.c_int)]
        L.ref_run_many.restype = ctypes.c_double
        for name in ("ref_dump_dispatch", "ref_diagnostics"):
            getattr(L, name).argtypes = [ctypes.c_char_p]
            getattr(L, name).restype = ctypes.c_void_p
        L.ref_generate.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64]
        L.ref_generate.restype = ctypes.c_void_p
        L.ref_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def run(text: str, engine: str = "seq", workers: int = 1, chunk: int = 256, capacity: int = 0,
        fixed_capacity: bool = False, step_budget: int = 1_000_000_000, words: bool = True) -> RefRun:
    L = lib()
    r = _RefResult()
    L.ref_run(text.encode(), engine.encode(), workers, chunk, capacity, int(fixed_capacity),
              step_budget, int(words), ctypes.byref(r))
    out = RefRun(r.status, r.message.decode(errors="replace"), r.rewrites, r.sweeps, r.micros,
                 n_nodes=r.n_nodes, max_width=r.max_width, median_width=r.median_width)
    if r.n_widths:
        out.widths = np.ctypeslib.as_array(r.widths, (r.n_widths,)).copy()
        out.live = np.ctypeslib.as_array(r.live, (r.n_widths,)).copy()
    if r.n_words:
        out.words = np.ctypeslib.as_array(r.words, (r.n_words,)).copy()
    L.ref_result_free(ctypes.byref(r))
    return out


def run_many(texts: list[str], engine: str = "seq", workers: int = 1):
    """Concurrent runs (one big-stack thread each); returns (wall_s, rewrites[], status[])."""
    L = lib()
    k = len(texts)
    arr = (ctypes.c_char_p * k)(*[t.encode() for t in texts])
    rw = (ctypes.c_uint64 * k)()
    st = (ctypes.c_int * k)()
    wall = L.ref_run_many(arr, k, engine.encode(), workers, rw, st)
    return wall, list(rw), list(st)


def _take_string(ptr) -> str | None:
    if not ptr:
        return None
    s = ctypes.string_at(ptr).decode()
    lib().ref_free(ptr)
    return s


def dump_dispatch(text: str) -> str | None:
    return _take_string(lib().ref_dump_dispatch(text.encode()))


def diagnostics(text: str) -> str:
    return _take_string(lib().ref_diagnostics(text.encode())) or ""


def generate(family: str, length: int = 0, depth: int = 0, seed: int = 1) -> str:
    fam = {"mergesort": 0, "treemergesort": 1, "transform": 2}[family]
    return _take_string(lib().ref_generate(fam, length, depth, seed))

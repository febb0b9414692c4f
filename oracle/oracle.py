"""TEST INFRASTRUCTURE ONLY: ctypes access to the C oracle (oracle/liboracle.so).

The oracle restates the reference's sweep and seq engines in plain C over
the flattened program of include/trs_gpu.h (see trs_oracle.h).  Inputs are
parsed/loaded with the product's host front end (the oracle checks the
engine, and tests/test_host.py checks the front end against the reference).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")


class Counts(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "eligible", "child_nf_reads", "checkhead", "path_hops", "rc_rmw", "collapse_reads", "frontier_sum",
        "own_args", "rewrites", "fresh_nodes", "visits", "dead_visits")]


class _Result(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int),
        ("rewrites", ctypes.c_uint64),
        ("sweeps", ctypes.c_uint32),
        ("widths", ctypes.POINTER(ctypes.c_uint64)),
        ("live", ctypes.POINTER(ctypes.c_uint32)),
        ("n", ctypes.POINTER(ctypes.c_uint32)),
        ("free_len", ctypes.POINTER(ctypes.c_uint32)),
        ("num_roots", ctypes.c_uint32),
        ("words", ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32))),
        ("n_words", ctypes.POINTER(ctypes.c_uint64)),
        ("counts", Counts),
        ("seconds", ctypes.c_double),
    ]


@dataclass
class OracleRun:
    status: int
    rewrites: int
    sweeps: int
    seconds: float
    widths: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    live: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    n: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    free_len: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    words: list = field(default_factory=list)
    counts: dict = field(default_factory=dict)

    @property
    def accesses(self) -> int:
        """A of SURVEY.md §8(d): random accesses counted per eligible derive."""
        c = self.counts
        return c["child_nf_reads"] + c["checkhead"] + c["path_hops"] + c["rc_rmw"] + c["collapse_reads"]

    def s_min(self, maxarity: int) -> int:
        """S_min of SURVEY.md §8(d): minimal streaming bytes of a frontier-only engine."""
        c = self.counts
        return (5 * c["frontier_sum"] + 4 * c["eligible"] + 4 * c["own_args"]
                + (5 + 4 * maxarity) * c["rewrites"] + (9 + 4 * maxarity) * c["fresh_nodes"])


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle oracle)")
        L = ctypes.CDLL(LIB_PATH)
        P, U32, U64, I = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        for name in ("oracle_sweep", "oracle_seq", "oracle_logical"):
            fn = getattr(L, name)
            fn.argtypes = [P, U32, P, U32, P, P, U32, P, U64, I, ctypes.POINTER(_Result)]
            fn.restype = I
        L.oracle_free.argtypes = [ctypes.POINTER(_Result)]
        _lib = L
    return _lib


def _run(fn_name: str, texts, step_budget: int = 0, words: bool = True) -> OracleRun:
    from paper_2009_07174_b200 import api

    if isinstance(texts, str):
        texts = [texts]
    systems = [api.System(t) for t in texts]
    store = api.Store.load(systems)
    v = store.view()
    prog = api.lib().trsb_program(systems[0].handle)
    r = _Result()
    getattr(lib(), fn_name)(prog, v["n"], v["roots_ptr"], v["num_roots"], v["hss_ptr"], v["args_ptr"],
                            v["maxarity"], v["rc_ptr"], step_budget, int(words), ctypes.byref(r))
    out = OracleRun(r.status, r.rewrites, r.sweeps, r.seconds,
                    counts={k: getattr(r.counts, k) for k, _ in Counts._fields_})
    if r.sweeps:
        out.widths = np.ctypeslib.as_array(r.widths, (r.sweeps,)).copy()
        if r.live:  # oracle_sweep only
            out.live = np.ctypeslib.as_array(r.live, (r.sweeps,)).copy()
            out.n = np.ctypeslib.as_array(r.n, (r.sweeps,)).copy()
            out.free_len = np.ctypeslib.as_array(r.free_len, (r.sweeps,)).copy()
    if r.words:
        for k in range(r.num_roots):
            out.words.append(np.ctypeslib.as_array(r.words[k], (r.n_words[k],)).copy())
    out.maxarity = v["maxarity"]
    lib().oracle_free(ctypes.byref(r))
    return out


def run_text(texts, step_budget: int = 0, words: bool = True) -> OracleRun:
    """Reference sweep engine (workers = 1) restated in C."""
    return _run("oracle_sweep", texts, step_budget, words)


def run_logical(texts, step_budget: int = 0, words: bool = True) -> OracleRun:
    """Reference sweep engine restated in logical time (dependency order, no
    sweep-by-sweep scans): same widths, sweeps, rewrites and words."""
    return _run("oracle_logical", texts, step_budget, words)


def run_seq(texts, step_budget: int = 0, words: bool = True) -> OracleRun:
    """Reference seq engine restated in C."""
    return _run("oracle_seq", texts, step_budget, words)

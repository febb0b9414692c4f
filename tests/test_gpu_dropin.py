"""Drop-in check: the reference's own C++ API (load_system -> compile ->
load -> run -> extract) with the B200 engine behind trs::run via
integration/trs_gpu_adapter.hpp.  Uses the prebuilt
integration/_ref/libref_gpu.so (unmodified reference objects + adapter),
built where /root/reference exists and shipped with the snapshot."""
import ctypes
import json
import os

import pytest

from paper_2009_07174_b200 import workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "integration", "_ref", "libref_gpu.so")
CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "small.json")))["cases"]


class _Res(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("message", ctypes.c_char * 512), ("term_equal_seq", ctypes.c_int),
                ("rewrites_equal", ctypes.c_int), ("widths_equal", ctypes.c_int),
                ("rewrites", ctypes.c_ulonglong), ("sweeps", ctypes.c_uint)]


@pytest.fixture(scope="module")
def dropin():
    if not os.path.exists(LIB):
        pytest.skip("integration/_ref/libref_gpu.so not built (needs /root/reference at build time)")
    L = ctypes.CDLL(LIB)
    L.ref_gpu_normalize.argtypes = [ctypes.c_char_p, ctypes.c_ulonglong, ctypes.POINTER(_Res)]
    return L


@pytest.mark.parametrize("name", ["unit_collapse", "unit_constructive", "unit_dupvar", "unit_erase",
                                  "unit_two_waiters", "transform6", "mergesort50_s42", "treemergesort_4_5_s7",
                                  "fib12", "buildsum8", "reverse64", "ackermann23", "fibbatch64_s3"])
def test_reference_api_with_b200_engine(dropin, name):
    r = _Res()
    dropin.ref_gpu_normalize(CASES[name]["text"].encode(), 0, ctypes.byref(r))
    assert r.status == 0, r.message
    assert r.term_equal_seq and r.rewrites_equal and r.widths_equal
    assert r.rewrites == CASES[name]["rewrites"]


def test_reference_api_full_size(dropin):
    r = _Res()
    dropin.ref_gpu_normalize(W.fib(18).encode(), 0, ctypes.byref(r))
    assert r.status == 0 and r.term_equal_seq and r.rewrites_equal and r.widths_equal


def test_reference_api_step_budget(dropin):
    r = _Res()
    text = "sort T = A() | F(T);\nvar X : T;\neqn F(X) = F(F(X));\ninput F(A());\n"
    dropin.ref_gpu_normalize(text.encode(), 500, ctypes.byref(r))
    assert r.status == 1  # EngineError(EngineFault::StepBudget) raised through the adapter

"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute without a GPU), and the synthetic workload texts are
byte-identical to the reference generator's."""
import ctypes
import os
import re

import pytest

from oracle import ref
from paper_2009_07174_b200 import api
from paper_2009_07174_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header: str) -> list[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(trs_gpu_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(api.LIB_PATH)
    names = declared_functions("trs_gpu.h")
    assert len(names) >= 16
    for n in names:
        assert hasattr(L, n), n
    assert set(api.exported_symbols()) <= set(names)


def test_no_device_is_reported_not_faked():
    """Without a GPU the engine refuses to open (there is no CPU fallback)."""
    if api.device_count() > 0:
        pytest.skip("a GPU is visible here")
    with pytest.raises(api.CudaError):
        api.Engine(0)


def test_error_strings():
    L = api.lib()
    for code in range(6):
        assert L.trs_gpu_error_string(code)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("args", [("mergesort", 50, 0, 42), ("mergesort", 1, 0, 1), ("treemergesort", 16, 4, 3),
                                  ("treemergesort", 5, 2, 9), ("transform", 0, 3, 0), ("transform", 0, 22, 0)])
def test_generator_texts_match_reference(args):
    fam, length, depth, seed = args
    mine = {"mergesort": lambda: W.mergesort(length, seed), "treemergesort": lambda: W.treemergesort(depth, length, seed),
            "transform": lambda: W.transform(depth)}[fam]()
    assert mine == ref.generate(fam, length, depth, seed)


def test_appendix_a_texts_resolve():
    for text in (W.fib(18), W.buildsum(22), W.reverse(64), W.ackermann(3, 6), W.fib_batch(1, roots=16)):
        api.System(text)


def test_splitmix_reference_stream():
    # generators.cpp:14-22 on seed 1: first values mod 32
    r = W.SplitMix64(1)
    assert [r.numeral() for _ in range(5)] == W.generated_numerals("mergesort", 5, seed=1)

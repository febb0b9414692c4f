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


# ---- the reference's own commands with a "gpu" engine (integration/trs_bench_gpu)

EXE = os.path.join(ROOT, "integration", "_ref", "trs_bench_gpu")


def _exe(args, tmp_path, name, text):
    import subprocess

    if not os.path.exists(EXE):
        pytest.skip("integration/_ref/trs_bench_gpu not built (needs /root/reference at build time)")
    path = tmp_path / f"{name}.trs"
    path.write_text(text)
    return subprocess.run([EXE, args[0], str(path), *args[1:]], capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("name", ["fib12", "mergesort64_s1", "transform6", "treemergesort_4_5_s7", "unit_dupvar"])
def test_cmd_bench_divergence_check_with_gpu(tmp_path, name):
    """The reference's cmd_bench (bench.cpp:117-185) over seq, sweep and gpu,
    two repetitions each: every run's normal form (term_equal) and rewrite
    count must equal the first's, else exit 4 (bench.cpp:147-159)."""
    out = _exe(["bench", "--engines", "seq,sweep,gpu", "--reps", "2", "--csv", str(tmp_path / "b.csv")],
               tmp_path, name, CASES[name]["text"])
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert [ln.split(":")[0] for ln in lines] == ["seq", "sweep", "gpu"]
    assert f"{CASES[name]['rewrites']} rewrites" in lines[2]
    rows = (tmp_path / "b.csv").read_text().splitlines()
    assert rows[0] == "engine,run,rewrites,micros,terms_per_s,max_width,median_width"
    assert sum(r.startswith("gpu,") for r in rows) == 2


def test_cmd_bench_full_size_fib18(tmp_path):
    out = _exe(["bench", "--engines", "seq,gpu"], tmp_path, "fib18", W.fib(18))
    assert out.returncode == 0, out.stderr
    assert "24363 rewrites" in out.stdout.splitlines()[1]


@pytest.mark.parametrize("name", ["transform6", "mergesort50_s42", "fib12"])
def test_gpu_trace_csv_through_reference_writer(tmp_path, name):
    """normalize --engine gpu --trace: the GPU trace written by the
    reference's own write_trace_csv (sweep_engine.cpp:432-437): its header,
    one row per sweep, and the rewrites column = the reference's widths."""
    csv = tmp_path / "t.csv"
    out = _exe(["normalize", "--engine", "gpu", "--trace", str(csv)], tmp_path, name, CASES[name]["text"])
    assert out.returncode == 0, out.stderr
    rows = csv.read_text().splitlines()
    assert rows[0] == "sweep,rewrites,live_terms,n,free_len,micros"
    widths = [int(r.split(",")[1]) for r in rows[1:]]
    assert widths == CASES[name]["widths"]


@pytest.mark.parametrize("name", ["mergesort10_s3", "transform3", "fib10", "unit_two_waiters", "buildsum3"])
def test_device_program_dump_equals_reference_dump(tmp_path, name):
    """The dispatch tables as staged on the device, read back and rendered
    (trs_gpu_dump_program), equal the reference's dump-dispatch text
    (dispatch.cpp:98-134) byte for byte."""
    host = _exe(["dump-dispatch"], tmp_path, name, CASES[name]["text"])
    dev = _exe(["dump-dispatch", "--device"], tmp_path, name, CASES[name]["text"])
    assert host.returncode == 0 and dev.returncode == 0, dev.stderr
    assert dev.stdout == host.stdout and host.stdout

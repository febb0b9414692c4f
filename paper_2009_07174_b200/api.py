"""Python mirror of the rewriter's public API over `libtrs_b200.so`.

It mirrors the reference's C++ "load a TRS, build a term, normalise it"
path with the same names and error behaviour:

    System(text)            ~ trs::load_system + trs::compile   (parser.hpp:100, dispatch.hpp:80)
    Store.load(systems)     ~ trs::load                         (term_store.hpp:52)
    Engine.run(options)     ~ trs::run                          (sweep_engine.hpp:47)
    Engine.canonical(k)     ~ extract + canonical relabelling   (term_store.hpp:57)
    EngineError(fault)      ~ trs::EngineError                  (error.hpp:8-20)

Every call goes through the C ABI of `include/trs_gpu.h` (plus the host
library's `trsb_*` entry points).  There is no CPU fallback: when the
extension or a CUDA device is missing the calls raise.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TRS_B200_PROFILE_BUILD=1 selects the profiling build (phase cycle counters)
LIB_PATH = os.path.join(_HERE, "libtrs_b200_prof.so" if os.environ.get("TRS_B200_PROFILE_BUILD") == "1"
                        else "libtrs_b200.so")

OK, STEP_BUDGET, CAPACITY, DANGLING, INVALID, CUDA = range(6)


class EngineFault(enum.Enum):
    StepBudget = STEP_BUDGET
    Capacity = CAPACITY
    DanglingReference = DANGLING


class EngineError(RuntimeError):
    """trs::EngineError: fault is an EngineFault."""

    def __init__(self, fault: EngineFault, message: str):
        super().__init__(message)
        self.fault = fault


class CudaError(RuntimeError):
    pass


class Options(ctypes.Structure):
    """trs_gpu_options (include/trs_gpu.h)."""

    _fields_ = [
        ("step_budget", ctypes.c_uint64),
        ("fixed_capacity", ctypes.c_uint32),
        ("validate", ctypes.c_uint32),
        ("small_enter", ctypes.c_uint32),
        ("small_exit", ctypes.c_uint32),
        ("disable_small", ctypes.c_uint32),
        ("gc_interval", ctypes.c_uint32),
        ("disable_gc", ctypes.c_uint32),
        ("blocks_per_sm", ctypes.c_uint32),
        ("variant", ctypes.c_uint32),
        ("max_blocks", ctypes.c_uint32),
        ("profile", ctypes.c_uint32),
        ("disable_warp_mode", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32 * 4),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("total_rewrites", ctypes.c_uint64),
        ("max_width", ctypes.c_uint64),
        ("sweeps", ctypes.c_uint32),
        ("gc_runs", ctypes.c_uint32),
        ("small_sweeps", ctypes.c_uint32),
        ("launches", ctypes.c_uint32),
        ("regrows", ctypes.c_uint32),
        ("grid_blocks", ctypes.c_uint32),
        ("block_threads", ctypes.c_uint32),
        ("record_words", ctypes.c_uint32),
        ("peak_slots", ctypes.c_uint64),
        ("live_terms", ctypes.c_uint64),
        ("kernel_ms", ctypes.c_double),
        ("gc_ms", ctypes.c_double),
        ("load_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


SWEEP_RECORD = np.dtype(
    [("sweep", np.uint32), ("live_terms", np.uint32), ("rewrites", np.uint64), ("n", np.uint32),
     ("free_len", np.uint32), ("active", np.uint32), ("mode", np.uint32), ("ns", np.uint64)]
)
assert SWEEP_RECORD.itemsize == 40

_lib = None


def lib():
    """Load libtrs_b200.so (raises when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, U32, U64, I = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    u32p = ctypes.POINTER(ctypes.c_uint32)
    sig = {
        "trs_gpu_device_count": ([], I),
        "trs_gpu_open": ([I, ctypes.POINTER(P)], I),
        "trs_gpu_close": ([P], None),
        "trs_gpu_error_string": ([I], ctypes.c_char_p),
        "trs_gpu_last_error": ([P], ctypes.c_char_p),
        "trs_gpu_set_program": ([P, P], I),
        "trs_gpu_load": ([P, U32, P, U32, P, P, U32, P, U64], I),
        "trs_gpu_load_device": ([P, U32, P, U32, P, P, U32, P, U64], I),
        "trs_gpu_run": ([P, ctypes.POINTER(Options), ctypes.POINTER(Stats)], I),
        "trs_gpu_run_async": ([P, ctypes.POINTER(Options)], I),
        "trs_gpu_run_wait": ([P, ctypes.POINTER(Stats)], I),
        "trs_gpu_hold": ([P], I),
        "trs_gpu_jit_info": ([P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, U64], I),
        "trs_gpu_release": ([P], I),
        "trs_gpu_trace": ([P, P, U64, ctypes.POINTER(U64)], I),
        "trs_gpu_phys_trace": ([P, P, U64, ctypes.POINTER(U64)], I),
        "trs_gpu_canonical": ([P, U32, P, U64, ctypes.POINTER(U64), u32p], I),
        "trs_gpu_fetch_store": ([P, u32p, P, P, P, P, P, U32], I),
        "trs_gpu_canonical_all": ([P, P, U64, ctypes.POINTER(U64), P, P, P], I),
        "trs_gpu_live_count": ([P, ctypes.POINTER(U64)], I),
        "trs_gpu_layout_probe": ([P, U32, U32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(U64)], I),
        "trs_gpu_gather_probe": ([I, U64, U32, U32, ctypes.POINTER(ctypes.c_double)], I),
        "trs_gpu_gather_probe_ex": ([I, U64, U32, U32, U32, ctypes.POINTER(ctypes.c_double)], I),
        "trs_gpu_stream": ([P], P),
        "trs_gpu_profile_counters": ([P, P], I),
        "trs_gpu_overhead_probe": ([P, U32, U32, U32, ctypes.POINTER(ctypes.c_double)], I),
        "trs_gpu_compact": ([P, U32, ctypes.POINTER(Stats)], I),
        "trs_gpu_fetch_records": ([P, P, U64, ctypes.POINTER(U64), u32p, P], I),
        "trsb_system_load": ([ctypes.c_char_p, ctypes.POINTER(P), ctypes.c_char_p, ctypes.c_size_t], I),
        "trsb_system_free": ([P], None),
        "trsb_num_symbols": ([P], U32),
        "trsb_symbol_name": ([P, U32], ctypes.c_char_p),
        "trsb_symbol_arity": ([P, U32], U32),
        "trsb_num_rules": ([P], U32),
        "trsb_max_new_slots": ([P], U32),
        "trsb_max_arity": ([P], U32),
        "trsb_program": ([P], P),
        "trsb_dump_dispatch": ([P], P),
        "trsb_print_input": ([P], P),
        "trsb_free": ([P], None),
        "trsb_input_canonical": ([P, P, U64, ctypes.POINTER(U64), u32p], I),
        "trsb_store_load": ([P, U32, U32, ctypes.POINTER(P), ctypes.c_char_p, ctypes.c_size_t], I),
        "trsb_store_free": ([P], None),
        "trsb_store_view": ([P, u32p, u32p, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                             ctypes.POINTER(P), u32p, ctypes.POINTER(P)], None),
        "trsb_store_canonical": ([P, U32, P, U64, ctypes.POINTER(U64), u32p], I),
        "trsb_store_extract_canonical": ([P, U32, P, U64, ctypes.POINTER(U64), u32p], I),
        "trsb_dump_store": ([P, P], P),
        "trsb_store_poke_arg": ([P, U32, U32, U32], None),
        "trsb_gpu_run_store": ([P, P, P, ctypes.POINTER(Options), ctypes.POINTER(Stats), ctypes.c_char_p,
                                ctypes.c_size_t], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def exported_symbols() -> list[str]:
    return [n for n in ("trs_gpu_device_count", "trs_gpu_open", "trs_gpu_close", "trs_gpu_error_string",
                        "trs_gpu_last_error", "trs_gpu_set_program", "trs_gpu_load", "trs_gpu_load_device",
                        "trs_gpu_run", "trs_gpu_run_async", "trs_gpu_run_wait", "trs_gpu_hold",
                        "trs_gpu_release", "trs_gpu_jit_info", "trs_gpu_trace", "trs_gpu_canonical", "trs_gpu_fetch_store",
                        "trs_gpu_canonical_all", "trs_gpu_live_count", "trs_gpu_phys_trace", "trs_gpu_gather_probe_ex", "trs_gpu_layout_probe",
                        "trs_gpu_gather_probe", "trs_gpu_stream", "trs_gpu_compact", "trs_gpu_fetch_records",
                        "trs_gpu_profile_counters", "trs_gpu_overhead_probe")]


def device_count() -> int:
    return lib().trs_gpu_device_count()


def _take_string(ptr) -> str:
    s = ctypes.string_at(ptr).decode()
    lib().trsb_free(ptr)
    return s


def _words(fn, *args) -> tuple[np.ndarray, int]:
    n_words = ctypes.c_uint64(0)
    n_nodes = ctypes.c_uint32(0)
    rc = fn(*args, None, 0, ctypes.byref(n_words), ctypes.byref(n_nodes))
    if rc:
        return rc, None
    out = np.zeros(max(1, n_words.value), np.uint32)
    rc = fn(*args, out.ctypes.data, n_words.value, ctypes.byref(n_words), ctypes.byref(n_nodes))
    return rc, (out[: n_words.value], n_nodes.value)


class System:
    """A parsed, resolved and compiled rewrite system (load_system + compile)."""

    def __init__(self, text: str):
        L = lib()
        h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(8192)
        rc = L.trsb_system_load(text.encode(), ctypes.byref(h), err, len(err))
        if rc:
            raise ValueError(err.value.decode())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.trsb_system_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def num_symbols(self) -> int:
        return lib().trsb_num_symbols(self._h)

    @property
    def num_rules(self) -> int:
        return lib().trsb_num_rules(self._h)

    @property
    def max_new_slots(self) -> int:
        return lib().trsb_max_new_slots(self._h)

    @property
    def max_arity(self) -> int:
        return lib().trsb_max_arity(self._h)

    def symbol_name(self, f: int) -> str:
        return lib().trsb_symbol_name(self._h, f).decode()

    def symbol_arity(self, f: int) -> int:
        return lib().trsb_symbol_arity(self._h, f)

    def symbol_id(self, name: str) -> int:
        for f in range(self.num_symbols):
            if self.symbol_name(f) == name:
                return f
        raise KeyError(name)

    def dump_dispatch(self) -> str:
        return _take_string(lib().trsb_dump_dispatch(self._h))

    def print_input(self) -> str:
        return _take_string(lib().trsb_print_input(self._h))

    def input_canonical(self) -> np.ndarray:
        rc, res = _words(lib().trsb_input_canonical, self._h)
        return res[0]

    def print_words(self, words: np.ndarray) -> str:
        """Render canonical words back to term text (iterative)."""
        names = [self.symbol_name(f) for f in range(self.num_symbols)]
        ar = [self.symbol_arity(f) for f in range(self.num_symbols)]
        # offsets of each node's record
        offs = []
        k = 0
        while k < len(words):
            offs.append(k)
            k += 1 + ar[int(words[k])]
        out = []
        stack = [(0, 0)]
        while stack:
            node, nxt = stack.pop()
            sym = int(words[offs[node]])
            if nxt == 0:
                out.append(names[sym] + "(")
            if nxt < ar[sym]:
                if nxt > 0:
                    out.append(", ")
                stack.append((node, nxt + 1))
                stack.append((int(words[offs[node] + 1 + nxt]), 0))
            else:
                out.append(")")
        return "".join(out)


class Store:
    """Host SoA term store in the reference layout (TermStore)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def load(cls, systems, capacity: int = 0) -> "Store":
        if isinstance(systems, System):
            systems = [systems]
        L = lib()
        arr = (ctypes.c_void_p * len(systems))(*[s.handle for s in systems])
        h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(4096)
        rc = L.trsb_store_load(arr, len(systems), capacity, ctypes.byref(h), err, len(err))
        if rc == CAPACITY:
            raise EngineError(EngineFault.Capacity, err.value.decode())
        if rc:
            raise ValueError(err.value.decode())
        st = cls(h)
        st._systems = systems
        return st

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.trsb_store_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def view(self) -> dict:
        """Zero-copy numpy views of the host arrays (valid while the store lives)."""
        n = ctypes.c_uint32()
        ma = ctypes.c_uint32()
        nr = ctypes.c_uint32()
        ptrs = [ctypes.c_void_p() for _ in range(5)]
        nfp = ctypes.c_void_p()
        lib().trsb_store_view(self._h, ctypes.byref(n), ctypes.byref(ma), ctypes.byref(ptrs[0]),
                              ctypes.byref(ptrs[1]), ctypes.byref(ptrs[2]), ctypes.byref(ptrs[3]),
                              ctypes.byref(nr), ctypes.byref(nfp))
        N, MA, NR = n.value, ma.value, nr.value

        def arr(p, count, ct=ctypes.c_uint32):
            if count == 0 or not p.value:
                return np.zeros(0, np.uint32 if ct is ctypes.c_uint32 else np.uint8)
            return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ct)), (count,))

        return {
            "n": N, "maxarity": MA, "hss": arr(ptrs[0], N), "args": arr(ptrs[1], N * MA),
            "refcounts": arr(ptrs[2], N), "roots": arr(ptrs[3], NR), "nf": arr(nfp, N, ctypes.c_uint8),
            "hss_ptr": ptrs[0].value, "args_ptr": ptrs[1].value, "rc_ptr": ptrs[2].value,
            "roots_ptr": ptrs[3].value, "num_roots": NR,
        }

    def canonical(self, root_index: int = 0) -> np.ndarray:
        rc, res = _words(lib().trsb_store_canonical, self._h, root_index)
        if rc == DANGLING:
            raise EngineError(EngineFault.DanglingReference, "dangling reference in the store")
        return res[0]

    def extract_canonical(self, root_index: int = 0) -> np.ndarray:
        rc, res = _words(lib().trsb_store_extract_canonical, self._h, root_index)
        if rc == DANGLING:
            raise EngineError(EngineFault.DanglingReference, "dangling reference in the store")
        return res[0]

    def dump(self, system: System) -> str:
        return _take_string(lib().trsb_dump_store(system.handle, self._h))

    def poke_arg(self, j: int, slot: int, value: int):
        lib().trsb_store_poke_arg(self._h, j, slot, value)


def _raise(rc: int, message: str):
    if rc == OK:
        return
    if rc in (STEP_BUDGET, CAPACITY, DANGLING):
        raise EngineError(EngineFault(rc), message)
    if rc == INVALID:
        raise ValueError(message)
    raise CudaError(message)


# reserved[1] bits (include/trs_gpu.h)
_RESERVED1_BITS = {"no_resident": 1, "interpreted": 2, "no_runahead": 4}


def make_options(**kw) -> Options:
    """Options by field name; no_resident / interpreted / no_runahead set the
    corresponding reserved[1] bits."""
    o = Options()
    for k, v in kw.items():
        if k in _RESERVED1_BITS:
            if v:
                o.reserved[1] |= _RESERVED1_BITS[k]
        else:
            setattr(o, k, v)
    return o


@dataclass
class RunResult:
    stats: dict
    trace: np.ndarray
    words: list = field(default_factory=list)  # canonical words per root
    nodes: list = field(default_factory=list)

    @property
    def widths(self) -> np.ndarray:
        return self.trace["rewrites"].astype(np.uint64)

    @property
    def total_rewrites(self) -> int:
        return int(self.stats["total_rewrites"])

    @property
    def sweeps(self) -> int:
        return int(self.stats["sweeps"])


class Engine:
    """One device engine (trs_gpu_open ... trs_gpu_close)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = ctypes.c_void_p()
        rc = L.trs_gpu_open(device, ctypes.byref(h))
        if rc:
            raise CudaError(f"cannot open CUDA device {device}: {L.trs_gpu_error_string(rc).decode()}")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.trs_gpu_close(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _err(self) -> str:
        return lib().trs_gpu_last_error(self._h).decode()

    def set_program(self, system: System):
        rc = lib().trs_gpu_set_program(self._h, lib().trsb_program(system.handle))
        _raise(rc, self._err())

    def load(self, store: Store, capacity: int = 0):
        v = store.view()
        rc = lib().trs_gpu_load(self._h, v["n"], v["roots_ptr"], v["num_roots"], v["hss_ptr"], v["args_ptr"],
                                v["maxarity"], v["rc_ptr"], capacity)
        _raise(rc, self._err())

    def load_device(self, n, roots: np.ndarray, d_hss: int, d_args: int, maxarity: int, d_rc: int,
                    capacity: int = 0):
        roots = np.ascontiguousarray(roots, np.uint32)
        rc = lib().trs_gpu_load_device(self._h, n, roots.ctypes.data, len(roots), d_hss, d_args, maxarity, d_rc,
                                       capacity)
        _raise(rc, self._err())

    def run(self, options: Options | None = None) -> dict:
        st = Stats()
        rc = lib().trs_gpu_run(self._h, ctypes.byref(options or Options()), ctypes.byref(st))
        _raise(rc, self._err())
        return st.as_dict()

    def run_async(self, options: Options | None = None):
        _raise(lib().trs_gpu_run_async(self._h, ctypes.byref(options or Options())), self._err())

    def run_wait(self) -> dict:
        st = Stats()
        rc = lib().trs_gpu_run_wait(self._h, ctypes.byref(st))
        _raise(rc, self._err())
        return st.as_dict()

    def jit_info(self) -> dict:
        """Whether set_program compiled the specialised step loop (jit.hpp)."""
        act = ctypes.c_int(0)
        sec = ctypes.c_double(0)
        log = ctypes.create_string_buffer(1 << 16)
        _raise(lib().trs_gpu_jit_info(self._h, ctypes.byref(act), ctypes.byref(sec), log, len(log)), self._err())
        return {"active": bool(act.value), "seconds": sec.value, "log": log.value.decode(errors="replace")}

    def hold(self):
        _raise(lib().trs_gpu_hold(self._h), self._err())

    def release(self):
        _raise(lib().trs_gpu_release(self._h), self._err())

    @property
    def stream(self) -> int:
        """cudaStream_t of this engine (for torch.cuda.ExternalStream + events)."""
        return lib().trs_gpu_stream(self._h)

    def overhead_probe(self, iters: int = 2000, mode: int = 0, max_blocks: int = 0) -> float:
        ns = ctypes.c_double(0)
        rc = lib().trs_gpu_overhead_probe(self._h, iters, mode, max_blocks, ctypes.byref(ns))
        _raise(rc, self._err())
        return ns.value

    def profile_counters(self) -> dict:
        out = np.zeros(26, np.uint64)
        lib().trs_gpu_profile_counters(self._h, out.ctypes.data)
        keys = ("match", "claim", "apply", "push", "sweep", "sweeps", "steps", "spare",
                "m_record", "m_children", "m_slots", "m_rules",
                "gc_claim_ns", "gc_count_ns", "gc_scatter_ns", "gc_remap_ns", "gc_hops", "gc_max_hops",
                "wmax_match", "wmax_claim", "wmax_apply", "wmax_push", "wmax_record", "wmax_children",
                "wmax_slots", "wmax_rules")
        return {k: int(v) for k, v in zip(keys, out)}

    def compact(self, max_rounds: int = 8) -> dict:
        st = Stats()
        rc = lib().trs_gpu_compact(self._h, max_rounds, ctypes.byref(st))
        _raise(rc, self._err())
        return st.as_dict()

    def fetch_records(self, dst_ptr: int | None = None, cap_bytes: int = 0, roots_ptr: int | None = None):
        """Raw arena copy into a (pinned) host buffer; returns (bytes, record_words)."""
        nb = ctypes.c_uint64(0)
        rw = ctypes.c_uint32(0)
        rc = lib().trs_gpu_fetch_records(self._h, dst_ptr, cap_bytes, ctypes.byref(nb), ctypes.byref(rw), roots_ptr)
        _raise(rc, self._err())
        return nb.value, rw.value

    def trace(self) -> np.ndarray:
        n = ctypes.c_uint64(0)
        lib().trs_gpu_trace(self._h, None, 0, ctypes.byref(n))
        out = np.zeros(n.value, SWEEP_RECORD)
        if n.value:
            rc = lib().trs_gpu_trace(self._h, out.ctypes.data, n.value, ctypes.byref(n))
            _raise(rc, self._err())
        return out

    def phys_trace(self) -> np.ndarray:
        """Per physical sweep (step-loop iteration) records of the last run."""
        n = ctypes.c_uint64(0)
        lib().trs_gpu_phys_trace(self._h, None, 0, ctypes.byref(n))
        out = np.zeros(n.value, SWEEP_RECORD)
        if n.value:
            rc = lib().trs_gpu_phys_trace(self._h, out.ctypes.data, n.value, ctypes.byref(n))
            _raise(rc, self._err())
        return out

    def canonical(self, root_index: int = 0) -> np.ndarray:
        rc, res = _words(lib().trs_gpu_canonical, self._h, root_index)
        _raise(rc, self._err())
        return res[0]

    def canonical_all(self, num_roots: int, words: bool = True) -> dict:
        """Canonical words of every root, relabelled on the device
        (trs_gpu_canonical_all): {'words': [per-root arrays] or None,
        'hashes': uint64[num_roots], 'nodes': uint32[num_roots]}."""
        L = lib()
        nw = ctypes.c_uint64(0)
        offs = np.zeros(num_roots + 1, np.uint64)
        hashes = np.zeros(num_roots, np.uint64)
        nodes = np.zeros(num_roots, np.uint32)
        rc = L.trs_gpu_canonical_all(self._h, None, 0, ctypes.byref(nw), offs.ctypes.data, hashes.ctypes.data,
                                     nodes.ctypes.data)
        _raise(rc, self._err())
        out = {"hashes": hashes, "nodes": nodes, "offsets": offs, "words": None}
        if words:
            flat = np.zeros(max(1, nw.value), np.uint32)
            rc = L.trs_gpu_canonical_all(self._h, flat.ctypes.data, nw.value, ctypes.byref(nw), None, None, None)
            _raise(rc, self._err())
            out["words"] = [flat[int(offs[k]):int(offs[k + 1])] for k in range(num_roots)]
        return out

    def layout_probe(self, layout: int, iters: int = 5) -> dict:
        """AoS (0) vs SoA (1) probe pass over the current store, in slot order or (+2) a hashed order
        (trs_gpu_layout_probe)."""
        ms = ctypes.c_double(0)
        n = ctypes.c_uint64(0)
        _raise(lib().trs_gpu_layout_probe(self._h, layout, iters, ctypes.byref(ms), ctypes.byref(n)), self._err())
        return {"ms": ms.value, "slots": n.value}

    def live_count(self) -> int:
        """Slots with refcount > 0 (the reference's live_terms, sweep_engine.cpp:122-123)."""
        v = ctypes.c_uint64(0)
        _raise(lib().trs_gpu_live_count(self._h, ctypes.byref(v)), self._err())
        return v.value

    def fetch_store(self, maxarity: int, num_roots: int) -> dict:
        """The live store in the reference TermStore layout (trs_gpu_fetch_store):
        slots renumbered 1..n-1, args column-major [maxarity, n], refcounts
        recounted over the exported store, renumbered roots."""
        L = lib()
        n = ctypes.c_uint32(0)
        rc = L.trs_gpu_fetch_store(self._h, ctypes.byref(n), None, None, None, None, None, 0)
        _raise(rc, self._err())
        N = n.value
        roots = np.zeros(max(1, num_roots), np.uint32)
        hss = np.zeros(N, np.uint32)
        args = np.zeros((maxarity, N), np.uint32)
        rcs = np.zeros(N, np.uint32)
        nf = np.zeros(N, np.uint8)
        rc = L.trs_gpu_fetch_store(self._h, ctypes.byref(n), roots.ctypes.data, hss.ctypes.data,
                                   args.ctypes.data if maxarity else None, rcs.ctypes.data, nf.ctypes.data, N)
        _raise(rc, self._err())
        return {"n": N, "hss": hss, "args": args, "refcounts": rcs, "nf": nf, "roots": roots[:num_roots]}

    def normalize(self, system: System, store: Store, options: Options | None = None,
                  words: bool = True) -> RunResult:
        self.set_program(system)
        self.load(store)
        stats = self.run(options)
        res = RunResult(stats=stats, trace=self.trace())
        if words:
            res.words = self.canonical_all(store.view()["num_roots"])["words"]
        return res


def canonical_hash(words: np.ndarray) -> int:
    """The per-root hash trs_gpu_canonical_all reports, restated in numpy:
    sum over positions k of SplitMix64((k << 32) ^ w_k ^ 0x9e3779b97f4a7c15)
    modulo 2^64 (canon.cuh, canon_mix)."""
    w = np.asarray(words, np.uint64)
    with np.errstate(over="ignore"):
        z = (np.arange(w.size, dtype=np.uint64) << np.uint64(32)) ^ w ^ np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return int(z.sum(dtype=np.uint64))


def gather_probe(device: int = 0, bytes_: int = 4 << 30, bytes_per_access: int = 4, iters: int = 5,
                 ilp: int = 4) -> float:
    g = ctypes.c_double(0)
    rc = lib().trs_gpu_gather_probe_ex(device, bytes_, bytes_per_access, ilp, iters, ctypes.byref(g))
    _raise(rc, "gather probe failed")
    return g.value


def normalize_texts(texts, device: int = 0, options: Options | None = None, engine: Engine | None = None,
                    words: bool = True) -> RunResult:
    """Parse each text, load all inputs as one multi-root store, normalise on the GPU."""
    if isinstance(texts, str):
        texts = [texts]
    systems = [System(t) for t in texts]
    store = Store.load(systems)
    eng = engine or Engine(device)
    return eng.normalize(systems[0], store, options, words=words)

// gpu::run — the reference's run(TermStore&, const DispatchTable&,
// const SweepOptions&) (proj/include/trs/sweep_engine.hpp:47) on the B200
// engine behind trs_gpu.h, plus the extern "C" surface the Python mirror,
// the tests and bench.py bind with ctypes.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <memory>
#include <mutex>

#include "trs_host.hpp"

namespace trs_b200 {

namespace {

void throw_status(int status, trs_gpu_engine* e) {
    std::string msg = std::string(trs_gpu_error_string(status));
    const char* detail = e ? trs_gpu_last_error(e) : "";
    if (detail && *detail) msg = detail;
    switch (status) {
        case TRS_GPU_OK: return;
        case TRS_GPU_STEP_BUDGET: throw EngineError(EngineFault::StepBudget, msg);
        case TRS_GPU_CAPACITY: throw EngineError(EngineFault::Capacity, msg);
        case TRS_GPU_DANGLING: throw EngineError(EngineFault::DanglingReference, msg);
        case TRS_GPU_INVALID: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}

struct EngineCache {
    std::mutex mu;
    std::map<int, trs_gpu_engine*> engines;
    ~EngineCache() {
        for (auto& [d, e] : engines) trs_gpu_close(e);
    }
};

trs_gpu_engine* engine_for(int device) {
    static EngineCache cache;
    std::lock_guard<std::mutex> g(cache.mu);
    auto it = cache.engines.find(device);
    if (it != cache.engines.end()) return it->second;
    trs_gpu_engine* e = nullptr;
    int rc = trs_gpu_open(device, &e);
    if (rc) throw std::runtime_error("cannot open CUDA device " + std::to_string(device) + " for the B200 rewriter");
    cache.engines[device] = e;
    return e;
}

}  // namespace

// Page-locked allocations carry a 16-byte tag so that frees know which
// allocator they came from (cudaHostAlloc, or malloc without a device).
void* pinned_alloc(std::size_t bytes) {
    constexpr std::size_t kTag = 16;
    void* p = nullptr;
    const bool have_device = trs_gpu_device_count() > 0;
    if (have_device && cudaHostAlloc(&p, bytes + kTag, cudaHostAllocDefault) == cudaSuccess) {
        *static_cast<std::uint32_t*>(p) = 0x50494e4eu;  // "PINN"
    } else {
        if (have_device) cudaGetLastError();
        p = std::malloc(bytes + kTag);
        if (!p) throw std::bad_alloc();
        *static_cast<std::uint32_t*>(p) = 0x48454150u;  // "HEAP"
    }
    return static_cast<char*>(p) + kTag;
}

void pinned_free(void* q) noexcept {
    if (!q) return;
    void* p = static_cast<char*>(q) - 16;
    if (*static_cast<std::uint32_t*>(p) == 0x50494e4eu)
        cudaFreeHost(p);
    else
        std::free(p);
}

// Load, run and write the normal form back into `store` with the given engine.
SweepTrace run_with(trs_gpu_engine* e, TermStore& store, const FlatProgram& flat, const gpu::GpuOptions& o) {
    trs_gpu_program view = flat.view();
    throw_status(trs_gpu_set_program(e, &view), e);
    std::uint64_t cap = o.fixed_capacity ? store.capacity : 0;
    throw_status(trs_gpu_load(e, store.n, store.roots.data(), static_cast<std::uint32_t>(store.roots.size()),
                              store.hss.data(), store.args.data(), store.maxarity, store.refcounts.data(), cap),
                 e);
    trs_gpu_options opt = o.raw;
    opt.step_budget = o.step_budget;
    opt.fixed_capacity = o.fixed_capacity ? 1 : 0;
    opt.validate = o.validate ? 1 : 0;
    SweepTrace trace;
    int rc = trs_gpu_run(e, &opt, &trace.stats);
    std::uint64_t count = 0;
    trs_gpu_trace(e, nullptr, 0, &count);
    std::vector<trs_gpu_sweep_record> recs(count);
    if (count) trs_gpu_trace(e, recs.data(), count, &count);
    for (const trs_gpu_sweep_record& r : recs)
        trace.records.push_back({r.sweep, r.rewrites, r.live_terms, r.n, r.free_len, r.micros_x1000 / 1000});
    if (rc != TRS_GPU_OK && rc != TRS_GPU_STEP_BUDGET && rc != TRS_GPU_CAPACITY) throw_status(rc, e);
    // write the (possibly partial) store back, renumbered, like the reference's in-place mutation
    std::uint32_t n = 0;
    throw_status(trs_gpu_fetch_store(e, &n, nullptr, nullptr, nullptr, nullptr, nullptr, 0), e);
    store.n = n;
    store.capacity = std::max(store.capacity, n);
    store.hss.assign(n, 0);
    store.args.assign(static_cast<std::size_t>(store.maxarity) * n, 0);
    store.refcounts.assign(n, 0);
    store.nf.assign(n, 0);
    throw_status(trs_gpu_fetch_store(e, &n, store.roots.data(), store.hss.data(),
                                     store.maxarity ? store.args.data() : nullptr, store.refcounts.data(),
                                     store.nf.data(), n),
                 e);
    throw_status(rc, e);
    return trace;
}

namespace gpu {

SweepTrace run(TermStore& store, const RewriteSystem& system, const DispatchTable& table, const GpuOptions& options) {
    FlatProgram flat = flatten(system, table);
    return run_with(engine_for(options.device), store, flat, options);
}

}  // namespace gpu

}  // namespace trs_b200

// ===========================================================================
// extern "C" surface of the host library (ctypes in Python, bench.py)

using namespace trs_b200;

struct trsb_system {
    RewriteSystem sys;
    DispatchTable table;
    FlatProgram flat;
    trs_gpu_program view;
};

struct trsb_store {
    TermStore store;
};

namespace {

void write_err(char* err, size_t len, const std::string& m) {
    if (err && len) {
        std::strncpy(err, m.c_str(), len - 1);
        err[len - 1] = 0;
    }
}

char* dup_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

int copy_words(const std::vector<std::uint32_t>& w, std::uint32_t nodes, std::uint32_t* out, std::uint64_t cap,
               std::uint64_t* n_words, std::uint32_t* n_nodes) {
    if (n_words) *n_words = w.size();
    if (n_nodes) *n_nodes = nodes;
    if (out && cap >= w.size()) std::memcpy(out, w.data(), w.size() * sizeof(std::uint32_t));
    return 0;
}

}  // namespace

extern "C" {

// Parse, resolve and compile a .trs text.  Returns 0, or 4 with the
// formatted diagnostics in err.
int trsb_system_load(const char* text, trsb_system** out, char* err, size_t errlen) {
    *out = nullptr;
    try {
        ResolveResult r = load_system(text);
        if (!r.system) {
            std::string m;
            for (const ParseError& e : r.errors) m += format_error("<text>", e) + "\n";
            write_err(err, errlen, m);
            return TRS_GPU_INVALID;
        }
        auto* s = new trsb_system();
        s->sys = std::move(*r.system);
        s->table = compile(s->sys);
        s->flat = flatten(s->sys, s->table);
        s->view = s->flat.view();
        *out = s;
        return TRS_GPU_OK;
    } catch (const std::exception& e) {
        write_err(err, errlen, e.what());
        return TRS_GPU_INVALID;
    }
}

void trsb_system_free(trsb_system* s) { delete s; }

uint32_t trsb_num_symbols(const trsb_system* s) { return static_cast<uint32_t>(s->sys.signature.symbols.size()); }
const char* trsb_symbol_name(const trsb_system* s, uint32_t f) { return s->sys.signature.symbols.at(f).name.c_str(); }
uint32_t trsb_symbol_arity(const trsb_system* s, uint32_t f) { return s->sys.signature.symbols.at(f).arity; }
uint32_t trsb_num_rules(const trsb_system* s) { return static_cast<uint32_t>(s->sys.rules.size()); }
uint32_t trsb_max_new_slots(const trsb_system* s) { return s->table.max_new_slots; }
uint32_t trsb_max_arity(const trsb_system* s) { return s->sys.signature.max_arity; }
const trs_gpu_program* trsb_program(const trsb_system* s) { return &s->view; }

char* trsb_dump_dispatch(const trsb_system* s) { return dup_string(dump_dispatch(s->sys, s->table)); }
char* trsb_print_input(const trsb_system* s) { return dup_string(print_term(s->sys.signature, s->sys.terms, s->sys.input_term)); }
void trsb_free(void* p) { std::free(p); }

int trsb_input_canonical(const trsb_system* s, uint32_t* words, uint64_t cap, uint64_t* n_words, uint32_t* n_nodes) {
    std::uint32_t nodes = 0;
    auto w = canonical_words(s->sys.terms, s->sys.input_term, &nodes);
    return copy_words(w, nodes, words, cap, n_words, n_nodes);
}

// Load the input terms of k systems (same signature) as one store with k
// pinned roots.  capacity 0 = automatic.
int trsb_store_load(trsb_system* const* systems, uint32_t k, uint32_t capacity, trsb_store** out, char* err,
                    size_t errlen) {
    *out = nullptr;
    try {
        if (k == 0) throw std::invalid_argument("no systems");
        const Signature& sig = systems[0]->sys.signature;
        std::vector<std::pair<const TermArena*, TermRef>> inputs;
        for (uint32_t i = 0; i < k; ++i) {
            const Signature& si = systems[i]->sys.signature;
            if (si.symbols.size() != sig.symbols.size())
                throw std::invalid_argument("batched inputs need identical signatures");
            for (std::size_t f = 0; f < si.symbols.size(); ++f)
                if (si.symbols[f].name != sig.symbols[f].name || si.symbols[f].arity != sig.symbols[f].arity)
                    throw std::invalid_argument("batched inputs need identical signatures");
            inputs.emplace_back(&systems[i]->sys.terms, systems[i]->sys.input_term);
        }
        auto* st = new trsb_store();
        st->store = load_many(sig, inputs, capacity);
        *out = st;
        return TRS_GPU_OK;
    } catch (const EngineError& e) {
        write_err(err, errlen, e.what());
        return TRS_GPU_CAPACITY;
    } catch (const std::exception& e) {
        write_err(err, errlen, e.what());
        return TRS_GPU_INVALID;
    }
}

void trsb_store_free(trsb_store* s) { delete s; }

void trsb_store_view(const trsb_store* s, uint32_t* n, uint32_t* maxarity, const uint32_t** hss,
                     const uint32_t** args, const uint32_t** refcounts, const uint32_t** roots, uint32_t* num_roots,
                     const uint8_t** nf) {
    const TermStore& t = s->store;
    if (n) *n = t.n;
    if (maxarity) *maxarity = t.maxarity;
    if (hss) *hss = t.hss.data();
    if (args) *args = t.args.data();
    if (refcounts) *refcounts = t.refcounts.data();
    if (roots) *roots = t.roots.data();
    if (num_roots) *num_roots = static_cast<uint32_t>(t.roots.size());
    if (nf) *nf = t.nf.data();
}

int trsb_store_canonical(const trsb_store* s, uint32_t root_index, uint32_t* words, uint64_t cap, uint64_t* n_words,
                         uint32_t* n_nodes) {
    try {
        std::uint32_t nodes = 0;
        auto w = canonical_words(s->store, root_index, &nodes);
        return copy_words(w, nodes, words, cap, n_words, n_nodes);
    } catch (const EngineError&) {
        return TRS_GPU_DANGLING;
    } catch (const std::exception&) {
        return TRS_GPU_INVALID;
    }
}

// extract() into a fresh arena, then canonical words of that tree: checks
// extract's own dangling detection and the load/extract round trip.
int trsb_store_extract_canonical(const trsb_store* s, uint32_t root_index, uint32_t* words, uint64_t cap,
                                 uint64_t* n_words, uint32_t* n_nodes) {
    try {
        TermArena a;
        TermRef t = extract(s->store, a, root_index);
        std::uint32_t nodes = 0;
        auto w = canonical_words(a, t, &nodes);
        return copy_words(w, nodes, words, cap, n_words, n_nodes);
    } catch (const EngineError&) {
        return TRS_GPU_DANGLING;
    } catch (const std::exception&) {
        return TRS_GPU_INVALID;
    }
}

char* trsb_dump_store(const trsb_system* sys, const trsb_store* s) { return dup_string(dump_store(sys->sys.signature, s->store)); }

// Corrupt one argument (tests of the dangling-reference path).
void trsb_store_poke_arg(trsb_store* s, uint32_t j, uint32_t slot, uint32_t value) {
    s->store.args.at(static_cast<std::size_t>(j) * s->store.n + slot) = value;
}

// gpu::run on an explicit engine: load the store, normalise, write the
// normal form back into it.  Returns a trs_gpu.h status; err gets details.
int trsb_gpu_run_store(trs_gpu_engine* e, const trsb_system* sys, trsb_store* st, const trs_gpu_options* opt,
                       trs_gpu_stats* stats, char* err, size_t errlen) {
    try {
        gpu::GpuOptions o;
        if (opt) {
            o.raw = *opt;
            o.step_budget = opt->step_budget ? opt->step_budget : 1000000000ull;
            o.fixed_capacity = opt->fixed_capacity != 0;
            o.validate = opt->validate != 0;
        }
        SweepTrace t = run_with(e, st->store, sys->flat, o);
        if (stats) *stats = t.stats;
        return TRS_GPU_OK;
    } catch (const EngineError& ex) {
        write_err(err, errlen, ex.what());
        return ex.fault == EngineFault::StepBudget ? TRS_GPU_STEP_BUDGET
               : ex.fault == EngineFault::Capacity ? TRS_GPU_CAPACITY
                                                   : TRS_GPU_DANGLING;
    } catch (const std::invalid_argument& ex) {
        write_err(err, errlen, ex.what());
        return TRS_GPU_INVALID;
    } catch (const std::exception& ex) {
        write_err(err, errlen, ex.what());
        return TRS_GPU_CUDA;
    }
}

}  // extern "C"

// Drop-in adapter: the reference's own sweep-engine signature
//
//   trs::SweepTrace trs::run(TermStore&, const DispatchTable&, const SweepOptions&)
//                                           (proj/include/trs/sweep_engine.hpp:38-47)
//
// served by the B200 engine through the C ABI of include/trs_gpu.h.  Header
// only; include it in a translation unit that already sees the reference's
// headers (trs/term_store.hpp, trs/dispatch.hpp, trs/sweep_engine.hpp) and
// link libtrs_b200.so.  INTEGRATION.md shows the one-line "gpu" branch in
// run_engine (proj/src/bench.cpp:49-69) that calls it.
//
// What it does, in the reference's terms:
//  * flattens DispatchTable::by_symbol (dispatch.hpp:73-78) into
//    trs_gpu_program: MatchStep paths become (parent step, child index)
//    pairs, RhsRef becomes TRS_GPU_REF_NODE | index or a var slot;
//  * passes TermStore's SoA columns (term_store.hpp:15-45) as is (args are
//    concatenated column by column);
//  * runs, then writes the normal form back into the TermStore (slots
//    renumbered densely; root, hss, args, refcounts, nf, n updated) so the
//    reference's extract (term_store.cpp:77-116) works unchanged;
//  * maps status codes onto trs::EngineError(EngineFault) (error.hpp:8-20).
#pragma once

#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "trs_gpu.h"

namespace trs::gpu {

struct GpuOptions {
    int device = 0;
    trs::SweepOptions sweep{};  // step_budget, fixed_capacity, validate are honoured
    trs_gpu_options raw{};      // device knobs
};

namespace detail {

inline void check(int status, trs_gpu_engine* e) {
    if (status == TRS_GPU_OK) return;
    std::string msg = trs_gpu_last_error(e);
    if (msg.empty()) msg = trs_gpu_error_string(status);
    switch (status) {
        case TRS_GPU_STEP_BUDGET: throw trs::EngineError(trs::EngineFault::StepBudget, msg);
        case TRS_GPU_CAPACITY: throw trs::EngineError(trs::EngineFault::Capacity, msg);
        case TRS_GPU_DANGLING: throw trs::EngineError(trs::EngineFault::DanglingReference, msg);
        case TRS_GPU_INVALID: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}

struct Flat {
    std::vector<uint32_t> arity, rule_begin, refs;
    std::vector<trs_gpu_rule> rules;
    std::vector<trs_gpu_step> steps;
    std::vector<trs_gpu_instr> instrs;
};

inline Flat flatten(const trs::TermStore& store, const trs::DispatchTable& table) {
    Flat f;
    f.arity = store.arity_of;
    f.rule_begin.push_back(0);
    for (std::size_t sym = 0; sym < table.by_symbol.size(); ++sym) {
        for (const trs::CompiledRule& c : table.by_symbol[sym]) {
            trs_gpu_rule r{};
            r.source_order = c.rule_index;
            r.first_step = static_cast<uint32_t>(f.steps.size());
            r.num_steps = static_cast<uint32_t>(c.program.steps.size());
            r.first_instr = static_cast<uint32_t>(f.instrs.size());
            r.num_instrs = static_cast<uint32_t>(c.rhs.instructions.size());
            r.num_vars = static_cast<uint32_t>(c.program.slot_vars.size());
            r.root_ref = c.rhs.collapses() ? c.rhs.root_ref.index : (TRS_GPU_REF_NODE | c.rhs.root_ref.index);
            // a step's parent is the (CheckHead) step whose path is its path minus the last index
            std::map<std::vector<uint8_t>, int32_t> step_of_path;
            for (std::size_t t = 0; t < c.program.steps.size(); ++t) {
                const trs::MatchStep& st = c.program.steps[t];
                trs_gpu_step s{};
                s.kind = st.kind == trs::MatchStep::Kind::CheckHead ? TRS_GPU_STEP_CHECK_HEAD : TRS_GPU_STEP_BIND_VAR;
                std::vector<uint8_t> parent_path(st.path.begin(), st.path.end() - 1);
                s.parent = parent_path.empty() ? -1 : step_of_path.at(parent_path);
                s.child = st.path.back();
                s.value = st.kind == trs::MatchStep::Kind::CheckHead ? st.symbol : st.var_slot;
                step_of_path[st.path] = static_cast<int32_t>(t);
                f.steps.push_back(s);
            }
            for (const trs::RhsInstr& in : c.rhs.instructions) {
                trs_gpu_instr i{};
                i.symbol = in.symbol;
                i.indegree = in.indegree;
                i.first_ref = static_cast<uint32_t>(f.refs.size());
                for (const trs::RhsRef& ref : in.children)
                    f.refs.push_back(ref.kind == trs::RhsRef::Kind::Node ? (TRS_GPU_REF_NODE | ref.index) : ref.index);
                f.instrs.push_back(i);
            }
            f.rules.push_back(r);
        }
        f.rule_begin.push_back(static_cast<uint32_t>(f.rules.size()));
    }
    return f;
}

inline trs_gpu_program program_of(const Flat& f) {
    trs_gpu_program p{};
    p.num_symbols = static_cast<uint32_t>(f.arity.size());
    p.arity = f.arity.data();
    p.rule_begin = f.rule_begin.data();
    p.num_rules = static_cast<uint32_t>(f.rules.size());
    p.rules = f.rules.data();
    p.num_steps = static_cast<uint32_t>(f.steps.size());
    p.steps = f.steps.data();
    p.num_instrs = static_cast<uint32_t>(f.instrs.size());
    p.instrs = f.instrs.data();
    p.num_refs = static_cast<uint32_t>(f.refs.size());
    p.refs = f.refs.data();
    return p;
}

// The flattened program as one word string: equal strings, equal programs.
inline std::vector<uint32_t> fingerprint(const Flat& f) {
    std::vector<uint32_t> k;
    auto put = [&](const void* p, std::size_t bytes) {
        k.push_back(static_cast<uint32_t>(bytes));
        const std::size_t w = k.size();
        k.resize(w + (bytes + 3) / 4, 0u);
        if (bytes) std::memcpy(k.data() + w, p, bytes);
    };
    put(f.arity.data(), f.arity.size() * 4);
    put(f.rule_begin.data(), f.rule_begin.size() * 4);
    put(f.refs.data(), f.refs.size() * 4);
    put(f.rules.data(), f.rules.size() * sizeof(trs_gpu_rule));
    put(f.steps.data(), f.steps.size() * sizeof(trs_gpu_step));
    put(f.instrs.data(), f.instrs.size() * sizeof(trs_gpu_instr));
    return k;
}

// One engine per process, kept open across calls, and the program it holds:
// set_program (which specialises and compiles the step loop, jit.hpp) runs
// only when a different DispatchTable comes.  Calls are serialised.
struct Cache {
    std::mutex mu;
    trs_gpu_engine* e = nullptr;
    int device = -1;
    std::vector<uint32_t> program;
};

inline Cache& cache() {
    static Cache* c = new Cache();  // never destroyed: no CUDA calls after the runtime's teardown
    return *c;
}

}  // namespace detail

// trs::run's contract on the B200: mutates `store` into the normal form and
// returns the per-sweep trace (widths bit-exact to the reference's).
inline trs::SweepTrace run(trs::TermStore& store, const trs::DispatchTable& table, const GpuOptions& opt = {}) {
    detail::Cache& cache = detail::cache();
    std::lock_guard<std::mutex> guard(cache.mu);
    if (!cache.e || cache.device != opt.device) {
        if (cache.e) trs_gpu_close(cache.e);
        cache.e = nullptr;
        cache.program.clear();
        detail::check(trs_gpu_open(opt.device, &cache.e), nullptr);
        cache.device = opt.device;
    }
    trs_gpu_engine* e = cache.e;
    detail::Flat f = detail::flatten(store, table);
    std::vector<uint32_t> fp = detail::fingerprint(f);
    if (fp != cache.program) {
        trs_gpu_program p = detail::program_of(f);
        cache.program.clear();
        detail::check(trs_gpu_set_program(e, &p), e);
        cache.program = std::move(fp);
    }
    // TermStore columns args[j][i] -> column-major [maxarity * n]
    const uint32_t n = store.n;
    std::vector<uint32_t> args(static_cast<std::size_t>(store.maxarity) * n);
    for (uint32_t j = 0; j < store.maxarity; ++j)
        std::memcpy(args.data() + static_cast<std::size_t>(j) * n, store.args[j].data(), sizeof(uint32_t) * n);
    uint32_t root = store.root;
    const uint64_t cap = opt.sweep.fixed_capacity ? store.capacity : 0;
    detail::check(trs_gpu_load(e, n, &root, 1, store.hss.data(), args.data(), store.maxarity,
                               store.refcounts.data(), cap),
                  e);
    trs_gpu_options o = opt.raw;
    o.step_budget = opt.sweep.step_budget;
    o.fixed_capacity = opt.sweep.fixed_capacity ? 1 : 0;
    o.validate = opt.sweep.validate ? 1 : 0;
    trs_gpu_stats stats{};
    const int rc = trs_gpu_run(e, &o, &stats);
    trs::SweepTrace trace;
    uint64_t count = 0;
    trs_gpu_trace(e, nullptr, 0, &count);
    std::vector<trs_gpu_sweep_record> recs(count);
    if (count) trs_gpu_trace(e, recs.data(), count, &count);
    // one record per logical sweep (the reference's sweeps): the width is
    // exact; live_terms/n/free_len/micros are per physical sweep on the GPU
    // (trs_gpu_phys_trace) and are filled for the last record only, from the
    // written-back store below (n = its slots, live_terms = its terms)
    for (const trs_gpu_sweep_record& r : recs) {
        trs::SweepRecord sr;
        sr.sweep = r.sweep;
        sr.rewrites = r.rewrites;
        sr.live_terms = 0;
        sr.n = 0;
        sr.free_len = 0;
        sr.micros = 0;
        trace.records.push_back(sr);
    }
    if (rc != TRS_GPU_OK && rc != TRS_GPU_STEP_BUDGET && rc != TRS_GPU_CAPACITY) detail::check(rc, e);
    // write the normal form back in the reference layout
    uint32_t nn = 0;
    detail::check(trs_gpu_fetch_store(e, &nn, nullptr, nullptr, nullptr, nullptr, nullptr, 0), e);
    std::vector<uint32_t> hss(nn), cols(static_cast<std::size_t>(store.maxarity) * nn), rcs(nn);
    std::vector<uint8_t> nf(nn);
    detail::check(trs_gpu_fetch_store(e, &nn, &root, hss.data(), store.maxarity ? cols.data() : nullptr, rcs.data(),
                                      nf.data(), nn),
                  e);
    if (store.capacity < nn) store.grow(nn);
    for (uint32_t i = 0; i < nn; ++i) {
        store.hss[i] = hss[i];
        store.refcounts[i] = rcs[i];
        store.nf[i] = nf[i];
        store.collected[i] = 0;
        for (uint32_t j = 0; j < store.maxarity; ++j) store.args[j][i] = cols[static_cast<std::size_t>(j) * nn + i];
    }
    store.n = nn;
    store.root = root;
    if (!trace.records.empty()) {
        trace.records.back().n = nn;
        trace.records.back().live_terms = nn > 0 ? nn - 1 : 0;
        trace.records.back().micros = static_cast<std::uint64_t>(stats.kernel_ms * 1e3);
    }
    store.next_free_begin = store.next_free_end = 0;
    store.next_fresh = 0;
    detail::check(rc, e);
    return trace;
}

}  // namespace trs::gpu

// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Thin extern "C" driver over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libtrs_ref.so).  It lets the Python tests, the golden-fixture
// generator and bench.py's `--impl reference` arm call the reference's own
// public API:
//
//   load_system        (proj/include/trs/parser.hpp:100, proj/src/parser.cpp:569)
//   compile            (proj/include/trs/dispatch.hpp:80, proj/src/dispatch.cpp:63)
//   normalize          (proj/include/trs/seq_engine.hpp:29, proj/src/seq_engine.cpp:136)
//   load / run / extract (proj/include/trs/term_store.hpp:52,57, sweep_engine.hpp:47)
//   dump_dispatch      (proj/src/dispatch.cpp:98)
//   generate           (proj/src/generators.cpp:146)
//
// Everything runs on a thread with a 2 GiB stack: the reference resolver
// (parser.cpp:443-491) and shared_ptr teardown recurse once per nesting level
// (SURVEY.md §8c "Stack hazard").
//
// The canonical form of a normal form is the DAG-level relabelling of
// iterative pre-order from the root, children
// left to right, ids assigned on first visit; emitted as (symbol, child ids…)
// per id.  The product computes the same words from its device store.

#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "trs/bench.hpp"
#include "trs/dispatch.hpp"
#include "trs/generators.hpp"
#include "trs/parser.hpp"
#include "trs/seq_engine.hpp"
#include "trs/sweep_engine.hpp"
#include "trs/term_store.hpp"

namespace {

void run_on_big_stack(const std::function<void()>& fn) {
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, std::size_t(2) << 30);
    struct Box {
        const std::function<void()>* fn;
    } box{&fn};
    pthread_t th;
    auto tramp = [](void* p) -> void* {
        (*static_cast<Box*>(p)->fn)();
        return nullptr;
    };
    if (pthread_create(&th, &attr, tramp, &box) != 0) {
        fn();  // fall back to the caller's stack
    } else {
        pthread_join(th, nullptr);
    }
    pthread_attr_destroy(&attr);
}

std::vector<std::uint32_t> canonical_words(const trs::Term& root, std::uint32_t* n_nodes) {
    std::unordered_map<const trs::TermNode*, std::uint32_t> ids;
    std::vector<const trs::TermNode*> order;
    std::vector<const trs::TermNode*> stack{root.get()};
    while (!stack.empty()) {
        const trs::TermNode* node = stack.back();
        stack.pop_back();
        if (ids.count(node)) continue;
        ids.emplace(node, static_cast<std::uint32_t>(order.size()));
        order.push_back(node);
        const auto& ch = node->children();
        for (auto it = ch.rbegin(); it != ch.rend(); ++it) stack.push_back(it->get());
    }
    std::vector<std::uint32_t> words;
    for (const trs::TermNode* node : order) {
        words.push_back(node->symbol());
        for (const trs::Term& c : node->children()) words.push_back(ids.at(c.get()));
    }
    *n_nodes = static_cast<std::uint32_t>(order.size());
    return words;
}

}  // namespace

extern "C" {

struct ref_result {
    int status;  // 0 ok, 1 step budget, 2 capacity, 3 dangling, 4 invalid input, 6 other
    char message[512];
    std::uint64_t rewrites;
    std::uint32_t sweeps;
    std::uint64_t micros;  // engine time only (bench.cpp:56-61: excludes parse/load/extract)
    std::uint64_t max_width;
    std::uint64_t median_width;
    std::uint64_t* widths;  // per-sweep rewrites (sweep engine only)
    std::uint32_t* live;    // per-sweep live_terms (sweep engine only)
    std::uint32_t n_widths;
    std::uint32_t* words;   // canonical DAG words of the normal form
    std::uint64_t n_words;
    std::uint32_t n_nodes;
    std::uint32_t num_symbols;
    std::uint64_t peak_depth;  // seq engine only
};

static void set_error(ref_result* out, int status, const char* msg) {
    out->status = status;
    std::snprintf(out->message, sizeof(out->message), "%s", msg);
}

static int fault_status(trs::EngineFault f) {
    switch (f) {
        case trs::EngineFault::StepBudget: return 1;
        case trs::EngineFault::Capacity: return 2;
        case trs::EngineFault::DanglingReference: return 3;
    }
    return 6;
}

// engine: "seq" or "sweep".  workers/chunk/capacity/fixed_capacity mirror
// SweepOptions (sweep_engine.hpp:29-36) and EngineConfig (bench.hpp:19-23).
int ref_run(const char* text, const char* engine, unsigned workers, unsigned chunk,
            std::uint32_t capacity, int fixed_capacity, std::uint64_t step_budget, int want_words,
            ref_result* out) {
    std::memset(out, 0, sizeof(*out));
    std::string eng(engine);
    std::string input(text);
    run_on_big_stack([&] {
        try {
            trs::ResolveResult rr = trs::load_system(input);
            if (!rr.system) {
                std::string m = "resolve failed";
                for (const auto& e : rr.errors) m += "; " + trs::format_error("<text>", e);
                set_error(out, 4, m.c_str());
                return;
            }
            const trs::RewriteSystem& sys = *rr.system;
            out->num_symbols = static_cast<std::uint32_t>(sys.signature.symbols.size());
            trs::DispatchTable table = trs::compile(sys);
            trs::Term nf;
            if (eng == "seq") {
                trs::SeqOptions so;
                so.step_budget = step_budget;
                trs::SeqResult r = trs::normalize(sys, table, sys.input_term, so);
                out->rewrites = r.stats.rewritten_terms;
                out->micros = r.stats.micros;
                out->peak_depth = r.stats.peak_depth;
                nf = r.normal_form;
            } else if (eng == "sweep") {
                trs::SweepOptions so;
                so.workers = workers;
                so.chunk_size = chunk ? chunk : 256;
                so.step_budget = step_budget;
                so.fixed_capacity = fixed_capacity != 0;
                trs::TermStore store = trs::load(sys, sys.input_term, capacity);
                auto t0 = std::chrono::steady_clock::now();
                trs::SweepTrace trace = trs::run(store, table, so);
                auto t1 = std::chrono::steady_clock::now();
                out->micros = static_cast<std::uint64_t>(
                    std::chrono::duration_cast<std::chrono::microseconds>(t1 - t0).count());
                out->rewrites = trace.total_rewrites();
                out->sweeps = static_cast<std::uint32_t>(trace.records.size());
                out->max_width = trace.max_width();
                out->median_width = trace.median_width();
                out->n_widths = out->sweeps;
                out->widths = static_cast<std::uint64_t*>(
                    std::malloc(sizeof(std::uint64_t) * std::max<std::size_t>(1, out->sweeps)));
                out->live = static_cast<std::uint32_t*>(
                    std::malloc(sizeof(std::uint32_t) * std::max<std::size_t>(1, out->sweeps)));
                for (std::uint32_t k = 0; k < out->sweeps; ++k) {
                    out->widths[k] = trace.records[k].rewrites;
                    out->live[k] = trace.records[k].live_terms;
                }
                if (want_words) nf = trs::extract(store);
            } else {
                set_error(out, 4, "unknown engine");
                return;
            }
            if (want_words && nf) {
                std::vector<std::uint32_t> w = canonical_words(nf, &out->n_nodes);
                out->n_words = w.size();
                out->words = static_cast<std::uint32_t*>(
                    std::malloc(sizeof(std::uint32_t) * std::max<std::size_t>(1, w.size())));
                std::memcpy(out->words, w.data(), sizeof(std::uint32_t) * w.size());
            }
        } catch (const trs::EngineError& e) {
            set_error(out, fault_status(e.fault), e.what());
        } catch (const std::exception& e) {
            set_error(out, 6, e.what());
        }
    });
    return out->status;
}

void ref_result_free(ref_result* r) {
    std::free(r->widths);
    std::free(r->live);
    std::free(r->words);
    r->widths = nullptr;
    r->live = nullptr;
    r->words = nullptr;
}

// Several independent inputs at once, one big-stack thread each: the
// "nproc concurrent seq processes" CPU baseline of BASELINE.md §2 for the
// batched config.  Parse/compile happen before a barrier; the timed region is
// the engine calls only (bench.cpp:56-61).  Returns the wall seconds of the
// timed region; per-input rewrites land in rewrites_out.
double ref_run_many(const char** texts, int k, const char* engine, unsigned workers,
                    std::uint64_t* rewrites_out, int* status_out) {
    std::string eng(engine);
    std::barrier sync(k + 1);
    std::vector<std::thread> pool;
    std::atomic<std::int64_t> end_ns{0};
    std::vector<std::function<void()>> jobs(k);
    for (int i = 0; i < k; ++i) {
        jobs[i] = [&, i] {
            std::unique_ptr<trs::RewriteSystem> sys;
            std::unique_ptr<trs::DispatchTable> table;
            std::unique_ptr<trs::TermStore> store;
            trs::ResolveResult rr = trs::load_system(texts[i]);
            if (rr.system) {
                sys = std::make_unique<trs::RewriteSystem>(std::move(*rr.system));
                table = std::make_unique<trs::DispatchTable>(trs::compile(*sys));
                if (eng == "sweep") store = std::make_unique<trs::TermStore>(trs::load(*sys, sys->input_term));
            }
            sync.arrive_and_wait();
            status_out[i] = 0;
            rewrites_out[i] = 0;
            if (!sys) {
                status_out[i] = 4;
            } else {
                try {
                    if (eng == "seq") {
                        trs::SeqResult r = trs::normalize(*sys, *table, sys->input_term);
                        rewrites_out[i] = r.stats.rewritten_terms;
                    } else {
                        trs::SweepOptions so;
                        so.workers = workers;
                        rewrites_out[i] = trs::run(*store, *table, so).total_rewrites();
                    }
                } catch (const trs::EngineError& e) {
                    status_out[i] = fault_status(e.fault);
                }
            }
            std::int64_t now = std::chrono::duration_cast<std::chrono::nanoseconds>(
                                   std::chrono::steady_clock::now().time_since_epoch())
                                   .count();
            std::int64_t prev = end_ns.load();
            while (prev < now && !end_ns.compare_exchange_weak(prev, now)) {
            }
            sync.arrive_and_wait();
        };
    }
    std::vector<pthread_t> threads(k);
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, std::size_t(2) << 30);
    for (int i = 0; i < k; ++i) {
        pthread_create(
            &threads[i], &attr,
            [](void* p) -> void* {
                (*static_cast<std::function<void()>*>(p))();
                return nullptr;
            },
            &jobs[i]);
    }
    sync.arrive_and_wait();  // everyone parsed
    std::int64_t start = std::chrono::duration_cast<std::chrono::nanoseconds>(
                             std::chrono::steady_clock::now().time_since_epoch())
                             .count();
    sync.arrive_and_wait();  // everyone done
    for (int i = 0; i < k; ++i) pthread_join(threads[i], nullptr);
    pthread_attr_destroy(&attr);
    return static_cast<double>(end_ns.load() - start) * 1e-9;
}

// Reference dump-dispatch text (dispatch.cpp:98-134); malloc'd, NULL on a
// resolve failure.
char* ref_dump_dispatch(const char* text) {
    char* result = nullptr;
    std::string input(text);
    run_on_big_stack([&] {
        trs::ResolveResult rr = trs::load_system(input);
        if (!rr.system) return;
        std::string d = trs::dump_dispatch(*rr.system, trs::compile(*rr.system));
        result = static_cast<char*>(std::malloc(d.size() + 1));
        std::memcpy(result, d.c_str(), d.size() + 1);
    });
    return result;
}

// Reference generator text (generators.cpp:146-174).  family: 0 mergesort,
// 1 treemergesort, 2 transform.
char* ref_generate(int family, std::uint32_t length, std::uint32_t depth, std::uint64_t seed) {
    trs::GenSpec spec = family == 0   ? trs::GenSpec::mergesort(length, seed)
                        : family == 1 ? trs::GenSpec::treemergesort(depth, length, seed)
                                      : trs::GenSpec::transform(depth);
    std::string t = trs::generate(spec);
    char* out = static_cast<char*>(std::malloc(t.size() + 1));
    std::memcpy(out, t.c_str(), t.size() + 1);
    return out;
}

// Resolve diagnostics as "line:col: kind: message" lines; empty when the
// text resolves.  malloc'd.
char* ref_diagnostics(const char* text) {
    std::string out;
    std::string input(text);
    run_on_big_stack([&] {
        trs::ResolveResult rr = trs::load_system(input);
        for (const auto& e : rr.errors) out += trs::format_error("<text>", e) + "\n";
    });
    char* r = static_cast<char*>(std::malloc(out.size() + 1));
    std::memcpy(r, out.c_str(), out.size() + 1);
    return r;
}

void ref_free(void* p) { std::free(p); }

}  // extern "C"

// Integration check: the UNMODIFIED reference API end to end with the B200
// engine as its sweep engine (TEST INFRASTRUCTURE; built by
// integration/Makefile where /root/reference exists, then travels to the
// GPU box prebuilt).
//
//   load_system -> compile -> load -> trs::gpu::run (adapter) -> extract
//
// and, beside it, the reference's own seq engine (normalize) and sweep
// engine (run) on the same input.  Returns whether the normal forms are
// term_equal and the rewrite counts and per-sweep widths agree.
#include <pthread.h>

#include <cstdio>
#include <cstring>
#include <functional>
#include <string>

#include "trs/bench.hpp"
#include "trs/seq_engine.hpp"
#include "trs/sweep_engine.hpp"
#include "trs/term_store.hpp"
#include "trs_gpu_adapter.hpp"

namespace {

void on_big_stack(const std::function<void()>& fn) {
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, std::size_t(2) << 30);
    pthread_t th;
    auto tramp = [](void* p) -> void* {
        (*static_cast<const std::function<void()>*>(p))();
        return nullptr;
    };
    pthread_create(&th, &attr, tramp, const_cast<std::function<void()>*>(&fn));
    pthread_join(th, nullptr);
    pthread_attr_destroy(&attr);
}

}  // namespace

extern "C" {

struct ref_gpu_result {
    int status;            // 0 ok, 1 step budget, 2 capacity, 3 dangling, 4 invalid, 6 other
    char message[512];
    int term_equal_seq;    // extract(gpu store) term_equal seq normal form
    int rewrites_equal;    // gpu trace total == seq rewritten_terms == reference sweep total
    int widths_equal;      // gpu per-sweep widths == reference sweep engine's
    unsigned long long rewrites;
    unsigned sweeps;
};

int ref_gpu_normalize(const char* text, unsigned long long step_budget, ref_gpu_result* out) {
    std::memset(out, 0, sizeof(*out));
    std::string input(text);
    on_big_stack([&] {
        try {
            trs::ResolveResult rr = trs::load_system(input);
            if (!rr.system) {
                out->status = 4;
                std::snprintf(out->message, sizeof(out->message), "resolve failed");
                return;
            }
            const trs::RewriteSystem& sys = *rr.system;
            trs::DispatchTable table = trs::compile(sys);
            if (step_budget) {
                // error path only: the B200 engine must raise the reference's EngineError
                trs::TermStore store = trs::load(sys, sys.input_term);
                trs::gpu::GpuOptions go;
                go.sweep.step_budget = step_budget;
                trs::gpu::run(store, table, go);
                return;
            }
            trs::SeqResult seq = trs::normalize(sys, table, sys.input_term);
            trs::TermStore ref_store = trs::load(sys, sys.input_term);
            trs::SweepOptions so;
            so.workers = 1;
            trs::SweepTrace ref_trace = trs::run(ref_store, table, so);

            trs::TermStore store = trs::load(sys, sys.input_term);  // the reference's own load
            trs::gpu::GpuOptions go;
            if (step_budget) go.sweep.step_budget = step_budget;
            trs::SweepTrace trace = trs::gpu::run(store, table, go);  // the drop-in
            trs::Term nf = trs::extract(store);                        // the reference's own extract
            out->term_equal_seq = trs::term_equal(nf, seq.normal_form);
            out->rewrites = trace.total_rewrites();
            out->sweeps = static_cast<unsigned>(trace.records.size());
            out->rewrites_equal = trace.total_rewrites() == seq.stats.rewritten_terms &&
                                  trace.total_rewrites() == ref_trace.total_rewrites();
            bool w = trace.records.size() == ref_trace.records.size();
            for (std::size_t k = 0; w && k < trace.records.size(); ++k)
                w = trace.records[k].rewrites == ref_trace.records[k].rewrites;
            out->widths_equal = w;
        } catch (const trs::EngineError& e) {
            out->status = e.fault == trs::EngineFault::StepBudget ? 1 : e.fault == trs::EngineFault::Capacity ? 2 : 3;
            std::snprintf(out->message, sizeof(out->message), "%s", e.what());
        } catch (const std::exception& e) {
            out->status = 6;
            std::snprintf(out->message, sizeof(out->message), "%s", e.what());
        }
    });
    return out->status;
}

}  // extern "C"

// trs_bench_gpu: the reference's OWN commands (cmd_bench, cmd_normalize,
// proj/src/bench.cpp:75-185) with a "gpu" engine next to "seq" and "sweep".
//
// Nothing of the reference is copied or modified.  Its library is the
// unmodified oracle/_ref/libtrs_ref.so, whose cmd_bench / cmd_normalize call
// run_engine (bench.cpp:45-73) through the PLT; this executable exports its
// own trs::run_engine, which the dynamic linker binds those calls to:
//   engine "gpu"  -> load -> trs::gpu::run (integration/trs_gpu_adapter.hpp,
//                    the B200 engine through include/trs_gpu.h) -> extract,
//                    timed like the sweep branch (bench.cpp:56-61);
//   anything else -> the reference's run_engine (dlsym RTLD_NEXT).
// So cmd_bench's divergence check (bench.cpp:147-159: normal form and rewrite
// count of every engine and repetition against the first) runs the GPU
// against the reference's seq and sweep engines in one process.
//
//   trs_bench_gpu bench FILE --engines seq,sweep,gpu [--reps N] [--csv PATH]
//   trs_bench_gpu normalize FILE [--engine gpu] [--trace PATH]
//   trs_bench_gpu dump-dispatch FILE [--device]
//
// `normalize --trace` writes the gpu run's trace with the reference's own
// write_trace_csv (sweep_engine.cpp:432-437) -- cmd_normalize itself writes
// traces for "sweep" only.  `dump-dispatch --device` renders the program the
// engine staged on the device (trs_gpu_dump_program) next to the reference's
// dump (dispatch.cpp:98-134); the two must be identical.
#include <dlfcn.h>
#include <pthread.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "trs/bench.hpp"
#include "trs/dispatch.hpp"
#include "trs/sweep_engine.hpp"
#include "trs/term_store.hpp"
#include "trs_gpu_adapter.hpp"

namespace trs {

using RunEngineFn = EngineRun (*)(const RewriteSystem&, const DispatchTable&, const std::string&,
                                  const EngineConfig&);

// Interposes the reference's run_engine for every caller in libtrs_ref.so.
EngineRun run_engine(const RewriteSystem& system, const DispatchTable& table, const std::string& engine,
                     const EngineConfig& config) {
    if (engine != "gpu") {
        static RunEngineFn next = reinterpret_cast<RunEngineFn>(dlsym(
            RTLD_NEXT,
            "_ZN3trs10run_engineERKNS_13RewriteSystemERKNS_13DispatchTableERKNSt7__cxx1112basic_stringIcSt11char_"
            "traitsIcESaIcEEERKNS_12EngineConfigE"));
        if (!next) throw std::runtime_error("reference run_engine not found");
        return next(system, table, engine, config);
    }
    EngineRun r;
    r.report.engine = engine;
    TermStore store = load(system, system.input_term, config.capacity);  // the reference's load
    gpu::GpuOptions go;
    go.sweep = config.sweep;
    const auto t0 = std::chrono::steady_clock::now();
    r.trace = gpu::run(store, table, go);
    r.report.micros = static_cast<std::uint64_t>(
        std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count());
    r.normal_form = extract(store);  // the reference's extract of the written-back store
    r.report.total_rewrites = r.trace.total_rewrites();
    r.report.sweep_count = static_cast<std::uint32_t>(r.trace.records.size());
    r.report.max_sweep_width = r.trace.max_width();
    r.report.median_sweep_width = r.trace.median_width();
    r.report.terms_per_second =
        r.report.micros ? r.report.total_rewrites * 1e6 / static_cast<double>(r.report.micros) : 0.0;
    return r;
}

}  // namespace trs

namespace {

int on_big_stack(const std::function<int()>& fn) {
    // the reference's resolver and Term teardown recurse per nesting level
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, std::size_t(2) << 30);
    struct Box {
        const std::function<int()>* fn;
        int rc;
    } box{&fn, 0};
    pthread_t th;
    pthread_create(
        &th, &attr,
        [](void* p) -> void* {
            auto* b = static_cast<Box*>(p);
            b->rc = (*b->fn)();
            return nullptr;
        },
        &box);
    pthread_join(th, nullptr);
    pthread_attr_destroy(&attr);
    return box.rc;
}

std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(item);
    return out;
}

int usage() {
    std::cerr << "usage: trs_bench_gpu bench FILE --engines seq,sweep,gpu [--reps N] [--csv PATH]\n"
                 "       trs_bench_gpu normalize FILE [--engine gpu] [--trace PATH]\n"
                 "       trs_bench_gpu dump-dispatch FILE [--device]\n";
    return trs::kExitInputError;
}

int dump_device(const std::string& path) {
    std::ifstream in(path);
    std::stringstream text;
    text << in.rdbuf();
    trs::ResolveResult rr = trs::load_system(text.str());
    if (!rr.system) return trs::kExitInputError;
    const trs::RewriteSystem& sys = *rr.system;
    const trs::DispatchTable table = trs::compile(sys);
    trs_gpu_engine* e = nullptr;
    trs::gpu::detail::check(trs_gpu_open(0, &e), nullptr);
    trs::TermStore store = trs::load(sys, sys.input_term);
    trs::gpu::detail::Flat f = trs::gpu::detail::flatten(store, table);
    trs_gpu_program p = trs::gpu::detail::program_of(f);
    trs::gpu::detail::check(trs_gpu_set_program(e, &p), e);
    // names from the reference's signature, rule texts from its printer
    std::vector<std::string> syms, vars, texts;
    for (const auto& s : sys.signature.symbols) syms.push_back(s.name);
    for (const auto& v : sys.signature.variables) vars.push_back(v.name);
    for (const auto& r : sys.rules)
        texts.push_back(trs::print_term(sys.signature, r.lhs) + " = " + trs::print_term(sys.signature, r.rhs));
    std::vector<const char*> sp, vp, tp;
    for (auto& x : syms) sp.push_back(x.c_str());
    for (auto& x : vars) vp.push_back(x.c_str());
    for (auto& x : texts) tp.push_back(x.c_str());
    // device rule r's variable slot k -> signature variable (the program's slot_vars)
    std::vector<uint32_t> begin{0}, slot_var;
    for (const auto& rules : table.by_symbol)
        for (const auto& c : rules) {
            for (auto v : c.program.slot_vars) slot_var.push_back(v);
            begin.push_back(static_cast<uint32_t>(slot_var.size()));
        }
    uint64_t need = 0;
    trs::gpu::detail::check(
        trs_gpu_dump_program(e, sp.data(), vp.data(), begin.data(), slot_var.data(), tp.data(), nullptr, 0, &need), e);
    std::string out(need, '\0');
    trs::gpu::detail::check(
        trs_gpu_dump_program(e, sp.data(), vp.data(), begin.data(), slot_var.data(), tp.data(), out.data(), need, &need),
        e);
    std::cout << out.c_str();
    trs_gpu_close(e);
    return trs::kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) return usage();
    const std::string cmd = argv[1], file = argv[2];
    std::vector<std::string> engines{"seq", "sweep", "gpu"};
    std::string engine = "gpu", csv, trace;
    unsigned reps = 1;
    bool device = false;
    for (int i = 3; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string { return i + 1 < argc ? argv[++i] : ""; };
        if (a == "--engines") engines = split(val());
        else if (a == "--engine") engine = val();
        else if (a == "--reps") reps = static_cast<unsigned>(std::stoul(val()));
        else if (a == "--csv") csv = val();
        else if (a == "--trace") trace = val();
        else if (a == "--device") device = true;
        else return usage();
    }
    trs::EngineConfig cfg;  // the reference CLI's defaults (trs_cli.cpp:9-30)
    cfg.sweep.step_budget = 1'000'000'000;
    cfg.seq.step_budget = 1'000'000'000;
    return on_big_stack([&]() -> int {
        if (cmd == "bench") return trs::cmd_bench(file, engines, reps, cfg, csv, std::cout, std::cerr);
        if (cmd == "normalize") {
            const int rc = trs::cmd_normalize(file, engine, cfg, engine == "sweep" ? trace : "", std::cout, std::cerr);
            if (rc == trs::kExitOk && !trace.empty() && engine == "gpu") {
                // the gpu run's trace through the reference's own CSV writer
                std::ifstream in(file);
                std::stringstream text;
                text << in.rdbuf();
                trs::ResolveResult rr = trs::load_system(text.str());
                const trs::DispatchTable table = trs::compile(*rr.system);
                trs::EngineRun r = trs::run_engine(*rr.system, table, "gpu", cfg);
                std::ofstream out(trace);
                trs::write_trace_csv(out, r.trace);
            }
            return rc;
        }
        if (cmd == "dump-dispatch") return device ? dump_device(file) : trs::cmd_dump_dispatch(file, std::cout, std::cerr);
        return usage();
    });
}

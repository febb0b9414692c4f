// Per-program specialisation of the step loop (host side).
//
// The paper generated one `rewrite_f` device function per symbol from each
// TRS and compiled it with nvcc.  Here the same idea
// runs at set_program: from the flattened program (the DispatchTable of
// dispatch.hpp:73-78 as the blob of device_program.hpp) this emits
//   gen_bind   -- the chosen rule's variable bindings as register moves
//                 (constant indices into the matcher's register arrays),
//   gen_csrc   -- a collapsing rule's source variable,
//   gen_build  -- a constructive rule's right-hand side as straight-line
//                 record stores and reference additions,
// and NVRTC compiles them into the step loop (sweep.cuh with TRS_GEN = 1).
// Everything else -- rule choice by match tables, claims, waiters, pushes,
// collections -- is the same code as the interpreted kernel, so the two are
// interchangeable launch by launch.
#pragma once

#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "device_program.hpp"

namespace trs_b200_jit {
extern const int kNumHeaders;
extern const char* const kHeaderNames[];
extern const char* const kHeaderSources[];
}  // namespace trs_b200_jit

namespace trs_b200 {

struct BlobView {
    const ProgHeader* h;
    const uint8_t* arity;
    const uint16_t* rule_begin;
    const DRule* rules;
    const DStep* steps;
    const DInstr* instrs;
    const uint16_t* refs;
    const DPlan* plans;
    explicit BlobView(const uint8_t* blob) {
        h = reinterpret_cast<const ProgHeader*>(blob);
        arity = blob + h->off_arity;
        rule_begin = reinterpret_cast<const uint16_t*>(blob + h->off_rule_begin);
        rules = reinterpret_cast<const DRule*>(blob + h->off_rules);
        steps = reinterpret_cast<const DStep*>(blob + h->off_steps);
        instrs = reinterpret_cast<const DInstr*>(blob + h->off_instrs);
        refs = reinterpret_cast<const uint16_t*>(blob + h->off_refs);
        plans = reinterpret_cast<const DPlan*>(blob + h->off_plans);
    }
};

inline std::string jit_src_expr(uint8_t src) {
    char b[32];
    if (src < kSrcSlot)
        std::snprintf(b, sizeof b, "a[%u]", (unsigned)src);
    else if (src < kSrcSArg)
        std::snprintf(b, sizeof b, "ca[%u]", (unsigned)(src & 15u));
    else
        std::snprintf(b, sizeof b, "ga[%u]", (unsigned)(src & 7u));
    return b;
}

// CUDA source of the specialised step loop for record width W.
inline std::string jit_source(const uint8_t* blob, int W, uint32_t max_vars) {
    const BlobView B(blob);
    const uint32_t nsym = B.h->num_symbols;
    const int MAXA = rec_args(W);
    std::string bind, csrc, build, choose;
    char line[256];
    for (uint32_t f = 0; f < nsym; ++f) {
        // rule choice of a table-planned symbol: its rules' head checks in
        // source order (dispatch.hpp:119-130), registers against constants
        if (B.plans[f].fast & kPlanTables) {
            std::string body = "        case " + std::to_string(f) + ":\n";
            for (uint32_t r = B.rule_begin[f]; r < B.rule_begin[f + 1]; ++r) {
                const DRule& R = B.rules[r];
                std::string cond;
                for (uint32_t t = 0; t < R.num_steps; ++t) {
                    const DStep& d = B.steps[R.first_step + t];
                    if (d.kind != 0) continue;
                    const std::string v = d.src < kSrcSlot ? "ch[" + std::to_string(d.src) + "]"
                                                           : "gh[" + std::to_string(d.src - kSrcSlot) + "]";
                    cond += (cond.empty() ? "" : " && ") + v + " == " + std::to_string(d.value) + "u";
                }
                if (cond.empty()) {
                    body += "            return " + std::to_string(r) + ";\n";
                    break;  // later rules are unreachable
                }
                body += "            if (" + cond + ") return " + std::to_string(r) + ";\n";
            }
            body += "            return -1;\n";
            choose += body;
        }
        for (uint32_t r = B.rule_begin[f]; r < B.rule_begin[f + 1]; ++r) {
            const DRule& R = B.rules[r];
            if (B.plans[f].fast & kPlanTables) {
                std::string body;
                for (uint32_t t = 0; t < R.num_steps; ++t) {
                    const DStep& d = B.steps[R.first_step + t];
                    if (d.kind == 0) continue;
                    std::snprintf(line, sizeof line, " gb[%u] = %s;", d.value, jit_src_expr(d.src).c_str());
                    body += line;
                }
                if (R.collapse && R.csrc != kNone) {
                    // the collapse source's record, already in registers
                    const unsigned cs = R.csrc;
                    if (cs < kSrcSlot) {
                        std::snprintf(line, sizeof line, " cs_head = ch[%u];", cs);
                        body += line;
                        for (int k = 0; k < 4; ++k) {
                            std::snprintf(line, sizeof line, " cs_b[%d] = ca[%u];", k, (cs & 3u) * 4 + k);
                            body += line;
                        }
                    } else {
                        std::snprintf(line, sizeof line, " cs_head = gh[%u];", cs & 3u);
                        body += line;
                        for (int k = 0; k < 4; ++k) {
                            std::snprintf(line, sizeof line, " cs_b[%d] = ga[%u];", k, (cs & 1u) * 4 + k);
                            body += line;
                        }
                    }
                }
                if (!body.empty()) bind += "        case " + std::to_string(r) + ":" + body + " break;\n";
            }
            if (R.collapse) {
                std::snprintf(line, sizeof line, "        case %u: return gb[%u];\n", r, (unsigned)R.root_ref);
                csrc += line;
                continue;
            }
            // constructive: fresh nodes 0..new_slots-1, then the root in place
            std::string body;
            std::vector<uint32_t> var_refs;
            for (uint32_t k = 0; k <= R.new_slots; ++k) {
                const DInstr& I = B.instrs[R.first_instr + k];
                const uint32_t iar = B.arity[I.symbol];
                std::vector<std::string> args(MAXA, "0u");
                for (uint32_t j = 0; j < iar; ++j) {
                    const uint16_t ref = B.refs[I.first_ref + j];
                    if (ref & kRefNode) {
                        args[j] = "fresh + " + std::to_string(ref & 0x7fff) + "u";
                    } else {
                        args[j] = "gb[" + std::to_string(ref) + "]";
                        var_refs.push_back(ref);
                    }
                }
                if (k < R.new_slots) {
                    std::string sub = I.subscriber == kNone ? "0u"
                                      : I.subscriber == kRootSub ? "i"
                                                                 : "fresh + " + std::to_string(I.subscriber) + "u";
                    std::snprintf(line, sizeof line,
                                  "            { uint32_t* F = rec<W>(arena, fresh + %uu);\n"
                                  "              *reinterpret_cast<uint4*>(F) = make_uint4(%uu, tnext, %uu, %s);\n",
                                  k, I.symbol | ((uint32_t)I.cursor << kSymBits), (unsigned)I.indegree, sub.c_str());
                    body += line;
                    // the first argument quad always (zeros past the arity: sweep.cuh's build)
                    for (uint32_t q = 0; q == 0 || q * 4 < iar; ++q)
                        body += "              *reinterpret_cast<uint4*>(F + kWArgs + " + std::to_string(q * 4) +
                                ") = make_uint4(" + args[q * 4] + ", " + args[q * 4 + 1] + ", " + args[q * 4 + 2] +
                                ", " + args[q * 4 + 3] + ");\n";
                    body += "            }\n";
                } else {
                    std::snprintf(line, sizeof line,
                                  "            { uint32_t* R = rec<W>(arena, i);\n"
                                  "              *reinterpret_cast<uint2*>(R) = make_uint2(%uu, tnext);\n"
                                  "              const uint32_t b[%d] = {",
                                  I.symbol | ((uint32_t)R.root_cursor << kSymBits), MAXA);
                    body += line;
                    for (int j = 0; j < MAXA; ++j) body += (j ? ", " : "") + args[j];
                    body += "};\n              store_args<W>(R, b, ar > " + std::to_string(iar) + "u ? ar : " +
                            std::to_string(iar) + "u);\n            }\n";
                }
            }
            // every reuse of a bound variable adds one reference (sweep_engine.cpp:251-253)
            for (uint32_t v : var_refs)
                body += "            if (rc) rc_upd<S>(rec<W>(arena, gb[" + std::to_string(v) + "]) + kWRc, 1);\n";
            build += "        case " + std::to_string(r) + ": {\n" + body + "            break;\n        }\n";
        }
    }
    std::string src;
    bool all_tables = true;  // every symbol with rules chooses by tables: the rule walks compile out
    for (uint32_t f = 0; f < nsym; ++f)
        if (B.rule_begin[f + 1] > B.rule_begin[f] && !(B.plans[f].fast & kPlanTables)) all_tables = false;
    src += "#define TRS_GEN 1\n#define TRS_GEN_MAXV " + std::to_string(max_vars) + "\n#define TRS_GEN_MAXA " +
           std::to_string(B.h->max_arity ? B.h->max_arity : 1) + "\n#define TRS_GEN_ALL_TABLES " +
           (all_tables ? "1" : "0") + "\n";
    src += "#include \"device_common.cuh\"\nnamespace trs_b200 {\n";
    src += "template <int W>\n__device__ __forceinline__ void gen_bind(uint32_t rule, const uint32_t (&a)[rec_args(W)],\n"
           "    const uint32_t (&ch)[rec_args(W)], const uint32_t (&ca)[kPlanChildren * 4],\n"
           "    const uint32_t (&gh)[kPlanSlots], const uint32_t (&ga)[kPlanArgSlots * 4],\n"
           "    uint32_t (&gb)[TRS_GEN_MAXV], uint32_t& cs_head, uint32_t (&cs_b)[4]) {\n    switch (rule) {\n" +
           bind + "        default: break;\n    }\n}\n";
    src += "template <int N>\n__device__ __forceinline__ int gen_choose(uint32_t sym, const uint32_t (&ch)[N],\n"
           "    const uint32_t (&gh)[kPlanSlots]) {\n    switch (sym) {\n" +
           choose + "        default: return -1;\n    }\n}\n";
    src += "__device__ __forceinline__ uint32_t gen_csrc(uint32_t rule, const uint32_t (&gb)[TRS_GEN_MAXV]) {\n"
           "    switch (rule) {\n" +
           csrc + "        default: return 0u;\n    }\n}\n";
    src += "template <int W, bool S>\n__device__ __forceinline__ void gen_build(uint32_t rule, uint32_t* arena, uint32_t fresh,\n"
           "    uint32_t i, uint32_t ar, const uint32_t (&gb)[TRS_GEN_MAXV], uint32_t tnext, bool rc) {\n"
           "    switch (rule) {\n" +
           build + "        default: break;\n    }\n}\n}  // namespace trs_b200\n#include \"sweep.cuh\"\n";
    return src;
}

struct JitResult {
    const void* kernel = nullptr;     // step_loop<W, MINB, false>: the lean synchronous build
    const void* kernel_ra = nullptr;  // step_loop<W, MINB, true>: the run-ahead build
    std::string log;
    double seconds = 0;
};

// Compile (or fetch from the process-wide cache) the specialised step loop.
inline JitResult jit_compile(const std::string& src, int W, int minb = 1) {
    static std::mutex mu;
    static std::unordered_map<std::string, std::pair<const void*, const void*>> cache;
    // compile-time knobs for A/B experiments (e.g. "-DTRS_B200_RA_PREFETCH=0"), space separated
    const char* defs_env = std::getenv("TRS_B200_JIT_DEFINES");
    const std::string defs = defs_env ? defs_env : "";
    const std::string key =
        std::to_string(W) + "/" + std::to_string(minb) + (TRS_B200_PROFILE ? "p" : "") + defs + "\n" + src;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return JitResult{it->second.first, it->second.second, "", 0};
    }
    JitResult out;
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "trs_gen.cu", trs_b200_jit::kNumHeaders, trs_b200_jit::kHeaderSources,
                           trs_b200_jit::kHeaderNames) != NVRTC_SUCCESS) {
        out.log = "nvrtcCreateProgram failed";
        return out;
    }
    const std::string name = "trs_b200::step_loop<" + std::to_string(W) + ", " + std::to_string(minb) + ", false>";
    const std::string name_ra = "trs_b200::step_loop<" + std::to_string(W) + ", " + std::to_string(minb) + ", true>";
    nvrtcAddNameExpression(prog, name.c_str());
    nvrtcAddNameExpression(prog, name_ra.c_str());
    // the specialisation is built like the library that loads it (profiling build or not)
    const char* verbose = std::getenv("TRS_B200_JIT_VERBOSE");  // ptxas register/spill report in the log
    std::vector<std::string> extra;
    for (size_t a = 0; a < defs.size();) {
        const size_t b = defs.find(' ', a);
        const std::string t = defs.substr(a, b == std::string::npos ? std::string::npos : b - a);
        if (!t.empty()) extra.push_back(t);
        if (b == std::string::npos) break;
        a = b + 1;
    }
    std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                                     TRS_B200_PROFILE ? "-DTRS_B200_PROFILE=1" : "-DTRS_B200_PROFILE=0"};
    for (const std::string& t : extra) opts.push_back(t.c_str());
    if (verbose && verbose[0] == '1') opts.push_back("--ptxas-options=-v");
    const nvrtcResult rc = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    out.log.resize(n);
    if (n) nvrtcGetProgramLog(prog, &out.log[0]);
    if (rc != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return out;
    }
    const char* lowered = nullptr;
    nvrtcGetLoweredName(prog, name.c_str(), &lowered);
    const std::string lname = lowered ? lowered : "";
    lowered = nullptr;
    nvrtcGetLoweredName(prog, name_ra.c_str(), &lowered);
    const std::string lname_ra = lowered ? lowered : "";
    size_t cb = 0;
    nvrtcGetCUBINSize(prog, &cb);
    std::vector<char> cubin(cb);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    cudaLibrary_t lib = nullptr;
    if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
        out.log += "\ncudaLibraryLoadData failed";
        cudaGetLastError();
        return out;
    }
    cudaKernel_t k = nullptr, kra = nullptr;
    if (cudaLibraryGetKernel(&k, lib, lname.c_str()) != cudaSuccess ||
        cudaLibraryGetKernel(&kra, lib, lname_ra.c_str()) != cudaSuccess) {
        out.log += "\ncudaLibraryGetKernel failed for " + lname + " / " + lname_ra;
        cudaGetLastError();
        return out;
    }
    out.kernel = reinterpret_cast<const void*>(k);
    out.kernel_ra = reinterpret_cast<const void*>(kra);
    std::lock_guard<std::mutex> g(mu);
    cache[key] = {out.kernel, out.kernel_ra};
    return out;
}

}  // namespace trs_b200

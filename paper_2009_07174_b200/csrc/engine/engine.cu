// B200 term-rewriting engine: device step loop, allocator, GC, C ABI.
//
// Replaces the reference's host worker-pool sweep engine
// (proj/src/sweep_engine.cpp) and the device-facing half of its term store
// (proj/src/term_store.cpp) with sm_100a kernels.  Semantics follow
// one inner-most rewrite per eligible slot per sweep, first
// matching rule in source order, eligibility judged on the state at the
// start of the sweep, identical per-sweep widths.
//
// Design (DESIGN.md has the long form):
//  * Store: AoS records of W = 8/16/32 u32 words per slot in HBM
//    (head|cursor, nf epoch, refcount, waiter, args...).  One 32-byte
//    sector holds everything a random visit of an arity<=4 node needs, so a
//    child probe yields head + nf + args in one gather.
//  * Snapshot without copies: nf is an epoch; nf_read(c) at sweep s is
//    0 < epoch(c) < s (sweep_engine.cpp:80-81 become free).
//  * Frontier list instead of a full-store scan: only awake non-nf slots are
//    visited.  A slot whose scan stops on a non-nf child c subscribes to c
//    (CAS on c's waiter word) and sleeps; when c becomes nf it wakes the
//    subscriber for the next sweep.  A slot that loses the CAS polls (stays
//    on the list), which is exactly the reference's re-check.  Widths are
//    unchanged because a sleeping slot is, by construction, ineligible
//    (sweep_engine.cpp:173-178).
//  * Allocator: bump pointer with a per-sweep rotating claim counter
//    (the reference's next_fresh fold, sweep_engine.cpp:94-102); claims are
//    aggregated per CTA iteration by a block scan, one atomic per CTA.
//  * GC: refcount-zero slots are claimed and their argument references
//    dropped (term_store.cpp:140-157), then the arena is stream-compacted
//    (block scans + a grid-wide block-sum prefix) into the twin arena with
//    an old->new index map applied to args, waiters, frontier and roots.
//  * Step loop: one cooperative persistent launch runs every sweep with a
//    software grid barrier; when the frontier is small, CTA 0 alone runs
//    sweeps with __syncthreads while the rest of the grid parks.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device_program.hpp"
#include "sweep.cuh"
#include "export.cuh"
#include "canon.cuh"
#include "jit.hpp"
#include "trs_gpu.h"

using namespace trs_b200;

namespace {

// ---------------------------------------------------------------------------
// load: SoA (reference TermStore layout) -> AoS records, then the sweep-1
// frontier.  Every input slot is non-nf (term_store.cpp:55-72); an inner
// slot's first sweep stops on its first child, so it subscribes to it right
// away; leaves (and slots that lose the subscription race on a shared
// child) start on the list.

template <int W>
__global__ void load_records(uint32_t* __restrict__ arena, uint32_t n, const uint32_t* __restrict__ hss,
                             const uint32_t* __restrict__ args, uint32_t max_arity,
                             const uint32_t* __restrict__ rc) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t w[W];
#pragma unroll
        for (int k = 0; k < W; ++k) w[k] = 0;
        if (i != 0) {
            w[kWHead] = hss[i];
            w[kWRc] = rc[i];
            for (uint32_t j = 0; j < max_arity && j < (uint32_t)rec_args(W); ++j)
                w[kWArgs + j] = args[(size_t)j * n + i];
        } else {
            w[kWEpoch] = 1;  // slot 0 is never a term; keep it inert
        }
        uint4* dst = reinterpret_cast<uint4*>(arena + (size_t)i * W);
#pragma unroll
        for (int q = 0; q < W / 4; ++q) dst[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
}

template <int W>
__global__ void load_frontier(uint32_t* __restrict__ arena, uint32_t n, const uint8_t* __restrict__ arity,
                              uint32_t* __restrict__ list, uint32_t* __restrict__ count, uint32_t rich) {
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        uint32_t i = base + threadIdx.x;
        bool push = false;
        if (i >= 1 && i < n) {
            uint32_t* R = arena + (size_t)i * W;
            if (R[kWRc] != 0) {
                uint32_t ar = arity[R[kWHead] & kSymMask];
                if (ar == 0) {
                    push = true;
                } else {
                    uint32_t c = R[kWArgs];
                    push = atomicCAS(arena + (size_t)c * W + kWWaiter, 0u, i) != 0u;
                }
            }
        }
        unsigned mask = __ballot_sync(0xffffffffu, push);
        if (mask) {
            uint32_t lane = threadIdx.x & 31;
            uint32_t off = 0;
            if (lane == 0) off = atomicAdd(count, __popc(mask));
            off = __shfl_sync(0xffffffffu, off, 0);
            if (push && !rich) list[off + __popc(mask & ((1u << lane) - 1))] = i;
            if (push && rich) {
                // rich entry with payload (sweep.cuh): slot, head, flag, args
                uint32_t* E = list + (size_t)(off + __popc(mask & ((1u << lane) - 1))) * W;
                const uint32_t* R = arena + (size_t)i * W;
                *reinterpret_cast<uint4*>(E) = make_uint4(i, R[kWHead], 1u, 0u);
#pragma unroll
                for (int q = 1; q < W / 4; ++q)
                    reinterpret_cast<uint4*>(E)[q] = reinterpret_cast<const uint4*>(R)[q];
            }
        }
    }
}

__global__ void init_ctl(Ctl* ctl, uint32_t* regions, const uint32_t* count, uint32_t n) {
    ctl->bump = n;
    ctl->peak_bump = n;
    ctl->status = kRunning;
    ctl->nregions[0] = 1;
    regions[0] = 0;                  // buffer 0, offset of region 0
    regions[kMaxGrid] = *count;      // buffer 0, count of region 0
}

// Random-gather roofline: uniformly random VEC-word accesses over a
// power-of-two array far larger than L2, indices streamed coalesced.  Each
// thread keeps kProbeILP independent gathers in flight (the engine's warp
// step issues its child probes together the same way), and addressing is a
// mask, so the probe is bound by the memory system, not by issue.
template <int VEC, int kProbeILP>
__global__ void __launch_bounds__(512) gather_probe_kernel(const uint32_t* __restrict__ data, uint64_t mask,
                                                           const uint32_t* __restrict__ idx, uint32_t n,
                                                           uint32_t* __restrict__ sink) {
    uint32_t acc = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride * kProbeILP) {
        uint32_t e[kProbeILP];
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) {
            const uint32_t kk = k + (uint32_t)u * stride;
            e[u] = kk < n ? __ldcs(idx + kk) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) {
            const uint64_t w = ((uint64_t)e[u] * VEC) & mask;
            if (VEC == 1) {
                acc += data[w];
            } else if (VEC == 2) {
                const uint2 v = *reinterpret_cast<const uint2*>(data + w);
                acc += v.x ^ v.y;
            } else if (VEC == 4) {
                const uint4 v = *reinterpret_cast<const uint4*>(data + w);
                acc += v.x ^ v.y ^ v.z ^ v.w;
            } else {
                const uint4 v = *reinterpret_cast<const uint4*>(data + w);
                const uint4 x = *reinterpret_cast<const uint4*>(data + w + 4);
                acc += v.x ^ v.y ^ v.z ^ v.w ^ x.x ^ x.y ^ x.z ^ x.w;
            }
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
}

// Start of a run (begin = 1) or of a relaunch within one (begin = 0): the
// host never reads the control block before launching, so a run costs one
// host synchronisation (the status read-back at the end).
__global__ void prep_launch(Ctl* c, uint32_t* claim_ctrs, uint32_t* region_flags, uint32_t begin) {
    if (threadIdx.x == 0) {
        if (begin) {
            // logical sweeps continue from the previous run's (epochs stay comparable)
            c->sweep0 = c->sweep;
            c->tmax = c->sweep;
            c->psweep = 0;
            c->total_rewrites = 0;
            c->max_width = 0;
            c->gc_runs = 0;
            c->small_sweeps = 0;
            c->gc_ns = 0;
            c->abort_capacity = 0;
            c->last_gc_sweep = 0;
            c->hist_need = 0;
            c->ra_narrow = 0;
            c->ra_on = 0;
            c->ra_used = 0;
            c->ra_mref = 0;
            c->ra_sref = 0;
            c->ra_go = 0;
            c->val_kind = 0;
            c->val_slot = 0;
        }
        c->status = kRunning;
        c->bar_arrive = 0;
    }
    if (threadIdx.x < 8) claim_ctrs[threadIdx.x] = 0;
    // the flags that ended the previous launch have been acted on
    for (uint32_t k = threadIdx.x; k < 2 * kMaxGrid; k += blockDim.x) region_flags[k] = 0;
}

// After every step-loop launch: the logical sweep count (the run ends at the
// first sweep after its last nf event, sweep_engine.cpp:147) and the widest
// logical sweep (SweepTrace::max_width, sweep_engine.cpp:407-426).
__global__ void finish_run(Ctl* c, const unsigned long long* __restrict__ hist, uint32_t hist_cap) {
    const uint32_t t = max(c->tmax, c->sweep0);
    const uint32_t n = min(t - c->sweep0, hist_cap);
    unsigned long long mx = 0;
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) mx = max(mx, hist[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ unsigned long long wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < blockDim.x / 32; ++w) mx = max(mx, wm[w]);
        c->max_width = mx;
        c->sweep = t + 1;
    }
}

// Device-side write-back in the reference TermStore layout (term_store.hpp:
// 15-45): hss, column-major args, refcounts and nf of slots [0, n) of a
// compacted arena, packed into a staging buffer for one D2H per column.
template <int W>
__global__ void pack_store(const uint32_t* __restrict__ A, uint32_t n, const uint8_t* __restrict__ arity,
                           uint32_t ma, uint32_t* __restrict__ hss, uint32_t* __restrict__ args,
                           uint32_t* __restrict__ rcs, uint8_t* __restrict__ nf) {
    for (uint32_t y = blockIdx.x * blockDim.x + threadIdx.x; y < n; y += gridDim.x * blockDim.x) {
        if (y == 0) {
            hss[0] = 0;
            rcs[0] = 0;
            nf[0] = 0;
            for (uint32_t j = 0; j < ma; ++j) args[(size_t)j * n] = 0;
            continue;
        }
        const uint32_t* R = A + (size_t)y * W;
        const uint4 q0 = *reinterpret_cast<const uint4*>(R);  // head, epoch, rc, waiter
        const uint32_t sym = q0.x & kSymMask;
        const uint32_t ar = arity[sym];
        hss[y] = sym;
        rcs[y] = q0.z;
        nf[y] = epoch_nf(q0.y);
        for (uint32_t j = 0; j < ma; ++j) args[(size_t)j * n + y] = j < ar ? R[kWArgs + j] : 0u;
    }
}

// Layout evidence: the derive's probe pattern -- a node's
// head, epoch word and arguments, then each argument's head and epoch word --
// over the store of the last run, read from the engine's AoS records or from
// SoA columns built from them (the reference's TermStore layout,
// term_store.hpp:15-45: hss, nf, args[j] as separate arrays).
template <int W>
__global__ void to_soa(const uint32_t* __restrict__ A, uint32_t n, uint32_t* __restrict__ hss,
                       uint32_t* __restrict__ ep, uint32_t* __restrict__ args, uint32_t na) {
    for (uint32_t y = blockIdx.x * blockDim.x + threadIdx.x; y < n; y += gridDim.x * blockDim.x) {
        const uint32_t* R = A + (size_t)y * W;
        hss[y] = R[kWHead];
        ep[y] = R[kWEpoch];
        for (uint32_t j = 0; j < na; ++j) args[(size_t)j * n + y] = R[kWArgs + j];
    }
}

// The probes visit every slot either in slot order or in a hashed order
// (every parent a random slot, as a sweep's frontier order is at worst).
__device__ __forceinline__ uint32_t probe_slot(uint32_t k, uint32_t n) {
    uint64_t z = 0x9e3779b97f4a7c15ull * k;
    z = (z ^ (z >> 31)) * 0xbf58476d1ce4e5b9ull;
    return 1u + (uint32_t)((z ^ (z >> 29)) % (uint64_t)(n - 1));
}

template <int W>
__global__ void probe_aos(const uint32_t* __restrict__ A, uint32_t n, const uint8_t* __restrict__ arity,
                          uint32_t* __restrict__ sink, bool random_order) {
    uint32_t acc = 0;
    for (uint32_t k = 1 + blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t y = random_order ? probe_slot(k, n) : k;
        const uint4 h = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)y * W));
        if (h.x == kDeadHead) continue;
        const uint4 a = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)y * W + kWArgs));
        const uint32_t ar = arity[h.x & kSymMask];
        const uint32_t c[4] = {a.x, a.y, a.z, a.w};
        acc += h.y;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((uint32_t)j < ar) {
                const uint2 ch = __ldcg(reinterpret_cast<const uint2*>(A + (size_t)c[j] * W));
                acc += ch.x ^ ch.y;
            }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
}

__global__ void probe_soa(const uint32_t* __restrict__ hss, const uint32_t* __restrict__ ep,
                          const uint32_t* __restrict__ args, uint32_t n, uint32_t na, const uint8_t* __restrict__ arity,
                          uint32_t* __restrict__ sink, bool random_order) {
    uint32_t acc = 0;
    for (uint32_t k = 1 + blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t y = random_order ? probe_slot(k, n) : k;
        const uint32_t head = __ldcg(hss + y);
        if (head == kDeadHead) continue;
        const uint32_t ar = arity[head & kSymMask];
        acc += __ldcg(ep + y);
        for (uint32_t j = 0; j < na && j < 4; ++j)
            if (j < ar) {
                const uint32_t c = __ldcg(args + (size_t)j * n + y);
                acc += __ldcg(hss + c) ^ __ldcg(ep + c);
            }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
}

__global__ void fill_random(uint32_t* idx, uint32_t n, uint64_t seed) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        uint64_t z = seed + 0x9e3779b97f4a7c15ull * (k + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        idx[k] = (uint32_t)(z ^ (z >> 31));
    }
}

}  // namespace

// ===========================================================================
// host side

struct RunState {
    trs_gpu_options opt{};
    bool runahead = false;
    int blocks = 0;
    uint32_t launches = 0;
    float total_ms = 0.f;
    cudaEvent_t a = nullptr, b = nullptr;
    bool active = false;
};

struct trs_gpu_engine {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    std::string last_error;

    // program
    std::vector<uint8_t> blob;
    uint8_t* d_prog = nullptr;
    uint32_t max_arity = 0;
    uint32_t max_new = 0;
    uint32_t num_symbols = 0;
    std::vector<uint32_t> arity;
    std::vector<uint32_t> rule_source;  // source order of each device rule (trs_gpu_dump_program)
    int W = 8;
    int minb = 1;  // register budget variant of the step loop (see step_loop_for)
    bool resident_on = false;  // this run reserves the shared-memory resident arena
    uint64_t pg_capacity = 0;  // prefer_grow() cache key (capacity, W) and value
    int pg_W = 0;
    bool pg_value = false;
    // grid_blocks() cache: kernel, dynamic shared memory, blocks-per-SM cap -> blocks
    const void* gb_fn = nullptr;
    size_t gb_dyn = 0;
    uint32_t gb_cap = 0;
    int gb_blocks = 0;
    const void* jit_kernel = nullptr;  // the program's specialised step loop (jit.hpp), if compiled
    const void* jit_kernel_ra = nullptr;  // ... its run-ahead build
    bool use_ra = false;               // the pending run is in its run-ahead phase
    bool has_chains = false;           // the program has constant chains (device_program.hpp)
    bool rc_stale = false;             // a run without refcount tracking: live_count recounts first
    bool jit_off = false;              // this run uses the interpreted step loop
    double jit_seconds = 0;
    int jit_minb = 1;
    std::string jit_log;
    uint32_t max_vars = 1;     // binding columns the step loop keeps in shared memory
    uint32_t input_n = 0;      // slots of the loaded store
    uint32_t rich = 0;  // frontier entry format of the loaded store (fixed at load time)

    // store
    uint64_t capacity = 0;        // logical capacity (slots) the step loop may use
    uint64_t alloc_capacity = 0;  // slots physically allocated per arena
    int alloc_W = 0;
    uint32_t roots_cap = 0;
    uint32_t* d_arena[2] = {nullptr, nullptr};
    uint32_t* d_list[2] = {nullptr, nullptr};
    uint32_t* d_gcmap = nullptr;
    uint32_t* d_roots = nullptr;
    uint32_t* d_blocksum = nullptr;       // GC per-CTA sums + rotating claim counters
    uint32_t* d_regions = nullptr;        // [2][2][kMaxGrid] frontier region tables
    unsigned long long* d_region_rew = nullptr;  // [2][kMaxGrid]
    uint32_t num_roots = 0;
    Ctl* d_ctl = nullptr;
    Ctl* h_ctl = nullptr;                 // pinned read-back of the control block
    Ctl export_ctl{};                     // control block of the exported state
    RunState run{};                       // the pending run (trs_gpu_run_async .. trs_gpu_run_wait)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    volatile uint32_t* h_gate = nullptr;  // trs_gpu_hold / trs_gpu_release
    uint32_t* d_gate = nullptr;
    uint32_t* d_roots_out = nullptr;      // renumbered roots of the export
    uint32_t* d_stage = nullptr;          // trs_gpu_load H2D staging
    size_t stage_words = 0;
    uint32_t roots_out_cap = 0;
    bool exported = false;                // staging holds the export of the current state (marked, renumbered)
    bool packed = false;                  // ... and its columns are packed
    std::vector<uint32_t> export_cta_live;  // live slots per renumbering range (rows of a range are contiguous)
    uint32_t export_blocks = 0;
    cudaStream_t stream2 = nullptr;       // D2H of packed column ranges, overlapping the next range's pack
    cudaEvent_t pack_ev[8] = {};
    bool canon_ready = false;             // d_words holds the canonical words of that export
    uint32_t* d_canon = nullptr;          // canonical relabelling scratch (canon.cuh)
    size_t canon_words_cap = 0;
    uint32_t* d_words = nullptr;
    size_t words_cap = 0;
    unsigned long long* d_woff = nullptr; // [roots + 1] word offsets, then [roots] hashes
    uint32_t* d_nodes = nullptr;
    uint32_t canon_roots_cap = 0;
    uint64_t canon_total = 0;
    trs_gpu_sweep_record* d_trace = nullptr;  // physical sweep records
    uint32_t trace_cap = 0;
    unsigned long long* d_hist = nullptr;     // rewrites per logical sweep (the reference's widths)
    uint32_t hist_cap = 0;
    uint32_t hist_used = 0;                   // entries the last run wrote (zeroed before the next)
    uint32_t* d_region_flags = nullptr;       // [2][kMaxGrid]
    uint32_t* d_val = nullptr;                // validate=2 scratch (validate.cuh), 3 words per slot
    uint64_t val_cap = 0;
    uint32_t last_psweeps = 0;
    bool loaded = false;
    uint32_t last_sweeps = 0;
    int record_width = 8;
    float load_ms = 0.f;
    cudaEvent_t load_a = nullptr, load_b = nullptr;  // bracket the last load (read lazily)
};

namespace {

int fail(trs_gpu_engine* e, int code, const std::string& msg) {
    if (e) e->last_error = msg;
    return code;
}

// Entry points that read or replace device state refuse while a run is
// pending (trs_gpu_run_async .. trs_gpu_run_wait): the step loop may be
// relaunched on the same buffers between the two.
#define REFUSE_PENDING(e)                                                            \
    do {                                                                              \
        if ((e)->run.active) return fail((e), TRS_GPU_INVALID, "a run is pending (call trs_gpu_run_wait first)"); \
    } while (0)

#define CUDA_TRY(e, call)                                                              \
    do {                                                                              \
        cudaError_t err_ = (call);                                                    \
        if (err_ != cudaSuccess)                                                      \
            return fail((e), TRS_GPU_CUDA, std::string(#call ": ") + cudaGetErrorString(err_)); \
    } while (0)

void free_store(trs_gpu_engine* e) {
    for (int k = 0; k < 2; ++k) {
        cudaFree(e->d_arena[k]);
        cudaFree(e->d_list[k]);
        e->d_arena[k] = e->d_list[k] = nullptr;
    }
    cudaFree(e->d_gcmap);
    cudaFree(e->d_roots);
    cudaFree(e->d_blocksum);
    cudaFree(e->d_regions);
    cudaFree(e->d_region_rew);
    e->d_regions = nullptr;
    e->d_region_rew = nullptr;
    cudaFree(e->d_ctl);
    cudaFree(e->d_trace);
    cudaFree(e->d_hist);
    cudaFree(e->d_region_flags);
    cudaFree(e->d_val);
    e->d_val = nullptr;
    e->val_cap = 0;
    e->d_hist = nullptr;
    e->d_region_flags = nullptr;
    e->hist_cap = e->hist_used = 0;
    e->d_gcmap = e->d_roots = e->d_blocksum = nullptr;
    e->d_ctl = nullptr;
    e->d_trace = nullptr;
    e->loaded = false;
    e->capacity = e->alloc_capacity = 0;
    e->alloc_W = 0;
    e->roots_cap = 0;
    e->trace_cap = 0;
}

int words_for_arity(uint32_t max_arity) {
    if (max_arity <= 4) return 8;
    if (max_arity <= 8) return 16;
    if (max_arity <= 28) return 32;
    return 0;
}

// Build the device blob from the flattened reference DispatchTable.
// Level-synchronous matching plan of symbol f (device_program.hpp, DPlan):
// assigns every step of f's rules a register source and the collapse
// source of each collapsing rule, or leaves f on the interpreted matcher.
DPlan plan_symbol(const trs_gpu_program* p, uint32_t f, std::vector<DStep>& steps, std::vector<DRule>& rules) {
    DPlan pl{};
    struct Path {
        int depth;
        uint32_t c[3];
    };
    std::vector<std::pair<uint32_t, bool>> slots;  // (4j+k, needs its argument quad)
    auto slot_of = [&](uint32_t jk, bool args) -> int {
        for (size_t q = 0; q < slots.size(); ++q)
            if (slots[q].first == jk) {
                slots[q].second = slots[q].second || args;
                return (int)q;
            }
        slots.push_back({jk, args});
        return (int)slots.size() - 1;
    };
    bool fast = true;
    std::vector<std::vector<Path>> paths;
    for (uint32_t r = p->rule_begin[f]; r < p->rule_begin[f + 1]; ++r) {
        const trs_gpu_rule& R = p->rules[r];
        std::vector<Path> ps(R.num_steps);
        for (uint32_t t = 0; t < R.num_steps; ++t) {
            const trs_gpu_step& S = p->steps[R.first_step + t];
            Path q{};
            if (S.parent < 0) {
                q.depth = 1;
                q.c[0] = S.child;
            } else {
                q = ps[S.parent];
                if (q.depth >= 3) {
                    fast = false;
                    q.depth = 4;
                } else {
                    q.c[q.depth++] = S.child;
                }
            }
            ps[t] = q;
            if (q.depth >= 2 && (q.c[0] >= kPlanChildren || q.c[1] >= 4)) fast = false;
            if (q.depth == 3 && (S.kind == TRS_GPU_STEP_CHECK_HEAD || q.c[2] >= 4)) fast = false;
            if (q.depth > 3) fast = false;
            if (!fast) break;
            if (q.depth == 2) {
                pl.child_args |= (uint8_t)(1u << q.c[0]);
                if (S.kind == TRS_GPU_STEP_CHECK_HEAD) slot_of(q.c[0] * 4 + q.c[1], false);
            } else if (q.depth == 3) {
                pl.child_args |= (uint8_t)(1u << q.c[0]);
                slot_of(q.c[0] * 4 + q.c[1], true);
            }
        }
        paths.push_back(std::move(ps));
        if (!fast) break;
    }
    auto arg_slots = [&]() {
        uint32_t n = 0;
        for (auto& sl : slots) n += sl.second;
        return n;
    };
    if (!fast || slots.size() > kPlanSlots || arg_slots() > kPlanArgSlots) return DPlan{};
    // collapse sources: the record of the bound node is already in registers
    // when it is a child (with its argument quad) or an argument slot
    std::vector<int> csrc_slot(paths.size(), -1);
    for (uint32_t r = p->rule_begin[f], x = 0; r < p->rule_begin[f + 1]; ++r, ++x) {
        const trs_gpu_rule& R = p->rules[r];
        if (R.root_ref & TRS_GPU_REF_NODE) continue;
        int bind_t = -1;
        for (uint32_t t = 0; t < R.num_steps; ++t) {
            const trs_gpu_step& S = p->steps[R.first_step + t];
            if (S.kind == TRS_GPU_STEP_BIND_VAR && S.value == R.root_ref) bind_t = (int)t;
        }
        if (bind_t < 0) continue;
        const Path& q = paths[x][bind_t];
        if (q.depth == 1 && q.c[0] < kPlanChildren) {
            pl.child_args |= (uint8_t)(1u << q.c[0]);
            csrc_slot[x] = -2;  // child
        } else if (q.depth == 2) {
            auto saved = slots;
            int sl = slot_of(q.c[0] * 4 + q.c[1], true);
            if (slots.size() > kPlanSlots || arg_slots() > kPlanArgSlots) {
                slots = saved;
            } else {
                csrc_slot[x] = sl;
            }
        }
    }
    // argument-carrying slots first: only the first kPlanArgSlots may load arguments
    std::vector<int> order(slots.size());
    for (size_t q = 0; q < order.size(); ++q) order[q] = (int)q;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return slots[x].second > slots[y].second; });
    std::vector<int> rank(slots.size());
    for (size_t q = 0; q < order.size(); ++q) rank[order[q]] = (int)q;
    pl.fast = 1;
    pl.nslots = (uint8_t)slots.size();
    for (size_t q = 0; q < slots.size(); ++q) {
        pl.slot_jk[rank[q]] = (uint8_t)slots[q].first;
        if (slots[q].second) pl.slot_args |= (uint8_t)(1u << rank[q]);
    }
    auto find_slot = [&](uint32_t jk) {
        for (size_t q = 0; q < slots.size(); ++q)
            if (slots[q].first == jk) return rank[q];
        return -1;
    };
    for (uint32_t r = p->rule_begin[f], x = 0; r < p->rule_begin[f + 1]; ++r, ++x) {
        const trs_gpu_rule& R = p->rules[r];
        for (uint32_t t = 0; t < R.num_steps; ++t) {
            const trs_gpu_step& S = p->steps[R.first_step + t];
            const Path& q = paths[x][t];
            uint8_t src;
            if (q.depth == 1)
                src = (uint8_t)(kSrcChild + q.c[0]);
            else if (q.depth == 2)
                src = S.kind == TRS_GPU_STEP_CHECK_HEAD ? (uint8_t)(kSrcSlot + find_slot(q.c[0] * 4 + q.c[1]))
                                                       : (uint8_t)(kSrcCArg + q.c[0] * 4 + q.c[1]);
            else
                src = (uint8_t)(kSrcSArg + find_slot(q.c[0] * 4 + q.c[1]) * 4 + q.c[2]);
            steps[R.first_step + t].src = src;
        }
        if (csrc_slot[x] == -2) {
            for (uint32_t t = 0; t < R.num_steps; ++t) {
                const trs_gpu_step& S = p->steps[R.first_step + t];
                if (S.kind == TRS_GPU_STEP_BIND_VAR && S.value == R.root_ref) rules[r].csrc = (uint8_t)(kSrcChild + paths[x][t].c[0]);
            }
        } else if (csrc_slot[x] >= 0) {
            rules[r].csrc = (uint8_t)(kSrcSlot + rank[csrc_slot[x]]);
        }
    }
    return pl;
}

constexpr size_t kSmemBudget = 227 * 1024 - 12 * 1024;  // dynamic bytes, leaving room for static smem
size_t dyn_base(const trs_gpu_engine* e);
int run_canon(trs_gpu_engine* e);

int build_blob(trs_gpu_engine* e, const trs_gpu_program* p) {
    if (!p || !p->arity || !p->rule_begin) return fail(e, TRS_GPU_INVALID, "null program");
    if (p->num_symbols == 0 || p->num_symbols > (1u << 16) - 2)
        return fail(e, TRS_GPU_INVALID, "symbol count out of range");
    uint32_t max_arity = 0;
    for (uint32_t f = 0; f < p->num_symbols; ++f) max_arity = std::max(max_arity, p->arity[f]);
    if (!words_for_arity(max_arity)) return fail(e, TRS_GPU_INVALID, "max arity above 28");
    if (p->rule_begin[p->num_symbols] != p->num_rules)
        return fail(e, TRS_GPU_INVALID, "rule_begin does not cover the rules");
    std::vector<DRule> rules(p->num_rules);
    std::vector<DStep> steps(p->num_steps);
    std::vector<DInstr> instrs(p->num_instrs);
    std::vector<uint16_t> refs(p->num_refs);
    if (p->num_steps > 65535 || p->num_instrs > 65535 || p->num_refs > 65535)
        return fail(e, TRS_GPU_INVALID, "program too large");
    uint32_t max_new = 0;
    for (uint32_t r = 0; r < p->num_rules; ++r) {
        const trs_gpu_rule& R = p->rules[r];
        if (R.num_steps > kMaxRuleSteps || R.num_instrs > kMaxRuleInstrs || R.num_vars > kMaxVars)
            return fail(e, TRS_GPU_INVALID, "rule beyond device limits");
        if (R.first_step + R.num_steps > p->num_steps || R.first_instr + R.num_instrs > p->num_instrs)
            return fail(e, TRS_GPU_INVALID, "rule indexes out of range");
        DRule& D = rules[r];
        std::memset(&D, 0, sizeof(D));
        D.first_step = (uint16_t)R.first_step;
        D.num_steps = (uint8_t)R.num_steps;
        D.num_vars = (uint8_t)R.num_vars;
        D.first_instr = (uint16_t)R.first_instr;
        D.num_instrs = (uint8_t)R.num_instrs;
        const bool collapse = !(R.root_ref & TRS_GPU_REF_NODE);
        D.collapse = collapse;
        D.root_ref = collapse ? (uint16_t)R.root_ref : (uint16_t)(kRefNode | (R.root_ref & 0x7fff));
        if (collapse && R.root_ref >= R.num_vars) return fail(e, TRS_GPU_INVALID, "collapse var out of range");
        if (!collapse && (R.root_ref & 0x7fffffff) + 1 != R.num_instrs)
            return fail(e, TRS_GPU_INVALID, "constructive root must be the last instruction");
        D.new_slots = collapse ? 0 : (uint8_t)(R.num_instrs - 1);
        D.root_wait = kNone;
        D.root_cursor = 0;
        D.csrc = kNone;
        max_new = std::max<uint32_t>(max_new, D.new_slots);
        for (uint32_t t = 0; t < R.num_steps; ++t) {
            const trs_gpu_step& S = p->steps[R.first_step + t];
            DStep& d = steps[R.first_step + t];
            std::memset(&d, 0, sizeof(d));
            if (S.parent >= (int32_t)t || S.parent < -1) return fail(e, TRS_GPU_INVALID, "step parent order");
            if (S.child >= 28) return fail(e, TRS_GPU_INVALID, "step child index");
            if (S.kind == TRS_GPU_STEP_BIND_VAR && S.value >= R.num_vars)
                return fail(e, TRS_GPU_INVALID, "bind var slot out of range");
            d.kind = (uint8_t)S.kind;
            d.src = kNone;
            d.child = (uint8_t)S.child;
            d.parent = (int8_t)S.parent;
            d.value = S.value;
        }
        // subscription plan (device_program.hpp): the first fresh child in
        // argument order is where the reference's next-sweep scan stops
        std::vector<int> claimed(R.num_instrs, -1);
        for (uint32_t k = 0; k < R.num_instrs; ++k) {
            const trs_gpu_instr& I = p->instrs[R.first_instr + k];
            if (I.symbol >= p->num_symbols) return fail(e, TRS_GPU_INVALID, "instr symbol");
            DInstr& d = instrs[R.first_instr + k];
            std::memset(&d, 0, sizeof(d));
            d.symbol = I.symbol;
            d.first_ref = (uint16_t)I.first_ref;
            if (I.indegree > 255) return fail(e, TRS_GPU_INVALID, "indegree above 255");
            d.indegree = (uint8_t)I.indegree;
            d.subscriber = kNone;
            d.cursor = 0;
            uint32_t ar = p->arity[I.symbol];
            if (I.first_ref + ar > p->num_refs) return fail(e, TRS_GPU_INVALID, "instr refs");
            int wait_on = -1;
            uint32_t wait_pos = 0;
            for (uint32_t j = 0; j < ar; ++j) {
                uint32_t ref = p->refs[I.first_ref + j];
                if (ref & TRS_GPU_REF_NODE) {
                    uint32_t target = ref & 0x7fffffff;
                    if (target >= k) return fail(e, TRS_GPU_INVALID, "template not topological");
                    if (wait_on < 0) {
                        wait_on = (int)target;
                        wait_pos = j;
                    }
                } else if (ref >= R.num_vars) {
                    return fail(e, TRS_GPU_INVALID, "template var out of range");
                }
            }
            const bool is_root = !collapse && k + 1 == R.num_instrs;
            d.cursor = (uint8_t)wait_pos;
            bool subscribed = false;
            if (wait_on >= 0 && claimed[wait_on] < 0) {
                claimed[wait_on] = (int)k;
                instrs[R.first_instr + wait_on].subscriber = is_root ? kRootSub : (uint8_t)k;
                subscribed = true;
            }
            if (is_root) {
                D.root_wait = subscribed ? (uint8_t)wait_on : kNone;
                D.root_cursor = (uint8_t)wait_pos;
            } else if (!subscribed) {
                D.push_mask |= 1u << k;
            }
        }
    }
    std::vector<DPlan> plans(p->num_symbols);
    for (uint32_t f = 0; f < p->num_symbols; ++f) plans[f] = plan_symbol(p, f, steps, rules);
    // match tables (device_program.hpp): only for W <= 16 and within a budget
    const int Wl = words_for_arity(max_arity);
    const uint32_t nsym = p->num_symbols;
    const uint32_t npos = Wl <= 16 ? (uint32_t)rec_args(Wl) + kPlanSlots : 0u;
    std::vector<uint16_t> mrow;
    std::vector<uint32_t> mtab;
    if (npos) {
        mrow.assign((size_t)nsym * npos, kNoRow);
        for (uint32_t f = 0; f < nsym; ++f) {
            if (!(plans[f].fast & kPlanFast)) continue;
            const uint32_t r0 = p->rule_begin[f], nr = p->rule_begin[f + 1] - r0;
            if (nr == 0 || nr > 32) continue;
            const uint32_t all = nr == 32 ? 0xFFFFFFFFu : (1u << nr) - 1u;
            std::vector<std::vector<uint32_t>> rows(npos);
            for (uint32_t r = 0; r < nr; ++r) {
                const trs_gpu_rule& R = p->rules[r0 + r];
                for (uint32_t t = 0; t < R.num_steps; ++t) {
                    const DStep& d = steps[R.first_step + t];
                    if (d.kind != 0) continue;
                    const uint32_t pos = d.src < kSrcSlot ? d.src : (uint32_t)rec_args(Wl) + (d.src - kSrcSlot);
                    if (pos >= npos || d.value >= nsym) continue;
                    if (rows[pos].empty()) rows[pos].assign(nsym, all);
                    for (uint32_t h = 0; h < nsym; ++h)
                        if (h != d.value) rows[pos][h] &= ~(1u << r);
                }
            }
            const size_t need = mtab.size();
            bool ok = true;
            for (uint32_t q = 0; q < npos && ok; ++q)
                if (!rows[q].empty() && mtab.size() + nsym > 0xFFFE) ok = false;
            if (!ok) continue;
            (void)need;
            for (uint32_t q = 0; q < npos; ++q) {
                if (rows[q].empty()) continue;
                mrow[(size_t)f * npos + q] = (uint16_t)mtab.size();
                mtab.insert(mtab.end(), rows[q].begin(), rows[q].end());
            }
            plans[f].fast |= kPlanTables;
        }
        // stay inside the program budget: without tables every symbol keeps the rule walk
        if (mtab.size() * 4 + mrow.size() * 2 > 16 * 1024) {
            for (auto& pl : plans) pl.fast &= (uint8_t)~kPlanTables;
            mrow.clear();
            mtab.clear();
        }
    }
    for (uint32_t k = 0; k < p->num_refs; ++k) {
        uint32_t ref = p->refs[k];
        refs[k] = (ref & TRS_GPU_REF_NODE) ? (uint16_t)(kRefNode | (ref & 0x7fff)) : (uint16_t)ref;
    }
    // pack
    auto align16 = [](uint32_t x) { return (x + 15u) & ~15u; };
    ProgHeader h{};
    h.num_symbols = p->num_symbols;
    h.num_rules = p->num_rules;
    h.num_steps = p->num_steps;
    h.num_instrs = p->num_instrs;
    h.num_refs = p->num_refs;
    h.max_arity = max_arity;
    h.max_new_slots = max_new;
    uint32_t off = align16(sizeof(ProgHeader));
    h.off_arity = off;
    off = align16(off + p->num_symbols);
    h.off_rule_begin = off;
    off = align16(off + 2 * (p->num_symbols + 1));
    h.off_rules = off;
    off = align16(off + sizeof(DRule) * p->num_rules);
    h.off_steps = off;
    off = align16(off + sizeof(DStep) * p->num_steps);
    h.off_instrs = off;
    off = align16(off + sizeof(DInstr) * p->num_instrs);
    h.off_refs = off;
    off = align16(off + 2 * p->num_refs);
    h.off_plans = off;
    off = align16(off + sizeof(DPlan) * p->num_symbols);
    h.npos = mtab.empty() ? 0u : npos;
    h.off_mrow = off;
    off = align16(off + 2 * (uint32_t)mrow.size());
    h.off_mtab = off;
    off = align16(off + 4 * (uint32_t)mtab.size());
    // constant chains (device_program.hpp)
    std::vector<uint16_t> chain(p->num_symbols, kChainNone);
    for (uint32_t f = 0; f < p->num_symbols; ++f) {
        if (p->arity[f] != 0) continue;
        if (p->rule_begin[f] == p->rule_begin[f + 1]) {
            chain[f] = kChainNf;
            continue;
        }
        const trs_gpu_rule& R = p->rules[p->rule_begin[f]];
        if (!(R.root_ref & TRS_GPU_REF_NODE) || R.num_instrs != 1) continue;
        const uint32_t g = p->instrs[R.first_instr].symbol;
        if (p->arity[g] == 0 && g < kChainNf) {
            chain[f] = (uint16_t)g;
            h.chains = 1;
        }
    }
    h.off_chain = off;
    off = align16(off + 2 * (uint32_t)chain.size());
    h.bytes = off;
    if (h.bytes > kMaxProgramBytes) return fail(e, TRS_GPU_INVALID, "program blob above 40 KiB");
    std::vector<uint8_t> blob(h.bytes, 0);
    std::memcpy(blob.data(), &h, sizeof(h));
    for (uint32_t f = 0; f < p->num_symbols; ++f) blob[h.off_arity + f] = (uint8_t)p->arity[f];
    for (uint32_t f = 0; f <= p->num_symbols; ++f) {
        if (p->rule_begin[f] > 65535) return fail(e, TRS_GPU_INVALID, "too many rules");
        uint16_t v = (uint16_t)p->rule_begin[f];
        std::memcpy(blob.data() + h.off_rule_begin + 2 * f, &v, 2);
    }
    if (!rules.empty()) std::memcpy(blob.data() + h.off_rules, rules.data(), sizeof(DRule) * rules.size());
    if (!steps.empty()) std::memcpy(blob.data() + h.off_steps, steps.data(), sizeof(DStep) * steps.size());
    if (!instrs.empty()) std::memcpy(blob.data() + h.off_instrs, instrs.data(), sizeof(DInstr) * instrs.size());
    if (!refs.empty()) std::memcpy(blob.data() + h.off_refs, refs.data(), 2 * refs.size());
    std::memcpy(blob.data() + h.off_plans, plans.data(), sizeof(DPlan) * plans.size());
    if (!mrow.empty()) std::memcpy(blob.data() + h.off_mrow, mrow.data(), 2 * mrow.size());
    if (!mtab.empty()) std::memcpy(blob.data() + h.off_mtab, mtab.data(), 4 * mtab.size());
    std::memcpy(blob.data() + h.off_chain, chain.data(), 2 * chain.size());
    e->blob = std::move(blob);
    e->max_arity = max_arity;
    e->max_new = max_new;
    e->max_vars = 1;
    for (uint32_t r = 0; r < p->num_rules; ++r) e->max_vars = std::max<uint32_t>(e->max_vars, p->rules[r].num_vars);
    if (dyn_base(e) > kSmemBudget)
        return fail(e, TRS_GPU_INVALID, "program + binding columns exceed the step loop's shared memory");
    e->num_symbols = p->num_symbols;
    e->has_chains = reinterpret_cast<const ProgHeader*>(e->blob.data())->chains != 0;
    e->arity.assign(p->arity, p->arity + p->num_symbols);
    e->rule_source.resize(p->num_rules);
    for (uint32_t r = 0; r < p->num_rules; ++r) e->rule_source[r] = p->rules[r].source_order;
    e->W = words_for_arity(max_arity);
    return TRS_GPU_OK;
}

// Two register budgets per record width: MINB = 1 (no spills, 1 CTA of 512
// threads per SM) and MINB = 2 (64 registers, 2 CTAs per SM, some spills).
template <int W, int MINB, bool RA>
const void* step_loop_ptr() {
    return reinterpret_cast<const void*>(&step_loop<W, MINB, RA>);
}

// The lean synchronous build (ra = false) or the run-ahead build.
template <bool RA>
const void* step_loop_for_ra(int W, int minb) {
    if (minb >= 2) {
        switch (W) {
            case 8: return step_loop_ptr<8, 2, RA>();
            case 16: return step_loop_ptr<16, 2, RA>();
            default: return step_loop_ptr<32, 2, RA>();
        }
    }
    switch (W) {
        case 8: return step_loop_ptr<8, 1, RA>();
        case 16: return step_loop_ptr<16, 1, RA>();
        default: return step_loop_ptr<32, 1, RA>();
    }
}

const void* step_loop_for(int W, int minb, bool ra) {
    return ra ? step_loop_for_ra<true>(W, minb) : step_loop_for_ra<false>(W, minb);
}

// Dynamic shared memory of the step loop: program blob, the two single-CTA
// frontier lists, and (when enabled) the resident arena of the single-CTA
// mode (sweep.cuh, run_small).
size_t dyn_base(const trs_gpu_engine* e) {
    return e->blob.size() + 2 * kSmallCap * sizeof(uint32_t) + (size_t)e->max_vars * kBlock * sizeof(uint32_t);
}
uint32_t resident_slots(const trs_gpu_engine* e) {
    const size_t base = dyn_base(e);
    if (base >= kSmemBudget) return 0;
    size_t slots = (kSmemBudget - base) / ((size_t)e->W * 4);
    slots = std::min<size_t>(slots, kSmallCap);  // local_gc keeps its map in an idle frontier list
    return slots >= 256 ? (uint32_t)slots : 0u;
}
size_t dyn_smem(const trs_gpu_engine* e) {
    return dyn_base(e) + (e->resident_on ? (size_t)resident_slots(e) * e->W * 4 : 0);
}

int alloc_store(trs_gpu_engine* e, uint64_t capacity) {
    size_t rec_bytes = (size_t)e->W * 4;
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(e, cudaMalloc(&e->d_arena[k], rec_bytes * capacity));
        CUDA_TRY(e, cudaMalloc(&e->d_list[k], sizeof(uint32_t) * e->W * capacity));
        // once per allocation: record words past an arity are never written, but
        // whole-record copies (resident arena, compaction) move them
        CUDA_TRY(e, cudaMemsetAsync(e->d_arena[k], 0, rec_bytes * capacity, e->stream));
    }
    CUDA_TRY(e, cudaMalloc(&e->d_gcmap, sizeof(uint32_t) * capacity));
    e->capacity = capacity;
    e->alloc_capacity = capacity;
    e->alloc_W = e->W;
    return TRS_GPU_OK;
}

// The step loop of this engine's next launch: the program's specialised
// kernel when one was compiled (and not switched off for the run), else the
// interpreted kernel of the record width.
const void* loop_kernel(const trs_gpu_engine* e) {
    if (e->jit_kernel && e->jit_kernel_ra && !e->jit_off) return e->use_ra ? e->jit_kernel_ra : e->jit_kernel;
    return step_loop_for(e->W, e->minb, e->use_ra);
}

int grid_blocks(trs_gpu_engine* e, uint32_t blocks_per_sm) {
    int occ = 0;
    size_t dyn = dyn_smem(e);
    const void* fn = loop_kernel(e);
    if (fn == e->gb_fn && dyn == e->gb_dyn && blocks_per_sm == e->gb_cap && e->gb_blocks) return e->gb_blocks;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, dyn) != cudaSuccess || occ < 1)
        occ = 1;
    if (blocks_per_sm) occ = std::min<int>(occ, (int)blocks_per_sm);
    e->gb_fn = fn;
    e->gb_dyn = dyn;
    e->gb_cap = blocks_per_sm;
    e->gb_blocks = std::min<int>(occ * e->sm_count, (int)kMaxGrid);
    return e->gb_blocks;
}

// Frontier of the next sweep (list buffer c.cur): total entries and the
// end of its furthest region.
uint64_t frontier_extent(trs_gpu_engine* e, const Ctl& c, uint64_t* total = nullptr) {
    uint32_t R = c.nregions[c.cur];
    std::vector<uint32_t> off(R), cnt(R);
    if (R) {
        cudaMemcpy(off.data(), e->d_regions + c.cur * 2 * kMaxGrid, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost);
        cudaMemcpy(cnt.data(), e->d_regions + c.cur * 2 * kMaxGrid + kMaxGrid, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost);
    }
    uint64_t ext = 0, tot = 0;
    for (uint32_t r = 0; r < R; ++r) {
        ext = std::max<uint64_t>(ext, (uint64_t)off[r] + cnt[r]);
        tot += cnt[r];
    }
    if (total) *total = tot;
    return ext;
}

// Grow every device array so that the next sweep fits (the reference's
// ensure_headroom + TermStore::grow, sweep_engine.cpp:290-303,
// term_store.cpp:8-27).
int grow_store(trs_gpu_engine* e, uint64_t needed) {
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    uint64_t cap = std::max<uint64_t>(needed, e->capacity * 2);
    if (cap > 0xFFFFFFF0ull) cap = 0xFFFFFFF0ull;
    if (cap <= e->capacity) return fail(e, TRS_GPU_CAPACITY, "term store would exceed 2^32 slots");
    if (cap <= e->alloc_capacity) {
        e->capacity = cap;
        return TRS_GPU_OK;
    }
    size_t rec_bytes = (size_t)e->W * 4;
    uint32_t* na[2] = {nullptr, nullptr};
    uint32_t* nl[2] = {nullptr, nullptr};
    uint32_t* nm = nullptr;
    for (int k = 0; k < 2; ++k) {
        if (cudaMalloc(&na[k], rec_bytes * cap) != cudaSuccess || cudaMalloc(&nl[k], rec_bytes * cap) != cudaSuccess) {
            for (int j = 0; j < 2; ++j) { cudaFree(na[j]); cudaFree(nl[j]); }
            cudaGetLastError();
            return fail(e, TRS_GPU_CAPACITY, "device memory exhausted while growing the term store");
        }
    }
    if (cudaMalloc(&nm, sizeof(uint32_t) * cap) != cudaSuccess) {
        for (int j = 0; j < 2; ++j) { cudaFree(na[j]); cudaFree(nl[j]); }
        cudaGetLastError();
        return fail(e, TRS_GPU_CAPACITY, "device memory exhausted while growing the term store");
    }
    // the frontier of the next sweep: regions of list buffer c.cur
    uint64_t extent = frontier_extent(e, c);
    for (int k = 0; k < 2; ++k) CUDA_TRY(e, cudaMemsetAsync(na[k], 0, rec_bytes * cap, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(na[c.arena], e->d_arena[c.arena], rec_bytes * c.bump, cudaMemcpyDeviceToDevice, e->stream));
    // frontier entries are one word (bare slots) or a record (rich entries)
    const size_t entry_bytes = e->rich ? rec_bytes : sizeof(uint32_t);
    if (extent)
        CUDA_TRY(e, cudaMemcpyAsync(nl[c.cur], e->d_list[c.cur], std::min(entry_bytes * extent, rec_bytes * e->alloc_capacity),
                                    cudaMemcpyDeviceToDevice, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    for (int k = 0; k < 2; ++k) {
        cudaFree(e->d_arena[k]);
        cudaFree(e->d_list[k]);
        e->d_arena[k] = na[k];
        e->d_list[k] = nl[k];
    }
    cudaFree(e->d_gcmap);
    e->d_gcmap = nm;
    e->capacity = cap;
    e->alloc_capacity = cap;
    return TRS_GPU_OK;
}

// Host reads/writes of the control block use synchronous copies on the
// legacy stream, which does not order against the engine's non-blocking
// stream: drain the engine stream first at every entry point.
int drain(trs_gpu_engine* e) {
    cudaError_t err = cudaStreamSynchronize(e->stream);
    if (err != cudaSuccess) return fail(e, TRS_GPU_CUDA, std::string("engine stream: ") + cudaGetErrorString(err));
    return TRS_GPU_OK;
}

// Before every step-loop launch: barrier counter and rotating claim
// counters start at zero.
void reset_barrier(trs_gpu_engine* e) {
    cudaMemsetAsync(reinterpret_cast<uint8_t*>(e->d_ctl) + offsetof(Ctl, bar_arrive), 0, sizeof(uint32_t), e->stream);
    cudaMemsetAsync(e->d_blocksum + kMaxGrid, 0, sizeof(uint32_t) * 8, e->stream);
}

Params make_params(trs_gpu_engine* e, int blocks) {
    Params P{};
    P.arena[0] = e->d_arena[0];
    P.arena[1] = e->d_arena[1];
    P.list[0] = e->d_list[0];
    P.list[1] = e->d_list[1];
    P.gcmap = e->d_gcmap;
    P.blocksum = e->d_blocksum;
    P.regions = e->d_regions;
    P.region_rew = e->d_region_rew;
    P.roots = e->d_roots;
    P.num_roots = e->num_roots;
    P.ctl = e->d_ctl;
    P.trace = e->d_trace;
    P.trace_cap = e->trace_cap;
    P.prog = e->d_prog;
    P.prog_bytes = (uint32_t)e->blob.size();
    P.capacity = e->capacity;
    P.max_new = e->max_new;
    P.step_budget = 1000000000ull;
    P.rich = e->rich;
    P.max_vars = e->max_vars;
    P.region_flags = e->d_region_flags;
    P.hist = e->d_hist;
    P.hist_cap = e->hist_cap;
    P.list_cap = e->rich ? e->alloc_capacity : (uint64_t)e->alloc_W * e->alloc_capacity;
    // slab: 256 slots per warp unless the arena is small
    uint64_t per_warp = e->capacity / (4ull * (uint64_t)blocks * kWarps);
    P.slab = (uint32_t)std::max<uint64_t>(16, std::min<uint64_t>(256, per_warp));
    return P;
}

// Growing is preferred over collecting while the twin arenas, lists and
// map of the grown store fit comfortably in free HBM; the compacting GC is
// the memory-pressure path (and what fixed-capacity stores rely on).
bool prefer_grow(trs_gpu_engine* e) {
    // cudaMemGetInfo can stall the host for milliseconds: ask once per
    // capacity, not once per launch
    if (e->pg_capacity != e->capacity || e->pg_W != e->W) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
            cudaGetLastError();
            free_b = 0;
        }
        const uint64_t next = e->capacity * 2;
        const uint64_t need = next * ((uint64_t)e->W * 4 * 2 + 4 * 3);
        e->pg_value = need < free_b / 2;
        e->pg_capacity = e->capacity;
        e->pg_W = e->W;
    }
    return e->pg_value;
}

int grow_trace(trs_gpu_engine* e) {
    uint32_t cap = e->trace_cap * 2;
    trs_gpu_sweep_record* nt = nullptr;
    CUDA_TRY(e, cudaMalloc(&nt, sizeof(trs_gpu_sweep_record) * cap));
    CUDA_TRY(e, cudaMemcpy(nt, e->d_trace, sizeof(trs_gpu_sweep_record) * e->trace_cap, cudaMemcpyDeviceToDevice));
    cudaFree(e->d_trace);
    e->d_trace = nt;
    e->trace_cap = cap;
    return TRS_GPU_OK;
}

int grow_hist(trs_gpu_engine* e, uint32_t need) {
    if (need >= kEpochMask - 2)
        return fail(e, TRS_GPU_STEP_BUDGET, "more than 2^27 logical sweeps; the derivation may not terminate");
    uint32_t cap = e->hist_cap;
    while (cap < need) cap *= 2;
    unsigned long long* nh = nullptr;
    CUDA_TRY(e, cudaMalloc(&nh, sizeof(unsigned long long) * cap));
    CUDA_TRY(e, cudaMemsetAsync(nh, 0, sizeof(unsigned long long) * cap, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(nh, e->d_hist, sizeof(unsigned long long) * e->hist_cap, cudaMemcpyDeviceToDevice,
                                e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    cudaFree(e->d_hist);
    e->d_hist = nh;
    e->hist_cap = cap;
    return TRS_GPU_OK;
}

template <int W>
void launch_load(trs_gpu_engine* e, uint32_t n, const uint32_t* hss, const uint32_t* args, uint32_t max_arity,
                 const uint32_t* rc, const uint8_t* d_arity, uint32_t* count) {
    int blocks = std::max(1, std::min<int>((int)((n + 255) / 256), e->sm_count * 8));
    load_records<W><<<blocks, 256, 0, e->stream>>>(e->d_arena[0], n, hss, args, max_arity, rc);
    load_frontier<W><<<blocks, 256, 0, e->stream>>>(e->d_arena[0], n, d_arity, e->d_list[0], count, e->rich);
}

int load_impl(trs_gpu_engine* e, uint32_t n, const uint32_t* roots, uint32_t num_roots,
              const uint32_t* d_hss, const uint32_t* d_args, uint32_t max_arity, const uint32_t* d_rc,
              uint64_t capacity) {
    if (e->blob.empty()) return fail(e, TRS_GPU_INVALID, "no program set");
    if (n < 2 || num_roots == 0) return fail(e, TRS_GPU_INVALID, "empty store");
    if (max_arity > (uint32_t)rec_args(e->W))
        return fail(e, TRS_GPU_INVALID, "store arity exceeds program record width");
    for (uint32_t r = 0; r < num_roots; ++r)
        if (roots[r] == 0 || roots[r] >= n) return fail(e, TRS_GPU_INVALID, "root out of range");
    if (capacity != 0 && capacity < n)
        return fail(e, TRS_GPU_CAPACITY, "store capacity " + std::to_string(capacity) + " cannot hold " +
                                             std::to_string(n - 1) + " input term nodes");
    uint64_t want = capacity;
    if (want == 0) {
        // auto: room for the input and a generous allocation window; the
        // step loop collects and grows on demand
        want = std::max<uint64_t>((uint64_t)n * 4 + 1024, 1ull << 22);
        if (e->alloc_W == e->W && e->alloc_capacity > want) want = e->alloc_capacity;
    }
    if (e->alloc_W != e->W || e->alloc_capacity < want) {
        free_store(e);
        int rc = alloc_store(e, want);
        if (rc) return rc;
    }
    e->capacity = want;
    if (!e->d_ctl) CUDA_TRY(e, cudaMalloc(&e->d_ctl, sizeof(Ctl)));
    CUDA_TRY(e, cudaMemsetAsync(e->d_ctl, 0, sizeof(Ctl), e->stream));
    if (e->roots_cap < num_roots) {
        cudaFree(e->d_roots);
        CUDA_TRY(e, cudaMalloc(&e->d_roots, sizeof(uint32_t) * num_roots));
        e->roots_cap = num_roots;
    }
    CUDA_TRY(e, cudaMemcpyAsync(e->d_roots, roots, sizeof(uint32_t) * num_roots, cudaMemcpyHostToDevice, e->stream));
    if (!e->d_blocksum) CUDA_TRY(e, cudaMalloc(&e->d_blocksum, sizeof(uint32_t) * (kMaxGrid + 8)));
    if (!e->d_regions) CUDA_TRY(e, cudaMalloc(&e->d_regions, sizeof(uint32_t) * 4 * kMaxGrid));
    if (!e->d_region_rew) CUDA_TRY(e, cudaMalloc(&e->d_region_rew, sizeof(unsigned long long) * 2 * kMaxGrid));
    if (!e->d_region_flags) CUDA_TRY(e, cudaMalloc(&e->d_region_flags, sizeof(uint32_t) * 2 * kMaxGrid));
    CUDA_TRY(e, cudaMemsetAsync(e->d_region_flags, 0, sizeof(uint32_t) * 2 * kMaxGrid, e->stream));
    if (!e->d_hist) {
        e->hist_cap = 1u << 16;
        CUDA_TRY(e, cudaMalloc(&e->d_hist, sizeof(unsigned long long) * e->hist_cap));
        CUDA_TRY(e, cudaMemsetAsync(e->d_hist, 0, sizeof(unsigned long long) * e->hist_cap, e->stream));
        e->hist_used = 0;
    }
    CUDA_TRY(e, cudaMemsetAsync(e->d_blocksum, 0, sizeof(uint32_t) * (kMaxGrid + 8), e->stream));
    if (!e->d_trace) {
        e->trace_cap = 1u << 16;
        CUDA_TRY(e, cudaMalloc(&e->d_trace, sizeof(trs_gpu_sweep_record) * e->trace_cap));
    }
    if (e->d_prog == nullptr) return fail(e, TRS_GPU_INVALID, "program not staged");
    // frontier count of sweep 1: a scratch word of the blocksum array (zeroed above)
    uint32_t* d_count = e->d_blocksum + kMaxGrid + 7;
    const uint8_t* d_arity = e->d_prog + reinterpret_cast<const ProgHeader*>(e->blob.data())->off_arity;
    cudaEvent_t a = e->load_a, b = e->load_b;
    if (!a) cudaEventCreate(&a);
    if (!b) cudaEventCreate(&b);
    cudaEventRecord(a, e->stream);
    switch (e->W) {
        case 8: launch_load<8>(e, n, d_hss, d_args, max_arity, d_rc, d_arity, d_count); break;
        case 16: launch_load<16>(e, n, d_hss, d_args, max_arity, d_rc, d_arity, d_count); break;
        default: launch_load<32>(e, n, d_hss, d_args, max_arity, d_rc, d_arity, d_count); break;
    }
    // persistent state: sweep 0 done, bump pointer n, one frontier region
    init_ctl<<<1, 1, 0, e->stream>>>(e->d_ctl, e->d_regions, d_count, n);
    cudaEventRecord(b, e->stream);
    CUDA_TRY(e, cudaGetLastError());
    e->load_a = a;
    e->load_b = b;
    e->num_roots = num_roots;
    e->input_n = n;
    e->loaded = true;
    e->exported = false;
    e->rc_stale = false;
    e->last_sweeps = 0;
    return TRS_GPU_OK;
}

// Host-side canonical relabelling over a fetched arena.
struct HostArena {
    std::vector<uint32_t> words;  // W per slot
    uint32_t base = 0;
    int W = 8;
    const uint32_t* rec(uint32_t i) const { return words.data() + (size_t)i * W; }
};

int fetch_arena(trs_gpu_engine* e, HostArena& h, std::vector<uint32_t>& roots) {
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    h.W = e->W;
    h.base = c.bump;
    h.words.resize((size_t)c.bump * e->W);
    CUDA_TRY(e, cudaMemcpy(h.words.data(), e->d_arena[c.arena], sizeof(uint32_t) * h.words.size(), cudaMemcpyDeviceToHost));
    roots.resize(e->num_roots);
    CUDA_TRY(e, cudaMemcpy(roots.data(), e->d_roots, sizeof(uint32_t) * e->num_roots, cudaMemcpyDeviceToHost));
    return TRS_GPU_OK;
}

// Refcounts of a store that runs without tracking left stale (e->rc_stale):
// recounted from the store (gc.cuh recount_refs), synchronously.
int ensure_refcounts(trs_gpu_engine* e) {
    if (!e->rc_stale) return TRS_GPU_OK;
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    uint32_t* A = e->d_arena[c.arena];
    const uint8_t* arity = e->d_prog + reinterpret_cast<const ProgHeader*>(e->blob.data())->off_arity;
    const int blocks = e->sm_count * 8;
    switch (e->W) {
        case 8:
            recount_clear<8><<<blocks, 256, 0, e->stream>>>(A, c.bump);
            recount_add<8><<<blocks, 256, 0, e->stream>>>(A, c.bump, arity, e->d_roots, e->num_roots);
            break;
        case 16:
            recount_clear<16><<<blocks, 256, 0, e->stream>>>(A, c.bump);
            recount_add<16><<<blocks, 256, 0, e->stream>>>(A, c.bump, arity, e->d_roots, e->num_roots);
            break;
        default:
            recount_clear<32><<<blocks, 256, 0, e->stream>>>(A, c.bump);
            recount_add<32><<<blocks, 256, 0, e->stream>>>(A, c.bump, arity, e->d_roots, e->num_roots);
            break;
    }
    CUDA_TRY(e, cudaGetLastError());
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    e->rc_stale = false;
    return TRS_GPU_OK;
}

// Post-run refcount ghost invariant (sweep_engine.cpp:335-359): rc of every
// uncollected slot = references from uncollected slots + root pins, and no
// live slot references slot 0 or a collected slot.
int validate_store(trs_gpu_engine* e) {
    HostArena h;
    std::vector<uint32_t> roots;
    if (int r = fetch_arena(e, h, roots)) return r;
    std::vector<uint64_t> counted(h.base, 0);
    for (uint32_t i = 1; i < h.base; ++i) {
        const uint32_t* R = h.rec(i);
        if (R[kWHead] == kDeadHead) continue;
        uint32_t ar = e->arity[R[kWHead] & kSymMask];
        for (uint32_t j = 0; j < ar; ++j) {
            uint32_t ch = R[kWArgs + j];
            if (ch == 0 || ch >= h.base || h.rec(ch)[kWHead] == kDeadHead)
                return fail(e, TRS_GPU_DANGLING, "slot " + std::to_string(i) + " references invalid slot " + std::to_string(ch));
            counted[ch]++;
        }
    }
    for (uint32_t r2 : roots) counted[r2]++;
    for (uint32_t i = 1; i < h.base; ++i) {
        const uint32_t* R = h.rec(i);
        if (R[kWHead] == kDeadHead) continue;
        if (counted[i] != R[kWRc])
            return fail(e, TRS_GPU_DANGLING, "refcount ghost invariant: slot " + std::to_string(i) + " has rc " +
                                                 std::to_string(R[kWRc]) + ", expected " + std::to_string(counted[i]));
    }
    return TRS_GPU_OK;
}

}  // namespace

extern "C" {

int trs_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

const char* trs_gpu_error_string(int status) {
    switch (status) {
        case TRS_GPU_OK: return "ok";
        case TRS_GPU_STEP_BUDGET: return "step budget exceeded; the derivation may not terminate";
        case TRS_GPU_CAPACITY: return "term store capacity exhausted";
        case TRS_GPU_DANGLING: return "dangling reference in the term store";
        case TRS_GPU_INVALID: return "invalid argument";
        case TRS_GPU_CUDA: return "CUDA error";
    }
    return "unknown status";
}

const char* trs_gpu_last_error(trs_gpu_engine* e) { return e ? e->last_error.c_str() : ""; }

int trs_gpu_open(int device, trs_gpu_engine** out) {
    if (!out) return TRS_GPU_INVALID;
    *out = nullptr;
    int n = trs_gpu_device_count();
    if (device < 0 || device >= n) return TRS_GPU_CUDA;
    auto* e = new trs_gpu_engine();
    e->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete e;
        return TRS_GPU_CUDA;
    }
    cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, device);
    // experimental frontier format (sweep.cuh, rich entries); off by default
#if TRS_B200_RICH_ENTRIES
    if (const char* r = std::getenv("TRS_B200_RICH_ENTRIES")) e->rich = std::atoi(r) ? 1u : 0u;
#endif
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (!coop || cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete e;
        return TRS_GPU_CUDA;
    }
    *out = e;
    return TRS_GPU_OK;
}

void trs_gpu_close(trs_gpu_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    free_store(e);
    cudaFree(e->d_prog);
    if (e->h_ctl) cudaFreeHost(e->h_ctl);
    if (e->h_gate) cudaFreeHost((void*)e->h_gate);
    if (e->ev_a) cudaEventDestroy(e->ev_a);
    if (e->ev_b) cudaEventDestroy(e->ev_b);
    cudaFree(e->d_roots_out);
    cudaFree(e->d_stage);
    cudaFree(e->d_canon);
    cudaFree(e->d_words);
    cudaFree(e->d_woff);
    cudaFree(e->d_nodes);
    if (e->load_a) cudaEventDestroy(e->load_a);
    if (e->load_b) cudaEventDestroy(e->load_b);
    for (cudaEvent_t& ev : e->pack_ev)
        if (ev) cudaEventDestroy(ev);
    if (e->stream2) cudaStreamDestroy(e->stream2);
    cudaStreamDestroy(e->stream);
    delete e;
}

int trs_gpu_set_program(trs_gpu_engine* e, const trs_gpu_program* p) {
    if (!e) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    int rc = build_blob(e, p);
    if (rc) return rc;
    cudaFree(e->d_prog);
    e->d_prog = nullptr;
    CUDA_TRY(e, cudaMalloc(&e->d_prog, e->blob.size()));
    CUDA_TRY(e, cudaMemcpy(e->d_prog, e->blob.data(), e->blob.size(), cudaMemcpyHostToDevice));
    e->loaded = false;
    // specialise the step loop for this program (jit.hpp); TRS_B200_JIT=0
    // keeps the interpreted kernel, and a failed compilation falls back to it
    e->jit_kernel = nullptr;
    e->jit_kernel_ra = nullptr;
    e->jit_log.clear();
    e->jit_seconds = 0;
    const char* env = std::getenv("TRS_B200_JIT");
    if (!(env && env[0] == '0')) {
        const auto t0 = std::chrono::steady_clock::now();
        // experiment hook: the specialisation's register budget (MINB = 2 spills
        // and measured 1.5-2x slower on every config; the default is 1)
        const char* mb = std::getenv("TRS_B200_JIT_MINB");
        e->jit_minb = (mb && mb[0] == '2') ? 2 : 1;
        JitResult jr = jit_compile(jit_source(e->blob.data(), e->W, e->max_vars), e->W, e->jit_minb);
        e->jit_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        e->jit_kernel = jr.kernel;
        e->jit_kernel_ra = jr.kernel_ra;
        e->jit_log = jr.log;
        if (e->jit_kernel && e->jit_kernel_ra) {
            // load the module now (lazy loading would otherwise happen at the
            // first launch, possibly behind a held stream gate)
            cudaFuncAttributes fa;
            if (cudaFuncGetAttributes(&fa, e->jit_kernel) != cudaSuccess ||
                cudaFuncGetAttributes(&fa, e->jit_kernel_ra) != cudaSuccess) {
                cudaGetLastError();
                e->jit_kernel = e->jit_kernel_ra = nullptr;
                e->jit_log += "\nspecialised kernel failed to load";
            }
        } else {
            e->jit_kernel = e->jit_kernel_ra = nullptr;
        }
    }
    return TRS_GPU_OK;
}

int trs_gpu_jit_info(trs_gpu_engine* e, int* active, double* seconds, char* log, uint64_t log_cap) {
    if (!e) return TRS_GPU_INVALID;
    if (active) *active = e->jit_kernel ? 1 : 0;
    if (seconds) *seconds = e->jit_seconds;
    if (log && log_cap) {
        const size_t n = std::min<size_t>(e->jit_log.size(), log_cap - 1);
        std::memcpy(log, e->jit_log.data(), n);
        log[n] = 0;
    }
    return TRS_GPU_OK;
}

int trs_gpu_load(trs_gpu_engine* e, uint32_t n, const uint32_t* roots, uint32_t num_roots, const uint32_t* hss,
                 const uint32_t* args, uint32_t max_arity, const uint32_t* refcounts, uint64_t capacity) {
    if (!e || !hss || !refcounts || (max_arity && !args) || !roots) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    // H2D into a grow-only staging buffer owned by the engine (no per-call
    // allocation: allocator round trips show up as e2e jitter)
    const size_t na = (size_t)max_arity * n;
    const size_t words = (size_t)n * 2 + std::max<size_t>(na, 1);
    if (e->stage_words < words) {
        cudaFree(e->d_stage);
        e->d_stage = nullptr;
        e->stage_words = 0;
        CUDA_TRY(e, cudaMalloc(&e->d_stage, sizeof(uint32_t) * words));
        e->stage_words = words;
    }
    uint32_t* dh = e->d_stage;
    uint32_t* dr = dh + n;
    uint32_t* da = dr + n;
    CUDA_TRY(e, cudaMemcpyAsync(dh, hss, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e->stream));
    if (na) CUDA_TRY(e, cudaMemcpyAsync(da, args, sizeof(uint32_t) * na, cudaMemcpyHostToDevice, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(dr, refcounts, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e->stream));
    int rc = load_impl(e, n, roots, num_roots, dh, da, max_arity, dr, capacity);
    // the caller may reuse its host buffers on return
    cudaStreamSynchronize(e->stream);
    return rc;
}

int trs_gpu_load_device(trs_gpu_engine* e, uint32_t n, const uint32_t* roots, uint32_t num_roots,
                        const uint32_t* d_hss, const uint32_t* d_args, uint32_t max_arity,
                        const uint32_t* d_refcounts, uint64_t capacity) {
    if (!e || !d_hss || !d_refcounts || !roots) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    return load_impl(e, n, roots, num_roots, d_hss, d_args, max_arity, d_refcounts, capacity);
}

}  // extern "C"

namespace {

// One step-loop launch of the pending run on the engine stream: prep, the
// cooperative launch, the status read-back into pinned memory, the timing
// events.  Nothing here waits.
int enqueue_launch(trs_gpu_engine* e) {
    RunState& R = e->run;
    const trs_gpu_options& opt = R.opt;
    Params P = make_params(e, R.blocks);
    P.step_budget = opt.step_budget ? opt.step_budget : 1000000000ull;
    // single-CTA mode below 128 entries, back to the grid above 256
    // (profiles/r2_opts_ab2.log: build+sum(22) 5.17 -> 5.00 ms against 512 /
    // 1024, the other configs within 1 %)
    P.small_enter = opt.disable_small ? 0 : (opt.small_enter ? opt.small_enter : kBlock / 4);
    P.small_exit = opt.disable_small ? 0 : (opt.small_exit ? opt.small_exit : kBlock / 2);
    if (P.small_exit < P.small_enter) P.small_exit = P.small_enter;
    P.warp_mode = opt.disable_warp_mode ? 0 : 1;
    {
        // Warp mode takes frontiers of up to 32 entries in the lean build
        // (lanes in step: mergesort 2^14 10 % faster than spreading them over
        // the CTA's warps), but only single entries in the run-ahead build,
        // where each lane follows its own chain and a warp of diverging
        // chains pays for every path (fib(18) 7.9 -> 6.7 ms;
        // profiles/r2_ab_warpmax.log)
        const char* wm = std::getenv("TRS_B200_WARP_MAX");  // tuning hooks
        const char* wr = std::getenv("TRS_B200_WARP_MAX_RA");
        const uint32_t v = wm ? (uint32_t)std::strtoul(wm, nullptr, 10) : 32u;
        const uint32_t vr = wr ? (uint32_t)std::strtoul(wr, nullptr, 10) : 1u;
        P.warp_max = std::min<uint32_t>(std::max<uint32_t>(v, 1u), 32u);
        P.warp_max_ra = std::min<uint32_t>(std::max<uint32_t>(vr, 1u), 32u);
    }
    P.gc_interval = opt.gc_interval;
    P.allow_gc = opt.disable_gc ? 0 : 1;
    P.fixed_capacity = opt.fixed_capacity;
    P.prefer_grow = (!opt.fixed_capacity && !opt.gc_interval && prefer_grow(e)) ? 1u : 0u;
    P.profile = opt.profile;
    P.local_cap = e->resident_on ? resident_slots(e) : 0u;
    P.local_enter = P.local_cap / 2;
    if (opt.reserved[2]) P.slab = opt.reserved[2];  // experiment: slab override
    // run-ahead (lanes continue into slots their step made ready; logical
    // time keeps the widths exact) except where the reference's abort state
    // is part of the contract: an explicit step budget or a fixed capacity
    P.runahead = (R.runahead && !e->rich) ? 1u : 0u;
    if (opt.validate >= 2) {
        // quiescent-point scans before every grid sweep (validate.cuh): the
        // whole run in the grid mode, no run-ahead
        if (e->val_cap < e->alloc_capacity) {
            cudaFree(e->d_val);
            e->d_val = nullptr;
            e->val_cap = 0;
            CUDA_TRY(e, cudaMalloc(&e->d_val, sizeof(uint32_t) * 3 * e->alloc_capacity));
            e->val_cap = e->alloc_capacity;
        }
        CUDA_TRY(e, cudaMemsetAsync(e->d_val, 0, sizeof(uint32_t) * 3 * e->val_cap, e->stream));
        P.validate = 2;
        P.val = e->d_val;
        P.small_enter = P.small_exit = 0;
        P.runahead = 0;
    }
    {
        const char* rm = std::getenv("TRS_B200_RA_MAX");  // tuning hook
        // defaults from tools/ra_sweep.py (profiles/r2_ra_sweep*.log): run-ahead in
        // sweeps of up to one entry per lane, handed over after 64 sweeps of at
        // most two per lane, 32 continued steps per lane and physical sweep
        P.ra_max = rm ? (uint32_t)std::strtoul(rm, nullptr, 10) : (uint32_t)R.blocks * kWarps * 32u;
        const char* rk = std::getenv("TRS_B200_RA_KILL");
        P.ra_kill = rk ? (uint32_t)std::strtoul(rk, nullptr, 10) : (uint32_t)R.blocks * kWarps * 64u;
        const char* rw = std::getenv("TRS_B200_RA_WARM");
        P.ra_warm = rw ? (uint32_t)std::strtoul(rw, nullptr, 10) : 64u;
        const char* rp = std::getenv("TRS_B200_RA_WARM_PAST");
        P.ra_warm_past = rp ? (uint32_t)std::strtoul(rp, nullptr, 10) : 16u;
        const char* rs = std::getenv("TRS_B200_RA_STEPS");
        P.ra_steps = rs ? (uint32_t)std::strtoul(rs, nullptr, 10) : 32u;
        // refcounts are kept step by step only for the validate modes (their
        // checks read them); otherwise collectors and live_count recount
        const char* tr = std::getenv("TRS_B200_TRACK_RC");  // A/B hook (tools/rc_ab.py)
        P.track_rc = (opt.validate || (tr && tr[0] == '1')) ? 1u : 0u;
        if (!P.track_rc) e->rc_stale = true;
    }
    void* args[] = {&P};
    cudaEventRecord(R.a, e->stream);
    prep_launch<<<1, 256, 0, e->stream>>>(e->d_ctl, e->d_blocksum + kMaxGrid, e->d_region_flags,
                                          R.launches == 0 ? 1u : 0u);
    cudaError_t err =
        cudaLaunchCooperativeKernel(loop_kernel(e), R.blocks, kBlock, args, dyn_smem(e), e->stream);
    if (err == cudaSuccess) {
        finish_run<<<1, 256, 0, e->stream>>>(e->d_ctl, e->d_hist, e->hist_cap);
        err = cudaGetLastError();
    }
    if (err == cudaSuccess) err = cudaMemcpyAsync(e->h_ctl, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream);
    cudaEventRecord(R.b, e->stream);
    R.launches++;
    if (err != cudaSuccess) return fail(e, TRS_GPU_CUDA, std::string("step loop launch: ") + cudaGetErrorString(err));
    return TRS_GPU_OK;
}

}  // namespace

extern "C" {

int trs_gpu_run_async(trs_gpu_engine* e, const trs_gpu_options* opt_in) {
    if (!e) return TRS_GPU_INVALID;
    if (!e->loaded) return fail(e, TRS_GPU_INVALID, "no store loaded");
    if (e->run.active) return fail(e, TRS_GPU_INVALID, "a run is already pending (trs_gpu_run_wait)");
    cudaSetDevice(e->device);
    // no drain: everything below is ordered on the engine stream
    e->exported = false;
    e->last_error.clear();
    RunState& R = e->run;
    R = RunState{};
    if (opt_in) R.opt = *opt_in;
    e->minb = R.opt.variant == 2 ? 2 : 1;
    e->use_ra = false;  // every run starts in the lean build (but see below)
    e->jit_off = (R.opt.reserved[1] & 2u) != 0;
    // the resident arena costs L1 capacity on every grid sweep: reserve it
    // only for stores small enough to start resident (single-term runs)
    e->resident_on = !(R.opt.reserved[1] & 1u) && resident_slots(e) != 0 && e->input_n <= resident_slots(e) / 2;
    {
        const char* ra = std::getenv("TRS_B200_RUNAHEAD");
        // an explicit budget below the default (sweep_engine.hpp:32) asks for the
        // reference's abort point: no run-ahead then
        const bool budget = R.opt.step_budget != 0 && R.opt.step_budget < 1000000000ull;
        // (8-word records only: the wide-record run-ahead build spills and
        // measured slower than the synchronous one on the sort configs)
        R.runahead = !budget && !R.opt.fixed_capacity && !(R.opt.reserved[1] & 4u) && !(ra && ra[0] == '0') &&
                     R.opt.validate < 2 && (e->W == 8 || (ra && ra[0] == '1'));
    }
    // a program with constant chains starts in the run-ahead build: it takes
    // a chain in registers (transform's leaves) where the lean build would
    // sweep it rewrite by rewrite
    if (R.runahead && e->has_chains) e->use_ra = true;
    // a validating run checks refcounts: a store an untracked run left gets them recounted
    if (R.opt.validate)
        if (int r = ensure_refcounts(e)) return r;
    R.blocks = grid_blocks(e, R.opt.blocks_per_sm);
    if (R.opt.max_blocks && (int)R.opt.max_blocks < R.blocks) R.blocks = (int)R.opt.max_blocks;
    if (!e->h_ctl) CUDA_TRY(e, cudaMallocHost(&e->h_ctl, sizeof(Ctl)));
    if (!e->ev_a) CUDA_TRY(e, cudaEventCreate(&e->ev_a));
    if (!e->ev_b) CUDA_TRY(e, cudaEventCreate(&e->ev_b));
    R.a = e->ev_a;
    R.b = e->ev_b;
    // widths of the last run go; the histogram is all zeros again
    if (e->hist_used)
        CUDA_TRY(e, cudaMemsetAsync(e->d_hist, 0, sizeof(unsigned long long) * e->hist_used, e->stream));
    e->hist_used = 0;
    R.active = true;
    int r = enqueue_launch(e);
    if (r) R.active = false;
    return r;
}

int trs_gpu_run_wait(trs_gpu_engine* e, trs_gpu_stats* stats) {
    if (!e) return TRS_GPU_INVALID;
    RunState& R = e->run;
    if (!R.active) return fail(e, TRS_GPU_INVALID, "no run pending");
    cudaSetDevice(e->device);
    const trs_gpu_options opt = R.opt;
    trs_gpu_stats st{};
    st.grid_blocks = R.blocks;
    st.block_threads = kBlock;
    st.record_words = e->W;
    int result = TRS_GPU_OK;
    const Ctl& c = *e->h_ctl;
    for (;;) {
        cudaError_t err = cudaEventSynchronize(R.b);  // the run's only host synchronisation (per launch)
        if (err != cudaSuccess) {
            result = fail(e, TRS_GPU_CUDA, std::string("step loop: ") + cudaGetErrorString(err));
            break;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, R.a, R.b);
        R.total_ms += ms;
        if (c.status == kDone) break;
        if (c.status == kStepBudget) {
            result = fail(e, TRS_GPU_STEP_BUDGET,
                          "step budget of " + std::to_string(opt.step_budget ? opt.step_budget : 1000000000ull) +
                              " rewrites exceeded; the derivation may not terminate");
            break;
        }
        if (c.status == kCapacity) {
            result = fail(e, TRS_GPU_CAPACITY,
                          "term store capacity " + std::to_string(e->capacity) +
                              " exhausted (fixed capacity; rerun with a larger capacity)");
            break;
        }
        if (c.status == kNeedTrace) {
            int r = TRS_GPU_OK;
            if (c.hist_need > e->hist_cap) {
                // a slot's logical derive sweep lies past the width histogram
                r = grow_hist(e, c.hist_need);
            } else {
                r = grow_trace(e);
            }
            if (!r) r = enqueue_launch(e);
            if (r) { result = r; break; }
            continue;
        }
        if (c.status == kNeedRA) {
            // a latency-bound phase began: continue in the run-ahead build
            e->use_ra = true;
            e->gb_blocks = 0;  // its occupancy may differ
            R.blocks = grid_blocks(e, opt.blocks_per_sm);
            if (opt.max_blocks && (int)opt.max_blocks < R.blocks) R.blocks = (int)opt.max_blocks;
            if (int r = enqueue_launch(e)) {
                result = r;
                break;
            }
            continue;
        }
        if (c.status == kValidate) {
            static const char* kinds[] = {"", "a live slot references slot 0, a slot past the store or a collected slot",
                                          "refcount ghost invariant broken", "nf monotonicity: a slot left normal form",
                                          "inner-most safety: an nf slot has an argument that was not nf before it",
                                          "garbage that is not in normal form", "a live slot is neither on the frontier "
                                          "nor subscribed to an argument"};
            result = fail(e, TRS_GPU_DANGLING, std::string("sweep invariant violation: ") +
                                                   kinds[c.val_kind < 7 ? c.val_kind : 0] + " (slot " +
                                                   std::to_string(c.val_slot) + ")");
            break;
        }
        if (c.status == kNeedGrow) {
            uint64_t m = 0;
            const Ctl cg = c;
            frontier_extent(e, cg, &m);
            st.regrows++;
            int r = grow_store(e, (uint64_t)cg.bump + 2 * m * e->max_new + (uint64_t)R.blocks * kWarps * 256 + (1u << 20));
            if (!r) r = enqueue_launch(e);
            if (r) { result = r; break; }
            continue;
        }
        result = fail(e, TRS_GPU_CUDA, "step loop ended in an unknown state");
        break;
    }
    R.active = false;
    st.launches = R.launches;
    st.total_rewrites = c.total_rewrites;
    st.max_width = c.max_width;
    st.sweeps = c.sweep - c.sweep0;  // logical (finish_run)
    st.gc_runs = c.gc_runs;
    st.small_sweeps = c.small_sweeps;
    st.peak_slots = c.peak_bump;
    st.live_terms = c.bump - 1;
    st.kernel_ms = R.total_ms;
    st.gc_ms = c.gc_ns * 1e-6;
    if (e->load_a && e->load_b && cudaEventElapsedTime(&e->load_ms, e->load_a, e->load_b) == cudaSuccess)
        st.load_ms = e->load_ms;
    cudaGetLastError();
    e->last_sweeps = c.sweep - c.sweep0;
    e->last_psweeps = c.psweep;
    // a completed run rewrote only in sweeps up to its last nf epoch; a run
    // that stopped early (budget, capacity) may have counted rewrites past it
    e->hist_used = result == TRS_GPU_OK ? std::min<uint32_t>(e->hist_cap, e->last_sweeps) : e->hist_cap;
    if (result == TRS_GPU_OK && opt.validate) result = validate_store(e);
    if (stats) *stats = st;
    return result;
}

int trs_gpu_run(trs_gpu_engine* e, const trs_gpu_options* opt, trs_gpu_stats* stats) {
    int r = trs_gpu_run_async(e, opt);
    if (r) return r;
    return trs_gpu_run_wait(e, stats);
}

// Stream gate: the engine stream spins on a host-mapped word until
// trs_gpu_release, so a caller can enqueue a whole step before the device
// starts it (host scheduling noise then stays outside device timings).
__global__ void gate_kernel(volatile uint32_t* flag) {
    uint32_t ns = 64;
    while (*flag == 0u) {
        __nanosleep(ns);
        if (ns < 2048) ns <<= 1;
    }
}

int trs_gpu_hold(trs_gpu_engine* e) {
    if (!e) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    if (!e->h_gate) {
        void* hp = nullptr;
        CUDA_TRY(e, cudaHostAlloc(&hp, sizeof(uint32_t), cudaHostAllocMapped));
        e->h_gate = static_cast<volatile uint32_t*>(hp);
        CUDA_TRY(e, cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->d_gate), (void*)e->h_gate, 0));
    }
    *e->h_gate = 0u;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    gate_kernel<<<1, 1, 0, e->stream>>>(e->d_gate);
    CUDA_TRY(e, cudaGetLastError());
    return TRS_GPU_OK;
}

int trs_gpu_release(trs_gpu_engine* e) {
    if (!e || !e->h_gate) return TRS_GPU_INVALID;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    *e->h_gate = 1u;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    return TRS_GPU_OK;
}

void* trs_gpu_stream(trs_gpu_engine* e) { return e ? (void*)e->stream : nullptr; }

int trs_gpu_profile_counters(trs_gpu_engine* e, uint64_t* out26) {
    if (!e || !e->d_ctl || !out26) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    uint64_t* out12 = out26;
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 12; ++k) out12[k] = c.prof[k];
    for (int k = 0; k < 6; ++k) out12[12 + k] = c.gcprof[k];
    for (int k = 0; k < 8; ++k) out12[18 + k] = c.wmax_sum[k];
    return TRS_GPU_OK;
}

int trs_gpu_compact(trs_gpu_engine* e, uint32_t max_rounds, trs_gpu_stats* stats) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    Ctl c0;
    CUDA_TRY(e, cudaMemcpy(&c0, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    const int blocks = grid_blocks(e, 0);
    // the compaction scatters into the twin arena, where an export stages its columns
    e->exported = false;
    Params P = make_params(e, blocks);
    P.allow_gc = 1;
    P.compact_only = max_rounds ? max_rounds : 8;
    void* args[] = {&P};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, e->stream);
    reset_barrier(e);
    cudaError_t err = cudaLaunchCooperativeKernel(loop_kernel(e), blocks, kBlock, args, dyn_smem(e), e->stream);
    cudaEventRecord(b, e->stream);
    if (err == cudaSuccess) err = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (err != cudaSuccess) return fail(e, TRS_GPU_CUDA, std::string("compaction: ") + cudaGetErrorString(err));
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->gc_runs = c.gc_runs - c0.gc_runs;
        stats->gc_ms = (c.gc_ns - c0.gc_ns) * 1e-6;
        stats->kernel_ms = ms;
        stats->launches = 1;
        stats->live_terms = c.bump - 1;
        stats->peak_slots = c.bump;
        stats->grid_blocks = blocks;
        stats->block_threads = kBlock;
        stats->record_words = e->W;
    }
    return TRS_GPU_OK;
}

int trs_gpu_overhead_probe(trs_gpu_engine* e, uint32_t iters, uint32_t mode, uint32_t max_blocks, double* ns_per_iter) {
    if (!e || !e->loaded || !ns_per_iter) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    int blocks = grid_blocks(e, 0);
    if (max_blocks && (int)max_blocks < blocks) blocks = (int)max_blocks;
    Params P = make_params(e, blocks);
    P.probe_iters = iters ? iters : 1000;
    P.probe_mode = mode;
    void* args[] = {&P};
    reset_barrier(e);
    cudaError_t err = cudaLaunchCooperativeKernel(loop_kernel(e), blocks, kBlock, args, dyn_smem(e), e->stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize(e->stream);
    if (err != cudaSuccess) return fail(e, TRS_GPU_CUDA, std::string("probe: ") + cudaGetErrorString(err));
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    *ns_per_iter = (double)c.gc_ns / P.probe_iters;
    return TRS_GPU_OK;
}

int trs_gpu_fetch_records(trs_gpu_engine* e, void* dst, uint64_t cap_bytes, uint64_t* bytes, uint32_t* record_words,
                          uint32_t* roots_out) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    Ctl c;
    CUDA_TRY(e, cudaMemcpyAsync(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    uint64_t need = (uint64_t)c.bump * e->W * 4;
    if (bytes) *bytes = need;
    if (record_words) *record_words = (uint32_t)e->W;
    if (!dst || cap_bytes < need) return TRS_GPU_OK;
    if (int r = ensure_refcounts(e)) return r;  // the records' refcount words as the reference keeps them
    CUDA_TRY(e, cudaMemcpyAsync(dst, e->d_arena[c.arena], need, cudaMemcpyDeviceToHost, e->stream));
    if (roots_out)
        CUDA_TRY(e, cudaMemcpyAsync(roots_out, e->d_roots, sizeof(uint32_t) * e->num_roots, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    return TRS_GPU_OK;
}

int trs_gpu_trace(trs_gpu_engine* e, trs_gpu_sweep_record* out, uint64_t cap, uint64_t* count) {
    if (!e || !e->d_trace) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    // one record per logical sweep: rewrites = the width (hist); the run's
    // last sweep is the empty one that ends it (sweep_engine.cpp:147)
    const uint64_t n = e->last_sweeps;
    if (count) *count = n;
    if (!out || !cap) return TRS_GPU_OK;
    const uint64_t k = std::min(n, cap);
    std::vector<unsigned long long> h(std::max<uint64_t>(1, k), 0ull);
    const uint64_t have = std::min<uint64_t>(k, e->hist_cap);
    if (have) CUDA_TRY(e, cudaMemcpy(h.data(), e->d_hist, sizeof(unsigned long long) * have, cudaMemcpyDeviceToHost));
    for (uint64_t j = 0; j < k; ++j) {
        trs_gpu_sweep_record r{};
        r.sweep = (uint32_t)(j + 1);
        r.rewrites = h[j];
        out[j] = r;
    }
    return TRS_GPU_OK;
}

int trs_gpu_phys_trace(trs_gpu_engine* e, trs_gpu_sweep_record* out, uint64_t cap, uint64_t* count) {
    if (!e || !e->d_trace) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    uint64_t n = std::min<uint64_t>(e->last_psweeps, e->trace_cap);
    if (count) *count = n;
    if (out && cap)
        CUDA_TRY(e, cudaMemcpy(out, e->d_trace, sizeof(trs_gpu_sweep_record) * std::min(n, cap), cudaMemcpyDeviceToHost));
    return TRS_GPU_OK;
}

int trs_gpu_canonical(trs_gpu_engine* e, uint32_t root_index, uint32_t* words, uint64_t cap, uint64_t* n_words,
                      uint32_t* n_nodes) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    if (root_index >= e->num_roots) return fail(e, TRS_GPU_INVALID, "root index out of range");
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    if (int r = run_canon(e)) return r;
    unsigned long long off[2];
    uint32_t nodes = 0;
    CUDA_TRY(e, cudaMemcpy(off, e->d_woff + root_index, sizeof(off), cudaMemcpyDeviceToHost));
    CUDA_TRY(e, cudaMemcpy(&nodes, e->d_nodes + root_index, sizeof(nodes), cudaMemcpyDeviceToHost));
    const uint64_t nw = off[1] - off[0];
    if (n_words) *n_words = nw;
    if (n_nodes) *n_nodes = nodes;
    if (!words || cap < nw) return TRS_GPU_OK;
    CUDA_TRY(e, cudaMemcpy(words, e->d_words + off[0], sizeof(uint32_t) * nw, cudaMemcpyDeviceToHost));
    return TRS_GPU_OK;
}

}  // extern "C"

namespace {

template <int W>
const void* export_ptr() {
    return reinterpret_cast<const void*>(&export_store<W>);
}

// Staging layout of an export in the twin arena (bump = slots scanned):
// hss [bump] | rcs [bump] | args [ma * n] | nf [bump] bytes.
struct ExportStaging {
    uint32_t* hss;
    uint32_t* rcs;
    uint32_t* args;
    uint8_t* nf;
};

ExportStaging export_staging(trs_gpu_engine* e, const Ctl& c) {
    ExportStaging st;
    st.hss = e->d_arena[c.arena ^ 1];
    st.rcs = st.hss + c.bump;
    st.args = st.rcs + c.bump;
    st.nf = reinterpret_cast<uint8_t*>(st.args + (size_t)e->max_arity * c.bump);
    return st;
}

ExportArgs export_args(trs_gpu_engine* e, const Ctl& c) {
    ExportArgs X{};
    uint32_t* scratch = e->d_list[c.cur ^ 1];  // the frontier lives in list[c.cur]
    for (int k = 0; k < 3; ++k) X.queue[k] = scratch + (size_t)k * c.bump;
    X.map = scratch + (((size_t)c.bump + 3) & ~(size_t)3);  // 16-byte aligned (export.cuh stores quads); queue[1] unused
    X.newrc = e->d_gcmap;
    X.counters = e->d_blocksum + kMaxGrid;
    const ExportStaging st = export_staging(e, c);
    X.hss = st.hss;
    X.rcs = st.rcs;
    X.args = st.args;
    X.nf = st.nf;
    X.roots_out = e->d_roots_out;
    X.ma = e->max_arity;
    return X;
}

// Mark from the roots, recount references and renumber (export.cuh); the
// columns are packed later, range by range (pack_export).
int run_export(trs_gpu_engine* e, Ctl& c) {
    CUDA_TRY(e, cudaMemcpyAsync(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    const void* fn = e->W == 8 ? export_ptr<8>() : e->W == 16 ? export_ptr<16>() : export_ptr<32>();
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, 0) != cudaSuccess || occ < 1) occ = 1;
    const int blocks = std::min<int>(occ * e->sm_count, (int)kMaxGrid);
    Params P = make_params(e, blocks);
    ExportArgs X = export_args(e, c);
    uint32_t bump = c.bump;
    void* args[] = {&P, &X, &bump};
    CUDA_TRY(e, cudaMemsetAsync(X.counters, 0, sizeof(uint32_t) * 4, e->stream));
    CUDA_TRY(e, cudaMemsetAsync(X.queue[0], 0, sizeof(uint32_t) * c.bump, e->stream));
    reset_barrier(e);
    CUDA_TRY(e, cudaLaunchCooperativeKernel(fn, blocks, kBlock, args, 0, e->stream));
    uint32_t dangling = 0;
    e->export_cta_live.assign(blocks, 0u);
    e->export_blocks = (uint32_t)blocks;
    CUDA_TRY(e, cudaMemcpyAsync(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(&dangling, X.counters + 3, sizeof(uint32_t), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(e->export_cta_live.data(), e->d_blocksum, sizeof(uint32_t) * blocks,
                                cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    if (dangling) {
        e->exported = false;
        return fail(e, TRS_GPU_DANGLING,
                    dangling == 0xFFFFFFFFu ? std::string("a live term references slot 0 or a slot past the store")
                                            : "slot " + std::to_string(dangling) + " is not a live term");
    }
    e->exported = true;
    e->packed = false;
    e->canon_ready = false;
    e->export_ctl = c;
    return TRS_GPU_OK;
}

template <int W>
void launch_pack(trs_gpu_engine* e, const ExportArgs& X, uint32_t n, const uint8_t* arity, uint32_t lo, uint32_t hi) {
    const uint32_t A_idx = e->export_ctl.arena;
    const int grid = std::max(1, std::min<int>(e->sm_count * 4, (int)(((hi - lo) / 8 + kBlock - 1) / kBlock)));
    pack_range<W><<<grid, kBlock, 0, e->stream>>>(e->d_arena[A_idx], X, n, arity, lo, hi);
}

// Pack the exported columns, in up to 8 slot ranges; with host buffers, each
// range's rows (contiguous: renumbering keeps arena order) are copied out on
// a second stream while the next range packs.
struct HostColumns {
    uint32_t* hss;
    uint32_t* args;
    uint32_t* rcs;
    uint8_t* nf;
};

int pack_export(trs_gpu_engine* e, const HostColumns* host) {
    const Ctl& c = e->export_ctl;
    const uint32_t n = c.export_n, bump = c.bump, ma = e->max_arity;
    const ExportArgs X = export_args(e, c);
    const uint8_t* arity = e->d_prog + reinterpret_cast<const ProgHeader*>(e->blob.data())->off_arity;
    if (!e->stream2) CUDA_TRY(e, cudaStreamCreateWithFlags(&e->stream2, cudaStreamNonBlocking));
    const uint32_t B = std::max(1u, e->export_blocks);
    // the export kernel renumbered CTA b's 8-slot groups [b * gchunk, (b + 1) * gchunk)
    const uint32_t ngroups = (bump + 7) / 8, gchunk = (ngroups + B - 1) / B;
    const uint32_t G = std::min<uint32_t>(8, B);
    uint32_t row = 1;  // row 0 is slot 0 (zeros, written by the export kernel)
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t b0 = g * B / G, b1 = (g + 1) * B / G;
        const uint32_t lo = std::max<uint64_t>(1, std::min<uint64_t>(bump, 8ull * b0 * gchunk));
        const uint32_t hi = std::min<uint64_t>(bump, 8ull * b1 * gchunk);
        uint32_t rows = 0;
        for (uint32_t b = b0; b < b1; ++b) rows += e->export_cta_live[b];
        if (hi > lo) {
            switch (e->W) {
                case 8: launch_pack<8>(e, X, n, arity, lo, hi); break;
                case 16: launch_pack<16>(e, X, n, arity, lo, hi); break;
                default: launch_pack<32>(e, X, n, arity, lo, hi); break;
            }
        }
        if (host) {
            if (!e->pack_ev[g]) CUDA_TRY(e, cudaEventCreateWithFlags(&e->pack_ev[g], cudaEventDisableTiming));
            CUDA_TRY(e, cudaEventRecord(e->pack_ev[g], e->stream));
            CUDA_TRY(e, cudaStreamWaitEvent(e->stream2, e->pack_ev[g], 0));
            // this range's rows, plus row 0 with the first range
            const uint32_t r0 = g == 0 ? 0 : row, r1 = row + rows;
            if (r1 > r0) {
                const size_t k = r1 - r0;
                CUDA_TRY(e, cudaMemcpyAsync(host->hss + r0, X.hss + r0, 4 * k, cudaMemcpyDeviceToHost, e->stream2));
                if (host->rcs)
                    CUDA_TRY(e, cudaMemcpyAsync(host->rcs + r0, X.rcs + r0, 4 * k, cudaMemcpyDeviceToHost, e->stream2));
                if (host->nf) CUDA_TRY(e, cudaMemcpyAsync(host->nf + r0, X.nf + r0, k, cudaMemcpyDeviceToHost, e->stream2));
                if (host->args && ma)
                    CUDA_TRY(e, cudaMemcpy2DAsync(host->args + r0, 4 * (size_t)n, X.args + r0, 4 * (size_t)n, 4 * k, ma,
                                                  cudaMemcpyDeviceToHost, e->stream2));
            }
        }
        row += rows;
    }
    if (row != n) return fail(e, TRS_GPU_CUDA, "export: renumbering ranges do not cover the exported rows");
    if (host) CUDA_TRY(e, cudaStreamSynchronize(e->stream2));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    CUDA_TRY(e, cudaGetLastError());
    e->packed = true;
    return TRS_GPU_OK;
}

// Canonical words of every root from the export staging (canon.cuh); the
// result stays on the device until the store changes.
int run_canon(trs_gpu_engine* e) {
    if (e->roots_out_cap < e->num_roots) {
        cudaFree(e->d_roots_out);
        CUDA_TRY(e, cudaMalloc(&e->d_roots_out, sizeof(uint32_t) * e->num_roots));
        e->roots_out_cap = e->num_roots;
        e->exported = false;
    }
    if (!e->exported) {
        Ctl c;
        if (int r = run_export(e, c)) return r;
    }
    if (e->canon_ready) return TRS_GPU_OK;
    if (!e->packed)
        if (int r = pack_export(e, nullptr)) return r;
    const Ctl& c = e->export_ctl;
    const uint32_t n = c.export_n;
    const uint32_t ma = e->max_arity;
    const uint32_t R = e->num_roots;
    if ((uint64_t)n * (1 + ma) >= 0xFFFFFFFFull) return fail(e, TRS_GPU_INVALID, "normal forms beyond 2^32 words");
    const size_t need = (size_t)n * 8 + (size_t)ma * n + R + 8;
    if (e->canon_words_cap < need) {
        cudaFree(e->d_canon);
        e->d_canon = nullptr;
        e->canon_words_cap = 0;
        CUDA_TRY(e, cudaMalloc(&e->d_canon, sizeof(uint32_t) * need));
        e->canon_words_cap = need;
    }
    const size_t wneed = (size_t)n * (1 + ma) + 1;
    if (e->words_cap < wneed) {
        cudaFree(e->d_words);
        e->d_words = nullptr;
        e->words_cap = 0;
        CUDA_TRY(e, cudaMalloc(&e->d_words, sizeof(uint32_t) * wneed));
        e->words_cap = wneed;
    }
    if (e->canon_roots_cap < R) {
        cudaFree(e->d_woff);
        cudaFree(e->d_nodes);
        e->d_woff = nullptr;
        e->d_nodes = nullptr;
        e->canon_roots_cap = 0;
        CUDA_TRY(e, cudaMalloc(&e->d_woff, sizeof(unsigned long long) * (2 * (size_t)R + 1)));
        CUDA_TRY(e, cudaMalloc(&e->d_nodes, sizeof(uint32_t) * R));
        e->canon_roots_cap = R;
    }
    const ExportStaging st = export_staging(e, c);
    CanonArgs X{};
    X.hss = st.hss;
    X.args = st.args;
    X.rcs = st.rcs;
    X.roots = e->d_roots_out;
    X.num_roots = R;
    X.n = n;
    X.ma = ma;
    X.arity = e->d_prog + reinterpret_cast<const ProgHeader*>(e->blob.data())->off_arity;
    uint32_t* s = e->d_canon;
    X.par = s;
    X.size = s + (size_t)n;
    X.wsz = s + 2 * (size_t)n;
    X.pending = s + 3 * (size_t)n;
    X.id = s + 4 * (size_t)n;
    X.wpos = s + 5 * (size_t)n;
    X.rootof = s + 6 * (size_t)n;
    X.queue = s + 7 * (size_t)n;
    X.counters = s + 8 * (size_t)n;
    X.stack = X.counters + 8;
    X.nodes = e->d_nodes;
    X.woff = e->d_woff;
    X.hash = e->d_woff + R + 1;
    X.words = e->d_words;
    const int blocks = e->sm_count * 4;
    CUDA_TRY(e, cudaMemsetAsync(X.counters, 0, sizeof(uint32_t) * 8, e->stream));
    CUDA_TRY(e, cudaMemsetAsync(X.par, 0, sizeof(uint32_t) * n, e->stream));
    CUDA_TRY(e, cudaMemsetAsync(X.queue, 0, sizeof(uint32_t) * n, e->stream));
    canon_init<<<blocks, 256, 0, e->stream>>>(X);
    uint32_t shared = 0;
    CUDA_TRY(e, cudaMemcpyAsync(&shared, X.counters + 3, sizeof(uint32_t), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    if (shared) {
        // sharing: the reference's sequential stack walk (canon_seq)
        CUDA_TRY(e, cudaMemsetAsync(X.par, 0, sizeof(uint32_t) * n, e->stream));
        canon_seq<<<1, 32, 0, e->stream>>>(X);
    } else {
        canon_up<<<blocks, 256, 0, e->stream>>>(X);
        canon_offsets<<<1, kBlock, 0, e->stream>>>(X);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, canon_down, kBlock, 0) != cudaSuccess || occ < 1) occ = 1;
        const int dblocks = std::min<int>(occ * e->sm_count, 1024);
        void* kargs[] = {&X};
        CUDA_TRY(e, cudaLaunchCooperativeKernel((const void*)canon_down, dblocks, kBlock, kargs, 0, e->stream));
    }
    unsigned long long total = 0;
    CUDA_TRY(e, cudaMemcpyAsync(&total, e->d_woff + R, sizeof(total), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    CUDA_TRY(e, cudaGetLastError());
    e->canon_total = total;
    e->canon_ready = true;
    return TRS_GPU_OK;
}

}  // namespace

extern "C" {

int trs_gpu_fetch_store(trs_gpu_engine* e, uint32_t* n, uint32_t* roots_out, uint32_t* hss, uint32_t* args,
                        uint32_t* refcounts, uint8_t* nf, uint32_t cap) {
    if (!e || !e->loaded || !n) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (e->roots_out_cap < e->num_roots) {
        cudaFree(e->d_roots_out);
        CUDA_TRY(e, cudaMalloc(&e->d_roots_out, sizeof(uint32_t) * e->num_roots));
        e->roots_out_cap = e->num_roots;
    }
    if (!e->exported) {
        Ctl c;
        if (int r = run_export(e, c)) return r;
    }
    const Ctl& c = e->export_ctl;
    const uint32_t N = c.export_n;
    *n = N;
    if (!hss) return TRS_GPU_OK;
    if (cap < N) return fail(e, TRS_GPU_INVALID, "fetch buffer too small");
    if (!e->packed) {
        // pack range by range, each range's rows copied out while the next packs
        const HostColumns host{hss, args, refcounts, nf};
        if (int r = pack_export(e, &host)) return r;
        if (roots_out)
            CUDA_TRY(e, cudaMemcpyAsync(roots_out, e->d_roots_out, sizeof(uint32_t) * e->num_roots,
                                        cudaMemcpyDeviceToHost, e->stream));
        CUDA_TRY(e, cudaStreamSynchronize(e->stream));
        return TRS_GPU_OK;
    }
    const ExportStaging st = export_staging(e, c);
    const uint32_t ma = e->max_arity;
    CUDA_TRY(e, cudaMemcpyAsync(hss, st.hss, sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, e->stream));
    if (refcounts) CUDA_TRY(e, cudaMemcpyAsync(refcounts, st.rcs, sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, e->stream));
    if (args && ma)
        CUDA_TRY(e, cudaMemcpyAsync(args, st.args, sizeof(uint32_t) * ma * (size_t)N, cudaMemcpyDeviceToHost, e->stream));
    if (nf) CUDA_TRY(e, cudaMemcpyAsync(nf, st.nf, N, cudaMemcpyDeviceToHost, e->stream));
    if (roots_out)
        CUDA_TRY(e, cudaMemcpyAsync(roots_out, e->d_roots_out, sizeof(uint32_t) * e->num_roots, cudaMemcpyDeviceToHost,
                                    e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    return TRS_GPU_OK;
}

int trs_gpu_dump_program(trs_gpu_engine* e, const char* const* symbol_names, const char* const* var_names,
                         const uint32_t* rule_var_begin, const uint32_t* rule_vars, const char* const* rule_texts,
                         char* out, uint64_t cap, uint64_t* need) {
    if (!e || !e->d_prog || !symbol_names || !var_names || !rule_var_begin || !rule_vars || !rule_texts || !need)
        return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    // render what the device holds, not the host copy
    std::vector<uint8_t> blob(e->blob.size());
    CUDA_TRY(e, cudaMemcpy(blob.data(), e->d_prog, blob.size(), cudaMemcpyDeviceToHost));
    const ProgHeader* h = reinterpret_cast<const ProgHeader*>(blob.data());
    const uint8_t* arity = blob.data() + h->off_arity;
    const uint16_t* rule_begin = reinterpret_cast<const uint16_t*>(blob.data() + h->off_rule_begin);
    const DRule* rules = reinterpret_cast<const DRule*>(blob.data() + h->off_rules);
    const DStep* steps = reinterpret_cast<const DStep*>(blob.data() + h->off_steps);
    const DInstr* instrs = reinterpret_cast<const DInstr*>(blob.data() + h->off_instrs);
    const uint16_t* refs = reinterpret_cast<const uint16_t*>(blob.data() + h->off_refs);
    // the reference's dump format (dispatch.cpp:98-134)
    std::string o;
    for (uint32_t f = 0; f < h->num_symbols; ++f) {
        const uint32_t r0 = rule_begin[f], r1 = rule_begin[f + 1];
        if (r0 == r1) continue;
        o += std::string("symbol ") + symbol_names[f] + "/" + std::to_string(arity[f]) + ": " +
             std::to_string(r1 - r0) + " rule(s)\n";
        for (uint32_t r = r0; r < r1; ++r) {
            const DRule& R = rules[r];
            const uint32_t src = e->rule_source[r];
            o += "  rule #" + std::to_string(src) + ": " + rule_texts[src] + "\n";
            auto var_of = [&](uint32_t slot) { return std::string(var_names[rule_vars[rule_var_begin[r] + slot]]); };
            std::vector<std::string> path(R.num_steps);
            for (uint32_t t = 0; t < R.num_steps; ++t) {
                const DStep& S = steps[R.first_step + t];
                const std::string up = S.parent < 0 ? std::string() : path[S.parent];
                path[t] = up.empty() ? std::to_string(S.child) : up + "." + std::to_string(S.child);
                if (S.kind == TRS_GPU_STEP_CHECK_HEAD)
                    o += "    check [" + path[t] + "] = " + symbol_names[S.value] + "\n";
                else
                    o += "    bind  [" + path[t] + "] -> " + var_of(S.value) + "\n";
            }
            for (uint32_t k = 0; k < R.num_instrs; ++k) {
                const DInstr& I = instrs[R.first_instr + k];
                const bool is_root = !R.collapse && k + 1 == R.num_instrs;
                o += is_root ? "    root  " : "    new   ";
                o += "n" + std::to_string(k) + " = " + symbol_names[I.symbol] + "(";
                for (uint32_t j = 0; j < arity[I.symbol]; ++j) {
                    if (j) o += ", ";
                    const uint16_t ref = refs[I.first_ref + j];
                    o += (ref & kRefNode) ? "n" + std::to_string(ref & 0x7fff) : var_of(ref);
                }
                o += ")\n";
            }
            if (R.collapse) o += "    root  reuse " + var_of(R.root_ref) + "\n";
        }
    }
    *need = o.size() + 1;
    if (out && cap >= o.size() + 1) std::memcpy(out, o.c_str(), o.size() + 1);
    return TRS_GPU_OK;
}

int trs_gpu_canonical_all(trs_gpu_engine* e, uint32_t* words, uint64_t cap, uint64_t* n_words,
                          uint64_t* root_offsets, uint64_t* hashes, uint32_t* root_nodes) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    if (int r = run_canon(e)) return r;
    const uint32_t R = e->num_roots;
    if (n_words) *n_words = e->canon_total;
    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "u64");
    if (root_offsets) CUDA_TRY(e, cudaMemcpy(root_offsets, e->d_woff, sizeof(uint64_t) * (R + 1), cudaMemcpyDeviceToHost));
    if (hashes) CUDA_TRY(e, cudaMemcpy(hashes, e->d_woff + R + 1, sizeof(uint64_t) * R, cudaMemcpyDeviceToHost));
    if (root_nodes) CUDA_TRY(e, cudaMemcpy(root_nodes, e->d_nodes, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost));
    if (words && cap >= e->canon_total)
        CUDA_TRY(e, cudaMemcpy(words, e->d_words, sizeof(uint32_t) * e->canon_total, cudaMemcpyDeviceToHost));
    return TRS_GPU_OK;
}

int trs_gpu_layout_probe(trs_gpu_engine* e, uint32_t layout, uint32_t iters, double* ms_per_pass, uint64_t* nodes) {
    if (!e || !e->loaded || !ms_per_pass || layout > 3) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    if (e->W != 8) return fail(e, TRS_GPU_INVALID, "layout probe: 8-word records only");
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    const uint32_t n = c.bump;
    const uint32_t na = std::min<uint32_t>(e->max_arity, 4);
    const uint32_t* A = e->d_arena[c.arena];
    const uint8_t* arity = e->d_prog + reinterpret_cast<const ProgHeader*>(e->blob.data())->off_arity;
    uint32_t* soa = nullptr;
    uint32_t* sink = nullptr;
    CUDA_TRY(e, cudaMalloc(&sink, 4));
    const bool soa_layout = layout & 1u, random_order = layout & 2u;
    if (soa_layout) {
        CUDA_TRY(e, cudaMalloc(&soa, sizeof(uint32_t) * (size_t)n * (2 + na)));
        to_soa<8><<<e->sm_count * 8, 256, 0, e->stream>>>(A, n, soa, soa + n, soa + 2 * (size_t)n, na);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto pass = [&]() {
        if (!soa_layout)
            probe_aos<8><<<e->sm_count * 8, 256, 0, e->stream>>>(A, n, arity, sink, random_order);
        else
            probe_soa<<<e->sm_count * 8, 256, 0, e->stream>>>(soa, soa + n, soa + 2 * (size_t)n, n, na, arity, sink,
                                                              random_order);
    };
    pass();  // warm-up
    cudaEventRecord(a, e->stream);
    for (uint32_t k = 0; k < std::max(1u, iters); ++k) pass();
    cudaEventRecord(b, e->stream);
    cudaError_t err = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(soa);
    cudaFree(sink);
    if (err != cudaSuccess) return fail(e, TRS_GPU_CUDA, std::string("layout probe: ") + cudaGetErrorString(err));
    *ms_per_pass = ms / std::max(1u, iters);
    if (nodes) *nodes = n;
    return TRS_GPU_OK;
}

int trs_gpu_live_count(trs_gpu_engine* e, uint64_t* live) {
    if (!e || !e->loaded || !live) return TRS_GPU_INVALID;
    REFUSE_PENDING(e);
    cudaSetDevice(e->device);
    if (int r = drain(e)) return r;
    if (int r = ensure_refcounts(e)) return r;
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    unsigned long long* d = reinterpret_cast<unsigned long long*>(e->d_blocksum + kMaxGrid);  // scratch words
    CUDA_TRY(e, cudaMemsetAsync(d, 0, sizeof(*d), e->stream));
    const uint32_t* A = e->d_arena[c.arena];
    const int blocks = e->sm_count * 8;
    switch (e->W) {
        case 8: count_live<8><<<blocks, 256, 0, e->stream>>>(A, c.bump, d); break;
        case 16: count_live<16><<<blocks, 256, 0, e->stream>>>(A, c.bump, d); break;
        default: count_live<32><<<blocks, 256, 0, e->stream>>>(A, c.bump, d); break;
    }
    unsigned long long v = 0;
    CUDA_TRY(e, cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    *live = v;
    return TRS_GPU_OK;
}

}  // extern "C"

namespace {

template <int ILP>
void launch_probe(uint32_t vec, int grid, const uint32_t* data, uint64_t mask, const uint32_t* idx, uint32_t n,
                  uint32_t* sink) {
    switch (vec) {
        case 1: gather_probe_kernel<1, ILP><<<grid, 512>>>(data, mask, idx, n, sink); break;
        case 2: gather_probe_kernel<2, ILP><<<grid, 512>>>(data, mask, idx, n, sink); break;
        case 4: gather_probe_kernel<4, ILP><<<grid, 512>>>(data, mask, idx, n, sink); break;
        default: gather_probe_kernel<8, ILP><<<grid, 512>>>(data, mask, idx, n, sink); break;
    }
}

}  // namespace

extern "C" {

int trs_gpu_gather_probe_ex(int device, uint64_t bytes, uint32_t bytes_per_access, uint32_t ilp, uint32_t iters,
                            double* gbps) {
    if (!gbps || (bytes_per_access != 4 && bytes_per_access != 8 && bytes_per_access != 16 && bytes_per_access != 32))
        return TRS_GPU_INVALID;
    if (ilp != 1 && ilp != 2 && ilp != 4 && ilp != 8 && ilp != 16) return TRS_GPU_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return TRS_GPU_CUDA;
    uint64_t words = 1;
    while (words * 2 <= bytes / 4) words *= 2;  // power of two: addressing is a mask
    const uint32_t n = 1u << 28;                // accesses per launch
    uint32_t *data = nullptr, *idx = nullptr, *sink = nullptr;
    if (cudaMalloc(&data, words * 4) != cudaSuccess) return TRS_GPU_CUDA;
    if (cudaMalloc(&idx, (size_t)n * 4) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) {
        cudaFree(data);
        cudaFree(idx);
        return TRS_GPU_CUDA;
    }
    cudaMemset(data, 1, words * 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    fill_random<<<sms * 8, 256>>>(idx, n, 12345);
    const uint32_t vec = bytes_per_access / 4;
    const uint64_t mask = (words - 1) & ~(uint64_t)(vec - 1);
    auto launch = [&]() {
        const int grid = sms * 4;  // 4 x 512 threads = a full SM
        switch (ilp) {
            case 1: launch_probe<1>(vec, grid, data, mask, idx, n, sink); break;
            case 2: launch_probe<2>(vec, grid, data, mask, idx, n, sink); break;
            case 4: launch_probe<4>(vec, grid, data, mask, idx, n, sink); break;
            case 8: launch_probe<8>(vec, grid, data, mask, idx, n, sink); break;
            default: launch_probe<16>(vec, grid, data, mask, idx, n, sink); break;
        }
    };
    launch();  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (uint32_t k = 0; k < iters; ++k) launch();
    cudaEventRecord(b);
    cudaError_t err = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(data);
    cudaFree(idx);
    cudaFree(sink);
    if (err != cudaSuccess) return TRS_GPU_CUDA;
    *gbps = (double)n * iters * bytes_per_access / (ms * 1e-3) / 1e9;
    return TRS_GPU_OK;
}

int trs_gpu_gather_probe(int device, uint64_t bytes, uint32_t bytes_per_access, uint32_t iters, double* gbps) {
    return trs_gpu_gather_probe_ex(device, bytes, bytes_per_access, 4, iters, gbps);
}

}  // extern "C"

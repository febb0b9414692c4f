// Device-side building blocks shared by the step loop and the collector:
// control block, launch parameters, grid barrier, block scans, record access.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device_program.hpp"
#include "trs_gpu.h"

#ifndef TRS_B200_PROFILE
#define TRS_B200_PROFILE 0
#endif

namespace trs_b200 {

constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;
constexpr uint32_t kMaxGrid = 1024;    // CTAs; sizes the frontier region tables
constexpr uint32_t kSmallCap = 4096;   // frontier entries per shared-memory list (single-CTA mode)

// Sweep outcome flags, raised by lanes in a CTA-shared word and published
// with the CTA's frontier region, so every CTA reads the same set after the
// grid barrier (a global sticky word could be raised by the next sweep of a
// fast CTA before a slow one has read it).
constexpr uint32_t kFlagCapacity = 1;  // a claim did not fit a fixed capacity
constexpr uint32_t kFlagHist = 2;      // a derive sweep lies past the width histogram

enum Status : uint32_t {
    kRunning = 0,
    kDone = 1,
    kStepBudget = 2,
    kCapacity = 3,
    kNeedGrow = 4,
    kNeedTrace = 5,
    kValidate = 6,   // a validate=2 scan found a violation (Ctl::val_kind)
    kNeedRA = 7,     // the lean build hands over to the run-ahead build
};

// Control block in device memory.  Persistent fields are written by one
// thread at quiescent points only (kernel exit, single-CTA hand-back, end of
// a collection); every CTA keeps an identical private copy (Local) in
// between, so no CTA ever needs a fresh read of shared bookkeeping to decide
// what the grid does next.
struct Ctl {
    uint32_t sweep;           // completed sweeps
    uint32_t cur;             // frontier list buffer of the next sweep
    uint32_t arena;           // current arena buffer
    uint32_t status;
    uint32_t gc_runs;
    uint32_t small_sweeps;
    uint32_t last_gc_sweep;
    uint32_t abort_capacity;  // a claim did not fit a fixed capacity
    unsigned long long total_rewrites;
    unsigned long long max_width;
    unsigned long long gc_ns;
    uint32_t peak_bump;
    uint32_t sweep0;          // sweeps completed before this run (epochs keep counting)
    // allocator: slots [0, bump) are handed out (in per-warp slabs)
    uint32_t bump;
    // grid barrier: monotonic arrival counter, zeroed by the host per launch
    uint32_t bar_arrive;
    // frontier layout: list buffer b holds nregions[b] regions whose
    // (offset, count) pairs live in Params::regions
    uint32_t nregions[2];
    // a collection left a refcount cascade unfinished (hop cap): garbage remains
    uint32_t gc_truncated;
    uint32_t export_n;        // slots of the last export (export.cuh)
    // logical time: `sweep` is the logical sweep count (epochs) at the end of
    // a run; `psweep` counts the physical sweeps (loop iterations) of the run,
    // `tmax` the latest nf epoch so far; widths live in Params::hist
    uint32_t psweep;
    uint32_t tmax;
    uint32_t need_hist;       // a slot's derive sweep lies past the width histogram
    uint32_t hist_need;       // the histogram entries it needs
    uint32_t ra_narrow, ra_on, ra_used;  // run-ahead state (sweep.cuh, ra_track)
    uint32_t ra_mref, ra_sref, ra_go;    // shrinking-phase window (sweep.cuh, ra_track)
    uint32_t val_kind, val_slot;         // first validate=2 violation (validate.cuh)
    // phase cycle accounting (Params::profile): match, claim, apply, push,
    // sweep, sweeps, warp steps (chunks) of the profiled warp, spare, then
    // the match sub-phases: record, children, slots, rules
    unsigned long long prof[12];
    // profiling build: collection phase ns (claim, count, scatter, remap),
    // cascade hops, longest cascade
    unsigned long long gcprof[6];
    // profiling build: per-sweep maxima over warps of the warp-step phases
    // (match, claim, apply, push, record, children, slots, rules), rotating
    // slots, and their sums over the profiled sweeps
    unsigned long long wmax[2][8];
    unsigned long long wmax_sum[8];
};

struct Params {
    uint32_t* arena[2];
    uint32_t* list[2];
    uint32_t* gcmap;
    uint32_t* blocksum;
    uint32_t* regions;               // [2 buffers][off | cnt][kMaxGrid]
    uint32_t* region_flags;          // [2 buffers][kMaxGrid] kFlag* raised by the sweep that wrote the buffer
    unsigned long long* region_rew;  // [2 buffers][kMaxGrid] rewrites of the sweep that wrote the buffer
    uint32_t* roots;
    uint32_t num_roots;
    Ctl* ctl;
    trs_gpu_sweep_record* trace;
    uint32_t trace_cap;
    const uint8_t* prog;  // blob in global memory
    uint32_t prog_bytes;
    uint64_t capacity;  // logical slots per arena
    uint64_t step_budget;
    uint32_t small_enter, small_exit;
    uint32_t warp_mode;  // tiny frontiers run on one warp
    uint32_t gc_interval;
    uint32_t allow_gc;
    uint32_t fixed_capacity;
    uint32_t max_new;
    uint32_t compact_only;  // >0: run at most this many compaction rounds and exit
    uint32_t prefer_grow;   // out of headroom: grow (host) rather than collect
    uint32_t profile;       // phase cycle accounting of CTA 0 (debug): 1 every sweep, >1 grid sweeps of <= profile entries
    uint32_t slab;          // fresh slots a warp claims at a time
    uint32_t probe_iters;   // >0: time this many grid barriers and exit (trs_gpu_overhead_probe)
    uint32_t probe_mode;
    uint32_t rich;          // grid frontier entries carry record payloads (W words) instead of bare slots
    uint32_t local_cap;     // >0: slots of the shared-memory resident arena of the single-CTA mode
    uint32_t local_enter;   // allocated slots at or below which the single-CTA mode goes resident
    uint32_t max_vars;      // binding columns in shared memory (largest rule's variable count)
    unsigned long long* hist;  // per logical sweep (from sweep0 + 1): rewrites (the reference's widths)
    uint32_t hist_cap;
    uint32_t runahead;      // lanes continue into slots their step made ready (logical time)
    uint32_t ra_max;        // ... in sweeps of at most this many frontier entries
    uint32_t ra_kill;       // a sweep wider than this switches run-ahead off (Local::ra_on)
    uint32_t ra_warm;       // consecutive sweeps no wider than ra_kill switch it on
    uint32_t ra_steps;      // consecutive run-ahead steps of a lane before it pushes instead (a long
                            // chain must not hold back the work its steps pushed to the next sweep)
    uint64_t list_cap;      // entries per frontier list buffer
    uint32_t validate;      // 2: quiescent-point scans before every grid sweep (validate.cuh)
    uint32_t* val;          // their scratch, 3 words per slot
    uint32_t track_rc;      // steps keep refcounts (validate modes); otherwise collectors recount (gc.cuh)
    uint32_t ra_warm_past;  // hand-over after this many sweeps of a steady frontier past the widest sweep
    uint32_t warp_max;      // frontiers of at most this many entries run on one warp (1..32; warp_mode)
    uint32_t warp_max_ra;   // ... in the run-ahead build, whose lanes follow diverging chains
};

__device__ __forceinline__ uint32_t* region_off(const Params& P, uint32_t buf) {
    return P.regions + buf * 2 * kMaxGrid;
}
__device__ __forceinline__ uint32_t* region_cnt(const Params& P, uint32_t buf) {
    return P.regions + buf * 2 * kMaxGrid + kMaxGrid;
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Software grid barrier (all CTAs are co-resident: cooperative launch).
// Arrivals are fire-and-forget increments of one monotonic counter; the
// k-th barrier completes when it reaches k * nblocks, so nobody resets it.
// `park` is for CTAs idling while CTA 0 runs single-CTA sweeps: they back
// off to microsecond sleeps so their polling does not load the L2 slice
// CTA 0 is working against.
__device__ __forceinline__ void grid_sync(Ctl* ctl, uint32_t nblocks, uint32_t& epoch, bool park = false) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        red_release_add(&ctl->bar_arrive, 1u);
        const uint32_t target = epoch * nblocks;
        // the acquire load pairs with every CTA's release increment; the
        // CTA barrier below extends it to the whole CTA
        if (park) {
            uint32_t ns = 64;
            while ((int)(ld_acquire(&ctl->bar_arrive) - target) < 0) {
                __nanosleep(ns);
                if (ns < 4096) ns <<= 1;
            }
        } else {
            while ((int)(ld_acquire(&ctl->bar_arrive) - target) < 0) {
            }
        }
    }
    __syncthreads();
}

struct Smem {
    uint32_t scan[kWarps];
    uint32_t bcast[4];
    unsigned long long red[kWarps];
};

// Exclusive block scan of v; *total gets the block sum.  Ends synchronised.
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* total, Smem& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm.scan[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kWarps ? sm.scan[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kWarps) sm.scan[lane] = w;
    }
    __syncthreads();
    uint32_t prefix = warp > 0 ? sm.scan[warp - 1] : 0;
    *total = sm.scan[kWarps - 1];
    __syncthreads();
    return prefix + x - v;
}

// Block-wide sum, valid in every thread.  Ends synchronised.
__device__ __forceinline__ unsigned long long block_sum64(unsigned long long v, Smem& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red[warp] = v;
    __syncthreads();
    // every thread reduces the warp sums with a full 32-lane butterfly
    // (lanes >= kWarps hold zero), so every lane of the block gets the total:
    // the single-CTA loop keeps per-thread counters from it and breaks on them
    unsigned long long t = lane < kWarps ? sm.red[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    __syncthreads();
    return t;
}

// Refcount update (rc_add / rc_sub, sweep_engine.cpp:267-275), aggregated
// over the lanes of the warp that hit the same slot as the first active lane.
// A bound variable shared by a whole level of a tree (transform's and
// build+sum's `n` under Expand/Build) is otherwise one same-address atomic
// per redex, serialised in its L2 slice; this issues one per warp.  The test
// is a shuffle and a ballot (a full match_any costs more than it saves when
// slots are distinct, the common case).
__device__ __forceinline__ void rc_update(uint32_t* rc, int delta) {
    const uint32_t act = __activemask();
    const int first = __ffs(act) - 1;
    const unsigned long long mine = reinterpret_cast<unsigned long long>(rc);
    const unsigned long long lead = __shfl_sync(act, mine, first);
    const uint32_t same = __ballot_sync(act, mine == lead);
    // one reduction instruction for the warp: the first lane carries its
    // group's sum, the group's other lanes nothing, everyone else its delta
    const int v = mine != lead ? delta : (int)(threadIdx.x & 31) == first ? delta * __popc(same) : 0;
    if (v) atomicAdd(rc, (uint32_t)v);
}

template <bool kSolo>
__device__ __forceinline__ void rc_upd(uint32_t* rc, int delta) {
    if (kSolo)
        atomicAdd(rc, (uint32_t)delta);  // one lane: nothing to aggregate
    else
        rc_update(rc, delta);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Typed views of the program blob staged in shared memory.
struct Prog {
    const uint8_t* arity;
    const uint16_t* rule_begin;
    const DRule* rules;
    const DStep* steps;
    const DInstr* instrs;
    const uint16_t* refs;
    const DPlan* plans;
    const uint16_t* mrow;
    const uint32_t* mtab;
    const uint16_t* chain;  // null: no constant chains
    uint32_t npos;
    uint32_t max_new;
};

__device__ __forceinline__ Prog view_prog(const uint8_t* blob) {
    const ProgHeader* h = reinterpret_cast<const ProgHeader*>(blob);
    Prog p;
    p.arity = blob + h->off_arity;
    p.rule_begin = reinterpret_cast<const uint16_t*>(blob + h->off_rule_begin);
    p.rules = reinterpret_cast<const DRule*>(blob + h->off_rules);
    p.steps = reinterpret_cast<const DStep*>(blob + h->off_steps);
    p.instrs = reinterpret_cast<const DInstr*>(blob + h->off_instrs);
    p.refs = reinterpret_cast<const uint16_t*>(blob + h->off_refs);
    p.plans = reinterpret_cast<const DPlan*>(blob + h->off_plans);
    p.mrow = reinterpret_cast<const uint16_t*>(blob + h->off_mrow);
    p.mtab = reinterpret_cast<const uint32_t*>(blob + h->off_mtab);
    p.npos = h->npos;
    p.chain = h->chains ? reinterpret_cast<const uint16_t*>(blob + h->off_chain) : nullptr;
    p.max_new = h->max_new_slots;
    return p;
}

template <int N>
__device__ __forceinline__ uint32_t pick(const uint32_t (&v)[N], uint32_t k) {
    uint32_t r = v[0];
#pragma unroll
    for (int t = 1; t < N; ++t)
        if (k == (uint32_t)t) r = v[t];
    return r;
}

template <int W>
__device__ __forceinline__ uint32_t* rec(uint32_t* arena, uint32_t i) {
    return arena + (size_t)i * W;
}

// Load the first `ar` argument words of a record (whole 16-byte quads).
template <int W>
__device__ __forceinline__ void load_args(const uint32_t* r, uint32_t ar, uint32_t (&a)[rec_args(W)]) {
#pragma unroll
    for (int q = 0; q < rec_args(W) / 4; ++q) {
        if ((uint32_t)(q * 4) < ar) {
            uint4 v = *reinterpret_cast<const uint4*>(r + kWArgs + q * 4);
            a[q * 4 + 0] = v.x;
            a[q * 4 + 1] = v.y;
            a[q * 4 + 2] = v.z;
            a[q * 4 + 3] = v.w;
        } else {
            a[q * 4 + 0] = a[q * 4 + 1] = a[q * 4 + 2] = a[q * 4 + 3] = 0;
        }
    }
}

template <int W>
__device__ __forceinline__ void store_args(uint32_t* r, const uint32_t (&a)[rec_args(W)], uint32_t ar) {
#pragma unroll
    for (int q = 0; q < rec_args(W) / 4; ++q) {
        if ((uint32_t)(q * 4) < ar || q == 0) {
            *reinterpret_cast<uint4*>(r + kWArgs + q * 4) =
                make_uint4(a[q * 4 + 0], a[q * 4 + 1], a[q * 4 + 2], a[q * 4 + 3]);
        }
    }
}

// Entries of a sweep are handed out in chunks of q <= 32 entries (one per
// lane), round-robin over all warps of the participating CTAs.  q is the
// smallest chunk that covers the frontier in one round, so a medium sweep
// spreads over every warp of the grid: fewer lanes per warp means fewer
// divergent symbol/rule paths in each warp's instruction stream, which is
// what bounds a sweep that is one chunk deep.  CTA b of n then processes
// exactly cta_entries(b) of m entries and the entries of CTAs < b number
// cta_prefix(b); its next-frontier pushes (at most max_new + 1 per entry)
// therefore fit the output region [(max_new+1) * prefix, +(max_new+1) * count).
__device__ __forceinline__ uint32_t chunk_lanes(uint32_t m, uint32_t nblocks) {
    const uint32_t gw = nblocks * kWarps;
    const uint32_t q = (m + gw - 1) / gw;
    return q < 1 ? 1 : q > 32 ? 32 : q;
}

__device__ __forceinline__ uint32_t cta_prefix(uint32_t m, uint32_t b, uint32_t nblocks, uint32_t q) {
    // 32-bit: m < 2^32 entries and round <= kMaxGrid * kBlock
    const uint32_t round = nblocks * kWarps * q;
    const uint32_t full = m / round;
    const uint32_t rem = m - full * round;
    const uint32_t before = b * kWarps * q;
    return full * before + (rem < before ? rem : before);
}

}  // namespace trs_b200

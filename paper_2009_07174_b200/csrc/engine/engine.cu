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
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "device_program.hpp"
#include "trs_gpu.h"

using namespace trs_b200;

namespace {

constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;

enum Status : uint32_t {
    kRunning = 0,
    kDone = 1,
    kStepBudget = 2,
    kCapacity = 3,
    kNeedGrow = 4,
    kNeedTrace = 5,
};

struct __align__(16) SweepCtr {
    uint32_t count;  // frontier list length of sweep s
    uint32_t alloc;  // slots claimed during sweep s
    unsigned long long rew;  // rewrites of sweep s
};

__device__ __forceinline__ SweepCtr ld_ctr(const SweepCtr* p) {
    uint4 v = __ldcg(reinterpret_cast<const uint4*>(p));
    SweepCtr c;
    c.count = v.x;
    c.alloc = v.y;
    c.rew = (unsigned long long)v.z | ((unsigned long long)v.w << 32);
    return c;
}

// Control block in device memory.  Persistent fields are written only at
// quiescent points (kernel exit, single-CTA hand-back); per-sweep counters
// rotate over 4 sweeps so that resetting the one two sweeps ahead never
// races with late readers (see reset in step_loop).
struct Ctl {
    // persistent state
    uint32_t sweep;     // completed sweeps
    uint32_t cur;       // current list buffer
    uint32_t arena;     // current arena buffer
    uint32_t base;      // bump pointer: slots [1, base) are allocated
    uint32_t status;
    uint32_t gc_runs;
    uint32_t small_sweeps;
    uint32_t abort_capacity;
    unsigned long long total_rewrites;
    unsigned long long max_width;
    unsigned long long gc_ns;
    uint32_t peak_base;
    uint32_t last_gc_sweep;
    // barrier: monotonic arrival counter, reset by the host before a launch
    uint32_t bar_arrive;
    uint32_t bar_pad;
    // rotating per-sweep counters (index sweep & 3), one 16-byte load each
    SweepCtr ctr[4];
    // GC scratch
    uint32_t gc_live;
    uint32_t prof_pad;
    // phase cycle accounting (P.profile): match, claim, apply, push, sweep total, sweeps
    unsigned long long prof[6];
};

struct Params {
    uint32_t* arena[2];
    uint32_t* list[2];
    uint32_t* gcmap;
    uint32_t* blocksum;
    uint32_t* roots;
    uint32_t num_roots;
    Ctl* ctl;
    trs_gpu_sweep_record* trace;
    uint32_t trace_cap;
    const uint8_t* prog;  // blob in global memory
    uint32_t prog_bytes;
    uint64_t capacity;  // slots per arena
    uint64_t step_budget;
    uint32_t small_enter, small_exit;
    uint32_t gc_interval;
    uint32_t allow_gc;
    uint32_t fixed_capacity;
    uint32_t max_new;
    uint32_t sweep0;  // sweeps completed before this run (epochs keep counting)
    uint32_t compact_only;  // >0: run at most this many compaction rounds and exit
    uint32_t prefer_grow;   // out of headroom: grow (host) rather than collect
    uint32_t profile;       // phase cycle accounting of CTA 0 (debug)
};

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long* p) { return __ldcg(p); }
__device__ __forceinline__ long long ld_cg(const long long* p) { return __ldcg(p); }

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

// Software grid barrier (all CTAs are co-resident: cooperative launch).
// Arrivals are fire-and-forget increments of one monotonic counter; the
// k-th barrier completes when it reaches k * nblocks, so nobody resets it.
// `park` is for CTAs idling while CTA 0 runs single-CTA sweeps: they back
// off to microsecond sleeps so their polling does not load the L2 slice
// CTA 0 is working against.
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ void grid_sync(Ctl* ctl, uint32_t nblocks, uint32_t& epoch, bool park = false) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        red_release_add(&ctl->bar_arrive, 1u);
        const uint32_t target = epoch * nblocks;
        uint32_t ns = 32;
        while ((int)(ld_acquire(&ctl->bar_arrive) - target) < 0) {
            __nanosleep(ns);
            if (park && ns < 4096) ns <<= 1;
        }
        __threadfence();
    }
    __syncthreads();
}

struct Smem {
    uint32_t scan[kWarps];
    uint32_t bcast[4];
    unsigned long long red[kWarps];
};

// Exclusive block scan of v; *total gets the block sum.  Ends synchronised
// so the scratch can be reused immediately.
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

__device__ __forceinline__ unsigned long long block_sum64(unsigned long long v, Smem& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red[warp] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kWarps; ++w) t += sm.red[w];
    __syncthreads();
    return t;  // valid in thread 0
}

// Typed views of the program blob staged in shared memory.
struct Prog {
    const uint8_t* arity;
    const uint16_t* rule_begin;
    const DRule* rules;
    const DStep* steps;
    const DInstr* instrs;
    const uint16_t* refs;
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

// Load the first `ar` argument words of slot i (whole 16-byte quads).
template <int W>
__device__ __forceinline__ void load_args(const uint32_t* r, uint32_t ar, uint32_t (&a)[W - 4]) {
#pragma unroll
    for (int q = 0; q < (W - 4) / 4; ++q) {
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
__device__ __forceinline__ void store_args(uint32_t* r, const uint32_t (&a)[W - 4], uint32_t ar) {
#pragma unroll
    for (int q = 0; q < (W - 4) / 4; ++q) {
        if ((uint32_t)(q * 4) < ar || q == 0) {
            *reinterpret_cast<uint4*>(r + kWArgs + q * 4) =
                make_uint4(a[q * 4 + 0], a[q * 4 + 1], a[q * 4 + 2], a[q * 4 + 3]);
        }
    }
}

enum Act : uint32_t { kActNone = 0, kActWait, kActNf, kActCollapse, kActBuild };

struct Acc {
    unsigned long long rewrites = 0;
    // optional phase accounting (thread 0 of CTA 0, P.profile): cycles in
    // [0] match, [1] claim, [2] apply, [3] push
    long long t[4] = {0, 0, 0, 0};
};

// One sweep over frontier entries [0, m) of `in`, by CTAs block_rank,
// block_rank + nblocks, ...  Pushes next-sweep entries to `out`.
template <int W>
__device__ void process_sweep(const Params& P, const Prog& G, Smem& sm, uint32_t* arena,
                              uint32_t s, uint32_t m, const uint32_t* __restrict__ in,
                              uint32_t* __restrict__ out, uint32_t* out_count, uint32_t base,
                              uint32_t* alloc_ctr, uint32_t block_rank, uint32_t nblocks,
                              Acc& acc, uint32_t* abort_flag = nullptr) {
    constexpr int MAXA = W - 4;
    const bool prof = P.profile && threadIdx.x == 0 && block_rank == 0;
    for (uint32_t start = block_rank * kBlock; start < m; start += nblocks * kBlock) {
        long long c0 = prof ? clock64() : 0;
        const uint32_t idx = start + threadIdx.x;
        uint32_t act = kActNone;
        uint32_t i = 0, sym = 0, ar = 0, rule = 0, wchild = 0, wpos = 0, cursor = 0;
        uint32_t a[MAXA];
        uint32_t bind[kMaxVars];
        if (idx < m) {
            i = in[idx];
            uint32_t* R = rec<W>(arena, i);
            uint2 he = *reinterpret_cast<const uint2*>(R);
            sym = he.x & kSymMask;
            cursor = he.x >> kSymBits;
            ar = G.arity[sym];
            load_args<W>(R, ar, a);
            // subterm scan (sweep_engine.cpp:173-178); all child probes issue together
            uint32_t ch[MAXA];
            uint32_t cep[MAXA];
#pragma unroll
            for (int j = 0; j < MAXA; ++j) {
                ch[j] = 0;
                cep[j] = 1;
                if ((uint32_t)j < ar) {
                    uint2 c = *reinterpret_cast<const uint2*>(rec<W>(arena, a[j]));
                    ch[j] = c.x & kSymMask;
                    cep[j] = c.y;
                }
            }
            bool pending = false;
#pragma unroll
            for (int j = MAXA - 1; j >= 0; --j) {
                if ((uint32_t)j >= cursor && (uint32_t)j < ar && (cep[j] == 0 || cep[j] >= s)) {
                    pending = true;
                    wpos = j;
                }
            }
            if (pending) {
                act = kActWait;
                wchild = pick(a, wpos);
            } else {
                // first matching rule in source order (dispatch.hpp:119-130)
                uint32_t stepnode[kMaxRuleSteps];
                int chosen = -1;
                for (uint32_t r = G.rule_begin[sym]; r < G.rule_begin[sym + 1]; ++r) {
                    const DRule& Rl = G.rules[r];
                    bool ok = true;
                    for (uint32_t t = 0; t < Rl.num_steps; ++t) {
                        const DStep st = G.steps[Rl.first_step + t];
                        uint32_t node, head;
                        if (st.parent < 0) {
                            node = pick(a, st.child);
                            head = pick(ch, st.child);
                        } else {
                            node = rec<W>(arena, stepnode[st.parent])[kWArgs + st.child];
                            head = st.kind == 0 ? (rec<W>(arena, node)[kWHead] & kSymMask) : 0;
                        }
                        stepnode[t] = node;
                        if (st.kind == 0) {
                            if (head != st.value) {
                                ok = false;
                                break;
                            }
                        } else {
                            bind[st.value] = node;
                        }
                    }
                    if (ok) {
                        chosen = (int)r;
                        break;
                    }
                }
                if (chosen < 0) {
                    act = kActNf;
                } else {
                    rule = (uint32_t)chosen;
                    act = G.rules[rule].collapse ? kActCollapse : kActBuild;
                }
            }
        }

        long long c1 = prof ? clock64() : 0;
        if (prof) acc.t[0] += c1 - c0;
        // ---- allocation: one claim per CTA iteration (get_new_index, term_store.cpp:118-138)
        uint32_t need = act == kActBuild ? G.rules[rule].new_slots : 0;
        uint32_t total;
        uint32_t excl = block_scan(need, &total, sm);
        if (threadIdx.x == 0) sm.bcast[0] = total ? atomicAdd(alloc_ctr, total) : 0;
        __syncthreads();
        const uint32_t fresh = base + sm.bcast[0] + excl;
        __syncthreads();
        if (act == kActBuild && (uint64_t)fresh + need > P.capacity) {
            // fixed capacity exhausted: the reference raises Capacity (sweep_engine.cpp:221-226)
            atomicExch(&P.ctl->abort_capacity, 1u);
            if (abort_flag) *abort_flag = 1u;
            act = kActNone;
        }

        long long c2 = prof ? clock64() : 0;
        if (prof) acc.t[1] += c2 - c1;
        // ---- apply (sweep_engine.cpp:190-258)
        uint32_t npush = 0, push1 = 0, push_mask = 0;
        if (act == kActWait) {
            if (wpos != cursor) rec<W>(arena, i)[kWHead] = sym | (wpos << kSymBits);
            uint32_t old = atomicCAS(rec<W>(arena, wchild) + kWWaiter, 0u, i);
            if (old != 0) {  // polled: lost the subscription or the child just turned nf
                npush = 1;
                push1 = i;
            }
        } else if (act == kActNf) {
            uint32_t* R = rec<W>(arena, i);
            R[kWEpoch] = s;
            uint32_t w = atomicExch(R + kWWaiter, kWoken);
            if (w != 0 && w != kWoken) {
                npush = 1;
                push1 = w;
            }
        } else if (act == kActCollapse) {
            const DRule& Rl = G.rules[rule];
            uint32_t src = bind[Rl.root_ref];
            uint32_t* S = rec<W>(arena, src);
            uint32_t shead = S[kWHead] & kSymMask;
            uint32_t sar = G.arity[shead];
            uint32_t b[MAXA];
            load_args<W>(S, sar, b);
#pragma unroll
            for (int j = 0; j < MAXA; ++j)
                if ((uint32_t)j >= sar) b[j] = 0;
            uint32_t* R = rec<W>(arena, i);
            *reinterpret_cast<uint2*>(R) = make_uint2(shead, s);
            store_args<W>(R, b, ar > sar ? ar : sar);
#pragma unroll
            for (int j = 0; j < MAXA; ++j)
                if ((uint32_t)j < sar) atomicAdd(rec<W>(arena, b[j]) + kWRc, 1u);
#pragma unroll
            for (int j = 0; j < MAXA; ++j)
                if ((uint32_t)j < ar) atomicSub(rec<W>(arena, a[j]) + kWRc, 1u);
            uint32_t w = atomicExch(R + kWWaiter, kWoken);
            if (w != 0 && w != kWoken) {
                npush = 1;
                push1 = w;
            }
            acc.rewrites++;
        } else if (act == kActBuild) {
            const DRule& Rl = G.rules[rule];
            const uint32_t nfresh = Rl.new_slots;
            for (uint32_t k = 0; k <= nfresh; ++k) {
                const DInstr I = G.instrs[Rl.first_instr + k];
                const uint32_t iar = G.arity[I.symbol];
                uint32_t b[MAXA];
#pragma unroll
                for (int j = 0; j < MAXA; ++j) {
                    b[j] = 0;
                    if ((uint32_t)j < iar) {
                        uint16_t ref = G.refs[I.first_ref + j];
                        b[j] = (ref & kRefNode) ? fresh + (ref & 0x7fff) : bind[ref];
                    }
                }
                if (k < nfresh) {
                    uint32_t sub = I.subscriber == kNone      ? 0u
                                   : I.subscriber == kRootSub ? i
                                                              : fresh + I.subscriber;
                    uint32_t* F = rec<W>(arena, fresh + k);
                    *reinterpret_cast<uint4*>(F) =
                        make_uint4(I.symbol | ((uint32_t)I.cursor << kSymBits), 0u, I.indegree, sub);
#pragma unroll
                    for (int q = 0; q < MAXA / 4; ++q)
                        *reinterpret_cast<uint4*>(F + kWArgs + q * 4) =
                            make_uint4(b[q * 4], b[q * 4 + 1], b[q * 4 + 2], b[q * 4 + 3]);
                } else {
                    uint32_t* R = rec<W>(arena, i);
                    R[kWHead] = I.symbol | ((uint32_t)Rl.root_cursor << kSymBits);
                    store_args<W>(R, b, ar > iar ? ar : iar);
                }
                // every reuse of a bound variable adds one reference (sweep_engine.cpp:251-253)
#pragma unroll
                for (int j = 0; j < MAXA; ++j) {
                    if ((uint32_t)j < iar) {
                        uint16_t ref = G.refs[I.first_ref + j];
                        if (!(ref & kRefNode)) atomicAdd(rec<W>(arena, b[j]) + kWRc, 1u);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < MAXA; ++j)
                if ((uint32_t)j < ar) atomicSub(rec<W>(arena, a[j]) + kWRc, 1u);
            push_mask = Rl.push_mask;
            npush = __popc(push_mask) + (Rl.root_wait == kNone ? 1u : 0u);
            push1 = i;
            acc.rewrites++;
        }

        long long c3 = prof ? clock64() : 0;
        if (prof) acc.t[2] += c3 - c2;
        // ---- next frontier: one reservation per CTA iteration
        uint32_t ptotal;
        uint32_t pexcl = block_scan(npush, &ptotal, sm);
        if (threadIdx.x == 0) sm.bcast[1] = ptotal ? atomicAdd(out_count, ptotal) : 0;
        __syncthreads();
        uint32_t pos = sm.bcast[1] + pexcl;
        __syncthreads();
        if (npush) {
            if (act == kActBuild) {
                uint32_t mask = push_mask;
                while (mask) {
                    uint32_t k = __ffs(mask) - 1;
                    mask &= mask - 1;
                    out[pos++] = fresh + k;
                }
                if (G.rules[rule].root_wait == kNone) out[pos++] = i;
            } else {
                out[pos] = push1;
            }
        }
        if (prof) acc.t[3] += clock64() - c3;
    }
}

// ---------------------------------------------------------------------------
// compacting GC (grid-wide).  Returns the new bump pointer.

template <int W>
__device__ uint32_t gc_compact(const Params& P, Smem& sm, uint32_t& arena_idx, uint32_t base,
                               uint32_t cur_list, uint32_t m, uint32_t block_rank,
                               uint32_t nblocks, const Prog& G, uint32_t& epoch) {
    uint32_t* A = P.arena[arena_idx];
    uint32_t* B = P.arena[arena_idx ^ 1];
    const uint32_t tid = block_rank * kBlock + threadIdx.x;
    const uint32_t nthreads = nblocks * kBlock;
    auto sync = [&]() { grid_sync(P.ctl, nblocks, epoch); };
    // phase 1: claim refcount-zero slots and drop their argument references
    // (collect_free_indices, term_store.cpp:140-157); a thread follows the
    // cascade it triggers for a bounded number of hops, the rest waits for
    // a later collection, exactly as the reference defers it.
    unsigned long long freed = 0;
    for (uint32_t x = 1 + tid; x < base; x += nthreads) {
        uint32_t* R = rec<W>(A, x);
        uint32_t head = __ldcg(R + kWHead);
        if (head == kDeadHead || __ldcg(R + kWRc) != 0) continue;
        if (atomicCAS(R + kWHead, head, kDeadHead) != head) continue;
        uint32_t cur = x, chead = head;
        for (int hop = 0; hop < 64; ++hop) {
            freed++;
            uint32_t* C = rec<W>(A, cur);
            uint32_t car = G.arity[chead & kSymMask];
            uint32_t next = 0, nhead = 0;
            for (uint32_t j = 0; j < car; ++j) {
                uint32_t c = __ldcg(C + kWArgs + j);
                if (atomicSub(rec<W>(A, c) + kWRc, 1u) == 1u && next == 0) {
                    uint32_t h = __ldcg(rec<W>(A, c) + kWHead);
                    if (h != kDeadHead && atomicCAS(rec<W>(A, c) + kWHead, h, kDeadHead) == h) {
                        next = c;
                        nhead = h;
                    }
                }
            }
            if (!next) break;
            cur = next;
            chead = nhead;
        }
    }
    sync();
    // phase 2: live count per CTA range
    const uint32_t span = base - 1;
    const uint32_t chunk = (span + nblocks - 1) / nblocks;
    const uint32_t lo = 1 + block_rank * chunk;
    const uint32_t hi = min(base, lo + chunk);
    uint32_t cnt = 0;
    for (uint32_t x = lo + threadIdx.x; x < hi; x += kBlock)
        cnt += __ldcg(rec<W>(A, x) + kWHead) != kDeadHead;
    uint32_t tot;
    block_scan(cnt, &tot, sm);
    if (threadIdx.x == 0) P.blocksum[block_rank] = tot;
    sync();
    // phase 3: prefix over CTA sums, then order-preserving scatter into the
    // twin arena with the old->new map
    uint32_t prefix = 0, all = 0;
    for (uint32_t b = threadIdx.x; b < nblocks; b += kBlock) {
        uint32_t v = __ldcg(P.blocksum + b);
        all += v;
        if (b < block_rank) prefix += v;
    }
    uint32_t dummy;
    // reduce prefix and all over the block
    {
        uint32_t t1, t2;
        block_scan(prefix, &t1, sm);
        block_scan(all, &t2, sm);
        prefix = t1;
        all = t2;
    }
    (void)dummy;
    uint32_t running = 1 + prefix;
    for (uint32_t x0 = lo; x0 < hi; x0 += kBlock) {
        uint32_t x = x0 + threadIdx.x;
        bool live = x < hi && __ldcg(rec<W>(A, x) + kWHead) != kDeadHead;
        uint32_t t;
        uint32_t e = block_scan(live ? 1u : 0u, &t, sm);
        if (x < hi) P.gcmap[x] = live ? running + e : 0u;
        if (live) {
            const uint4* src = reinterpret_cast<const uint4*>(rec<W>(A, x));
            uint4* dst = reinterpret_cast<uint4*>(rec<W>(B, running + e));
#pragma unroll
            for (int q = 0; q < W / 4; ++q) dst[q] = __ldcg(src + q);
        }
        running += t;
    }
    sync();
    // phase 4: remap args, waiters, frontier entries, roots
    const uint32_t nbase = 1 + all;
    for (uint32_t y = 1 + tid; y < nbase; y += nthreads) {
        uint32_t* R = rec<W>(B, y);
        uint32_t car = G.arity[R[kWHead] & kSymMask];
        for (uint32_t j = 0; j < car; ++j) R[kWArgs + j] = __ldcg(P.gcmap + R[kWArgs + j]);
        uint32_t w = R[kWWaiter];
        if (w != 0 && w != kWoken) R[kWWaiter] = __ldcg(P.gcmap + w);
    }
    uint32_t* L = P.list[cur_list];
    for (uint32_t e = tid; e < m; e += nthreads) L[e] = __ldcg(P.gcmap + L[e]);
    for (uint32_t e = tid; e < P.num_roots; e += nthreads) P.roots[e] = __ldcg(P.gcmap + P.roots[e]);
    sync();
    arena_idx ^= 1;
    (void)freed;
    return nbase;
}

// ---------------------------------------------------------------------------

struct Local {
    uint32_t sweep, cur, arena, base;
    unsigned long long total, maxw;
    uint32_t gc_runs, small_sweeps, last_gc, peak_base;
    unsigned long long gc_ns;
};

__device__ void load_local(Local& L, Ctl* c) {
    L.sweep = ld_cg(&c->sweep);
    L.cur = ld_cg(&c->cur);
    L.arena = ld_cg(&c->arena);
    L.base = ld_cg(&c->base);
    L.total = ld_cg(&c->total_rewrites);
    L.maxw = ld_cg(&c->max_width);
    L.gc_runs = ld_cg(&c->gc_runs);
    L.small_sweeps = ld_cg(&c->small_sweeps);
    L.last_gc = ld_cg(&c->last_gc_sweep);
    L.peak_base = ld_cg(&c->peak_base);
    L.gc_ns = ld_cg(&c->gc_ns);
}

__device__ void store_local(const Local& L, Ctl* c) {
    c->sweep = L.sweep;
    c->cur = L.cur;
    c->arena = L.arena;
    c->base = L.base;
    c->total_rewrites = L.total;
    c->max_width = L.maxw;
    c->gc_runs = L.gc_runs;
    c->small_sweeps = L.small_sweeps;
    c->last_gc_sweep = L.last_gc;
    c->peak_base = L.peak_base;
    c->gc_ns = L.gc_ns;
    __threadfence();
}

// What to do before sweep s, identical in every CTA.
enum Plan : uint32_t { kPlanSweep, kPlanGc, kPlanGrow, kPlanFinish, kPlanBudget, kPlanTrace };

__device__ __forceinline__ uint32_t plan(const Params& P, const Local& L, uint32_t m,
                                         bool just_collected) {
    const uint32_t s = L.sweep + 1;
    if (s - P.sweep0 > P.trace_cap) return kPlanTrace;
    if (m == 0) return kPlanFinish;
    // worst case: every frontier slot rewrites with the largest template
    // (ensure_headroom, sweep_engine.cpp:290-303)
    const uint64_t worst = (uint64_t)L.base + (uint64_t)m * P.max_new + 1;
    if (worst > P.capacity) {
        if (P.allow_gc && !just_collected && !P.prefer_grow) return kPlanGc;
        if (!P.fixed_capacity) return kPlanGrow;
        // fixed capacity: go ahead; a claim that does not fit aborts with
        // Capacity like the reference (sweep_engine.cpp:221-226)
    }
    // a collection that left the arena more than half full: grow instead of
    // collecting again next sweep
    if (just_collected && !P.fixed_capacity && (uint64_t)L.base * 2 > P.capacity) return kPlanGrow;
    if (P.allow_gc && P.gc_interval && !just_collected && s - L.last_gc >= P.gc_interval)
        return kPlanGc;
    return kPlanSweep;
}

__device__ void record(const Params& P, uint32_t s, unsigned long long width, const Local& L,
                       uint32_t m, uint32_t mode, uint64_t ns) {
    const uint32_t k = s - P.sweep0;
    if (k == 0 || k > P.trace_cap) return;
    trs_gpu_sweep_record r;
    r.sweep = k;
    r.live_terms = L.base - 1;  // allocated and not yet reclaimed by a compaction
    r.rewrites = width;
    r.n = L.base;
    r.free_len = 0;
    r.active = m;
    r.mode = mode;
    r.micros_x1000 = ns;
    P.trace[k - 1] = r;
}

// Shared-memory state of the single-CTA mode.
struct SmallState {
    uint32_t count[2];    // frontier counts: [cur] being read, [cur^1] being pushed
    uint32_t alloc;
    uint32_t abort;       // a claim did not fit the fixed capacity
    unsigned long long width;
};

constexpr uint32_t kSmallCap = 4096;  // frontier entries per shared-memory list

template <int W>
__device__ void run_small(const Params& P, const Prog& G, Smem& sm, Local& L, bool& just_collected,
                          uint32_t* slist /* 2 * kSmallCap */, SmallState& ss) {
    Ctl* ctl = P.ctl;
    const uint32_t s0 = L.sweep + 1;
    uint32_t m = ld_ctr(&ctl->ctr[s0 & 3]).count;
    const uint32_t cap_m = kSmallCap / (P.max_new + 1);
    const uint32_t exit_m = min(P.small_exit, cap_m);
    if (m > exit_m) return;  // too wide for the shared-memory lists; nothing touched
    // stage the frontier into shared memory
    uint32_t* gin = P.list[L.cur];
    for (uint32_t e = threadIdx.x; e < m; e += kBlock) slist[e] = gin[e];
    uint32_t sc = 0;  // shared list holding the current frontier
    if (threadIdx.x == 0) {
        ss.count[0] = m;
        ss.abort = 0;
    }
    __syncthreads();
    for (;;) {
        const uint32_t s = L.sweep + 1;
        m = ss.count[sc];
        if (m > exit_m) break;
        if (plan(P, L, m, just_collected) != kPlanSweep) break;
        just_collected = false;
        uint64_t t0 = threadIdx.x == 0 ? global_ns() : 0;
        long long cs = (P.profile && threadIdx.x == 0) ? clock64() : 0;
        __syncthreads();  // everyone has read ss.count[sc]
        if (threadIdx.x == 0) {
            ss.count[sc ^ 1] = 0;
            ss.alloc = 0;
        }
        __syncthreads();
        Acc acc;
        process_sweep<W>(P, G, sm, P.arena[L.arena], s, m, slist + sc * kSmallCap,
                         slist + (sc ^ 1) * kSmallCap, &ss.count[sc ^ 1], L.base, &ss.alloc, 0, 1, acc,
                         &ss.abort);
        unsigned long long rw = block_sum64(acc.rewrites, sm);
        if (threadIdx.x == 0) ss.width = rw;
        __syncthreads();
        const unsigned long long width = ss.width;
        L.base += ss.alloc;
        L.peak_base = max(L.peak_base, L.base);
        L.total += width;
        L.maxw = width > L.maxw ? width : L.maxw;
        L.sweep = s;
        L.small_sweeps++;
        sc ^= 1;
        if (threadIdx.x == 0) record(P, s, width, L, m, 1, global_ns() - t0);
        if (P.profile && threadIdx.x == 0) {
            for (int k = 0; k < 4; ++k) ctl->prof[k] += acc.t[k];
            ctl->prof[4] += clock64() - cs;
            ctl->prof[5] += 1;
        }
        if (L.total > P.step_budget) break;
        if (ss.abort) break;
    }
    // hand the frontier back to the grid through the global list
    m = ss.count[sc];
    uint32_t* gout = P.list[L.cur];
    // L.cur is unchanged while the lists live in shared memory
    for (uint32_t e = threadIdx.x; e < m; e += kBlock) gout[e] = slist[sc * kSmallCap + e];
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t s = L.sweep + 1;
        for (int k = 0; k < 4; ++k) ctl->ctr[k] = SweepCtr{0u, 0u, 0ull};
        ctl->ctr[s & 3].count = m;
        store_local(L, ctl);
    }
}

template <int W, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) step_loop(Params P) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ Smem sm;
    __shared__ SmallState ss;
    // stage the program tables; the single-CTA frontier lists follow them
    for (uint32_t o = threadIdx.x * 16; o < P.prog_bytes; o += kBlock * 16)
        *reinterpret_cast<uint4*>(smem_raw + o) = *reinterpret_cast<const uint4*>(P.prog + o);
    __syncthreads();
    const Prog G = view_prog(smem_raw);
    uint32_t* slist = reinterpret_cast<uint32_t*>(smem_raw + P.prog_bytes);
    const uint32_t nblocks = gridDim.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    Ctl* ctl = P.ctl;

    Local L;
    load_local(L, ctl);
    bool just_collected = false;
    uint32_t exit_status = kRunning;
    uint32_t epoch = 0;  // barriers passed in this launch (the host zeroes bar_arrive)

    if (P.compact_only) {
        // final compaction: collect until a pass reclaims nothing
        for (uint32_t round = 0; round < P.compact_only; ++round) {
            uint32_t before = L.base;
            const uint32_t s = L.sweep + 1;
            uint64_t t0 = global_ns();
            L.base = gc_compact<W>(P, sm, L.arena, L.base, L.cur, ld_ctr(&ctl->ctr[s & 3]).count, blockIdx.x,
                                   nblocks, G, epoch);
            L.gc_runs++;
            L.gc_ns += global_ns() - t0;
            if (L.base == before) break;
        }
        if (leader) {
            store_local(L, ctl);
            ctl->status = kDone;
        }
        return;
    }

    // frontier length of the next sweep; read after every barrier that
    // precedes a sweep (a grid sweep carries it over from its bookkeeping load)
    uint32_t m = ld_ctr(&ctl->ctr[(L.sweep + 1) & 3]).count;
    for (;;) {
        const uint32_t s = L.sweep + 1;
        const uint32_t pl = plan(P, L, m, just_collected);
        if (pl == kPlanFinish) {
            // the first sweep whose frontier is empty (sweep_engine.cpp:147)
            if (leader) record(P, s, 0, L, 0, 0, 0);
            L.sweep = s;
            exit_status = kDone;
            break;
        }
        if (pl == kPlanTrace) { exit_status = kNeedTrace; break; }
        if (pl == kPlanGrow) { exit_status = kNeedGrow; break; }
        if (pl == kPlanGc) {
            uint64_t t0 = global_ns();
            L.base = gc_compact<W>(P, sm, L.arena, L.base, L.cur, m, blockIdx.x, nblocks, G, epoch);
            L.gc_runs++;
            L.last_gc = L.sweep + 1;
            L.gc_ns += global_ns() - t0;
            just_collected = true;
            continue;
        }

        if (m <= P.small_enter) {
            // ---- single-CTA mode: CTA 0 runs sweeps out of shared memory,
            // the rest of the grid parks in the barrier
            const uint32_t before = L.sweep;
            if (blockIdx.x == 0) run_small<W>(P, G, sm, L, just_collected, slist, ss);
            grid_sync(ctl, nblocks, epoch, /*park=*/blockIdx.x != 0);
            load_local(L, ctl);
            m = ld_ctr(&ctl->ctr[(L.sweep + 1) & 3]).count;
            if (L.sweep != before) just_collected = false;  // keep every CTA's plan identical
            if (ld_cg(&ctl->abort_capacity)) { exit_status = kCapacity; break; }
            if (L.total > P.step_budget) { exit_status = kStepBudget; break; }
            if (L.sweep != before) continue;
            // no progress in single-CTA mode (frontier too wide for its
            // lists): fall through to one grid-wide sweep
        }
        just_collected = false;

        // ---- grid-wide sweep
        uint64_t t0 = leader ? global_ns() : 0;
        if (leader) ctl->ctr[(s + 2) & 3] = SweepCtr{0u, 0u, 0ull};
        Acc acc;
        process_sweep<W>(P, G, sm, P.arena[L.arena], s, m, P.list[L.cur], P.list[L.cur ^ 1],
                         &ctl->ctr[(s + 1) & 3].count, L.base, &ctl->ctr[s & 3].alloc, blockIdx.x,
                         nblocks, acc);
        unsigned long long rw = block_sum64(acc.rewrites, sm);
        if (threadIdx.x == 0 && rw) atomicAdd(&ctl->ctr[s & 3].rew, rw);
        grid_sync(ctl, nblocks, epoch);
        const SweepCtr done_ctr = ld_ctr(&ctl->ctr[s & 3]);
        const SweepCtr next_ctr = ld_ctr(&ctl->ctr[(s + 1) & 3]);
        const unsigned long long width = done_ctr.rew;
        const uint32_t allocd = done_ctr.alloc;
        m = next_ctr.count;
        L.base += allocd;
        L.peak_base = max(L.peak_base, L.base);
        L.total += width;
        L.maxw = width > L.maxw ? width : L.maxw;
        L.sweep = s;
        L.cur ^= 1;
        if (leader) record(P, s, width, L, m, 0, global_ns() - t0);
        if (P.profile && leader) {
            for (int k = 0; k < 4; ++k) ctl->prof[k] += acc.t[k];
            ctl->prof[5] += 1;
        }
        if (ld_cg(&ctl->abort_capacity)) { exit_status = kCapacity; break; }
        if (L.total > P.step_budget) { exit_status = kStepBudget; break; }
    }
    if (leader) {
        store_local(L, ctl);
        ctl->status = exit_status;
    }
}

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
            for (uint32_t j = 0; j < max_arity && j < (uint32_t)(W - 4); ++j)
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
                              uint32_t* __restrict__ list, uint32_t* __restrict__ count) {
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
            if (push) list[off + __popc(mask & ((1u << lane) - 1))] = i;
        }
    }
}

__global__ void gather_probe_kernel(const uint32_t* __restrict__ data, uint64_t words, const uint32_t* __restrict__ idx,
                                    uint32_t n, uint32_t vec, uint32_t* __restrict__ sink) {
    uint32_t acc = 0;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        uint64_t e = idx[k];
        if (vec == 1) {
            acc += data[e % words];
        } else if (vec == 2) {
            uint2 v = reinterpret_cast<const uint2*>(data)[e % (words / 2)];
            acc += v.x ^ v.y;
        } else {
            uint4 v = reinterpret_cast<const uint4*>(data)[e % (words / 4)];
            acc += v.x ^ v.y ^ v.z ^ v.w;
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
    int W = 8;
    int minb = 1;  // register budget variant of the step loop (see step_loop_for)

    // store
    uint64_t capacity = 0;        // logical capacity (slots) the step loop may use
    uint64_t alloc_capacity = 0;  // slots physically allocated per arena
    int alloc_W = 0;
    uint32_t roots_cap = 0;
    uint32_t* d_arena[2] = {nullptr, nullptr};
    uint32_t* d_list[2] = {nullptr, nullptr};
    uint32_t* d_gcmap = nullptr;
    uint32_t* d_roots = nullptr;
    uint32_t* d_blocksum = nullptr;
    uint32_t num_roots = 0;
    Ctl* d_ctl = nullptr;
    trs_gpu_sweep_record* d_trace = nullptr;
    uint32_t trace_cap = 0;
    bool loaded = false;
    uint32_t last_sweeps = 0;
    int record_width = 8;
    float load_ms = 0.f;
};

namespace {

int fail(trs_gpu_engine* e, int code, const std::string& msg) {
    if (e) e->last_error = msg;
    return code;
}

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
    cudaFree(e->d_ctl);
    cudaFree(e->d_trace);
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
    if (max_arity <= 12) return 16;
    if (max_arity <= 28) return 32;
    return 0;
}

// Build the device blob from the flattened reference DispatchTable.
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
    e->blob = std::move(blob);
    e->max_arity = max_arity;
    e->max_new = max_new;
    e->num_symbols = p->num_symbols;
    e->arity.assign(p->arity, p->arity + p->num_symbols);
    e->W = words_for_arity(max_arity);
    return TRS_GPU_OK;
}

// Two register budgets per record width: MINB = 1 (no spills, 1 CTA of 512
// threads per SM) and MINB = 2 (64 registers, 2 CTAs per SM, some spills).
template <int W, int MINB>
const void* step_loop_ptr() {
    return reinterpret_cast<const void*>(&step_loop<W, MINB>);
}

const void* step_loop_for(int W, int minb) {
    if (minb >= 2) {
        switch (W) {
            case 8: return step_loop_ptr<8, 2>();
            case 16: return step_loop_ptr<16, 2>();
            default: return step_loop_ptr<32, 2>();
        }
    }
    switch (W) {
        case 8: return step_loop_ptr<8, 1>();
        case 16: return step_loop_ptr<16, 1>();
        default: return step_loop_ptr<32, 1>();
    }
}

size_t dyn_smem(const trs_gpu_engine* e) { return e->blob.size() + 2 * kSmallCap * sizeof(uint32_t); }

int alloc_store(trs_gpu_engine* e, uint64_t capacity) {
    size_t rec_bytes = (size_t)e->W * 4;
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(e, cudaMalloc(&e->d_arena[k], rec_bytes * capacity));
        CUDA_TRY(e, cudaMalloc(&e->d_list[k], sizeof(uint32_t) * capacity));
    }
    CUDA_TRY(e, cudaMalloc(&e->d_gcmap, sizeof(uint32_t) * capacity));
    e->capacity = capacity;
    e->alloc_capacity = capacity;
    e->alloc_W = e->W;
    return TRS_GPU_OK;
}

int grid_blocks(trs_gpu_engine* e, uint32_t blocks_per_sm) {
    int occ = 0;
    size_t dyn = dyn_smem(e);
    const void* fn = step_loop_for(e->W, e->minb);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, dyn) != cudaSuccess || occ < 1)
        occ = 1;
    if (blocks_per_sm) occ = std::min<int>(occ, (int)blocks_per_sm);
    return occ * e->sm_count;
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
        if (cudaMalloc(&na[k], rec_bytes * cap) != cudaSuccess || cudaMalloc(&nl[k], sizeof(uint32_t) * cap) != cudaSuccess) {
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
    uint32_t s = c.sweep + 1;
    uint32_t m = c.ctr[s & 3].count;
    CUDA_TRY(e, cudaMemcpyAsync(na[c.arena], e->d_arena[c.arena], rec_bytes * c.base, cudaMemcpyDeviceToDevice, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(nl[c.cur], e->d_list[c.cur], sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, e->stream));
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

void reset_barrier(trs_gpu_engine* e) {
    cudaMemsetAsync(reinterpret_cast<uint8_t*>(e->d_ctl) + offsetof(Ctl, bar_arrive), 0, sizeof(uint32_t), e->stream);
}

// Growing is preferred over collecting while the twin arenas, lists and
// map of the grown store fit comfortably in free HBM; the compacting GC is
// the memory-pressure path (and what fixed-capacity stores rely on).
bool prefer_grow(trs_gpu_engine* e) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    uint64_t next = e->capacity * 2;
    uint64_t need = next * ((uint64_t)e->W * 4 * 2 + 4 * 3);
    return need < free_b / 2;
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

template <int W>
void launch_load(trs_gpu_engine* e, uint32_t n, const uint32_t* hss, const uint32_t* args, uint32_t max_arity,
                 const uint32_t* rc, const uint8_t* d_arity, uint32_t* count) {
    int blocks = std::max(1, std::min<int>((int)((n + 255) / 256), e->sm_count * 8));
    load_records<W><<<blocks, 256, 0, e->stream>>>(e->d_arena[0], n, hss, args, max_arity, rc);
    load_frontier<W><<<blocks, 256, 0, e->stream>>>(e->d_arena[0], n, d_arity, e->d_list[0], count);
}

int load_impl(trs_gpu_engine* e, uint32_t n, const uint32_t* roots, uint32_t num_roots,
              const uint32_t* d_hss, const uint32_t* d_args, uint32_t max_arity, const uint32_t* d_rc,
              uint64_t capacity) {
    if (e->blob.empty()) return fail(e, TRS_GPU_INVALID, "no program set");
    if (n < 2 || num_roots == 0) return fail(e, TRS_GPU_INVALID, "empty store");
    if (max_arity > (uint32_t)(e->W - 4))
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
    if (!e->d_blocksum) CUDA_TRY(e, cudaMalloc(&e->d_blocksum, sizeof(uint32_t) * (e->sm_count * 32 + 1)));
    if (!e->d_trace) {
        e->trace_cap = 1u << 16;
        CUDA_TRY(e, cudaMalloc(&e->d_trace, sizeof(trs_gpu_sweep_record) * e->trace_cap));
    }
    if (e->d_prog == nullptr) return fail(e, TRS_GPU_INVALID, "program not staged");
    // frontier count of sweep 1 lives in ctl->ctr[1].count
    uint32_t* d_count = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(e->d_ctl) + offsetof(Ctl, ctr) +
                                                    sizeof(SweepCtr) * 1 + offsetof(SweepCtr, count));
    const uint8_t* d_arity = e->d_prog + reinterpret_cast<const ProgHeader*>(e->blob.data())->off_arity;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, e->stream);
    switch (e->W) {
        case 8: launch_load<8>(e, n, d_hss, d_args, max_arity, d_rc, d_arity, d_count); break;
        case 16: launch_load<16>(e, n, d_hss, d_args, max_arity, d_rc, d_arity, d_count); break;
        default: launch_load<32>(e, n, d_hss, d_args, max_arity, d_rc, d_arity, d_count); break;
    }
    cudaEventRecord(b, e->stream);
    CUDA_TRY(e, cudaGetLastError());
    // persistent state: sweep 0 done, bump pointer n, live = slots with rc>0
    Ctl init{};
    init.base = n;
    init.peak_base = n;
    init.status = kRunning;
    CUDA_TRY(e, cudaEventSynchronize(b));
    cudaEventElapsedTime(&e->load_ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    uint32_t count1 = 0;
    CUDA_TRY(e, cudaMemcpy(&count1, d_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    init.ctr[1].count = count1;
    CUDA_TRY(e, cudaMemcpy(e->d_ctl, &init, sizeof(Ctl), cudaMemcpyHostToDevice));
    e->num_roots = num_roots;
    e->loaded = true;
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
    h.base = c.base;
    h.words.resize((size_t)c.base * e->W);
    CUDA_TRY(e, cudaMemcpy(h.words.data(), e->d_arena[c.arena], sizeof(uint32_t) * h.words.size(), cudaMemcpyDeviceToHost));
    roots.resize(e->num_roots);
    CUDA_TRY(e, cudaMemcpy(roots.data(), e->d_roots, sizeof(uint32_t) * e->num_roots, cudaMemcpyDeviceToHost));
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
    cudaStreamDestroy(e->stream);
    delete e;
}

int trs_gpu_set_program(trs_gpu_engine* e, const trs_gpu_program* p) {
    if (!e) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    int rc = build_blob(e, p);
    if (rc) return rc;
    cudaFree(e->d_prog);
    e->d_prog = nullptr;
    CUDA_TRY(e, cudaMalloc(&e->d_prog, e->blob.size()));
    CUDA_TRY(e, cudaMemcpy(e->d_prog, e->blob.data(), e->blob.size(), cudaMemcpyHostToDevice));
    e->loaded = false;
    return TRS_GPU_OK;
}

int trs_gpu_load(trs_gpu_engine* e, uint32_t n, const uint32_t* roots, uint32_t num_roots, const uint32_t* hss,
                 const uint32_t* args, uint32_t max_arity, const uint32_t* refcounts, uint64_t capacity) {
    if (!e || !hss || !refcounts || (max_arity && !args) || !roots) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    uint32_t *dh = nullptr, *da = nullptr, *dr = nullptr;
    size_t na = (size_t)max_arity * n;
    CUDA_TRY(e, cudaMallocAsync(&dh, sizeof(uint32_t) * n, e->stream));
    CUDA_TRY(e, cudaMallocAsync(&da, sizeof(uint32_t) * std::max<size_t>(na, 1), e->stream));
    CUDA_TRY(e, cudaMallocAsync(&dr, sizeof(uint32_t) * n, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(dh, hss, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e->stream));
    if (na) CUDA_TRY(e, cudaMemcpyAsync(da, args, sizeof(uint32_t) * na, cudaMemcpyHostToDevice, e->stream));
    CUDA_TRY(e, cudaMemcpyAsync(dr, refcounts, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e->stream));
    int rc = load_impl(e, n, roots, num_roots, dh, da, max_arity, dr, capacity);
    cudaFreeAsync(dh, e->stream);
    cudaFreeAsync(da, e->stream);
    cudaFreeAsync(dr, e->stream);
    cudaStreamSynchronize(e->stream);
    return rc;
}

int trs_gpu_load_device(trs_gpu_engine* e, uint32_t n, const uint32_t* roots, uint32_t num_roots,
                        const uint32_t* d_hss, const uint32_t* d_args, uint32_t max_arity,
                        const uint32_t* d_refcounts, uint64_t capacity) {
    if (!e || !d_hss || !d_refcounts || !roots) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    return load_impl(e, n, roots, num_roots, d_hss, d_args, max_arity, d_refcounts, capacity);
}

int trs_gpu_run(trs_gpu_engine* e, const trs_gpu_options* opt_in, trs_gpu_stats* stats) {
    if (!e) return TRS_GPU_INVALID;
    if (!e->loaded) return fail(e, TRS_GPU_INVALID, "no store loaded");
    cudaSetDevice(e->device);
    trs_gpu_options opt{};
    if (opt_in) opt = *opt_in;
    e->last_error.clear();
    e->minb = opt.variant == 2 ? 2 : 1;
    int blocks = grid_blocks(e, opt.blocks_per_sm);
    if (opt.max_blocks && (int)opt.max_blocks < blocks) blocks = (int)opt.max_blocks;
    trs_gpu_stats st{};
    st.grid_blocks = blocks;
    st.block_threads = kBlock;
    st.record_words = e->W;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int result = TRS_GPU_OK;
    float total_ms = 0.f;
    uint32_t sweep0 = 0;
    {
        Ctl c0;
        CUDA_TRY(e, cudaMemcpy(&c0, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
        sweep0 = c0.sweep;
        c0.total_rewrites = 0;
        c0.max_width = 0;
        c0.gc_runs = 0;
        c0.small_sweeps = 0;
        c0.gc_ns = 0;
        c0.status = kRunning;
        c0.abort_capacity = 0;
        c0.last_gc_sweep = c0.sweep;
        CUDA_TRY(e, cudaMemcpy(e->d_ctl, &c0, sizeof(Ctl), cudaMemcpyHostToDevice));
    }
    for (;;) {
        Params P{};
        P.arena[0] = e->d_arena[0];
        P.arena[1] = e->d_arena[1];
        P.list[0] = e->d_list[0];
        P.list[1] = e->d_list[1];
        P.gcmap = e->d_gcmap;
        P.blocksum = e->d_blocksum;
        P.roots = e->d_roots;
        P.num_roots = e->num_roots;
        P.ctl = e->d_ctl;
        P.trace = e->d_trace;
        P.trace_cap = e->trace_cap;
        P.prog = e->d_prog;
        P.prog_bytes = (uint32_t)e->blob.size();
        P.capacity = e->capacity;
        P.step_budget = opt.step_budget ? opt.step_budget : 1000000000ull;
        P.small_enter = opt.disable_small ? 0 : (opt.small_enter ? opt.small_enter : kBlock);
        P.small_exit = opt.disable_small ? 0 : (opt.small_exit ? opt.small_exit : 2 * kBlock);
        if (P.small_exit < P.small_enter) P.small_exit = P.small_enter;
        P.gc_interval = opt.gc_interval;
        P.allow_gc = opt.disable_gc ? 0 : 1;
        P.fixed_capacity = opt.fixed_capacity;
        P.max_new = e->max_new;
        P.sweep0 = sweep0;
        P.prefer_grow = (!opt.fixed_capacity && !opt.gc_interval && prefer_grow(e)) ? 1u : 0u;
        P.profile = opt.profile;
        void* args[] = {&P};
        cudaEventRecord(a, e->stream);
        reset_barrier(e);
        reset_barrier(e);
    cudaError_t err = cudaLaunchCooperativeKernel(step_loop_for(e->W, e->minb), blocks, kBlock, args, dyn_smem(e), e->stream);
        cudaEventRecord(b, e->stream);
        st.launches++;
        if (err != cudaSuccess) {
            result = fail(e, TRS_GPU_CUDA, std::string("step loop launch: ") + cudaGetErrorString(err));
            break;
        }
        err = cudaEventSynchronize(b);
        if (err != cudaSuccess) {
            result = fail(e, TRS_GPU_CUDA, std::string("step loop: ") + cudaGetErrorString(err));
            break;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        total_ms += ms;
        Ctl c;
        if (cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost) != cudaSuccess) {
            result = fail(e, TRS_GPU_CUDA, "control block copy");
            break;
        }
        if (c.status == kDone) break;
        if (c.status == kStepBudget) {
            result = fail(e, TRS_GPU_STEP_BUDGET,
                          "step budget of " + std::to_string(P.step_budget) +
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
            int r = grow_trace(e);
            if (r) { result = r; break; }
            continue;
        }
        if (c.status == kNeedGrow) {
            uint32_t s = c.sweep + 1;
            uint64_t m = c.ctr[s & 3].count;
            st.regrows++;
            int r = grow_store(e, (uint64_t)c.base + m * e->max_new + 1 + (1u << 20));
            if (r) { result = r; break; }
            continue;
        }
        result = fail(e, TRS_GPU_CUDA, "step loop ended in an unknown state");
        break;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    Ctl c{};
    cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost);
    st.total_rewrites = c.total_rewrites;
    st.max_width = c.max_width;
    st.sweeps = c.sweep - sweep0;
    st.gc_runs = c.gc_runs;
    st.small_sweeps = c.small_sweeps;
    st.peak_slots = c.peak_base;
    st.live_terms = c.base - 1;
    st.kernel_ms = total_ms;
    st.gc_ms = c.gc_ns * 1e-6;
    st.load_ms = e->load_ms;
    e->last_sweeps = c.sweep - sweep0;
    if (result == TRS_GPU_OK && opt.validate) {
        // refcount ghost invariant (sweep_engine.cpp:335-359): rc of every
        // uncollected slot = references from uncollected slots + root pins
        HostArena h;
        std::vector<uint32_t> roots;
        int r = fetch_arena(e, h, roots);
        if (r) return r;
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
    }
    if (stats) *stats = st;
    return result;
}

void* trs_gpu_stream(trs_gpu_engine* e) { return e ? (void*)e->stream : nullptr; }

int trs_gpu_profile_counters(trs_gpu_engine* e, uint64_t* out6) {
    if (!e || !e->d_ctl || !out6) return TRS_GPU_INVALID;
    Ctl c;
    CUDA_TRY(e, cudaMemcpy(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 6; ++k) out6[k] = c.prof[k];
    return TRS_GPU_OK;
}

int trs_gpu_compact(trs_gpu_engine* e, uint32_t max_rounds, trs_gpu_stats* stats) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    Ctl c0;
    CUDA_TRY(e, cudaMemcpy(&c0, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    Params P{};
    P.arena[0] = e->d_arena[0];
    P.arena[1] = e->d_arena[1];
    P.list[0] = e->d_list[0];
    P.list[1] = e->d_list[1];
    P.gcmap = e->d_gcmap;
    P.blocksum = e->d_blocksum;
    P.roots = e->d_roots;
    P.num_roots = e->num_roots;
    P.ctl = e->d_ctl;
    P.trace = e->d_trace;
    P.trace_cap = e->trace_cap;
    P.prog = e->d_prog;
    P.prog_bytes = (uint32_t)e->blob.size();
    P.capacity = e->capacity;
    P.max_new = e->max_new;
    P.sweep0 = c0.sweep;
    P.allow_gc = 1;
    P.compact_only = max_rounds ? max_rounds : 8;
    const int blocks = grid_blocks(e, 0);
    void* args[] = {&P};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, e->stream);
    reset_barrier(e);
    cudaError_t err = cudaLaunchCooperativeKernel(step_loop_for(e->W, e->minb), blocks, kBlock, args, dyn_smem(e), e->stream);
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
        stats->live_terms = c.base - 1;
        stats->peak_slots = c.base;
        stats->grid_blocks = blocks;
        stats->block_threads = kBlock;
        stats->record_words = e->W;
    }
    return TRS_GPU_OK;
}

int trs_gpu_fetch_records(trs_gpu_engine* e, void* dst, uint64_t cap_bytes, uint64_t* bytes, uint32_t* record_words,
                          uint32_t* roots_out) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    Ctl c;
    CUDA_TRY(e, cudaMemcpyAsync(&c, e->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    uint64_t need = (uint64_t)c.base * e->W * 4;
    if (bytes) *bytes = need;
    if (record_words) *record_words = (uint32_t)e->W;
    if (!dst || cap_bytes < need) return TRS_GPU_OK;
    CUDA_TRY(e, cudaMemcpyAsync(dst, e->d_arena[c.arena], need, cudaMemcpyDeviceToHost, e->stream));
    if (roots_out)
        CUDA_TRY(e, cudaMemcpyAsync(roots_out, e->d_roots, sizeof(uint32_t) * e->num_roots, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(e, cudaStreamSynchronize(e->stream));
    return TRS_GPU_OK;
}

int trs_gpu_trace(trs_gpu_engine* e, trs_gpu_sweep_record* out, uint64_t cap, uint64_t* count) {
    if (!e || !e->d_trace) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    uint64_t n = std::min<uint64_t>(e->last_sweeps, e->trace_cap);
    if (count) *count = n;
    if (out && cap) CUDA_TRY(e, cudaMemcpy(out, e->d_trace, sizeof(trs_gpu_sweep_record) * std::min(n, cap), cudaMemcpyDeviceToHost));
    return TRS_GPU_OK;
}

int trs_gpu_canonical(trs_gpu_engine* e, uint32_t root_index, uint32_t* words, uint64_t cap, uint64_t* n_words,
                      uint32_t* n_nodes) {
    if (!e || !e->loaded) return TRS_GPU_INVALID;
    if (root_index >= e->num_roots) return fail(e, TRS_GPU_INVALID, "root index out of range");
    cudaSetDevice(e->device);
    HostArena h;
    std::vector<uint32_t> roots;
    int rc = fetch_arena(e, h, roots);
    if (rc) return rc;
    // iterative pre-order, first-visit ids
    std::vector<uint32_t> id(h.base, UINT32_MAX);
    std::vector<uint32_t> order;
    std::vector<uint32_t> stack{roots[root_index]};
    auto check = [&](uint32_t slot) {
        return slot != 0 && slot < h.base && h.rec(slot)[kWHead] != kDeadHead;
    };
    if (!check(roots[root_index])) return fail(e, TRS_GPU_DANGLING, "root is not a live term");
    uint64_t nw = 0;
    while (!stack.empty()) {
        uint32_t x = stack.back();
        stack.pop_back();
        if (id[x] != UINT32_MAX) continue;
        id[x] = (uint32_t)order.size();
        order.push_back(x);
        const uint32_t* R = h.rec(x);
        uint32_t ar = e->arity[R[kWHead] & kSymMask];
        nw += 1 + ar;
        for (uint32_t j = ar; j-- > 0;) {
            uint32_t c = R[kWArgs + j];
            if (!check(c))
                return fail(e, TRS_GPU_DANGLING, "slot " + std::to_string(c) + " is not a live term");
            stack.push_back(c);
        }
    }
    if (n_words) *n_words = nw;
    if (n_nodes) *n_nodes = (uint32_t)order.size();
    if (!words || cap < nw) return TRS_GPU_OK;
    uint64_t k = 0;
    for (uint32_t x : order) {
        const uint32_t* R = h.rec(x);
        uint32_t sym = R[kWHead] & kSymMask;
        words[k++] = sym;
        uint32_t ar = e->arity[sym];
        for (uint32_t j = 0; j < ar; ++j) words[k++] = id[R[kWArgs + j]];
    }
    return TRS_GPU_OK;
}

int trs_gpu_fetch_store(trs_gpu_engine* e, uint32_t* n, uint32_t* roots_out, uint32_t* hss, uint32_t* args,
                        uint32_t* refcounts, uint8_t* nf, uint32_t cap) {
    if (!e || !e->loaded || !n) return TRS_GPU_INVALID;
    cudaSetDevice(e->device);
    HostArena h;
    std::vector<uint32_t> roots;
    int rc = fetch_arena(e, h, roots);
    if (rc) return rc;
    // renumber live slots 1..n-1 in arena order
    std::vector<uint32_t> map(h.base, 0);
    uint32_t next = 1;
    for (uint32_t i = 1; i < h.base; ++i)
        if (h.rec(i)[kWHead] != kDeadHead) map[i] = next++;
    *n = next;
    if (!hss) return TRS_GPU_OK;
    if (cap < next) return fail(e, TRS_GPU_INVALID, "fetch buffer too small");
    const uint32_t ma = e->max_arity;
    hss[0] = 0;
    if (refcounts) refcounts[0] = 0;
    if (nf) nf[0] = 0;
    if (args)
        for (uint32_t j = 0; j < ma; ++j) args[(size_t)j * next] = 0;
    for (uint32_t i = 1; i < h.base; ++i) {
        const uint32_t* R = h.rec(i);
        if (R[kWHead] == kDeadHead) continue;
        uint32_t k = map[i];
        uint32_t sym = R[kWHead] & kSymMask;
        hss[k] = sym;
        if (refcounts) refcounts[k] = R[kWRc];
        if (nf) nf[k] = R[kWEpoch] != 0;
        uint32_t ar = e->arity[sym];
        if (args)
            for (uint32_t j = 0; j < ma; ++j) args[(size_t)j * next + k] = j < ar ? map[R[kWArgs + j]] : 0;
    }
    if (roots_out)
        for (uint32_t r = 0; r < roots.size(); ++r) roots_out[r] = map[roots[r]];
    return TRS_GPU_OK;
}

int trs_gpu_gather_probe(int device, uint64_t bytes, uint32_t bytes_per_access, uint32_t iters, double* gbps) {
    if (!gbps || (bytes_per_access != 4 && bytes_per_access != 8 && bytes_per_access != 16)) return TRS_GPU_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return TRS_GPU_CUDA;
    uint64_t words = bytes / 4;
    const uint32_t n = 1u << 28;  // accesses per launch
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
    uint32_t vec = bytes_per_access / 4;
    gather_probe_kernel<<<sms * 8, 512>>>(data, words, idx, n, vec, sink);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (uint32_t k = 0; k < iters; ++k) gather_probe_kernel<<<sms * 8, 512>>>(data, words, idx, n, vec, sink);
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

}  // extern "C"

// The step loop: one persistent cooperative launch runs every sweep.
//
// A sweep (the reference's derive_phase + fold, sweep_engine.cpp:69-188)
// processes the awake frontier in chunks of q <= 32 entries, one entry per
// lane, with warps running independently: no CTA-wide barrier inside a sweep.
//  * Derive: record, children and (planned) grandchildren loaded level by
//    level; the rule chosen by match tables, or by generated compare chains
//    in the per-program specialisation (TRS_GEN, jit.hpp).
//  * Fresh slots come from per-warp slabs (one atomic per slab, not per
//    rewrite; get_new_index, term_store.cpp:118-138).
//  * Next-frontier pushes go to the CTA's own region of the output list,
//    sized in closed form (cta_prefix), through a shared-memory counter; the
//    region table (offset, count, rewrites) is read back after the grid
//    barrier, so a sweep has no contended global atomics at all.
//  * Tiny frontiers run on CTA 0 alone out of shared memory (single-CTA
//    mode), frontiers of <= 32 slots on one warp of it (warp mode), a single
//    slot on one lane (solo), with __syncthreads / __syncwarp / nothing
//    instead of the grid barrier; small stores move into shared memory
//    altogether (the resident arena).
#pragma once

#include "gc.cuh"
#include "validate.cuh"

namespace trs_b200 {

// Variable bindings of the lane's chosen rule live in dynamic shared memory
// (Params::max_vars columns of kBlock words, one column entry per thread:
// bank-conflict free for equal indices).  As a dynamically indexed
// per-thread array they would live in local memory, whose lines the random
// gathers evict from L1, and every RHS reference to a variable would become
// an L2 round trip on the rewrite's critical path.
#define TRS_BIND(v) C.bind[(v) * kBlock]

// Dynamic shared memory after the program: two frontier lists of the
// single-CTA mode, the binding columns, then the resident arena.
__device__ __forceinline__ uint32_t* bind_base(const Params& P, uint32_t* slist) {
    return slist + 2 * kSmallCap + threadIdx.x;
}

enum Act : uint32_t { kActNone = 0, kActWait, kActNf, kActCollapse, kActBuild, kActDefer, kActChain };

// The slot a lane last published nf in this physical sweep, with the head
// and epoch words it wrote (run-ahead: its parent is usually the lane's next
// step, and reads them without a round trip)
struct NfCarry {
    uint32_t slot, head, epoch;
};

struct Slab {
    uint32_t cur, end;  // warp-uniform: [cur, end) are this warp's unused fresh slots
    uint32_t room;      // warp-uniform: the sweep's claims leave room for run-ahead
};

// Mark a warp's unused slab slots dead so collections and copies skip them.
template <int W, bool kSolo = false>
__device__ __forceinline__ void abandon_slab(uint32_t* arena, Slab& slab) {
    const uint32_t lane = kSolo ? 0u : (threadIdx.x & 31);
    // the whole record: collections and copies read the first quad (and
    // move whole records) of every slot below the bump pointer
    for (uint32_t x = slab.cur + lane; x < slab.end; x += kSolo ? 1u : 32u) {
        uint4* R = reinterpret_cast<uint4*>(rec<W>(arena, x));
        R[0] = make_uint4(kDeadHead, 0u, 0u, 0u);
#pragma unroll
        for (int q = 1; q < W / 4; ++q) R[q] = make_uint4(0u, 0u, 0u, 0u);
    }
    slab.cur = slab.end = 0;
}

// Width accounting (logical time): one rewrite in the histogram entry h.
// Lanes whose entry equals the first rewriting lane's are folded into one
// add (a whole wide sweep's warp usually shares one logical sweep).  A grid
// sweep first adds into a CTA-shared window of kHistWin sweeps from its own
// logical sweep (flushed once per CTA and sweep): every warp of a wide sweep
// hitting the same global entry would serialise in one L2 slice.
constexpr uint32_t kHistWin = 32;
template <bool kSolo, typename Ctr>
__device__ __forceinline__ void hist_add(Ctr* h, bool on) {
    if (kSolo) {
        if (on) atomicAdd(h, (Ctr)1);
        return;
    }
    const uint32_t act = __ballot_sync(0xffffffffu, on);
    if (!act) return;
    const int first = __ffs(act) - 1;
    const unsigned long long mine = reinterpret_cast<unsigned long long>(h);
    const unsigned long long lead = __shfl_sync(0xffffffffu, mine, first);
    const uint32_t same = __ballot_sync(0xffffffffu, on && mine == lead);
    const int lane = threadIdx.x & 31;
    if (on && (mine != lead || lane == first)) atomicAdd(h, mine != lead ? (Ctr)1 : (Ctr)__popc(same));
}

// Warp collectives of the warp step, or their one-lane identities when a
// single entry is swept by lane 0 alone (kSolo: the narrow sweeps of the
// latency-bound configs, where the scans and ballots are pure path length).
template <bool kSolo>
__device__ __forceinline__ uint32_t w_scan(uint32_t x) {
    return kSolo ? x : warp_incl_scan(x);
}
template <bool kSolo>
__device__ __forceinline__ uint32_t w_bcast(uint32_t v, int src) {
    return kSolo ? v : __shfl_sync(0xffffffffu, v, src);
}

struct StepCtx {
    uint32_t s;           // logical sweep of this physical sweep when there is no run-ahead (then they coincide)
    uint32_t bump;        // slot base of claims made during this sweep
    uint32_t* claim_ctr;  // slots claimed during this sweep (relative to bump)
    uint32_t* out;        // output region of the next frontier
    uint32_t* push_ctr;   // entries pushed into `out` (shared memory)
    uint32_t* flags;      // CTA-shared kFlag* word of this sweep
    uint64_t cap;         // slots of the arena being swept (global or shared-memory resident)
    uint32_t slab;        // fresh slots a warp claims at a time (0: exactly what a step needs)
    uint32_t* bind;       // this thread's binding column (TRS_BIND)
    // logical time (oracle_logical): slots derive at T = max(earliest sweep,
    // argument nf epochs + 1); widths go to hist[T - t0]
    uint32_t t0;          // the run's first logical sweep (earliest sweep of an input slot)
    unsigned long long* hist;
    uint32_t hist_cap;
    uint32_t* hwin;       // CTA-shared width window [hbase, hbase + kHistWin) (null: global adds)
    uint32_t hbase;
    uint32_t stamp;       // physical sweep mod 16, published with nf epochs
    uint32_t ra;          // the run may run ahead: readiness by stamps, not by sweep number
    // run-ahead: a lane carries on with a slot its own step made ready
    // instead of pushing it to the next sweep; every step is backed by
    // cont_cost reserved push entries of the output list (cont_room, null:
    // no run-ahead), and slabs stop feeding it past claim_soft
    int* cont_room;
    uint32_t cont_cost;
    uint32_t lone;        // single-CTA modes: push_ctr counts the whole next frontier
    uint32_t claim_soft;
};

// Phase cycle accounting is compiled only into the profiling build
// (libtrs_b200_prof.so, -DTRS_B200_PROFILE=1) so that the production step
// loop carries none of its registers.
constexpr bool kProfBuild = TRS_B200_PROFILE != 0;
// TRS_GEN: this translation unit is the per-program specialisation compiled
// at set_program by NVRTC (engine.cu, jit_compile); the generated functions
// gen_bind / gen_csrc / gen_build are defined before this header.
#ifndef TRS_GEN
#define TRS_GEN 0
#endif
#ifndef TRS_GEN_ALL_TABLES
#define TRS_GEN_ALL_TABLES 0
#endif
// The rich frontier-entry format (record payloads in the list) is compiled
// only on request (-DTRS_B200_RICH_ENTRIES=1): its extra inlined copy of the
// warp step doubles the grid sweep's code for an opt-in format.
#ifndef TRS_B200_RICH_ENTRIES
#define TRS_B200_RICH_ENTRIES 0
#endif
#ifndef TRS_B200_LONE
#define TRS_B200_LONE 1
#endif
#ifndef TRS_B200_PUB_FAST
#define TRS_B200_PUB_FAST 1
#endif
#ifndef TRS_B200_NF_CARRY
#define TRS_B200_NF_CARRY 1
#endif
#ifndef TRS_B200_RA_PREFETCH_LONE
#define TRS_B200_RA_PREFETCH_LONE 0
#endif
#ifndef TRS_B200_RA_PREFETCH
#define TRS_B200_RA_PREFETCH 1
#endif

struct PhaseClock {
    long long t[4] = {0, 0, 0, 0};  // match, claim, apply, push (debug accounting)
    long long steps = 0;            // warp steps accounted
    long long sub[4] = {0, 0, 0, 0};  // match sub-phases: entry+record, children, slots, rules
    long long last = 0;
    // close a sub-phase once value v has arrived (the MOV waits on its scoreboard)
    __device__ __forceinline__ void mark(int k, uint32_t v) {
        uint32_t d;
        asm volatile("mov.b32 %0, %1;" : "=r"(d) : "r"(v));
        long long now = clock64() + (d & 0);
        sub[k] += now - last;
        last = now;
    }
};

// Frontier entries are bare slot ids.  The opt-in rich format
// (TRS_B200_RICH_ENTRIES) holds W words laid out like a record,
//   [slot, head|cursor, has_payload, 0, args...],
// where the pusher copies the node's head and arguments whenever it knows
// them (fresh nodes, rewritten roots, polls): the node cannot change
// before its own next derive, so the next sweep skips its record gather.
constexpr uint32_t kEntHasPayload = 1;

// One entry per lane: derive (sweep_engine.cpp:163-188), claim, apply
// (:190-258), push.  Every lane of the warp must call it (valid or not),
// except in the solo form (kSolo), which lane 0 runs alone for a one-entry
// sweep.  Returns the warp's number of rewrites.

// kRA: the run-ahead build of the step loop (continuations, publication
// stamps, logical derive sweeps); without it logical and physical sweeps
// coincide and the step is the lean synchronous one.
template <int W, bool kRich, bool kRA, int kSolo = 0>
__device__ __forceinline__ uint32_t warp_step(const Params& P, const Prog& G, uint32_t* arena, const StepCtx& C,
                                              Slab& slab, bool valid, const uint32_t* entry, bool prof_req,
                                              PhaseClock& pc, bool may_cont, uint32_t& cont, uint32_t& tmax,
                                              NfCarry& just_nf, uint32_t& pushes) {
    const bool prof = kProfBuild && prof_req;
    // kSolo 1: lane 0 alone on the device (plain counters); 2: one lane of
    // its warp in a grid sweep (atomics, but no warp collectives)
    constexpr bool kAlone = kSolo != 0;
    constexpr int MAXA = rec_args(W);
    // arguments any symbol of the program has: the specialisation knows it,
    // so loops over arguments stop there and their registers disappear
#if TRS_GEN
    constexpr int AE = TRS_GEN_MAXA < MAXA ? TRS_GEN_MAXA : MAXA;
#else
    constexpr int AE = MAXA;
#endif
    const uint32_t s = C.s;
    const uint32_t lane = threadIdx.x & 31;
    long long c0 = prof ? clock64() : 0;
    if (prof) {
        pc.steps++;
        pc.last = c0;
    }
    uint32_t act = kActNone;
    uint32_t i = 0, sym = 0, ar = 0, rule = 0, wchild = 0, wpos = 0, cursor = 0;
    uint32_t T = 0;  // logical sweep of this derive
    uint32_t chain_k = 0, chain_f = 0;  // run-ahead: constant-chain rewrites taken in registers, final symbol
    uint32_t a[MAXA];
    // level-synchronous matcher state (DPlan): children's first argument
    // quads, grandchild slot heads, and the argument quads of two slots
    uint32_t ch[MAXA];
    uint32_t ca[kPlanChildren * 4];
    uint32_t gh[kPlanSlots];
    uint32_t ga[kPlanArgSlots * 4];
    uint32_t cs_head = 0, cs_b[4] = {0, 0, 0, 0};  // collapse source record taken from registers
    uint32_t own_waiter = 0;  // the record's waiter word as loaded (the nf publication's first guess)
    uint32_t own_epoch = 0;   // the record's epoch word (earliest derive sweep while not nf)
#if TRS_GEN
    bool gb_ready = false;       // set by the match-table path; the walks bind through shared memory
    uint32_t gb[TRS_GEN_MAXV];  // the chosen rule's bindings, in registers (constant indices only)
#pragma unroll
    for (int v = 0; v < TRS_GEN_MAXV; ++v) gb[v] = 0;
#endif
    bool planned = false;
    if (valid) {
        uint32_t headw;
        bool have = false;
        if (kRich) {
            const uint4 q0 = *reinterpret_cast<const uint4*>(entry);
            i = q0.x;
            headw = q0.y;
            own_epoch = rec<W>(arena, i)[kWEpoch];
            have = q0.z == kEntHasPayload;
            if (have) {
#pragma unroll
                for (int q = 0; q < MAXA / 4; ++q) {
                    const uint4 v = *reinterpret_cast<const uint4*>(entry + kWArgs + q * 4);
                    a[q * 4 + 0] = v.x;
                    a[q * 4 + 1] = v.y;
                    a[q * 4 + 2] = v.z;
                    a[q * 4 + 3] = v.w;
                }
            }
        } else {
            i = *entry;
        }
        if (!have) {
            // head and the first argument quad share the record's first
            // sector: issue both loads together
            const uint32_t* R = rec<W>(arena, i);
            const uint4 h4 = *reinterpret_cast<const uint4*>(R);
            const uint4 a4 = *reinterpret_cast<const uint4*>(R + kWArgs);
            headw = h4.x;
            own_epoch = h4.y;
            own_waiter = h4.w;
            a[0] = a4.x;
            a[1] = a4.y;
            a[2] = a4.z;
            a[3] = a4.w;
            const uint32_t har = G.arity[headw & kSymMask];
#pragma unroll
            for (int q = 1; q < MAXA / 4; ++q) {
                if ((uint32_t)(q * 4) < har) {
                    const uint4 v = *reinterpret_cast<const uint4*>(R + kWArgs + q * 4);
                    a[q * 4 + 0] = v.x;
                    a[q * 4 + 1] = v.y;
                    a[q * 4 + 2] = v.z;
                    a[q * 4 + 3] = v.w;
                } else {
                    a[q * 4 + 0] = a[q * 4 + 1] = a[q * 4 + 2] = a[q * 4 + 3] = 0;
                }
            }
        }
        if (prof) pc.mark(0, headw ^ a[0]);
        sym = headw & kSymMask;
        cursor = headw >> kSymBits;
        ar = G.arity[sym];
        const DPlan pl = G.plans[sym];
        // level 1 -- subterm scan (sweep_engine.cpp:173-178): every child's
        // head and nf epoch, plus the argument quads the plan needs, issued
        // together
        uint32_t cep[MAXA];
#pragma unroll
        for (int j = 0; j < MAXA; ++j) {
            ch[j] = 0;
            cep[j] = 1;
        }
#pragma unroll
        for (int j = 0; j < (int)kPlanChildren * 4; ++j) ca[j] = 0;
#pragma unroll
        for (int j = 0; j < AE; ++j) {
            if ((uint32_t)j < ar) {
                const uint32_t* C = rec<W>(arena, a[j]);
                if (j < (int)kPlanChildren && ((pl.child_args >> j) & 1u)) {
                    const uint4 q0 = *reinterpret_cast<const uint4*>(C);
                    const uint4 q1 = *reinterpret_cast<const uint4*>(C + kWArgs);
                    ch[j] = q0.x & kSymMask;
                    cep[j] = q0.y;
                    ca[j * 4 + 0] = q1.x;
                    ca[j * 4 + 1] = q1.y;
                    ca[j * 4 + 2] = q1.z;
                    ca[j * 4 + 3] = q1.w;
                } else if (kRA && TRS_B200_NF_CARRY && a[j] == just_nf.slot) {
                    // the argument this lane has just made nf: its head and
                    // epoch are in registers (an nf record no longer changes)
                    ch[j] = just_nf.head;
                    cep[j] = just_nf.epoch;
                } else {
                    const uint2 c = *reinterpret_cast<const uint2*>(C);
                    ch[j] = c.x & kSymMask;
                    cep[j] = c.y;
                }
            }
        }
        if (prof) pc.mark(1, cep[0] ^ cep[MAXA - 1] ^ ca[0]);
        // run-ahead in a grid sweep: a lane that carries on into a node it
        // builds from these grandchildren (a spine, Plus(S(X), Y) ->
        // S(Plus(X, Y))) reads their records in its next step: start those
        // misses now (words past an arity are slot 0).  Grid sweeps only: the
        // single-CTA modes' chains run from L1 or the resident arena, where
        // the extra instructions measured slower (tools/knob_ab.py)
        if (kRA && kSolo != 1 && (!C.lone || TRS_B200_RA_PREFETCH_LONE) && may_cont && C.cont_room &&
            TRS_B200_RA_PREFETCH) {
#pragma unroll
            for (int q = 0; q < (int)kPlanChildren * 4; ++q)
                if (ca[q]) asm volatile("prefetch.L1 [%0];" ::"l"(rec<W>(arena, ca[q])));
        }
        // Logical derive sweep (oracle_logical): one past the slot's build or
        // last rewrite, and past every argument's nf epoch.  An argument that
        // is not nf -- or whose nf is too fresh to read: published in this
        // physical sweep (without run-ahead: in this sweep, nf_read,
        // sweep_engine.cpp:80-81; with run-ahead: by another lane, whose
        // record writes need not be visible yet) -- is pending, and the slot
        // waits on the first such argument (:173-178).
        // (synchronous build: every derive of physical sweep s happens at
        // logical sweep s, the reference's own schedule)
        T = kRA ? ((own_epoch & kTminBit) ? max(own_epoch & ~kTminBit, C.t0) : C.t0) : s;
        bool pending = false;
#pragma unroll
        for (int j = AE - 1; j >= 0; --j) {
            if ((uint32_t)j < ar) {
                const uint32_t e = cep[j];
                const bool ready = epoch_nf(e) && (kRA ? (((e >> kEpochBits) & kStampMask) != C.stamp ||
                                                          a[j] == just_nf.slot)
                                                       : (e & kEpochMask) < s);
                if (kRA && ready) T = max(T, (e & kEpochMask) + 1);
                if (!ready) {
                    pending = true;
                    wpos = j;
                }
            }
        }
        if (pending) {
            act = kActWait;
            wchild = pick(a, wpos);
        } else if (T - C.t0 >= C.hist_cap || T >= kEpochMask - 1) {
            // past the width histogram: the host grows it (kPlanTrace)
            act = kActDefer;
        } else if (kRA && ar == 0 && G.chain && G.chain[sym] < kChainNf) {
            // a constant chain: its rewrites happen at T, T + 1, ... whatever
            // else happens (nothing is read), so they are taken here, in
            // registers, and only the final state is written
            uint32_t f = sym, k = 0;
            while (k < kChainMax && G.chain[f] < kChainNf && T + k + 1 - C.t0 < C.hist_cap) {
                f = G.chain[f];
                ++k;
            }
            chain_k = k;
            chain_f = f;
            act = G.chain[f] == kChainNf ? kActNf : kActChain;
        } else if (pl.fast) {
            planned = true;
            // level 2: grandchild slots (nf below an nf child: stable)
#pragma unroll
            for (int q = 0; q < (int)kPlanSlots; ++q) {
                gh[q] = 0;
                if (q < (int)kPlanArgSlots) ga[q * 4 + 0] = ga[q * 4 + 1] = ga[q * 4 + 2] = ga[q * 4 + 3] = 0;
                if ((uint32_t)q < pl.nslots) {
                    const uint32_t node = pick(ca, pl.slot_jk[q]);
                    const uint32_t* N = rec<W>(arena, node);
                    if (q < (int)kPlanArgSlots && ((pl.slot_args >> q) & 1u)) {
                        const uint4 q0 = *reinterpret_cast<const uint4*>(N);
                        const uint4 q1 = *reinterpret_cast<const uint4*>(N + kWArgs);
                        gh[q] = q0.x & kSymMask;
                        ga[q * 4 + 0] = q1.x;
                        ga[q * 4 + 1] = q1.y;
                        ga[q * 4 + 2] = q1.z;
                        ga[q * 4 + 3] = q1.w;
                    } else {
                        gh[q] = N[kWHead] & kSymMask;
                    }
                }
            }
            if (prof) pc.mark(2, gh[0] ^ ga[0]);
            // first matching rule in source order (dispatch.hpp:119-130),
            // every step answered from registers
            int chosen = -1;
#if TRS_GEN
            if (pl.fast & kPlanTables) {
                // specialised: the symbol's checks as compare chains against
                // constants (first match in source order), then the bindings
                chosen = gen_choose(sym, ch, gh);
                if (chosen >= 0) {
                    gen_bind<W>((uint32_t)chosen, a, ch, ca, gh, ga, gb, cs_head, cs_b);
                    gb_ready = true;
                }
            }
#endif
#if TRS_GEN && TRS_GEN_ALL_TABLES
            // every symbol with rules has match tables: the walks below are
            // unreachable (a planned symbol without tables has no rules)
#else
#if TRS_GEN
            else
#endif
            if (pl.fast & kPlanTables) {
                // match tables: AND the rule masks of every checked position
                // (static register reads, no walk over the rules), then bind
                // the chosen rule's variables
                const uint16_t* rows = G.mrow + sym * G.npos;
                const uint32_t nr = G.rule_begin[sym + 1] - G.rule_begin[sym];
                uint32_t mask = nr >= 32 ? 0xFFFFFFFFu : (1u << nr) - 1u;
#pragma unroll
                for (int q = 0; q < AE; ++q) {
                    const uint16_t row = rows[q];
                    if (row != kNoRow) mask &= G.mtab[row + ch[q]];
                }
#pragma unroll
                for (int q = 0; q < (int)kPlanSlots; ++q) {
                    const uint16_t row = rows[MAXA + q];
                    if (row != kNoRow) mask &= G.mtab[row + gh[q]];
                }
                if (mask) {
                    chosen = (int)(G.rule_begin[sym] + __ffs(mask) - 1);
#if TRS_GEN
                    gen_bind<W>((uint32_t)chosen, a, ca, ga, gb);
                    gb_ready = true;
#else
                    const DRule& Rl = G.rules[chosen];
                    for (uint32_t t = 0; t < Rl.num_steps; ++t) {
                        const DStep st = G.steps[Rl.first_step + t];
                        if (st.kind == 0) continue;
                        const uint32_t src = st.src;
                        TRS_BIND(st.value) = src < kSrcSlot ? pick(a, src)
                                             : src < kSrcSArg ? pick(ca, src & 15u)
                                                              : pick(ga, src & 7u);
                    }
#endif
                }
            } else {
                for (uint32_t r = G.rule_begin[sym]; r < G.rule_begin[sym + 1]; ++r) {
                    const DRule& Rl = G.rules[r];
                    bool ok = true;
                    for (uint32_t t = 0; t < Rl.num_steps; ++t) {
                        const DStep st = G.steps[Rl.first_step + t];
                        const uint32_t src = st.src;
                        if (st.kind == 0) {
                            const uint32_t head = src < kSrcSlot ? pick(ch, src) : pick(gh, src & 3u);
                            if (head != st.value) {
                                ok = false;
                                break;
                            }
                        } else {
                            const uint32_t node = src < kSrcSlot ? pick(a, src)
                                                  : src < kSrcSArg ? pick(ca, src & 15u)
                                                                   : pick(ga, src & 7u);
                            TRS_BIND(st.value) = node;
                        }
                    }
                    if (ok) {
                        chosen = (int)r;
                        break;
                    }
                }
            }
#endif
            if (chosen < 0) {
                act = kActNf;
            } else {
                rule = (uint32_t)chosen;
                const DRule& Rl = G.rules[rule];
                act = Rl.collapse ? kActCollapse : kActBuild;
#if TRS_GEN
                if (!gb_ready && Rl.collapse && Rl.csrc != kNone) {  // gen_bind set them on the table path
#else
                if (Rl.collapse && Rl.csrc != kNone) {
#endif
                    const uint32_t cs = Rl.csrc;
                    cs_head = cs < kSrcSlot ? pick(ch, cs) : pick(gh, cs & 3u);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        cs_b[k] = cs < kSrcSlot ? pick(ca, (cs & 3u) * 4 + k) : pick(ga, (cs & 1u) * 4 + k);
                }
            }
        } else {
#if TRS_GEN && TRS_GEN_ALL_TABLES
            act = kActNf;  // unreachable: every symbol is planned
#else
            // interpreted matcher: one dependent gather per step below the root
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
                        TRS_BIND(st.value) = node;
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
#endif
        }
    }
#if TRS_GEN && !TRS_GEN_ALL_TABLES
    if (!gb_ready && (act == kActCollapse || act == kActBuild)) {
#pragma unroll
        for (int v = 0; v < TRS_GEN_MAXV; ++v) gb[v] = TRS_BIND(v);
    }
#endif
    if (prof) pc.mark(3, act);
    long long c1 = prof ? clock64() : 0;
    if (prof) pc.t[0] += c1 - c0;

    // ---- claim fresh slots from the warp's slab
    const uint32_t need = act == kActBuild ? G.rules[rule].new_slots : 0;
    const uint32_t incl = w_scan<kAlone>(need);
    const uint32_t total = w_bcast<kAlone>(incl, 31);
    uint32_t fresh = 0;
    if (total) {
        if (slab.end - slab.cur < total) {
            abandon_slab<W, kAlone>(arena, slab);
            const uint32_t size = max(C.slab, total);
            uint32_t off = 0;
            if (kSolo == 1) {
                // the solo step runs alone on the device: plain counters
                off = *C.claim_ctr;
                *C.claim_ctr = off + size;
            } else if (kAlone || lane == 0) {
                off = atomicAdd(C.claim_ctr, size);
            }
            off = w_bcast<kAlone>(off, 0);
            // run-ahead feeds on the slots the sweep's worst case leaves over
            if (kRA) slab.room = (uint64_t)off + size <= C.claim_soft ? 1u : 0u;
            const uint64_t start = (uint64_t)C.bump + off;
            if (start + total > C.cap) {
                // not even this step's slots fit: the reference raises
                // Capacity when get_new_index finds no slot (sweep_engine.cpp:221-226)
                if (kAlone || lane == 0) {
                    atomicExch(&P.ctl->abort_capacity, 1u);
                    atomicOr(C.flags, kFlagCapacity);
                }
                if (act == kActBuild) act = kActNone;
            } else {
                // a slab that runs past the capacity is cut at it (the sweep's
                // fold clamps the bump pointer the same way, sweep_engine.cpp:94-98)
                slab.cur = (uint32_t)start;
                slab.end = (uint32_t)min(start + size, C.cap);
            }
        }
        if (slab.end - slab.cur >= total) {
            fresh = slab.cur + incl - need;
            slab.cur += total;
        }
    }
    long long c2 = prof ? clock64() : 0;
    if (prof) pc.t[1] += c2 - c1;

    // ---- apply
    uint32_t npush = 0, push1 = 0, push_mask = 0;
    bool rewrote = false, root_push = false;
    // Each lane makes at most one round trip to a waiter word: subscribe to
    // a pending child (Wait) or publish its own nf (Nf, Collapse).  Both are
    // issued as ONE compare-and-swap after the branches below, so a warp
    // mixing the three outcomes pays one atomic latency, not three.
    uint32_t* wword = nullptr;
    uint32_t wcmp = 0, wval = 0;
    if (act == kActWait) {
        if (wpos != cursor) rec<W>(arena, i)[kWHead] = sym | (wpos << kSymBits);
        wword = rec<W>(arena, wchild) + kWWaiter;
        wcmp = 0u;
        wval = i;
    } else if (act == kActNf) {
        uint32_t* R = rec<W>(arena, i);
        if (kRA && chain_k) {
            // the chain ends in a constant without rules: nf after its last rewrite
            *reinterpret_cast<uint2*>(R) = make_uint2(chain_f, (T + chain_k) | (C.stamp << kEpochBits));
            rewrote = true;
        } else {
            R[kWEpoch] = T | (C.stamp << kEpochBits);
        }
        tmax = max(tmax, T + chain_k);
        if (kRA) just_nf = NfCarry{i, chain_k ? chain_f : sym, (T + chain_k) | (C.stamp << kEpochBits)};
        wword = R + kWWaiter;
        wcmp = own_waiter;
        wval = kWoken;
    } else if (kRA && act == kActChain) {
        // the chain stopped at a rule that builds or looks deeper (or at the
        // histogram's end): the slot carries on from there at T + chain_k
        *reinterpret_cast<uint2*>(rec<W>(arena, i)) = make_uint2(chain_f, kTminBit | (T + chain_k));
        rewrote = true;
        root_push = true;
    } else if (act == kActCollapse) {
        const DRule& Rl = G.rules[rule];
#if TRS_GEN
        const uint32_t src = gen_csrc(rule, gb);
#else
        const uint32_t src = TRS_BIND(Rl.root_ref);
#endif
        const uint32_t* S = rec<W>(arena, src);
        uint32_t shead, sar;
        uint32_t b[MAXA];
        if (planned && Rl.csrc != kNone) {
            // the source record was already in registers (a child or a slot)
            shead = cs_head;
#pragma unroll
            for (int k = 0; k < 4; ++k) b[k] = cs_b[k];
            sar = G.arity[shead];
#pragma unroll
            for (int q = 1; q < MAXA / 4; ++q) {
                if ((uint32_t)(q * 4) < sar) {
                    const uint4 v = *reinterpret_cast<const uint4*>(S + kWArgs + q * 4);
                    b[q * 4 + 0] = v.x;
                    b[q * 4 + 1] = v.y;
                    b[q * 4 + 2] = v.z;
                    b[q * 4 + 3] = v.w;
                }
            }
        } else {
            shead = S[kWHead] & kSymMask;
            sar = G.arity[shead];
            load_args<W>(S, sar, b);
        }
#pragma unroll
        for (int j = 0; j < MAXA; ++j)
            if ((uint32_t)j >= sar) b[j] = 0;
        uint32_t* R = rec<W>(arena, i);
        *reinterpret_cast<uint2*>(R) = make_uint2(shead, T | (C.stamp << kEpochBits));
        tmax = max(tmax, T);
        if (kRA) just_nf = NfCarry{i, shead, T | (C.stamp << kEpochBits)};
        store_args<W>(R, b, ar > sar ? ar : sar);
#pragma unroll
        for (int j = 0; j < MAXA; ++j) {
            if ((uint32_t)j >= sar) break;
            if (P.track_rc) rc_upd<kAlone>(rec<W>(arena, b[j]) + kWRc, 1);
        }
        wword = R + kWWaiter;
        wcmp = own_waiter;
        wval = kWoken;
        rewrote = true;
    } else if (act == kActBuild) {
        const DRule& Rl = G.rules[rule];
#if TRS_GEN
        gen_build<W, kAlone>(rule, arena, fresh, i, ar, gb, kTminBit | (T + 1), P.track_rc != 0);
#else
        const uint32_t nfresh = Rl.new_slots;
        for (uint32_t k = 0; k <= nfresh; ++k) {
            const DInstr I = G.instrs[Rl.first_instr + k];
            const uint32_t iar = G.arity[I.symbol];
            uint32_t b[MAXA];
            uint32_t vmask = 0;  // argument positions bound to variables
#pragma unroll
            for (int j = 0; j < MAXA; ++j) b[j] = 0;
#pragma unroll
            for (int j = 0; j < AE; ++j) {
                if ((uint32_t)j >= iar) break;
                const uint16_t ref = G.refs[I.first_ref + j];
                const bool var = !(ref & kRefNode);
                b[j] = var ? TRS_BIND(ref) : fresh + (ref & 0x7fff);
                vmask |= (uint32_t)var << j;
            }
            if (k < nfresh) {
                uint32_t sub = I.subscriber == kNone ? 0u : I.subscriber == kRootSub ? i : fresh + I.subscriber;
                uint32_t* F = rec<W>(arena, fresh + k);
                *reinterpret_cast<uint4*>(F) =
                    make_uint4(I.symbol | ((uint32_t)I.cursor << kSymBits), kTminBit | (T + 1), I.indegree, sub);
                // argument quads past the arity are never read, except the
                // first: a planned match loads a child's first quad whole and
                // follows a grandchild slot from it before the child's head is
                // checked, so the words past the arity must hold slot 0 (a
                // stale slot id would be dereferenced; store_args and the
                // loader keep the same invariant)
#pragma unroll
                for (int q = 0; q < MAXA / 4; ++q)
                    if (q == 0 || (uint32_t)(q * 4) < iar)
                        *reinterpret_cast<uint4*>(F + kWArgs + q * 4) =
                            make_uint4(b[q * 4], b[q * 4 + 1], b[q * 4 + 2], b[q * 4 + 3]);
            } else {
                uint32_t* R = rec<W>(arena, i);
                *reinterpret_cast<uint2*>(R) =
                    make_uint2(I.symbol | ((uint32_t)Rl.root_cursor << kSymBits), kTminBit | (T + 1));
                store_args<W>(R, b, ar > iar ? ar : iar);
            }
            // every reuse of a bound variable adds one reference (sweep_engine.cpp:251-253)
#pragma unroll
            for (int j = 0; j < AE; ++j) {
                if ((vmask >> j) == 0u) break;
                if (((vmask >> j) & 1u) && P.track_rc) rc_upd<kAlone>(rec<W>(arena, b[j]) + kWRc, 1);
            }
        }
#endif
        push_mask = Rl.push_mask;
        root_push = Rl.root_wait == kNone;
        push1 = i;
        rewrote = true;
    } else if (act == kActDefer) {
        atomicMax(&P.ctl->hist_need, T - C.t0 + 1);
        atomicOr(C.flags, kFlagHist);
    }
    // the rewritten root drops its old children (after the additions, as
    // the reference orders them; sweep_engine.cpp:255-256)
    if (rewrote && P.track_rc) {
#pragma unroll
        for (int j = 0; j < AE; ++j) {
            if ((uint32_t)j >= ar) break;
            rc_upd<kAlone>(rec<W>(arena, a[j]) + kWRc, -1);
        }
    }
    uint32_t wake = 0;  // the parent this lane's nf publication woke
    if (wword) {
        // run-ahead: the parent the nf publication will most likely wake is
        // the waiter word as loaded; its record is fetched while the CAS
        // confirms it (the next step of this lane's chain starts there)
        if (kRA && act != kActWait && own_waiter != 0u && own_waiter != kWoken)
            asm volatile("prefetch.L1 [%0];" ::"l"(rec<W>(arena, own_waiter)));  // generic: no-op on the resident arena
        uint32_t old;
        if (kSolo == 1) {
            // nothing else runs: the subscription and the publication are a
            // read and a write (an nf publication's word is the one loaded
            // with the record, unchanged since: only subscribers write it)
            old = act == kActWait ? *wword : wcmp;
            if (old == wcmp) *wword = wval;
        } else if (TRS_B200_PUB_FAST && act != kActWait && wcmp != 0u && wcmp != kWoken) {
            // the word held a subscriber when the record was loaded, and a
            // word holding a subscriber changes only by this publication
            // (a later subscriber's CAS expects 0): the swap needs no answer
            atomicExch(wword, kWoken);
            old = wcmp;
        } else {
            old = atomicCAS(wword, wcmp, wval);
        }
        if (act == kActWait) {
            // lost the subscription race (another subscriber, or the child
            // turned nf this very sweep): poll next sweep
            if (old != 0) {
                npush = 1;
                push1 = i;
            }
        } else {
            // publish nf: swap in kWoken whatever the word holds (only a
            // parent subscribing this sweep can change it under us)
            while (old != wcmp) {
                wcmp = old;
                old = atomicCAS(wword, wcmp, kWoken);
            }
            if (old != 0 && old != kWoken) wake = old;
        }
    }
    // ---- run-ahead: carry on with one slot this step made ready -- the woken
    // parent, else the rewritten root when it can derive next, else the first
    // ready fresh node -- at its logical sweep, instead of pushing it.  The
    // slot's own writes are this lane's or older than this physical sweep,
    // and its arguments' readiness is judged as above, so what it reads is
    // what the reference would read.  Every continued step is backed by
    // cont_cost reserved output entries (a refused reservation pushes).
    bool want = kRA && may_cont && slab.room != 0u &&
                (wake != 0u || ((act == kActBuild || act == kActChain) && (push_mask != 0u || root_push)));
    if (kRA && C.cont_room) {
        const uint32_t wm = kAlone ? (want ? 1u : 0u) : __ballot_sync(0xffffffffu, want);
        if (wm) {
            uint32_t ok = 0;
            if (kSolo == 1) {
                const int need = (int)C.cont_cost;
                if (*C.cont_room >= need) {
                    *C.cont_room -= need;
                    ok = 1;
                }
            } else if (kAlone || lane == 0) {
                const int need = __popc(wm) * (int)C.cont_cost;
                const int before = atomicSub(C.cont_room, need);
                if (before >= need)
                    ok = 1;
                else
                    atomicAdd(C.cont_room, need);
            }
            if (!w_bcast<kAlone>(ok, 0)) want = false;
        }
    } else {
        want = false;
    }
    cont = 0;
    if (kRA && want) {
        if (wake) {
            cont = wake;
        } else if (root_push) {
            cont = i;
            root_push = false;
        } else {
            cont = fresh + (uint32_t)(__ffs(push_mask) - 1);
            push_mask &= push_mask - 1;
        }
    } else if (wake) {
        npush = 1;
        push1 = wake;
    }
    if (act == kActBuild) npush = __popc(push_mask) + (root_push ? 1u : 0u);
    if (kRA && act == kActChain) {
        npush = root_push ? 1u : 0u;
        push1 = i;
    }
    if (act == kActDefer) {
        npush = 1;
        push1 = i;
    }
    long long c3 = prof ? clock64() : 0;
    if (prof) pc.t[2] += c3 - c2;

    pushes += npush;
    // ---- next frontier: one shared-memory reservation per warp step
    const uint32_t pincl = w_scan<kAlone>(npush);
    const uint32_t ptotal = w_bcast<kAlone>(pincl, 31);
    if (ptotal) {
        uint32_t base = 0;
        if (kSolo == 1) {
            base = *C.push_ctr;
            *C.push_ctr = base + ptotal;
        } else if (kAlone || lane == 0) {
            base = atomicAdd(C.push_ctr, ptotal);
        }
        base = w_bcast<kAlone>(base, 0);
        uint32_t pos = base + pincl - npush;
        if (npush) {
            if (act == kActBuild) {
                const DRule& Rl = G.rules[rule];
                uint32_t mask = push_mask | (root_push ? (1u << Rl.new_slots) : 0u);
                while (mask) {
                    const uint32_t k = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const bool root = k == Rl.new_slots;
                    const uint32_t slot = root ? i : fresh + k;
                    if (kRich) {
                        const DInstr I = G.instrs[Rl.first_instr + k];
                        const uint32_t iar = G.arity[I.symbol];
                        uint32_t b[MAXA];
#pragma unroll
                        for (int j = 0; j < MAXA; ++j) {
                            b[j] = 0;
                            if ((uint32_t)j < iar) {
                                const uint16_t ref = G.refs[I.first_ref + j];
                                b[j] = (ref & kRefNode) ? fresh + (ref & 0x7fff) : TRS_BIND(ref);
                            }
                        }
                        const uint32_t cur = root ? Rl.root_cursor : I.cursor;
                        uint32_t* E = C.out + (size_t)pos * W;
                        *reinterpret_cast<uint4*>(E) =
                            make_uint4(slot, I.symbol | (cur << kSymBits), kEntHasPayload, 0u);
#pragma unroll
                        for (int q = 0; q < MAXA / 4; ++q)
                            if ((uint32_t)(q * 4) < iar)
                                *reinterpret_cast<uint4*>(E + kWArgs + q * 4) =
                                    make_uint4(b[q * 4], b[q * 4 + 1], b[q * 4 + 2], b[q * 4 + 3]);
                    } else {
                        C.out[pos] = slot;
                    }
                    ++pos;
                }
            } else if (kRich) {
                uint32_t* E = C.out + (size_t)pos * W;
                if (act == kActWait) {
                    // polling: the record is exactly what this lane holds
                    *reinterpret_cast<uint4*>(E) = make_uint4(i, sym | (wpos << kSymBits), kEntHasPayload, 0u);
#pragma unroll
                    for (int q = 0; q < MAXA / 4; ++q)
                        if ((uint32_t)(q * 4) < ar)
                            *reinterpret_cast<uint4*>(E + kWArgs + q * 4) =
                                make_uint4(a[q * 4], a[q * 4 + 1], a[q * 4 + 2], a[q * 4 + 3]);
                } else {
                    *reinterpret_cast<uint4*>(E) = make_uint4(push1, 0u, 0u, 0u);  // woken: no payload
                }
            } else {
                C.out[pos] = push1;
            }
        }
    }
    if (prof) pc.t[3] += clock64() - c3;
    // (the lean build adds each sweep's width once, at its end: all its
    // rewrites happen at the sweep's own logical sweep)
    // (a constant chain's k rewrites at T .. T + k - 1, one entry at a time:
    // the lanes of a warp on the same chain add together)
    uint32_t nrw = rewrote ? (chain_k ? chain_k : 1u) : 0u;
    if (kRA) {
        const uint32_t steps = kAlone ? nrw : __reduce_max_sync(0xffffffffu, nrw);
        for (uint32_t j = 0; j < steps; ++j) {
            const bool on = j < nrw;
            const uint32_t Tj = T + j;
            if (C.hwin) {
                const bool win = on && Tj - C.hbase < kHistWin;
                hist_add<kAlone>(C.hwin + (Tj - C.hbase), win);
                hist_add<kAlone>(C.hist + (Tj - C.t0), on && !win);
            } else {
                hist_add<kAlone>(C.hist + (Tj - C.t0), on);
            }
        }
    }
    if (kAlone) return nrw;
    return kRA ? __reduce_add_sync(0xffffffffu, nrw) : __popc(__ballot_sync(0xffffffffu, rewrote));
}

// Run-ahead output entries per CTA per grid sweep, at most.
constexpr uint32_t kMaxSlack = 1u << 20;

// Whether a lane that has taken `steps` run-ahead steps for its current entry
// may take another (the physical sweep must still end, where the step budget
// and headroom are checked).
__device__ __forceinline__ bool ra_more(const Params& P, const StepCtx& C, uint32_t steps) {
    // a lone chain (single-CTA modes, nothing pushed for the next sweep yet)
    // holds nothing back and runs on; otherwise the pushed work would wait
    // for the chain's end, so a lane stops after P.ra_steps
    return steps < P.ra_steps || (C.lone && steps < 4096u && *(volatile uint32_t*)C.push_ctr == 0u);
}

// All warps of CTAs [block_rank, nblocks) process the frontier in q-entry
// chunks (chunk_lanes); returns this thread's share of the rewrite count
// (lane 0 of each warp holds its warp's count).
template <int W, bool kRich, bool kRA>
__device__ __forceinline__ unsigned long long cta_entries(const Params& P, const Prog& G, uint32_t* arena,
                                                          const StepCtx& C, const Frontier& F,
                                                          const uint32_t* __restrict__ in, uint32_t block_rank,
                                                          uint32_t nblocks, Slab& slab, bool prof, PhaseClock& pc,
                                                          uint32_t& tmax) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t gw = nblocks * kWarps;
    const uint32_t q = chunk_lanes(F.M, nblocks);
    unsigned long long rw = 0;
    uint32_t cont = 0, pushes = 0;
    NfCarry just_nf{};
    if (kRich) {
        for (uint32_t k = block_rank * kWarps + warp; k * q < F.M; k += gw) {
            const uint32_t v = k * q + lane;
            const bool valid = lane < q && v < F.M;
            const uint32_t* entry = valid ? in + (size_t)frontier_phys(F, v) * W : in;
            rw += warp_step<W, kRich, kRA>(P, G, arena, C, slab, valid, entry, prof && (TRS_B200_PROFILE || warp == 0), pc,
                                      false, cont, tmax, just_nf, pushes);
        }
        return lane == 0 ? rw : 0ull;
    }
    // Dense entries.  Each lane walks its own entries (k * q + lane, k += gw),
    // software-pipelined: the slot ids of the entry after next are loaded,
    // and the next entry's record prefetched into L2, while the current one
    // derives (a wide sweep hands each warp dozens of chunks).  A lane whose
    // step made a slot ready runs ahead with it before taking its next entry.
    auto slot_of = [&](uint32_t kk) -> uint32_t {
        const uint32_t v = kk * q + lane;
        return (lane < q && v < F.M) ? in[frontier_phys(F, v)] : 0u;  // generic: the list may be shared memory
    };
    uint32_t k = block_rank * kWarps + warp;
    uint32_t s0 = k * q < F.M ? slot_of(k) : 0u;
    uint32_t s1 = (k + gw) * q < F.M ? slot_of(k + gw) : 0u;
    if (!kRA) {
        // synchronous build: every lane of the warp steps through its entries together
        for (; k * q < F.M; k += gw) {
            const uint32_t s2 = (k + 2 * gw) * q < F.M ? slot_of(k + 2 * gw) : 0u;
            if (s1) asm volatile("prefetch.L2 [%0];" ::"l"(rec<W>(arena, s1)));
            uint32_t slot = s0;
            rw += warp_step<W, kRich, kRA>(P, G, arena, C, slab, slot != 0u, &slot,
                                           prof && (TRS_B200_PROFILE || warp == 0), pc, false, cont, tmax, just_nf,
                                           pushes);
            s0 = s1;
            s1 = s2;
        }
        return lane == 0 ? rw : 0ull;
    }
    uint32_t steps = 0;
    for (;;) {
        const bool own = lane < q && k * q + lane < F.M;
        const uint32_t busy = __ballot_sync(0xffffffffu, cont != 0u || own);
        if (!busy) break;
#if TRS_B200_LONE
        // A lone chain: one lane of the warp has work, and it is a
        // continuation.  It runs its chain without warp collectives (the
        // tails of the batches: a few chains per warp, one step per logical
        // sweep, the step's path length is the critical path), then hands
        // the warp-uniform slab state back.
        if (W == 8 && __popc(busy) == 1 && (busy & __ballot_sync(0xffffffffu, cont != 0u))) {
            uint32_t lrw = 0;
            if (cont) {
                do {
                    ++steps;
                    uint32_t slot = cont;
                    lrw += warp_step<W, kRich, kRA, 2>(P, G, arena, C, slab, true, &slot,
                                                       prof && (TRS_B200_PROFILE || warp == 0), pc,
                                                       ra_more(P, C, steps), cont, tmax, just_nf, pushes);
                } while (cont);
            }
            const int src = __ffs(busy) - 1;
            lrw = __shfl_sync(0xffffffffu, lrw, src);
            if (lane == 0) rw += lrw;
            slab.cur = __shfl_sync(0xffffffffu, slab.cur, src);
            slab.end = __shfl_sync(0xffffffffu, slab.end, src);
            slab.room = __shfl_sync(0xffffffffu, slab.room, src);
            continue;
        }
#endif
        uint32_t slot = cont;
        if (cont) {
            ++steps;
        } else if (own) {
            const uint32_t s2 = (k + 2 * gw) * q < F.M ? slot_of(k + 2 * gw) : 0u;
            // generic prefetch: a no-op when the arena is the shared-memory resident one
            if (s1) asm volatile("prefetch.L2 [%0];" ::"l"(rec<W>(arena, s1)));
            slot = s0;
            s0 = s1;
            s1 = s2;
            k += gw;
            steps = 0;
            pushes = 0;
        }
        rw += warp_step<W, kRich, kRA>(P, G, arena, C, slab, slot != 0u, &slot, prof && (TRS_B200_PROFILE || warp == 0),
                                  pc, ra_more(P, C, steps), cont, tmax, just_nf, pushes);
    }
    return lane == 0 ? rw : 0ull;
}

// ---------------------------------------------------------------------------

struct Local {
    uint32_t sweep, cur, arena, bump;  // sweep: physical sweeps of this run
    unsigned long long total, maxw;
    uint32_t gc_runs, small_sweeps, last_gc, peak_bump;
    unsigned long long gc_ns;
    uint32_t sweep0;  // logical sweeps before this run (input slots derive from sweep0 + 1)
    // run-ahead state: `ra_narrow` consecutive sweeps of at most ra_kill
    // entries switch it on (a latency-bound phase), a wider sweep off again;
    // once it has run, argument readiness is judged by publication stamps
    // (logical and physical sweeps no longer coincide)
    uint32_t ra_narrow, ra_on, ra_used;
    // a steady frontier past the widest sweep (chains, not a reduction):
    // the window's widest frontier and first sweep; ra_go: hand over now
    uint32_t ra_mref, ra_sref, ra_go;
};

__device__ __forceinline__ void load_local(Local& L, Ctl* c) {
    L.sweep = __ldcg(&c->psweep);
    L.cur = __ldcg(&c->cur);
    L.arena = __ldcg(&c->arena);
    L.bump = __ldcg(&c->bump);
    L.total = __ldcg(&c->total_rewrites);
    L.maxw = __ldcg(&c->max_width);
    L.gc_runs = __ldcg(&c->gc_runs);
    L.small_sweeps = __ldcg(&c->small_sweeps);
    L.last_gc = __ldcg(&c->last_gc_sweep);
    L.peak_bump = __ldcg(&c->peak_bump);
    L.gc_ns = __ldcg(&c->gc_ns);
    L.sweep0 = __ldcg(&c->sweep0);
    L.ra_narrow = __ldcg(&c->ra_narrow);
    L.ra_on = __ldcg(&c->ra_on);
    L.ra_used = __ldcg(&c->ra_used);
    L.ra_mref = __ldcg(&c->ra_mref);
    L.ra_sref = __ldcg(&c->ra_sref);
    L.ra_go = __ldcg(&c->ra_go);
}

__device__ __forceinline__ void store_local(const Local& L, Ctl* c) {
    c->psweep = L.sweep;
    c->cur = L.cur;
    c->arena = L.arena;
    c->bump = L.bump;
    c->total_rewrites = L.total;
    c->max_width = L.maxw;
    c->gc_runs = L.gc_runs;
    c->small_sweeps = L.small_sweeps;
    c->last_gc_sweep = L.last_gc;
    c->peak_bump = L.peak_bump;
    c->gc_ns = L.gc_ns;
    c->ra_narrow = L.ra_narrow;
    c->ra_on = L.ra_on;
    c->ra_used = L.ra_used;
    c->ra_mref = L.ra_mref;
    c->ra_sref = L.ra_sref;
    c->ra_go = L.ra_go;
    __threadfence();
}

// What to do before sweep s; identical in every CTA (pure function of Local).
enum Plan : uint32_t { kPlanSweep, kPlanGc, kPlanGrow, kPlanFinish, kPlanTrace };

__device__ __forceinline__ uint32_t plan(const Params& P, const Local& L, uint32_t m, bool just_collected,
                                         uint32_t nwarps) {
    const uint32_t s = L.sweep + 1;
    // the physical trace, and the width histogram entry of a synchronous
    // sweep (logical = physical), must exist before the sweep starts: a sweep
    // whose lanes deferred for want of an entry would shift every later
    // sweep of the lean build
    if (s > P.trace_cap || s > P.hist_cap) return kPlanTrace;
    if (m == 0) return kPlanFinish;
    // worst case: every frontier slot rewrites with the largest template,
    // plus what slab hand-offs can strand (ensure_headroom, sweep_engine.cpp:290-303)
    const uint64_t need = (uint64_t)m * P.max_new;
    const uint64_t worst = (uint64_t)L.bump + 2 * need + (uint64_t)nwarps * P.slab + 1;
    const uint64_t tight = (uint64_t)L.bump + need + 1;
    if ((P.fixed_capacity ? tight : worst) > P.capacity) {
        if (P.allow_gc && !just_collected && !P.prefer_grow) return kPlanGc;
        if (!P.fixed_capacity) return kPlanGrow;
        // fixed capacity: go ahead; a claim that does not fit aborts with
        // Capacity like the reference (sweep_engine.cpp:221-226)
    }
    // a collection that left the arena more than half full: grow instead of
    // collecting again next sweep
    if (just_collected && !P.fixed_capacity && (uint64_t)L.bump * 2 > P.capacity) return kPlanGrow;
    if (P.allow_gc && P.gc_interval && !just_collected && s - L.last_gc >= P.gc_interval) return kPlanGc;
    return kPlanSweep;
}

__device__ __forceinline__ void record(const Params& P, uint32_t s, unsigned long long width, const Local& L,
                                       uint32_t m, uint32_t mode, uint64_t ns) {
    // physical sweep record (diagnostics; the reference's widths are the
    // logical histogram, Params::hist)
    const uint32_t k = s;
    if (k == 0 || k > P.trace_cap) return;
    trs_gpu_sweep_record r;
    r.sweep = k;
    r.live_terms = L.bump - 1;  // allocated and not yet reclaimed by a compaction
    r.rewrites = width;
    r.n = L.bump;
    r.free_len = 0;
    r.active = m;
    r.mode = mode;
    r.micros_x1000 = ns;
    P.trace[k - 1] = r;
}

// Shared-memory staging of a frontier's region table: prefix over counts,
// offsets, and the sum of the per-region rewrite counts (the width of the
// sweep that wrote the buffer).  One round trip: the table is read for all
// `nblocks` possible regions together with its length, then one fused
// block scan (counts) + reduction (rewrites).  Ends synchronised.
__device__ Frontier stage_frontier(const Params& P, uint32_t buf, uint32_t nblocks, uint32_t* f_pref,
                                   uint32_t* f_off, Smem& sm, unsigned long long* width) {
    const uint32_t t0 = threadIdx.x, t1 = threadIdx.x + kBlock;
    const uint32_t R = __ldcg(&P.ctl->nregions[buf]);
    // the regions' flags, ORed over the CTA (every thread reads its regions)
    uint32_t fl = t0 < R ? __ldcg(P.region_flags + buf * kMaxGrid + t0) : 0u;
    if (t1 < R) fl |= __ldcg(P.region_flags + buf * kMaxGrid + t1);
    const uint32_t flags = (__syncthreads_or((int)(fl & kFlagCapacity)) ? kFlagCapacity : 0u) |
                           (__syncthreads_or((int)(fl & kFlagHist)) ? kFlagHist : 0u);
    if (nblocks <= kBlock) {
        // one region per thread: warp scans, then warp 0 scans the warp totals
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint32_t c = t0 < R ? __ldcg(region_cnt(P, buf) + t0) : 0u;
        if (t0 < R) f_off[t0] = __ldcg(region_off(P, buf) + t0);
        unsigned long long r = (width && t0 < R) ? __ldcg(P.region_rew + buf * kMaxGrid + t0) : 0ull;
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
            r += __shfl_xor_sync(0xffffffffu, r, o);
        }
        __shared__ uint32_t wpre[kWarps + 1];
        __shared__ unsigned long long wrw;
        if (lane == 31) sm.scan[warp] = x;
        if (lane == 0) sm.red[warp] = r;
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = lane < kWarps ? sm.scan[lane] : 0u;
            unsigned long long rr = lane < kWarps ? sm.red[lane] : 0ull;
            uint32_t xi = v;
#pragma unroll
            for (int o = 1; o < kWarps; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
                rr += __shfl_xor_sync(0xffffffffu, rr, o);
            }
            if (lane < kWarps) wpre[lane] = xi - v;
            if (lane == kWarps - 1) wpre[kWarps] = xi;
            if (lane == 0) wrw = rr;
        }
        __syncthreads();
        const uint32_t M = wpre[kWarps];
        if (t0 < R) f_pref[t0] = wpre[warp] + x - c;
        if (t0 == 0) f_pref[R] = M;
        if (width) *width = wrw;
        __syncthreads();
        Frontier F;
        F.R = R;
        F.M = M;
        F.flags = flags;
        F.pref = f_pref;
        F.off = f_off;
        return F;
    }
    uint32_t c0 = t0 < nblocks ? __ldcg(region_cnt(P, buf) + t0) : 0u;
    uint32_t c1 = t1 < nblocks ? __ldcg(region_cnt(P, buf) + t1) : 0u;
    const uint32_t o0 = t0 < nblocks ? __ldcg(region_off(P, buf) + t0) : 0u;
    const uint32_t o1 = t1 < nblocks ? __ldcg(region_off(P, buf) + t1) : 0u;
    unsigned long long rw = 0;
    if (width) {
        if (t0 < nblocks) rw += __ldcg(P.region_rew + buf * kMaxGrid + t0);
        if (t1 < nblocks) rw += __ldcg(P.region_rew + buf * kMaxGrid + t1);
    }
    if (t0 >= R) c0 = 0, rw = 0;
    if (t1 >= R) c1 = 0;
    if (t0 < R) f_off[t0] = o0;
    if (t1 < R) f_off[t1] = o1;
    // fused scan: each thread owns regions t0 and t1 = t0 + kBlock
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x0 = c0, x1 = c1;
    unsigned long long r = rw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o);
        uint32_t y1 = __shfl_up_sync(0xffffffffu, x1, o);
        if (lane >= o) x0 += y0, x1 += y1;
        r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if (lane == 31) {
        sm.scan[warp] = x0;
        sm.bcast[0] = 0;
    }
    __shared__ uint32_t scan1[kWarps];
    if (lane == 31) scan1[warp] = x1;
    if (lane == 0) sm.red[warp] = r;
    __syncthreads();
    uint32_t p0 = 0, p1 = 0, tot0 = 0, tot1 = 0;
    unsigned long long rtot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t a0 = sm.scan[w], a1 = scan1[w];
        if (w < warp) p0 += a0, p1 += a1;
        tot0 += a0;
        tot1 += a1;
        rtot += sm.red[w];
    }
    if (t0 < R) f_pref[t0] = p0 + x0 - c0;
    if (t1 < R) f_pref[t1] = tot0 + p1 + x1 - c1;
    if (threadIdx.x == 0) f_pref[R] = tot0 + tot1;
    if (width) *width = rtot;
    __syncthreads();
    Frontier F;
    F.R = R;
    F.M = tot0 + tot1;
    F.flags = flags;
    F.pref = f_pref;
    F.off = f_off;
    return F;
}

// Shared-memory state of the single-CTA mode.
struct SmallState {
    uint32_t count[2];  // frontier counts: [sc] being read, [sc ^ 1] being pushed
    uint32_t claim;     // slots claimed during the current sweep
    uint32_t flags;     // kFlag* raised in these sweeps
    uint32_t sc;
    int cont_room;      // output entries left for run-ahead steps this sweep
    uint32_t pad[2];
    Local L;            // hand-over from warp mode to the whole CTA
};

// Run-ahead switches on after P.ra_warm consecutive sweeps of at most
// P.ra_kill entries (a latency-bound phase: fib, Ackermann, reverse,
// mergesort) and off at a wider one: lanes that ran ahead reach a wide phase
// out of step, and a warp of lanes on different rules diverges.
// The lean (synchronous) build returns true instead: it hands the run over
// to the run-ahead build (kNeedRA), which switches on at its first sweep.
// An earlier hand-over, after P.ra_warm_past sweeps, applies to a steady
// frontier past the run's widest sweep: below an eighth of it and level
// within 1/16 over the window -- chains advancing one step per sweep, none
// ending (the plateaus of the batches' tails).  A reduction tree's frontier
// decays as its chains end at different sweeps, and keeps the full
// P.ra_warm: its lanes would run ahead only to poll at the next join
// (build+sum measured 15-28 % slower with a looser test).
__device__ __forceinline__ bool ra_steady(const Params& P, Local& L, uint32_t m) {
    const bool past = (unsigned long long)m * 8u < L.maxw;
    if (!past || m > L.ra_mref || (unsigned long long)m * 16u < (unsigned long long)L.ra_mref * 15u) {
        L.ra_mref = m;
        L.ra_sref = L.sweep;
        return false;
    }
    return L.sweep - L.ra_sref >= P.ra_warm_past;
}

template <bool kRA>
__device__ __forceinline__ bool ra_track(const Params& P, Local& L, uint32_t m) {
    if (!P.runahead) return false;
    const bool steady = ra_steady(P, L, m);
    if (m > P.ra_kill) {
        L.ra_narrow = 0;
        L.ra_on = 0;
        return false;
    }
    if (L.ra_narrow < P.ra_warm) ++L.ra_narrow;
    if (L.ra_narrow < P.ra_warm && !(steady && L.ra_narrow >= P.ra_warm_past)) return false;
    L.ra_go = 1;
    if (!kRA) return true;
    L.ra_on = 1;
    L.ra_used = 1;
    return false;
}

// The step context of physical sweep s over m frontier entries, swept by
// nwarps warps.  Run-ahead gets the arena slots the sweep's worst case
// (plan) leaves over, with a margin of two slabs (or two warp steps) per warp.
__device__ __forceinline__ StepCtx make_ctx(const Params& P, const Local& L, uint32_t s, uint32_t* claim_ctr,
                                            uint32_t* out, uint32_t* push_ctr, uint32_t* flags, uint64_t cap,
                                            uint32_t slab, uint32_t* slist, uint32_t m, uint32_t nwarps,
                                            int* cont_room) {
    StepCtx C;
    C.s = L.sweep0 + s;
    C.bump = L.bump;
    C.claim_ctr = claim_ctr;
    C.out = out;
    C.push_ctr = push_ctr;
    C.flags = flags;
    C.cap = cap;
    C.slab = slab;
    C.bind = bind_base(P, slist);
    C.t0 = L.sweep0 + 1;
    C.hist = P.hist;
    C.hist_cap = P.hist_cap;
    C.hwin = nullptr;
    C.hbase = C.s;
    C.stamp = s & kStampMask;
    C.ra = L.ra_used;
    // run-ahead pays in narrow sweeps of latency-bound phases (a lane's chain
    // of dependent steps without a barrier between them); in a wide sweep the
    // lanes of a warp stay on one rule path each only if they stay in step
    C.cont_room = (L.ra_on && m <= P.ra_max) ? cont_room : nullptr;
    C.cont_cost = P.max_new + 1;
    C.lone = nwarps <= kWarps ? 1u : 0u;
    const uint64_t worst = (uint64_t)m * P.max_new + 2ull * nwarps * max(slab, 32u * P.max_new) + 1;
    const uint64_t room = cap > (uint64_t)L.bump + worst ? cap - L.bump - worst : 0ull;
    C.claim_soft = room > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)room;
    return C;
}

// Copy records [0, n) between arenas (global <-> shared memory), CTA-wide.
template <int W>
__device__ __forceinline__ void copy_records(uint32_t* dst, const uint32_t* src, uint32_t n) {
    const uint32_t q = n * (W / 4);
    for (uint32_t k = threadIdx.x; k < q; k += kBlock)
        reinterpret_cast<uint4*>(dst)[k] = reinterpret_cast<const uint4*>(src)[k];  // generic: either side may be shared
}

// Collection of a shared-memory resident arena by CTA 0 (the grid-wide
// gc_compact restated for one CTA): recount references (unless the run keeps
// them), claim refcount-zero slots and follow
// their cascades to the end, renumber live slots in order (map in the idle
// frontier list `map`, so the resident arena holds at most kSmallCap
// slots), move records down chunk by chunk, and remap arguments, waiter
// words, the frontier `list` and the roots.  Returns the new bump pointer.
template <int W>
__device__ uint32_t local_gc(const Params& P, const Prog& G, Smem& sm, uint32_t* A, uint32_t bump, uint32_t* list,
                             uint32_t m, uint32_t* map) {
    if (!P.track_rc) recount_refs<W>(P, G, A, bump, threadIdx.x, kBlock, []() { __syncthreads(); });
    for (uint32_t x = 1 + threadIdx.x; x < bump; x += kBlock) {
        uint32_t* R = rec<W>(A, x);
        const uint32_t head = R[kWHead];
        if (head == kDeadHead || R[kWRc] != 0) continue;
        if (atomicCAS(R + kWHead, head, kDeadHead) != head) continue;
        uint32_t cur_slot = x, chead = head;
        for (;;) {
            const uint32_t* C = rec<W>(A, cur_slot);
            const uint32_t car = G.arity[chead & kSymMask];
            uint32_t next = 0, nhead = 0;
            for (uint32_t j = 0; j < car; ++j) {
                const uint32_t c = C[kWArgs + j];
                if (atomicSub(rec<W>(A, c) + kWRc, 1u) == 1u && next == 0) {
                    const uint32_t h = rec<W>(A, c)[kWHead];
                    if (h != kDeadHead && atomicCAS(rec<W>(A, c) + kWHead, h, kDeadHead) == h) {
                        next = c;
                        nhead = h;
                    }
                }
            }
            if (!next) break;
            cur_slot = next;
            chead = nhead;
        }
    }
    __syncthreads();
    uint32_t running = 1;
    for (uint32_t x0 = 0; x0 < bump; x0 += kBlock) {
        const uint32_t x = x0 + threadIdx.x;
        const bool live = x > 0 && x < bump && rec<W>(A, x)[kWHead] != kDeadHead;
        uint32_t t;
        const uint32_t e = block_scan(live ? 1u : 0u, &t, sm);
        if (x < bump) map[x] = live ? running + e : 0u;
        running += t;
    }
    __syncthreads();
    // order-preserving move: targets never exceed sources, and every earlier
    // chunk has landed before this chunk's records are read
    for (uint32_t x0 = 0; x0 < bump; x0 += kBlock) {
        const uint32_t x = x0 + threadIdx.x;
        const uint32_t to = x < bump ? map[x] : 0u;
        uint4 v[W / 4];
        if (to) {
#pragma unroll
            for (int q = 0; q < W / 4; ++q) v[q] = reinterpret_cast<const uint4*>(rec<W>(A, x))[q];
        }
        __syncthreads();
        if (to) {
#pragma unroll
            for (int q = 0; q < W / 4; ++q) reinterpret_cast<uint4*>(rec<W>(A, to))[q] = v[q];
        }
        __syncthreads();
    }
    for (uint32_t y = 1 + threadIdx.x; y < running; y += kBlock) {
        uint32_t* R = rec<W>(A, y);
        const uint32_t car = G.arity[R[kWHead] & kSymMask];
        for (uint32_t j = 0; j < car; ++j) R[kWArgs + j] = map[R[kWArgs + j]];
        const uint32_t w = R[kWWaiter];
        if (w != 0 && w != kWoken) R[kWWaiter] = map[w];
    }
    for (uint32_t v = threadIdx.x; v < m; v += kBlock) list[v] = map[list[v]];
    for (uint32_t r = threadIdx.x; r < P.num_roots; r += kBlock) P.roots[r] = map[__ldcg(P.roots + r)];
    __syncthreads();
    return running;
}

// Warp 0 of CTA 0 runs sweeps alone while the frontier fits one warp.
template <int W, bool kRA>
__device__ void warp_sweeps(const Params& P, const Prog& G, uint32_t* slist, SmallState& ss, Local& L,
                            bool& just_collected, Slab& slab, uint32_t* arena, uint64_t cap, uint32_t slab_size,
                            uint32_t& tmax) {
    const uint32_t lane = threadIdx.x & 31;
    PhaseClock pc;
    const bool prof = kProfBuild && P.profile == 1 && lane == 0;
    uint64_t t_prev = global_ns();  // one timer read per sweep: each sweep's ns runs from the previous one's end
    for (;;) {
        const uint32_t sc = ss.sc;
        const uint32_t m = ss.count[sc];
        if (m == 0 || m > (kRA ? P.warp_max_ra : P.warp_max)) break;
        if (W == 8 && m == 1) {
            // Solo sweeps: while the frontier is a single slot, lane 0 runs
            // sweep after sweep alone -- the warp step without collectives and
            // the loop's bookkeeping without warp synchronisation -- and hands
            // its state to the warp when the frontier widens or the run stops.
            // (Wide-record kernels take the one-sweep solo step below instead:
            // this loop's extra state costs them spills.)
            if (lane == 0) {
                for (;;) {
                    const uint32_t sc1 = ss.sc;
                    if (ss.count[sc1] != 1) break;
                    if (slab_size == 0 && (uint64_t)L.bump + P.max_new + 1 > cap) break;
                    if (plan(P, L, 1, just_collected, 1) != kPlanSweep) break;
                    just_collected = false;
                    if (ra_track<kRA>(P, L, 1)) break;  // hand over to the run-ahead build
                    const uint32_t s = L.sweep + 1;
                    const long long cs = prof ? clock64() : 0;
                    ss.count[sc1 ^ 1] = 0;
                    ss.claim = 0;
                    ss.cont_room = (int)(kSmallCap - (P.max_new + 1));
                    const StepCtx C = make_ctx(P, L, s, &ss.claim, slist + (sc1 ^ 1) * kSmallCap, &ss.count[sc1 ^ 1],
                                               &ss.flags, cap, slab_size, slist, 1, 1, &ss.cont_room);
                    uint32_t width = 0, cont = 0, steps = 0, pushes = 0;
                    NfCarry just_nf{};
                    uint32_t slot = slist[sc1 * kSmallCap];
                    for (;;) {
                        width += warp_step<W, false, kRA, 1>(P, G, arena, C, slab, true, &slot, prof, pc,
                                                           ra_more(P, C, steps), cont, tmax, just_nf, pushes);
                        if (!cont) break;
                        slot = cont;
                        ++steps;
                    }
                    L.bump = (uint32_t)min((uint64_t)L.bump + ss.claim, cap);
                    L.peak_bump = max(L.peak_bump, L.bump);
                    L.total += width;
                    L.maxw = width > L.maxw ? width : L.maxw;
                    if (!kRA && width) atomicAdd(P.hist + (s - 1), (unsigned long long)width);
                    L.sweep = s;
                    L.small_sweeps++;
                    ss.sc = sc1 ^ 1;
                    const uint64_t now = global_ns();
                    record(P, s, width, L, 1, 2, now - t_prev);
                    t_prev = now;
                    if (prof) {
                        for (int k = 0; k < 4; ++k) P.ctl->prof[k] += pc.t[k];
                        P.ctl->prof[4] += clock64() - cs;
                        P.ctl->prof[5] += 1;
                        P.ctl->prof[6] += pc.steps;
                        pc = PhaseClock{};
                    }
                    if (L.total > P.step_budget || ss.flags) break;
                }
                ss.L = L;
            }
            __syncwarp();
            L = ss.L;
            just_collected = false;
            t_prev = __shfl_sync(0xffffffffu, t_prev, 0);
            slab.cur = __shfl_sync(0xffffffffu, slab.cur, 0);
            slab.end = __shfl_sync(0xffffffffu, slab.end, 0);
            slab.room = __shfl_sync(0xffffffffu, slab.room, 0);
            __syncwarp();
            if (L.total > P.step_budget || ss.flags) break;
            if (ss.count[ss.sc] == 1) break;  // stopped by plan or headroom: the caller decides
            continue;
        }
        // a resident arena must hold the worst case of this sweep
        if (slab_size == 0 && (uint64_t)L.bump + (uint64_t)m * P.max_new + 1 > cap) break;
        if (plan(P, L, m, just_collected, 1) != kPlanSweep) break;
        just_collected = false;
        if (ra_track<kRA>(P, L, m)) break;
        const uint32_t s = L.sweep + 1;
        const long long cs = prof ? clock64() : 0;
        if (lane == 0) {
            ss.count[sc ^ 1] = 0;
            ss.claim = 0;
            ss.cont_room = (int)(kSmallCap - (P.max_new + 1) * m);
        }
        __syncwarp();
        const StepCtx C = make_ctx(P, L, s, &ss.claim, slist + (sc ^ 1) * kSmallCap, &ss.count[sc ^ 1], &ss.flags,
                                   cap, slab_size, slist, m, 1, &ss.cont_room);
        uint32_t width = 0;
        if (TRS_GEN && W != 8 && m == 1) {
            // one entry, specialised wide-record kernel: lane 0 alone for this sweep
            uint32_t w1 = 0;
            if (lane == 0) {
                uint32_t cont = 0, steps = 0, pushes = 0;
                NfCarry just_nf{};
                uint32_t slot = slist[sc * kSmallCap];
                for (;;) {
                    w1 += warp_step<W, false, kRA, 1>(P, G, arena, C, slab, true, &slot, prof, pc,
                                                    ra_more(P, C, steps), cont, tmax, just_nf, pushes);
                    if (!cont) break;
                    slot = cont;
                    ++steps;
                }
            }
            width = __shfl_sync(0xffffffffu, w1, 0);
            slab.cur = __shfl_sync(0xffffffffu, slab.cur, 0);  // the slab is warp-uniform state
            slab.end = __shfl_sync(0xffffffffu, slab.end, 0);
            slab.room = __shfl_sync(0xffffffffu, slab.room, 0);
        } else {
            uint32_t cont = 0, steps = 0, pushes = 0;
            NfCarry just_nf{};
            uint32_t slot = lane < m ? slist[sc * kSmallCap + lane] : 0u;
            for (;;) {
                width += warp_step<W, false, kRA>(P, G, arena, C, slab, slot != 0u, &slot, prof, pc,
                                             ra_more(P, C, steps), cont, tmax, just_nf, pushes);
                const uint32_t cm = __ballot_sync(0xffffffffu, cont != 0u);
                if (!cm) break;
#if TRS_B200_LONE
                if (W == 8 && kRA && __popc(cm) == 1) {
                    // one chain left: its lane runs it alone (the rest of
                    // the device is idle in warp mode: plain counters)
                    uint32_t lw = 0;
                    if (cont) {
                        do {
                            ++steps;
                            uint32_t sl = cont;
                            lw += warp_step<W, false, kRA, 1>(P, G, arena, C, slab, true, &sl, prof, pc,
                                                              ra_more(P, C, steps), cont, tmax, just_nf, pushes);
                        } while (cont);
                    }
                    const int src = __ffs(cm) - 1;
                    width += __shfl_sync(0xffffffffu, lw, src);
                    slab.cur = __shfl_sync(0xffffffffu, slab.cur, src);
                    slab.end = __shfl_sync(0xffffffffu, slab.end, src);
                    slab.room = __shfl_sync(0xffffffffu, slab.room, src);
                    break;
                }
#endif
                slot = cont;
                ++steps;
            }
        }
        __syncwarp();
        L.bump = (uint32_t)min((uint64_t)L.bump + ss.claim, cap);
        L.peak_bump = max(L.peak_bump, L.bump);
        L.total += width;
        L.maxw = width > L.maxw ? width : L.maxw;
        L.sweep = s;
        L.small_sweeps++;
        const uint64_t now = global_ns();
        if (lane == 0) {
            ss.sc = sc ^ 1;
            if (!kRA && width) atomicAdd(P.hist + (s - 1), (unsigned long long)width);
            record(P, s, width, L, m, 2, now - t_prev);
            if (prof) {
                for (int k = 0; k < 4; ++k) P.ctl->prof[k] += pc.t[k];
                P.ctl->prof[4] += clock64() - cs;
                P.ctl->prof[5] += 1;
                P.ctl->prof[6] += pc.steps;
                pc = PhaseClock{};
            }
        }
        t_prev = now;
        __syncwarp();
        if (L.total > P.step_budget || ss.flags) break;
    }
}

// Grid sweep s claims through counter s & 3, which grid sweep s - 2 zeroes
// (every CTA has read it by then).  Single-CTA sweeps skip that ring, so on
// hand-back CTA 0 zeroes the counters of the next two sweeps itself (before
// the grid barrier that releases them); a stale count would move the bump
// over slots nobody writes, and the collector would keep their old records.
__device__ __forceinline__ void zero_next_claims(const Params& P, uint32_t sweep) {
    P.blocksum[kMaxGrid + ((sweep + 1) & 3)] = 0;
    P.blocksum[kMaxGrid + ((sweep + 2) & 3)] = 0;
}

// CTA 0 runs sweeps out of shared memory while the frontier is small.
template <int W, bool kRA>
__device__ void run_small(const Params& P, const Prog& G, Smem& sm, Local& L, bool& just_collected,
                          uint32_t* slist, SmallState& ss, const Frontier& F, Slab& slab, uint32_t& tmax) {
    Ctl* ctl = P.ctl;
    const uint32_t cap_m = kSmallCap / (P.max_new + 1);
    const uint32_t exit_m = min(P.small_exit, cap_m);
    if (F.M > exit_m) {
        // too wide for the shared-memory lists; nothing touched
        if (threadIdx.x == 0) {
            zero_next_claims(P, L.sweep);
            store_local(L, ctl);
        }
        return;
    }
    const uint32_t* gin = P.list[L.cur];
    const uint32_t stride = P.rich ? W : 1;
    for (uint32_t v = threadIdx.x; v < F.M; v += kBlock) slist[v] = gin[(size_t)frontier_phys(F, v) * stride];
    if (threadIdx.x == 0) {
        ss.count[0] = F.M;
        ss.sc = 0;
        ss.flags = 0;
    }
    __syncthreads();
    uint32_t* arena = P.arena[L.arena];
    uint64_t cap = P.capacity;
    uint32_t slab_size = P.slab;
    // Resident mode: the whole allocated store fits the CTA's shared memory,
    // so it moves there (same slot ids) and every gather, claim and atomic of
    // these sweeps is a shared-memory access; claims are exact (no slabs),
    // a full resident arena is compacted in place (local_gc), and the store
    // moves back when the frontier outgrows this mode or stops fitting.
    uint32_t* const resident_arena = slist + 2 * kSmallCap + P.max_vars * kBlock;
    bool resident = P.local_cap != 0 && L.bump <= P.local_enter;
    if (resident) {
        abandon_slab<W>(arena, slab);
        __syncthreads();
        copy_records<W>(resident_arena, arena, L.bump);
        __syncthreads();
        arena = resident_arena;
        cap = min((uint64_t)P.local_cap, P.capacity);  // a fixed capacity binds here too
        slab_size = 0;
    }
    auto leave_resident = [&]() {
        copy_records<W>(P.arena[L.arena], resident_arena, L.bump);
        __syncthreads();
        arena = P.arena[L.arena];
        cap = P.capacity;
        slab_size = P.slab;
        resident = false;
    };
    const uint32_t warp = threadIdx.x >> 5;
    for (;;) {
        const uint32_t sc = ss.sc;
        const uint32_t m = ss.count[sc];
        if (m > exit_m) break;
        if (resident && (uint64_t)L.bump + (uint64_t)m * P.max_new + 1 > cap) {
            if (P.allow_gc) {
                const uint64_t t0 = global_ns();
                L.bump = local_gc<W>(P, G, sm, arena, L.bump, slist + sc * kSmallCap, m, slist + (sc ^ 1) * kSmallCap);
                L.gc_runs++;
                L.gc_ns += global_ns() - t0;
                L.last_gc = L.sweep + 1;
            }
            // keep half the resident arena free, else hand back to HBM (where
            // growth, collection or the fixed-capacity fault take over)
            if ((uint64_t)L.bump + (uint64_t)m * P.max_new + 1 > cap / 2) leave_resident();
        }
        if (plan(P, L, m, just_collected, kWarps) != kPlanSweep) break;
        if (P.warp_mode && m <= (kRA ? P.warp_max_ra : P.warp_max)) {
            if (warp == 0) {
                warp_sweeps<W, kRA>(P, G, slist, ss, L, just_collected, slab, arena, cap, slab_size, tmax);
                if ((threadIdx.x & 31) == 0) ss.L = L;
            }
            __syncthreads();
            L = ss.L;
            just_collected = false;
            if (L.total > P.step_budget || ss.flags) break;
            const uint32_t m2 = ss.count[ss.sc];
            if (m2 <= (kRA ? P.warp_max_ra : P.warp_max) && !(resident && m2 && (uint64_t)L.bump + (uint64_t)m2 * P.max_new + 1 > cap))
                break;  // warp mode stopped for another reason (plan / empty)
            continue;
        }
        just_collected = false;
        if (ra_track<kRA>(P, L, m)) break;
        const uint32_t s = L.sweep + 1;
        const uint64_t t0 = threadIdx.x == 0 ? global_ns() : 0;
        const bool profc = kProfBuild && P.profile == 1 && threadIdx.x == 0;
        const long long cs = profc ? clock64() : 0;
        __syncthreads();  // everyone has read ss.count[sc]
        if (threadIdx.x == 0) {
            ss.count[sc ^ 1] = 0;
            ss.claim = 0;
            ss.cont_room = (int)(kSmallCap - (P.max_new + 1) * m);
        }
        __syncthreads();
        Frontier Fs{1, m, 0u, nullptr, nullptr};
        uint32_t zero_off = 0;
        Fs.off = &zero_off;
        const StepCtx C = make_ctx(P, L, s, &ss.claim, slist + (sc ^ 1) * kSmallCap, &ss.count[sc ^ 1], &ss.flags, cap,
                                   slab_size, slist, m, kWarps, &ss.cont_room);
        PhaseClock pc;
        unsigned long long rw = cta_entries<W, false, kRA>(P, G, arena, C, Fs, slist + sc * kSmallCap, 0, 1, slab,
                                                      profc, pc, tmax);
        const unsigned long long width = block_sum64(rw, sm);
        L.bump = (uint32_t)min((uint64_t)L.bump + ss.claim, cap);
        L.peak_bump = max(L.peak_bump, L.bump);
        L.total += width;
        L.maxw = width > L.maxw ? width : L.maxw;
        L.sweep = s;
        L.small_sweeps++;
        if (threadIdx.x == 0) {
            ss.sc = sc ^ 1;
            if (!kRA && width) atomicAdd(P.hist + (s - 1), width);
            record(P, s, width, L, m, resident ? 3 : 1, global_ns() - t0);
            if (profc) {
                for (int k = 0; k < 4; ++k) ctl->prof[k] += pc.t[k];
                ctl->prof[4] += clock64() - cs;
                ctl->prof[5] += 1;
                ctl->prof[6] += pc.steps;
                for (int k = 0; k < 4; ++k) ctl->prof[8 + k] += pc.sub[k];
            }
        }
        __syncthreads();
        if (L.total > P.step_budget || ss.flags) break;
    }
    if (resident) leave_resident();
    // hand the frontier back to the grid as one region of the global list
    const uint32_t m = ss.count[ss.sc];
    uint32_t* gout = P.list[L.cur];
    for (uint32_t v = threadIdx.x; v < m; v += kBlock) {
        if (P.rich)
            *reinterpret_cast<uint4*>(gout + (size_t)v * W) = make_uint4(slist[ss.sc * kSmallCap + v], 0u, 0u, 0u);
        else
            gout[v] = slist[ss.sc * kSmallCap + v];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        region_off(P, L.cur)[0] = 0;
        region_cnt(P, L.cur)[0] = m;
        P.region_flags[L.cur * kMaxGrid] = ss.flags;
        ctl->nregions[L.cur] = 1;
        zero_next_claims(P, L.sweep);
        store_local(L, ctl);
    }
}

template <int W, int MINB, bool kRA>
__global__ void __launch_bounds__(kBlock, MINB) step_loop(Params P) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ Smem sm;
    __shared__ SmallState ss;
    __shared__ uint32_t f_pref[kMaxGrid + 1];
    __shared__ uint32_t f_off[kMaxGrid];
    __shared__ uint32_t s_push;
    __shared__ uint32_t s_flags;
    __shared__ int s_cont;
    __shared__ uint32_t s_hwin[kHistWin];
    // stage the program tables; the single-CTA frontier lists follow them
    for (uint32_t o = threadIdx.x * 16; o < P.prog_bytes; o += kBlock * 16)
        *reinterpret_cast<uint4*>(smem_raw + o) = *reinterpret_cast<const uint4*>(P.prog + o);
    __syncthreads();
    const Prog G = view_prog(smem_raw);
    uint32_t* slist = reinterpret_cast<uint32_t*>(smem_raw + P.prog_bytes);
    const uint32_t nblocks = gridDim.x;
    const uint32_t nwarps = nblocks * kWarps;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    Ctl* ctl = P.ctl;

    Local L;
    load_local(L, ctl);
    bool just_collected = false;
    uint32_t exit_status = kRunning;
    uint32_t epoch = 0;  // barriers passed in this launch (the host zeroes bar_arrive)
    Slab slab{0, 0, 1u};
    uint32_t tmax = 0;  // latest nf epoch this thread published (the run's logical sweep count)
    Frontier F = stage_frontier(P, L.cur, nblocks, f_pref, f_off, sm, nullptr);

    bool gc_truncated = false;
    auto collect = [&]() {
        abandon_slab<W>(P.arena[L.arena], slab);
        if (leader) ctl->gc_truncated = 0u;
        grid_sync(ctl, nblocks, epoch);  // every slab is marked before the collector scans
        const uint64_t t0 = global_ns();
        L.bump = gc_compact<W>(P, sm, G, L.arena, L.bump, F, L.cur, blockIdx.x, nblocks, epoch, gc_truncated,
                               P.compact_only ? 0xFFFFFFFFu : 64u);
        L.cur ^= 1;
        L.gc_runs++;
        L.gc_ns += global_ns() - t0;
        F = stage_frontier(P, L.cur, nblocks, f_pref, f_off, sm, nullptr);
    };

    if (P.probe_iters) {
        // overhead probe: grid barriers alone (mode 0) or a barrier plus the
        // frontier staging every grid sweep does (mode 1)
        const uint64_t t0 = global_ns();
        for (uint32_t it = 0; it < P.probe_iters; ++it) {
            grid_sync(ctl, nblocks, epoch);
            if (P.probe_mode == 1) {
                unsigned long long w;
                F = stage_frontier(P, L.cur, nblocks, f_pref, f_off, sm, &w);
            }
        }
        if (leader) ctl->gc_ns = global_ns() - t0;
        return;
    }

    if (P.compact_only) {
        // final compaction: collect until a pass reclaims nothing
        for (uint32_t round = 0; round < P.compact_only; ++round) {
            const uint32_t before = L.bump;
            collect();
            // done when every cascade ran to its end (no garbage left) or
            // a pass reclaimed nothing
            if (L.bump == before || !gc_truncated) break;
        }
        if (leader) {
            store_local(L, ctl);
            ctl->status = kDone;
        }
        return;
    }

    bool val_monotone = false;  // the first scan of a launch (or after a collection) has no previous epochs
    auto validate_now = [&]() -> bool {
        // every slab's unused slots are marked collected before the scan
        abandon_slab<W>(P.arena[L.arena], slab);
        grid_sync(ctl, nblocks, epoch);
        validate_store_device<W>(P, G, L.arena, L.bump, F, L.cur, blockIdx.x, nblocks, epoch, val_monotone);
        val_monotone = true;
        return __ldcg(&ctl->val_kind) == 0u;
    };
    for (;;) {
        const uint32_t s = L.sweep + 1;
        const uint32_t m = F.M;
        if (P.validate >= 2 && !validate_now()) {
            exit_status = kValidate;
            break;
        }
        const uint32_t pl = plan(P, L, m, just_collected, nwarps);
        if (pl == kPlanFinish) {
            // the first sweep whose frontier is empty (sweep_engine.cpp:147)
            if (leader) record(P, s, 0, L, 0, 0, 0);
            L.sweep = s;
            exit_status = kDone;
            break;
        }
        if (pl == kPlanTrace) {
            if (leader && s > P.hist_cap) atomicMax(&ctl->hist_need, s + 1);
            exit_status = kNeedTrace;
            break;
        }
        if (pl == kPlanGrow) {
            exit_status = kNeedGrow;
            break;
        }
        if (pl == kPlanGc) {
            collect();
            L.last_gc = L.sweep + 1;
            just_collected = true;
            val_monotone = false;  // slots were renumbered
            continue;
        }

        if (m <= P.small_enter) {
            // ---- single-CTA mode: CTA 0 runs sweeps out of shared memory,
            // the rest of the grid parks in the barrier
            const uint32_t before = L.sweep;
            if (blockIdx.x == 0) run_small<W, kRA>(P, G, sm, L, just_collected, slist, ss, F, slab, tmax);
            grid_sync(ctl, nblocks, epoch, /*park=*/blockIdx.x != 0);
            load_local(L, ctl);
            F = stage_frontier(P, L.cur, nblocks, f_pref, f_off, sm, nullptr);
            if (L.sweep != before) just_collected = false;  // keep every CTA's plan identical
            if (!kRA && P.runahead && L.ra_go) {
                exit_status = kNeedRA;
                break;
            }
            if (F.flags & kFlagCapacity) {
                exit_status = kCapacity;
                break;
            }
            if (F.flags & kFlagHist) {
                exit_status = kNeedTrace;
                break;
            }
            if (L.total > P.step_budget) {
                exit_status = kStepBudget;
                break;
            }
            if (L.sweep != before) continue;
            // no progress in single-CTA mode (frontier too wide for its
            // lists): fall through to one grid-wide sweep
        }
        just_collected = false;

        // ---- grid-wide sweep
        const uint64_t t0 = leader ? global_ns() : 0;
        const bool profsw = kProfBuild && P.profile && (P.profile == 1 || m <= P.profile);
        const long long cs = (profsw && leader) ? clock64() : 0;
        // output regions: CTA b's own entries need (max_new + 1) * count, and
        // every CTA gets the same slack of the list buffer for run-ahead steps
        const uint64_t base_ext = (uint64_t)(P.max_new + 1) * m;
        const uint32_t slack = (P.runahead && !P.rich && P.list_cap > base_ext)
                                   ? (uint32_t)min((P.list_cap - base_ext) / nblocks, (uint64_t)kMaxSlack)
                                   : 0u;
        if (ra_track<kRA>(P, L, m)) {  // every CTA sees the same m
            exit_status = kNeedRA;
            break;
        }
        if (threadIdx.x == 0) {
            s_push = 0;
            s_flags = 0;
            s_cont = (int)slack;
        }
        if (threadIdx.x < kHistWin) s_hwin[threadIdx.x] = 0u;
        __syncthreads();
        const uint32_t out_off =
            (P.max_new + 1) * cta_prefix(m, blockIdx.x, nblocks, chunk_lanes(m, nblocks)) + blockIdx.x * slack;
        uint32_t* claim_ctr = &P.blocksum[kMaxGrid + (s & 3)];
        if (leader) P.blocksum[kMaxGrid + ((s + 2) & 3)] = 0;
        StepCtx C = make_ctx(P, L, s, claim_ctr, P.list[L.cur ^ 1] + (size_t)out_off * (P.rich ? W : 1), &s_push,
                             &s_flags, P.capacity, P.slab, slist, m, nwarps, &s_cont);
        C.hwin = s_hwin;
        PhaseClock pc;
#if TRS_B200_PROFILE
        // profiling build: the slowest warp's entry time of this sweep
        // (max over the grid, rotating slot) lands in the trace's free_len,
        // and per-phase maxima over warps in ctl->wmax
        if (leader) {
            ctl->gcprof[(s + 1) & 1] = 0;
            for (int k = 0; k < 8; ++k) ctl->wmax[(s + 1) & 1][k] = 0;
        }
        const long long wt0 = clock64();
        PhaseClock wpc;
        const bool wprof = profsw && (threadIdx.x & 31) == 0;
#else
        PhaseClock& wpc = pc;
        const bool wprof = profsw && leader;
#endif
        unsigned long long rw =
#if TRS_B200_RICH_ENTRIES
            P.rich ? cta_entries<W, true, kRA>(P, G, P.arena[L.arena], C, F, P.list[L.cur], blockIdx.x, nblocks, slab,
                                          wprof, wpc, tmax)
                   :
#endif
                     cta_entries<W, false, kRA>(P, G, P.arena[L.arena], C, F, P.list[L.cur], blockIdx.x, nblocks, slab,
                                           wprof, wpc, tmax);
#if TRS_B200_PROFILE
        if ((threadIdx.x & 31) == 0) atomicMax(&ctl->gcprof[s & 1], (unsigned long long)(clock64() - wt0));
        if (wprof) {
            for (int k = 0; k < 4; ++k) atomicMax(&ctl->wmax[s & 1][k], (unsigned long long)wpc.t[k]);
            for (int k = 0; k < 4; ++k) atomicMax(&ctl->wmax[s & 1][4 + k], (unsigned long long)wpc.sub[k]);
        }
        if (leader) pc = wpc;
#endif
        rw = block_sum64(rw, sm);  // ends synchronised: the width window is complete
        if (kRA && threadIdx.x < kHistWin && s_hwin[threadIdx.x])
            atomicAdd(P.hist + (C.hbase - C.t0 + threadIdx.x), (unsigned long long)s_hwin[threadIdx.x]);
        if (threadIdx.x == 0) {
            region_off(P, L.cur ^ 1)[blockIdx.x] = out_off;
            region_cnt(P, L.cur ^ 1)[blockIdx.x] = s_push;
            P.region_rew[(L.cur ^ 1) * kMaxGrid + blockIdx.x] = rw;
            P.region_flags[(L.cur ^ 1) * kMaxGrid + blockIdx.x] = s_flags;
        }
        if (leader) ctl->nregions[L.cur ^ 1] = nblocks;
        grid_sync(ctl, nblocks, epoch);
        L.cur ^= 1;
        unsigned long long width = 0;
        F = stage_frontier(P, L.cur, nblocks, f_pref, f_off, sm, &width);
        const uint32_t allocd = __ldcg(claim_ctr);
        L.bump = (uint32_t)min((uint64_t)L.bump + allocd, P.capacity);  // n = min(n + next_fresh, capacity), sweep_engine.cpp:94-98
        L.peak_bump = max(L.peak_bump, L.bump);
        L.total += width;
        L.maxw = width > L.maxw ? width : L.maxw;
        L.sweep = s;
        if (leader) {
            if (!kRA && width) atomicAdd(P.hist + (s - 1), width);
            record(P, s, width, L, m, 0, global_ns() - t0);
#if TRS_B200_PROFILE
            if (s <= P.trace_cap) P.trace[s - 1].free_len = (uint32_t)__ldcg(&ctl->gcprof[s & 1]);
            if (profsw)
                for (int k = 0; k < 8; ++k) ctl->wmax_sum[k] += __ldcg(&ctl->wmax[s & 1][k]);
#endif
            if (profsw) {
                for (int k = 0; k < 4; ++k) ctl->prof[k] += pc.t[k];
                ctl->prof[4] += clock64() - cs;
                ctl->prof[5] += 1;
                ctl->prof[6] += pc.steps;
                for (int k = 0; k < 4; ++k) ctl->prof[8 + k] += pc.sub[k];
            }
        }
        if (F.flags & kFlagCapacity) {
            exit_status = kCapacity;
            break;
        }
        if (F.flags & kFlagHist) {
            exit_status = kNeedTrace;
            break;
        }
        if (L.total > P.step_budget) {
            exit_status = kStepBudget;
            break;
        }
    }
    // leave no half-used slab behind: the host may copy or the next launch
    // may collect [0, bump)
    abandon_slab<W>(P.arena[L.arena], slab);
    // the latest nf epoch of this launch; finish_run turns it into the
    // logical sweep count
    const uint32_t wt = __reduce_max_sync(0xffffffffu, tmax);
    if ((threadIdx.x & 31) == 0 && wt) atomicMax(&ctl->tmax, wt);
    if (leader) {
        store_local(L, ctl);
        ctl->status = exit_status;
    }
}

}  // namespace trs_b200

// Compacting garbage collector (grid-wide, inside the persistent step loop).
//
// Counterpart of the reference's collect_free_indices (term_store.cpp:140-157)
// plus its free ring, re-designed for bump allocation: refcount-zero slots
// are claimed (head := dead) and drop their argument references; then the
// live slots are stream-compacted, in order, into the twin arena with block
// scans and a grid-wide prefix over per-CTA counts, and an old -> new index
// map is applied to every argument, waiter word, frontier entry and root.
#pragma once

#include "device_common.cuh"

namespace trs_b200 {

// Frontier list of one sweep: R regions of a list buffer, with their
// exclusive prefix over counts staged in shared memory.
struct Frontier {
    uint32_t R;
    uint32_t M;
    uint32_t flags;        // OR of the regions' kFlag* (the sweep that wrote them)
    const uint32_t* pref;  // [R + 1], pref[R] = M
    const uint32_t* off;   // [R]
};

__device__ __forceinline__ uint32_t frontier_phys(const Frontier& f, uint32_t v) {
    if (f.R == 1) return f.off[0] + v;
    uint32_t lo = 0, hi = f.R - 1;  // largest r with pref[r] <= v
    while (lo < hi) {
        uint32_t mid = (lo + hi + 1) >> 1;
        if (f.pref[mid] <= v)
            lo = mid;
        else
            hi = mid - 1;
    }
    return f.off[lo] + (v - f.pref[lo]);
}

// Refcounts recounted from the store: rc(y) = references from uncollected
// slots + root pins, the reference's ghost invariant (sweep_engine.cpp:335-359)
// and so exactly what maintaining them rewrite by rewrite would leave.  The
// step loop keeps no refcounts unless Params::track_rc (validate modes): no
// derive reads them (garbage is always nf, so the frontier
// needs no liveness test), and the argument updates were a fifth of the
// batched configs' step-loop time (tools/rc_ab.py).  The collectors recount
// first.  Threads [tid, nthreads) of the caller's group; `sync` is its barrier.
template <int W, typename Sync>
__device__ __forceinline__ void recount_refs(const Params& P, const Prog& G, uint32_t* A, uint32_t bump, uint32_t tid,
                                             uint32_t nthreads, Sync sync) {
    for (uint32_t x = 1 + tid; x < bump; x += nthreads) rec<W>(A, x)[kWRc] = 0u;
    sync();
    for (uint32_t x = 1 + tid; x < bump; x += nthreads) {
        const uint32_t* R = rec<W>(A, x);
        const uint32_t head = R[kWHead];
        if (head == kDeadHead) continue;
        const uint32_t ar = G.arity[head & kSymMask];
        for (uint32_t j = 0; j < ar; ++j) atomicAdd(rec<W>(A, R[kWArgs + j]) + kWRc, 1u);
    }
    for (uint32_t r = tid; r < P.num_roots; r += nthreads) atomicAdd(rec<W>(A, __ldcg(P.roots + r)) + kWRc, 1u);
    sync();
}

// Returns the new bump pointer.  The caller has staged `in` (regions of
// list buffer `cur`) and abandoned every warp's slab; on return the
// frontier is one dense region of buffer cur ^ 1 and arena_idx is flipped.
template <int W>
__device__ uint32_t gc_compact(const Params& P, Smem& sm, const Prog& G, uint32_t& arena_idx, uint32_t bump,
                               const Frontier& in, uint32_t cur, uint32_t block_rank, uint32_t nblocks,
                               uint32_t& epoch, bool& truncated, uint32_t max_hops) {
    uint32_t* A = P.arena[arena_idx];
    uint32_t* B = P.arena[arena_idx ^ 1];
    const uint32_t tid = block_rank * kBlock + threadIdx.x;
    const uint32_t nthreads = nblocks * kBlock;
#if TRS_B200_PROFILE
    const bool gl = block_rank == 0 && threadIdx.x == 0;
    uint64_t gt = gl ? global_ns() : 0;
    unsigned long long hops_total = 0;
    uint32_t hops_max = 0;
#define TRS_GC_MARK(k)                                      \
    if (gl) {                                               \
        const uint64_t now = global_ns();                   \
        atomicAdd(&P.ctl->gcprof[k], (unsigned long long)(now - gt)); \
        gt = now;                                           \
    }
#else
#define TRS_GC_MARK(k)
#endif
    if (!P.track_rc) recount_refs<W>(P, G, A, bump, tid, nthreads, [&]() { grid_sync(P.ctl, nblocks, epoch); });
    // phase 1: claim refcount-zero slots and drop their argument references.
    // A thread follows the cascade it triggers for at most max_hops claimed
    // slots (64 inside the step loop, bounding the pause; unbounded for the
    // final compaction); the rest waits for a later collection, as the
    // reference defers it.
    for (uint32_t x = 1 + tid; x < bump; x += nthreads) {
        uint32_t* R = rec<W>(A, x);
        const uint4 hq = __ldcg(reinterpret_cast<const uint4*>(R));  // head, epoch, rc, waiter
        const uint32_t head = hq.x;
        if (head == kDeadHead || hq.z != 0) continue;
        if (atomicCAS(R + kWHead, head, kDeadHead) != head) continue;
        uint32_t cur_slot = x, chead = head;
        for (uint32_t hop = 0;; ++hop) {
            // a claimed slot always drops its references; at the hop cap the
            // children it frees stay unclaimed with refcount zero (live to
            // the compaction), and the next collection's scan takes them
            const bool last = hop + 1 >= max_hops;
            uint32_t* C = rec<W>(A, cur_slot);
            uint32_t car = G.arity[chead & kSymMask];
            uint32_t next = 0, nhead = 0;
            for (uint32_t j = 0; j < car; ++j) {
                uint32_t c = __ldcg(C + kWArgs + j);
                const bool freed = atomicSub(rec<W>(A, c) + kWRc, 1u) == 1u;
                if (!freed) continue;
                if (last || next != 0) {
                    // not followed (hop cap, or a second freed child): it stays
                    // garbage unless this pass's scan reaches it later
                    P.ctl->gc_truncated = 1u;
                } else {
                    uint32_t h = __ldcg(rec<W>(A, c) + kWHead);
                    if (h != kDeadHead && atomicCAS(rec<W>(A, c) + kWHead, h, kDeadHead) == h) {
                        next = c;
                        nhead = h;
                    }
                }
            }
#if TRS_B200_PROFILE
            hops_total++;
            hops_max = max(hops_max, hop + 1);
#endif
            if (!next) break;
            cur_slot = next;
            chead = nhead;
        }
    }
#if TRS_B200_PROFILE
    atomicAdd(&P.ctl->gcprof[4], hops_total);
    atomicMax(&P.ctl->gcprof[5], (unsigned long long)hops_max);
#endif
    grid_sync(P.ctl, nblocks, epoch);
    TRS_GC_MARK(0)
    // phase 1 is the flag's only writer; every CTA reads it before the
    // barriers below, so the clear of the next collection cannot race it
    truncated = __ldcg(&P.ctl->gc_truncated) != 0;
    // phase 2: live count per CTA range
    const uint32_t span = bump - 1;
    const uint32_t chunk = (span + nblocks - 1) / nblocks;
    const uint32_t lo = 1 + block_rank * chunk;
    const uint32_t hi = min(bump, lo + chunk);
    uint32_t cnt = 0;
    for (uint32_t x = lo + threadIdx.x; x < hi; x += kBlock) cnt += __ldcg(rec<W>(A, x) + kWHead) != kDeadHead;
    uint32_t tot;
    block_scan(cnt, &tot, sm);
    if (threadIdx.x == 0) P.blocksum[block_rank] = tot;
    grid_sync(P.ctl, nblocks, epoch);
    TRS_GC_MARK(1)
    // phase 3: prefix over CTA sums, then order-preserving scatter into the
    // twin arena with the old -> new map
    uint32_t prefix = 0, all = 0;
    for (uint32_t b = threadIdx.x; b < nblocks; b += kBlock) {
        uint32_t v = __ldcg(P.blocksum + b);
        all += v;
        if (b < block_rank) prefix += v;
    }
    {
        uint32_t t1, t2;
        block_scan(prefix, &t1, sm);
        block_scan(all, &t2, sm);
        prefix = t1;
        all = t2;
    }
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
    grid_sync(P.ctl, nblocks, epoch);
    TRS_GC_MARK(2)
    // phase 4: remap args and waiters, and the frontier into one dense
    // region of the other list buffer, and the roots
    const uint32_t nbump = 1 + all;
    for (uint32_t y = 1 + tid; y < nbump; y += nthreads) {
        uint32_t* R = rec<W>(B, y);
        uint32_t car = G.arity[R[kWHead] & kSymMask];
        for (uint32_t j = 0; j < car; ++j) R[kWArgs + j] = __ldcg(P.gcmap + R[kWArgs + j]);
        uint32_t w = R[kWWaiter];
        if (w != 0 && w != kWoken) R[kWWaiter] = __ldcg(P.gcmap + w);
    }
    const uint32_t* Lin = P.list[cur];
    uint32_t* Lout = P.list[cur ^ 1];
    for (uint32_t v = tid; v < in.M && !P.rich; v += nthreads) Lout[v] = __ldcg(P.gcmap + Lin[frontier_phys(in, v)]);
    for (uint32_t v = tid; v < in.M && P.rich; v += nthreads) {
        // rich entries (sweep.cuh): remap the slot and, with a payload, its arguments
        const uint32_t* E = Lin + (size_t)frontier_phys(in, v) * W;
        uint32_t* D = Lout + (size_t)v * W;
        const uint4 q0 = __ldcg(reinterpret_cast<const uint4*>(E));
        *reinterpret_cast<uint4*>(D) = make_uint4(__ldcg(P.gcmap + q0.x), q0.y, q0.z, 0u);
        if (q0.z) {
            const uint32_t car = G.arity[q0.y & kSymMask];
            for (uint32_t j = 0; j < car; ++j) D[kWArgs + j] = __ldcg(P.gcmap + __ldcg(E + kWArgs + j));
        }
    }
    for (uint32_t e = tid; e < P.num_roots; e += nthreads) P.roots[e] = __ldcg(P.gcmap + P.roots[e]);
    if (block_rank == 0 && threadIdx.x == 0) {
        region_off(P, cur ^ 1)[0] = 0;
        region_cnt(P, cur ^ 1)[0] = in.M;
        P.region_flags[(cur ^ 1) * kMaxGrid] = 0u;
        P.ctl->nregions[cur ^ 1] = 1;
    }
    grid_sync(P.ctl, nblocks, epoch);
    TRS_GC_MARK(3)
    arena_idx ^= 1;
    return nbump;
}

}  // namespace trs_b200

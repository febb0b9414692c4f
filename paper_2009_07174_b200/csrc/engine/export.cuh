// Normal-form export: the live store written back in the reference
// TermStore layout (term_store.hpp:15-45) without collecting garbage.
//
// After a run the arena holds the live term graph plus every slot the run
// discarded; on the batched configs garbage outnumbers live slots ~8:1, and a
// refcount collection (gc.cuh) pays one random atomic per garbage edge.  The
// export instead marks what is reachable from the roots -- the live set by
// definition (extract, term_store.cpp:77-116, follows the same edges) -- and
// recounts references on the way: rc(y) = edges from live slots + root pins,
// the reference's refcount invariant over the exported store
// (sweep_engine.cpp:335-359).  Then live slots are renumbered 1..n-1 in arena
// order and packed column by column for one D2H each.
//
// Marking runs on one work queue: a thread walks a chain of first-time
// children itself (S^k numerals, list spines) and queues only the other
// children, and idle threads take queued items as soon as they appear, so
// the marking time is about the longest path, not depth x chain length.
//
// Scratch: newrc in P.gcmap; the queue and the old -> new map in the list
// buffer the frontier does NOT occupy; output columns in the twin arena.
// The arena and the frontier are untouched, so a run can resume afterwards.
#pragma once

#include "device_common.cuh"

namespace trs_b200 {

struct ExportArgs {
    uint32_t* queue[3];  // queue[0]: [bump] work items, zeroed by the host
    uint32_t* map;       // [bump]
    uint32_t* newrc;     // [bump]
    uint32_t* counters;  // [4] tail, head, pending, dangling (zeroed by the host)
    uint32_t* hss;       // output columns (staging)
    uint32_t* args;      // [ma * n]
    uint32_t* rcs;
    uint8_t* nf;
    uint32_t* roots_out;
    uint32_t ma;
};

template <int W>
__global__ void __launch_bounds__(kBlock, 1) export_store(Params P, ExportArgs X, uint32_t bump) {
    __shared__ Smem sm;
    const uint32_t* A = P.arena[__ldcg(&P.ctl->arena)];
    // symbol arities in shared memory when they fit (a chain walk reads one per hop)
    __shared__ uint8_t s_arity[4096];
    const ProgHeader* ph = reinterpret_cast<const ProgHeader*>(P.prog);
    const uint8_t* g_arity = P.prog + ph->off_arity;
    const bool arity_in_smem = ph->num_symbols <= 4096;
    if (arity_in_smem)
        for (uint32_t f = threadIdx.x; f < ph->num_symbols; f += kBlock) s_arity[f] = g_arity[f];
    __syncthreads();
    const uint8_t* arity = arity_in_smem ? s_arity : g_arity;
    const uint32_t nblocks = gridDim.x;
    const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
    const uint32_t nthreads = nblocks * kBlock;
    uint32_t epoch = 0;
#if TRS_B200_PROFILE
    // profiling build: phase ns (clear, mark, renumber, pack) in ctl->gcprof
    const bool gl = blockIdx.x == 0 && threadIdx.x == 0;
    uint64_t gt = gl ? global_ns() : 0;
#define TRS_EXPORT_MARK(k)                       \
    if (gl) {                                    \
        const uint64_t now = global_ns();        \
        P.ctl->gcprof[k] = now - gt;             \
        gt = now;                                \
    }
#else
#define TRS_EXPORT_MARK(k)
#endif
    // clear the reference counters
    for (uint32_t y = tid; y < bump; y += nthreads) X.newrc[y] = 0;
    grid_sync(P.ctl, nblocks, epoch);
    TRS_EXPORT_MARK(0)
    // Marking runs on one shared work queue with no levels: an S^k numeral
    // under a deep tree would otherwise cost a whole chain walk per level.
    // Items are pushed by a tail counter into zeroed slots; a thread claims
    // the next slot by a head counter and waits for it to be filled, or for
    // `pending` (pushed but unfinished items) to reach zero, which means no
    // further push can happen.  Every root occurrence pins once.
    uint32_t* tail = X.counters + 0;
    uint32_t* head = X.counters + 1;
    uint32_t* pending = X.counters + 2;
    uint32_t* Q = X.queue[0];
    for (uint32_t r = tid; r < P.num_roots; r += nthreads) {
        const uint32_t x = P.roots[r];
        if (atomicAdd(X.newrc + x, 1u) == 0u) {
            atomicAdd(pending, 1u);
            Q[atomicAdd(tail, 1u)] = x;
        }
    }
    grid_sync(P.ctl, nblocks, epoch);
    for (;;) {
        const uint32_t i = atomicAdd(head, 1u);
        // at most bump - 1 items are ever pushed: a later index stays empty
        // (and lies past the queue, which a small store's grid outnumbers)
        if (i >= bump) break;
        uint32_t x = 0;
        uint32_t ns = 32;
        while ((x = ld_acquire(Q + i)) == 0u) {
            // pending reaches zero only after every push (release below):
            // one more look at the slot settles it
            if (ld_acquire(pending) == 0u) {
                x = ld_acquire(Q + i);
                break;
            }
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
        }
        if (x == 0u) break;
        uint4 h4 = make_uint4(0u, 0u, 0u, 0u), a4 = h4;
        if (x) {
            h4 = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)x * W));
            a4 = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)x * W + kWArgs));
        }
        while (x) {
            const uint32_t* R = A + (size_t)x * W;
            if (h4.x == kDeadHead) {
                // a live term references a collected slot: extract's
                // DanglingReference (term_store.cpp:84-88)
                atomicExch(X.counters + 3, x);
                break;
            }
            const uint32_t ar = arity[h4.x & kSymMask];
            // speculate that the walk continues into the first argument (S^k
            // numerals, list spines): its record load overlaps the reference
            // count round trip that decides it
            uint4 sh = make_uint4(0u, 0u, 0u, 0u), sa = sh;
            if (ar && a4.x != 0u && a4.x < bump) {
                sh = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)a4.x * W));
                sa = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)a4.x * W + kWArgs));
            }
            uint32_t next = 0;
            for (uint32_t j = 0; j < ar; ++j) {
                const uint32_t c = j == 0 ? a4.x : j == 1 ? a4.y : j == 2 ? a4.z : j == 3 ? a4.w : __ldcg(R + kWArgs + j);
                if (c == 0u || c >= bump) {
                    // slot 0 or past the store: DanglingReference (term_store.cpp:84-88)
                    atomicExch(X.counters + 3, 0xFFFFFFFFu);
                    if (j == 0) a4.x = 0u;  // no speculated walk into it
                    continue;
                }
                if (atomicAdd(X.newrc + c, 1u) == 0u) {
                    if (next == 0) {
                        next = c;  // keep walking: a chain stays in one thread
                    } else {
                        atomicAdd(pending, 1u);
                        const uint32_t t = atomicAdd(tail, 1u);
                        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(Q + t), "r"(c) : "memory");
                    }
                }
            }
            if (next && next == a4.x) {
                h4 = sh;
                a4 = sa;
            } else if (next) {
                h4 = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)next * W));
                a4 = __ldcg(reinterpret_cast<const uint4*>(A + (size_t)next * W + kWArgs));
            }
            x = next;
        }
        red_release_add(pending, 0xFFFFFFFFu);  // -1, ordered after this item's pushes
    }
    grid_sync(P.ctl, nblocks, epoch);
    TRS_EXPORT_MARK(1)
    // renumber live slots in arena order: per-CTA contiguous ranges of
    // 8-slot groups, each thread a group per pass (two 16-byte loads of the
    // reference counts, two 16-byte stores of the map), one block scan per
    // 4096 slots
    const uint32_t ngroups = (bump + 7) / 8;
    const uint32_t gchunk = (ngroups + nblocks - 1) / nblocks;
    const uint32_t glo = blockIdx.x * gchunk;
    const uint32_t ghi = min(ngroups, glo + gchunk);
    auto live_bits = [&](uint32_t g) -> uint32_t {
        const uint32_t y = g * 8;
        uint32_t rc[8];
        if (y + 8 <= bump) {
            const uint4 a = __ldcg(reinterpret_cast<const uint4*>(X.newrc + y));
            const uint4 b = __ldcg(reinterpret_cast<const uint4*>(X.newrc + y + 4));
            rc[0] = a.x, rc[1] = a.y, rc[2] = a.z, rc[3] = a.w, rc[4] = b.x, rc[5] = b.y, rc[6] = b.z, rc[7] = b.w;
        } else {
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) rc[k] = y + k < bump ? __ldcg(X.newrc + y + k) : 0u;
        }
        uint32_t bits = 0;
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k) bits |= (rc[k] != 0u ? 1u : 0u) << k;
        return y == 0 ? bits & ~1u : bits;  // slot 0 is never live
    };
    uint32_t cnt = 0;
    for (uint32_t g = glo + threadIdx.x; g < ghi; g += kBlock) cnt += __popc(live_bits(g));
    uint32_t tot;
    block_scan(cnt, &tot, sm);
    if (threadIdx.x == 0) P.blocksum[blockIdx.x] = tot;
    grid_sync(P.ctl, nblocks, epoch);
    uint32_t prefix = 0, all = 0;
    for (uint32_t b = threadIdx.x; b < nblocks; b += kBlock) {
        const uint32_t c = __ldcg(P.blocksum + b);
        all += c;
        if (b < blockIdx.x) prefix += c;
    }
    {
        uint32_t t1, t2;
        block_scan(prefix, &t1, sm);
        block_scan(all, &t2, sm);
        prefix = t1;
        all = t2;
    }
    uint32_t running = 1 + prefix;
    for (uint32_t g0 = glo; g0 < ghi; g0 += kBlock) {
        const uint32_t g = g0 + threadIdx.x;
        const uint32_t live = g < ghi ? live_bits(g) : 0u;  // bit k: slot 8g + k is live
        uint32_t t;
        uint32_t e = running + block_scan(__popc(live), &t, sm);
        if (g < ghi) {
            uint32_t m[8];
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) {
                m[k] = ((live >> k) & 1u) ? e : 0u;
                e += (live >> k) & 1u;
            }
            const uint32_t y = g * 8;
            if (y + 8 <= bump) {
                *reinterpret_cast<uint4*>(X.map + y) = make_uint4(m[0], m[1], m[2], m[3]);
                *reinterpret_cast<uint4*>(X.map + y + 4) = make_uint4(m[4], m[5], m[6], m[7]);
            } else {
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k)
                    if (y + k < bump) X.map[y + k] = m[k];
            }
        }
        running += t;
    }
    const uint32_t n = 1 + all;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.ctl->export_n = n;
        X.map[0] = 0;
    }
    grid_sync(P.ctl, nblocks, epoch);
    TRS_EXPORT_MARK(2)
    // the columns are packed by pack_range, slot range by slot range, so the
    // host can copy each range out while the next one packs
    if (tid == 0) {
        X.hss[0] = 0;
        X.rcs[0] = 0;
        X.nf[0] = 0;
        for (uint32_t j = 0; j < X.ma; ++j) X.args[(size_t)j * n] = 0;
    }
    for (uint32_t r = tid; r < P.num_roots; r += nthreads) X.roots_out[r] = __ldcg(X.map + P.roots[r]);
#if TRS_B200_PROFILE
    grid_sync(P.ctl, nblocks, epoch);
    TRS_EXPORT_MARK(3)
#endif
}

// Pack live slots [lo, hi) of the arena into the reference columns: slot y
// goes to row map[y]; rows of a slot range are contiguous (renumbering keeps
// arena order).  Eight slots per thread per pass, their reference counts
// loaded together (most slots are garbage and only cost that load).
template <int W>
__global__ void __launch_bounds__(kBlock) pack_range(const uint32_t* __restrict__ A, ExportArgs X, uint32_t n,
                                                     const uint8_t* __restrict__ arity, uint32_t lo, uint32_t hi) {
    constexpr uint32_t kPer = 8;
    const uint32_t nthreads = gridDim.x * blockDim.x;
    for (uint32_t y0 = lo + (blockIdx.x * blockDim.x + threadIdx.x) * kPer; y0 < hi; y0 += nthreads * kPer) {
        uint32_t rcs[kPer];
#pragma unroll
        for (uint32_t q = 0; q < kPer; ++q) rcs[q] = y0 + q < hi ? __ldcg(X.newrc + y0 + q) : 0u;
#pragma unroll
        for (uint32_t q = 0; q < kPer; ++q) {
            const uint32_t y = y0 + q;
            const uint32_t rc = rcs[q];
            if (!rc) continue;
            const uint32_t k = __ldcg(X.map + y);
            const uint32_t* R = A + (size_t)y * W;
            const uint4 q0 = __ldcg(reinterpret_cast<const uint4*>(R));  // head, epoch, rc, waiter
            const uint32_t sym = q0.x & kSymMask;
            const uint32_t ar = arity[sym];
            X.hss[k] = sym;
            X.rcs[k] = rc;
            X.nf[k] = epoch_nf(q0.y);
            for (uint32_t j = 0; j < X.ma; ++j)
                X.args[(size_t)j * n + k] = j < ar ? __ldcg(X.map + __ldcg(R + kWArgs + j)) : 0u;
        }
    }
}

}  // namespace trs_b200

// Canonical relabelling of the normal forms on the device (SURVEY.md §3b.9,
// §8(f)2): per root, pre-order from the root, children left to right, ids on
// first visit, words = (symbol, child ids...) per id -- the relabelling the
// reference's parity check applies to extract()'s Term DAG
// (term_store.cpp:77-116; oracle/ref_driver.cpp canonical_words).
//
// Input: the export staging (export.cuh): the live store in the reference
// column layout, slots 1..n-1, with references recounted (rc = live parents +
// root pins).  When every live slot has rc == 1 the roots' graphs are
// disjoint trees and the first-visit order is the tree pre-order, which is
// computed in parallel:
//   1. init: size = 1, wsz = 1 + arity (its words), pending = arity, parent
//      pointers (one writer per child in a forest);
//   2. up: from every leaf, walk towards the root adding subtree sizes; the
//      child that completes a parent (pending -> 0) carries on with it, so a
//      chain (S^k numerals, list spines) is one thread's walk;
//   3. root offsets: exclusive scan of the roots' word counts;
//   4. down: from the roots, a node's id and word position give its
//      children's (id(c_j) = id(x) + 1 + sum_{k<j} size(c_k), likewise word
//      positions), its words are written, and the walk continues into the
//      first child while the others go on a shared work queue (export.cuh's
//      queue discipline);
//   5. a 64-bit hash per root of its words (position-keyed SplitMix64 sum),
//      so a caller can compare normal forms without copying words back.
// A store with sharing (rc != 1 somewhere) takes canon_seq: one thread runs
// the reference's own stack walk root after root.  Every BASELINE normal
// form is a forest (tests/test_gpu_parity.py).
#pragma once

#include "device_common.cuh"

namespace trs_b200 {

struct CanonArgs {
    // export staging (column layout, n slots)
    const uint32_t* hss;
    const uint32_t* args;  // [ma * n]
    const uint32_t* rcs;
    const uint32_t* roots;  // renumbered roots
    uint32_t num_roots;
    uint32_t n;
    uint32_t ma;
    const uint8_t* arity;
    // scratch, n words each
    uint32_t* par;
    uint32_t* size;
    uint32_t* wsz;
    uint32_t* pending;
    uint32_t* id;
    uint32_t* wpos;
    uint32_t* rootof;
    uint32_t* queue;
    uint32_t* stack;        // canon_seq: [ma * n + num_roots]
    uint32_t* counters;     // [4]: tail, head, pending, shared flag
    uint32_t* nodes;        // [num_roots] nodes per root
    unsigned long long* woff;  // [num_roots + 1] word offsets (absolute)
    unsigned long long* hash;  // [num_roots]
    uint32_t* words;        // output
};

__host__ __device__ __forceinline__ unsigned long long canon_mix(unsigned long long k, uint32_t w) {
    // SplitMix64 finaliser of (position, word): the per-root hash is the sum
    // over the root's words (tests/test_gpu_parity.py restates it in numpy)
    unsigned long long z = (k << 32) ^ (unsigned long long)w ^ 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void canon_init(CanonArgs X) {
    const uint32_t stride = gridDim.x * blockDim.x;
    bool shared = false;
    for (uint32_t y = blockIdx.x * blockDim.x + threadIdx.x; y < X.n; y += stride) {
        if (y == 0) continue;
        const uint32_t ar = X.arity[X.hss[y]];
        X.size[y] = 1;
        X.wsz[y] = 1 + ar;
        X.pending[y] = ar;
        if (X.rcs[y] != 1) shared = true;
        for (uint32_t j = 0; j < ar; ++j) X.par[X.args[(size_t)j * X.n + y]] = y;
    }
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < X.num_roots; r += stride) X.par[X.roots[r]] = 0;
    if (__syncthreads_or(shared) && threadIdx.x == 0) atomicExch(X.counters + 3, 1u);
}

__global__ void canon_up(CanonArgs X) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t y = blockIdx.x * blockDim.x + threadIdx.x; y < X.n; y += stride) {
        if (y == 0 || X.arity[X.hss[y]] != 0) continue;
        uint32_t x = y;
        for (;;) {
            const uint32_t p = __ldcg(X.par + x);
            if (p == 0) break;  // a root
            atomicAdd(X.size + p, __ldcg(X.size + x));
            atomicAdd(X.wsz + p, __ldcg(X.wsz + x));
            __threadfence();
            if (atomicSub(X.pending + p, 1u) != 1u) break;  // a sibling completes p
            __threadfence();
            x = p;
        }
    }
}

// Exclusive scan of the roots' word counts into absolute offsets (one CTA).
__global__ void __launch_bounds__(kBlock) canon_offsets(CanonArgs X) {
    __shared__ Smem sm;
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t r0 = 0; r0 < X.num_roots; r0 += kBlock) {
        const uint32_t r = r0 + threadIdx.x;
        const unsigned long long v = r < X.num_roots ? __ldcg(X.wsz + X.roots[r]) : 0ull;
        // 64-bit exclusive scan via a 32-bit scan of counts split in two halves
        uint32_t tlo, thi;
        const uint32_t lo = block_scan((uint32_t)(v & 0xFFFFu), &tlo, sm);
        const uint32_t hi = block_scan((uint32_t)(v >> 16), &thi, sm);
        const unsigned long long ex = (unsigned long long)lo + ((unsigned long long)hi << 16);
        if (r < X.num_roots) {
            X.woff[r] = carry + ex;
            X.hash[r] = 0ull;
            const uint32_t x = X.roots[r];
            X.nodes[r] = __ldcg(X.size + x);
            X.id[x] = 0;
            X.wpos[x] = (uint32_t)(carry + ex);  // n * (1 + ma) < 2^32 words (checked by the host)
            X.rootof[x] = r;
            X.queue[r] = x;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += (unsigned long long)tlo + ((unsigned long long)thi << 16);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        X.woff[X.num_roots] = carry;
        X.counters[0] = X.num_roots;  // tail
        X.counters[1] = 0;            // head
        X.counters[2] = X.num_roots;  // pending
    }
}

// Top-down numbering and word emission on one shared work queue (the
// export's discipline: tail/head counters over zeroed slots, `pending` =
// pushed but unfinished items).  Cooperative launch: every thread that waits
// on a queue slot has its producers co-resident.
__global__ void __launch_bounds__(kBlock) canon_down(CanonArgs X) {
    uint32_t* tail = X.counters + 0;
    uint32_t* head = X.counters + 1;
    uint32_t* pending = X.counters + 2;
    // the roots are queue items [0, num_roots), counted in `pending` by the
    // host, so `pending` cannot reach zero before every root was taken
    for (;;) {
        const uint32_t i = atomicAdd(head, 1u);
        if (i >= X.n) break;  // at most n - 1 items are ever pushed
        uint32_t x = 0;
        uint32_t ns = 32;
        while ((x = ld_acquire(X.queue + i)) == 0u) {
            if (ld_acquire(pending) == 0u) {
                x = ld_acquire(X.queue + i);
                break;
            }
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
        }
        if (x == 0u) break;
        uint32_t xid = __ldcg(X.id + x), xw = __ldcg(X.wpos + x), r = __ldcg(X.rootof + x);
        const unsigned long long base = X.woff[r];
        unsigned long long h = 0;
        while (x) {
            const uint32_t sym = X.hss[x];
            const uint32_t ar = X.arity[sym];
            X.words[xw] = sym;
            h += canon_mix(xw - base, sym);
            uint32_t cid = xid + 1, cw = xw + 1 + ar;
            uint32_t next = 0, nid = 0, nw = 0;
            for (uint32_t j = 0; j < ar; ++j) {
                const uint32_t c = X.args[(size_t)j * X.n + x];
                X.words[xw + 1 + j] = cid;
                h += canon_mix(xw + 1 + j - base, cid);
                if (j == 0) {
                    next = c, nid = cid, nw = cw;
                } else {
                    X.id[c] = cid;
                    X.wpos[c] = cw;
                    X.rootof[c] = r;
                    __threadfence();
                    atomicAdd(pending, 1u);
                    const uint32_t t = atomicAdd(tail, 1u);
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(X.queue + t), "r"(c) : "memory");
                }
                cid += __ldcg(X.size + c);
                cw += __ldcg(X.wsz + c);
            }
            x = next, xid = nid, xw = nw;
        }
        atomicAdd(X.hash + r, h);
        red_release_add(pending, 0xFFFFFFFFu);  // -1, ordered after this item's pushes
    }
}

// Stores with sharing: the reference's own walk (an explicit stack, children
// pushed right to left, ids on first visit), one root after another on one
// thread; `stamp` (X.par) = root index + 1 marks this root's visits.
__global__ void canon_seq(CanonArgs X) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    unsigned long long wbase = 0;  // X.par is zeroed by the host
    for (uint32_t r = 0; r < X.num_roots; ++r) {
        const uint32_t stamp = r + 1;
        uint32_t sp = 0, nid = 0;
        X.stack[sp++] = X.roots[r];
        while (sp) {
            const uint32_t x = X.stack[--sp];
            if (X.par[x] == stamp) continue;
            X.par[x] = stamp;
            X.id[x] = nid;
            X.queue[nid++] = x;  // visit order
            const uint32_t ar = X.arity[X.hss[x]];
            for (uint32_t j = ar; j-- > 0;) X.stack[sp++] = X.args[(size_t)j * X.n + x];
        }
        X.woff[r] = wbase;
        unsigned long long h = 0, k = 0;
        for (uint32_t q = 0; q < nid; ++q) {
            const uint32_t x = X.queue[q];
            const uint32_t sym = X.hss[x];
            const uint32_t ar = X.arity[sym];
            X.words[wbase + k] = sym;
            h += canon_mix(k++, sym);
            for (uint32_t j = 0; j < ar; ++j) {
                const uint32_t cid = X.id[X.args[(size_t)j * X.n + x]];
                X.words[wbase + k] = cid;
                h += canon_mix(k++, cid);
            }
        }
        X.hash[r] = h;
        X.nodes[r] = nid;
        wbase += k;
    }
    X.woff[X.num_roots] = wbase;
}

// Exact live count (the reference's live_terms, sweep_engine.cpp:122-123:
// slots with refcount > 0) over [1, bump) of an arena.
template <int W>
__global__ void count_live(const uint32_t* __restrict__ A, uint32_t bump, unsigned long long* out) {
    uint32_t c = 0;
    for (uint32_t y = 1 + blockIdx.x * blockDim.x + threadIdx.x; y < bump; y += gridDim.x * blockDim.x) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(A + (size_t)y * W));
        c += (q.x != kDeadHead && q.z != 0) ? 1u : 0u;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// Host-launched refcount recount (gc.cuh recount_refs as two kernels), for
// a store left by runs that kept no refcounts: before live_count, and before
// a validating run continues such a store.
template <int W>
__global__ void recount_clear(uint32_t* __restrict__ A, uint32_t bump) {
    for (uint32_t y = 1 + blockIdx.x * blockDim.x + threadIdx.x; y < bump; y += gridDim.x * blockDim.x)
        A[(size_t)y * W + kWRc] = 0u;
}
template <int W>
__global__ void recount_add(uint32_t* __restrict__ A, uint32_t bump, const uint8_t* __restrict__ arity,
                            const uint32_t* __restrict__ roots, uint32_t num_roots) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    for (uint32_t y = 1 + tid; y < bump; y += nthreads) {
        const uint32_t* R = A + (size_t)y * W;
        const uint32_t head = R[kWHead];
        if (head == kDeadHead) continue;
        const uint32_t ar = arity[head & kSymMask];
        for (uint32_t j = 0; j < ar; ++j) atomicAdd(A + (size_t)R[kWArgs + j] * W + kWRc, 1u);
    }
    for (uint32_t r = tid; r < num_roots; r += nthreads) atomicAdd(A + (size_t)roots[r] * W + kWRc, 1u);
}

}  // namespace trs_b200

// Device validate mode (trs_gpu_options.validate = 2): quiescent-point scans
// of the whole store before every grid sweep and at the end of the run, the
// device counterpart of the reference's SweepOptions::validate
// (sweep_engine.cpp:307-379):
//   * refcount ghost invariant: rc of every uncollected slot = references
//     from uncollected slots + root pins (:335-359);
//   * no live slot references slot 0, a slot past the store or a collected
//     slot (:341-344, extract's DanglingReference);
//   * nf monotonicity: a slot nf at one quiescent point is nf with the same
//     epoch at the next (:361-366, nf never falls within a slot lifetime);
//   * inner-most safety and snapshot discipline, checked on the store: an nf
//     slot's arguments are nf with EARLIER epochs (it was derived, or copied
//     from an nf source, only after they were nf_read, :314-329);
//   * garbage is nf (refcount 0 implies nf);
//   * no lost slot: every live slot that is not nf is on the frontier of the
//     next sweep or subscribed to one of its arguments (the frontier-list
//     engine's own liveness invariant; the reference has no counterpart
//     because it rescans every slot).
// The first violation is recorded (kind, slot) and the run stops; the host
// maps it onto TRS_GPU_DANGLING with the reference's message text.
#pragma once

#include "gc.cuh"

namespace trs_b200 {

enum ValidateKind : uint32_t {
    kValOk = 0,
    kValDangling = 1,
    kValGhost = 2,
    kValMonotone = 3,
    kValInnerMost = 4,
    kValGarbage = 5,
    kValLost = 6,
};

__device__ __forceinline__ void val_fail(const Params& P, uint32_t kind, uint32_t slot) {
    if (atomicCAS(&P.ctl->val_kind, 0u, kind) == 0u) P.ctl->val_slot = slot;
}

// All CTAs; `F` is the staged frontier of the next sweep (list buffer cur).
// Scratch: P.val (3 words per slot: counted references, frontier mark,
// previous epoch word), zeroed by the host before the run.
template <int W>
__device__ void validate_store_device(const Params& P, const Prog& G, uint32_t arena_idx, uint32_t bump,
                                      const Frontier& F, uint32_t cur, uint32_t block_rank, uint32_t nblocks,
                                      uint32_t& epoch, bool monotone) {
    const uint32_t* A = P.arena[arena_idx];
    uint32_t* counted = P.val;
    uint32_t* on_list = P.val + P.capacity;
    uint32_t* prev = P.val + 2 * P.capacity;
    const uint32_t tid = block_rank * kBlock + threadIdx.x;
    const uint32_t nthreads = nblocks * kBlock;
    if (!monotone) {
        // a collection renumbered the slots (or the launch is new): no epoch
        // recorded before it is comparable, above the new bump pointer either
        for (uint64_t x = tid; x < P.capacity; x += nthreads) prev[x] = 0u;
        grid_sync(P.ctl, nblocks, epoch);
    }
    // phase 1: count references, mark the frontier, check the arguments
    for (uint32_t x = 1 + tid; x < bump; x += nthreads) {
        const uint32_t* R = A + (size_t)x * W;
        const uint32_t head = __ldcg(R + kWHead);
        if (head == kDeadHead) continue;
        const uint32_t ep = __ldcg(R + kWEpoch);
        const uint32_t ar = G.arity[head & kSymMask];
        for (uint32_t j = 0; j < ar; ++j) {
            const uint32_t c = __ldcg(R + kWArgs + j);
            if (c == 0 || c >= bump || __ldcg(A + (size_t)c * W + kWHead) == kDeadHead) {
                val_fail(P, kValDangling, x);
                continue;
            }
            atomicAdd(counted + c, 1u);
            if (epoch_nf(ep)) {
                const uint32_t ce = __ldcg(A + (size_t)c * W + kWEpoch);
                if (!epoch_nf(ce) || (ce & kEpochMask) >= (ep & kEpochMask)) val_fail(P, kValInnerMost, x);
            }
        }
    }
    for (uint32_t r = tid; r < P.num_roots; r += nthreads) atomicAdd(counted + __ldcg(P.roots + r), 1u);
    const uint32_t* L = P.list[cur];
    for (uint32_t v = tid; v < F.M; v += nthreads) on_list[__ldcg(L + frontier_phys(F, v))] = 1u;
    grid_sync(P.ctl, nblocks, epoch);
    // phase 2: per-slot invariants, then reset the scratch for the next scan
    for (uint32_t x = 1 + tid; x < bump; x += nthreads) {
        const uint32_t* R = A + (size_t)x * W;
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(R));  // head, epoch, rc, waiter
        const uint32_t pe = prev[x];
        if (q.x == kDeadHead) {
            prev[x] = 0u;
            counted[x] = 0u;
            on_list[x] = 0u;
            continue;
        }
        if (__ldcg(counted + x) != q.z) val_fail(P, kValGhost, x);
        if (monotone && epoch_nf(pe) && pe != q.y) val_fail(P, kValMonotone, x);
        if (q.z == 0u && !epoch_nf(q.y)) val_fail(P, kValGarbage, x);
        if (q.z != 0u && !epoch_nf(q.y) && !on_list[x]) {
            bool subscribed = false;
            const uint32_t ar = G.arity[q.x & kSymMask];
            for (uint32_t j = 0; j < ar && !subscribed; ++j) {
                const uint32_t c = __ldcg(R + kWArgs + j);
                if (c != 0 && c < bump) subscribed = __ldcg(A + (size_t)c * W + kWWaiter) == x;
            }
            if (!subscribed) val_fail(P, kValLost, x);
        }
        prev[x] = q.y;
        counted[x] = 0u;
        on_list[x] = 0u;
    }
    grid_sync(P.ctl, nblocks, epoch);
}

}  // namespace trs_b200

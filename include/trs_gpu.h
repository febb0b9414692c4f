/*
 * trs_gpu.h — C ABI of the B200 term-rewriting engine (libtrs_b200.so).
 *
 * This is the drop-in boundary named by SURVEY.md §8(b): POD in, POD out,
 * integer status codes, no exceptions, no torch or C++ types.  It replaces
 * the reference's sweep engine behind its own C++ API:
 *
 *   SweepTrace run(TermStore&, const DispatchTable&, const SweepOptions&)
 *                                   proj/include/trs/sweep_engine.hpp:38-47
 *   TermStore  load(const RewriteSystem&, const Term&, uint32_t capacity)
 *                                   proj/include/trs/term_store.hpp:47-52
 *   Term       extract(const TermStore&)
 *                                   proj/include/trs/term_store.hpp:54-57
 *   DispatchTable compile(const RewriteSystem&)   proj/include/trs/dispatch.hpp:80
 *
 * A C++ caller keeps those signatures (see INTEGRATION.md for the adapter
 * that flattens the reference's TermStore/DispatchTable into these structs
 * and the one-line "gpu" branch in run_engine, proj/src/bench.cpp:49-69).
 *
 * Status codes map 1:1 onto the reference's error model
 * (proj/include/trs/error.hpp:8-20):
 *   TRS_GPU_STEP_BUDGET -> EngineError(EngineFault::StepBudget)
 *   TRS_GPU_CAPACITY    -> EngineError(EngineFault::Capacity)
 *   TRS_GPU_DANGLING    -> EngineError(EngineFault::DanglingReference)
 *   TRS_GPU_INVALID     -> std::invalid_argument (bad program/store/options)
 *   TRS_GPU_CUDA        -> CUDA runtime failure (no device, OOM, launch error)
 *
 * Threading: one engine handle per device, used by one host thread at a
 * time (the reference's run is not reentrant on one store either,
 * sweep_engine.cpp:34-46).  Distinct handles may run concurrently.
 */
#ifndef TRS_GPU_H
#define TRS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRS_GPU_OK 0
#define TRS_GPU_STEP_BUDGET 1
#define TRS_GPU_CAPACITY 2
#define TRS_GPU_DANGLING 3
#define TRS_GPU_INVALID 4
#define TRS_GPU_CUDA 5

#define TRS_GPU_STEP_CHECK_HEAD 0u
#define TRS_GPU_STEP_BIND_VAR 1u

/* RHS reference: TRS_GPU_REF_NODE | instruction index, or a bare var slot. */
#define TRS_GPU_REF_NODE 0x80000000u

typedef struct trs_gpu_engine trs_gpu_engine;

/* One match step (reference MatchStep, dispatch.hpp:15-21).  The reference
 * stores a child-index path from the redex root; steps run in pre-order so
 * the node at path p.j is child j of the node an earlier CheckHead step (or
 * the redex root) reached at path p.  `parent` is the index (within the
 * rule) of that step, -1 for the redex root; `child` is j. */
typedef struct trs_gpu_step {
    uint32_t kind;   /* TRS_GPU_STEP_CHECK_HEAD / TRS_GPU_STEP_BIND_VAR */
    int32_t parent;  /* step index within the rule, -1 = redex root */
    uint32_t child;  /* child index at the parent */
    uint32_t value;  /* symbol (CheckHead) or var slot (BindVar) */
} trs_gpu_step;

/* One RHS build instruction (reference RhsInstr, dispatch.hpp:40-46).
 * Children are refs[first_ref .. first_ref + arity(symbol)). */
typedef struct trs_gpu_instr {
    uint32_t symbol;
    uint32_t indegree;
    uint32_t first_ref;
} trs_gpu_instr;

/* One compiled rule (reference CompiledRule, dispatch.hpp:66-70). */
typedef struct trs_gpu_rule {
    uint32_t source_order;
    uint32_t first_step, num_steps;
    uint32_t first_instr, num_instrs; /* topological; root last unless collapsing */
    uint32_t num_vars;
    uint32_t root_ref; /* TRS_GPU_REF_NODE|k (constructive) or var slot (collapse) */
} trs_gpu_rule;

/* Flattened DispatchTable (dispatch.hpp:73-78) plus the signature arities
 * (TermStore::arity_of, term_store.hpp:19).  Rules of symbol f are
 * rules[rule_begin[f] .. rule_begin[f+1]) in source order; first match wins
 * (dispatch.hpp:119-130). */
typedef struct trs_gpu_program {
    uint32_t num_symbols;
    const uint32_t* arity;      /* [num_symbols] */
    const uint32_t* rule_begin; /* [num_symbols + 1] */
    uint32_t num_rules;
    const trs_gpu_rule* rules;
    uint32_t num_steps;
    const trs_gpu_step* steps;
    uint32_t num_instrs;
    const trs_gpu_instr* instrs;
    uint32_t num_refs;
    const uint32_t* refs;
} trs_gpu_program;

/* Options (reference SweepOptions, sweep_engine.hpp:29-36, plus the device
 * knobs).  Zero-initialise and set what you need; 0 means "default". */
typedef struct trs_gpu_options {
    uint64_t step_budget;      /* 0 -> 1e9 (sweep_engine.hpp:32) */
    uint32_t fixed_capacity;   /* 1: never grow; CAPACITY when the arena fills */
    uint32_t validate;         /* 1: check the refcount ghost invariant after the run; 2: also scan the whole
                                  store before every sweep (ghost refcounts, dangling references, nf
                                  monotonicity, inner-most safety, garbage is nf, no lost slot; grid mode
                                  only), the reference's validate mode (sweep_engine.cpp:307-379);
                                  violations: TRS_GPU_DANGLING */
    uint32_t small_enter;      /* frontier size at/below which one CTA runs the sweeps (0 -> default) */
    uint32_t small_exit;       /* frontier size above which the whole grid takes over again */
    uint32_t disable_small;    /* 1: never use single-CTA mode */
    uint32_t gc_interval;      /* >0: force a compacting GC every this many sweeps (testing) */
    uint32_t disable_gc;       /* 1: never collect (grow instead) */
    uint32_t blocks_per_sm;    /* 0 -> occupancy maximum */
    uint32_t variant;          /* step-loop register budget: 0/1 = 1 CTA/SM no spills, 2 = 2 CTAs/SM */
    uint32_t max_blocks;       /* >0: cap the persistent grid (profiling the single-CTA mode) */
    uint32_t profile;          /* 1: accumulate per-phase cycle counters (trs_gpu_profile_counters); >1: only grid sweeps of <= profile entries */
    uint32_t disable_warp_mode; /* 1: frontiers <= 32 slots still run on the whole CTA */
    uint32_t reserved[4];       /* [0] zero; [1] bit 0: no shared-memory resident arena in
                                   the single-CTA mode, bit 1: interpreted (not specialised) step loop,
                                   bit 2: no run-ahead (also off with an explicit step_budget or a fixed
                                   capacity, or TRS_B200_RUNAHEAD=0); [2] slab override (0); [3] zero */
} trs_gpu_options;

/* Per-sweep record (reference SweepRecord, sweep_engine.hpp:10-17).
 * trs_gpu_trace returns one record per LOGICAL sweep -- the reference's
 * sweeps -- with `rewrites` the sweep width, bit-exact to the reference; the
 * engine may run ahead of the sweep it physically executes (a lane carries on
 * with a slot its own step made ready, at that slot's logical sweep), so the
 * other fields are 0 there.  trs_gpu_phys_trace returns one record per
 * PHYSICAL sweep (a step-loop iteration): rewrites performed in it, n = the
 * arena bump pointer, live_terms = bump - 1 (allocated slots not yet
 * reclaimed by a compaction; the reference's refcount > 0 count is
 * trs_gpu_live_count), free_len = 0 (bump allocation leaves no free list),
 * active = frontier entries, mode 0 grid-wide, 1 single-CTA, 2 warp / solo,
 * 3 single-CTA over the shared-memory resident arena, and the duration. */
typedef struct trs_gpu_sweep_record {
    uint32_t sweep;
    uint32_t live_terms;
    uint64_t rewrites;
    uint32_t n;
    uint32_t free_len;
    uint32_t active;
    uint32_t mode;
    uint64_t micros_x1000; /* sweep duration in ns (device globaltimer) */
} trs_gpu_sweep_record;

typedef struct trs_gpu_stats {
    uint64_t total_rewrites;
    uint64_t max_width;
    uint32_t sweeps;
    uint32_t gc_runs;
    uint32_t small_sweeps;     /* sweeps run by the single-CTA mode */
    uint32_t launches;         /* kernels launched by this run (all are ours) */
    uint32_t regrows;          /* host-side arena growths */
    uint32_t grid_blocks;
    uint32_t block_threads;
    uint32_t record_words;
    uint64_t peak_slots;       /* highest bump pointer reached */
    uint64_t live_terms;       /* allocated slots at the end (bump - 1); exact refcount > 0 count: trs_gpu_live_count */
    double kernel_ms;          /* device time of the step-loop launches (CUDA events) */
    double gc_ms;              /* device time spent inside compacting GC (globaltimer) */
    double load_ms;            /* device time of the load kernel */
} trs_gpu_stats;

/* The entry points below are host functions; the device code of the
 * per-program specialisation (NVRTC) includes this header for the types only. */
#ifndef __CUDACC_RTC__

/* Number of visible CUDA devices (0 when none / no driver). */
int trs_gpu_device_count(void);

int trs_gpu_open(int device, trs_gpu_engine** out);
void trs_gpu_close(trs_gpu_engine* engine);
const char* trs_gpu_error_string(int status);
/* Last detailed error message of this engine (empty when none). */
const char* trs_gpu_last_error(trs_gpu_engine* engine);

/* Stage the flattened DispatchTable in device memory (replaces the previous
 * program).  TRS_GPU_INVALID for a malformed program or one beyond the
 * device limits (max arity 28, 32 instructions / 48 steps / 48 vars per
 * rule, program blob <= 40 KiB). */
int trs_gpu_set_program(trs_gpu_engine* engine, const trs_gpu_program* program);

/* Load a term store (reference TermStore layout, term_store.hpp:15-45):
 * slots [1, n) hold terms, slot 0 is never a term; hss[i] is the head
 * symbol; args is column-major, args[j * n + i] for j < max_arity (0 =
 * absent); refcounts already include one pin per root.  `roots` lists the
 * root slots (one per independent term).  capacity 0 sizes the arena
 * automatically; an explicit capacity < n fails with TRS_GPU_CAPACITY
 * (term_store.cpp:50-53).  Buffers are HOST pointers; they are copied. */
int trs_gpu_load(trs_gpu_engine* engine, uint32_t n, const uint32_t* roots, uint32_t num_roots,
                 const uint32_t* hss, const uint32_t* args, uint32_t max_arity,
                 const uint32_t* refcounts, uint64_t capacity);

/* Same, from DEVICE pointers already resident in HBM (bench `value` path). */
int trs_gpu_load_device(trs_gpu_engine* engine, uint32_t n, const uint32_t* roots,
                        uint32_t num_roots, const uint32_t* d_hss, const uint32_t* d_args,
                        uint32_t max_arity, const uint32_t* d_refcounts, uint64_t capacity);

/* Normalise every loaded root (reference run, sweep_engine.cpp:428-430).
 * Synchronous.  On TRS_GPU_STEP_BUDGET / TRS_GPU_CAPACITY the store is left
 * as the failing sweep left it, like the reference. */
int trs_gpu_run(trs_gpu_engine* engine, const trs_gpu_options* options, trs_gpu_stats* stats);

/* trs_gpu_run split in two: _async enqueues the step loop on the engine
 * stream and returns at once; _wait blocks until the run ends (relaunching
 * on the rare arena growth / trace growth) and reports like trs_gpu_run.
 * One pending run per engine. */
int trs_gpu_run_async(trs_gpu_engine* engine, const trs_gpu_options* options);
int trs_gpu_run_wait(trs_gpu_engine* engine, trs_gpu_stats* stats);

/* Per-program specialisation (the paper's generated rewrite functions,
 * PAPER.md:305-327): trs_gpu_set_program compiles the step loop with the
 * program's rule bindings and right-hand sides as straight-line code (NVRTC);
 * TRS_B200_JIT=0 in the environment keeps the interpreted kernel, and
 * trs_gpu_options.reserved[1] bit 1 selects it for one run.  Reports whether
 * the specialised kernel is active, its compile time and the compiler log. */
int trs_gpu_jit_info(trs_gpu_engine* engine, int* active, double* seconds, char* log, uint64_t log_cap);

/* Stream gate: _hold enqueues a wait on a host-mapped flag so a whole step
 * (load + run) can be enqueued before the device starts it; _release opens
 * it.  Nothing that synchronises the engine stream may be called between
 * the two (e.g. trs_gpu_load, which waits for its copies). */
int trs_gpu_hold(trs_gpu_engine* engine);
int trs_gpu_release(trs_gpu_engine* engine);

/* Per-sweep records of the last run, one per logical sweep (the reference's
 * trace); *count receives the number of records (copies min(count, cap)). */
int trs_gpu_trace(trs_gpu_engine* engine, trs_gpu_sweep_record* out, uint64_t cap, uint64_t* count);

/* Per-physical-sweep records of the last run (diagnostics: duration, mode,
 * frontier size, rewrites executed in that step-loop iteration). */
int trs_gpu_phys_trace(trs_gpu_engine* engine, trs_gpu_sweep_record* out, uint64_t cap, uint64_t* count);

/* Canonical DAG words of root `root_index` (pre-order from
 * the root, children left to right, ids on first visit, words = symbol then
 * child ids per id).  Two-call protocol: if cap < needed, nothing is copied
 * and *n_words receives the size.  TRS_GPU_DANGLING when the root's graph
 * references slot 0 or a dead slot (term_store.cpp:84-88). */
int trs_gpu_canonical(trs_gpu_engine* engine, uint32_t root_index, uint32_t* words, uint64_t cap,
                      uint64_t* n_words, uint32_t* n_nodes);

/* Canonical words of EVERY root, computed on the device (canon.cuh; SURVEY.md
 * §8(f)2) from the export of the current store: words of root r are
 * words[root_offsets[r] .. root_offsets[r+1]); hashes[r] is a 64-bit
 * position-keyed hash of them (sum over k of SplitMix64((k << 32) ^ w_k ^
 * 0x9e3779b97f4a7c15)) for comparisons without the copy; root_nodes[r] the
 * node count.  Any output pointer may be NULL; words are copied only when
 * cap >= *n_words.  Replaces extract + relabelling (term_store.cpp:77-116). */
int trs_gpu_canonical_all(trs_gpu_engine* engine, uint32_t* words, uint64_t cap, uint64_t* n_words,
                          uint64_t* root_offsets, uint64_t* hashes, uint32_t* root_nodes);

/* The program as staged on the device (read back from device memory),
 * rendered in the reference's dump-dispatch format (dispatch.cpp:98-134), so
 * it can be compared byte for byte with the reference's own dump of the same
 * system.  Names come from the caller's signature: symbol_names[symbol],
 * var_names[variable]; device rule r (rules in trs_gpu_program order) maps
 * variable slot k to variable rule_vars[rule_var_begin[r] + k]; rule_texts
 * [source_order] is "lhs = rhs" as the reference prints it.  Two-call
 * protocol on cap (*need includes the terminating NUL). */
int trs_gpu_dump_program(trs_gpu_engine* engine, const char* const* symbol_names, const char* const* var_names,
                         const uint32_t* rule_var_begin, const uint32_t* rule_vars, const char* const* rule_texts,
                         char* out, uint64_t cap, uint64_t* need);

/* Layout evidence: one pass of the derive's probe pattern (a slot's head,
 * epoch word and arguments, then each argument's head and epoch word) over
 * every slot of the current store, read from the engine's 8-word AoS records
 * (layout 0) or from SoA columns built from them, the reference TermStore
 * layout (layout 1); layouts 2 and 3 are the same two visiting the slots in
 * a hashed (random) order instead of slot order.  Reports ms per pass (CUDA events, `iters` passes) and
 * the slots scanned; ncu on trs_gpu_layout_probe's kernels gives the DRAM
 * bytes and sectors of each layout. */
int trs_gpu_layout_probe(trs_gpu_engine* engine, uint32_t layout, uint32_t iters, double* ms_per_pass,
                         uint64_t* nodes);

/* Exact count of slots with refcount > 0 in the current store: the
 * reference's live_terms (sweep_engine.cpp:122-123), which includes
 * garbage not yet collected.  Runs without validate keep no refcounts step
 * by step; they are recounted from the store first (references from
 * uncollected slots + root pins, the reference's ghost invariant). */
int trs_gpu_live_count(trs_gpu_engine* engine, uint64_t* live);

/* Raw store copy-back (reference TermStore layout): after a compacting pass
 * the live slots are renumbered 1..n-1 in their arena order, roots updated.
 * Pass NULL arrays to query n first.  args is column-major [max_arity * n]. */
int trs_gpu_fetch_store(trs_gpu_engine* engine, uint32_t* n, uint32_t* roots, uint32_t* hss,
                        uint32_t* args, uint32_t* refcounts, uint8_t* nf, uint32_t cap);

/* The CUDA stream (cudaStream_t) every call of this engine runs on, for
 * callers that bracket calls with their own CUDA events. */
void* trs_gpu_stream(trs_gpu_engine* engine);

/* Debug phase counters, accumulated over runs; filled only by the profiling
 * build (libtrs_b200_prof.so), zeros otherwise.  out18: cycles of the
 * profiled warp in match, claim, apply, push, whole sweep; sweeps; warp
 * steps; spare; match sub-phases record, children, slots, rules; then the
 * collector's phase ns (claim, count, scatter, remap), cascade hops and the
 * longest cascade; then, per profiled grid sweep summed, the maxima over
 * warps of match, claim, apply, push, record, children, slots, rules. */
int trs_gpu_profile_counters(trs_gpu_engine* engine, uint64_t* out26);

/* Fixed per-sweep overhead probe on the loaded store: `iters` grid barriers
 * (mode 0) or barriers plus the frontier-table staging of a grid sweep
 * (mode 1) in one step-loop launch; reports ns per iteration.  Leaves the
 * store untouched except for timing fields. */
int trs_gpu_overhead_probe(trs_gpu_engine* engine, uint32_t iters, uint32_t mode, uint32_t max_blocks,
                           double* ns_per_iter);

/* Compacting collection on demand (up to max_rounds passes, 0 -> 8, stops
 * when a pass reclaims nothing): afterwards the arena holds only slots
 * still referenced, renumbered densely, roots updated. */
int trs_gpu_compact(trs_gpu_engine* engine, uint32_t max_rounds, trs_gpu_stats* stats);

/* Raw copy of the device arena [0, n) into dst (record_words u32 per slot:
 * head|cursor<<24, nf epoch, refcount, waiter, args...) and of the root
 * slots into roots_out (may be NULL).  Two-call protocol on cap_bytes.
 * Refcount words are recounted first when the last run kept none. */
int trs_gpu_fetch_records(trs_gpu_engine* engine, void* dst, uint64_t cap_bytes, uint64_t* bytes,
                          uint32_t* record_words, uint32_t* roots_out);

/* Device-side roofline probe: `iters` launches of a uniformly random 4-byte
 * (bytes_per_access = 4), 8-, 16- or 32-byte gather over a power-of-two array
 * of at most `bytes` in HBM (indices streamed coalesced, 4 independent
 * gathers in flight per thread, a full SM of threads).  Returns achieved GB/s
 * counting bytes_per_access per access. */
int trs_gpu_gather_probe(int device, uint64_t bytes, uint32_t bytes_per_access, uint32_t iters,
                         double* gbps);

/* The same probe with `ilp` (1, 2, 4, 8 or 16) independent gathers in flight
 * per thread (trs_gpu_gather_probe uses 4): the roofline curve over footprint,
 * access size and memory-level parallelism. */
int trs_gpu_gather_probe_ex(int device, uint64_t bytes, uint32_t bytes_per_access, uint32_t ilp, uint32_t iters,
                            double* gbps);

#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif

#endif /* TRS_GPU_H */

/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle restating the reference rewriters.
 * See trs_oracle.h for scope; every function cites the reference lines it
 * follows.  Plain C11, single-threaded, deterministic.
 */
#define _POSIX_C_SOURCE 199309L
#include "trs_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORACLE_MAX_VARS 64
#define ORACLE_MAX_STEPS 256
#define ORACLE_MAX_INSTRS 256

static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static void* xrealloc(void* p, size_t bytes) {
    void* q = realloc(p, bytes ? bytes : 1);
    if (!q) abort();
    return q;
}

/* ---- growable vectors --------------------------------------------------- */

typedef struct {
    uint64_t* v;
    size_t n, cap;
} vec64;

typedef struct {
    uint32_t* v;
    size_t n, cap;
} vec32;

static void push64(vec64* a, uint64_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 1024;
        a->v = xrealloc(a->v, a->cap * sizeof(uint64_t));
    }
    a->v[a->n++] = x;
}

static void push32(vec32* a, uint32_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 1024;
        a->v = xrealloc(a->v, a->cap * sizeof(uint32_t));
    }
    a->v[a->n++] = x;
}

/* ---- the reference TermStore (term_store.hpp:15-45) ---------------------- */

typedef struct {
    uint32_t capacity, n, maxarity;
    uint32_t* hss;
    uint32_t** args; /* args[j][i] */
    uint8_t *nf, *nf_read;
    uint32_t *rc, *rc_read;
    uint8_t* collected;
    uint32_t* free_indices;
    uint64_t next_free_begin, next_free_end;
    uint32_t next_fresh;
    uint8_t* cursor;
} Store;

/* TermStore::grow (term_store.cpp:8-27) */
static void store_grow(Store* s, uint32_t cap) {
    if (cap <= s->capacity) return;
    size_t old = s->capacity;
#define GROW(p, T)                                          \
    do {                                                    \
        p = xrealloc(p, (size_t)cap * sizeof(T));           \
        memset(p + old, 0, ((size_t)cap - old) * sizeof(T)); \
    } while (0)
    GROW(s->hss, uint32_t);
    for (uint32_t j = 0; j < s->maxarity; ++j) GROW(s->args[j], uint32_t);
    GROW(s->nf, uint8_t);
    GROW(s->nf_read, uint8_t);
    GROW(s->rc, uint32_t);
    GROW(s->rc_read, uint32_t);
    GROW(s->collected, uint8_t);
    GROW(s->cursor, uint8_t);
#undef GROW
    /* compact the live ring window under the new geometry */
    uint64_t w = s->next_free_end > s->next_free_begin ? s->next_free_end - s->next_free_begin : 0;
    uint32_t* win = malloc((size_t)(w ? w : 1) * sizeof(uint32_t));
    for (uint64_t p = 0; p < w; ++p) win[p] = s->free_indices[(s->next_free_begin + p) % s->capacity];
    free(s->free_indices);
    s->free_indices = calloc(cap, sizeof(uint32_t));
    memcpy(s->free_indices, win, (size_t)w * sizeof(uint32_t));
    free(win);
    s->next_free_begin = 0;
    s->next_free_end = w;
    s->capacity = cap;
}

static void store_free(Store* s) {
    free(s->hss);
    for (uint32_t j = 0; j < s->maxarity; ++j) free(s->args[j]);
    free(s->args);
    free(s->nf);
    free(s->nf_read);
    free(s->rc);
    free(s->rc_read);
    free(s->collected);
    free(s->free_indices);
    free(s->cursor);
}

/* get_new_index (term_store.cpp:118-138), single-threaded */
static uint32_t get_new_index(Store* s, uint32_t region_n) {
    uint32_t id = 0;
    if (s->next_free_begin < s->next_free_end) {
        uint64_t b = s->next_free_begin++;
        if (b < s->next_free_end) id = s->free_indices[b % s->capacity];
    }
    if (id == 0) {
        uint64_t slot = (uint64_t)region_n + s->next_fresh++;
        if (slot >= s->capacity) return 0;
        id = (uint32_t)slot;
    }
    s->collected[id] = 0;
    return id;
}

/* collect_free_indices (term_store.cpp:140-157) */
static void collect_free_indices(Store* s, const uint32_t* arity, uint32_t lo, uint32_t hi) {
    for (uint32_t i = lo; i < hi; ++i) {
        if (s->rc[i] != 0 || s->collected[i]) continue;
        s->collected[i] = 1;
        for (uint32_t j = 0; j < arity[s->hss[i]]; ++j) s->rc[s->args[j][i]]--;
        s->free_indices[s->next_free_end % s->capacity] = i;
        s->next_free_end++;
    }
}

/* ---- matcher (dispatch.hpp:95-130) over the (parent, child) step form ----- */

typedef struct {
    const trs_gpu_program* p;
    uint32_t* step_depth; /* depth of each step's path */
} Prog;

/* Returns the chosen rule index or -1; fills bind[].  `head`/`child` read
 * the subject store; counters follow SURVEY.md §8(d). */
typedef uint32_t (*head_fn)(void* ctx, uint32_t node);
typedef uint32_t (*child_fn)(void* ctx, uint32_t node, uint32_t j);

static int try_rules(const Prog* P, uint32_t sym, uint32_t subject, void* ctx, head_fn head, child_fn child,
                     uint32_t* bind, oracle_counts* c) {
    const trs_gpu_program* p = P->p;
    uint32_t node[ORACLE_MAX_STEPS];
    for (uint32_t r = p->rule_begin[sym]; r < p->rule_begin[sym + 1]; ++r) {
        const trs_gpu_rule* R = &p->rules[r];
        int ok = 1;
        for (uint32_t t = 0; t < R->num_steps && ok; ++t) {
            const trs_gpu_step* st = &p->steps[R->first_step + t];
            uint32_t at = st->parent < 0 ? subject : node[st->parent];
            uint32_t x = child(ctx, at, st->child);
            node[t] = x;
            if (c) c->path_hops += P->step_depth[R->first_step + t] - 1;
            if (st->kind == TRS_GPU_STEP_CHECK_HEAD) {
                if (c) c->checkhead++;
                if (head(ctx, x) != st->value) ok = 0;
            } else {
                bind[st->value] = x;
            }
        }
        if (ok) return (int)r;
    }
    return -1;
}

static void prog_init(Prog* P, const trs_gpu_program* p) {
    P->p = p;
    P->step_depth = calloc(p->num_steps ? p->num_steps : 1, sizeof(uint32_t));
    for (uint32_t r = 0; r < p->num_rules; ++r) {
        const trs_gpu_rule* R = &p->rules[r];
        for (uint32_t t = 0; t < R->num_steps; ++t) {
            const trs_gpu_step* st = &p->steps[R->first_step + t];
            P->step_depth[R->first_step + t] = st->parent < 0 ? 1 : P->step_depth[R->first_step + st->parent] + 1;
        }
    }
}

static uint32_t max_new_slots(const trs_gpu_program* p) {
    uint32_t m = 0;
    for (uint32_t r = 0; r < p->num_rules; ++r)
        if (p->rules[r].root_ref & TRS_GPU_REF_NODE)
            if (p->rules[r].num_instrs - 1 > m) m = p->rules[r].num_instrs - 1;
    return m;
}

static uint32_t st_head(void* ctx, uint32_t node) { return ((Store*)ctx)->hss[node]; }
static uint32_t st_child(void* ctx, uint32_t node, uint32_t j) { return ((Store*)ctx)->args[j][node]; }

/* canonical DAG words of a slot graph */
static void canonical(uint32_t root, uint32_t limit, const uint32_t* arity, void* ctx, head_fn head,
                      child_fn child, uint32_t** words_out, uint64_t* n_out) {
    uint32_t* id = malloc((size_t)limit * sizeof(uint32_t));
    memset(id, 0xff, (size_t)limit * sizeof(uint32_t));
    vec32 order = {0}, stack = {0}, w = {0};
    push32(&stack, root);
    while (stack.n) {
        uint32_t x = stack.v[--stack.n];
        if (id[x] != UINT32_MAX) continue;
        id[x] = (uint32_t)order.n;
        push32(&order, x);
        uint32_t ar = arity[head(ctx, x)];
        for (uint32_t j = ar; j-- > 0;) push32(&stack, child(ctx, x, j));
    }
    for (size_t k = 0; k < order.n; ++k) {
        uint32_t x = order.v[k];
        uint32_t f = head(ctx, x);
        push32(&w, f);
        for (uint32_t j = 0; j < arity[f]; ++j) push32(&w, id[child(ctx, x, j)]);
    }
    free(id);
    free(order.v);
    free(stack.v);
    *words_out = w.v;
    *n_out = w.n;
}

/* ---- sweep engine (sweep_engine.cpp:69-258), workers = 1 ----------------- */

int oracle_sweep(const trs_gpu_program* prog, uint32_t n, const uint32_t* roots, uint32_t num_roots,
                 const uint32_t* hss, const uint32_t* args, uint32_t max_arity, const uint32_t* refcounts,
                 uint64_t step_budget, int want_words, oracle_result* out) {
    memset(out, 0, sizeof(*out));
    if (!step_budget) step_budget = 1000000000ull;
    Prog P;
    prog_init(&P, prog);
    const uint32_t* arity = prog->arity;
    const uint32_t max_new = max_new_slots(prog);
    Store s;
    memset(&s, 0, sizeof(s));
    s.maxarity = max_arity;
    s.args = calloc(max_arity ? max_arity : 1, sizeof(uint32_t*));
    store_grow(&s, n); /* load: capacity = needed (term_store.cpp:59) */
    s.n = n;
    for (uint32_t i = 0; i < n; ++i) {
        s.hss[i] = hss[i];
        s.rc[i] = refcounts[i];
        for (uint32_t j = 0; j < max_arity; ++j) s.args[j][i] = args[(size_t)j * n + i];
    }
    vec64 widths = {0};
    vec32 live = {0}, nvec = {0}, flen = {0};
    oracle_counts* C = &out->counts;
    uint64_t total = 0;
    uint32_t sweep = 0;
    uint32_t bind[ORACLE_MAX_VARS];
    uint32_t fresh[ORACLE_MAX_INSTRS];
    uint32_t old_children[64];
    int status = 0;
    double t0 = now_s();
    for (;;) {
        ++sweep;
        /* ensure_headroom (:290-303) */
        uint64_t needed = (uint64_t)s.n + (uint64_t)(s.n - 1) * max_new + 1;
        if (needed > s.capacity) {
            uint64_t target = needed;
            if ((uint64_t)s.capacity * 2 > target) target = (uint64_t)s.capacity * 2;
            if (target < 64) target = 64;
            if (target > UINT32_MAX) {
                status = TRS_GPU_CAPACITY;
                break;
            }
            store_grow(&s, (uint32_t)target);
        }
        /* snapshot (:80-81) */
        memcpy(s.nf_read, s.nf, s.n);
        memcpy(s.rc_read, s.rc, (size_t)s.n * sizeof(uint32_t));
        int done = 1, gc = 0, aborted = 0;
        uint64_t width = 0;
        const uint32_t region_n = s.n;
        for (uint32_t i = 1; i < region_n; ++i) C->frontier_sum += s.rc_read[i] && !s.nf_read[i];
        /* derive_phase / derive_slot (:153-188) */
        for (uint32_t i = 1; i < region_n && !aborted; ++i) {
            C->visits++;
            if (s.rc_read[i] == 0) {
                C->dead_visits++;
                if (!s.collected[i]) gc = 1;
                continue;
            }
            if (s.nf_read[i]) continue;
            done = 0;
            uint32_t sym = s.hss[i];
            uint32_t ar = arity[sym];
            uint32_t j = s.cursor[i];
            while (j < ar && s.nf_read[s.args[j][i]]) ++j;
            s.cursor[i] = (uint8_t)j;
            if (j < ar) continue;
            C->eligible++;
            C->child_nf_reads += ar;
            C->own_args += ar;
            int r = try_rules(&P, sym, i, &s, st_head, st_child, bind, C);
            if (r < 0) {
                s.nf[i] = 1;
                continue;
            }
            /* apply_rule_at (:190-258) */
            const trs_gpu_rule* R = &prog->rules[r];
            for (uint32_t k = 0; k < ar; ++k) old_children[k] = s.args[k][i];
            if (!(R->root_ref & TRS_GPU_REF_NODE)) {
                uint32_t src = bind[R->root_ref];
                uint32_t f = s.hss[src];
                uint32_t sar = arity[f];
                s.hss[i] = f;
                for (uint32_t k = 0; k < sar; ++k) {
                    uint32_t c = s.args[k][src];
                    s.args[k][i] = c;
                    s.rc[c]++;
                }
                for (uint32_t k = sar; k < s.maxarity; ++k) s.args[k][i] = 0;
                s.nf[i] = 1;
                C->collapse_reads += 1 + sar;
                C->rc_rmw += sar;
            } else {
                uint32_t nnew = R->num_instrs - 1;
                for (uint32_t k = 0; k < nnew; ++k) {
                    fresh[k] = get_new_index(&s, region_n);
                    if (fresh[k] == 0) {
                        aborted = 1;
                        break;
                    }
                }
                if (aborted) break;
                for (uint32_t k = 0; k <= nnew; ++k) {
                    const trs_gpu_instr* I = &prog->instrs[R->first_instr + k];
                    uint32_t at = k < nnew ? fresh[k] : i;
                    uint32_t iar = arity[I->symbol];
                    s.hss[at] = I->symbol;
                    for (uint32_t q = 0; q < iar; ++q) {
                        uint32_t ref = prog->refs[I->first_ref + q];
                        uint32_t v = (ref & TRS_GPU_REF_NODE) ? fresh[ref & 0x7fffffffu] : bind[ref];
                        s.args[q][at] = v;
                        if (!(ref & TRS_GPU_REF_NODE)) {
                            s.rc[v]++;
                            C->rc_rmw++;
                        }
                    }
                    for (uint32_t q = iar; q < s.maxarity; ++q) s.args[q][at] = 0;
                    if (k < nnew) {
                        s.rc[at] = I->indegree;
                        s.nf[at] = 0;
                        s.cursor[at] = 0;
                    }
                }
                s.nf[i] = 0;
                C->fresh_nodes += nnew;
            }
            s.cursor[i] = 0;
            for (uint32_t k = 0; k < ar; ++k) s.rc[old_children[k]]--;
            C->rc_rmw += ar;
            width++;
        }
        /* fold (:94-106) */
        uint64_t folded = (uint64_t)s.n + s.next_fresh;
        s.n = (uint32_t)(folded < s.capacity ? folded : s.capacity);
        s.next_fresh = 0;
        if (s.next_free_begin > s.next_free_end) s.next_free_begin = s.next_free_end;
        total += width;
        C->rewrites += width;
        if (gc) collect_free_indices(&s, arity, 1, s.n); /* (:108-115), one ordered pass with one worker */
        uint32_t lv = 0;
        for (uint32_t i = 1; i < s.n; ++i) lv += s.rc[i] > 0;
        push64(&widths, width);
        push32(&live, lv);
        push32(&nvec, s.n);
        push32(&flen, s.next_free_begin < s.next_free_end ? (uint32_t)(s.next_free_end - s.next_free_begin) : 0);
        if (aborted) {
            status = TRS_GPU_CAPACITY;
            break;
        }
        if (total > step_budget) {
            status = TRS_GPU_STEP_BUDGET;
            break;
        }
        if (done) break;
    }
    out->seconds = now_s() - t0;
    out->status = status;
    out->rewrites = total;
    out->sweeps = (uint32_t)widths.n;
    out->widths = widths.v;
    out->live = live.v;
    out->n = nvec.v;
    out->free_len = flen.v;
    out->num_roots = num_roots;
    if (want_words && status == 0) {
        out->words = calloc(num_roots, sizeof(uint32_t*));
        out->n_words = calloc(num_roots, sizeof(uint64_t));
        /* roots keep their slots (the reference rewrites in place) */
        for (uint32_t r = 0; r < num_roots; ++r)
            canonical(roots[r], s.n, arity, &s, st_head, st_child, &out->words[r], &out->n_words[r]);
    }
    store_free(&s);
    free(P.step_depth);
    return status;
}

/* ---- sequential engine (seq_engine.cpp:104-192) -------------------------- */

typedef struct {
    uint32_t maxarity;
    vec32 sym;
    vec32 kids; /* maxarity per node */
    vec32 nf;
} Graph;

static uint32_t g_new(Graph* g, uint32_t f) {
    uint32_t id = (uint32_t)g->sym.n;
    push32(&g->sym, f);
    push32(&g->nf, 0);
    for (uint32_t j = 0; j < (g->maxarity ? g->maxarity : 1); ++j) push32(&g->kids, 0);
    return id;
}
static uint32_t* g_kids(Graph* g, uint32_t x) { return g->kids.v + (size_t)x * (g->maxarity ? g->maxarity : 1); }
static uint32_t g_head(void* ctx, uint32_t x) { return ((Graph*)ctx)->sym.v[x]; }
static uint32_t g_child(void* ctx, uint32_t x, uint32_t j) { return g_kids((Graph*)ctx, x)[j]; }

int oracle_seq(const trs_gpu_program* prog, uint32_t n, const uint32_t* roots, uint32_t num_roots,
               const uint32_t* hss, const uint32_t* args, uint32_t max_arity, const uint32_t* refcounts,
               uint64_t step_budget, int want_words, oracle_result* out) {
    (void)refcounts;
    memset(out, 0, sizeof(*out));
    if (!step_budget) step_budget = 1000000000ull;
    Prog P;
    prog_init(&P, prog);
    const uint32_t* arity = prog->arity;
    Graph g;
    memset(&g, 0, sizeof(g));
    g.maxarity = max_arity;
    /* import: one node per slot (slot sharing = TermNode* sharing, seq_engine.cpp:34-65) */
    for (uint32_t i = 0; i < n; ++i) g_new(&g, hss[i]);
    for (uint32_t i = 1; i < n; ++i)
        for (uint32_t j = 0; j < arity[hss[i]]; ++j) g_kids(&g, i)[j] = args[(size_t)j * n + i];
    uint32_t bind[ORACLE_MAX_VARS];
    uint32_t built[ORACLE_MAX_INSTRS];
    uint64_t rewrites = 0;
    int status = 0;
    double t0 = now_s();
    typedef struct {
        uint32_t node, next;
    } Frame;
    Frame* stack = NULL;
    size_t sn = 0, scap = 0;
    for (uint32_t r = 0; r < num_roots && !status; ++r) {
        sn = 0;
#define PUSH(x)                                                    \
    do {                                                           \
        if (sn == scap) {                                          \
            scap = scap ? 2 * scap : 1024;                         \
            stack = xrealloc(stack, scap * sizeof(Frame));         \
        }                                                          \
        stack[sn].node = (x);                                      \
        stack[sn].next = 0;                                        \
        ++sn;                                                      \
    } while (0)
        PUSH(roots[r]);
        while (sn) {
            Frame* f = &stack[sn - 1];
            uint32_t x = f->node;
            if (g.nf.v[x]) {
                --sn;
                continue;
            }
            uint32_t ar = arity[g.sym.v[x]];
            while (f->next < ar && g.nf.v[g_kids(&g, x)[f->next]]) ++f->next;
            if (f->next < ar) {
                uint32_t c = g_kids(&g, x)[f->next];
                PUSH(c);
                continue;
            }
            int rule = try_rules(&P, g.sym.v[x], x, &g, g_head, g_child, bind, NULL);
            if (rule < 0) {
                g.nf.v[x] = 1;
                --sn;
                continue;
            }
            if (++rewrites > step_budget) {
                status = TRS_GPU_STEP_BUDGET;
                break;
            }
            const trs_gpu_rule* R = &prog->rules[rule];
            if (!(R->root_ref & TRS_GPU_REF_NODE)) {
                uint32_t src = bind[R->root_ref];
                g.sym.v[x] = g.sym.v[src];
                memcpy(g_kids(&g, x), g_kids(&g, src), sizeof(uint32_t) * (max_arity ? max_arity : 1));
                g.nf.v[x] = 1;
            } else {
                uint32_t nnew = R->num_instrs - 1;
                for (uint32_t k = 0; k <= nnew; ++k) {
                    const trs_gpu_instr* I = &prog->instrs[R->first_instr + k];
                    uint32_t at = k < nnew ? g_new(&g, I->symbol) : x;
                    if (k < nnew) built[k] = at;
                    uint32_t tmp[64];
                    uint32_t iar = arity[I->symbol];
                    for (uint32_t q = 0; q < iar; ++q) {
                        uint32_t ref = prog->refs[I->first_ref + q];
                        tmp[q] = (ref & TRS_GPU_REF_NODE) ? built[ref & 0x7fffffffu] : bind[ref];
                    }
                    g.sym.v[at] = I->symbol;
                    for (uint32_t q = 0; q < iar; ++q) g_kids(&g, at)[q] = tmp[q];
                    if (k == nnew) g.nf.v[at] = 0;
                }
            }
            stack[sn - 1].next = 0;
        }
#undef PUSH
    }
    out->seconds = now_s() - t0;
    free(stack);
    out->status = status;
    out->rewrites = rewrites;
    out->num_roots = num_roots;
    if (want_words && status == 0) {
        out->words = calloc(num_roots, sizeof(uint32_t*));
        out->n_words = calloc(num_roots, sizeof(uint64_t));
        for (uint32_t r = 0; r < num_roots; ++r)
            canonical(roots[r], (uint32_t)g.sym.n, arity, &g, g_head, g_child, &out->words[r], &out->n_words[r]);
    }
    free(g.sym.v);
    free(g.kids.v);
    free(g.nf.v);
    free(P.step_depth);
    return status;
}

/* ---- logical-time sweep engine ------------------------------------------
 *
 * The reference sweep engine (sweep_engine.cpp:69-258) re-examines every
 * slot every sweep.  Slot i rewrites (or is marked nf) in sweep t exactly
 * when, at the start of t,
 *   (a) it is live and not nf (:164-171; garbage is always nf, SURVEY.md
 *       §3b.10, so "not nf" implies live),
 *   (b) it was not claimed or rewritten in place during an earlier part of
 *       t (fresh slots lie at >= region_n and recycled ones read rc_read == 0,
 *       :86, :156; a rewritten root is visited once per sweep, :153-161), and
 *   (c) every argument is nf_read, i.e. became nf in a sweep before t
 *       (:80-81, :173-178).
 * All three are functions of event times: with b(i) the sweep in which i was
 * built or last rewritten in place (0 for the input) and e(c) the sweep in
 * which argument c became nf, i derives at
 *       T(i) = max(b(i) + 1, max_j e(arg_j) + 1),
 * and what it does there depends only on its own content and its nf
 * arguments (nf slots never change, :170, :202-215).  So the reference's
 * per-sweep widths, sweep count, rewrite total and normal form follow from
 * processing slots in ANY order that respects those dependencies: a slot
 * with a non-nf argument subscribes to it and is re-examined when it turns
 * nf.  This is the semantics the B200 engine's barrier-free run-ahead relies
 * on; tests/test_oracle.py pins it against the reference sweep engine's
 * traces (the golden fixtures) and oracle_sweep. */
int oracle_logical(const trs_gpu_program* prog, uint32_t n, const uint32_t* roots, uint32_t num_roots,
                   const uint32_t* hss, const uint32_t* args, uint32_t max_arity, const uint32_t* refcounts,
                   uint64_t step_budget, int want_words, oracle_result* out) {
    memset(out, 0, sizeof(*out));
    if (!step_budget) step_budget = 1000000000ull;
    Prog P;
    prog_init(&P, prog);
    const uint32_t* arity = prog->arity;
    Graph g;
    memset(&g, 0, sizeof(g));
    g.maxarity = max_arity;
    for (uint32_t i = 0; i < n; ++i) g_new(&g, hss[i]);
    for (uint32_t i = 1; i < n; ++i)
        for (uint32_t j = 0; j < arity[hss[i]]; ++j) g_kids(&g, i)[j] = args[(size_t)j * n + i];
    /* per node: nf epoch (g.nf, 0 = not nf), earliest derive sweep, waiter list */
    vec32 tmin = {0}, whead = {0}, wnext = {0};
    for (uint32_t i = 0; i < n; ++i) {
        push32(&tmin, 1);
        push32(&whead, 0);
        push32(&wnext, 0);
    }
    vec64 hist = {0};
    vec32 work = {0};
    for (uint32_t i = n; i-- > 1;)
        if (refcounts[i]) push32(&work, i);
    uint32_t bind[ORACLE_MAX_VARS];
    uint32_t built[ORACLE_MAX_INSTRS];
    uint64_t rewrites = 0;
    uint32_t last = 0; /* latest sweep with an event */
    int status = 0;
    double t0 = now_s();
#define WAKE(x)                                        \
    do {                                               \
        for (uint32_t w_ = whead.v[x]; w_;) {          \
            uint32_t nx_ = wnext.v[w_];                \
            push32(&work, w_);                         \
            w_ = nx_;                                  \
        }                                              \
        whead.v[x] = 0;                                \
    } while (0)
    while (work.n && !status) {
        uint32_t x = work.v[--work.n];
        if (g.nf.v[x]) continue;
        uint32_t f = g.sym.v[x], ar = arity[f];
        uint32_t T = tmin.v[x], pending = 0;
        for (uint32_t j = 0; j < ar; ++j) {
            uint32_t c = g_kids(&g, x)[j];
            if (!g.nf.v[c]) {
                pending = c;
                break;
            }
            if (g.nf.v[c] + 1 > T) T = g.nf.v[c] + 1;
        }
        if (pending) { /* sleep on the first non-nf argument (the reference's scan stops there, :173-178) */
            wnext.v[x] = whead.v[pending];
            whead.v[pending] = x;
            continue;
        }
        if (T > last) last = T;
        int rule = try_rules(&P, f, x, &g, g_head, g_child, bind, NULL);
        if (rule < 0) { /* no match: nf from this sweep on (:182-186) */
            g.nf.v[x] = T;
            WAKE(x);
            continue;
        }
        while (hist.n <= T) push64(&hist, 0);
        hist.v[T]++;
        if (++rewrites > step_budget) {
            status = TRS_GPU_STEP_BUDGET;
            break;
        }
        const trs_gpu_rule* R = &prog->rules[rule];
        if (!(R->root_ref & TRS_GPU_REF_NODE)) { /* collapse: copy, nf (:202-215) */
            uint32_t src = bind[R->root_ref];
            g.sym.v[x] = g.sym.v[src];
            memcpy(g_kids(&g, x), g_kids(&g, src), sizeof(uint32_t) * (max_arity ? max_arity : 1));
            g.nf.v[x] = T;
            WAKE(x);
            continue;
        }
        /* constructive: fresh nodes and the root in place, all derivable from T + 1 (:217-249) */
        uint32_t nnew = R->num_instrs - 1;
        for (uint32_t k = 0; k <= nnew; ++k) {
            const trs_gpu_instr* I = &prog->instrs[R->first_instr + k];
            uint32_t at = x;
            if (k < nnew) {
                at = g_new(&g, I->symbol);
                push32(&tmin, T + 1);
                push32(&whead, 0);
                push32(&wnext, 0);
                built[k] = at;
            }
            uint32_t tmp[64];
            uint32_t iar = arity[I->symbol];
            for (uint32_t q = 0; q < iar; ++q) {
                uint32_t ref = prog->refs[I->first_ref + q];
                tmp[q] = (ref & TRS_GPU_REF_NODE) ? built[ref & 0x7fffffffu] : bind[ref];
            }
            g.sym.v[at] = I->symbol;
            for (uint32_t q = 0; q < iar; ++q) g_kids(&g, at)[q] = tmp[q];
            push32(&work, at);
        }
        tmin.v[x] = T + 1;
    }
#undef WAKE
    out->seconds = now_s() - t0;
    out->status = status;
    out->rewrites = rewrites;
    out->num_roots = num_roots;
    /* the run ends at the first sweep after the last event (:147) */
    out->sweeps = status ? 0 : last + 1;
    if (!status) {
        out->widths = calloc(out->sweeps, sizeof(uint64_t));
        for (uint32_t t = 1; t < hist.n && t <= last; ++t) out->widths[t - 1] = hist.v[t];
    }
    if (want_words && status == 0) {
        out->words = calloc(num_roots, sizeof(uint32_t*));
        out->n_words = calloc(num_roots, sizeof(uint64_t));
        for (uint32_t r = 0; r < num_roots; ++r)
            canonical(roots[r], (uint32_t)g.sym.n, arity, &g, g_head, g_child, &out->words[r], &out->n_words[r]);
    }
    free(g.sym.v);
    free(g.kids.v);
    free(g.nf.v);
    free(tmin.v);
    free(whead.v);
    free(wnext.v);
    free(hist.v);
    free(work.v);
    free(P.step_depth);
    return status;
}

void oracle_free(oracle_result* r) {
    free(r->widths);
    free(r->live);
    free(r->n);
    free(r->free_len);
    if (r->words)
        for (uint32_t k = 0; k < r->num_roots; ++k) free(r->words[k]);
    free(r->words);
    free(r->n_words);
    memset(r, 0, sizeof(*r));
}

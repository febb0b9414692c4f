// Host-side C++ API of the B200 rewriter, mirroring the reference's
// "load a TRS, build a term, normalise it" interface:
//
//   load_system   proj/include/trs/parser.hpp:100     (parse + resolve, diagnostics)
//   compile       proj/include/trs/dispatch.hpp:80    (per-head rule programs, RHS templates)
//   dump_dispatch proj/include/trs/dispatch.hpp:84    (stable text, golden-tested)
//   load          proj/include/trs/term_store.hpp:52  (DAG -> SoA slots, root = 1, pin)
//   extract       proj/include/trs/term_store.hpp:57  (slots -> term DAG, dangling check)
//   gpu::run      proj/include/trs/sweep_engine.hpp:47 (the B200 engine behind trs_gpu.h)
//
// Representation differs on purpose: terms are nodes of a flat, append-only
// arena (children before parents) instead of shared_ptr trees, so deep
// inputs (2^14-element lists, S^2584 numerals) never recurse, and extracting
// an 8 M-node normal form is a linear pass.
// Physical sharing = same arena index, the counterpart of the reference's
// TermNode* identity (term_store.cpp:33-47).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "trs_gpu.h"

namespace trs_b200 {

using SymbolId = std::uint32_t;
using VarId = std::uint32_t;
using SortId = std::uint32_t;
using TermRef = std::uint32_t;

// ---- error model (proj/include/trs/error.hpp:8-20) -------------------------

enum class EngineFault { StepBudget, Capacity, DanglingReference };

class EngineError : public std::runtime_error {
public:
    EngineError(EngineFault f, const std::string& message) : std::runtime_error(message), fault(f) {}
    EngineFault fault;
};

// ---- signature / terms (proj/include/trs/term.hpp) ------------------------

struct SymbolInfo {
    std::string name;
    std::uint32_t arity = 0;
    SortId sort = 0;
    std::vector<SortId> argument_sorts;
};

struct VarInfo {
    std::string name;
    SortId sort = 0;
};

struct Signature {
    std::vector<std::string> sorts;
    std::vector<SymbolInfo> symbols;
    std::vector<VarInfo> variables;
    std::uint32_t max_arity = 0;
    std::unordered_map<std::string, SortId> sort_ids;
    std::unordered_map<std::string, SymbolId> symbol_ids;
    std::unordered_map<std::string, VarId> variable_ids;

    SortId add_sort(const std::string& name);
    SymbolId add_symbol(const std::string& name, SortId sort, std::vector<SortId> argument_sorts);
    VarId add_variable(const std::string& name, SortId sort);
};

// Append-only term DAG.  A node is a variable or a symbol application whose
// children were added earlier.
class TermArena {
public:
    TermRef variable(VarId v);
    TermRef apply(SymbolId f, const TermRef* children, std::uint32_t count);
    TermRef apply(SymbolId f, std::initializer_list<TermRef> children) {
        return apply(f, children.begin(), static_cast<std::uint32_t>(children.size()));
    }

    bool is_variable(TermRef t) const { return is_var_[t] != 0; }
    std::uint32_t id(TermRef t) const { return id_[t]; }  // symbol or variable
    std::uint32_t arity(TermRef t) const { return first_[t + 1] - first_[t]; }
    TermRef child(TermRef t, std::uint32_t j) const { return kids_[first_[t] + j]; }
    std::size_t size() const { return id_.size(); }
    void reserve(std::size_t nodes, std::size_t edges);

private:
    std::vector<std::uint32_t> id_;
    std::vector<std::uint8_t> is_var_;
    std::vector<std::uint32_t> first_{0};
    std::vector<TermRef> kids_;
};

bool is_ground(const TermArena& a, TermRef t);
// Structural (tree) equality, insensitive to sharing (term.cpp:102-120).
bool term_equal(const TermArena& a, TermRef x, const TermArena& b, TermRef y);
std::string print_term(const Signature& sig, const TermArena& a, TermRef t);

struct Rule {
    TermRef lhs = 0;
    TermRef rhs = 0;
    std::uint32_t source_order = 0;
};

struct RewriteSystem {
    Signature signature;
    TermArena terms;
    std::vector<Rule> rules;
    std::vector<std::vector<std::uint32_t>> rules_by_head;
    TermRef input_term = 0;
};

// ---- front end (proj/include/trs/parser.hpp) -------------------------------

struct SourceSpan {
    std::uint32_t line = 1, column = 1, length = 1;
};

enum class ErrorKind { Lex, Syntax, UnknownName, ArityMismatch, SortMismatch, RuleViolation, DuplicateName };
const char* error_kind_name(ErrorKind kind);

struct ParseError {
    SourceSpan span;
    ErrorKind kind = ErrorKind::Syntax;
    std::string message;
};

std::string format_error(std::string_view file, const ParseError& e);

struct ResolveResult {
    std::optional<RewriteSystem> system;
    std::vector<ParseError> errors;
};

ResolveResult load_system(std::string_view text);

// ---- compiled programs (proj/include/trs/dispatch.hpp) ---------------------

struct MatchStep {
    enum class Kind { CheckHead, BindVar };
    Kind kind;
    std::vector<std::uint8_t> path;
    SymbolId symbol = 0;
    std::uint32_t var_slot = 0;
    std::int32_t parent = -1;  // step reaching path[:-1] (-1 = redex root)
};

struct MatchProgram {
    SymbolId head = 0;
    std::vector<MatchStep> steps;
    std::vector<VarId> slot_vars;
};

struct RhsRef {
    enum class Kind { Var, Node };
    Kind kind;
    std::uint32_t index;
    bool operator<(const RhsRef& o) const {
        return kind != o.kind ? kind < o.kind : index < o.index;
    }
    bool operator==(const RhsRef& o) const { return kind == o.kind && index == o.index; }
};

struct RhsInstr {
    SymbolId symbol = 0;
    std::vector<RhsRef> children;
    std::uint32_t indegree = 0;
};

struct RhsTemplate {
    std::vector<RhsInstr> instructions;
    RhsRef root_ref{RhsRef::Kind::Var, 0};
    bool collapses() const { return root_ref.kind == RhsRef::Kind::Var; }
    std::uint32_t new_slots() const {
        return collapses() ? 0 : static_cast<std::uint32_t>(instructions.size()) - 1;
    }
};

struct CompiledRule {
    std::uint32_t rule_index = 0;
    MatchProgram program;
    RhsTemplate rhs;
};

struct DispatchTable {
    std::vector<std::vector<CompiledRule>> by_symbol;
    std::uint32_t max_new_slots = 0;
    const std::vector<CompiledRule>& rules_for(SymbolId f) const { return by_symbol[f]; }
};

DispatchTable compile(const RewriteSystem& system);
std::string dump_dispatch(const RewriteSystem& system, const DispatchTable& table);

// Flattened POD view for trs_gpu_set_program (owns its arrays).
struct FlatProgram {
    std::vector<std::uint32_t> arity, rule_begin, refs;
    std::vector<trs_gpu_rule> rules;
    std::vector<trs_gpu_step> steps;
    std::vector<trs_gpu_instr> instrs;
    trs_gpu_program view() const;
};

FlatProgram flatten(const RewriteSystem& system, const DispatchTable& table);

// ---- term store (proj/include/trs/term_store.hpp) ---------------------------

// Page-locked host memory for the store's columns (cudaHostAlloc), so load
// flattens the input straight into memory the device copies from without a
// staging copy (trs_gpu_load's H2D is then a direct DMA); plain heap memory
// where no CUDA device is present.  Defined in gpu_run.cpp.
void* pinned_alloc(std::size_t bytes);
void pinned_free(void* p) noexcept;

template <class T>
struct PinnedAlloc {
    using value_type = T;
    PinnedAlloc() = default;
    template <class U>
    PinnedAlloc(const PinnedAlloc<U>&) noexcept {}
    T* allocate(std::size_t n) { return static_cast<T*>(pinned_alloc(n * sizeof(T))); }
    void deallocate(T* p, std::size_t) noexcept { pinned_free(p); }
    template <class U>
    bool operator==(const PinnedAlloc<U>&) const noexcept { return true; }
    template <class U>
    bool operator!=(const PinnedAlloc<U>&) const noexcept { return false; }
};
template <class T>
using pinned_vector = std::vector<T, PinnedAlloc<T>>;

// Host mirror of the reference TermStore layout: slot 0 is never a term,
// args column-major (args[j * n + i]), refcounts include one pin per root.
struct TermStore {
    std::uint32_t n = 1;
    std::uint32_t capacity = 0;
    std::uint32_t maxarity = 0;
    std::vector<std::uint32_t> roots;
    std::vector<std::uint32_t> arity_of;
    pinned_vector<std::uint32_t> hss;
    pinned_vector<std::uint32_t> args;
    pinned_vector<std::uint32_t> refcounts;
    pinned_vector<std::uint8_t> nf;

    std::uint32_t root() const { return roots.empty() ? 0 : roots[0]; }
    std::uint32_t arg(std::uint32_t j, std::uint32_t i) const { return args[static_cast<std::size_t>(j) * n + i]; }
};

// Pre-order flattening, root first at slot 1, shared subterms once with
// in-degree refcounts (term_store.cpp:29-75).  Several inputs (same
// signature) load as one store with one pinned root each; their slots are
// numbered root after root.
TermStore load(const RewriteSystem& system, TermRef input, std::uint32_t capacity = 0);
TermStore load_many(const Signature& sig, const std::vector<std::pair<const TermArena*, TermRef>>& inputs,
                    std::uint32_t capacity = 0);

// Tree unfolding of root `root_index` into `out` (term_store.cpp:77-116);
// throws EngineError(DanglingReference) on slot 0 / out-of-range references.
TermRef extract(const TermStore& store, TermArena& out, std::uint32_t root_index = 0);

// Canonical DAG words, identical to trs_gpu_canonical.
std::vector<std::uint32_t> canonical_words(const TermArena& a, TermRef root, std::uint32_t* n_nodes = nullptr);
std::vector<std::uint32_t> canonical_words(const TermStore& s, std::uint32_t root_index = 0,
                                           std::uint32_t* n_nodes = nullptr);

// `idx  symbol  arg...  rc=k  nf|-` per slot (term_store.cpp:159-171).
std::string dump_store(const Signature& sig, const TermStore& store);

// ---- the B200 engine (proj/include/trs/sweep_engine.hpp) --------------------

struct SweepRecord {
    std::uint32_t sweep = 0;
    std::uint64_t rewrites = 0;
    std::uint32_t live_terms = 0;
    std::uint32_t n = 0;
    std::uint32_t free_len = 0;
    std::uint64_t micros = 0;
};

struct SweepTrace {
    std::vector<SweepRecord> records;
    trs_gpu_stats stats{};
    std::uint64_t total_rewrites() const;
    std::uint64_t max_width() const;
    std::uint64_t median_width() const;
};

namespace gpu {

struct GpuOptions {
    int device = 0;
    std::uint64_t step_budget = 1'000'000'000;
    bool fixed_capacity = false;
    bool validate = false;
    trs_gpu_options raw{};  // device knobs (small-frontier mode, GC interval, ...)
};

// Normalise every root of `store` on the GPU and write the normal form back
// into it (renumbered slots), like the reference's in-place run.  Throws
// EngineError on step budget / capacity / dangling, std::runtime_error on
// CUDA failures.
SweepTrace run(TermStore& store, const RewriteSystem& system, const DispatchTable& table,
               const GpuOptions& options = {});

}  // namespace gpu

void write_trace_csv(std::string& out, const SweepTrace& trace);

}  // namespace trs_b200

// Host term store: load / extract / canonical words / dump (counterpart of
// proj/src/term_store.cpp load, extract, dump_store).  The device side of
// the store (allocator, GC) lives in csrc/engine/engine.cu.
#include <algorithm>

#include "trs_host.hpp"

namespace trs_b200 {

TermStore load(const RewriteSystem& system, TermRef input, std::uint32_t capacity) {
    return load_many(system.signature, {{&system.terms, input}}, capacity);
}

TermStore load_many(const Signature& sig, const std::vector<std::pair<const TermArena*, TermRef>>& inputs,
                    std::uint32_t capacity) {
    if (inputs.empty()) throw std::invalid_argument("no input term");
    for (const auto& [a, t] : inputs)
        if (!is_ground(*a, t)) throw std::invalid_argument("derivations need a ground input term");
    // pre-order numbering, root first (term_store.cpp:33-47); shared nodes
    // (same arena index) get one slot
    std::vector<std::vector<std::uint32_t>> slot_of(inputs.size());
    std::vector<std::pair<std::uint32_t, TermRef>> order;  // (input, node)
    std::vector<std::uint32_t> roots;
    std::uint32_t next = 1;
    for (std::uint32_t r = 0; r < inputs.size(); ++r) {
        const TermArena& a = *inputs[r].first;
        auto& slots = slot_of[r];
        slots.assign(a.size(), 0);
        std::vector<TermRef> stack{inputs[r].second};
        while (!stack.empty()) {
            TermRef x = stack.back();
            stack.pop_back();
            if (slots[x]) continue;
            slots[x] = next++;
            order.emplace_back(r, x);
            for (std::uint32_t j = a.arity(x); j-- > 0;) stack.push_back(a.child(x, j));
        }
        roots.push_back(slots[inputs[r].second]);
    }
    const std::uint32_t needed = next;
    if (capacity != 0 && capacity < needed)
        throw EngineError(EngineFault::Capacity, "store capacity " + std::to_string(capacity) + " cannot hold " +
                                                     std::to_string(needed - 1) + " input term nodes");
    TermStore s;
    s.n = needed;
    s.capacity = capacity == 0 ? needed : capacity;
    s.maxarity = sig.max_arity;
    for (const SymbolInfo& si : sig.symbols) s.arity_of.push_back(si.arity);
    s.hss.assign(needed, 0);
    s.args.assign(static_cast<std::size_t>(s.maxarity) * needed, 0);
    s.refcounts.assign(needed, 0);
    s.nf.assign(needed, 0);
    for (const auto& [r, x] : order) {
        const TermArena& a = *inputs[r].first;
        std::uint32_t slot = slot_of[r][x];
        s.hss[slot] = a.id(x);
        for (std::uint32_t j = 0; j < a.arity(x); ++j) {
            std::uint32_t c = slot_of[r][a.child(x, j)];
            s.args[static_cast<std::size_t>(j) * needed + slot] = c;
            ++s.refcounts[c];
        }
    }
    for (std::uint32_t root : roots) ++s.refcounts[root];  // pin (term_store.cpp:73)
    s.roots = std::move(roots);
    return s;
}

TermRef extract(const TermStore& s, TermArena& out, std::uint32_t root_index) {
    if (root_index >= s.roots.size()) throw std::invalid_argument("root index out of range");
    auto check = [&](std::uint32_t slot) {
        if (slot == 0 || slot >= s.n)
            throw EngineError(EngineFault::DanglingReference, "slot " + std::to_string(slot) + " is not a live term");
    };
    std::vector<TermRef> memo(s.n, UINT32_MAX);
    struct Frame {
        std::uint32_t slot, next;
    };
    const std::uint32_t root = s.roots[root_index];
    check(root);
    std::vector<Frame> stack{{root, 0}};
    std::vector<TermRef> kids;
    while (!stack.empty()) {
        Frame& f = stack.back();
        std::uint32_t ar = s.arity_of[s.hss[f.slot]];
        if (f.next < ar) {
            std::uint32_t c = s.arg(f.next, f.slot);
            ++f.next;
            check(c);
            if (memo[c] == UINT32_MAX) stack.push_back({c, 0});
            continue;
        }
        kids.clear();
        for (std::uint32_t j = 0; j < ar; ++j) kids.push_back(memo[s.arg(j, f.slot)]);
        memo[f.slot] = out.apply(s.hss[f.slot], kids.data(), ar);
        stack.pop_back();
    }
    return memo[root];
}

std::vector<std::uint32_t> canonical_words(const TermArena& a, TermRef root, std::uint32_t* n_nodes) {
    std::unordered_map<TermRef, std::uint32_t> id;
    std::vector<TermRef> order;
    std::vector<TermRef> stack{root};
    while (!stack.empty()) {
        TermRef x = stack.back();
        stack.pop_back();
        if (id.count(x)) continue;
        id.emplace(x, static_cast<std::uint32_t>(order.size()));
        order.push_back(x);
        for (std::uint32_t j = a.arity(x); j-- > 0;) stack.push_back(a.child(x, j));
    }
    std::vector<std::uint32_t> w;
    for (TermRef x : order) {
        w.push_back(a.id(x));
        for (std::uint32_t j = 0; j < a.arity(x); ++j) w.push_back(id.at(a.child(x, j)));
    }
    if (n_nodes) *n_nodes = static_cast<std::uint32_t>(order.size());
    return w;
}

std::vector<std::uint32_t> canonical_words(const TermStore& s, std::uint32_t root_index, std::uint32_t* n_nodes) {
    std::vector<std::uint32_t> id(s.n, UINT32_MAX);
    std::vector<std::uint32_t> order;
    std::vector<std::uint32_t> stack{s.roots.at(root_index)};
    while (!stack.empty()) {
        std::uint32_t x = stack.back();
        stack.pop_back();
        if (x == 0 || x >= s.n)
            throw EngineError(EngineFault::DanglingReference, "slot " + std::to_string(x) + " is not a live term");
        if (id[x] != UINT32_MAX) continue;
        id[x] = static_cast<std::uint32_t>(order.size());
        order.push_back(x);
        for (std::uint32_t j = s.arity_of[s.hss[x]]; j-- > 0;) stack.push_back(s.arg(j, x));
    }
    std::vector<std::uint32_t> w;
    for (std::uint32_t x : order) {
        w.push_back(s.hss[x]);
        for (std::uint32_t j = 0; j < s.arity_of[s.hss[x]]; ++j) w.push_back(id[s.arg(j, x)]);
    }
    if (n_nodes) *n_nodes = static_cast<std::uint32_t>(order.size());
    return w;
}

std::string dump_store(const Signature& sig, const TermStore& s) {
    std::string out;
    for (std::uint32_t i = 1; i < s.n; ++i) {
        out += std::to_string(i) + "  " + sig.symbols[s.hss[i]].name;
        for (std::uint32_t j = 0; j < s.arity_of[s.hss[i]]; ++j) out += "  " + std::to_string(s.arg(j, i));
        out += "  rc=" + std::to_string(s.refcounts[i]);
        out += s.nf[i] ? "  nf" : "  -";
        out += '\n';
    }
    return out;
}

std::uint64_t SweepTrace::total_rewrites() const {
    std::uint64_t t = 0;
    for (const SweepRecord& r : records) t += r.rewrites;
    return t;
}

std::uint64_t SweepTrace::max_width() const {
    std::uint64_t m = 0;
    for (const SweepRecord& r : records) m = std::max(m, r.rewrites);
    return m;
}

std::uint64_t SweepTrace::median_width() const {
    if (records.empty()) return 0;
    std::vector<std::uint64_t> w;
    for (const SweepRecord& r : records) w.push_back(r.rewrites);
    std::sort(w.begin(), w.end());
    return w[w.size() / 2];
}

void write_trace_csv(std::string& out, const SweepTrace& trace) {
    out += "sweep,rewrites,live_terms,n,free_len,micros\n";
    for (const SweepRecord& r : trace.records)
        out += std::to_string(r.sweep) + "," + std::to_string(r.rewrites) + "," + std::to_string(r.live_terms) + "," +
               std::to_string(r.n) + "," + std::to_string(r.free_len) + "," + std::to_string(r.micros) + "\n";
}

}  // namespace trs_b200

// Signature and flat term arena (counterpart of proj/src/term.cpp).
#include <algorithm>

#include "trs_host.hpp"

namespace trs_b200 {

SortId Signature::add_sort(const std::string& name) {
    SortId id = static_cast<SortId>(sorts.size());
    sort_ids.emplace(name, id);
    sorts.push_back(name);
    return id;
}

SymbolId Signature::add_symbol(const std::string& name, SortId sort, std::vector<SortId> argument_sorts) {
    SymbolId id = static_cast<SymbolId>(symbols.size());
    SymbolInfo info;
    info.name = name;
    info.arity = static_cast<std::uint32_t>(argument_sorts.size());
    info.sort = sort;
    info.argument_sorts = std::move(argument_sorts);
    max_arity = std::max(max_arity, info.arity);
    symbol_ids.emplace(name, id);
    symbols.push_back(std::move(info));
    return id;
}

VarId Signature::add_variable(const std::string& name, SortId sort) {
    VarId id = static_cast<VarId>(variables.size());
    variable_ids.emplace(name, id);
    variables.push_back(VarInfo{name, sort});
    return id;
}

TermRef TermArena::variable(VarId v) {
    TermRef t = static_cast<TermRef>(id_.size());
    id_.push_back(v);
    is_var_.push_back(1);
    first_.push_back(first_.back());
    return t;
}

TermRef TermArena::apply(SymbolId f, const TermRef* children, std::uint32_t count) {
    TermRef t = static_cast<TermRef>(id_.size());
    for (std::uint32_t j = 0; j < count; ++j)
        if (children[j] >= t) throw std::invalid_argument("term children must precede their parent");
    id_.push_back(f);
    is_var_.push_back(0);
    kids_.insert(kids_.end(), children, children + count);
    first_.push_back(static_cast<std::uint32_t>(kids_.size()));
    return t;
}

void TermArena::reserve(std::size_t nodes, std::size_t edges) {
    id_.reserve(nodes);
    is_var_.reserve(nodes);
    first_.reserve(nodes + 1);
    kids_.reserve(edges);
}

bool is_ground(const TermArena& a, TermRef t) {
    std::vector<TermRef> stack{t};
    std::vector<std::uint8_t> seen;
    while (!stack.empty()) {
        TermRef x = stack.back();
        stack.pop_back();
        if (a.is_variable(x)) return false;
        if (seen.size() <= x) seen.resize(x + 1, 0);
        if (seen[x]) continue;
        seen[x] = 1;
        for (std::uint32_t j = 0; j < a.arity(x); ++j) stack.push_back(a.child(x, j));
    }
    return true;
}

bool term_equal(const TermArena& a, TermRef x, const TermArena& b, TermRef y) {
    std::vector<std::pair<TermRef, TermRef>> work{{x, y}};
    while (!work.empty()) {
        auto [p, q] = work.back();
        work.pop_back();
        if (&a == &b && p == q) continue;  // shared subterms unfold identically
        if (a.is_variable(p) != b.is_variable(q) || a.id(p) != b.id(q)) return false;
        if (a.is_variable(p)) continue;
        if (a.arity(p) != b.arity(q)) return false;
        for (std::uint32_t j = 0; j < a.arity(p); ++j) work.emplace_back(a.child(p, j), b.child(q, j));
    }
    return true;
}

std::string print_term(const Signature& sig, const TermArena& a, TermRef t) {
    std::string out;
    struct Frame {
        TermRef node;
        std::uint32_t next;
    };
    std::vector<Frame> stack{{t, 0}};
    while (!stack.empty()) {
        Frame& f = stack.back();
        if (f.next == 0) {
            if (a.is_variable(f.node)) {
                out += sig.variables[a.id(f.node)].name;
                stack.pop_back();
                continue;
            }
            out += sig.symbols[a.id(f.node)].name;
            out += '(';
        }
        if (f.next < a.arity(f.node)) {
            if (f.next > 0) out += ", ";
            TermRef c = a.child(f.node, f.next);
            ++f.next;
            stack.push_back({c, 0});
        } else {
            out += ')';
            stack.pop_back();
        }
    }
    return out;
}

}  // namespace trs_b200

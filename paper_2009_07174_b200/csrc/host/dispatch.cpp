// Rule compiler (counterpart of proj/src/dispatch.cpp): per-head match
// programs in source order, RHS build templates with structural sharing
// and in-template indegrees, the stable dump-dispatch text, and the
// flattening into the trs_gpu.h POD program the device stages in shared
// memory.
#include <algorithm>
#include <map>

#include "trs_host.hpp"

namespace trs_b200 {

namespace {

// Pre-order over the pattern; every child position yields one step
// (dispatch.cpp:10-26).  `parent` records the CheckHead step that reached
// the enclosing position, which lets the device walk each step from its
// parent's node instead of re-walking the path from the root.
void compile_pattern(const TermArena& a, TermRef lhs, MatchProgram& prog,
                     std::unordered_map<VarId, std::uint32_t>& var_slots) {
    struct Frame {
        TermRef node;
        std::uint32_t next;
        std::int32_t step;  // step index that reached `node` (-1: root)
    };
    std::vector<Frame> stack{{lhs, 0, -1}};
    std::vector<std::uint8_t> path;
    while (!stack.empty()) {
        Frame& f = stack.back();
        if (f.next >= a.arity(f.node)) {
            stack.pop_back();
            if (!path.empty()) path.pop_back();
            continue;
        }
        std::uint8_t j = static_cast<std::uint8_t>(f.next++);
        TermRef c = a.child(f.node, j);
        std::int32_t parent = f.step;
        path.push_back(j);
        MatchStep st;
        st.path = path;
        st.parent = parent;
        if (a.is_variable(c)) {
            std::uint32_t slot = static_cast<std::uint32_t>(prog.slot_vars.size());
            var_slots.emplace(a.id(c), slot);
            prog.slot_vars.push_back(a.id(c));
            st.kind = MatchStep::Kind::BindVar;
            st.var_slot = slot;
            prog.steps.push_back(st);
            path.pop_back();
        } else {
            st.kind = MatchStep::Kind::CheckHead;
            st.symbol = a.id(c);
            prog.steps.push_back(st);
            stack.push_back({c, 0, static_cast<std::int32_t>(prog.steps.size() - 1)});
        }
    }
}

// Post-order emission with structural memo (dispatch.cpp:28-49): identical
// RHS subterms become one instruction; children precede parents.
RhsTemplate compile_rhs(const TermArena& a, TermRef rhs, const std::unordered_map<VarId, std::uint32_t>& var_slots) {
    RhsTemplate tmpl;
    std::map<std::pair<SymbolId, std::vector<RhsRef>>, RhsRef> memo;
    struct Frame {
        TermRef node;
        std::uint32_t next;
        std::vector<RhsRef> kids;
    };
    std::vector<Frame> stack{{rhs, 0, {}}};
    RhsRef done{RhsRef::Kind::Var, 0};
    bool have = false;
    if (a.is_variable(rhs)) {
        tmpl.root_ref = {RhsRef::Kind::Var, var_slots.at(a.id(rhs))};
        return tmpl;
    }
    while (!stack.empty()) {
        Frame& f = stack.back();
        if (have) {
            f.kids.push_back(done);
            have = false;
        }
        if (f.next < a.arity(f.node)) {
            TermRef c = a.child(f.node, f.next++);
            if (a.is_variable(c)) {
                f.kids.push_back({RhsRef::Kind::Var, var_slots.at(a.id(c))});
            } else {
                stack.push_back({c, 0, {}});
            }
            continue;
        }
        auto key = std::make_pair(a.id(f.node), f.kids);
        auto it = memo.find(key);
        if (it != memo.end()) {
            done = it->second;
        } else {
            done = {RhsRef::Kind::Node, static_cast<std::uint32_t>(tmpl.instructions.size())};
            tmpl.instructions.push_back({a.id(f.node), f.kids, 0});
            memo.emplace(std::move(key), done);
        }
        stack.pop_back();
        have = true;
    }
    tmpl.root_ref = done;
    for (const RhsInstr& ins : tmpl.instructions)
        for (const RhsRef& r : ins.children)
            if (r.kind == RhsRef::Kind::Node) ++tmpl.instructions[r.index].indegree;
    return tmpl;
}

std::string path_text(const std::vector<std::uint8_t>& p) {
    std::string out = "[";
    for (std::size_t i = 0; i < p.size(); ++i) {
        if (i) out += ".";
        out += std::to_string(p[i]);
    }
    return out + "]";
}

}  // namespace

DispatchTable compile(const RewriteSystem& sys) {
    DispatchTable t;
    t.by_symbol.resize(sys.signature.symbols.size());
    for (const Rule& r : sys.rules) {
        CompiledRule c;
        c.rule_index = r.source_order;
        c.program.head = sys.terms.id(r.lhs);
        std::unordered_map<VarId, std::uint32_t> slots;
        compile_pattern(sys.terms, r.lhs, c.program, slots);
        c.rhs = compile_rhs(sys.terms, r.rhs, slots);
        t.max_new_slots = std::max(t.max_new_slots, c.rhs.new_slots());
        t.by_symbol[c.program.head].push_back(std::move(c));
    }
    return t;
}

std::string dump_dispatch(const RewriteSystem& sys, const DispatchTable& t) {
    const Signature& sig = sys.signature;
    auto ref_text = [&](const RhsRef& r, const MatchProgram& p) {
        return r.kind == RhsRef::Kind::Var ? sig.variables[p.slot_vars[r.index]].name : "n" + std::to_string(r.index);
    };
    std::string out;
    for (SymbolId f = 0; f < t.by_symbol.size(); ++f) {
        const auto& rules = t.by_symbol[f];
        if (rules.empty()) continue;
        out += "symbol " + sig.symbols[f].name + "/" + std::to_string(sig.symbols[f].arity) + ": " +
               std::to_string(rules.size()) + " rule(s)\n";
        for (const CompiledRule& c : rules) {
            const Rule& src = sys.rules[c.rule_index];
            out += "  rule #" + std::to_string(c.rule_index) + ": " + print_term(sig, sys.terms, src.lhs) + " = " +
                   print_term(sig, sys.terms, src.rhs) + "\n";
            for (const MatchStep& st : c.program.steps) {
                if (st.kind == MatchStep::Kind::CheckHead)
                    out += "    check " + path_text(st.path) + " = " + sig.symbols[st.symbol].name + "\n";
                else
                    out += "    bind  " + path_text(st.path) + " -> " +
                           sig.variables[c.program.slot_vars[st.var_slot]].name + "\n";
            }
            const RhsTemplate& tm = c.rhs;
            for (std::uint32_t k = 0; k < tm.instructions.size(); ++k) {
                const RhsInstr& ins = tm.instructions[k];
                bool root = !tm.collapses() && k + 1 == tm.instructions.size();
                out += root ? "    root  " : "    new   ";
                out += "n" + std::to_string(k) + " = " + sig.symbols[ins.symbol].name + "(";
                for (std::size_t i = 0; i < ins.children.size(); ++i) {
                    if (i) out += ", ";
                    out += ref_text(ins.children[i], c.program);
                }
                out += ")\n";
            }
            if (tm.collapses()) out += "    root  reuse " + ref_text(tm.root_ref, c.program) + "\n";
        }
    }
    return out;
}

FlatProgram flatten(const RewriteSystem& sys, const DispatchTable& t) {
    FlatProgram p;
    const std::uint32_t ns = static_cast<std::uint32_t>(sys.signature.symbols.size());
    for (const SymbolInfo& s : sys.signature.symbols) p.arity.push_back(s.arity);
    p.rule_begin.push_back(0);
    for (SymbolId f = 0; f < ns; ++f) {
        for (const CompiledRule& c : t.by_symbol[f]) {
            trs_gpu_rule r{};
            r.source_order = c.rule_index;
            r.first_step = static_cast<std::uint32_t>(p.steps.size());
            r.num_steps = static_cast<std::uint32_t>(c.program.steps.size());
            r.first_instr = static_cast<std::uint32_t>(p.instrs.size());
            r.num_instrs = static_cast<std::uint32_t>(c.rhs.instructions.size());
            r.num_vars = static_cast<std::uint32_t>(c.program.slot_vars.size());
            r.root_ref = c.rhs.collapses() ? c.rhs.root_ref.index : (TRS_GPU_REF_NODE | c.rhs.root_ref.index);
            for (const MatchStep& st : c.program.steps) {
                trs_gpu_step s{};
                s.kind = st.kind == MatchStep::Kind::CheckHead ? TRS_GPU_STEP_CHECK_HEAD : TRS_GPU_STEP_BIND_VAR;
                s.parent = st.parent;
                s.child = st.path.back();
                s.value = st.kind == MatchStep::Kind::CheckHead ? st.symbol : st.var_slot;
                p.steps.push_back(s);
            }
            for (const RhsInstr& ins : c.rhs.instructions) {
                trs_gpu_instr in{};
                in.symbol = ins.symbol;
                in.indegree = ins.indegree;
                in.first_ref = static_cast<std::uint32_t>(p.refs.size());
                for (const RhsRef& ref : ins.children)
                    p.refs.push_back(ref.kind == RhsRef::Kind::Node ? (TRS_GPU_REF_NODE | ref.index) : ref.index);
                p.instrs.push_back(in);
            }
            p.rules.push_back(r);
        }
        p.rule_begin.push_back(static_cast<std::uint32_t>(p.rules.size()));
    }
    return p;
}

trs_gpu_program FlatProgram::view() const {
    trs_gpu_program v{};
    v.num_symbols = static_cast<std::uint32_t>(arity.size());
    v.arity = arity.data();
    v.rule_begin = rule_begin.data();
    v.num_rules = static_cast<std::uint32_t>(rules.size());
    v.rules = rules.data();
    v.num_steps = static_cast<std::uint32_t>(steps.size());
    v.steps = steps.data();
    v.num_instrs = static_cast<std::uint32_t>(instrs.size());
    v.instrs = instrs.data();
    v.num_refs = static_cast<std::uint32_t>(refs.size());
    v.refs = refs.data();
    return v;
}

}  // namespace trs_b200

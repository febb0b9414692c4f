// .trs front end: lexer, parser, resolver (counterpart of proj/src/parser.cpp).
//
// Same language and diagnostics as the reference (sections `sort`, `var`,
// `eqn`, `input`/`Input`; optional `struct`; `%` line comments; constants
// written `Name()`, bare names are variables), but every stage is
// iterative: raw terms are flat post-order node arrays and resolution walks
// them with an explicit stack in the reference's pre-order, so the
// reference's resolver recursion (parser.cpp:443-491, which overflows an
// 8 MiB stack near 16k nesting) has no counterpart here.
#include <cctype>

#include "trs_host.hpp"

namespace trs_b200 {

const char* error_kind_name(ErrorKind kind) {
    switch (kind) {
        case ErrorKind::Lex: return "lex";
        case ErrorKind::Syntax: return "syntax";
        case ErrorKind::UnknownName: return "unknown-name";
        case ErrorKind::ArityMismatch: return "arity-mismatch";
        case ErrorKind::SortMismatch: return "sort-mismatch";
        case ErrorKind::RuleViolation: return "rule-violation";
        case ErrorKind::DuplicateName: return "duplicate-name";
    }
    return "error";
}

std::string format_error(std::string_view file, const ParseError& e) {
    return std::string(file) + ":" + std::to_string(e.span.line) + ":" + std::to_string(e.span.column) + ": " +
           error_kind_name(e.kind) + ": " + e.message;
}

namespace {

enum class Tok { Ident, LParen, RParen, Comma, Semi, Equals, Pipe, Colon, End };

struct Token {
    Tok kind = Tok::End;
    std::string_view text;
    SourceSpan span;
};

bool reserved(std::string_view w) {
    return w == "sort" || w == "var" || w == "eqn" || w == "input" || w == "Input" || w == "struct";
}

class Lexer {
public:
    Lexer(std::string_view src, std::vector<ParseError>& errors) : src_(src), errors_(errors) { next(); }
    const Token& peek() const { return tok_; }
    Token take() {
        Token t = tok_;
        next();
        return t;
    }

private:
    void bump() {
        if (src_[pos_] == '\n') {
            ++line_;
            col_ = 1;
        } else {
            ++col_;
        }
        ++pos_;
    }
    void next() {
        for (;;) {
            for (;;) {
                while (pos_ < src_.size() && (src_[pos_] == ' ' || src_[pos_] == '\t' || src_[pos_] == '\r' || src_[pos_] == '\n'))
                    bump();
                if (pos_ < src_.size() && src_[pos_] == '%') {
                    while (pos_ < src_.size() && src_[pos_] != '\n') bump();
                    continue;
                }
                break;
            }
            tok_.span = {line_, col_, 1};
            if (pos_ >= src_.size()) {
                tok_.kind = Tok::End;
                tok_.text = {};
                return;
            }
            const char c = src_[pos_];
            Tok k;
            switch (c) {
                case '(': k = Tok::LParen; break;
                case ')': k = Tok::RParen; break;
                case ',': k = Tok::Comma; break;
                case ';': k = Tok::Semi; break;
                case '=': k = Tok::Equals; break;
                case '|': k = Tok::Pipe; break;
                case ':': k = Tok::Colon; break;
                default:
                    if (std::isalpha(static_cast<unsigned char>(c))) {
                        std::size_t start = pos_;
                        while (pos_ < src_.size() && (std::isalnum(static_cast<unsigned char>(src_[pos_])) || src_[pos_] == '_'))
                            bump();
                        tok_.kind = Tok::Ident;
                        tok_.text = src_.substr(start, pos_ - start);
                        tok_.span.length = static_cast<std::uint32_t>(pos_ - start);
                        return;
                    }
                    errors_.push_back({tok_.span, ErrorKind::Lex, std::string("unexpected character '") + c + "'"});
                    bump();
                    continue;  // resynchronise on the next token
            }
            tok_.kind = k;
            tok_.text = src_.substr(pos_, 1);
            bump();
            return;
        }
    }

    std::string_view src_;
    std::vector<ParseError>& errors_;
    std::size_t pos_ = 0;
    std::uint32_t line_ = 1, col_ = 1;
    Token tok_;
};

// Raw (unresolved) term: flat nodes in post-order; kids index into `kids`.
struct RawNode {
    std::string_view name;
    bool has_args = false;
    SourceSpan span;
    std::uint32_t first = 0, count = 0;
};

struct RawTerm {
    std::vector<RawNode> nodes;
    std::vector<std::uint32_t> kids;
    std::uint32_t root = 0;
    const RawNode& at(std::uint32_t k) const { return nodes[k]; }
    std::uint32_t child(std::uint32_t k, std::uint32_t j) const { return kids[nodes[k].first + j]; }
};

struct RawCtor {
    std::string name;
    SourceSpan span;
    std::vector<std::pair<std::string, SourceSpan>> arg_sorts;
};

struct RawSort {
    std::string name;
    SourceSpan span;
    std::vector<RawCtor> ctors;
};

struct RawVar {
    std::string name, sort;
    SourceSpan span, sort_span;
};

struct RawEqn {
    RawTerm lhs, rhs;
};

struct RawSpec {
    std::vector<RawSort> sorts;
    std::vector<RawVar> vars;
    std::vector<RawEqn> eqns;
    RawTerm input;
};

class Parser {
public:
    Parser(std::string_view text, std::vector<ParseError>& errors) : errors_(errors), lex_(text, errors) {}

    std::optional<RawSpec> run() {
        RawSpec spec;
        if (!section("sort")) return std::nullopt;
        sorts(spec);
        if (!section("var")) return std::nullopt;
        vars(spec);
        if (!section("eqn")) return std::nullopt;
        eqns(spec);
        if (!at("input") && !at("Input")) {
            error(lex_.peek().span, ErrorKind::Syntax, "missing required sections: expected 'input'");
            return std::nullopt;
        }
        lex_.take();
        term(spec.input);
        expect(Tok::Semi, "';'");
        if (lex_.peek().kind != Tok::End)
            error(lex_.peek().span, ErrorKind::Syntax, "trailing input after 'input' section");
        if (!errors_.empty()) return std::nullopt;
        return spec;
    }

private:
    bool at(std::string_view w) const { return lex_.peek().kind == Tok::Ident && lex_.peek().text == w; }
    bool at_name() const { return lex_.peek().kind == Tok::Ident && !reserved(lex_.peek().text); }
    void error(SourceSpan s, ErrorKind k, std::string m) { errors_.push_back({s, k, std::move(m)}); }
    std::string context() const {
        const Token& t = lex_.peek();
        return t.kind == Tok::End ? " before end of input" : " before '" + std::string(t.text) + "'";
    }
    bool section(std::string_view kw) {
        if (at(kw)) {
            lex_.take();
            return true;
        }
        error(lex_.peek().span, ErrorKind::Syntax, "missing required sections: expected '" + std::string(kw) + "'");
        return false;
    }
    bool expect(Tok k, const char* what) {
        if (lex_.peek().kind == k) {
            lex_.take();
            return true;
        }
        error(lex_.peek().span, ErrorKind::Syntax, std::string("expected ") + what + context());
        return false;
    }
    void skip_statement() {
        for (;;) {
            const Token& t = lex_.peek();
            if (t.kind == Tok::End) return;
            if (t.kind == Tok::Semi) {
                lex_.take();
                return;
            }
            if (t.kind == Tok::Ident && reserved(t.text)) return;
            lex_.take();
        }
    }

    void sorts(RawSpec& spec) {
        while (at_name()) {
            RawSort decl;
            Token name = lex_.take();
            decl.name = std::string(name.text);
            decl.span = name.span;
            if (!expect(Tok::Equals, "'='")) {
                skip_statement();
                continue;
            }
            if (at("struct")) lex_.take();
            bool ok = true;
            for (;;) {
                if (!at_name()) {
                    error(lex_.peek().span, ErrorKind::Syntax, "expected constructor name" + context());
                    ok = false;
                    break;
                }
                RawCtor ctor;
                Token cn = lex_.take();
                ctor.name = std::string(cn.text);
                ctor.span = cn.span;
                if (!expect(Tok::LParen, "'(' (constants are written with explicit '()')")) {
                    ok = false;
                    break;
                }
                bool arg_ok = true;
                if (lex_.peek().kind != Tok::RParen) {
                    for (;;) {
                        if (lex_.peek().kind != Tok::Ident) {
                            error(lex_.peek().span, ErrorKind::Syntax, "expected sort name" + context());
                            arg_ok = false;
                            break;
                        }
                        Token s = lex_.take();
                        ctor.arg_sorts.emplace_back(std::string(s.text), s.span);
                        if (lex_.peek().kind == Tok::Comma) {
                            lex_.take();
                            continue;
                        }
                        break;
                    }
                }
                if (!arg_ok || !expect(Tok::RParen, "')'")) {
                    ok = false;
                    break;
                }
                decl.ctors.push_back(std::move(ctor));
                if (lex_.peek().kind == Tok::Pipe) {
                    lex_.take();
                    continue;
                }
                break;
            }
            if (!ok || !expect(Tok::Semi, "';'")) {
                skip_statement();
                continue;
            }
            spec.sorts.push_back(std::move(decl));
        }
    }

    void vars(RawSpec& spec) {
        while (at_name()) {
            RawVar v;
            Token name = lex_.take();
            v.name = std::string(name.text);
            v.span = name.span;
            if (!expect(Tok::Colon, "':'")) {
                skip_statement();
                continue;
            }
            if (lex_.peek().kind != Tok::Ident) {
                error(lex_.peek().span, ErrorKind::Syntax, "expected sort name" + context());
                skip_statement();
                continue;
            }
            Token s = lex_.take();
            v.sort = std::string(s.text);
            v.sort_span = s.span;
            if (!expect(Tok::Semi, "';'")) {
                skip_statement();
                continue;
            }
            spec.vars.push_back(std::move(v));
        }
    }

    void eqns(RawSpec& spec) {
        while (at_name()) {
            RawEqn e;
            if (!term(e.lhs)) {
                skip_statement();
                continue;
            }
            if (!expect(Tok::Equals, "'='")) {
                skip_statement();
                continue;
            }
            if (!term(e.rhs)) {
                skip_statement();
                continue;
            }
            if (!expect(Tok::Semi, "';'")) {
                skip_statement();
                continue;
            }
            spec.eqns.push_back(std::move(e));
        }
    }

    // IDENT [ '(' term (',' term)* ')' ] with an explicit frame stack.
    bool term(RawTerm& out) {
        struct Open {
            std::string_view name;
            SourceSpan span;
            std::vector<std::uint32_t> kids;
        };
        std::vector<Open> open;
        auto finish = [&](std::string_view name, bool has_args, SourceSpan span, const std::vector<std::uint32_t>& kids) {
            RawNode n;
            n.name = name;
            n.has_args = has_args;
            n.span = span;
            n.first = static_cast<std::uint32_t>(out.kids.size());
            n.count = static_cast<std::uint32_t>(kids.size());
            out.kids.insert(out.kids.end(), kids.begin(), kids.end());
            out.nodes.push_back(n);
            return static_cast<std::uint32_t>(out.nodes.size() - 1);
        };
        static const std::vector<std::uint32_t> none;
        for (;;) {
            if (!at_name()) {
                error(lex_.peek().span, ErrorKind::Syntax, "expected a term" + context());
                return false;
            }
            Token name = lex_.take();
            std::uint32_t node;
            if (lex_.peek().kind == Tok::LParen) {
                lex_.take();
                if (lex_.peek().kind != Tok::RParen) {
                    open.push_back({name.text, name.span, {}});
                    continue;
                }
                lex_.take();
                node = finish(name.text, true, name.span, none);
            } else {
                node = finish(name.text, false, name.span, none);
            }
            for (;;) {
                if (open.empty()) {
                    out.root = node;
                    return true;
                }
                open.back().kids.push_back(node);
                if (lex_.peek().kind == Tok::Comma) {
                    lex_.take();
                    break;
                }
                if (lex_.peek().kind == Tok::RParen) {
                    lex_.take();
                    Open f = std::move(open.back());
                    open.pop_back();
                    node = finish(f.name, true, f.span, f.kids);
                    continue;
                }
                error(lex_.peek().span, ErrorKind::Syntax, "expected ',' or ')' in argument list" + context());
                return false;
            }
        }
    }

    std::vector<ParseError>& errors_;
    Lexer lex_;
};

class Resolver {
public:
    explicit Resolver(const RawSpec& spec) : spec_(spec) {}

    ResolveResult run() {
        for (const RawSort& d : spec_.sorts) {
            if (sig().sort_ids.count(d.name)) {
                error(d.span, ErrorKind::DuplicateName, "duplicate sort '" + d.name + "'");
                continue;
            }
            sig().add_sort(d.name);
        }
        for (const RawSort& d : spec_.sorts) {
            auto sit = sig().sort_ids.find(d.name);
            if (sit == sig().sort_ids.end()) continue;
            for (const RawCtor& c : d.ctors) {
                if (sig().symbol_ids.count(c.name)) {
                    error(c.span, ErrorKind::DuplicateName, "duplicate function symbol '" + c.name + "'");
                    continue;
                }
                std::vector<SortId> as;
                bool ok = true;
                for (const auto& [sn, sp] : c.arg_sorts) {
                    auto it = sig().sort_ids.find(sn);
                    if (it == sig().sort_ids.end()) {
                        error(sp, ErrorKind::UnknownName, "unknown sort '" + sn + "'");
                        ok = false;
                        continue;
                    }
                    as.push_back(it->second);
                }
                if (ok) sig().add_symbol(c.name, sit->second, std::move(as));
            }
        }
        for (const RawVar& v : spec_.vars) {
            if (sig().symbol_ids.count(v.name)) {
                error(v.span, ErrorKind::DuplicateName, "variable '" + v.name + "' collides with a function symbol");
                continue;
            }
            if (sig().variable_ids.count(v.name)) {
                error(v.span, ErrorKind::DuplicateName, "duplicate variable '" + v.name + "'");
                continue;
            }
            auto it = sig().sort_ids.find(v.sort);
            if (it == sig().sort_ids.end()) {
                error(v.sort_span, ErrorKind::UnknownName, "unknown sort '" + v.sort + "'");
                continue;
            }
            sig().add_variable(v.name, it->second);
        }
        sys_.rules_by_head.assign(sig().symbols.size(), {});
        for (const RawEqn& e : spec_.eqns) {
            std::optional<TermRef> lhs = resolve(e.lhs, std::nullopt);
            if (!lhs) continue;
            SortId ls = sys_.terms.is_variable(*lhs) ? sig().variables[sys_.terms.id(*lhs)].sort
                                                      : sig().symbols[sys_.terms.id(*lhs)].sort;
            std::optional<TermRef> rhs = resolve(e.rhs, ls);
            if (!rhs) continue;
            if (!validate(e)) continue;
            std::uint32_t index = static_cast<std::uint32_t>(sys_.rules.size());
            sys_.rules.push_back({*lhs, *rhs, index});
            sys_.rules_by_head[sys_.terms.id(*lhs)].push_back(index);
        }
        if (std::optional<TermRef> in = resolve(spec_.input, std::nullopt)) {
            if (!is_ground(sys_.terms, *in))
                error(spec_.input.at(spec_.input.root).span, ErrorKind::RuleViolation,
                      "input term must be ground (derivations need closed terms)");
            else
                sys_.input_term = *in;
        }
        ResolveResult r;
        r.errors = std::move(errors_);
        if (r.errors.empty()) r.system = std::move(sys_);
        return r;
    }

private:
    Signature& sig() { return sys_.signature; }
    void error(SourceSpan s, ErrorKind k, std::string m) { errors_.push_back({s, k, std::move(m)}); }

    // Pre-order resolution with an explicit stack; checks happen on entry in
    // the reference's order (variable, unknown symbol, arity, sort), and a
    // failed child fails its parent without further diagnostics.
    std::optional<TermRef> resolve(const RawTerm& raw, std::optional<SortId> expected) {
        struct Frame {
            std::uint32_t node;
            SymbolId symbol;
            std::uint32_t next;
            bool ok;
            std::vector<TermRef> kids;
        };
        std::vector<Frame> stack;
        std::optional<TermRef> result;
        bool have_result = false;
        // enter returns true when a frame was pushed; otherwise result is set
        auto enter = [&](std::uint32_t k, std::optional<SortId> exp) -> bool {
            const RawNode& n = raw.at(k);
            std::string name(n.name);
            if (!n.has_args) {
                auto it = sig().variable_ids.find(name);
                if (it == sig().variable_ids.end()) {
                    if (sig().symbol_ids.count(name))
                        error(n.span, ErrorKind::UnknownName,
                              "unknown variable '" + name + "' (a constant must be written with parentheses: '" + name + "()')");
                    else
                        error(n.span, ErrorKind::UnknownName, "unknown variable '" + name + "'");
                    result.reset();
                    return false;
                }
                SortId s = sig().variables[it->second].sort;
                if (exp && *exp != s) {
                    error(n.span, ErrorKind::SortMismatch,
                          "variable '" + name + "' has sort " + sig().sorts[s] + ", expected " + sig().sorts[*exp]);
                    result.reset();
                    return false;
                }
                result = sys_.terms.variable(it->second);
                return false;
            }
            auto it = sig().symbol_ids.find(name);
            if (it == sig().symbol_ids.end()) {
                error(n.span, ErrorKind::UnknownName, "unknown function symbol '" + name + "'");
                result.reset();
                return false;
            }
            const SymbolInfo& info = sig().symbols[it->second];
            if (n.count != info.arity) {
                error(n.span, ErrorKind::ArityMismatch,
                      "'" + name + "' takes " + std::to_string(info.arity) + " argument(s), got " + std::to_string(n.count));
                result.reset();
                return false;
            }
            if (exp && *exp != info.sort) {
                error(n.span, ErrorKind::SortMismatch,
                      "'" + name + "' has sort " + sig().sorts[info.sort] + ", expected " + sig().sorts[*exp]);
                result.reset();
                return false;
            }
            stack.push_back({k, it->second, 0, true, {}});
            stack.back().kids.reserve(info.arity);
            return true;
        };
        if (!enter(raw.root, expected)) return result;
        for (;;) {
            Frame& f = stack.back();
            if (have_result) {
                have_result = false;
                if (result)
                    f.kids.push_back(*result);
                else
                    f.ok = false;
            }
            const RawNode& n = raw.at(f.node);
            if (f.next < n.count) {
                std::uint32_t c = raw.child(f.node, f.next);
                SortId exp = sig().symbols[f.symbol].argument_sorts[f.next];
                ++f.next;
                if (!enter(c, exp)) have_result = true;
                continue;
            }
            if (f.ok)
                result = sys_.terms.apply(f.symbol, f.kids.data(), static_cast<std::uint32_t>(f.kids.size()));
            else
                result.reset();
            stack.pop_back();
            if (stack.empty()) return result;
            have_result = true;
        }
    }

    // validate_rule (term.cpp:167-179) on the raw trees, which mirror the
    // resolved terms node for node; diagnostics at the offending occurrence.
    bool validate(const RawEqn& e) {
        const RawNode& lroot = e.lhs.at(e.lhs.root);
        if (!lroot.has_args) {
            error(lroot.span, ErrorKind::RuleViolation, "left-hand side of a rule must not be a variable");
            return false;
        }
        bool ok = true;
        std::unordered_map<std::string_view, int> seen;
        std::vector<std::uint32_t> stack{e.lhs.root};
        while (!stack.empty()) {
            std::uint32_t k = stack.back();
            stack.pop_back();
            const RawNode& n = e.lhs.at(k);
            if (!n.has_args) {
                if (seen[n.name]++) {
                    error(n.span, ErrorKind::RuleViolation,
                          "variable '" + std::string(n.name) + "' occurs more than once in the left-hand side");
                    ok = false;
                }
                continue;
            }
            for (std::uint32_t j = n.count; j-- > 0;) stack.push_back(e.lhs.child(k, j));
        }
        stack.assign(1, e.rhs.root);
        while (!stack.empty()) {
            std::uint32_t k = stack.back();
            stack.pop_back();
            const RawNode& n = e.rhs.at(k);
            if (!n.has_args) {
                if (!seen.count(n.name)) {
                    error(n.span, ErrorKind::RuleViolation,
                          "variable '" + std::string(n.name) + "' of the right-hand side does not occur in the left-hand side");
                    ok = false;
                }
                continue;
            }
            for (std::uint32_t j = n.count; j-- > 0;) stack.push_back(e.rhs.child(k, j));
        }
        return ok;
    }

    const RawSpec& spec_;
    RewriteSystem sys_;
    std::vector<ParseError> errors_;
};

}  // namespace

ResolveResult load_system(std::string_view text) {
    std::vector<ParseError> errors;
    Parser parser(text, errors);
    std::optional<RawSpec> spec = parser.run();
    if (!spec || !errors.empty()) {
        ResolveResult r;
        r.errors = std::move(errors);
        return r;
    }
    return Resolver(*spec).run();
}

}  // namespace trs_b200

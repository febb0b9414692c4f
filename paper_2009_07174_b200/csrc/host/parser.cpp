// .trs front end: scanner, statement parser, resolver -- the language of
// proj/src/parser.cpp (sections `sort`, `var`, `eqn`, `input`/`Input`;
// optional `struct`; `%` line comments; constants written `Name()`, bare
// names are variables) with the same located diagnostics, word for word
// (tests/test_host.py checks them against the reference, including 600
// mutated systems).  The design is this file's own: the text is scanned in
// one pass into a token array through a character-class table, sections are
// driven by a table of statement parsers over token indices, raw terms are
// flat post-order node arrays, and resolution walks them with an explicit
// stack in the reference's pre-order -- nothing recurses, so the reference
// resolver's stack overflow near 16k nesting (parser.cpp:443-491, SURVEY.md
// §8c) has no counterpart here.
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

// ---- scanner ---------------------------------------------------------------
// The whole text is scanned up front into a token array (the parser then
// works on index ranges of it).  Characters are classified by one table;
// anything that is neither blank, `%` comment, punctuation nor a letter is
// a lex error that is reported and skipped.

enum class Tok : std::uint8_t { Ident, LParen, RParen, Comma, Semi, Equals, Pipe, Colon, End };

struct Token {
    Tok kind = Tok::End;
    std::string_view text;
    SourceSpan span;
};

enum CharClass : std::uint8_t { kBad, kBlank, kNewline, kComment, kAlpha, kDigit, kUnder, kPunct };

struct CharTable {
    CharClass cls[256];
    Tok punct[256];
    CharTable() {
        for (int c = 0; c < 256; ++c) {
            cls[c] = kBad;
            punct[c] = Tok::End;
            if (std::isalpha(c)) cls[c] = kAlpha;
            if (std::isdigit(c)) cls[c] = kDigit;
        }
        cls[(unsigned char)' '] = cls[(unsigned char)'\t'] = cls[(unsigned char)'\r'] = kBlank;
        cls[(unsigned char)'\n'] = kNewline;
        cls[(unsigned char)'%'] = kComment;
        cls[(unsigned char)'_'] = kUnder;
        const std::pair<char, Tok> p[] = {{'(', Tok::LParen}, {')', Tok::RParen}, {',', Tok::Comma}, {';', Tok::Semi},
                                          {'=', Tok::Equals}, {'|', Tok::Pipe},   {':', Tok::Colon}};
        for (auto [c, t] : p) {
            cls[(unsigned char)c] = kPunct;
            punct[(unsigned char)c] = t;
        }
    }
};

const CharTable& char_table() {
    static const CharTable t;
    return t;
}

// Section keywords (and `struct`) are not names.
bool reserved(std::string_view w) {
    static const std::string_view kw[] = {"sort", "var", "eqn", "input", "Input", "struct"};
    for (std::string_view k : kw)
        if (w == k) return true;
    return false;
}

std::vector<Token> scan(std::string_view src, std::vector<ParseError>& errors) {
    const CharTable& T = char_table();
    std::vector<Token> out;
    std::uint32_t line = 1, col = 1;
    std::size_t i = 0;
    auto advance = [&](std::size_t n) {
        for (std::size_t k = 0; k < n; ++k, ++i) {
            if (src[i] == '\n') {
                ++line;
                col = 1;
            } else {
                ++col;
            }
        }
    };
    while (i < src.size()) {
        const unsigned char c = static_cast<unsigned char>(src[i]);
        switch (T.cls[c]) {
            case kBlank:
            case kNewline: advance(1); break;
            case kComment: {
                std::size_t e = src.find('\n', i);
                advance((e == std::string_view::npos ? src.size() : e) - i);
                break;
            }
            case kPunct:
                out.push_back({T.punct[c], src.substr(i, 1), {line, col, 1}});
                advance(1);
                break;
            case kAlpha: {
                std::size_t e = i + 1;
                while (e < src.size()) {
                    const CharClass k = T.cls[static_cast<unsigned char>(src[e])];
                    if (k != kAlpha && k != kDigit && k != kUnder) break;
                    ++e;
                }
                out.push_back({Tok::Ident, src.substr(i, e - i), {line, col, static_cast<std::uint32_t>(e - i)}});
                advance(e - i);
                break;
            }
            default:
                errors.push_back({{line, col, 1}, ErrorKind::Lex, std::string("unexpected character '") + src[i] + "'"});
                advance(1);
                break;
        }
    }
    out.push_back({Tok::End, {}, {line, col, 1}});
    return out;
}

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

// ---- statement parser ------------------------------------------------------
// Grammar (the reference's language; proj/src/parser.cpp):
//   file   := 'sort' sortdecl* 'var' vardecl* 'eqn' eqn* ('input'|'Input') term ';'
//   sortdecl := NAME '=' ['struct'] ctor ('|' ctor)* ';'
//   ctor   := NAME '(' [NAME (',' NAME)*] ')'
//   vardecl := NAME ':' NAME ';'
//   eqn    := term '=' term ';'
//   term   := NAME ['(' [term (',' term)*] ')']
// A statement with an error is reported once, at the first offending
// token, and dropped: parsing resumes after the next ';' or at the next
// keyword (the statement cannot extend past either), and its section goes on
// with the next statement.  A section runs while the next statement starts
// with a name.  Diagnostics are the reference's, word for word
// (tests/test_host.py compares them with parser.cpp's).

class StatementParser {
public:
    StatementParser(std::string_view text, std::vector<ParseError>& errors)
        : toks_(scan(text, errors)), errors_(errors) {}

    std::optional<RawSpec> run() {
        RawSpec spec;
        using Stmt = bool (StatementParser::*)(RawSpec&);
        const std::pair<std::string_view, Stmt> sections[] = {
            {"sort", &StatementParser::sort_decl}, {"var", &StatementParser::var_decl}, {"eqn", &StatementParser::eqn}};
        for (const auto& [keyword, stmt] : sections) {
            if (!keyword_at(pos_, keyword)) return missing(keyword);
            ++pos_;
            while (name_at(pos_))
                if (!(this->*stmt)(spec)) resync();
        }
        if (!keyword_at(pos_, "input") && !keyword_at(pos_, "Input")) return missing("input");
        ++pos_;
        term(spec.input);
        expect(Tok::Semi, "';'");
        if (toks_[pos_].kind != Tok::End)
            report(toks_[pos_].span, ErrorKind::Syntax, "trailing input after 'input' section");
        if (!errors_.empty()) return std::nullopt;
        return spec;
    }

private:
    // after an error: past the statement's ';', or up to a keyword or the end
    void resync() {
        for (; toks_[pos_].kind != Tok::End; ++pos_) {
            if (toks_[pos_].kind == Tok::Semi) {
                ++pos_;
                return;
            }
            if (toks_[pos_].kind == Tok::Ident && reserved(toks_[pos_].text)) return;
        }
    }
    bool keyword_at(std::size_t i, std::string_view w) const {
        return toks_[i].kind == Tok::Ident && toks_[i].text == w;
    }
    bool name_at(std::size_t i) const { return toks_[i].kind == Tok::Ident && !reserved(toks_[i].text); }
    std::optional<RawSpec> missing(std::string_view keyword) {
        report(toks_[pos_].span, ErrorKind::Syntax, "missing required sections: expected '" + std::string(keyword) + "'");
        return std::nullopt;
    }
    void report(SourceSpan at, ErrorKind kind, std::string message) {
        errors_.push_back({at, kind, std::move(message)});
    }
    // an error at the current token, with the reference's " before ..." tail
    bool fail(std::string what) {
        const Token& t = toks_[pos_];
        report(t.span, ErrorKind::Syntax,
               what + (t.kind == Tok::End ? " before end of input" : " before '" + std::string(t.text) + "'"));
        return false;
    }
    bool expect(Tok k, const char* what) {
        if (toks_[pos_].kind == k) {
            ++pos_;
            return true;
        }
        return fail(std::string("expected ") + what);
    }
    bool accept(Tok k) {
        if (toks_[pos_].kind != k) return false;
        ++pos_;
        return true;
    }

    bool sort_decl(RawSpec& spec) {
        RawSort decl;
        decl.name = std::string(toks_[pos_].text);
        decl.span = toks_[pos_++].span;
        if (!expect(Tok::Equals, "'='")) return false;
        if (keyword_at(pos_, "struct")) ++pos_;
        do {
            if (!name_at(pos_)) return fail("expected constructor name");
            RawCtor ctor;
            ctor.name = std::string(toks_[pos_].text);
            ctor.span = toks_[pos_++].span;
            if (!expect(Tok::LParen, "'(' (constants are written with explicit '()')")) return false;
            if (toks_[pos_].kind != Tok::RParen) {
                do {
                    if (toks_[pos_].kind != Tok::Ident) return fail("expected sort name");
                    ctor.arg_sorts.emplace_back(std::string(toks_[pos_].text), toks_[pos_].span);
                    ++pos_;
                } while (accept(Tok::Comma));
            }
            if (!expect(Tok::RParen, "')'")) return false;
            decl.ctors.push_back(std::move(ctor));
        } while (accept(Tok::Pipe));
        if (!expect(Tok::Semi, "';'")) return false;
        spec.sorts.push_back(std::move(decl));
        return true;
    }

    bool var_decl(RawSpec& spec) {
        RawVar v;
        v.name = std::string(toks_[pos_].text);
        v.span = toks_[pos_++].span;
        if (!expect(Tok::Colon, "':'")) return false;
        if (toks_[pos_].kind != Tok::Ident) return fail("expected sort name");
        v.sort = std::string(toks_[pos_].text);
        v.sort_span = toks_[pos_++].span;
        if (!expect(Tok::Semi, "';'")) return false;
        spec.vars.push_back(std::move(v));
        return true;
    }

    bool eqn(RawSpec& spec) {
        RawEqn e;
        if (!term(e.lhs) || !expect(Tok::Equals, "'='") || !term(e.rhs) || !expect(Tok::Semi, "';'")) return false;
        spec.eqns.push_back(std::move(e));
        return true;
    }

    // term := NAME ['(' [term (',' term)*] ')'], with an explicit frame stack
    // (terms nest as deep as the input); nodes are emitted in post-order.
    bool term(RawTerm& out) {
        struct Frame {
            std::uint32_t tok;               // the applied name
            std::vector<std::uint32_t> kids;
        };
        std::vector<Frame> frames;
        auto emit = [&](std::uint32_t tok, bool has_args, const std::vector<std::uint32_t>& kids) {
            RawNode n;
            n.name = toks_[tok].text;
            n.has_args = has_args;
            n.span = toks_[tok].span;
            n.first = static_cast<std::uint32_t>(out.kids.size());
            n.count = static_cast<std::uint32_t>(kids.size());
            out.kids.insert(out.kids.end(), kids.begin(), kids.end());
            out.nodes.push_back(n);
            return static_cast<std::uint32_t>(out.nodes.size() - 1);
        };
        for (;;) {
            // an operand: a name, a constant `Name()`, or the opening of an application
            if (!name_at(pos_)) return fail("expected a term");
            const std::uint32_t tok = static_cast<std::uint32_t>(pos_++);
            std::uint32_t node;
            if (accept(Tok::LParen)) {
                if (!accept(Tok::RParen)) {
                    frames.push_back({tok, {}});
                    continue;
                }
                node = emit(tok, true, {});
            } else {
                node = emit(tok, false, {});
            }
            // close the applications this operand completes
            for (;;) {
                if (frames.empty()) {
                    out.root = node;
                    return true;
                }
                frames.back().kids.push_back(node);
                if (accept(Tok::Comma)) break;
                if (!accept(Tok::RParen)) return fail("expected ',' or ')' in argument list");
                node = emit(frames.back().tok, true, frames.back().kids);
                frames.pop_back();
            }
        }
    }

    std::vector<Token> toks_;
    std::vector<ParseError>& errors_;
    std::size_t pos_ = 0;
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
    StatementParser parser(text, errors);
    std::optional<RawSpec> spec = parser.run();
    if (!spec || !errors.empty()) {
        ResolveResult r;
        r.errors = std::move(errors);
        return r;
    }
    return Resolver(*spec).run();
}

}  // namespace trs_b200

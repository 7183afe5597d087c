// OpenQASM 2.0 frontend (behaviour of proj/src/qasm.cpp as
// documented in proj/include/naqs/qasm.hpp and pinned by
// proj/tests/test_qasm.cpp + the conformance corpus).
//
// A hand-written recursive-descent parser over an on-demand tokenizer: every
// token carries its 1-based line and column, and every failure (including
// circuit validation, e.g. a unitary after a terminal measurement) surfaces
// as a positioned QasmParseError.
#include "naqs/qasm.hpp"

#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace naqs {

namespace {

enum class Tok { Id, Num, Str, Sym, End };

struct Token {
    Tok kind = Tok::End;
    std::string text;  // identifier / string contents / symbol
    double value = 0.0;
    bool integral = false;
    int line = 1, col = 1;
};

class Lexer {
  public:
    explicit Lexer(const std::string& src) : s_(src) {}

    const Token& peek() {
        if (!have_) {
            tok_ = scan();
            have_ = true;
        }
        return tok_;
    }
    Token next() {
        peek();
        have_ = false;
        return tok_;
    }

  private:
    char at(size_t k) const { return k < s_.size() ? s_[k] : '\0'; }
    void advance() {
        if (at(i_) == '\n') {
            ++line_;
            col_ = 1;
        } else {
            ++col_;
        }
        ++i_;
    }

    Token scan() {
        for (;;) {  // whitespace and // comments
            const char c = at(i_);
            if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
                advance();
            } else if (c == '/' && at(i_ + 1) == '/') {
                while (i_ < s_.size() && at(i_) != '\n') advance();
            } else {
                break;
            }
        }
        Token t;
        t.line = line_;
        t.col = col_;
        if (i_ >= s_.size()) return t;
        const char c = at(i_);
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            t.kind = Tok::Id;
            while (std::isalnum(static_cast<unsigned char>(at(i_))) || at(i_) == '_') {
                t.text += at(i_);
                advance();
            }
            return t;
        }
        if (std::isdigit(static_cast<unsigned char>(c)) || (c == '.' && std::isdigit(static_cast<unsigned char>(at(i_ + 1))))) {
            std::string num;
            bool integral = true;
            while (std::isdigit(static_cast<unsigned char>(at(i_)))) {
                num += at(i_);
                advance();
            }
            if (at(i_) == '.') {
                integral = false;
                num += '.';
                advance();
                while (std::isdigit(static_cast<unsigned char>(at(i_)))) {
                    num += at(i_);
                    advance();
                }
            }
            if (at(i_) == 'e' || at(i_) == 'E') {
                const char n1 = at(i_ + 1), n2 = at(i_ + 2);
                if (std::isdigit(static_cast<unsigned char>(n1)) ||
                    ((n1 == '+' || n1 == '-') && std::isdigit(static_cast<unsigned char>(n2)))) {
                    integral = false;
                    num += 'e';
                    advance();
                    if (at(i_) == '+' || at(i_) == '-') {
                        num += at(i_);
                        advance();
                    }
                    while (std::isdigit(static_cast<unsigned char>(at(i_)))) {
                        num += at(i_);
                        advance();
                    }
                }
            }
            t.kind = Tok::Num;
            t.text = num;
            t.value = std::strtod(num.c_str(), nullptr);
            t.integral = integral;
            return t;
        }
        if (c == '"') {
            advance();
            while (i_ < s_.size() && at(i_) != '"' && at(i_) != '\n') {
                t.text += at(i_);
                advance();
            }
            if (at(i_) != '"') throw QasmParseError(t.line, t.col, "unterminated string");
            advance();
            t.kind = Tok::Str;
            return t;
        }
        if (c == '-' && at(i_ + 1) == '>') {
            advance();
            advance();
            t.kind = Tok::Sym;
            t.text = "->";
            return t;
        }
        if (c == '=' && at(i_ + 1) == '=') {
            advance();
            advance();
            t.kind = Tok::Sym;
            t.text = "==";
            return t;
        }
        static const std::string syms = ";,()[]{}+-*/^=";
        if (syms.find(c) != std::string::npos) {
            advance();
            t.kind = Tok::Sym;
            t.text = std::string(1, c);
            return t;
        }
        throw QasmParseError(t.line, t.col, std::string("unexpected character '") + c + "'");
    }

    const std::string& s_;
    size_t i_ = 0;
    int line_ = 1, col_ = 1;
    Token tok_;
    bool have_ = false;
};

// the qelib1 gates of the supported subset
const std::map<std::string, GateKind>& gate_table() {
    static const std::map<std::string, GateKind> t = {
        {"id", GateKind::ID},   {"x", GateKind::X},     {"y", GateKind::Y},     {"z", GateKind::Z},
        {"h", GateKind::H},     {"s", GateKind::S},     {"sdg", GateKind::SDG}, {"t", GateKind::T},
        {"tdg", GateKind::TDG}, {"rx", GateKind::RX},   {"ry", GateKind::RY},   {"rz", GateKind::RZ},
        {"u1", GateKind::U1},   {"u2", GateKind::U2},   {"u3", GateKind::U3},   {"cx", GateKind::CX},
        {"cz", GateKind::CZ},   {"swap", GateKind::SWAP}, {"ccx", GateKind::CCX},
    };
    return t;
}

struct Reg {
    int offset = 0;
    int size = 0;
};

// one operand: a whole register, or one element of it
struct Arg {
    const Reg* reg = nullptr;
    int index = -1;  // -1: whole register
    int line = 1, col = 1;
};

struct PendingOp {
    GateOp op;
    int line, col;
};

class Parser {
  public:
    explicit Parser(const std::string& text) : lex_(text) {}

    Circuit run() {
        header();
        while (lex_.peek().kind != Tok::End) statement();
        if (nq_ == 0) {
            const Token& e = lex_.peek();
            throw QasmParseError(e.line, e.col, "no quantum register declared");
        }
        Circuit c(nq_);
        for (auto& p : ops_) {
            try {
                c.add(std::move(p.op));
            } catch (const ContractError& err) {
                throw QasmParseError(p.line, p.col, err.what());
            }
        }
        return c;
    }

  private:
    [[noreturn]] void fail(const Token& t, const std::string& msg) { throw QasmParseError(t.line, t.col, msg); }

    Token expect_sym(const std::string& s) {
        Token t = lex_.next();
        if (t.kind != Tok::Sym || t.text != s)
            fail(t, "expected '" + s + "'" + (t.kind == Tok::End ? " before end of input" : ""));
        return t;
    }
    Token expect_id() {
        Token t = lex_.next();
        if (t.kind != Tok::Id) fail(t, "expected an identifier");
        return t;
    }
    int expect_int() {
        Token t = lex_.next();
        if (t.kind != Tok::Num || !t.integral) fail(t, "expected an integer");
        if (t.value > 1e9) fail(t, "integer too large");
        return int(t.value);
    }

    void header() {
        Token t = lex_.next();
        if (t.kind != Tok::Id || t.text != "OPENQASM") fail(t, "expected the 'OPENQASM 2.0;' header");
        Token v = lex_.next();
        if (v.kind != Tok::Num || v.value != 2.0) fail(v, "unsupported OpenQASM version (expected 2.0)");
        expect_sym(";");
    }

    void statement() {
        const Token t = lex_.next();
        if (t.kind != Tok::Id) fail(t, "expected a statement");
        const std::string& w = t.text;
        if (w == "OPENQASM") fail(t, "duplicate OPENQASM header");
        if (w == "include") {
            Token f = lex_.next();
            if (f.kind != Tok::Str) fail(f, "expected a file name string");
            if (f.text != "qelib1.inc") fail(f, "unsupported include \"" + f.text + "\" (only qelib1.inc)");
            expect_sym(";");
            return;
        }
        if (w == "qreg" || w == "creg") {
            declare(w == "qreg");
            return;
        }
        if (w == "gate" || w == "opaque" || w == "if" || w == "reset")
            fail(t, "unsupported statement '" + w + "'");
        if (w == "measure") {
            measure(t);
            return;
        }
        if (w == "barrier") {
            barrier(t);
            return;
        }
        const auto g = gate_table().find(w);
        if (g == gate_table().end()) fail(t, "unsupported gate '" + w + "'");
        apply(t, g->second);
    }

    void declare(bool quantum) {
        const Token name = expect_id();
        expect_sym("[");
        const int size = expect_int();
        expect_sym("]");
        expect_sym(";");
        if (size < 1) fail(name, "register size must be positive");
        if (qregs_.count(name.text) || cregs_.count(name.text)) fail(name, "duplicate register '" + name.text + "'");
        if (quantum) {
            qregs_[name.text] = Reg{nq_, size};
            nq_ += size;
        } else {
            cregs_[name.text] = Reg{nc_, size};
            nc_ += size;
        }
    }

    Arg arg(const std::map<std::string, Reg>& regs, const char* what) {
        const Token name = expect_id();
        const auto r = regs.find(name.text);
        if (r == regs.end()) fail(name, std::string("unknown ") + what + " register '" + name.text + "'");
        Arg a;
        a.reg = &r->second;
        a.line = name.line;
        a.col = name.col;
        if (lex_.peek().kind == Tok::Sym && lex_.peek().text == "[") {
            lex_.next();
            const Token it = lex_.peek();
            const int idx = expect_int();
            expect_sym("]");
            if (idx >= a.reg->size)
                fail(it, "index " + std::to_string(idx) + " out of range for register '" + name.text + "' of size " +
                             std::to_string(a.reg->size));
            a.index = idx;
        }
        return a;
    }

    std::vector<Arg> arglist() {
        std::vector<Arg> out;
        out.push_back(arg(qregs_, "quantum"));
        while (lex_.peek().kind == Tok::Sym && lex_.peek().text == ",") {
            lex_.next();
            out.push_back(arg(qregs_, "quantum"));
        }
        expect_sym(";");
        return out;
    }

    // constant angle expressions
    double expr() {
        double v = term();
        for (;;) {
            const Token& t = lex_.peek();
            if (t.kind == Tok::Sym && (t.text == "+" || t.text == "-")) {
                const bool add = lex_.next().text == "+";
                const double r = term();
                v = add ? v + r : v - r;
            } else {
                return v;
            }
        }
    }
    double term() {
        double v = unary();
        for (;;) {
            const Token& t = lex_.peek();
            if (t.kind == Tok::Sym && (t.text == "*" || t.text == "/")) {
                const Token op = lex_.next();
                const double r = unary();
                if (op.text == "*") {
                    v *= r;
                } else {
                    if (r == 0.0) fail(op, "division by zero in angle expression");
                    v /= r;
                }
            } else {
                return v;
            }
        }
    }
    double unary() {
        const Token& t = lex_.peek();
        if (t.kind == Tok::Sym && (t.text == "-" || t.text == "+")) {
            const bool neg = lex_.next().text == "-";
            const double v = unary();
            return neg ? -v : v;
        }
        return primary();
    }
    double primary() {
        const Token t = lex_.next();
        if (t.kind == Tok::Num) return t.value;
        if (t.kind == Tok::Id && t.text == "pi") return M_PI;
        if (t.kind == Tok::Sym && t.text == "(") {
            const double v = expr();
            expect_sym(")");
            return v;
        }
        fail(t, "expected a number, 'pi' or '(' in angle expression");
    }

    void apply(const Token& name, GateKind kind) {
        std::vector<double> params;
        if (lex_.peek().kind == Tok::Sym && lex_.peek().text == "(") {
            const Token open = lex_.next();
            if (lex_.peek().kind == Tok::Sym && lex_.peek().text == ")") fail(lex_.peek(), "missing parameter");
            params.push_back(expr());
            while (lex_.peek().kind == Tok::Sym && lex_.peek().text == ",") {
                lex_.next();
                params.push_back(expr());
            }
            expect_sym(")");
            (void)open;
        }
        const int np = gate_param_count(kind);
        if (int(params.size()) != np)
            fail(name, "gate '" + name.text + "' takes " + std::to_string(np) + " parameter(s), got " +
                           std::to_string(params.size()));
        const std::vector<Arg> args = arglist();
        const int arity = gate_arity(kind);
        if (int(args.size()) != arity)
            fail(name, "gate '" + name.text + "' takes " + std::to_string(arity) + " qubit(s), got " +
                           std::to_string(args.size()));
        // broadcast over whole-register operands (all of the same size)
        int width = 1;
        bool whole = false;
        for (const Arg& a : args) {
            if (a.index >= 0) continue;
            if (whole && a.reg->size != width) fail(name, "register operands of different sizes in broadcast");
            width = a.reg->size;
            whole = true;
        }
        for (int i = 0; i < width; ++i) {
            GateOp op{kind, {}, params};
            for (const Arg& a : args) op.qubits.push_back(a.reg->offset + (a.index >= 0 ? a.index : i));
            ops_.push_back(PendingOp{std::move(op), name.line, name.col});
        }
    }

    void measure(const Token& kw) {
        const Arg q = arg(qregs_, "quantum");
        expect_sym("->");
        const Arg c = arg(cregs_, "classical");
        expect_sym(";");
        if ((q.index < 0) != (c.index < 0)) fail(kw, "measure of a register needs a whole classical register");
        if (q.index >= 0) {
            ops_.push_back(PendingOp{GateOp{GateKind::MEASURE, {q.reg->offset + q.index}, {}}, kw.line, kw.col});
            return;
        }
        if (q.reg->size != c.reg->size) fail(kw, "measure between registers of different sizes");
        for (int i = 0; i < q.reg->size; ++i)
            ops_.push_back(PendingOp{GateOp{GateKind::MEASURE, {q.reg->offset + i}, {}}, kw.line, kw.col});
    }

    void barrier(const Token& kw) {
        for (const Arg& a : arglist()) {
            const int lo = a.index >= 0 ? a.index : 0, hi = a.index >= 0 ? a.index + 1 : a.reg->size;
            for (int i = lo; i < hi; ++i)
                ops_.push_back(PendingOp{GateOp{GateKind::BARRIER, {a.reg->offset + i}, {}}, kw.line, kw.col});
        }
    }

    Lexer lex_;
    std::map<std::string, Reg> qregs_, cregs_;
    int nq_ = 0, nc_ = 0;
    std::vector<PendingOp> ops_;
};

std::string fmt_angle(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

} // namespace

Circuit parse_qasm(const std::string& text) { return Parser(text).run(); }

Circuit parse_qasm_file(const std::string& path) {
    std::ifstream in(path);
    if (!in.good()) throw Error("cannot open QASM file '" + path + "'");
    std::ostringstream buf;
    buf << in.rdbuf();
    Circuit c = parse_qasm(buf.str());
    std::string stem = path;
    const size_t slash = stem.find_last_of("/\\");
    if (slash != std::string::npos) stem = stem.substr(slash + 1);
    const size_t dot = stem.find_last_of('.');
    if (dot != std::string::npos && dot > 0) stem = stem.substr(0, dot);
    c.set_name(stem);
    return c;
}

std::string emit_qasm(const Circuit& c) {
    std::ostringstream o;
    o << "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[" << c.num_qubits() << "];\n";
    bool measures = false;
    for (const auto& op : c.ops()) measures = measures || op.kind == GateKind::MEASURE;
    if (measures) o << "creg c[" << c.num_qubits() << "];\n";
    for (const auto& op : c.ops()) {
        if (op.kind == GateKind::MEASURE) {
            o << "measure q[" << op.qubits[0] << "] -> c[" << op.qubits[0] << "];\n";
            continue;
        }
        o << gate_name(op.kind);
        if (!op.params.empty()) {
            o << "(";
            for (size_t i = 0; i < op.params.size(); ++i) o << (i ? "," : "") << fmt_angle(op.params[i]);
            o << ")";
        }
        for (size_t i = 0; i < op.qubits.size(); ++i) o << (i ? "," : " ") << "q[" << op.qubits[i] << "]";
        o << ";\n";
    }
    return o.str();
}

} // namespace naqs

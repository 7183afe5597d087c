// C++ mirror of the reference engine's public API (include/naqs/*.hpp) over
// the C ABI.  Host-side logic that is inherently sequential or tiny
// (circuit validation, channel construction, calibration parsing, the RNG
// draws that fix sampling order) lives here; every operation on amplitudes or
// density-matrix entries goes through nq_* calls into the device.
//
// Semantics and error messages follow the reference: proj/src/circuit.cpp,
// gates.cpp, pauli.cpp, noise.cpp, statevector.cpp, densitymatrix.cpp.
#include "naqs/densitymatrix.hpp"
#include "naqs/gates.hpp"
#include "naqs/noise.hpp"
#include "naqs/pauli.hpp"
#include "naqs/statevector.hpp"

#include "../../include/naqs_b200.h"

#include <json.hpp>

#include <algorithm>
#include <chrono>
#include <map>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <numeric>
#include <sstream>
#include <unordered_set>

namespace naqs {

namespace {

using Eigen::MatrixXcd;
constexpr cplx kImag{0.0, 1.0};

// Map a C-ABI status onto the reference's exception hierarchy.
void check(nq_status st) {
    if (st == NQ_OK) return;
    const std::string msg = nq_last_error();
    if (st == NQ_ERR_CONTRACT) throw ContractError(msg);
    throw Error(msg);
}

nq_op to_abi(const GateOp& op) {
    nq_op o{};
    o.kind = static_cast<int32_t>(op.kind);
    o.nqubits = static_cast<int32_t>(op.qubits.size());
    for (size_t j = 0; j < op.qubits.size() && j < 3; ++j) o.qubits[j] = op.qubits[j];
    for (size_t j = 0; j < op.params.size() && j < 3; ++j) o.params[j] = op.params[j];
    return o;
}

nq_opts abi_opts(const EngineOptions& e) {
    nq_opts o;
    nq_default_opts(&o);
    o.device = e.device;
    o.max_qubits = e.max_qubits;
    o.tile_qubits = e.tile_qubits;
    o.fuse = e.fuse ? 1 : 0;
    return o;
}

// Row-major interleaved copy of an Eigen-subset matrix.
std::vector<double> flatten(const MatrixXcd& m) {
    std::vector<double> out(size_t(m.rows() * m.cols()) * 2);
    for (Eigen::Index r = 0; r < m.rows(); ++r)
        for (Eigen::Index c = 0; c < m.cols(); ++c) {
            const cplx v = m(r, c);
            out[size_t(r * m.cols() + c) * 2] = v.real();
            out[size_t(r * m.cols() + c) * 2 + 1] = v.imag();
        }
    return out;
}

struct PauliMasks {
    uint64_t flip = 0, signs = 0;
    int32_t ny = 0;
};

PauliMasks masks_of(const PauliString& p) {
    PauliMasks m;
    for (int i = 0; i < p.n; ++i) {
        const char L = p.letters[size_t(i)];
        if (L == 'X' || L == 'Y') m.flip |= uint64_t(1) << i;
        if (L == 'Y' || L == 'Z') m.signs |= uint64_t(1) << i;
        if (L == 'Y') ++m.ny;
    }
    return m;
}

} // namespace

// ============================================================================
// Circuit (proj/src/circuit.cpp)
// ============================================================================
int gate_arity(GateKind kind) {
    switch (kind) {
    case GateKind::CX: case GateKind::CZ: case GateKind::SWAP: return 2;
    case GateKind::CCX: return 3;
    default: return 1;
    }
}

int gate_param_count(GateKind kind) {
    switch (kind) {
    case GateKind::RX: case GateKind::RY: case GateKind::RZ: case GateKind::U1: return 1;
    case GateKind::U2: return 2;
    case GateKind::U3: return 3;
    default: return 0;
    }
}

bool gate_is_unitary(GateKind kind) { return kind != GateKind::MEASURE && kind != GateKind::BARRIER; }

namespace {
constexpr std::string_view kGateNames[] = {"x",  "y",  "z",  "h",  "s",  "sdg", "t",
                                           "tdg", "id", "rx", "ry", "rz", "u1",  "u2",
                                           "u3", "cx", "cz", "swap", "ccx", "measure", "barrier"};
}

std::string_view gate_name(GateKind kind) {
    const int i = static_cast<int>(kind);
    if (i < 0 || i >= int(std::size(kGateNames))) return "?";
    return kGateNames[i];
}

GateKind gate_kind_from_name(std::string_view name) {
    for (size_t i = 0; i < std::size(kGateNames); ++i)
        if (kGateNames[i] == name) return static_cast<GateKind>(i);
    throw ContractError("unknown gate name: " + std::string(name));
}

Circuit::Circuit(int num_qubits, std::string name)
    : nq_(num_qubits), name_(std::move(name)), measured_(size_t(std::max(num_qubits, 0)), false) {
    if (num_qubits < 1) throw ContractError("circuit qubit count must be positive");
}

void Circuit::add(GateOp op) {
    const std::string nm(gate_name(op.kind));
    const int arity = gate_arity(op.kind);
    if (int(op.qubits.size()) != arity)
        throw ContractError(nm + " expects " + std::to_string(arity) + " qubit(s), got " +
                            std::to_string(op.qubits.size()));
    const int np = gate_param_count(op.kind);
    if (int(op.params.size()) != np)
        throw ContractError(nm + " expects " + std::to_string(np) + " parameter(s), got " +
                            std::to_string(op.params.size()));
    std::unordered_set<int> seen;
    for (int q : op.qubits) {
        if (q < 0 || q >= nq_)
            throw ContractError("qubit index " + std::to_string(q) + " out of range for " + std::to_string(nq_) +
                                "-qubit circuit");
        if (!seen.insert(q).second) throw ContractError("duplicate qubit index " + std::to_string(q) + " in " + nm);
    }
    if (op.kind == GateKind::MEASURE) {
        measured_[size_t(op.qubits[0])] = true;
    } else if (gate_is_unitary(op.kind)) {
        for (int q : op.qubits)
            if (measured_[size_t(q)])
                throw ContractError("unitary after measurement on qubit " + std::to_string(q) +
                                    " (measurements are terminal)");
    }
    ops_.push_back(std::move(op));
}

void Circuit::add(GateKind kind, std::vector<int> qubits, std::vector<double> params) {
    add(GateOp{kind, std::move(qubits), std::move(params)});
}

std::size_t Circuit::unitary_count() const {
    return size_t(std::count_if(ops_.begin(), ops_.end(), [](const GateOp& o) { return gate_is_unitary(o.kind); }));
}

Circuit Circuit::unitaries_only() const {
    Circuit out(nq_, name_);
    for (const auto& op : ops_)
        if (gate_is_unitary(op.kind)) out.add(op);
    return out;
}

Circuit Circuit::inverse() const {
    Circuit out(nq_, name_.empty() ? "" : name_ + "_inv");
    for (auto it = ops_.rbegin(); it != ops_.rend(); ++it) {
        const GateOp& op = *it;
        switch (op.kind) {
        case GateKind::MEASURE: throw ContractError("cannot invert a circuit containing measurements");
        case GateKind::S: out.add(GateKind::SDG, op.qubits); break;
        case GateKind::SDG: out.add(GateKind::S, op.qubits); break;
        case GateKind::T: out.add(GateKind::TDG, op.qubits); break;
        case GateKind::TDG: out.add(GateKind::T, op.qubits); break;
        case GateKind::RX: case GateKind::RY: case GateKind::RZ: case GateKind::U1:
            out.add(op.kind, op.qubits, {-op.params[0]});
            break;
        case GateKind::U2:  // u2(phi, lambda)^-1 = u3(-pi/2, -lambda, -phi)
            out.add(GateKind::U3, op.qubits, {-M_PI / 2.0, -op.params[1], -op.params[0]});
            break;
        case GateKind::U3: out.add(GateKind::U3, op.qubits, {-op.params[0], -op.params[2], -op.params[1]}); break;
        default: out.add(op); break;  // self-inverse kinds and BARRIER
        }
    }
    return out;
}

// ============================================================================
// Gate matrices (proj/src/gates.cpp:12-118)
// ============================================================================
namespace {
MatrixXcd m2(cplx a, cplx b, cplx c, cplx d) {
    MatrixXcd m(2, 2);
    m(0, 0) = a; m(0, 1) = b; m(1, 0) = c; m(1, 1) = d;
    return m;
}
MatrixXcd perm_matrix(int dim, int a, int b) {  // identity with rows a, b swapped
    MatrixXcd m = MatrixXcd::Identity(dim, dim);
    m(a, a) = 0; m(b, b) = 0; m(a, b) = 1; m(b, a) = 1;
    return m;
}
} // namespace

Eigen::MatrixXcd gate_matrix(GateKind kind, const std::vector<double>& params) {
    if (!gate_is_unitary(kind)) throw ContractError(std::string(gate_name(kind)) + " has no unitary matrix");
    const int want = gate_param_count(kind);
    if (int(params.size()) != want)
        throw ContractError(std::string(gate_name(kind)) + " expects " + std::to_string(want) +
                            " parameter(s), got " + std::to_string(params.size()));
    auto u3 = [](double th, double ph, double la) {
        const double c = std::cos(th / 2.0), s = std::sin(th / 2.0);
        return m2(c, -std::exp(kImag * la) * s, std::exp(kImag * ph) * s, std::exp(kImag * (ph + la)) * c);
    };
    const double r = 1.0 / std::sqrt(2.0);
    switch (kind) {
    case GateKind::ID: return MatrixXcd::Identity(2, 2);
    case GateKind::X: return m2(0, 1, 1, 0);
    case GateKind::Y: return m2(0, -kImag, kImag, 0);
    case GateKind::Z: return m2(1, 0, 0, -1);
    case GateKind::H: return m2(r, r, r, -r);
    case GateKind::S: return m2(1, 0, 0, kImag);
    case GateKind::SDG: return m2(1, 0, 0, -kImag);
    case GateKind::T: return m2(1, 0, 0, std::exp(kImag * (M_PI / 4.0)));
    case GateKind::TDG: return m2(1, 0, 0, std::exp(-kImag * (M_PI / 4.0)));
    case GateKind::RX: {
        const double c = std::cos(params[0] / 2.0), s = std::sin(params[0] / 2.0);
        return m2(c, -kImag * s, -kImag * s, c);
    }
    case GateKind::RY: {
        const double c = std::cos(params[0] / 2.0), s = std::sin(params[0] / 2.0);
        return m2(c, -s, s, c);
    }
    case GateKind::RZ: return m2(std::exp(-kImag * (params[0] / 2.0)), 0, 0, std::exp(kImag * (params[0] / 2.0)));
    case GateKind::U1: return m2(1, 0, 0, std::exp(kImag * params[0]));
    case GateKind::U2: return u3(M_PI / 2.0, params[0], params[1]);
    case GateKind::U3: return u3(params[0], params[1], params[2]);
    case GateKind::CX: return perm_matrix(4, 1, 3);    // control = local bit 0
    case GateKind::CZ: {
        MatrixXcd m = MatrixXcd::Identity(4, 4);
        m(3, 3) = -1;
        return m;
    }
    case GateKind::SWAP: return perm_matrix(4, 1, 2);
    case GateKind::CCX: return perm_matrix(8, 3, 7);
    default: throw ContractError("unhandled gate kind");
    }
}

Eigen::MatrixXcd gate_matrix(const GateOp& op) { return gate_matrix(op.kind, op.params); }

double unitarity_residual(const Eigen::MatrixXcd& u) {
    return (u.adjoint() * u - MatrixXcd::Identity(u.rows(), u.cols())).cwiseAbs().maxCoeff();
}

// ============================================================================
// Pauli words (proj/src/pauli.cpp)
// ============================================================================
namespace {
bool pauli_letter_ok(char c) { return c == 'I' || c == 'X' || c == 'Y' || c == 'Z'; }
MatrixXcd letter_matrix(char L) {
    switch (L) {
    case 'I': return m2(1, 0, 0, 1);
    case 'X': return m2(0, 1, 1, 0);
    case 'Y': return m2(0, cplx(0, -1), cplx(0, 1), 0);
    case 'Z': return m2(1, 0, 0, -1);
    default: throw ContractError(std::string("illegal Pauli letter: ") + L);
    }
}
} // namespace

PauliString::PauliString(std::string letters_, double coeff)
    : n(int(letters_.size())), letters(std::move(letters_)), coefficient(coeff) {
    for (char c : letters)
        if (!pauli_letter_ok(c)) throw ContractError(std::string("illegal Pauli letter: ") + c);
    if (!std::isfinite(coefficient)) throw ContractError("Pauli coefficient must be finite");
}

PauliString pauli_parse(const std::string& text) {
    if (text.empty()) throw ContractError("empty Pauli string");
    const auto star = text.find('*');
    if (star == std::string::npos) {
        return PauliString(text, 1.0);
    }
    const std::string head = text.substr(0, star), tail = text.substr(star + 1);
    char* end = nullptr;
    const double coeff = std::strtod(head.c_str(), &end);
    if (end == head.c_str() || *end != '\0') throw ContractError("bad Pauli coefficient: '" + head + "'");
    if (tail.empty()) throw ContractError("empty Pauli letters in '" + text + "'");
    return PauliString(tail, coeff);
}

std::string pauli_format(const PauliString& p) {
    char buf[48];
    std::snprintf(buf, sizeof(buf), "%.17g", p.coefficient);
    return std::string(buf) + "*" + p.letters;
}

void Hamiltonian::add(const PauliString& term) {
    if (terms.empty() && n == 0) n = term.n;
    if (term.n != n)
        throw ContractError("Hamiltonian term length " + std::to_string(term.n) + " does not match n=" +
                            std::to_string(n));
    terms.push_back(term);
}

void Hamiltonian::add(const std::string& letters, double coeff) { add(PauliString(letters, coeff)); }

Eigen::MatrixXcd pauli_dense(const PauliString& p) {
    MatrixXcd acc = MatrixXcd::Constant(1, 1, p.coefficient);
    for (char L : p.letters) {  // each new letter becomes the new most-significant factor
        const MatrixXcd f = letter_matrix(L);
        MatrixXcd next(acc.rows() * 2, acc.cols() * 2);
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) next.block(i * acc.rows(), j * acc.cols(), acc.rows(), acc.cols()) = f(i, j) * acc;
        acc = std::move(next);
    }
    return acc;
}

Eigen::MatrixXcd hamiltonian_dense(const Hamiltonian& h) {
    if (h.n > kDenseOracleLimit)
        throw ContractError("hamiltonian_dense limited to n <= " + std::to_string(kDenseOracleLimit) + ", got n=" +
                            std::to_string(h.n));
    if (h.n < 1) throw ContractError("hamiltonian_dense requires n >= 1");
    const Eigen::Index dim = Eigen::Index(1) << h.n;
    MatrixXcd m = MatrixXcd::Zero(dim, dim);
    for (const auto& t : h.terms) m += pauli_dense(t);
    return m;
}

// ============================================================================
// Noise channels, readout, calibration, attach_noise (proj/src/noise.cpp)
// ============================================================================
double KrausChannel::completeness_residual() const {
    if (kraus.empty()) return 1.0;
    const Eigen::Index d = kraus.front().rows();
    MatrixXcd s = MatrixXcd::Zero(d, d);
    for (const auto& k : kraus) s += k.adjoint() * k;
    return (s - MatrixXcd::Identity(d, d)).cwiseAbs().maxCoeff();
}

bool KrausChannel::is_identity(double tol) const {
    if (kraus.size() != 1) return false;
    const auto& k = kraus.front();
    return (k - MatrixXcd::Identity(k.rows(), k.cols())).cwiseAbs().maxCoeff() <= tol;
}

void validate_channel(const KrausChannel& ch, double tol) {
    if (ch.arity != 1 && ch.arity != 2)
        throw ContractError("channel arity must be 1 or 2, got " + std::to_string(ch.arity));
    if (ch.kraus.empty()) throw ContractError("channel needs at least one Kraus operator");
    const Eigen::Index d = Eigen::Index(1) << ch.arity;
    for (const auto& k : ch.kraus) {
        if (k.rows() != d || k.cols() != d) throw ContractError("Kraus operator has wrong dimension");
        if (!k.allFinite()) throw ContractError("Kraus operator has non-finite entries");
    }
    const double res = ch.completeness_residual();
    if (res > tol)
        throw ContractError("Kraus completeness residual " + std::to_string(res) + " exceeds " + std::to_string(tol));
}

KrausChannel identity_channel(int arity) {
    const Eigen::Index d = Eigen::Index(1) << arity;
    return KrausChannel{arity, {MatrixXcd::Identity(d, d)}};
}

KrausChannel depolarizing(double p, int arity) {
    if (p < 0.0 || p > 1.0) throw ContractError("depolarizing probability must be in [0,1], got " + std::to_string(p));
    if (arity != 1 && arity != 2) throw ContractError("depolarizing arity must be 1 or 2");
    if (p == 0.0) return identity_channel(arity);
    const MatrixXcd P[4] = {letter_matrix('I'), letter_matrix('X'), letter_matrix('Y'), letter_matrix('Z')};
    KrausChannel ch;
    ch.arity = arity;
    if (arity == 1) {
        if (p < 1.0) ch.kraus.push_back(std::sqrt(1.0 - p) * P[0]);
        const double w = std::sqrt(p / 3.0);
        for (int a = 1; a < 4; ++a) ch.kraus.push_back(w * P[a]);
        return ch;
    }
    if (p < 1.0) ch.kraus.push_back(std::sqrt(1.0 - p) * MatrixXcd::Identity(4, 4));
    const double w = std::sqrt(p / 15.0);
    // Kraus order: a (qubit 0 letter) outer, b (qubit 1 letter) inner; the
    // operator on local bits (q0 = low, q1 = high) is kron(P_b, P_a).
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            if (a == 0 && b == 0) continue;
            MatrixXcd k(4, 4);
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) k.block(2 * i, 2 * j, 2, 2) = P[b](i, j) * P[a];
            ch.kraus.push_back(w * k);
        }
    return ch;
}

KrausChannel amplitude_damping(double gamma) {
    if (gamma < 0.0 || gamma > 1.0) throw ContractError("damping probability must be in [0,1]");
    MatrixXcd k0 = MatrixXcd::Identity(2, 2);
    k0(1, 1) = std::sqrt(1.0 - gamma);
    MatrixXcd k1 = MatrixXcd::Zero(2, 2);
    k1(0, 1) = std::sqrt(gamma);
    KrausChannel ch{1, {k0}};
    if (gamma > 0.0) ch.kraus.push_back(k1);
    return ch;
}

KrausChannel thermal_relaxation(double t1_us, double t2_us, double duration_ns) {
    if (t1_us <= 0.0 || t2_us <= 0.0) throw ContractError("thermal relaxation requires positive T1 and T2");
    if (duration_ns < 0.0) throw ContractError("duration must be non-negative");
    if (duration_ns == 0.0) return identity_channel(1);
    const double d = duration_ns / 1000.0;
    const double t2e = std::min(t2_us, t1_us);
    const double gamma = 1.0 - std::exp(-d / t1_us);
    const double lambda = 1.0 - std::exp(d / t1_us - 2.0 * d / t2e);
    const MatrixXcd amp[2] = {m2(1, 0, 0, std::sqrt(1.0 - gamma)), m2(0, std::sqrt(gamma), 0, 0)};
    const MatrixXcd ph[2] = {m2(1, 0, 0, std::sqrt(1.0 - lambda)), m2(0, 0, 0, std::sqrt(lambda))};
    KrausChannel ch;
    ch.arity = 1;
    for (const auto& P : ph)
        for (const auto& A : amp) {
            MatrixXcd k = P * A;
            if (k.cwiseAbs().maxCoeff() > 1e-15) ch.kraus.push_back(std::move(k));
        }
    return ch;
}

bool ReadoutModel::is_trivial() const {
    return std::all_of(qubits.begin(), qubits.end(), [](const QubitReadout& q) { return q.p01 == 0.0 && q.p10 == 0.0; });
}

std::vector<double> readout_apply_dist(const std::vector<double>& dist, const ReadoutModel& r) {
    const size_t n = r.qubits.size();
    if (dist.size() != (size_t(1) << n))
        throw ContractError("distribution length " + std::to_string(dist.size()) + " does not match 2^" +
                            std::to_string(n));
    std::vector<double> p01(n), p10(n), out(dist.size());
    for (size_t q = 0; q < n; ++q) {
        p01[q] = r.qubits[q].p01;
        p10[q] = r.qubits[q].p10;
    }
    check(nq_readout_apply_dist(dist.data(), int(n), p01.data(), p10.data(), out.data()));
    return out;
}

std::map<std::string, std::uint64_t> readout_apply_samples(const std::map<std::string, std::uint64_t>& counts,
                                                           const ReadoutModel& r, std::uint64_t seed) {
    // Sequential by contract: one RNG stream over (bitstring in map order) x
    // shot x qubit ascending, drawing only when the flip probability is > 0.
    Rng rng(seed);
    std::map<std::string, std::uint64_t> out;
    const size_t n = r.qubits.size();
    for (const auto& [bits, count] : counts) {
        if (bits.size() != n) throw ContractError("bitstring length does not match readout model");
        for (std::uint64_t s = 0; s < count; ++s) {
            std::string b = bits;
            for (size_t q = 0; q < n; ++q) {
                char& ch = b[n - 1 - q];
                const double p = ch == '1' ? r.qubits[q].p01 : r.qubits[q].p10;
                if (p > 0.0 && rng.next_double() < p) ch = ch == '1' ? '0' : '1';
            }
            ++out[b];
        }
    }
    return out;
}

DeviceNoiseModel DeviceNoiseModel::zero_noise(int n) {
    DeviceNoiseModel m;
    m.name = "zero-noise";
    m.qubits.assign(size_t(n), QubitParams{1.0, 1.0, 0.0, 0.0});
    m.default_1q = GateParams{"default_1q", {}, 0.0, 0.0};
    m.default_2q = GateParams{"default_2q", {}, 0.0, 0.0};
    return m;
}

std::optional<DeviceNoiseModel::GateParams> DeviceNoiseModel::find_gate(std::string_view gate,
                                                                         const std::vector<int>& qs) const {
    for (const auto& g : gates)
        if (g.name == gate && g.qubits == qs) return g;
    if (qs.size() == 1 && default_1q) return default_1q;
    if (qs.size() == 2 && default_2q) return default_2q;
    return std::nullopt;
}

ReadoutModel DeviceNoiseModel::readout() const {
    ReadoutModel r;
    for (const auto& q : qubits) r.qubits.push_back({q.readout_p01, q.readout_p10});
    return r;
}

namespace {
using json = nlohmann::json;

double field_number(const json& o, const std::string& f, const std::string& where) {
    if (!o.contains(f)) throw CalibrationError("missing field '" + f + "' in " + where);
    if (!o[f].is_number()) throw CalibrationError("field '" + f + "' in " + where + " must be a number");
    return o[f].get<double>();
}

double field_prob(const json& o, const std::string& f, const std::string& where) {
    const double v = field_number(o, f, where);
    if (v < 0.0 || v > 1.0)
        throw CalibrationError("field '" + f + "' in " + where + " must be in [0,1], got " + std::to_string(v));
    return v;
}

DeviceNoiseModel::GateParams gate_default(const json& o, const std::string& where) {
    DeviceNoiseModel::GateParams g;
    g.name = where;
    g.error = field_prob(o, "error", where);
    g.duration_ns = field_number(o, "duration_ns", where);
    if (g.duration_ns < 0.0) throw CalibrationError("field 'duration_ns' in " + where + " must be non-negative");
    return g;
}
} // namespace

DeviceNoiseModel load_calibration(const std::string& text) {
    json doc;
    try {
        doc = json::parse(text);
    } catch (const json::parse_error& e) {
        throw CalibrationError(std::string("malformed calibration document: ") + e.what());
    }
    if (!doc.is_object()) throw CalibrationError("calibration document must be a JSON object");
    DeviceNoiseModel m;
    m.name = doc.value("name", std::string("unnamed"));
    if (!doc.contains("qubits") || !doc["qubits"].is_array() || doc["qubits"].empty())
        throw CalibrationError("missing field 'qubits' (non-empty array required)");
    int qi = 0;
    for (const auto& q : doc["qubits"]) {
        const std::string where = "qubits[" + std::to_string(qi++) + "]";
        DeviceNoiseModel::QubitParams qp;
        qp.t1_us = field_number(q, "t1_us", where);
        qp.t2_us = field_number(q, "t2_us", where);
        if (qp.t1_us <= 0.0 || qp.t2_us <= 0.0) throw CalibrationError("T1/T2 in " + where + " must be positive");
        qp.readout_p01 = field_prob(q, "readout_p01", where);
        qp.readout_p10 = field_prob(q, "readout_p10", where);
        if (qp.t2_us > qp.t1_us) {
            m.warnings.push_back(where + ": t2_us " + std::to_string(qp.t2_us) + " exceeds t1_us " +
                                 std::to_string(qp.t1_us) + "; clamped to t1_us");
            qp.t2_us = qp.t1_us;
        }
        m.qubits.push_back(qp);
    }
    if (doc.contains("gates")) {
        if (!doc["gates"].is_array()) throw CalibrationError("field 'gates' must be an array");
        int gi = 0;
        for (const auto& g : doc["gates"]) {
            const std::string where = "gates[" + std::to_string(gi++) + "]";
            DeviceNoiseModel::GateParams gp;
            if (!g.contains("name") || !g["name"].is_string()) throw CalibrationError("missing field 'name' in " + where);
            gp.name = g["name"].get<std::string>();
            if (!g.contains("qubits") || !g["qubits"].is_array() || g["qubits"].empty() || g["qubits"].size() > 2)
                throw CalibrationError("field 'qubits' in " + where + " must be an array of 1 or 2 indices");
            for (const auto& v : g["qubits"]) {
                if (!v.is_number_integer()) throw CalibrationError("qubit indices in " + where + " must be integers");
                const int idx = v.get<int>();
                if (idx < 0 || idx >= m.num_qubits())
                    throw CalibrationError("qubit index " + std::to_string(idx) + " in " + where + " out of range");
                gp.qubits.push_back(idx);
            }
            gp.error = field_prob(g, "error", where);
            gp.duration_ns = field_number(g, "duration_ns", where);
            if (gp.duration_ns < 0.0) throw CalibrationError("field 'duration_ns' in " + where + " must be non-negative");
            m.gates.push_back(std::move(gp));
        }
    }
    if (doc.contains("default_1q")) m.default_1q = gate_default(doc["default_1q"], "default_1q");
    if (doc.contains("default_2q")) m.default_2q = gate_default(doc["default_2q"], "default_2q");
    return m;
}

DeviceNoiseModel load_calibration_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw CalibrationError("cannot open calibration file: " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return load_calibration(buf.str());
}

std::vector<GateOp> NoisySchedule::project_ops() const {
    std::vector<GateOp> ops;
    for (const auto& it : items)
        if (const auto* op = std::get_if<GateOp>(&it)) ops.push_back(*op);
    return ops;
}

NoisySchedule attach_noise(const Circuit& c, const DeviceNoiseModel& m) {
    if (c.num_qubits() > m.num_qubits())
        throw ContractError("device model covers " + std::to_string(m.num_qubits()) + " qubits, circuit needs " +
                            std::to_string(c.num_qubits()));
    NoisySchedule s;
    s.num_qubits = c.num_qubits();
    const ReadoutModel full = m.readout();
    s.readout.qubits.assign(full.qubits.begin(), full.qubits.begin() + c.num_qubits());
    // The channels of a gate depend only on (kind, qubits): build them once per
    // distinct pair (a long Trotter circuit repeats a handful of them).
    std::map<std::pair<int, std::vector<int>>, std::vector<ChannelApplication>> memo;
    for (const auto& op : c.ops()) {
        s.items.push_back(op);
        if (!gate_is_unitary(op.kind)) continue;
        const int arity = int(op.qubits.size());
        if (arity > 2)
            throw ContractError("no noise channel for " + std::string(gate_name(op.kind)) +
                                ": gates on more than 2 qubits are not calibratable");
        auto key = std::make_pair(int(op.kind), op.qubits);
        auto it = memo.find(key);
        if (it == memo.end()) {
            const auto gp = m.find_gate(gate_name(op.kind), op.qubits);
            if (!gp)
                throw ContractError("no calibration entry or default for gate '" + std::string(gate_name(op.kind)) +
                                    "' on qubits [" + std::to_string(op.qubits[0]) +
                                    (arity == 2 ? "," + std::to_string(op.qubits[1]) : "") + "]");
            std::vector<ChannelApplication> chans;
            chans.push_back(ChannelApplication{depolarizing(gp->error, arity), op.qubits});
            for (int q : op.qubits) {
                const auto& qp = m.qubits[size_t(q)];
                chans.push_back(ChannelApplication{thermal_relaxation(qp.t1_us, qp.t2_us, gp->duration_ns), {q}});
            }
            it = memo.emplace(std::move(key), std::move(chans)).first;
        }
        for (const auto& ch : it->second) s.items.push_back(ch);
    }
    return s;
}

// ============================================================================
// StateVector (proj/src/statevector.cpp) over nq_sv
// ============================================================================
StateVector::StateVector(int num_qubits) : StateVector(num_qubits, EngineOptions{}) {}

StateVector::StateVector(int num_qubits, const EngineOptions& opts) : n_(num_qubits) {
    const nq_opts o = abi_opts(opts);
    check(nq_sv_create(num_qubits, &o, &h_));
}

StateVector::StateVector(const StateVector& other) : n_(other.n_) {
    check(nq_sv_clone(other.h_, &h_));
}

StateVector::StateVector(StateVector&& other) noexcept
    : n_(other.n_), h_(other.h_), mirror_(std::move(other.mirror_)), mirror_ok_(other.mirror_ok_) {
    other.h_ = nullptr;
    other.mirror_ok_ = false;
}

StateVector& StateVector::operator=(const StateVector& other) {
    if (this == &other) return *this;
    nq_sv* h = nullptr;
    check(nq_sv_clone(other.h_, &h));
    if (h_) nq_sv_destroy(h_);
    h_ = h;
    n_ = other.n_;
    mirror_ok_ = false;
    return *this;
}

StateVector& StateVector::operator=(StateVector&& other) noexcept {
    if (this == &other) return *this;
    if (h_) nq_sv_destroy(h_);
    h_ = other.h_;
    n_ = other.n_;
    mirror_ = std::move(other.mirror_);
    mirror_ok_ = other.mirror_ok_;
    other.h_ = nullptr;
    other.mirror_ok_ = false;
    return *this;
}

StateVector::~StateVector() {
    if (h_) nq_sv_destroy(h_);
}

void StateVector::reset() {
    check(nq_sv_reset(h_));
    invalidate();
}

const std::vector<cplx>& StateVector::amplitudes() const {
    if (!mirror_ok_) {
        mirror_.resize(dim());
        check(nq_sv_get_amplitudes(h_, 0, dim(), reinterpret_cast<double*>(mirror_.data())));
        mirror_ok_ = true;
    }
    return mirror_;
}

cplx StateVector::amplitude(std::size_t index) const { return amplitudes()[index]; }

void StateVector::apply(const GateOp& op) {
    const nq_op o = to_abi(op);
    check(nq_sv_apply_ops(h_, &o, 1));
    invalidate();
}

void StateVector::run(const Circuit& c) {
    if (c.num_qubits() != n_)
        throw ContractError("circuit acts on " + std::to_string(c.num_qubits()) + " qubits, state has " +
                            std::to_string(n_));
    std::vector<nq_op> ops;
    ops.reserve(c.size());
    for (const auto& op : c.ops()) {
        if (op.kind == GateKind::MEASURE) throw ContractError("run() takes measurement-free circuits; use sample()");
        ops.push_back(to_abi(op));
    }
    check(nq_sv_apply_ops(h_, ops.data(), int64_t(ops.size())));
    invalidate();
}

double StateVector::norm_sq() const {
    double v = 0.0;
    check(nq_sv_norm_sq(h_, &v));
    return v;
}

double StateVector::expectation(const PauliString& p) const {
    if (p.n != n_)
        throw ContractError("Pauli string length " + std::to_string(p.n) + " does not match state qubit count " +
                            std::to_string(n_));
    return expectations({p})[0];
}

std::vector<double> StateVector::expectations(const std::vector<PauliString>& terms) const {
    std::vector<uint64_t> flip, signs;
    std::vector<int32_t> ny;
    std::vector<double> coeff;
    for (const auto& p : terms) {
        if (p.n != n_)
            throw ContractError("Pauli string length " + std::to_string(p.n) + " does not match state qubit count " +
                                std::to_string(n_));
        const PauliMasks m = masks_of(p);
        flip.push_back(m.flip);
        signs.push_back(m.signs);
        ny.push_back(m.ny);
        coeff.push_back(p.coefficient);
    }
    std::vector<double> out(terms.size());
    if (!terms.empty())
        check(nq_sv_expectation_batch(h_, flip.data(), signs.data(), ny.data(), coeff.data(), int(terms.size()),
                                      out.data()));
    return out;
}

std::vector<double> StateVector::probabilities() const {
    std::vector<double> p(dim());
    check(nq_sv_probabilities(h_, p.data()));
    return p;
}

std::string index_to_bitstring(std::size_t index, int n) {
    std::string s(size_t(n), '0');
    for (int q = 0; q < n; ++q)
        if ((index >> q) & 1) s[size_t(n - 1 - q)] = '1';
    return s;
}

namespace {
std::vector<double> sorted_uniforms(std::uint64_t shots, std::uint64_t seed) {
    Rng rng(seed);
    std::vector<double> u(shots);
    for (auto& v : u) v = rng.next_double();
    std::sort(u.begin(), u.end());
    return u;
}

std::map<std::string, std::uint64_t> counts_map(const std::vector<uint64_t>& idx, const std::vector<uint64_t>& cnt,
                                                uint64_t k, int n) {
    std::map<std::string, std::uint64_t> out;
    for (uint64_t i = 0; i < k; ++i) out[index_to_bitstring(size_t(idx[i]), n)] += cnt[i];
    return out;
}
} // namespace

std::map<std::string, std::uint64_t> sample_distribution(const std::vector<double>& dist, int n, std::uint64_t shots,
                                                         std::uint64_t seed) {
    if (shots < 1) throw ContractError("shots must be >= 1");
    if (dist.size() != (size_t(1) << n)) throw ContractError("distribution length does not match qubit count");
    const auto u = sorted_uniforms(shots, seed);
    std::vector<uint64_t> idx(shots), cnt(shots);
    uint64_t k = 0;
    check(nq_sample_dist_sorted(dist.data(), dist.size(), u.data(), shots, idx.data(), cnt.data(), &k));
    return counts_map(idx, cnt, k, n);
}

std::map<std::string, std::uint64_t> StateVector::sample(std::uint64_t shots, std::uint64_t seed) const {
    if (shots < 1) throw ContractError("shots must be >= 1");
    const auto u = sorted_uniforms(shots, seed);
    std::vector<uint64_t> idx(shots), cnt(shots);
    uint64_t k = 0;
    check(nq_sv_sample_sorted(h_, u.data(), shots, idx.data(), cnt.data(), &k));
    return counts_map(idx, cnt, k, n_);
}

void StateVector::apply_kraus_trajectory(const KrausChannel& ch, const std::vector<int>& qubits, Rng& rng) {
    if (int(qubits.size()) != ch.arity)
        throw ContractError("channel arity " + std::to_string(ch.arity) + " does not match " +
                            std::to_string(qubits.size()) + " qubits");
    const int k = int(qubits.size());
    std::vector<int32_t> q(qubits.begin(), qubits.end());
    std::vector<double> flat;
    for (const auto& K : ch.kraus) {
        auto f = flatten(K);
        flat.insert(flat.end(), f.begin(), f.end());
    }
    std::vector<double> w(ch.kraus.size());
    check(nq_sv_kraus_weights(h_, q.data(), k, int(ch.kraus.size()), flat.data(), w.data()));
    const double total = std::accumulate(w.begin(), w.end(), 0.0);
    if (std::abs(total - 1.0) > 1e-8)
        throw ContractError("Kraus branch probabilities sum to " + std::to_string(total) +
                            "; channel is not trace preserving on this state");
    const double u = rng.next_double() * total;
    size_t chosen = w.size() - 1;
    double cum = 0.0;
    for (size_t i = 0; i < w.size(); ++i) {
        cum += w[i];
        if (u < cum) {
            chosen = i;
            break;
        }
    }
    // K / sqrt(w) in one device op: apply and renormalise in the same pass.
    const double scale = 1.0 / std::sqrt(w[chosen]);
    std::vector<double> m = flatten(ch.kraus[chosen]);
    for (double& v : m) v *= scale;
    check(nq_sv_apply_matrix(h_, q.data(), k, m.data()));
    invalidate();
}

void StateVector::run_trajectory(const NoisySchedule& schedule, Rng& rng) {
    if (schedule.num_qubits != n_) throw ContractError("schedule qubit count mismatch");
    for (const auto& item : schedule.items) {
        if (const auto* op = std::get_if<GateOp>(&item)) {
            if (op->kind == GateKind::MEASURE || op->kind == GateKind::BARRIER) continue;
            apply(*op);
        } else {
            const auto& app = std::get<ChannelApplication>(item);
            apply_kraus_trajectory(app.channel, app.qubits, rng);
        }
    }
}

StateVector sv_run(const Circuit& c) {
    StateVector s(c.num_qubits());
    s.run(c);
    return s;
}

// ============================================================================
// DensityMatrix (proj/src/densitymatrix.cpp) over nq_dm
// ============================================================================
DensityMatrix::DensityMatrix(int num_qubits) : DensityMatrix(num_qubits, EngineOptions{}) {}

DensityMatrix::DensityMatrix(int num_qubits, const EngineOptions& opts) : n_(num_qubits) {
    const nq_opts o = abi_opts(opts);
    check(nq_dm_create(num_qubits, &o, &h_));
}

DensityMatrix::DensityMatrix(const DensityMatrix& other) : n_(other.n_) { check(nq_dm_clone(other.h_, &h_)); }

DensityMatrix::DensityMatrix(DensityMatrix&& other) noexcept
    : n_(other.n_), h_(other.h_), mirror_(std::move(other.mirror_)), mirror_ok_(other.mirror_ok_) {
    other.h_ = nullptr;
    other.mirror_ok_ = false;
}

DensityMatrix& DensityMatrix::operator=(const DensityMatrix& other) {
    if (this == &other) return *this;
    nq_dm* h = nullptr;
    check(nq_dm_clone(other.h_, &h));
    if (h_) nq_dm_destroy(h_);
    h_ = h;
    n_ = other.n_;
    mirror_ok_ = false;
    return *this;
}

DensityMatrix& DensityMatrix::operator=(DensityMatrix&& other) noexcept {
    if (this == &other) return *this;
    if (h_) nq_dm_destroy(h_);
    h_ = other.h_;
    n_ = other.n_;
    mirror_ = std::move(other.mirror_);
    mirror_ok_ = other.mirror_ok_;
    other.h_ = nullptr;
    other.mirror_ok_ = false;
    return *this;
}

DensityMatrix::~DensityMatrix() {
    if (h_) nq_dm_destroy(h_);
}

void DensityMatrix::reset() {
    check(nq_dm_reset(h_));
    mirror_ok_ = false;
}

const std::vector<cplx>& DensityMatrix::data() const {
    if (!mirror_ok_) {
        mirror_.resize(dim() * dim());
        check(nq_dm_get_entries(h_, 0, dim() * dim(), reinterpret_cast<double*>(mirror_.data())));
        mirror_ok_ = true;
    }
    return mirror_;
}

cplx DensityMatrix::entry(std::size_t row, std::size_t col) const { return data()[row * dim() + col]; }

void DensityMatrix::apply(const GateOp& op) {
    const nq_op o = to_abi(op);
    check(nq_dm_apply_ops(h_, &o, 1));
    mirror_ok_ = false;
}

void DensityMatrix::apply_channel(const KrausChannel& ch, const std::vector<int>& qubits) {
    if (int(qubits.size()) != ch.arity)
        throw ContractError("channel arity " + std::to_string(ch.arity) + " does not match " +
                            std::to_string(qubits.size()) + " qubits");
    for (int q : qubits)
        if (q < 0 || q >= n_) throw ContractError("qubit index " + std::to_string(q) + " out of range");
    validate_channel(ch);
    if (ch.is_identity()) return;
    std::vector<int32_t> q(qubits.begin(), qubits.end());
    std::vector<double> flat;
    for (const auto& K : ch.kraus) {
        auto f = flatten(K);
        flat.insert(flat.end(), f.begin(), f.end());
    }
    check(nq_dm_apply_channel(h_, q.data(), ch.arity, int(ch.kraus.size()), flat.data()));
    mirror_ok_ = false;
}

void DensityMatrix::run(const Circuit& c) {
    if (c.num_qubits() != n_) throw ContractError("circuit qubit count mismatch");
    std::vector<nq_op> ops;
    for (const auto& op : c.ops()) {
        if (op.kind == GateKind::MEASURE) throw ContractError("run() takes measurement-free circuits");
        ops.push_back(to_abi(op));
    }
    check(nq_dm_apply_ops(h_, ops.data(), int64_t(ops.size())));
    mirror_ok_ = false;
}

std::vector<std::vector<double>> run_trajectories(const NoisySchedule& schedule, std::uint64_t ntraj, Rng& rng,
                                                  const std::vector<PauliString>& observables) {
    const int n = schedule.num_qubits;
    std::vector<nq_sched_item> items;
    std::vector<double> pool;
    size_t nch = 0;
    for (const auto& item : schedule.items) {
        nq_sched_item it{};
        if (const auto* op = std::get_if<GateOp>(&item)) {
            if (op->kind == GateKind::MEASURE || op->kind == GateKind::BARRIER) continue;
            it.type = 0;
            it.op = to_abi(*op);
        } else {
            // every channel draws one uniform, identity channels included
            // (apply_kraus_trajectory, statevector.cpp:339-386)
            const auto& app = std::get<ChannelApplication>(item);
            if (int(app.qubits.size()) != app.channel.arity)
                throw ContractError("channel arity " + std::to_string(app.channel.arity) + " does not match " +
                                    std::to_string(app.qubits.size()) + " qubits");
            it.type = 1;
            it.nkraus = int32_t(app.channel.kraus.size());
            it.kraus_offset = int64_t(pool.size() / 2);
            it.op.nqubits = int32_t(app.qubits.size());
            for (size_t j = 0; j < app.qubits.size(); ++j) it.op.qubits[j] = app.qubits[j];
            for (const auto& K : app.channel.kraus) {
                auto f = flatten(K);
                pool.insert(pool.end(), f.begin(), f.end());
            }
            ++nch;
        }
        items.push_back(it);
    }
    std::vector<double> u(size_t(ntraj) * nch);
    for (auto& x : u) x = rng.next_double();
    std::vector<uint64_t> flip, signs;
    std::vector<int32_t> ny;
    std::vector<double> coeff;
    for (const auto& p : observables) {
        if (p.n != n)
            throw ContractError("Pauli string length " + std::to_string(p.n) + " does not match state qubit count " +
                                std::to_string(n));
        const PauliMasks m = masks_of(p);
        flip.push_back(m.flip);
        signs.push_back(m.signs);
        ny.push_back(m.ny);
        coeff.push_back(p.coefficient);
    }
    std::vector<double> flat(size_t(ntraj) * observables.size());
    check(nq_traj_run(n, items.data(), int64_t(items.size()), pool.empty() ? nullptr : pool.data(), int64_t(ntraj),
                      u.data(), flip.data(), signs.data(), ny.data(), coeff.data(), int(observables.size()),
                      flat.data(), nullptr, nullptr, -1));
    std::vector<std::vector<double>> out{static_cast<size_t>(ntraj)};
    for (size_t t = 0; t < size_t(ntraj); ++t)
        out[t].assign(flat.begin() + long(t * observables.size()), flat.begin() + long((t + 1) * observables.size()));
    return out;
}

std::vector<std::vector<double>> batch_expectations(const std::vector<Circuit>& circuits,
                                                    const std::vector<PauliString>& observables) {
    if (circuits.empty()) return {};
    const int n = circuits.front().num_qubits();
    std::vector<nq_sched_item> items;
    std::vector<int64_t> off{0};
    for (const auto& c : circuits) {
        if (c.num_qubits() != n) throw ContractError("batched circuits must have the same qubit count");
        for (const auto& op : c.ops()) {
            nq_sched_item it{};
            it.type = 0;
            it.op = to_abi(op);
            items.push_back(it);
        }
        off.push_back(int64_t(items.size()));
    }
    std::vector<uint64_t> flip, signs;
    std::vector<int32_t> ny;
    std::vector<double> coeff;
    for (const auto& p : observables) {
        if (p.n != n)
            throw ContractError("Pauli string length " + std::to_string(p.n) + " does not match state qubit count " +
                                std::to_string(n));
        const PauliMasks m = masks_of(p);
        flip.push_back(m.flip);
        signs.push_back(m.signs);
        ny.push_back(m.ny);
        coeff.push_back(p.coefficient);
    }
    const size_t B = circuits.size(), T = observables.size();
    std::vector<double> flat(B * T);
    check(nq_batch_run(n, 0, int64_t(B), off.data(), items.data(), nullptr, flip.data(), signs.data(), ny.data(),
                       coeff.data(), int(T), flat.data(), nullptr, nullptr, -1));
    std::vector<std::vector<double>> out{B};
    for (size_t b = 0; b < B; ++b) out[b].assign(flat.begin() + long(b * T), flat.begin() + long((b + 1) * T));
    return out;
}

std::vector<std::vector<double>> batch_noisy_distributions(const std::vector<Circuit>& circuits,
                                                           const DeviceNoiseModel& m) {
    if (circuits.empty()) return {};
    const auto t_start = std::chrono::steady_clock::now();
    const int n = circuits.front().num_qubits();
    if (n > m.num_qubits())
        throw ContractError("device model covers " + std::to_string(m.num_qubits()) + " qubits, circuit needs " +
                            std::to_string(n));
    std::vector<nq_sched_item> items;
    std::vector<double> pool;
    std::vector<int64_t> off{0};
    // attach_noise (noise.cpp:383-426) without materialising the schedule: the
    // channels of a gate depend only on (kind, qubits), so each distinct pair
    // is built, validated and flattened once.
    struct Chan {
        int64_t at;  // pool offset (complex elements); -1: identity channel (skipped)
        int32_t nkraus;
        int q[2];
        int k;
    };
    std::map<std::tuple<int, int, int>, std::vector<Chan>> memo;
    auto add_channel = [&](const KrausChannel& ch, const std::vector<int>& qs, std::vector<Chan>& out) {
        validate_channel(ch);
        Chan c{-1, int32_t(ch.kraus.size()), {qs[0], qs.size() > 1 ? qs[1] : -1}, int(qs.size())};
        if (!ch.is_identity()) {
            c.at = int64_t(pool.size() / 2);
            for (const auto& K : ch.kraus) {
                auto f = flatten(K);
                pool.insert(pool.end(), f.begin(), f.end());
            }
        }
        out.push_back(c);
    };
    for (const auto& circ : circuits) {
        if (circ.num_qubits() != n) throw ContractError("batched circuits must have the same qubit count");
        for (const auto& op : circ.ops()) {
            if (!gate_is_unitary(op.kind)) continue;  // unitaries_only()
            nq_sched_item it{};
            it.type = 0;
            it.op = to_abi(op);
            items.push_back(it);
            const int arity = int(op.qubits.size());
            if (arity > 2)
                throw ContractError("no noise channel for " + std::string(gate_name(op.kind)) +
                                    ": gates on more than 2 qubits are not calibratable");
            const auto key = std::make_tuple(int(op.kind), op.qubits[0], arity == 2 ? op.qubits[1] : -1);
            auto f = memo.find(key);
            if (f == memo.end()) {
                const auto gp = m.find_gate(gate_name(op.kind), op.qubits);
                if (!gp)
                    throw ContractError("no calibration entry or default for gate '" + std::string(gate_name(op.kind)) +
                                        "' on qubits [" + std::to_string(op.qubits[0]) +
                                        (arity == 2 ? "," + std::to_string(op.qubits[1]) : "") + "]");
                std::vector<Chan> chans;
                add_channel(depolarizing(gp->error, arity), op.qubits, chans);
                for (int q : op.qubits) {
                    const auto& qp = m.qubits[size_t(q)];
                    add_channel(thermal_relaxation(qp.t1_us, qp.t2_us, gp->duration_ns), {q}, chans);
                }
                f = memo.emplace(key, std::move(chans)).first;
            }
            for (const Chan& c : f->second) {
                if (c.at < 0) continue;
                nq_sched_item ci{};
                ci.type = 1;
                ci.nkraus = c.nkraus;
                ci.kraus_offset = c.at;
                ci.op.nqubits = c.k;
                for (int j = 0; j < c.k; ++j) ci.op.qubits[j] = c.q[j];
                items.push_back(ci);
            }
        }
        off.push_back(int64_t(items.size()));
    }
    ReadoutModel readout = m.readout();
    readout.qubits.resize(size_t(n));
    const size_t B = circuits.size(), dq = size_t(1) << n;
    std::vector<double> probs(B * dq);
    const auto t_host = std::chrono::steady_clock::now();
    check(nq_batch_run(n, 1, int64_t(B), off.data(), items.data(), pool.empty() ? nullptr : pool.data(), nullptr,
                       nullptr, nullptr, nullptr, 0, nullptr, nullptr, probs.data(), -1));
    if (std::getenv("NQ_BATCH_TIMING"))
        std::fprintf(stderr, "[batch dm] schedules %.2f ms, nq_batch_run %.2f ms, %zu items\n",
                     std::chrono::duration<double, std::milli>(t_host - t_start).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host).count(),
                     items.size());
    std::vector<std::vector<double>> out;
    out.reserve(B);
    for (size_t b = 0; b < B; ++b)
        out.push_back(readout_apply_dist(
            std::vector<double>(probs.begin() + long(b * dq), probs.begin() + long((b + 1) * dq)), readout));
    return out;
}

void DensityMatrix::run_schedule(const NoisySchedule& schedule) {
    if (schedule.num_qubits != n_) throw ContractError("schedule qubit count mismatch");
    std::vector<nq_sched_item> items;
    std::vector<double> pool;
    items.reserve(schedule.items.size());
    for (const auto& item : schedule.items) {
        nq_sched_item it{};
        if (const auto* op = std::get_if<GateOp>(&item)) {
            if (op->kind == GateKind::MEASURE || op->kind == GateKind::BARRIER) continue;
            it.type = 0;
            it.op = to_abi(*op);
        } else {
            const auto& app = std::get<ChannelApplication>(item);
            if (int(app.qubits.size()) != app.channel.arity)
                throw ContractError("channel arity " + std::to_string(app.channel.arity) + " does not match " +
                                    std::to_string(app.qubits.size()) + " qubits");
            for (int q : app.qubits)
                if (q < 0 || q >= n_) throw ContractError("qubit index " + std::to_string(q) + " out of range");
            validate_channel(app.channel);
            if (app.channel.is_identity()) continue;
            it.type = 1;
            it.nkraus = int32_t(app.channel.kraus.size());
            it.kraus_offset = int64_t(pool.size() / 2);
            it.op.nqubits = int32_t(app.qubits.size());
            for (size_t j = 0; j < app.qubits.size(); ++j) it.op.qubits[j] = app.qubits[j];
            for (const auto& K : app.channel.kraus) {
                auto f = flatten(K);
                pool.insert(pool.end(), f.begin(), f.end());
            }
        }
        items.push_back(it);
    }
    check(nq_dm_apply_schedule(h_, items.data(), int64_t(items.size()), pool.data()));
    mirror_ok_ = false;
}

double DensityMatrix::trace() const {
    double v = 0.0;
    check(nq_dm_trace(h_, &v));
    return v;
}

double DensityMatrix::purity() const {
    double v = 0.0;
    check(nq_dm_purity(h_, &v));
    return v;
}

double DensityMatrix::hermiticity_residual() const {
    double v = 0.0;
    check(nq_dm_hermiticity_residual(h_, &v));
    return v;
}

double DensityMatrix::expectation(const PauliString& p) const {
    if (p.n != n_) throw ContractError("Pauli string length does not match qubit count");
    return expectations({p})[0];
}

std::vector<double> DensityMatrix::expectations(const std::vector<PauliString>& terms) const {
    std::vector<uint64_t> flip, signs;
    std::vector<int32_t> ny;
    std::vector<double> coeff;
    for (const auto& p : terms) {
        if (p.n != n_) throw ContractError("Pauli string length does not match qubit count");
        const PauliMasks m = masks_of(p);
        flip.push_back(m.flip);
        signs.push_back(m.signs);
        ny.push_back(m.ny);
        coeff.push_back(p.coefficient);
    }
    std::vector<double> re(terms.size()), im(terms.size());
    if (!terms.empty())
        check(nq_dm_expectation_batch(h_, flip.data(), signs.data(), ny.data(), coeff.data(), int(terms.size()),
                                      re.data(), im.data()));
    for (double v : im)
        if (std::abs(v) > 1e-8) throw ContractError("Pauli expectation has non-real residue " + std::to_string(v));
    return re;
}

std::vector<double> DensityMatrix::probabilities() const {
    std::vector<double> p(dim());
    check(nq_dm_probabilities(h_, p.data()));
    return p;
}

DensityMatrix dm_run_noisy(const Circuit& c, const DeviceNoiseModel& m) {
    DensityMatrix d(c.num_qubits());
    d.run_schedule(attach_noise(c, m));
    return d;
}

} // namespace naqs

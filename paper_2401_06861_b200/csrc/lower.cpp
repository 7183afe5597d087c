// Lowering of reference-level operations into planner elementary ops.
//
//  * SV: one GateOp -> one elementary op on the state bits (kind dispatch of
//    proj/src/statevector.cpp:90-180: X / CX / CCX / SWAP are permutations,
//    the Z/S/SDG/T/TDG/RZ/U1 family and CZ are diagonals, the rest dense 2x2).
//  * DM: rho is stored row-major, so vec(rho) index = r * 2^n + c: column bits
//    are state bits 0..n-1 and row bits n..2n-1.  rho -> K rho K^dagger acts
//    as K on the row bits and conj(K) on the column bits, i.e. a channel on
//    qubits qs is the 2k-bit operator S = sum_K kron(K, conj K) on the bit list
//    [qs..., qs+n...] (column bits low).  This reproduces
//    apply_operators_blockwise (proj/src/densitymatrix.cpp:60-110) exactly in
//    exact arithmetic; see SURVEY.md Appendix A.5.
#include "lower.hpp"

#include <cmath>
#include <stdexcept>

namespace nqe {

namespace {
constexpr cplx kI{0.0, 1.0};
}

bool gate_is_diagonal(int kind) {
    switch (kind) {
    case NQ_Z: case NQ_S: case NQ_SDG: case NQ_T: case NQ_TDG: case NQ_RZ: case NQ_U1:
    case NQ_ID: case NQ_CZ:
        return true;
    default:
        return false;
    }
}

// Gate matrices of proj/src/gates.cpp:51-110 (OpenQASM 2.0 u3 convention,
// SURVEY.md A.2), evaluated with the same expression forms so that unfused
// application is bit-identical to the reference.
void gate_matrix_2x2(int kind, const double* params, cplx out[4]) {
    auto set = [&](cplx a, cplx b, cplx c, cplx d) {
        out[0] = a; out[1] = b; out[2] = c; out[3] = d;
    };
    auto u3 = [&](double theta, double phi, double lambda) {
        const double c = std::cos(theta / 2.0);
        const double s = std::sin(theta / 2.0);
        set(c, -std::exp(kI * lambda) * s, std::exp(kI * phi) * s, std::exp(kI * (phi + lambda)) * c);
    };
    const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
    switch (kind) {
    case NQ_ID: set(1, 0, 0, 1); break;
    case NQ_X: set(0, 1, 1, 0); break;
    case NQ_Y: set(0, -kI, kI, 0); break;
    case NQ_Z: set(1, 0, 0, -1); break;
    case NQ_H: set(inv_sqrt2, inv_sqrt2, inv_sqrt2, -inv_sqrt2); break;
    case NQ_S: set(1, 0, 0, kI); break;
    case NQ_SDG: set(1, 0, 0, -kI); break;
    case NQ_T: set(1, 0, 0, std::exp(kI * (M_PI / 4.0))); break;
    case NQ_TDG: set(1, 0, 0, std::exp(-kI * (M_PI / 4.0))); break;
    case NQ_RX: {
        const double c = std::cos(params[0] / 2.0), s = std::sin(params[0] / 2.0);
        set(c, -kI * s, -kI * s, c);
        break;
    }
    case NQ_RY: {
        const double c = std::cos(params[0] / 2.0), s = std::sin(params[0] / 2.0);
        set(c, -s, s, c);
        break;
    }
    case NQ_RZ:
        set(std::exp(-kI * (params[0] / 2.0)), 0, 0, std::exp(kI * (params[0] / 2.0)));
        break;
    case NQ_U1: set(1, 0, 0, std::exp(kI * params[0])); break;
    case NQ_U2: u3(M_PI / 2.0, params[0], params[1]); break;
    case NQ_U3: u3(params[0], params[1], params[2]); break;
    default: throw std::logic_error("gate_matrix_2x2: not a one-qubit kind");
    }
}

int kind_arity(int kind) {
    switch (kind) {
    case NQ_CX: case NQ_CZ: case NQ_SWAP: return 2;
    case NQ_CCX: return 3;
    default: return 1;
    }
}

int kind_params(int kind) {
    switch (kind) {
    case NQ_RX: case NQ_RY: case NQ_RZ: case NQ_U1: return 1;
    case NQ_U2: return 2;
    case NQ_U3: return 3;
    default: return 0;
    }
}

// Full 2^k x 2^k matrix of any unitary kind, local bit j <-> qubits[j]
// (proj/src/gates.cpp:26-47: CX control = bit 0, CCX controls = bits 0, 1).
std::vector<cplx> full_gate_matrix(const nq_op& op) {
    const int k = kind_arity(op.kind);
    const int d = 1 << k;
    std::vector<cplx> m(size_t(d) * d, cplx(0.0, 0.0));
    auto at = [&](int r, int c) -> cplx& { return m[size_t(r) * d + c]; };
    switch (op.kind) {
    case NQ_CX:
        for (int c = 0; c < 4; ++c) at((c & 1) ? c ^ 2 : c, c) = 1.0;
        break;
    case NQ_CZ:
        for (int c = 0; c < 4; ++c) at(c, c) = c == 3 ? -1.0 : 1.0;
        break;
    case NQ_SWAP:
        for (int c = 0; c < 4; ++c) at(((c & 1) << 1) | (c >> 1), c) = 1.0;
        break;
    case NQ_CCX:
        for (int c = 0; c < 8; ++c) at((c & 3) == 3 ? c ^ 4 : c, c) = 1.0;
        break;
    default: {
        cplx g[4];
        gate_matrix_2x2(op.kind, op.params, g);
        m.assign(g, g + 4);
    }
    }
    return m;
}

// ---- state vector ------------------------------------------------------------
void lower_sv_op(const nq_op& op, std::vector<EOp>& out) {
    EOp e;
    const int* q = op.qubits;
    switch (op.kind) {
    case NQ_BARRIER:
        return;
    case NQ_ID:
        e.type = E_NOP;
        break;
    case NQ_X:
        e.type = E_XPERM; e.k = 1; e.bits[0] = q[0];
        break;
    case NQ_CX:
        e.type = E_XPERM; e.k = 1; e.bits[0] = q[1]; e.ctrl = uint64_t(1) << q[0];
        break;
    case NQ_CCX:
        e.type = E_XPERM; e.k = 1; e.bits[0] = q[2];
        e.ctrl = (uint64_t(1) << q[0]) | (uint64_t(1) << q[1]);
        break;
    case NQ_SWAP:
        e.type = E_SWAP; e.k = 2; e.bits[0] = q[0]; e.bits[1] = q[1];
        break;
    case NQ_CZ:
        e.type = E_DIAG; e.k = 2; e.bits[0] = q[0]; e.bits[1] = q[1];
        e.mat = {cplx(1, 0), cplx(1, 0), cplx(1, 0), cplx(-1, 0)};
        break;
    default: {
        cplx m[4];
        gate_matrix_2x2(op.kind, op.params, m);
        e.k = 1; e.bits[0] = q[0];
        if (gate_is_diagonal(op.kind)) {
            e.type = E_DIAG;
            e.mat = {m[0], m[3]};
        } else {
            e.type = E_DENSE;
            e.mat.assign(m, m + 4);
        }
    }
    }
    out.push_back(std::move(e));
}

EOp sv_matrix_op(const int* qubits, int k, const cplx* mat) {
    EOp e;
    e.type = E_DENSE;
    e.k = k;
    for (int j = 0; j < k; ++j) e.bits[j] = qubits[j];
    e.mat.assign(mat, mat + (size_t(1) << (2 * k)));
    e.src = 0;
    return e;
}

// ---- density matrix ------------------------------------------------------------
// Superoperator of a unitary / Kraus set on k qubits: 2k bits [qs, qs+n],
// S[(c,r),(c',r')] = sum_K K[r][r'] * conj(K[c][c']), local index l = c + 2^k r.
std::vector<cplx> superop(int k, const std::vector<const cplx*>& kraus) {
    const int d = 1 << k;
    const int D = d * d;
    std::vector<cplx> s(size_t(D) * D, cplx(0.0, 0.0));
    for (const cplx* K : kraus) {
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c)
                for (int rp = 0; rp < d; ++rp)
                    for (int cp = 0; cp < d; ++cp) {
                        const cplx v = K[r * d + rp] * std::conj(K[c * d + cp]);
                        s[size_t(c + d * r) * D + size_t(cp + d * rp)] += v;
                    }
    }
    return s;
}

// Does S equal a*I + b*Pi with Pi[(c,r),(c',r')] = [c==r][c'==r']?
bool depol_form(int k, const std::vector<cplx>& s, double* a, double* b) {
    const int d = 1 << k;
    const int D = d * d;
    // b from an off-diagonal Pi entry: (c=r=0) <- (c'=r'=1)
    const cplx bb = s[size_t(0) * D + size_t(1 + d * 1)];
    const cplx aa = s[0] - bb;
    if (std::abs(aa.imag()) > 1e-15 || std::abs(bb.imag()) > 1e-15) return false;
    const double tol = 1e-14;
    for (int l = 0; l < D; ++l) {
        const int c = l % d, r = l / d;
        for (int lp = 0; lp < D; ++lp) {
            const int cp = lp % d, rp = lp / d;
            cplx want(0.0, 0.0);
            if (l == lp) want += aa;
            if (c == r && cp == rp) want += bb;
            if (std::abs(s[size_t(l) * D + lp] - want) > tol) return false;
        }
    }
    *a = aa.real();
    *b = bb.real();
    return true;
}

void lower_dm_op(const nq_op& op, int n, std::vector<EOp>& out) {
    const int* q = op.qubits;
    auto perm_pair = [&](EOp e) {
        // row copy first (carries the source count), then the column copy
        EOp row = e;
        row.bits[0] += n;
        if (row.type == E_SWAP) row.bits[1] += n;
        uint64_t rc = 0;
        for (int b = 0; b < 64; ++b)
            if ((e.ctrl >> b) & 1) rc |= uint64_t(1) << (b + n);
        row.ctrl = rc;
        e.src = 0;
        row.pair_next = true;
        out.push_back(row);
        out.push_back(e);
    };
    switch (op.kind) {
    case NQ_BARRIER:
        return;
    case NQ_ID: {
        EOp e;
        e.type = E_NOP;
        out.push_back(e);
        return;
    }
    case NQ_X: case NQ_CX: case NQ_CCX: case NQ_SWAP: {
        std::vector<EOp> tmp;
        lower_sv_op(op, tmp);
        perm_pair(tmp[0]);
        return;
    }
    case NQ_CZ: {
        EOp e;
        e.type = E_DIAG; e.k = 4;
        e.bits[0] = q[0]; e.bits[1] = q[1]; e.bits[2] = q[0] + n; e.bits[3] = q[1] + n;
        e.mat.resize(16);
        const double dz[4] = {1, 1, 1, -1};
        for (int l = 0; l < 16; ++l) e.mat[size_t(l)] = cplx(dz[l & 3] * dz[l >> 2], 0.0);
        out.push_back(std::move(e));
        return;
    }
    default: {
        cplx m[4];
        gate_matrix_2x2(op.kind, op.params, m);
        EOp e;
        e.k = 2;
        e.bits[0] = q[0];
        e.bits[1] = q[0] + n;
        if (gate_is_diagonal(op.kind)) {
            e.type = E_DIAG;
            const cplx d[2] = {m[0], m[3]};
            e.mat.resize(4);
            for (int l = 0; l < 4; ++l) e.mat[size_t(l)] = d[l >> 1] * std::conj(d[l & 1]);
        } else {
            e.type = E_DENSE;
            const cplx* ks[1] = {m};
            e.mat = superop(1, std::vector<const cplx*>(ks, ks + 1));
        }
        out.push_back(std::move(e));
    }
    }
}

EOp dm_channel_op(const int* qubits, int k, int nkraus, const cplx* kraus, int n) {
    const int d = 1 << k;
    std::vector<const cplx*> ks;
    for (int i = 0; i < nkraus; ++i) ks.push_back(kraus + size_t(i) * d * d);
    std::vector<cplx> s = superop(k, ks);
    EOp e;
    e.src = 0;
    e.k = 2 * k;
    for (int j = 0; j < k; ++j) {
        e.bits[j] = qubits[j];
        e.bits[j + k] = qubits[j] + n;
    }
    double a = 0, b = 0;
    if (k == 2 && depol_form(k, s, &a, &b)) {
        e.type = E_DEPOL;
        e.mat = {cplx(a, 0.0), cplx(b, 0.0)};
    } else {
        e.type = E_DENSE;
        e.mat = std::move(s);
    }
    return e;
}

}  // namespace nqe

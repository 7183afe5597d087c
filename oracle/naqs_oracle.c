/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference hot path.
 * See naqs_oracle.h for scope and pinning.  The arithmetic follows the
 * reference expression by expression (same operand order, same chunked
 * reductions), so on the same host it reproduces the reference bit for bit
 * (tests/test_oracle_golden.py checks this against oracle/_ref).
 */
#include "naqs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { K_X, K_Y, K_Z, K_H, K_S, K_SDG, K_T, K_TDG, K_ID, K_RX, K_RY, K_RZ, K_U1, K_U2, K_U3,
       K_CX, K_CZ, K_SWAP, K_CCX, K_MEASURE, K_BARRIER };

/* ---- rng.hpp:12-61 (xoshiro256++ seeded by SplitMix64) ---------------------- */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
void or_rng_init(uint64_t* s, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9E3779B97F4A7C15ULL;
        s[i] = mix64(x);
    }
}
static uint64_t rng_next(uint64_t* s) {
    const uint64_t r = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return r;
}
double or_rng_next_double(uint64_t* s) { return (double)(rng_next(s) >> 11) * 0x1.0p-53; }
void or_rng_u64(uint64_t seed, int count, uint64_t* out) {
    uint64_t s[4];
    or_rng_init(s, seed);
    for (int i = 0; i < count; ++i) out[i] = rng_next(s);
}
void or_rng_double(uint64_t seed, int count, double* out) {
    uint64_t s[4];
    or_rng_init(s, seed);
    for (int i = 0; i < count; ++i) out[i] = or_rng_next_double(s);
}
uint64_t or_derive_seed(uint64_t base, uint64_t stream) { return mix64(base + 0x9E3779B97F4A7C15ULL * (stream + 1)); }

static int arity_of(int k) { return (k == K_CX || k == K_CZ || k == K_SWAP) ? 2 : (k == K_CCX ? 3 : 1); }
static int nparams_of(int k) {
    return (k == K_RX || k == K_RY || k == K_RZ || k == K_U1) ? 1 : k == K_U2 ? 2 : k == K_U3 ? 3 : 0;
}

/* ---- tests/test_util.hpp:59-86 ---------------------------------------------- */
int or_random_circuit(uint64_t seed, int n, int depth, int max_arity, or_op* out) {
    static const int pool[19] = {K_X, K_Y, K_Z, K_H, K_S, K_SDG, K_T, K_TDG, K_ID, K_RX,
                                 K_RY, K_RZ, K_U1, K_U2, K_U3, K_CX, K_CZ, K_SWAP, K_CCX};
    uint64_t s[4];
    or_rng_init(s, seed);
    for (int d = 0; d < depth; ++d) {
        int kind;
        do {
            kind = pool[rng_next(s) % 19u];
        } while (arity_of(kind) > n || arity_of(kind) > max_arity);
        or_op* o = &out[d];
        memset(o, 0, sizeof(*o));
        o->kind = kind;
        int cnt = 0;
        while (cnt < arity_of(kind)) {
            const int q = (int)(rng_next(s) % (uint64_t)n);
            int dup = 0;
            for (int j = 0; j < cnt; ++j) dup = dup || o->qubits[j] == q;
            if (!dup) o->qubits[cnt++] = q;
        }
        o->nqubits = cnt;
        for (int p = 0; p < nparams_of(kind); ++p) {
            const double lo = -2.0 * M_PI, hi = 2.0 * M_PI;
            o->params[p] = lo + (hi - lo) * or_rng_next_double(s);
        }
    }
    return 0;
}

/* ---- gates.cpp:19-110 -------------------------------------------------------- */
static void set2(double complex* m, double complex a, double complex b, double complex c, double complex d) {
    m[0] = a; m[1] = b; m[2] = c; m[3] = d;
}
static double complex cexpi(double x) { return cexp(I * x); }
static void u3m(double complex* m, double th, double ph, double la) {
    const double c = cos(th / 2.0), s = sin(th / 2.0);
    set2(m, c, -cexpi(la) * s, cexpi(ph) * s, cexpi(ph + la) * c);
}
int or_gate_matrix(const or_op* op, double complex* m) {
    const double r = 1.0 / sqrt(2.0);
    const double* p = op->params;
    int d;
    switch (op->kind) {
    case K_ID: set2(m, 1, 0, 0, 1); return 2;
    case K_X: set2(m, 0, 1, 1, 0); return 2;
    case K_Y: set2(m, 0, -I, I, 0); return 2;
    case K_Z: set2(m, 1, 0, 0, -1); return 2;
    case K_H: set2(m, r, r, r, -r); return 2;
    case K_S: set2(m, 1, 0, 0, I); return 2;
    case K_SDG: set2(m, 1, 0, 0, -I); return 2;
    case K_T: set2(m, 1, 0, 0, cexpi(M_PI / 4.0)); return 2;
    case K_TDG: set2(m, 1, 0, 0, cexp(-I * (M_PI / 4.0))); return 2;
    case K_RX: {
        const double c = cos(p[0] / 2.0), s = sin(p[0] / 2.0);
        set2(m, c, -I * s, -I * s, c);
        return 2;
    }
    case K_RY: {
        const double c = cos(p[0] / 2.0), s = sin(p[0] / 2.0);
        set2(m, c, -s, s, c);
        return 2;
    }
    case K_RZ: set2(m, cexp(-I * (p[0] / 2.0)), 0, 0, cexpi(p[0] / 2.0)); return 2;
    case K_U1: set2(m, 1, 0, 0, cexpi(p[0])); return 2;
    case K_U2: u3m(m, M_PI / 2.0, p[0], p[1]); return 2;
    case K_U3: u3m(m, p[0], p[1], p[2]); return 2;
    case K_CX: case K_CZ: case K_SWAP: case K_CCX:
        d = op->kind == K_CCX ? 8 : 4;
        for (int i = 0; i < d * d; ++i) m[i] = 0;
        for (int i = 0; i < d; ++i) m[i * d + i] = 1;
        if (op->kind == K_CX) { m[1 * 4 + 1] = 0; m[3 * 4 + 3] = 0; m[1 * 4 + 3] = 1; m[3 * 4 + 1] = 1; }
        if (op->kind == K_CZ) m[15] = -1;
        if (op->kind == K_SWAP) { m[1 * 4 + 1] = 0; m[2 * 4 + 2] = 0; m[1 * 4 + 2] = 1; m[2 * 4 + 1] = 1; }
        if (op->kind == K_CCX) { m[3 * 8 + 3] = 0; m[7 * 8 + 7] = 0; m[3 * 8 + 7] = 1; m[7 * 8 + 3] = 1; }
        return d;
    default: return -1;
    }
}

/* ---- statevector.cpp:17-40 ---------------------------------------------------- */
static void sort_ints(int* a, int k) {
    for (int i = 1; i < k; ++i)
        for (int j = i; j > 0 && a[j - 1] > a[j]; --j) {
            const int t = a[j];
            a[j] = a[j - 1];
            a[j - 1] = t;
        }
}
static uint64_t expand_index(uint64_t rest, const int* sorted, int k) {
    uint64_t idx = rest;
    for (int j = 0; j < k; ++j) {
        const int q = sorted[j];
        const uint64_t low = idx & ((UINT64_C(1) << q) - 1);
        idx = ((idx >> q) << (q + 1)) | low;
    }
    return idx;
}
static void local_offsets(const int* qubits, int k, uint64_t* off) {
    for (int b = 0; b < (1 << k); ++b) {
        uint64_t v = 0;
        for (int j = 0; j < k; ++j)
            if ((b >> j) & 1) v |= UINT64_C(1) << qubits[j];
        off[b] = v;
    }
}

/* statevector.cpp:50-88 */
void or_sv_apply_matrix(double complex* amps, int n, const int* qubits, int k, const double complex* u) {
    const uint64_t dim = UINT64_C(1) << n;
    int sorted[4];
    uint64_t off[16];
    memcpy(sorted, qubits, sizeof(int) * (size_t)k);
    sort_ints(sorted, k);
    local_offsets(qubits, k, off);
    if (k == 1) {
        const double complex u00 = u[0], u01 = u[1], u10 = u[2], u11 = u[3];
        const uint64_t stride = off[1];
        const int q = sorted[0];
        for (uint64_t r = 0; r < (dim >> 1); ++r) {
            const uint64_t low = r & ((UINT64_C(1) << q) - 1);
            const uint64_t base = ((r >> q) << (q + 1)) | low;
            const double complex a0 = amps[base], a1 = amps[base + stride];
            amps[base] = u00 * a0 + u01 * a1;
            amps[base + stride] = u10 * a0 + u11 * a1;
        }
        return;
    }
    const int block = 1 << k;
    for (uint64_t r = 0; r < (dim >> k); ++r) {
        const uint64_t base = expand_index(r, sorted, k);
        double complex v[16], w[16];
        for (int b = 0; b < block; ++b) v[b] = amps[base + off[b]];
        for (int row = 0; row < block; ++row) {
            double complex acc = 0;
            for (int col = 0; col < block; ++col) acc += u[row * block + col] * v[col];
            w[row] = acc;
        }
        for (int b = 0; b < block; ++b) amps[base + off[b]] = w[b];
    }
}

/* statevector.cpp:90-180 */
static void sv_gate(double complex* amps, int n, const or_op* op) {
    const uint64_t dim = UINT64_C(1) << n;
    int sorted[3];
    const int k = op->nqubits;
    memcpy(sorted, op->qubits, sizeof(int) * (size_t)k);
    sort_ints(sorted, k);
    switch (op->kind) {
    case K_ID: return;
    case K_X: {
        const int q = op->qubits[0];
        const uint64_t bit = UINT64_C(1) << q;
        for (uint64_t r = 0; r < (dim >> 1); ++r) {
            const uint64_t base = ((r >> q) << (q + 1)) | (r & (bit - 1));
            const double complex t = amps[base];
            amps[base] = amps[base + bit];
            amps[base + bit] = t;
        }
        return;
    }
    case K_Z: case K_S: case K_SDG: case K_T: case K_TDG: case K_RZ: case K_U1: {
        double complex u[4];
        or_gate_matrix(op, u);
        const double complex d0 = u[0], d1 = u[3];
        const uint64_t bit = UINT64_C(1) << op->qubits[0];
        for (uint64_t i = 0; i < dim; ++i) amps[i] *= (i & bit) ? d1 : d0;
        return;
    }
    case K_CX: {
        const uint64_t cb = UINT64_C(1) << op->qubits[0], tb = UINT64_C(1) << op->qubits[1];
        for (uint64_t r = 0; r < (dim >> 2); ++r) {
            const uint64_t base = expand_index(r, sorted, 2) | cb;
            const double complex t = amps[base];
            amps[base] = amps[base | tb];
            amps[base | tb] = t;
        }
        return;
    }
    case K_CZ: {
        const uint64_t mask = (UINT64_C(1) << op->qubits[0]) | (UINT64_C(1) << op->qubits[1]);
        for (uint64_t r = 0; r < (dim >> 2); ++r) {
            const uint64_t idx = expand_index(r, sorted, 2) | mask;
            amps[idx] = -amps[idx];
        }
        return;
    }
    case K_SWAP: {
        const uint64_t b0 = UINT64_C(1) << op->qubits[0], b1 = UINT64_C(1) << op->qubits[1];
        for (uint64_t r = 0; r < (dim >> 2); ++r) {
            const uint64_t base = expand_index(r, sorted, 2);
            const double complex t = amps[base | b0];
            amps[base | b0] = amps[base | b1];
            amps[base | b1] = t;
        }
        return;
    }
    case K_CCX: {
        const uint64_t c0 = UINT64_C(1) << op->qubits[0], c1 = UINT64_C(1) << op->qubits[1];
        const uint64_t tb = UINT64_C(1) << op->qubits[2];
        for (uint64_t r = 0; r < (dim >> 3); ++r) {
            const uint64_t base = expand_index(r, sorted, 3) | c0 | c1;
            const double complex t = amps[base];
            amps[base] = amps[base | tb];
            amps[base | tb] = t;
        }
        return;
    }
    default: {
        double complex u[4];
        or_gate_matrix(op, u);
        or_sv_apply_matrix(amps, n, op->qubits, 1, u);
    }
    }
}

int or_sv_apply(double complex* amps, int n, const or_op* ops, int64_t nops) {
    for (int64_t i = 0; i < nops; ++i) {
        if (ops[i].kind == K_BARRIER) continue;
        if (ops[i].kind == K_MEASURE) return -1;
        sv_gate(amps, n, &ops[i]);
    }
    return 0;
}

/* statevector.cpp:224-239: 4096-element chunks combined in chunk order */
#define REDUCE_CHUNK 4096u
double or_sv_norm_sq(const double complex* a, int n) {
    const uint64_t dim = UINT64_C(1) << n;
    double total = 0.0;
    for (uint64_t lo = 0; lo < dim; lo += REDUCE_CHUNK) {
        const uint64_t hi = lo + REDUCE_CHUNK < dim ? lo + REDUCE_CHUNK : dim;
        double acc = 0.0;
        for (uint64_t i = lo; i < hi; ++i) acc += creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]);
        total += acc;
    }
    return total;
}

static void masks(const char* L, int n, uint64_t* flip, uint64_t* signs, int* ny) {
    *flip = *signs = 0;
    *ny = 0;
    for (int i = 0; i < n; ++i) {
        if (L[i] == 'X') *flip |= UINT64_C(1) << i;
        if (L[i] == 'Y') {
            *flip |= UINT64_C(1) << i;
            *signs |= UINT64_C(1) << i;
            ++*ny;
        }
        if (L[i] == 'Z') *signs |= UINT64_C(1) << i;
    }
}
static const double complex kIPow[4] = {1, I, -1, -I};

/* statevector.cpp:241-277 */
double or_sv_expectation(const double complex* a, int n, const char* letters, double coeff) {
    uint64_t flip, signs;
    int ny;
    masks(letters, n, &flip, &signs, &ny);
    const uint64_t dim = UINT64_C(1) << n;
    double complex total = 0;
    for (uint64_t lo = 0; lo < dim; lo += REDUCE_CHUNK) {
        const uint64_t hi = lo + REDUCE_CHUNK < dim ? lo + REDUCE_CHUNK : dim;
        double complex acc = 0;
        for (uint64_t y = lo; y < hi; ++y) {
            const double sgn = (__builtin_popcountll(y & signs) & 1) ? -1.0 : 1.0;
            acc += sgn * conj(a[y ^ flip]) * a[y];
        }
        total += acc;
    }
    total *= kIPow[ny & 3];
    return coeff * creal(total);
}

void or_sv_probabilities(const double complex* a, int n, double* out) {
    for (uint64_t i = 0; i < (UINT64_C(1) << n); ++i) out[i] = creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]);
}

static int cmp_double(const void* x, const void* y) {
    const double a = *(const double*)x, b = *(const double*)y;
    return (a > b) - (a < b);
}

/* statevector.cpp:293-332 (counts written densely by basis index) */
int or_sample_distribution(const double* dist, int n, uint64_t shots, uint64_t seed, uint64_t* counts) {
    const uint64_t dim = UINT64_C(1) << n;
    memset(counts, 0, dim * sizeof(uint64_t));
    if (shots < 1) return -1;
    double* u = (double*)malloc(shots * sizeof(double));
    if (!u) return -2;
    or_rng_double(seed, (int)shots, u);
    qsort(u, shots, sizeof(double), cmp_double);
    double cum = 0.0;
    uint64_t next = 0;
    for (uint64_t i = 0; i < dim && next < shots; ++i) {
        cum += dist[i];
        while (next < shots && u[next] < cum) {
            ++counts[i];
            ++next;
        }
    }
    if (next < shots) {
        for (uint64_t i = dim; i-- > 0;) {
            if (dist[i] > 0.0) {
                counts[i] += shots - next;
                break;
            }
        }
    }
    free(u);
    return 0;
}

/* statevector.cpp:339-386 */
int or_sv_kraus_trajectory(double complex* amps, int n, const int* qubits, int k, int nk, const double complex* kraus,
                           uint64_t* rng) {
    const uint64_t dim = UINT64_C(1) << n;
    const int block = 1 << k;
    int sorted[4];
    uint64_t off[16];
    memcpy(sorted, qubits, sizeof(int) * (size_t)k);
    sort_ints(sorted, k);
    local_offsets(qubits, k, off);
    double weight[32];
    for (int ki = 0; ki < nk; ++ki) {
        const double complex* m = kraus + (size_t)ki * block * block;
        double acc = 0.0;
        for (uint64_t r = 0; r < (dim >> k); ++r) {
            const uint64_t base = expand_index(r, sorted, k);
            for (int row = 0; row < block; ++row) {
                double complex w = 0;
                for (int col = 0; col < block; ++col) w += m[row * block + col] * amps[base + off[col]];
                acc += creal(w) * creal(w) + cimag(w) * cimag(w);
            }
        }
        weight[ki] = acc;
    }
    double total = 0.0;
    for (int i = 0; i < nk; ++i) total += weight[i];
    if (fabs(total - 1.0) > 1e-8) return -1;
    const double u = or_rng_next_double(rng) * total;
    int chosen = nk - 1;
    double cum = 0.0;
    for (int i = 0; i < nk; ++i) {
        cum += weight[i];
        if (u < cum) {
            chosen = i;
            break;
        }
    }
    or_sv_apply_matrix(amps, n, qubits, k, kraus + (size_t)chosen * block * block);
    const double scale = 1.0 / sqrt(weight[chosen]);
    for (uint64_t i = 0; i < dim; ++i) amps[i] *= scale;
    return chosen;
}

/* ---- densitymatrix.cpp:60-110 ----------------------------------------------- */
void or_dm_apply_operators(double complex* rho, int n, const int* qubits, int k, int nops, const double complex* ops) {
    const uint64_t dim = UINT64_C(1) << n;
    const int block = 1 << k;
    int sorted[4];
    uint64_t off[16];
    memcpy(sorted, qubits, sizeof(int) * (size_t)k);
    sort_ints(sorted, k);
    local_offsets(qubits, k, off);
    const uint64_t rest = dim >> k;
    double complex in[8][8], mid[8][8], out[8][8];
    for (uint64_t rr = 0; rr < rest; ++rr) {
        const uint64_t rb = expand_index(rr, sorted, k);
        for (uint64_t cr = 0; cr < rest; ++cr) {
            const uint64_t cb = expand_index(cr, sorted, k);
            for (int i = 0; i < block; ++i)
                for (int j = 0; j < block; ++j) {
                    in[i][j] = rho[(rb + off[i]) * dim + (cb + off[j])];
                    out[i][j] = 0;
                }
            for (int o = 0; o < nops; ++o) {
                const double complex* m = ops + (size_t)o * block * block;
                for (int i = 0; i < block; ++i)
                    for (int j = 0; j < block; ++j) {
                        double complex acc = 0;
                        for (int l = 0; l < block; ++l) acc += m[i * block + l] * in[l][j];
                        mid[i][j] = acc;
                    }
                for (int i = 0; i < block; ++i)
                    for (int j = 0; j < block; ++j) {
                        double complex acc = 0;
                        for (int l = 0; l < block; ++l) acc += mid[i][l] * conj(m[j * block + l]);
                        out[i][j] += acc;
                    }
            }
            for (int i = 0; i < block; ++i)
                for (int j = 0; j < block; ++j) rho[(rb + off[i]) * dim + (cb + off[j])] = out[i][j];
        }
    }
}

/* densitymatrix.cpp:114-125 (apply) and :142-152 (run) */
int or_dm_apply(double complex* rho, int n, const or_op* ops, int64_t nops) {
    for (int64_t i = 0; i < nops; ++i) {
        const or_op* op = &ops[i];
        if (op->kind == K_BARRIER || op->kind == K_ID) continue;
        if (op->kind == K_MEASURE) return -1;
        double complex m[64];
        or_gate_matrix(op, m);
        or_dm_apply_operators(rho, n, op->qubits, op->nqubits, 1, m);
    }
    return 0;
}

double or_dm_trace(const double complex* rho, int n) {
    const uint64_t dim = UINT64_C(1) << n;
    double t = 0.0;
    for (uint64_t i = 0; i < dim; ++i) t += creal(rho[i * dim + i]);
    return t;
}

double or_dm_purity(const double complex* rho, int n) {
    const uint64_t len = UINT64_C(1) << (2 * n);
    double t = 0.0;
    for (uint64_t i = 0; i < len; ++i) t += creal(rho[i]) * creal(rho[i]) + cimag(rho[i]) * cimag(rho[i]);
    return t;
}

double or_dm_hermiticity(const double complex* rho, int n) {
    const uint64_t dim = UINT64_C(1) << n;
    double worst = 0.0;
    for (uint64_t r = 0; r < dim; ++r)
        for (uint64_t c = r; c < dim; ++c) {
            const double v = cabs(rho[r * dim + c] - conj(rho[c * dim + r]));
            if (v > worst) worst = v;
        }
    return worst;
}

int or_dm_expectation(const double complex* rho, int n, const char* letters, double coeff, double* out) {
    uint64_t flip, signs;
    int ny;
    masks(letters, n, &flip, &signs, &ny);
    const uint64_t dim = UINT64_C(1) << n;
    double complex total = 0;
    for (uint64_t y = 0; y < dim; ++y) {
        const double sgn = (__builtin_popcountll(y & signs) & 1) ? -1.0 : 1.0;
        total += sgn * rho[y * dim + (y ^ flip)];
    }
    total *= kIPow[ny & 3];
    if (fabs(cimag(total)) > 1e-8) return -1;
    *out = coeff * creal(total);
    return 0;
}

void or_dm_probabilities(const double complex* rho, int n, double* out) {
    const uint64_t dim = UINT64_C(1) << n;
    double sum = 0.0;
    for (uint64_t i = 0; i < dim; ++i) {
        const double v = creal(rho[i * dim + i]);
        out[i] = v > 0.0 ? v : 0.0;
        sum += out[i];
    }
    if (sum > 0.0)
        for (uint64_t i = 0; i < dim; ++i) out[i] /= sum;
}

/* ---- noise.cpp:87-170 --------------------------------------------------------- */
static void pauli2(int which, double complex* m) {
    switch (which) {
    case 0: set2(m, 1, 0, 0, 1); break;
    case 1: set2(m, 0, 1, 1, 0); break;
    case 2: set2(m, 0, -I, I, 0); break;
    default: set2(m, 1, 0, 0, -1); break;
    }
}

int or_depolarizing(double p, int arity, double complex* out) {
    const int d = 1 << arity;
    int nk = 0;
    if (p == 0.0) {
        for (int i = 0; i < d * d; ++i) out[i] = 0;
        for (int i = 0; i < d; ++i) out[i * d + i] = 1;
        return 1;
    }
    if (arity == 1) {
        double complex P[2][4];
        if (p < 1.0) {
            pauli2(0, P[0]);
            for (int i = 0; i < 4; ++i) out[nk * 4 + i] = sqrt(1.0 - p) * P[0][i];
            ++nk;
        }
        const double w = sqrt(p / 3.0);
        for (int a = 1; a < 4; ++a) {
            pauli2(a, P[1]);
            for (int i = 0; i < 4; ++i) out[nk * 4 + i] = w * P[1][i];
            ++nk;
        }
        return nk;
    }
    if (p < 1.0) {
        for (int i = 0; i < 16; ++i) out[i] = 0;
        for (int i = 0; i < 4; ++i) out[i * 4 + i] = sqrt(1.0 - p);
        ++nk;
    }
    const double w = sqrt(p / 15.0);
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            if (a == 0 && b == 0) continue;
            double complex hi[4], lo[4];
            pauli2(b, hi);
            pauli2(a, lo);
            double complex* K = out + nk * 16;
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j)
                    for (int r = 0; r < 2; ++r)
                        for (int c = 0; c < 2; ++c) K[(2 * i + r) * 4 + (2 * j + c)] = w * (hi[i * 2 + j] * lo[r * 2 + c]);
            ++nk;
        }
    return nk;
}

int or_amplitude_damping(double gamma, double complex* out) {
    set2(out, 1, 0, 0, sqrt(1.0 - gamma));
    if (gamma > 0.0) {
        set2(out + 4, 0, sqrt(gamma), 0, 0);
        return 2;
    }
    return 1;
}

int or_thermal_relaxation(double t1, double t2, double ns, double complex* out) {
    if (ns == 0.0) {
        set2(out, 1, 0, 0, 1);
        return 1;
    }
    const double d = ns / 1000.0;
    const double t2e = t2 < t1 ? t2 : t1;
    const double gamma = 1.0 - exp(-d / t1);
    const double lambda = 1.0 - exp(d / t1 - 2.0 * d / t2e);
    double complex amp[2][4], ph[2][4];
    set2(amp[0], 1, 0, 0, sqrt(1.0 - gamma));
    set2(amp[1], 0, sqrt(gamma), 0, 0);
    set2(ph[0], 1, 0, 0, sqrt(1.0 - lambda));
    set2(ph[1], 0, 0, 0, sqrt(lambda));
    int nk = 0;
    for (int p = 0; p < 2; ++p)
        for (int a = 0; a < 2; ++a) {
            double complex k[4];
            double mx = 0.0;
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) {
                    k[i * 2 + j] = ph[p][i * 2 + 0] * amp[a][0 * 2 + j] + ph[p][i * 2 + 1] * amp[a][1 * 2 + j];
                    if (cabs(k[i * 2 + j]) > mx) mx = cabs(k[i * 2 + j]);
                }
            if (mx > 1e-15) {
                memcpy(out + nk * 4, k, sizeof(k));
                ++nk;
            }
        }
    return nk;
}

static int is_identity_set(const double complex* k, int nk, int d) {
    if (nk != 1) return 0;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
            if (cabs(k[i * d + j] - (i == j ? 1.0 : 0.0)) > 1e-14) return 0;
    return 1;
}

/* noise.cpp:391-426 (defaults only) executed as densitymatrix.cpp:154-167 */
int or_dm_run_noisy(double complex* rho, int n, const or_op* ops, int64_t nops, const or_noise* m) {
    double complex kr[16 * 16];
    for (int64_t i = 0; i < nops; ++i) {
        const or_op* op = &ops[i];
        if (op->kind == K_MEASURE || op->kind == K_BARRIER) continue;
        if (op->nqubits > 2) return -1;
        if (or_dm_apply(rho, n, op, 1) != 0) return -1;
        const double err = op->nqubits == 1 ? m->e1 : m->e2;
        const double dur = op->nqubits == 1 ? m->d1 : m->d2;
        int nk = or_depolarizing(err, op->nqubits, kr);
        if (!is_identity_set(kr, nk, 1 << op->nqubits)) or_dm_apply_operators(rho, n, op->qubits, op->nqubits, nk, kr);
        for (int j = 0; j < op->nqubits; ++j) {
            const int q = op->qubits[j];
            double t2 = m->t2[q] > m->t1[q] ? m->t1[q] : m->t2[q];
            nk = or_thermal_relaxation(m->t1[q], t2, dur, kr);
            if (!is_identity_set(kr, nk, 2)) or_dm_apply_operators(rho, n, &q, 1, nk, kr);
        }
    }
    return 0;
}

/* noise.cpp:177-203 */
int or_readout_apply_dist(const double* dist, int n, const double* p01, const double* p10, double* out) {
    const uint64_t len = UINT64_C(1) << n;
    double sum = 0.0;
    for (uint64_t i = 0; i < len; ++i) sum += dist[i];
    if (fabs(sum - 1.0) > 1e-9) return -1;
    memcpy(out, dist, len * sizeof(double));
    for (int q = 0; q < n; ++q) {
        if (p01[q] == 0.0 && p10[q] == 0.0) continue;
        const uint64_t bit = UINT64_C(1) << q;
        for (uint64_t idx = 0; idx < len; ++idx) {
            if (idx & bit) continue;
            const double v0 = out[idx], v1 = out[idx | bit];
            out[idx] = (1.0 - p10[q]) * v0 + p01[q] * v1;
            out[idx | bit] = p10[q] * v0 + (1.0 - p01[q]) * v1;
        }
    }
    return 0;
}

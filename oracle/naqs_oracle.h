/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference engine's hot
 * path (arxiv 2401.06861 / naqs), used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker.  The product never links it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  Parity is pinned by
 * tests/test_oracle_golden.py against the reference's own golden vectors
 * (tests/test_statevector.cpp:234-246, tests/test_densitymatrix.cpp:90-98,
 * tests/test_noise.cpp, tests/python/test_reference.py) and, in the build
 * container, bit-for-bit against the reference compiled from its own sources
 * (oracle/_ref, see oracle/Makefile).
 */
#ifndef NAQS_ORACLE_H
#define NAQS_ORACLE_H

#include <complex.h>
#include <stdint.h>

typedef struct or_op {
    int32_t kind, nqubits, qubits[3], reserved;
    double params[3];
} or_op;

typedef struct or_noise {
    const double *t1, *t2, *p01, *p10; /* per qubit */
    double e1, d1, e2, d2;             /* default_1q / default_2q: error, duration_ns */
} or_noise;

/* rng.hpp:12-61 */
void or_rng_u64(uint64_t seed, int count, uint64_t* out);
void or_rng_double(uint64_t seed, int count, double* out);
uint64_t or_derive_seed(uint64_t base, uint64_t stream);
/* tests/test_util.hpp:59-86 */
int or_random_circuit(uint64_t seed, int n, int depth, int max_arity, or_op* out);

/* gates.cpp:51-110: 2^k x 2^k row-major */
int or_gate_matrix(const or_op* op, double complex* out);

/* statevector.cpp:50-180, 198-222 */
int or_sv_apply(double complex* amps, int n, const or_op* ops, int64_t nops);
void or_sv_apply_matrix(double complex* amps, int n, const int* qubits, int k, const double complex* u);
double or_sv_norm_sq(const double complex* amps, int n);                                   /* :224-239 */
double or_sv_expectation(const double complex* amps, int n, const char* letters, double c); /* :241-277 */
void or_sv_probabilities(const double complex* amps, int n, double* out);                  /* :279-283 */
int or_sample_distribution(const double* dist, int n, uint64_t shots, uint64_t seed, uint64_t* counts); /* :293-332 */
/* :339-386 (returns the chosen Kraus index, -1 on a non-trace-preserving channel) */
int or_sv_kraus_trajectory(double complex* amps, int n, const int* qubits, int k, int nk, const double complex* kraus,
                           uint64_t* rng_state);
void or_rng_init(uint64_t* state, uint64_t seed);
double or_rng_next_double(uint64_t* state);

/* densitymatrix.cpp:60-110 */
void or_dm_apply_operators(double complex* rho, int n, const int* qubits, int k, int nops, const double complex* ops);
int or_dm_apply(double complex* rho, int n, const or_op* ops, int64_t nops); /* :114-125, 142-152 */
double or_dm_trace(const double complex* rho, int n);                        /* :169-173 */
double or_dm_purity(const double complex* rho, int n);                       /* :175-180 */
double or_dm_hermiticity(const double complex* rho, int n);                  /* :182-190 */
int or_dm_expectation(const double complex* rho, int n, const char* letters, double c, double* out); /* :192-219 */
void or_dm_probabilities(const double complex* rho, int n, double* out);    /* :221-232 */

/* noise.cpp:87-170: Kraus sets, row-major; returns the operator count */
int or_depolarizing(double p, int arity, double complex* out);
int or_thermal_relaxation(double t1, double t2, double ns, double complex* out);
int or_amplitude_damping(double gamma, double complex* out);
/* noise.cpp:391-426 + densitymatrix.cpp:154-167 (channel on each gate, identity skipped) */
int or_dm_run_noisy(double complex* rho, int n, const or_op* ops, int64_t nops, const or_noise* m);
/* noise.cpp:177-203 */
int or_readout_apply_dist(const double* dist, int n, const double* p01, const double* p10, double* out);

#endif

// TEST INFRASTRUCTURE ONLY -- C wrapper around the UNMODIFIED reference engine.
//
// oracle/Makefile compiles the reference's own sources where they lie
// (/root/reference/proj/src/{circuit,gates,pauli,statevector,densitymatrix,
// noise}.cpp) against our Eigen-API subset (third_party/eigen_subset) and the
// nlohmann json.hpp shipped in this image, and links them with this file into
// oracle/_ref/libnaqs_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, as the checker and
// the CPU baseline -- never as the product path.
//
// Every entry point takes the same packed op array as the product ABI
// (nq_op, 48 bytes) and returns 0 on success, 1 on naqs::ContractError,
// 2 on any other exception (message via ref_last_error()).
#include "naqs/circuit.hpp"
#include "naqs/densitymatrix.hpp"
#include "naqs/gates.hpp"
#include "naqs/neldermead.hpp"
#include "naqs/noise.hpp"
#include "naqs/pauli.hpp"
#include "naqs/rng.hpp"
#include "naqs/statevector.hpp"
#include "test_util.hpp"  // proj/tests/test_util.hpp: random_circuit()

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace naqs;

namespace {

struct RefOp {
    int32_t kind, nqubits, qubits[3], reserved;
    double params[3];
};
static_assert(sizeof(RefOp) == 48, "op layout");

thread_local std::string g_err;

template <class F>
int wrap(F&& f) {
    try {
        f();
        return 0;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Circuit to_circuit(int n, const RefOp* ops, int64_t nops) {
    Circuit c(n);
    for (int64_t i = 0; i < nops; ++i) {
        const RefOp& o = ops[i];
        const GateKind k = static_cast<GateKind>(o.kind);
        std::vector<int> q(o.qubits, o.qubits + o.nqubits);
        std::vector<double> p(o.params, o.params + gate_param_count(k));
        c.add(k, q, p);
    }
    return c;
}

RefOp from_gate(const GateOp& g) {
    RefOp o{};
    o.kind = static_cast<int32_t>(g.kind);
    o.nqubits = int32_t(g.qubits.size());
    for (size_t j = 0; j < g.qubits.size(); ++j) o.qubits[j] = g.qubits[j];
    for (size_t j = 0; j < g.params.size(); ++j) o.params[j] = g.params[j];
    return o;
}

void copy_cplx(const std::vector<cplx>& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(cplx)); }

DeviceNoiseModel model_from(int n, const double* t1, const double* t2, const double* p01, const double* p10,
                            double e1, double d1, double e2, double d2) {
    DeviceNoiseModel m;
    m.name = "synthetic";
    for (int q = 0; q < n; ++q) m.qubits.push_back({t1[q], t2[q], p01[q], p10[q]});
    m.default_1q = DeviceNoiseModel::GateParams{"default_1q", {}, e1, d1};
    m.default_2q = DeviceNoiseModel::GateParams{"default_2q", {}, e2, d2};
    return m;
}

void counts_dense(const std::map<std::string, std::uint64_t>& counts, int n, uint64_t* out) {
    std::memset(out, 0, (size_t(1) << n) * sizeof(uint64_t));
    for (const auto& [bits, c] : counts) {
        size_t idx = 0;
        for (int q = 0; q < n; ++q)
            if (bits[size_t(n - 1 - q)] == '1') idx |= size_t(1) << q;
        out[idx] += c;
    }
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

int ref_rng_u64(uint64_t seed, int count, uint64_t* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.next_u64();
    return 0;
}

int ref_rng_double(uint64_t seed, int count, double* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.next_double();
    return 0;
}

uint64_t ref_derive_seed(uint64_t base, uint64_t stream) { return derive_seed(base, stream); }

// proj/tests/test_util.hpp:59-86 with Rng(seed); writes `depth` ops.
int ref_random_circuit(uint64_t seed, int n, int depth, int max_arity, RefOp* out) {
    return wrap([&] {
        Rng rng(seed);
        const Circuit c = test::random_circuit(rng, n, depth, max_arity);
        for (size_t i = 0; i < c.ops().size(); ++i) out[i] = from_gate(c.ops()[i]);
    });
}

int ref_gate_matrix(const RefOp* op, double* out) {
    return wrap([&] {
        const GateKind k = static_cast<GateKind>(op->kind);
        std::vector<double> p(op->params, op->params + gate_param_count(k));
        const Eigen::MatrixXcd m = gate_matrix(k, p);
        for (Eigen::Index r = 0; r < m.rows(); ++r)
            for (Eigen::Index c = 0; c < m.cols(); ++c) {
                out[2 * (r * m.cols() + c)] = m(r, c).real();
                out[2 * (r * m.cols() + c) + 1] = m(r, c).imag();
            }
    });
}

int ref_sv_run(int n, const RefOp* ops, int64_t nops, double* amps) {
    return wrap([&] { copy_cplx(sv_run(to_circuit(n, ops, nops)).amplitudes(), amps); });
}

int ref_sv_expectations(int n, const RefOp* ops, int64_t nops, const char* letters, const double* coeff, int nt,
                        double* out) {
    return wrap([&] {
        const StateVector s = sv_run(to_circuit(n, ops, nops));
        for (int t = 0; t < nt; ++t)
            out[t] = s.expectation(PauliString(std::string(letters + size_t(t) * size_t(n), size_t(n)), coeff[t]));
    });
}

int ref_sv_norm_sq(int n, const RefOp* ops, int64_t nops, double* out) {
    return wrap([&] { *out = sv_run(to_circuit(n, ops, nops)).norm_sq(); });
}

int ref_sv_sample(int n, const RefOp* ops, int64_t nops, uint64_t shots, uint64_t seed, uint64_t* counts) {
    return wrap([&] { counts_dense(sv_run(to_circuit(n, ops, nops)).sample(shots, seed), n, counts); });
}

int ref_sample_distribution(const double* dist, int n, uint64_t shots, uint64_t seed, uint64_t* counts) {
    return wrap([&] {
        std::vector<double> d(dist, dist + (size_t(1) << n));
        counts_dense(sample_distribution(d, n, shots, seed), n, counts);
    });
}

// Monte-Carlo trajectory of a noisy schedule (run_trajectory) from |0..0>.
int ref_sv_trajectory(int n, const RefOp* ops, int64_t nops, const double* t1, const double* t2, const double* p01,
                      const double* p10, double e1, double d1, double e2, double d2, uint64_t seed, double* amps) {
    return wrap([&] {
        const DeviceNoiseModel m = model_from(n, t1, t2, p01, p10, e1, d1, e2, d2);
        const NoisySchedule s = attach_noise(to_circuit(n, ops, nops), m);
        StateVector sv(n);
        Rng rng(seed);
        sv.run_trajectory(s, rng);
        copy_cplx(sv.amplitudes(), amps);
    });
}

int ref_dm_run(int n, const RefOp* ops, int64_t nops, double* rho) {
    return wrap([&] {
        DensityMatrix d(n);
        d.run(to_circuit(n, ops, nops));
        copy_cplx(d.data(), rho);
    });
}

int ref_dm_run_noisy(int n, const RefOp* ops, int64_t nops, const double* t1, const double* t2, const double* p01,
                     const double* p10, double e1, double d1, double e2, double d2, double* rho) {
    return wrap([&] {
        const DeviceNoiseModel m = model_from(n, t1, t2, p01, p10, e1, d1, e2, d2);
        copy_cplx(dm_run_noisy(to_circuit(n, ops, nops), m).data(), rho);
    });
}

// DensityMatrix from `rho_in`-free start: run ops, then apply one channel:
// kind 0 depolarizing(p=a, arity k), 1 thermal(a=t1, b=t2, c=ns), 2 amplitude damping(a).
int ref_dm_channel(int n, const RefOp* ops, int64_t nops, int kind, double a, double b, double c, int k,
                   const int* qubits, double* rho) {
    return wrap([&] {
        DensityMatrix d(n);
        d.run(to_circuit(n, ops, nops));
        KrausChannel ch = kind == 0 ? depolarizing(a, k) : kind == 1 ? thermal_relaxation(a, b, c) : amplitude_damping(a);
        d.apply_channel(ch, std::vector<int>(qubits, qubits + k));
        copy_cplx(d.data(), rho);
    });
}

// Kraus operators of the reference channel builders (row-major, interleaved).
int ref_channel_kraus(int kind, double a, double b, double c, int k, int* nkraus, double* out) {
    return wrap([&] {
        KrausChannel ch = kind == 0 ? depolarizing(a, k) : kind == 1 ? thermal_relaxation(a, b, c) : amplitude_damping(a);
        *nkraus = int(ch.kraus.size());
        size_t at = 0;
        for (const auto& K : ch.kraus)
            for (Eigen::Index r = 0; r < K.rows(); ++r)
                for (Eigen::Index cc = 0; cc < K.cols(); ++cc) {
                    out[at++] = K(r, cc).real();
                    out[at++] = K(r, cc).imag();
                }
    });
}

// Scalars of a noisy DM run: trace, purity, hermiticity residual; expectations; probabilities.
int ref_dm_noisy_reductions(int n, const RefOp* ops, int64_t nops, const double* t1, const double* t2,
                            const double* p01, const double* p10, double e1, double d1, double e2, double d2,
                            const char* letters, const double* coeff, int nt, double* scalars, double* expect,
                            double* probs) {
    return wrap([&] {
        const DeviceNoiseModel m = model_from(n, t1, t2, p01, p10, e1, d1, e2, d2);
        const DensityMatrix d = dm_run_noisy(to_circuit(n, ops, nops), m);
        scalars[0] = d.trace();
        scalars[1] = d.purity();
        scalars[2] = d.hermiticity_residual();
        for (int t = 0; t < nt; ++t)
            expect[t] = d.expectation(PauliString(std::string(letters + size_t(t) * size_t(n), size_t(n)), coeff[t]));
        const auto p = d.probabilities();
        std::memcpy(probs, p.data(), p.size() * sizeof(double));
    });
}

int ref_readout_apply_dist(const double* dist, int n, const double* p01, const double* p10, double* out) {
    return wrap([&] {
        ReadoutModel r;
        for (int q = 0; q < n; ++q) r.qubits.push_back({p01[q], p10[q]});
        const auto o = readout_apply_dist(std::vector<double>(dist, dist + (size_t(1) << n)), r);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

// CPU timing of reset + run (mirrors proj/src/bench.cpp:32-46): one warm-up,
// then `reps` timed runs; returns the per-run milliseconds.
int ref_sv_time(int n, const RefOp* ops, int64_t nops, int reps, double* ms) {
    return wrap([&] {
        const Circuit c = to_circuit(n, ops, nops);
        StateVector s(n);
        s.run(c);
        for (int r = 0; r < reps; ++r) {
            s.reset();
            const auto t0 = std::chrono::steady_clock::now();
            s.run(c);
            const auto t1 = std::chrono::steady_clock::now();
            ms[r] = std::chrono::duration<double, std::milli>(t1 - t0).count();
        }
    });
}

// Time the ops on an already-allocated state without reset (for large n the
// reset itself is a full sweep); `reps` runs of the op list.
int ref_sv_time_noreset(int n, const RefOp* ops, int64_t nops, int reps, double* ms, double* expect_z0) {
    return wrap([&] {
        const Circuit c = to_circuit(n, ops, nops);
        StateVector s(n);
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            s.run(c);
            const auto t1 = std::chrono::steady_clock::now();
            ms[r] = std::chrono::duration<double, std::milli>(t1 - t0).count();
        }
        std::string z(size_t(n), 'I');
        z[0] = 'Z';
        *expect_z0 = s.expectation(PauliString(z));
    });
}

int ref_dm_time_noisy(int n, const RefOp* ops, int64_t nops, const double* t1, const double* t2, const double* p01,
                      const double* p10, double e1, double d1, double e2, double d2, int reps, double* ms) {
    return wrap([&] {
        const DeviceNoiseModel m = model_from(n, t1, t2, p01, p10, e1, d1, e2, d2);
        const NoisySchedule s = attach_noise(to_circuit(n, ops, nops), m);
        DensityMatrix d(n);
        for (int r = 0; r < reps; ++r) {
            d.reset();
            const auto a = std::chrono::steady_clock::now();
            d.run_schedule(s);
            const auto b = std::chrono::steady_clock::now();
            ms[r] = std::chrono::duration<double, std::milli>(b - a).count();
        }
    });
}

// Sequential Monte-Carlo loop of acceptance criterion 5 (acceptance_main.cpp:
// 154-160): ntraj trajectories sharing one Rng(seed); returns the wall time
// and the per-trajectory <Z_0>.
int ref_traj_time(int n, const RefOp* ops, int64_t nops, const double* t1, const double* t2, const double* p01,
                  const double* p10, double e1, double d1, double e2, double d2, int64_t ntraj, uint64_t seed,
                  double* ms, double* z0) {
    return wrap([&] {
        const DeviceNoiseModel m = model_from(n, t1, t2, p01, p10, e1, d1, e2, d2);
        const NoisySchedule s = attach_noise(to_circuit(n, ops, nops), m);
        std::string z(size_t(n), 'I');
        z[0] = 'Z';
        const PauliString pz(z);
        Rng rng(seed);
        const auto a = std::chrono::steady_clock::now();
        for (int64_t t = 0; t < ntraj; ++t) {
            StateVector sv(n);
            sv.run_trajectory(s, rng);
            z0[t] = sv.expectation(pz);
        }
        const auto b = std::chrono::steady_clock::now();
        *ms = std::chrono::duration<double, std::milli>(b - a).count();
    });
}

// C1: the TFIM magnetization sweep of proj/src/tfim.cpp:139-184 without the
// dense exact column (its eigensolver is outside the Eigen subset), shots = 0,
// noise from calibration JSON.  build_trotter_circuit (tfim.cpp:36-62) is
// restated here because tfim.cpp is not part of this build.
int ref_tfim_sweep(const char* calib, int n, double t_max, double dt, int steps_per_unit, int max_rows,
                   double* t_out, double* ideal_out, double* noisy_out, int* nrows, double* ms) {
    return wrap([&] {
        const DeviceNoiseModel m = load_calibration(std::string(calib));
        const auto a = std::chrono::steady_clock::now();
        int r = 0;
        for (double t = 0.0; t <= t_max + 1e-12 && r < max_rows; t += dt, ++r) {
            Circuit c(n);
            if (t != 0.0) {
                const int steps = static_cast<int>(std::ceil(t * steps_per_unit));
                const double delta = t / steps;
                for (int s = 0; s < steps; ++s) {
                    for (int i = 0; i + 1 < n; ++i) {
                        c.cx(i, i + 1);
                        c.rz(i + 1, -2.0 * delta);
                        c.cx(i, i + 1);
                    }
                    for (int i = 0; i < n; ++i) c.rx(i, -2.0 * delta);
                }
            }
            StateVector sv(n);
            sv.run(c);
            double total = 0.0;
            for (int q = 0; q < n; ++q) {
                std::string z(size_t(n), 'I');
                z[size_t(q)] = 'Z';
                total += sv.expectation(PauliString(z));
            }
            const NoisySchedule sched = attach_noise(c, m);
            DensityMatrix rho(n);
            rho.run_schedule(sched);
            const std::vector<double> dist = readout_apply_dist(rho.probabilities(), sched.readout);
            double nz = 0.0;
            for (int q = 0; q < n; ++q) {
                double zq = 0.0;
                for (size_t idx = 0; idx < dist.size(); ++idx) zq += ((idx >> q) & 1) ? -dist[idx] : dist[idx];
                nz += zq;
            }
            t_out[r] = t;
            ideal_out[r] = total / n;
            noisy_out[r] = nz / n;
        }
        *nrows = r;
        const auto b = std::chrono::steady_clock::now();
        *ms = std::chrono::duration<double, std::milli>(b - a).count();
    });
}

// Persistent state for CPU timing (bench.py cpu_baseline / --impl reference):
// allocation and |0..0> fill happen once, outside the timed runs.
void* ref_sv_new(int n) {
    try {
        return new StateVector(n);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_sv_free(void* h) { delete static_cast<StateVector*>(h); }

int ref_sv_run_timed(void* h, const RefOp* ops, int64_t nops, double* ms) {
    return wrap([&] {
        auto* s = static_cast<StateVector*>(h);
        const Circuit c = to_circuit(s->num_qubits(), ops, nops);
        const auto t0 = std::chrono::steady_clock::now();
        s->run(c);
        const auto t1 = std::chrono::steady_clock::now();
        *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    });
}

// Readers of a persistent state (parity at benchmark scale): selected
// amplitudes (StateVector::amplitude), norm_sq and Pauli expectations of the
// reference engine's own state, without copying 2^n amplitudes out.
int ref_sv_gather(void* h, const int64_t* idx, int64_t count, double* out) {
    return wrap([&] {
        auto* s = static_cast<StateVector*>(h);
        for (int64_t i = 0; i < count; ++i) {
            const cplx a = s->amplitude(size_t(idx[i]));
            out[2 * i] = a.real();
            out[2 * i + 1] = a.imag();
        }
    });
}

int ref_sv_norm_sq_h(void* h, double* out) {
    return wrap([&] { *out = static_cast<StateVector*>(h)->norm_sq(); });
}

int ref_sv_expectations_h(void* h, const char* letters, const double* coeff, int nt, double* out) {
    return wrap([&] {
        auto* s = static_cast<StateVector*>(h);
        const size_t n = size_t(s->num_qubits());
        for (int t = 0; t < nt; ++t)
            out[t] = s->expectation(PauliString(std::string(letters + size_t(t) * n, n), coeff[t]));
    });
}

int ref_sv_reset_h(void* h) {
    return wrap([&] { static_cast<StateVector*>(h)->reset(); });
}

// The reference's Nelder-Mead (proj/src/neldermead.cpp) on a C callback:
// trace_out (capacity max_evals) receives every objective value, best_out
// the best point; returns 0 / 1 / 2 like the other entry points.
int ref_minimize(double (*f)(const double*, int, void*), void* ctx, const double* x0, int n, int max_evals,
                 double x_tol, double f_tol, double initial_step, double* trace_out, int* evals, double* best_out,
                 double* best_f, int* converged) {
    return wrap([&] {
        naqs::MinimizeOptions o;
        o.max_evals = max_evals;
        o.x_tol = x_tol;
        o.f_tol = f_tol;
        o.initial_step = initial_step;
        const naqs::Objective obj = [&](const std::vector<double>& x) { return f(x.data(), int(x.size()), ctx); };
        const naqs::MinimizeResult r = naqs::minimize(obj, std::vector<double>(x0, x0 + n), o);
        for (size_t i = 0; i < r.trace.size(); ++i) trace_out[i] = r.trace[i];
        *evals = r.iterations;
        for (size_t i = 0; i < r.best_params.size(); ++i) best_out[i] = r.best_params[i];
        *best_f = r.best_energy;
        *converged = r.converged ? 1 : 0;
    });
}

} // extern "C"

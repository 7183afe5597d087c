// Application layer above the simulation boundary: the reference's TFIM
// sweep (proj/src/tfim.cpp), VQE driver (proj/src/vqe.cpp) and Nelder-Mead
// minimizer (proj/src/neldermead.cpp), declared in include/naqs/{tfim,vqe,
// neldermead}.hpp with the reference's signatures.  They are host logic that
// calls the device engine; what changes for the B200:
//   * the sweep's ideal column runs every row's circuit in one batched launch
//     (batch_expectations), the noisy column every row's density matrix in
//     another (batch_noisy_distributions, n <= 6);
//   * the dense "exact" oracle is one cuSOLVER zheevd on the device for the
//     whole sweep (the reference re-decomposes H for every row);
//   * exact energies are one batched expectation launch over all terms.
// Values agree with the reference to rounding (tests/test_apps_gpu.py and the
// reference's own test_tfim.cpp / test_vqe.cpp / test_neldermead.cpp, built
// against these headers).
#include "naqs/densitymatrix.hpp"
#include "naqs/neldermead.hpp"
#include "naqs/rng.hpp"
#include "naqs/statevector.hpp"
#include "naqs/tfim.hpp"
#include "naqs/vqe.hpp"

#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <limits>
#include <mutex>
#include <numeric>
#include <string>

namespace naqs {

// ---- Nelder-Mead (proj/src/neldermead.cpp:85-182) ------------------------------
namespace {

struct Budgeted {
    Budgeted(const Objective& f_, int budget_) : f(f_), budget(budget_) {}
    const Objective& f;
    int budget;
    int used = 0;
    bool aborted = false;
    std::string diagnostic;
    std::vector<double> trace;
    std::vector<double> best_x;
    double best_f = std::numeric_limits<double>::infinity();

    bool done() const { return aborted || used >= budget; }
    double operator()(const std::vector<double>& x) {
        const double v = f(x);
        trace.push_back(v);
        ++used;
        if (!std::isfinite(v)) {
            aborted = true;
            diagnostic = "objective returned a non-finite value at evaluation " + std::to_string(used);
        } else if (v < best_f) {
            best_f = v;
            best_x = x;
        }
        return v;
    }
};

using Point = std::vector<double>;

// vertices ordered by value, ties keeping their previous order
void order_vertices(std::vector<Point>& xs, std::vector<double>& fs) {
    std::vector<size_t> idx(xs.size());
    std::iota(idx.begin(), idx.end(), size_t(0));
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return fs[a] < fs[b]; });
    std::vector<Point> x2;
    std::vector<double> f2;
    x2.reserve(xs.size());
    f2.reserve(fs.size());
    for (size_t i : idx) {
        x2.push_back(std::move(xs[i]));
        f2.push_back(fs[i]);
    }
    xs.swap(x2);
    fs.swap(f2);
}

// max over vertices and coordinates of |x_i - x_0|
double spread_from_first(const std::vector<Point>& xs) {
    double d = 0.0;
    for (size_t i = 1; i < xs.size(); ++i)
        for (size_t j = 0; j < xs[i].size(); ++j) d = std::max(d, std::abs(xs[i][j] - xs[0][j]));
    return d;
}

// c + s (a - c), coordinate-wise
Point along(const Point& c, const Point& a, double s) {
    Point r(c.size());
    for (size_t j = 0; j < c.size(); ++j) r[j] = c[j] + s * (a[j] - c[j]);
    return r;
}

}  // namespace

MinimizeResult minimize(const Objective& f, const std::vector<double>& x0, const MinimizeOptions& opts) {
    if (x0.empty()) throw ContractError("minimize needs at least one dimension");
    if (opts.max_evals < 1) throw ContractError("max_evals must be >= 1");
    const size_t dim = x0.size();
    Budgeted F(f, opts.max_evals);
    F.best_x = x0;
    F(x0);
    double step = opts.initial_step;
    bool by_tolerance = false;
    while (!F.done()) {
        // axis simplex around the best point (which may improve while it is built)
        std::vector<Point> xs{F.best_x};
        std::vector<double> fs{F.best_f};
        for (size_t i = 0; i < dim && !F.done(); ++i) {
            Point p = F.best_x;
            p[i] += step;
            fs.push_back(F(p));
            xs.push_back(std::move(p));
        }
        if (xs.size() < dim + 1) break;
        const double round_start = F.best_f;
        by_tolerance = false;
        while (!F.done()) {
            order_vertices(xs, fs);
            if (spread_from_first(xs) < opts.x_tol || std::abs(fs.back() - fs.front()) < opts.f_tol) {
                by_tolerance = true;
                break;
            }
            Point c(dim, 0.0);
            for (size_t i = 0; i < dim; ++i)
                for (size_t j = 0; j < dim; ++j) c[j] += xs[i][j];
            for (double& v : c) v /= double(dim);
            Point& worst = xs.back();
            // reflection: c + 1 (c - worst) = c - 1 (worst - c)
            Point xr = along(c, worst, -1.0);
            const double fr = F(xr);
            if (F.aborted) break;
            if (fr < fs.front()) {
                if (!F.done()) {
                    Point xe = along(c, worst, -2.0);  // expansion
                    const double fe = F(xe);
                    if (F.aborted) break;
                    if (fe < fr) {
                        worst = std::move(xe);
                        fs.back() = fe;
                        continue;
                    }
                }
                worst = std::move(xr);
                fs.back() = fr;
            } else if (fr < fs[dim - 1]) {
                worst = std::move(xr);
                fs.back() = fr;
            } else {
                if (F.done()) break;
                Point xc = along(c, fr < fs.back() ? xr : worst, 0.5);  // contraction
                const double fc = F(xc);
                if (F.aborted) break;
                if (fc < std::min(fr, fs.back())) {
                    worst = std::move(xc);
                    fs.back() = fc;
                } else {
                    // shrink toward the best vertex
                    for (size_t i = 1; i < xs.size() && !F.done(); ++i) {
                        xs[i] = along(xs[0], xs[i], 0.5);
                        fs[i] = F(xs[i]);
                        if (F.aborted) break;
                    }
                }
            }
        }
        if (F.aborted) break;
        if (F.best_f >= round_start) break;  // the restart did not improve
        step *= 0.5;
    }
    MinimizeResult r;
    r.best_params = F.best_x;
    r.best_energy = F.best_f;
    r.trace = std::move(F.trace);
    r.iterations = F.used;
    r.diagnostic = F.diagnostic;
    r.converged = !F.aborted && by_tolerance && F.used < opts.max_evals;
    return r;
}

// ---- dense Hermitian eigendecomposition on the device (cuSOLVER zheevd) ----------
// Replaces Eigen::SelfAdjointEigenSolver of the reference's dense oracles
// (proj/src/tfim.cpp:110-124, proj/src/vqe.cpp:142-149).  cuSOLVER is bound
// at first use so processes that never call the oracles do not load it.
namespace {

struct Solver {
    decltype(&::cusolverDnCreate) create = nullptr;
    decltype(&::cusolverDnDestroy) destroy = nullptr;
    decltype(&::cusolverDnZheevd_bufferSize) buffer = nullptr;
    decltype(&::cusolverDnZheevd) zheevd = nullptr;
};

const Solver& solver() {
    static Solver s;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            err = e ? e : "dlopen(libcusolver) failed";
            return;
        }
        s.create = reinterpret_cast<decltype(s.create)>(dlsym(h, "cusolverDnCreate"));
        s.destroy = reinterpret_cast<decltype(s.destroy)>(dlsym(h, "cusolverDnDestroy"));
        s.buffer = reinterpret_cast<decltype(s.buffer)>(dlsym(h, "cusolverDnZheevd_bufferSize"));
        s.zheevd = reinterpret_cast<decltype(s.zheevd)>(dlsym(h, "cusolverDnZheevd"));
    });
    if (!s.create || !s.destroy || !s.buffer || !s.zheevd) throw Error("cuSOLVER unavailable: " + err);
    return s;
}

struct DenseEigen {
    int dim = 0;
    std::vector<double> w;  // ascending
    std::vector<cplx> v;    // column-major eigenvectors (column j <-> w[j])
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

DenseEigen dense_eigen(const Hamiltonian& h, bool vectors) {
    const Eigen::MatrixXcd m = hamiltonian_dense(h);  // enforces the dense limit
    const int dim = int(m.rows());
    std::vector<cplx> a(size_t(dim) * size_t(dim));
    for (int c = 0; c < dim; ++c)
        for (int r = 0; r < dim; ++r) a[size_t(c) * size_t(dim) + size_t(r)] = m(r, c);
    const Solver& S = solver();
    cusolverDnHandle_t hd = nullptr;
    if (S.create(&hd) != CUSOLVER_STATUS_SUCCESS) throw Error("cusolverDnCreate failed");
    cuDoubleComplex *d_a = nullptr, *d_work = nullptr;
    double* d_w = nullptr;
    int* d_info = nullptr;
    DenseEigen out;
    out.dim = dim;
    out.w.resize(size_t(dim));
    try {
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&d_a), a.size() * sizeof(cuDoubleComplex)), "cudaMalloc");
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&d_w), size_t(dim) * sizeof(double)), "cudaMalloc");
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&d_info), sizeof(int)), "cudaMalloc");
        cuda_check(cudaMemcpy(d_a, a.data(), a.size() * sizeof(cuDoubleComplex), cudaMemcpyHostToDevice), "H2D");
        const cusolverEigMode_t job = vectors ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
        int lwork = 0;
        if (S.buffer(hd, job, CUBLAS_FILL_MODE_LOWER, dim, d_a, dim, d_w, &lwork) != CUSOLVER_STATUS_SUCCESS)
            throw Error("cusolverDnZheevd_bufferSize failed");
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&d_work), size_t(std::max(lwork, 1)) * sizeof(cuDoubleComplex)),
                   "cudaMalloc");
        if (S.zheevd(hd, job, CUBLAS_FILL_MODE_LOWER, dim, d_a, dim, d_w, d_work, lwork, d_info) !=
            CUSOLVER_STATUS_SUCCESS)
            throw Error("cusolverDnZheevd failed");
        int info = 0;
        cuda_check(cudaMemcpy(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
        if (info != 0) throw Error("eigendecomposition failed");
        cuda_check(cudaMemcpy(out.w.data(), d_w, size_t(dim) * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        if (vectors) {
            out.v.resize(a.size());
            cuda_check(cudaMemcpy(out.v.data(), d_a, a.size() * sizeof(cuDoubleComplex), cudaMemcpyDeviceToHost), "D2H");
        }
    } catch (...) {
        cudaFree(d_a);
        cudaFree(d_w);
        cudaFree(d_info);
        cudaFree(d_work);
        S.destroy(hd);
        throw;
    }
    cudaFree(d_a);
    cudaFree(d_w);
    cudaFree(d_info);
    cudaFree(d_work);
    S.destroy(hd);
    return out;
}

// (1/n) sum_q <Z_q> of V exp(-i W t) V^dagger psi0 (proj/src/tfim.cpp:100-137)
double evolved_magnetization(const DenseEigen& e, int n, double t, const std::vector<cplx>& psi0) {
    const size_t dim = size_t(e.dim);
    std::vector<cplx> coef(dim);
    for (size_t j = 0; j < dim; ++j) {
        cplx acc(0.0, 0.0);
        const cplx* col = e.v.data() + j * dim;
        for (size_t i = 0; i < dim; ++i) acc += std::conj(col[i]) * psi0[i];
        coef[j] = acc * std::exp(cplx(0.0, -e.w[j] * t));
    }
    std::vector<cplx> psit(dim, cplx(0.0, 0.0));
    for (size_t j = 0; j < dim; ++j) {
        const cplx* col = e.v.data() + j * dim;
        for (size_t i = 0; i < dim; ++i) psit[i] += col[i] * coef[j];
    }
    double total = 0.0;
    for (int q = 0; q < n; ++q) {
        double z = 0.0;
        for (size_t i = 0; i < dim; ++i) {
            const double p = std::norm(psit[i]);
            z += ((i >> q) & 1) ? -p : p;
        }
        total += z;
    }
    return total / n;
}

std::vector<PauliString> single_z_terms(int n) {
    std::vector<PauliString> zs;
    for (int q = 0; q < n; ++q) {
        std::string L(size_t(n), 'I');
        L[size_t(q)] = 'Z';
        zs.emplace_back(L);
    }
    return zs;
}

double mean_in_order(const std::vector<double>& v, int n) {
    double total = 0.0;
    for (double x : v) total += x;
    return total / n;
}

// site-averaged <Z> of a distribution (proj/src/tfim.cpp:77-88)
double dist_magnetization(const std::vector<double>& dist, int n) {
    double total = 0.0;
    for (int q = 0; q < n; ++q) {
        double z = 0.0;
        for (size_t i = 0; i < dist.size(); ++i) z += ((i >> q) & 1) ? -dist[i] : dist[i];
        total += z;
    }
    return total / n;
}

// bitstring counts -> distribution (MSB-first bitstrings; proj/src/tfim.cpp:90-98)
std::vector<double> counts_to_dist(const std::map<std::string, std::uint64_t>& counts, int n, std::uint64_t shots) {
    std::vector<double> dist(size_t(1) << n, 0.0);
    for (const auto& kv : counts) {
        size_t idx = 0;
        for (int q = 0; q < n; ++q)
            if (kv.first[size_t(n - 1 - q)] == '1') idx |= size_t(1) << q;
        dist[idx] = double(kv.second) / double(shots);
    }
    return dist;
}

}  // namespace

// ---- TFIM (proj/src/tfim.cpp) ------------------------------------------------------
Hamiltonian build_tfim_hamiltonian(int n, double coupling, double field, Boundary boundary) {
    if (n < 1) throw ContractError("TFIM chain needs at least one site");
    Hamiltonian h;
    h.n = n;
    auto word = [n](std::initializer_list<int> zs, char letter) {
        std::string L(size_t(n), 'I');
        for (int q : zs) L[size_t(q)] = letter;
        return L;
    };
    for (int i = 0; i + 1 < n; ++i) h.add(word({i, i + 1}, 'Z'), -coupling);
    if (boundary == Boundary::Periodic && n >= 3) h.add(word({n - 1, 0}, 'Z'), -coupling);
    for (int i = 0; i < n; ++i) h.add(word({i}, 'X'), -field);
    return h;
}

Circuit build_trotter_circuit(const TfimParams& p, double t) {
    if (t < 0.0) throw ContractError("evolution time must be non-negative");
    Circuit c(p.n, "tfim_trotter");
    if (t == 0.0) return c;
    const int steps = int(std::ceil(t * p.steps_per_unit_time));
    const double delta = t / steps;
    std::vector<std::pair<int, int>> bonds;
    for (int i = 0; i + 1 < p.n; ++i) bonds.emplace_back(i, i + 1);
    if (p.boundary == Boundary::Periodic && p.n >= 3) bonds.emplace_back(p.n - 1, 0);
    const double zz = -2.0 * p.coupling * delta, xf = -2.0 * p.field * delta;
    for (int s = 0; s < steps; ++s) {
        for (const auto& b : bonds) c.cx(b.first, b.second).rz(b.second, zz).cx(b.first, b.second);
        for (int i = 0; i < p.n; ++i) c.rx(i, xf);
    }
    return c;
}

double average_z(const StateVector& s) {
    const int n = s.num_qubits();
    return mean_in_order(s.expectations(single_z_terms(n)), n);
}

double exact_magnetization(const Hamiltonian& h, double t, const StateVector& initial) {
    if (h.n != initial.num_qubits()) throw ContractError("Hamiltonian and state qubit counts differ");
    const DenseEigen e = dense_eigen(h, true);
    return evolved_magnetization(e, h.n, t, initial.amplitudes());
}

std::vector<SweepRow> magnetization_sweep(const TfimParams& p, const std::optional<DeviceNoiseModel>& noise,
                                          std::uint64_t shots, std::uint64_t seed) {
    if (p.n < 1 || p.dt <= 0.0 || p.t_max < 0.0 || p.steps_per_unit_time < 1)
        throw ContractError("invalid sweep parameters");
    if (p.n > kDenseOracleLimit)
        throw ContractError("sweep's exact column is limited to n <= " + std::to_string(kDenseOracleLimit));
    if (noise && p.n > DensityMatrix::kMaxQubits)
        throw ContractError("noisy column is limited to n <= " + std::to_string(DensityMatrix::kMaxQubits));
    const Hamiltonian h = build_tfim_hamiltonian(p.n, p.coupling, p.field, p.boundary);
    // times as the reference accumulates them (t += dt: 0.30000000000000004 ...)
    std::vector<double> ts;
    for (double t = 0.0; t <= p.t_max + 1e-12; t += p.dt) ts.push_back(t);
    std::vector<Circuit> circs;
    circs.reserve(ts.size());
    for (double t : ts) circs.push_back(build_trotter_circuit(p, t));

    const DenseEigen e = dense_eigen(h, true);
    std::vector<cplx> psi0(size_t(1) << p.n, cplx(0.0, 0.0));
    psi0[0] = 1.0;

    std::vector<SweepRow> rows(ts.size());
    const std::vector<PauliString> zs = single_z_terms(p.n);
    const auto ideal = batch_expectations(circs, zs);  // every row, one launch
    for (size_t r = 0; r < ts.size(); ++r) {
        rows[r].t = ts[r];
        rows[r].exact = evolved_magnetization(e, p.n, ts[r], psi0);
        rows[r].ideal = mean_in_order(ideal[r], p.n);
    }
    if (noise) {
        std::vector<std::vector<double>> dists;
        if (p.n <= 6) {
            dists = batch_noisy_distributions(circs, *noise);  // every row, one launch
        } else {
            for (const auto& c : circs) {
                const NoisySchedule sched = attach_noise(c, *noise);
                DensityMatrix rho(p.n);
                rho.run_schedule(sched);
                dists.push_back(readout_apply_dist(rho.probabilities(), sched.readout));
            }
        }
        for (size_t r = 0; r < ts.size(); ++r) {
            std::vector<double>& dist = dists[r];
            if (shots > 0)
                dist = counts_to_dist(sample_distribution(dist, p.n, shots, derive_seed(seed, r)), p.n, shots);
            rows[r].noisy = dist_magnetization(dist, p.n);
        }
    }
    return rows;
}

// ---- VQE (proj/src/vqe.cpp) ----------------------------------------------------------
Circuit build_ansatz_circuit(const AnsatzSpec& a, const std::vector<double>& params) {
    if (a.n < 1 || a.layers < 1) throw ContractError("ansatz needs n >= 1 and layers >= 1");
    if (int(params.size()) != a.param_count())
        throw ContractError("ansatz expects " + std::to_string(a.param_count()) + " parameters, got " +
                            std::to_string(params.size()));
    Circuit c(a.n, "ansatz");
    size_t k = 0;
    for (int q = 0; q < a.n; ++q) c.ry(q, params[k++]);
    for (int l = 0; l < a.layers; ++l) {
        for (int i = 0; i + 1 < a.n; ++i) c.cx(i, i + 1);
        for (int q = 0; q < a.n; ++q) c.ry(q, params[k++]);
    }
    return c;
}

namespace {

// one Pauli term measured in its rotated basis from `shots` samples
// (proj/src/vqe.cpp:34-88: H for X, SDG then H for Y; parity of the support)
double sampled_term(const Circuit& ansatz, const PauliString& term, std::uint64_t shots, std::uint64_t term_seed,
                    const std::optional<DeviceNoiseModel>& noise) {
    Circuit c = ansatz;
    size_t support = 0;
    for (int q = 0; q < term.n; ++q) {
        const char L = term.letters[size_t(q)];
        if (L == 'X') {
            c.h(q);
        } else if (L == 'Y') {
            c.add(GateKind::SDG, {q});
            c.h(q);
        }
        if (L != 'I') support |= size_t(1) << q;
    }
    std::vector<double> dist;
    if (noise) {
        const NoisySchedule sched = attach_noise(c, *noise);
        DensityMatrix rho(c.num_qubits());
        rho.run_schedule(sched);
        dist = readout_apply_dist(rho.probabilities(), sched.readout);
    } else {
        dist = sv_run(c).probabilities();
    }
    const int n = c.num_qubits();
    double acc = 0.0;
    for (const auto& kv : sample_distribution(dist, n, shots, term_seed)) {
        size_t idx = 0;
        for (int q = 0; q < n; ++q)
            if (kv.first[size_t(n - 1 - q)] == '1') idx |= size_t(1) << q;
        acc += ((std::popcount(idx & support) & 1) ? -1.0 : 1.0) * double(kv.second);
    }
    return term.coefficient * (acc / double(shots));
}

}  // namespace

double vqe_energy(const std::vector<double>& params, const AnsatzSpec& a, const Hamiltonian& h,
                  const EnergyMode& mode, const std::optional<DeviceNoiseModel>& noise) {
    if (h.n != a.n) throw ContractError("Hamiltonian and ansatz qubit counts differ");
    const Circuit ansatz = build_ansatz_circuit(a, params);
    double energy = 0.0;
    if (mode.shots == 0) {
        // every term from one batched reduction, summed in term order
        const std::vector<double> e =
            noise ? dm_run_noisy(ansatz, *noise).expectations(h.terms) : sv_run(ansatz).expectations(h.terms);
        for (double v : e) energy += v;
        return energy;
    }
    for (size_t k = 0; k < h.terms.size(); ++k)
        energy += sampled_term(ansatz, h.terms[k], mode.shots, derive_seed(mode.seed, k), noise);
    return energy;
}

MinimizeResult run_vqe(int n, double coupling, double field, const VqeOptions& opts,
                       const std::optional<DeviceNoiseModel>& noise) {
    const Hamiltonian h = build_tfim_hamiltonian(n, coupling, field);
    const AnsatzSpec spec{n, opts.layers};
    Rng rng(opts.seed);
    std::vector<double> x0(size_t(spec.param_count()));
    for (double& v : x0) v = rng.uniform(-0.1, 0.1);
    MinimizeOptions mo;
    mo.max_evals = opts.max_evals;
    mo.x_tol = opts.x_tol;
    mo.f_tol = opts.f_tol;
    mo.seed = opts.seed;
    mo.initial_step = 2.0;  // proj/src/vqe.cpp:134
    return minimize([&](const std::vector<double>& x) { return vqe_energy(x, spec, h, opts.mode, noise); }, x0, mo);
}

double ground_energy(const Hamiltonian& h) { return dense_eigen(h, false).w.front(); }

}  // namespace naqs

// naqs-b200: pure-state simulator (API of proj/include/naqs/statevector.hpp).
//
// The amplitudes live in B200 HBM behind an nq_sv handle (C ABI,
// include/naqs_b200.h).  Gates are validated when applied and executed in
// fused passes when a result is requested.  amplitudes()/amplitude() read a
// host mirror that is refreshed lazily after the state changes.
#pragma once

#include "naqs/circuit.hpp"
#include "naqs/noise.hpp"
#include "naqs/pauli.hpp"
#include "naqs/rng.hpp"
#include "naqs/types.hpp"

#include <cstdint>
#include <map>
#include <string>
#include <vector>

struct nq_sv;

namespace naqs {

/// Execution options beyond the reference API (device, fusion, tile size,
/// and a raised qubit cap for states larger than the reference's guard).
struct EngineOptions {
    int device = -1;
    int max_qubits = 0;   // 0: the reference guard kMaxQubits
    int tile_qubits = 0;  // 0: planner default
    bool fuse = true;
};

class StateVector {
  public:
    static constexpr int kMaxQubits = 30;

    explicit StateVector(int num_qubits);
    StateVector(int num_qubits, const EngineOptions& opts);
    StateVector(const StateVector& other);
    StateVector(StateVector&& other) noexcept;
    StateVector& operator=(const StateVector& other);
    StateVector& operator=(StateVector&& other) noexcept;
    ~StateVector();

    void reset();

    int num_qubits() const { return n_; }
    std::size_t dim() const { return std::size_t(1) << n_; }
    const std::vector<cplx>& amplitudes() const;
    cplx amplitude(std::size_t index) const;

    void apply(const GateOp& op);
    void run(const Circuit& c);

    double norm_sq() const;
    double expectation(const PauliString& p) const;
    /// All terms in one batched device reduction (same values as calling
    /// expectation() per term).
    std::vector<double> expectations(const std::vector<PauliString>& terms) const;
    std::vector<double> probabilities() const;
    std::map<std::string, std::uint64_t> sample(std::uint64_t shots, std::uint64_t seed) const;

    void apply_kraus_trajectory(const KrausChannel& ch, const std::vector<int>& qubits, Rng& rng);
    void run_trajectory(const NoisySchedule& schedule, Rng& rng);

    /// Underlying C-ABI handle (for zero-copy consumers).
    nq_sv* handle() const { return h_; }

  private:
    void invalidate() { mirror_ok_ = false; }

    int n_ = 0;
    nq_sv* h_ = nullptr;
    mutable std::vector<cplx> mirror_;
    mutable bool mirror_ok_ = false;
};

StateVector sv_run(const Circuit& c);

std::string index_to_bitstring(std::size_t index, int n);

std::map<std::string, std::uint64_t> sample_distribution(const std::vector<double>& dist, int n,
                                                         std::uint64_t shots, std::uint64_t seed);

/// Batched Monte-Carlo trajectories (beyond the reference API; SURVEY.md §8
/// f1): `ntraj` runs of `schedule` from |0...0> in one device launch, drawing
/// from `rng` exactly as the sequential loop
/// `for (t) { StateVector s(n); s.run_trajectory(schedule, rng); }` does, so
/// row t holds the `observables` of the same trajectory that loop would give.
std::vector<std::vector<double>> run_trajectories(const NoisySchedule& schedule, std::uint64_t ntraj, Rng& rng,
                                                  const std::vector<PauliString>& observables);

/// Batches of small independent circuits in one launch (
/// TFIM sweep rows, VQE evaluations): row b = the observables of
/// sv_run(circuits[b]) (all circuits on the same qubit count, n <= 12).
std::vector<std::vector<double>> batch_expectations(const std::vector<Circuit>& circuits,
                                                    const std::vector<PauliString>& observables);

} // namespace naqs

// naqs-b200: mixed-state simulator (API of proj/include/naqs/densitymatrix.hpp).
//
// rho is row-major in B200 HBM (rho[r * 2^n + c]).  Gates and channels are
// compiled into Liouville-space superoperators on vec(rho) and executed by
// the same fused pass kernel as the state vector.
#pragma once

#include "naqs/circuit.hpp"
#include "naqs/noise.hpp"
#include "naqs/pauli.hpp"
#include "naqs/statevector.hpp"
#include "naqs/types.hpp"

#include <vector>

struct nq_dm;

namespace naqs {

class DensityMatrix {
  public:
    static constexpr int kMaxQubits = 14;

    explicit DensityMatrix(int num_qubits);
    DensityMatrix(int num_qubits, const EngineOptions& opts);
    DensityMatrix(const DensityMatrix& other);
    DensityMatrix(DensityMatrix&& other) noexcept;
    DensityMatrix& operator=(const DensityMatrix& other);
    DensityMatrix& operator=(DensityMatrix&& other) noexcept;
    ~DensityMatrix();

    void reset();

    int num_qubits() const { return n_; }
    std::size_t dim() const { return std::size_t(1) << n_; }
    const std::vector<cplx>& data() const;
    cplx entry(std::size_t row, std::size_t col) const;

    void apply(const GateOp& op);
    void apply_channel(const KrausChannel& ch, const std::vector<int>& qubits);
    void run(const Circuit& c);
    void run_schedule(const NoisySchedule& schedule);

    double trace() const;
    double purity() const;
    double hermiticity_residual() const;
    double expectation(const PauliString& p) const;
    std::vector<double> expectations(const std::vector<PauliString>& terms) const;
    std::vector<double> probabilities() const;

    nq_dm* handle() const { return h_; }

  private:
    int n_ = 0;
    nq_dm* h_ = nullptr;
    mutable std::vector<cplx> mirror_;
    mutable bool mirror_ok_ = false;
};

DensityMatrix dm_run_noisy(const Circuit& c, const DeviceNoiseModel& m);

/// Batches of small noisy circuits in one launch (the noisy
/// column of magnetization_sweep): row b = readout_apply_dist(probabilities of
/// dm_run_noisy(circuits[b], m), readout) (n <= 6).
std::vector<std::vector<double>> batch_noisy_distributions(const std::vector<Circuit>& circuits,
                                                           const DeviceNoiseModel& m);

} // namespace naqs

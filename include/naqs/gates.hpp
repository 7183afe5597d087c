// naqs-b200: dense gate matrices (API of proj/include/naqs/gates.hpp).
// Used by tests and by host-side channel/fusion code; the device kernels
// receive the same matrices through the C ABI.
#pragma once

#include "naqs/circuit.hpp"
#include "naqs/types.hpp"

#include <Eigen/Dense>
#include <vector>

namespace naqs {

/// 2^k x 2^k unitary of `kind` (local bit j = qubits[j]); OpenQASM 2.0 u3.
Eigen::MatrixXcd gate_matrix(GateKind kind, const std::vector<double>& params = {});
Eigen::MatrixXcd gate_matrix(const GateOp& op);

/// max |U^dagger U - I| entry.
double unitarity_residual(const Eigen::MatrixXcd& u);

} // namespace naqs

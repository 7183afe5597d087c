#pragma once

#include "../../include/naqs_b200.h"
#include "engine.hpp"

#include <vector>

namespace nqe {

int kind_arity(int kind);
int kind_params(int kind);

void lower_sv_op(const nq_op& op, std::vector<EOp>& out);
std::vector<cplx> full_gate_matrix(const nq_op& op);
EOp sv_matrix_op(const int* qubits, int k, const cplx* mat);

void lower_dm_op(const nq_op& op, int n, std::vector<EOp>& out);
EOp dm_channel_op(const int* qubits, int k, int nkraus, const cplx* kraus, int n);

std::vector<cplx> superop(int k, const std::vector<const cplx*>& kraus);
bool depol_form(int k, const std::vector<cplx>& s, double* a, double* b);

}  // namespace nqe

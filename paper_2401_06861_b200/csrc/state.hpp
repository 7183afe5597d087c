// Device context and state objects behind the C ABI handles.
#pragma once

#include "../../include/naqs_b200.h"
#include "engine.hpp"

#include <cuda_runtime.h>

#include <cstdint>
#include <new>
#include <string>
#include <utility>
#include <vector>

namespace nqe {

struct NqError {
    nq_status code;
    std::string msg;
};

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t cuda_try_e_ = (expr);                                                      \
        if (cuda_try_e_ != cudaSuccess) {                                                      \
            throw ::nqe::NqError{cuda_try_e_ == cudaErrorMemoryAllocation ? NQ_ERR_OOM         \
                                                                          : NQ_ERR_CUDA,       \
                                 std::string(#expr) + ": " + cudaGetErrorString(cuda_try_e_)}; \
        }                                                                                      \
    } while (0)

extern thread_local std::string g_last_error;

template <class F>
nq_status guard(F&& f) {
    try {
        f();
        return NQ_OK;
    } catch (const NqError& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return NQ_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return NQ_ERR_INTERNAL;
    }
}

// One per CUDA device: the stream every state on that device runs on, the
// pinned staging buffer for pass records, and reduction scratch.
struct DeviceCtx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t stage_ev = nullptr;
    bool stage_pending = false;
    unsigned char* h_stage = nullptr;
    size_t h_stage_cap = 0;
    unsigned char* d_ops = nullptr;
    size_t d_ops_cap = 0;
    double* d_scratch = nullptr;
    size_t scratch_cap = 0;
    double* h_small = nullptr;
    // measured region (nq_profile_begin/end)
    bool prof = false, prof_pass = false;
    cudaEvent_t prof_t0 = nullptr, prof_t1 = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
    size_t prof_used = 0;
    double prof_pass_bytes = 0.0;
    int64_t prof_launch0 = 0, h2d_bytes = 0, d2h_bytes = 0;

    void ensure_scratch(size_t doubles);
    void stage(const unsigned char* src, size_t bytes);
};

DeviceCtx& ctx_for(int dev);
std::pair<cudaEvent_t, cudaEvent_t>* prof_slot(DeviceCtx& c);

struct ShardComm;  // shard.cpp

struct State {
    int n = 0;       // qubits
    int nbits = 0;   // state bits (SV n, DM 2n)
    int nloc = 0;    // bits held on this device
    bool dm = false;
    int dev = 0;
    double2* d = nullptr;
    uint64_t count = 0;  // 2^nloc
    std::vector<EOp> queue;
    PlanOptions popt;
    int64_t last_passes = 0, last_microops = 0, last_source_ops = 0, last_launches = 0;
    // sharded states (world > 1)
    int rank = 0, world = 1;
    ShardComm* comm = nullptr;
    bool plain_alloc = false;  // cudaMalloc'd (IPC-exportable), freed with cudaFree
    // single-device state vectors: logical qubit -> physical bit after the
    // relabelling passes (identity otherwise); readouts normalise it
    std::vector<int> layout;
    // device probabilities for zero-copy consumers (nq_*_probabilities_device):
    // owned by the state, valid until it is next modified or destroyed
    double* dprob = nullptr;
    uint64_t dprob_cap = 0;
};

void sv_expect_raw(State& s, const uint64_t* flip, const uint64_t* signs, int nterms, std::vector<cplx>& totals);

void state_init(State& s, int n, bool dm, const nq_opts* opts);
void state_free(State& s);
// Z-type expectation terms a flush may compute in its last pass (fused
// epilogue): signs in logical qubits in, per-term sums on the device out
// (fused = false when the last pass could not carry them, e.g. its kernel is
// not compiled yet: the caller then reads the state separately)
struct FlushEpilogue {
    int nterms = 0;
    const uint64_t* signs = nullptr;
    bool fused = false;
    double* dev_sums = nullptr;
};
void state_flush(State& s, FlushEpilogue* fe = nullptr);
// flush, then restore the identity layout (amplitude-order readouts)
void state_flush_normal(State& s);
void configure_caps(PlanOptions& p);
double* result_slot(DeviceCtx& c, int i);
void fetch(DeviceCtx& c, const double* dsrc, size_t count, double* host);

// sampling (sample.cpp): either amplitudes `a` or probabilities `p` (one is
// null).  The cumulative sum is the reference's sequential one, bit for bit.
struct SeqCum {
    uint64_t n = 0, bs = 0, nb = 0;
    std::vector<double> bsum;                // approximate block sums (guesses only)
    std::vector<int> kb;                     // guessed binade per block (INT_MIN: replay)
    std::vector<unsigned long long> isum;    // integer increments in that binade
    std::vector<int> flags;                  // tie / overflow inside the block
    std::vector<double> ends;                // exact sequential cum at each block end
    int64_t replayed = 0;                    // blocks replayed on the host
};
void seqcum_prepare(DeviceCtx& c, const double2* a, const double* p, uint64_t n, double approx_start, SeqCum& sc);
// exact walk from the exact cumulative `start`; returns the final cumulative
double seqcum_walk(DeviceCtx& c, const double2* a, const double* p, SeqCum& sc, double start);
// leftovers: whether uniforms beyond the final cumulative are assigned here
void sample_assign(DeviceCtx& c, const double2* a, const double* p, const SeqCum& sc, double start,
                   const double* sorted_u, uint64_t shots, uint64_t* idx_out, uint64_t* count_out, uint64_t* nout,
                   bool leftovers);
void sample_sweep(DeviceCtx& c, const double2* a, const double* p, uint64_t n, const double* sorted_u,
                  uint64_t shots, uint64_t* idx_out, uint64_t* count_out, uint64_t* nout);

// multi-GPU (shard.cpp)
void shard_free(State& s);
void shard_reset(State& s);
void shard_flush(State& s);
double shard_norm_sq(State& s);
void shard_expectation(State& s, const uint64_t* flip, const uint64_t* signs, const int32_t* ny,
                       const double* coeff, int nterms, double* out);
void shard_sample(State& s, const double* sorted_u, uint64_t shots, uint64_t* idx_out, uint64_t* count_out,
                  uint64_t* nout);
void shard_get_amplitudes(State& s, uint64_t offset, uint64_t count, double* host_out);
void shard_probabilities(State& s, double* host_out);
void shard_set_amplitudes(State& s, uint64_t offset, uint64_t count, const double* host_in);
// restore the identity qubit map (physical order == logical order)
void shard_normalize(State& s);

}  // namespace nqe

// The opaque C-ABI handles.
extern "C" {
struct nq_sv {
    nqe::State s;
};
struct nq_dm {
    nqe::State s;
};
}

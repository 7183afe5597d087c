// Host-side launchers of the sm_100a kernels (kernels.cu).
#pragma once

#include "engine.hpp"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace nqe {

// Every kernel launched by this library (for the bench's gpu_launches claim).
extern std::atomic<int64_t> g_kernel_launches;

// rbits: register bits of the pass's layouts (its first MOP_LAYOUT's k: 3 or 4)
void launch_pass(double2* state, const unsigned char* dev_rec, const PassHdr& h, uint64_t rankbase,
                 cudaStream_t s, int rbits);
void launch_init_basis(double2* a, uint64_t n, uint64_t one_at, cudaStream_t s);

size_t scratch_doubles_needed(uint64_t n);
int terms_per_launch();

void launch_sumsq(const double2* a, uint64_t n, double* scratch, double* out, cudaStream_t s);
// il = 1: the density matrix is in the interleaved layout (column bit q at
// physical 2q, row bit q at 2q + 1)
void launch_trace(const double2* rho, uint64_t dim, double* scratch, double* out, cudaStream_t s, int il = 0);
void launch_expect_sv(const double2* a, int nbits, uint64_t flip, const uint64_t* signs,
                      const int* eps_im, int nt, double* scratch, double* out, cudaStream_t s);
void launch_expect_dm(const double2* rho, int n, uint64_t flip, const uint64_t* signs, int nt,
                      double* scratch, double* out, cudaStream_t s, int il = 0);
// Tiled multi-term expectations (expect.cu): every term's flip mask lies in
// the tile bits q[0..m); sign masks are split into tile and full-index parts.
constexpr int kMaxExpTerms = 32;
struct ExpTerm {
    uint32_t ftile;   // flip mask on tile bits (0: Z-type term)
    uint32_t stile;   // sign mask on tile bits
    uint64_t sglob;   // sign mask on full-index bits outside the tile
    int32_t f0;       // lowest set bit of ftile
    int32_t eps_im;   // accumulate Im(conj(a[y^F]) a[y]) instead of Re
};
struct ExpBatch {
    int32_t m, nrest, nt, pad;
    int8_t q[16];
    int8_t rest[56];
    ExpTerm t[kMaxExpTerms];
};
size_t expect_tiled_scratch();
void launch_expect_tiled(const double2* a, int nloc, const ExpBatch& b, double* part, double* out, cudaStream_t s);
// out[t] = sum over nblk rows of part (row stride kMaxExpTerms), fixed order
void launch_expect_final(const double* part, int nblk, int nt, double* out, cudaStream_t s);

// batched trajectories (traj.cu)
constexpr int kMaxTrajQubits = 13;  // state in shared memory
constexpr int kMaxTrajKraus = 64;
struct TrajItem {
    int32_t type;  // 0 gate (one matrix), 1 channel (nmat Kraus matrices)
    int32_t k;     // <= 3 for trajectories, <= 4 in batches (2-qubit superoperators)
    int32_t q[4];
    int32_t nmat;
    int32_t pad;
    int64_t mat;  // offset into the matrix pool (complex elements)
};
struct TrajArgs {
    int n, nitems, nchannels, nterms;
    const TrajItem* items;
    const double2* pool;
    const double* uniforms;  // ntraj x nchannels
    const uint64_t* flip;
    const uint64_t* signs;
    double* out_re;  // ntraj x nterms
    double* out_im;
    int32_t* branch_out;  // ntraj x nchannels or null
    double2* amps_out;    // ntraj x 2^n or null
    int* err;             // set when a channel's branch weights do not sum to 1
};
void launch_traj(const TrajArgs& p, int64_t ntraj, cudaStream_t s);

// batches of independent small circuits (traj.cu): CTA b runs
// items[prog_off[b] .. prog_off[b+1]) on its own state from |0..0>
constexpr int kMaxBatchBits = 12;  // SV n <= 12, DM n <= 6
struct BatchArgs {
    int bits;  // state bits: SV n, DM 2n
    int n;     // qubits
    int dm;
    int nterms;
    const int64_t* prog_off;
    const TrajItem* items;
    const double2* pool;
    const uint64_t* flip;
    const uint64_t* signs;
    double* out_re;  // batch x nterms
    double* out_im;
    double* probs;  // batch x 2^n or null
};
void launch_batch(const BatchArgs& p, int64_t batch, cudaStream_t s);

// half-shard pack/unpack for global<->local qubit swaps (comm_kernels.cu)
void launch_half_pack(const double2* st, double2* buf, uint64_t k0, uint64_t len, int v, uint64_t val,
                      cudaStream_t s);
void launch_half_unpack(double2* st, const double2* buf, uint64_t k0, uint64_t len, int v, uint64_t val,
                        cudaStream_t s);
// mine[ins(k, v, mval)] <-> peer[ins(k, v, pval)] for k in [k0, k1) (peer: IPC-mapped)
void launch_swap_peer(double2* mine, double2* peer, int v, uint64_t mval, uint64_t pval, uint64_t k0, uint64_t k1,
                      cudaStream_t s);

void launch_probs(const double2* a, uint64_t n, double* p, cudaStream_t s);
void launch_dm_probs(const double2* rho, uint64_t dim, double* p, double* scratch, cudaStream_t s, int il = 0);
void launch_sum_real(const double* x, uint64_t n, double* scratch, double* out, cudaStream_t s);
void launch_herm(const double2* rho, uint64_t dim, double* scratch, double* out, cudaStream_t s);
void launch_kraus_weights(const double2* a, int nbits, const int* qubits, int k, int nk,
                          const double2* dev_mats, double* scratch, double* out, cudaStream_t s);
void launch_block_psum(const double2* a, const double* p, uint64_t n, uint64_t bs, double* out,
                       cudaStream_t s);
void launch_block_isum(const double2* a, const double* p, uint64_t n, uint64_t bs, const int* kb,
                       unsigned long long* isum, int* flags, cudaStream_t s);
void launch_block_sweep(const double2* a, const double* p, uint64_t n, uint64_t bs, const int64_t* blk,
                        const double* cum0, const int64_t* ulo, const int64_t* uhi, const double* u,
                        int nb, uint64_t* idx_out, uint64_t* cnt_out, int64_t* npairs, cudaStream_t s);
void launch_last_nonzero(const double2* a, const double* p, uint64_t lo, uint64_t hi, uint64_t* out,
                         cudaStream_t s);
void launch_readout(double* d, int n, int q, double p01, double p10, cudaStream_t s);

}  // namespace nqe

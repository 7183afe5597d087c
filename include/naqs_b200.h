/*
 * naqs_b200.h — C ABI of the B200-native SV/DM simulation core.
 *
 * This is the drop-in boundary.  The reference engine (naqs, a C++20 CPU
 * engine; /root/reference/proj) has no C ABI: its boundary is the C++ class
 * API in proj/include/naqs/{statevector,densitymatrix,noise}.hpp plus the
 * pybind11 module naqs._core (proj/python/bindings.cpp:52-273).  Our C++
 * mirror of that API (headers in include/naqs/) and our Python mirror call
 * ONLY the functions below; any other host language binds the same symbols
 * (see INTEGRATION.md for the ctypes / C++ bindings).
 *
 * Conventions (bit-exact with the reference):
 *   - amplitude index bit i is qubit i (proj/include/naqs/circuit.hpp:11-14);
 *   - for a k-qubit operator, local index bit j is qubits[j]
 *     (proj/src/gates.cpp:26-33), so CX control = qubits[0];
 *   - density matrices are row-major rho[r * 2^n + c]
 *     (proj/include/naqs/densitymatrix.hpp:30);
 *   - complex numbers are interleaved (re, im) doubles.
 *
 * Every function returns an nq_status.  On failure, nq_last_error() returns
 * a thread-local message; NQ_ERR_CONTRACT corresponds to naqs::ContractError
 * (precondition violated, nothing was modified), the others to naqs::Error.
 *
 * Execution model: gate/channel applications are validated eagerly and
 * queued; the queue is compiled by the fusion planner into tiled passes
 * and executed on the state's CUDA stream when a result is requested
 * (any reduction / readout / nq_*_flush).  Results are bit-identical run to
 * run (fixed grids, fixed-order reductions, no floating-point atomics).
 */
#ifndef NAQS_B200_H
#define NAQS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NAQS_B200_ABI_VERSION 1

typedef enum nq_status {
    NQ_OK = 0,
    NQ_ERR_CONTRACT = 1, /* precondition violated (naqs::ContractError) */
    NQ_ERR_CUDA = 2,     /* CUDA runtime / kernel failure            */
    NQ_ERR_NCCL = 3,     /* NCCL failure in a sharded state           */
    NQ_ERR_OOM = 4,      /* device allocation failed                  */
    NQ_ERR_INTERNAL = 5
} nq_status;

/* Gate kinds: same ordinals as naqs::GateKind (proj/include/naqs/circuit.hpp:15-37). */
typedef enum nq_gate_kind {
    NQ_X = 0, NQ_Y, NQ_Z, NQ_H, NQ_S, NQ_SDG, NQ_T, NQ_TDG, NQ_ID,
    NQ_RX, NQ_RY, NQ_RZ, NQ_U1, NQ_U2, NQ_U3,
    NQ_CX, NQ_CZ, NQ_SWAP, NQ_CCX,
    NQ_MEASURE, NQ_BARRIER
} nq_gate_kind;

/* One gate application; mirrors naqs::GateOp{kind, qubits, params}
 * (proj/include/naqs/circuit.hpp:56-60).  48 bytes, no padding surprises. */
typedef struct nq_op {
    int32_t kind;       /* nq_gate_kind                         */
    int32_t nqubits;    /* must equal the kind's arity          */
    int32_t qubits[3];  /* qubits[j] is local operator bit j    */
    int32_t reserved;
    double params[3];   /* radians; count = kind's param count  */
} nq_op;

/* One schedule item of a noise-compiled circuit (naqs::NoisySchedule,
 * proj/include/naqs/noise.hpp:124-146): either a gate (type 0) or a Kraus
 * channel (type 1) whose operators live in a shared pool:
 * nkraus matrices of 2^k x 2^k complex, row-major, starting at
 * kraus_pool[2 * kraus_offset]. */
typedef struct nq_sched_item {
    int32_t type;          /* 0 = gate, 1 = channel               */
    int32_t nkraus;        /* channel only                        */
    int64_t kraus_offset;  /* channel only, in complex elements   */
    nq_op op;              /* gate: the op; channel: kind ignored, nqubits/qubits used */
} nq_sched_item;

typedef struct nq_opts {
    int32_t device;       /* CUDA device ordinal; -1 = current                  */
    int32_t max_qubits;   /* 0 = reference guard (SV 30, DM 14); else the cap   */
    int32_t tile_qubits;  /* 0 = planner default                                */
    int32_t fuse;         /* 1 = fuse (default), 0 = one op per micro-step      */
} nq_opts;

typedef struct nq_sv nq_sv;
typedef struct nq_dm nq_dm;

/* ---- library ---------------------------------------------------------- */
const char* nq_last_error(void);
int nq_abi_version(void);
nq_status nq_device_count(int* out);
nq_status nq_default_opts(nq_opts* out);

/* ---- state vector (replaces naqs::StateVector, statevector.hpp:20-79) -- */
/* StateVector(int)  — statevector.hpp:24; guard 1 <= n <= max (default 30). */
nq_status nq_sv_create(int num_qubits, const nq_opts* opts, nq_sv** out);
nq_status nq_sv_destroy(nq_sv* s);
/* Copy constructor (value semantics; tests/test_statevector.cpp:218). */
nq_status nq_sv_clone(const nq_sv* s, nq_sv** out);
/* reset() — statevector.hpp:27 */
nq_status nq_sv_reset(nq_sv* s);
nq_status nq_sv_num_qubits(const nq_sv* s, int* out);
/* apply(op) / run(circuit) — statevector.hpp:35-38.  BARRIER is a no-op,
 * MEASURE is a contract error, qubits are range-checked (statevector.cpp:198-209). */
nq_status nq_sv_apply_ops(nq_sv* s, const nq_op* ops, int64_t count);
/* Apply an arbitrary 2^k x 2^k complex matrix (k <= 4) on `qubits`
 * (local bit j = qubits[j]); the kernel of detail::apply_matrix_inplace
 * (statevector.cpp:50-88).  Not required to be unitary. */
nq_status nq_sv_apply_matrix(nq_sv* s, const int32_t* qubits, int k, const double* mat);
/* Multiply every amplitude by a real scale (trajectory renormalisation). */
nq_status nq_sv_scale(nq_sv* s, double factor);
/* Execute everything queued. */
nq_status nq_sv_flush(nq_sv* s);
/* norm_sq() — statevector.cpp:224-239 */
nq_status nq_sv_norm_sq(nq_sv* s, double* out);
/* Batched Pauli expectations (statevector.cpp:241-277): term t has
 * flip = X|Y bits, signs = Y|Z bits, ny = number of Y letters; the result is
 * coeff[t] * Re(i^ny * sum_y (-1)^popcount(y & signs) conj(a[y^flip]) a[y]). */
nq_status nq_sv_expectation_batch(nq_sv* s, const uint64_t* flip, const uint64_t* signs,
                                  const int32_t* ny, const double* coeff, int nterms,
                                  double* out);
/* probabilities() — statevector.cpp:279-283; writes 2^n doubles to host. */
nq_status nq_sv_probabilities(nq_sv* s, double* host_out);
/* Sorted-uniform sampling sweep (statevector.cpp:302-331): `sorted_u` holds
 * `shots` ascending uniforms in [0,1).  Writes (basis index, count) pairs in
 * ascending index order; *nout <= shots.  Leftover uniforms (beyond the
 * final cumulative) go to the highest index with nonzero probability. */
nq_status nq_sv_sample_sorted(nq_sv* s, const double* sorted_u, uint64_t shots,
                              uint64_t* idx_out, uint64_t* count_out, uint64_t* nout);
/* Kraus branch weights ||K_i psi||^2 (statevector.cpp:355-366). `kraus` holds
 * nkraus matrices 2^k x 2^k complex row-major. */
nq_status nq_sv_kraus_weights(nq_sv* s, const int32_t* qubits, int k, int nkraus,
                              const double* kraus, double* weights_out);
/* Copy amplitudes [offset, offset+count) to host (interleaved re,im). */
nq_status nq_sv_get_amplitudes(nq_sv* s, uint64_t offset, uint64_t count, double* host_out);
/* Overwrite amplitudes [offset, offset+count) from host. */
nq_status nq_sv_set_amplitudes(nq_sv* s, uint64_t offset, uint64_t count, const double* host_in);
/* Device pointer to the (flushed) amplitude array, for zero-copy consumers
 * (sharded states: this rank's 2^(n-g) block, qubit map restored first). */
nq_status nq_sv_device_ptr(nq_sv* s, void** out);
/* Device probabilities |a_i|^2 (std::norm rounding) in a buffer owned by the
 * state, valid until the state is next modified or destroyed (zero-copy
 * replacement of probabilities(), proj/python/bindings.cpp:25-42; sharded
 * states: this rank's block). */
nq_status nq_sv_probabilities_device(nq_sv* s, double** out);
/* Global index of this rank's first amplitude and the number it holds
 * (0 and 2^n for single-device states). */
nq_status nq_sv_local_range(const nq_sv* s, uint64_t* offset, uint64_t* count);
/* CUDA device ordinal holding the state (for DLPack / CUDA-array consumers). */
nq_status nq_sv_device(const nq_sv* s, int* device);
nq_status nq_dm_device(const nq_dm* d, int* device);
/* Planner/executor statistics of the last flush: passes, fused micro-ops,
 * source ops, kernel launches. */
nq_status nq_sv_last_stats(const nq_sv* s, int64_t* passes, int64_t* microops,
                           int64_t* source_ops, int64_t* launches);
/* Wait for all work queued on the state's stream. */
nq_status nq_sv_synchronize(nq_sv* s);

/* ---- density matrix (replaces naqs::DensityMatrix, densitymatrix.hpp:16-65) */
nq_status nq_dm_create(int num_qubits, const nq_opts* opts, nq_dm** out);
nq_status nq_dm_destroy(nq_dm* d);
nq_status nq_dm_clone(const nq_dm* d, nq_dm** out);
/* Device pointer to row-major rho (rho[r * 2^n + c], densitymatrix.hpp:30),
 * flushed and in amplitude order; valid until the state is modified. */
nq_status nq_dm_device_ptr(nq_dm* d, void** out);
/* Device probabilities max(0, Re rho_ii) / trace (DensityMatrix::probabilities,
 * densitymatrix.cpp:221-232) in a state-owned buffer. */
nq_status nq_dm_probabilities_device(nq_dm* d, double** out);
nq_status nq_dm_reset(nq_dm* d);
nq_status nq_dm_num_qubits(const nq_dm* d, int* out);
/* apply(op) — densitymatrix.cpp:114-125: BARRIER and ID skipped, MEASURE rejected. */
nq_status nq_dm_apply_ops(nq_dm* d, const nq_op* ops, int64_t count);
/* apply_channel(ch, qubits) — densitymatrix.cpp:127-140 (arity 1 or 2).
 * Validation (dimensions, finiteness, completeness <= 1e-10) is the caller's
 * (naqs::validate_channel); identity channels may be skipped by the caller. */
nq_status nq_dm_apply_channel(nq_dm* d, const int32_t* qubits, int k, int nkraus,
                              const double* kraus);
/* run_schedule(schedule) — densitymatrix.cpp:154-167, compiled into fused
 * superoperator passes. */
nq_status nq_dm_apply_schedule(nq_dm* d, const nq_sched_item* items, int64_t count,
                               const double* kraus_pool);
nq_status nq_dm_flush(nq_dm* d);
/* trace / purity / hermiticity_residual — densitymatrix.cpp:169-190 */
nq_status nq_dm_trace(nq_dm* d, double* out);
nq_status nq_dm_purity(nq_dm* d, double* out);
nq_status nq_dm_hermiticity_residual(nq_dm* d, double* out);
/* expectation — densitymatrix.cpp:192-219.  out_re[t] = coeff * Re(...),
 * out_im[t] = Im(i^ny * sum ...) (before coeff) for the 1e-8 residue check. */
nq_status nq_dm_expectation_batch(nq_dm* d, const uint64_t* flip, const uint64_t* signs,
                                  const int32_t* ny, const double* coeff, int nterms,
                                  double* out_re, double* out_im);
/* probabilities — densitymatrix.cpp:221-232 (clip at 0, renormalise). */
nq_status nq_dm_probabilities(nq_dm* d, double* host_out);
/* Copy row-major entries [offset, offset+count) to host (interleaved). */
nq_status nq_dm_get_entries(nq_dm* d, uint64_t offset, uint64_t count, double* host_out);
nq_status nq_dm_set_entries(nq_dm* d, uint64_t offset, uint64_t count, const double* host_in);
nq_status nq_dm_last_stats(const nq_dm* d, int64_t* passes, int64_t* microops,
                           int64_t* source_ops, int64_t* launches);
nq_status nq_dm_synchronize(nq_dm* d);

/* ---- batched Monte-Carlo trajectories ---------------- */
/* ntraj independent run_trajectory() calls (statevector.cpp:339-401) of one
 * schedule in one launch, each from |0...0>.  Every channel item consumes one
 * uniform: trajectory t uses uniforms[t*C .. t*C+C) (C = channel items), which
 * is exactly the sequential loop over trajectories sharing one Rng
 * (acceptance_main.cpp:154-160).  Gates: MEASURE and BARRIER skipped as in
 * run_trajectory.  Outputs per trajectory: the Pauli expectations (as
 * nq_sv_expectation_batch) in out[t*nterms + j]; optionally the chosen Kraus
 * branch per channel (branch_out, ntraj*C) and the final amplitudes
 * (amps_out, ntraj * 2^n complex).  1 <= n <= 13.  A channel whose branch
 * weights do not sum to 1 within 1e-8 fails with NQ_ERR_CONTRACT (the
 * reference's trace-preservation check). */
nq_status nq_traj_run(int num_qubits, const nq_sched_item* items, int64_t count, const double* kraus_pool,
                      int64_t ntraj, const double* uniforms, const uint64_t* flip, const uint64_t* signs,
                      const int32_t* ny, const double* coeff, int nterms, double* out, int32_t* branch_out,
                      double* amps_out, int device);

/* ---- batches of small independent circuits --------- */
/* `batch` circuits, circuit b = items[item_off[b] .. item_off[b+1]), each run
 * from |0...0> in one launch (one CTA per circuit, state in shared memory).
 * dm = 0: ideal state vectors (gates only; n <= 12); out[b*nterms + j] as
 * nq_sv_expectation_batch, probs[b*2^n + i] = |a_i|^2.
 * dm = 1: density matrices with gates and channels as run_schedule
 * (densitymatrix.cpp:154-167; n <= 6, channel arity <= 2); out as
 * nq_dm_expectation_batch (out_im receives the imaginary residue, may be
 * NULL), probs as DensityMatrix::probabilities (clip at 0, renormalise).
 * MEASURE / BARRIER / ID items are skipped; probs may be NULL. */
nq_status nq_batch_run(int num_qubits, int dm, int64_t batch, const int64_t* item_off, const nq_sched_item* items,
                       const double* kraus_pool, const uint64_t* flip, const uint64_t* signs, const int32_t* ny,
                       const double* coeff, int nterms, double* out, double* out_im, double* probs, int device);

/* ---- readout (replaces readout_apply_dist, noise.cpp:177-203) --------- */
/* Tensor-product confusion map on a 2^n distribution, on the device.
 * Validates length implicitly (n) and sum within 1e-9 (contract error). */
nq_status nq_readout_apply_dist(const double* dist_in, int n, const double* p01,
                                const double* p10, double* dist_out);

/* ---- sampling an explicit distribution (sample_distribution,
 *      statevector.cpp:293-332): dist has `len` = 2^n entries in host memory;
 *      same sorted-uniform sweep as nq_sv_sample_sorted, run on the device. */
nq_status nq_sample_dist_sorted(const double* dist, uint64_t len, const double* sorted_u, uint64_t shots,
                                uint64_t* idx_out, uint64_t* count_out, uint64_t* nout);

/* ---- multi-GPU (new) ----------------------------------- */
/* NCCL unique id (128 bytes) for a sharded state; rank 0 creates it and the
 * caller distributes it (e.g. through torch.distributed's store). */
nq_status nq_comm_unique_id(unsigned char out[128]);
/* Sharded state vector of `num_qubits` total qubits over `world` ranks
 * (world a power of two): rank r owns amplitudes whose top log2(world)
 * logical-index bits equal r (until the planner remaps qubits).  All
 * collective functions below must be called by every rank. */
nq_status nq_sv_create_sharded(int num_qubits, int rank, int world, const unsigned char uid[128],
                               const nq_opts* opts, nq_sv** out);
/* Number of global-qubit exchanges performed so far and bytes sent. */
nq_status nq_sv_comm_stats(const nq_sv* s, int64_t* exchanges, int64_t* bytes_sent);
/* Of those exchanges, how many were fused into the preceding pass, and how:
 * *has_alt_buffer = 1: the pass writes out of place, the moved half straight
 * into the partner's second buffer over NVLink; 2: no second copy fits
 * (e.g. 2^33 amplitudes per GPU): staged -- kept half in place, moved half
 * chunk by chunk through a staging ring that a pusher kernel copies into the
 * partner's state as both ranks finish each chunk; 0: standalone swaps. */
nq_status nq_sv_comm_fused(const nq_sv* s, int64_t* fused, int* has_alt_buffer);
/* Host-side schedule of a sharded flush (no device, no NCCL): the segments of
 * local work and the global<->local exchanges `ops` would produce on `world`
 * ranks, followed by the exchanges restoring the identity qubit map.
 * flags bit 0: rebalance the segments around each exchange, as flushes do.
 * Serialised as int64 records (see paper_2401_06861_b200/abi.py:shard_debug). */
nq_status nq_shard_debug(int num_qubits, int world, const nq_op* ops, int64_t count, int flags, int64_t* buf,
                         int64_t cap, int64_t* size);

/* ---- measurement (bench.py) -------------------------------------------- */
typedef struct nq_profile {
    double region_ms;        /* device time between begin and end: CUDA events on the device stream */
    double pass_ms;          /* summed device time of the fused-pass kernel launches in the region  */
    int64_t pass_launches;
    double pass_bytes;       /* algorithmic bytes of those launches: 32 * 2^nloc each (read+write), */
                             /* 24 * 2^nloc for Hermitian DM mirror passes (half the reads)         */
    int64_t kernel_launches; /* every kernel this library launched in the region                     */
    int64_t h2d_bytes;       /* bytes this library copied host->device in the region                 */
    int64_t d2h_bytes;       /* bytes copied device->host                                            */
} nq_profile;
/* Start a measured region on `device`'s stream; with per_pass_events != 0
 * every pass launch is bracketed by CUDA events (pass_ms / pass_launches). */
nq_status nq_profile_begin(int device, int per_pass_events);
/* Synchronise and report the region. */
nq_status nq_profile_end(int device, nq_profile* out);

/* Run-time specialised pass kernels (NVRTC, cached per pass structure;
 * policy NQ_JIT=off|auto|sync).  Wait for queued compilations / counters. */
nq_status nq_jit_wait(void);
/* Cancel queued compilations and wait for running ones; later flushes use the
 * already compiled kernels or the generic ones.  Call before process exit
 * when compilations may be in flight (the Python packages do this at exit). */
nq_status nq_jit_shutdown(void);
nq_status nq_jit_stats(int64_t* compiled, int64_t* failed, int64_t* misses, int64_t* launches);
/* Generated source of pass `pass_index` of an SV plan, optionally compiled
 * with NVRTC (no device needed); *compiled_ok = 1/0, or -1 when not compiled.
 * compile: bit 0 = compile, bit 1 = the exchange-store variant (the kernel a
 * sharded flush fuses with a global-qubit exchange). */
nq_status nq_jit_debug(int num_qubits, const nq_op* ops, int64_t count, int tile_qubits, int pass_index,
                       int compile, char* src_out, int64_t cap, int64_t* size, int* compiled_ok);

/* ---- planner introspection (host logic, CPU-testable) ------------------ */
/* Compile `ops` on an n-qubit state into the pass plan without executing it
 * and serialise it (see paper_2401_06861_b200/plan_format.py).  Writes
 * at most `cap` bytes; *size receives the full size.  fuse: bit 0 = fusion,
 * bit 1 = relabelling stores (as single-device state vectors run). */
nq_status nq_plan_debug(int num_qubits, const nq_op* ops, int64_t count, int tile_qubits,
                        int fuse, unsigned char* buf, int64_t cap, int64_t* size);

#ifdef __cplusplus
}
#endif

#endif /* NAQS_B200_H */

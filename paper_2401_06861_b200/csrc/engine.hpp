// Internal engine structures shared by the planner (host C++), the kernels
// (CUDA) and the C ABI.  Nothing here crosses the public boundary.
//
// Design: a state of `nbits` bits (SV: n qubits; DM: vec(rho),
// 2n bits, column bits low) is processed by PASSES.  A pass picks a set Q of
// m "tile bits"; each CTA stages the 2^m amplitudes that share one value of
// the remaining bits in shared memory, applies every micro-op of the pass
// there, and writes the tile back: one HBM read + one write of the state per
// pass, whatever the number of gates fused into it.
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace nqe {

using cplx = std::complex<double>;

constexpr int kMaxTileBits = 13;   // 2^13 * 16 B = 128 KiB of shared memory
constexpr int kMaxStateBits = 48;
constexpr int kMaxOpK = 4;         // dense micro-ops act on <= 4 tile bits
constexpr int kMaxDiagK = 6;       // diagonal micro-ops act on <= 6 bits (64-entry table; 7-8 measured
                                    // worse: bigger tables fill the pass pools sooner)

// ---- device micro-ops ------------------------------------------------------
enum MOpType : uint8_t {
    MOP_DENSE = 0,  // 2^k x 2^k complex matrix on tile bits pos[0..k)
    MOP_DIAG = 1,   // 2^k diagonal; pos[j] >= 0: tile bit, else full-index bit -1-pos[j]
    MOP_XPERM = 2,  // X on tile bit pos[0], controlled by cmask_tile / cmask_glob
    MOP_SWAP = 3,   // swap tile bits pos[0], pos[1]
    MOP_DEPOL = 4,  // x[c,r] -> a x[c,r] + b d_{c,r} sum_l x[l,l] on k col + k row bits
    MOP_LAYOUT = 5, // register layout: slot j <-> tile bit pos[j] (j < k)
};
// Encoding of register-slot ops (everything but DIAG and LAYOUT): pos[] holds
// register SLOTS (0..3), not tile bits; matrices are permuted by the planner so
// that local operator bit j is the j-th smallest slot (DEPOL: pos = slots of
// [col bits..., row bits...]).  DIAG keeps tile bits / full-index bits.

struct MOp {
    uint8_t type;
    uint8_t k;            // number of operator bits (DEPOL: 2 or 4)
    int8_t pos[8];        // tile bit positions (DIAG: negative = full-index bit)
    uint16_t pad0;
    uint32_t mat;         // offset into the pass's complex pool
    uint32_t cmask_tile;  // controls on tile bits (XPERM)
    uint64_t cmask_glob;  // controls on full-index bits outside the tile
};
static_assert(sizeof(MOp) == 32, "MOp layout");

struct PassHdr {
    int32_t m;          // tile bits
    int32_t nops;
    int32_t nloc;       // local state bits (device array has 2^nloc amplitudes)
    int32_t nrest;      // number of non-tile local bits
    int64_t ntiles;     // 2^(nloc - m)
    uint32_t op_off;    // byte offset of MOp[nops] from the pass header
    uint32_t pool_off;  // byte offset of the complex pool from the pass header
    uint32_t pool_n;    // complex entries in the pool
    uint32_t bytes;     // total bytes of this pass record (header+ops+pool, 16B aligned)
    int8_t q[16];       // tile bit i is loaded from state bit q[i] (ascending)
    int8_t rest[56];    // non-tile state bits, ascending
    int8_t qst[16];     // tile bit i is stored to state bit qst[i] (a permutation of q:
                        // the pass relabels qubits among its tile bits for free)
    int32_t flags;      // PASS_MIRROR: Hermitian pass (density matrix, interleaved layout)
    int8_t lab[16];     // the content stored from tile bit i carries the logical qubit
                        // label of tile bit lab[i] (identity unless SWAP micro-ops were
                        // folded into qst; host-side bookkeeping, kernels ignore it)
    int32_t pad_[3];
};
// The pass maps Hermitian matrices to Hermitian matrices and its tile and rest
// bits pair up as physical bits (2q, 2q+1) = (column, row) of qubit q: only
// tiles whose rest index r <= mirror(r) are read, and each is also stored,
// conjugated and transposed, as its mirror tile.
constexpr int32_t PASS_MIRROR = 1;
static_assert(sizeof(PassHdr) % 16 == 0, "PassHdr alignment");

// ---- elementary ops (planner input) ----------------------------------------
enum EOpType : uint8_t {
    E_DENSE = 0,  // matrix on bits[0..k) (local bit j = bits[j])
    E_DIAG = 1,   // diagonal on bits[0..k)
    E_XPERM = 2,  // X on bits[0], controls in ctrl
    E_SWAP = 3,   // swap bits[0], bits[1]
    E_DEPOL = 4,  // depolarizing in Liouville form: bits = [cols..., rows...]; mat = {a, b}
    E_NOP = 5,    // counted but does nothing (ID)
};

struct EOp {
    EOpType type = E_NOP;
    int k = 0;
    int bits[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // DIAG up to kMaxDiagK bits
    uint64_t ctrl = 0;
    std::vector<cplx> mat;  // DENSE: 4^k, DIAG: 2^k, DEPOL: 2
    int64_t src = 1;        // source (reference) ops this elementary op accounts for
    bool pair_next = false; // DM: the row copy of a permutation; its column copy follows
};

struct PlanOptions {
    int nbits = 0;        // state bits seen by the planner (local + global)
    int nloc = 0;         // local bits (== nbits on one device)
    int tile_bits = 12;   // m
    int low_bits = 4;     // minimum contiguous low bits in every tile (coalescing)
    bool fuse = true;
    int reg_bits = 4;     // amplitudes per thread = 2^reg_bits (3 or 4)
    int max_ops_per_pass = 192;
    int max_pool_per_pass = 1536;  // complex entries
    // Relabel qubits at pass stores (single-device state vectors): the qubits
    // held by the low (contiguous) physical bits become a per-pass choice.
    bool relabel = false;
    // Reorder commuting micro-ops to reduce register-layout switches (state
    // vectors; measured slower on the Liouville programs of density matrices).
    bool stage_sched = true;
    // Density matrices in the interleaved layout: n qubits, logical column bit
    // q pairs with row bit q + n; tiles are kept closed under that pairing and
    // passes that apply whole superoperators are flagged PASS_MIRROR.
    int dm_mirror_n = 0;
};

struct PlannedPass {
    std::vector<int> q;     // tile bits (physical, ascending) at load
    std::vector<int> qst;   // physical store bit of tile bit i (empty: same as q)
    std::vector<int> lab;   // see PassHdr::lab (empty: identity)
    int32_t flags = 0;
    std::vector<MOp> ops;
    std::vector<cplx> pool;
};

struct PlanStats {
    int64_t passes = 0;
    int64_t microops = 0;
    int64_t source_ops = 0;
};

// Plan a sequence of elementary ops (all on local bits < nloc for the
// non-diagonal targets; diagonal/control bits may be >= nloc).
// ops are in logical bits; `map` (logical -> physical bit, size nbits) is the
// layout of the state before the first pass and receives the layout after the
// last one.  Without a map (or without opt.relabel) the layout is the identity
// and stays so.
std::vector<PlannedPass> plan_passes(const std::vector<EOp>& ops, const PlanOptions& opt,
                                     PlanStats* stats, std::vector<int>* map = nullptr);

// Serialise passes into one contiguous buffer of PassHdr records.
std::vector<unsigned char> serialize_passes(const std::vector<PlannedPass>& passes, int nloc,
                                            std::vector<size_t>* offsets);

// Helpers shared by SV/DM lowering.
void gate_matrix_2x2(int kind, const double* params, cplx out[4]);
bool gate_is_diagonal(int kind);

}  // namespace nqe

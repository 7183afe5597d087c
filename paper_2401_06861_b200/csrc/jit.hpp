// Run-time specialised pass kernels (jit.cpp).
#pragma once

#include "engine.hpp"
#include "kernels.hpp"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>

namespace nqe {

enum class JitMode { Off, Auto, Sync };

struct JitStats {
    int64_t compiled = 0;
    int64_t failed = 0;
    int64_t misses = 0;
    int64_t launches = 0;
};

JitMode jit_mode();


// CUDA source of the kernel specialised to one pass record.  xstore: the
// exchange-store variant (sharded states, see JitXStore).
struct JitXStore;
// Diagonal (Z-type) expectation terms fused into a pass's stores (the last
// pass of a flush whose result is read as <Z...> terms): the sum over the
// pass's output of |a|^2 (-1)^popcount(o & signs[k]), o the physical index an
// amplitude is stored to; one partial per CTA at part[b * kMaxExpTerms + k]
// (fixed order: the sum is deterministic), `grid` set by the launch.
struct JitEpilogue {
    int nterms = 0;
    uint64_t signs[8] = {};
    double* part = nullptr;
    int grid = 0;
};
std::string jit_source(const PassHdr& h, const MOp* ops, const cplx* pool, bool xstore = false,
                       const JitXStore* stage = nullptr, const JitEpilogue* epi = nullptr);

// A pass fused with a global<->local qubit exchange (shard.cpp): the pass
// reads the state in place and writes out of place; element o of its output
// goes to out_local[o] when (o & xmask) == xval, else to the partner rank's
// buffer out_remote[o ^ xmask] (peer memory over NVLink).  xrot: rest-bit
// position of the tile counter's lowest bit (interleaves local and remote tiles).
struct JitXStore {
    double2* out_local = nullptr;
    double2* out_remote = nullptr;
    uint64_t xmask = 0, xval = 0;
    int xrot = 0;
    // Staged form, for shards too large for a second copy (shard.cpp): the
    // kept half is stored in place (out_local = the state) and the outgoing
    // half into this rank's staging ring (out_remote) of `slots` slots of
    // slot_elems, from which the grid's last `pushers` CTAs copy it into the
    // partner's state once the partner has consumed that chunk.
    // Chunk of tile counter r: r >> cshift; an outgoing element o lands at
    // slot (chunk % slots), index compress(o) = o with the physical bits
    // chunk_bits | xmask removed (physical order kept: coalesced both ways).
    // pass_done[c] counts the tiles this rank stored in chunk c; a tile of
    // chunk c >= slots first waits for push_done[c - slots] == pushers.
    bool staged = false;
    int cshift = 0, slots = 2;
    uint64_t chunk_bits = 0;
    uint64_t slot_elems = 0;
    unsigned* pass_done = nullptr;
    const unsigned* push_done = nullptr;
    unsigned pushers = 0;  // pusher CTAs appended to the pass grid (cooperative launch)
    double2* peer = nullptr;            // the partner's state (peer memory)
    const unsigned* peer_done = nullptr;  // the partner's pass_done counters
};
// Physical positions of the chunk bits of a staged exchange pass: the rest
// positions the top (nrest - cshift) bits of the rotated tile counter drive.
uint64_t jit_stage_chunk_bits(const PassHdr& h, int xrot, int cshift);
// Compile (synchronously) the exchange-store kernel of a pass ahead of its
// launch, so that ranks meet at the exchange with their kernels ready; the
// number of its CTAs that can be co-resident on the device.
int jit_xstore_prepare(const PassHdr& h, const MOp* ops, const cplx* pool, int device, const JitXStore* xs);
// Whether a pass can run as an exchange-store kernel (deterministic: every
// rank decides alike from the same pass record).
bool jit_xstore_ok(const PassHdr& h, const MOp* ops);

// Launch the specialised kernel for this pass if it is compiled (queueing the
// compilation otherwise, or compiling inline under NQ_JIT=sync).  Returns
// false when the caller must run the interpreter kernel instead.
// With xs: compiled synchronously if needed; throws when it cannot run.
// memo (optional, in-place passes only): the compiled kernel remembered by
// the caller for this exact pass record (plan cache): when set, the source is
// not regenerated and looked up again.  It holds a reference to the JIT
// entry, so the entry outlives any later eviction from the JIT cache.
struct JitMemo {
    std::mutex mu;
    std::shared_ptr<void> entry;
};
bool jit_launch(double2* state, const unsigned char* dev_rec, const PassHdr& h, const MOp* ops, const cplx* pool,
                uint64_t rankbase, cudaStream_t s, int device, const JitXStore* xs = nullptr,
                JitMemo* memo = nullptr, JitEpilogue* epi = nullptr);

// Expectation batch kernel specialised to the batch's term structure: source,
// and launch (plus the per-term final sums into out[0..nt)); false when the
// caller must use the generic tiled kernel (not compiled yet, or mode off).
std::string expect_source(const ExpBatch& b);
bool jit_expect_launch(const double2* state, int nloc, const ExpBatch& b, double* part, double* out,
                       cudaStream_t s, int device);

// NVRTC compile without loading (CPU-testable); false + log on failure.
bool jit_compile_only(const std::string& src, std::string* log);

// Block until every queued compilation has finished.
void jit_wait();
// Drop queued compilations, wait for running ones and accept no new ones
// (process exit; also registered with atexit when the workers start).
void jit_shutdown();
JitStats jit_stats();

}  // namespace nqe

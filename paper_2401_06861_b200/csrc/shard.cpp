// Multi-GPU layer (subsystem 5; no counterpart in the reference, which is a
// single-process engine: SPEC.md:188 non-goal).  SURVEY.md §8e.
//
// One process per GPU.  The 2^n state is split over world = 2^g ranks by its
// top g PHYSICAL bits: rank r owns the 2^(n-g) amplitudes whose physical
// index has top bits r.  A logical->physical qubit map lets the layer move a
// qubit between global and local positions:
//   * diagonal ops and controls on global bits need no communication: the
//     pass kernels see the rank-extended index (rankbase = r << nloc);
//   * a non-diagonal op on a global bit first swaps that bit with a local
//     "victim" bit (the local qubit whose next non-diagonal use is farthest
//     away, Belady): partners r and r ^ 2^j exchange the half of their shard
//     whose victim bit differs from their own rank bit (pack -> ncclSend /
//     ncclRecv -> unpack, chunked through two bounce buffers).
// Reductions gather per-rank partials and add them in rank order (results do
// not depend on timing).  Readouts that expose the index order (amplitudes,
// sampling) first restore the identity map.
//
// Scheduling is pure host logic (schedule()) and is exported for CPU testing
// through nq_shard_debug().
#include "jit.hpp"
#include "kernels.hpp"
#include "knobs.hpp"
#include "nvtx.hpp"
#include "lower.hpp"
#include "state.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <deque>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace nqe {

// NCCL is resolved at first use (dlopen), not at link time: a process that
// also imports torch must share torch's libnccl.so.2 (a newer build than the
// system one), so we bind to whichever libnccl.so.2 is already loaded, else
// NQ_NCCL_LIB (set by paper_2401_06861_b200/abi.py to torch's copy when
// present), else the system library.
namespace {
struct NcclApi {
    decltype(&::ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&::ncclCommInitRank) CommInitRank = nullptr;
    decltype(&::ncclCommDestroy) CommDestroy = nullptr;
    decltype(&::ncclGroupStart) GroupStart = nullptr;
    decltype(&::ncclGroupEnd) GroupEnd = nullptr;
    decltype(&::ncclSend) Send = nullptr;
    decltype(&::ncclRecv) Recv = nullptr;
    decltype(&::ncclAllGather) AllGather = nullptr;
    decltype(&::ncclAllReduce) AllReduce = nullptr;
    decltype(&::ncclBroadcast) Broadcast = nullptr;
    decltype(&::ncclGetErrorString) GetErrorString = nullptr;
    decltype(&::ncclCommGetAsyncError) CommGetAsyncError = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) {
            const char* env = std::getenv("NQ_NCCL_LIB");
            if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
            return;
        }
#define NQ_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
        NQ_SYM(GetUniqueId, "ncclGetUniqueId");
        NQ_SYM(CommInitRank, "ncclCommInitRank");
        NQ_SYM(CommDestroy, "ncclCommDestroy");
        NQ_SYM(GroupStart, "ncclGroupStart");
        NQ_SYM(GroupEnd, "ncclGroupEnd");
        NQ_SYM(Send, "ncclSend");
        NQ_SYM(Recv, "ncclRecv");
        NQ_SYM(AllGather, "ncclAllGather");
        NQ_SYM(AllReduce, "ncclAllReduce");
        NQ_SYM(Broadcast, "ncclBroadcast");
        NQ_SYM(GetErrorString, "ncclGetErrorString");
        NQ_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef NQ_SYM
    });
    if (!api.CommInitRank) throw NqError{NQ_ERR_NCCL, "NCCL unavailable: " + err};
    return api;
}
}  // namespace

#define ncclGetUniqueId nccl().GetUniqueId
#define ncclCommInitRank nccl().CommInitRank
#define ncclCommDestroy nccl().CommDestroy
#define ncclGroupStart nccl().GroupStart
#define ncclGroupEnd nccl().GroupEnd
#define ncclSend nccl().Send
#define ncclRecv nccl().Recv
#define ncclAllGather nccl().AllGather
#define ncclAllReduce nccl().AllReduce
#define ncclBroadcast nccl().Broadcast
#define ncclGetErrorString nccl().GetErrorString

#define NCCL_TRY(expr)                                                                                 \
    do {                                                                                               \
        ncclResult_t nccl_try_r_ = (expr);                                                             \
        if (nccl_try_r_ != ncclSuccess)                                                                \
            throw NqError{NQ_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(nccl_try_r_)}; \
    } while (0)

// Errors NCCL reports asynchronously (a peer failed, a network/NVLink fault)
// surface here instead of as a later hang: checked after every exchange and
// sharded flush.
void check_async(ncclComm_t comm) {
    ncclResult_t st = ncclSuccess;
    if (!comm || !nccl().CommGetAsyncError) return;
    NCCL_TRY(nccl().CommGetAsyncError(comm, &st));
    if (st != ncclSuccess && st != ncclInProgress)
        throw NqError{NQ_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(st)};
}

// ---- host-coordinated ranks (NQ_COMM=host) -----------------------------------
// Ranks that are processes on one node -- possibly sharing ONE GPU, which is
// how the sharded parity tests run on a single-GPU box -- coordinate through
// a POSIX shared-memory block (a counting barrier, the CUDA-IPC handles of a
// per-rank collective buffer) instead of NCCL.  Collectives are then
// host-synchronous copies through those buffers; exchanges still go through
// peer memory.  Staged exchanges are off in this mode: two ranks' cooperative
// grids cannot be co-resident on one shared GPU.
struct HostShm {
    std::atomic<uint64_t> arrived;
    std::atomic<uint64_t> generation;
    cudaIpcMemHandle_t coll[64];
};

struct HostGroup {
    std::string name;
    HostShm* shm = nullptr;
    int world = 1, rank = 0;
    double* coll = nullptr;  // this rank's collective buffer
    size_t coll_cap = 0;     // doubles
    std::vector<double*> peer_coll;

    void barrier() const {
        const uint64_t g = shm->generation.load();
        if (shm->arrived.fetch_add(1) + 1 == uint64_t(world)) {
            shm->arrived.store(0);
            shm->generation.fetch_add(1);
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        while (shm->generation.load() == g) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
                throw NqError{NQ_ERR_INTERNAL, "host-coordinated ranks: barrier timed out (a rank stopped)"};
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    double* buf(int r) const { return r == rank ? coll : peer_coll[size_t(r)]; }
};

bool host_comm_requested() { return env_option_str("NQ_COMM") == "host"; }

HostGroup* host_group_create(const unsigned char uid[128], int rank, int world) {
    auto g = std::make_unique<HostGroup>();
    g->world = world;
    g->rank = rank;
    char hex[33];
    for (int i = 0; i < 16; ++i) std::snprintf(hex + 2 * i, 3, "%02x", uid[i]);
    g->name = std::string("/naqs_b200_") + hex;
    const int fd = shm_open(g->name.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0) throw NqError{NQ_ERR_INTERNAL, "host-coordinated ranks: shm_open failed"};
    if (ftruncate(fd, sizeof(HostShm)) != 0) {
        close(fd);
        throw NqError{NQ_ERR_INTERNAL, "host-coordinated ranks: ftruncate failed"};
    }
    void* p = mmap(nullptr, sizeof(HostShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw NqError{NQ_ERR_INTERNAL, "host-coordinated ranks: mmap failed"};
    g->shm = static_cast<HostShm*>(p);  // zero-filled by ftruncate
    g->coll_cap = size_t(1) << 23;     // 64 MiB of doubles per rank
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&g->coll), g->coll_cap * sizeof(double)));
    CUDA_TRY(cudaIpcGetMemHandle(&g->shm->coll[rank], g->coll));
    g->barrier();
    g->peer_coll.assign(size_t(world), nullptr);
    for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        void* q = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&q, g->shm->coll[r], cudaIpcMemLazyEnablePeerAccess));
        g->peer_coll[size_t(r)] = static_cast<double*>(q);
    }
    g->barrier();
    return g.release();
}

void host_group_free(HostGroup* g) {
    if (!g) return;
    for (double* q : g->peer_coll)
        if (q) cudaIpcCloseMemHandle(q);
    if (g->coll) cudaFree(g->coll);
    if (g->rank == 0) shm_unlink(g->name.c_str());
    munmap(g->shm, sizeof(HostShm));
    delete g;
}

struct ShardComm {
    ncclComm_t comm = nullptr;
    HostGroup* hg = nullptr;  // NQ_COMM=host: no NCCL communicator
    std::vector<EOp> prev_ops;  // the previous flush (logical), for repeat prediction
    // peer-memory exchange: every rank's state mapped into this process (CUDA
    // IPC over NVLink); empty when unavailable or NQ_EXCHANGE=nccl
    std::vector<double2*> peer;
    // fused exchanges (NQ_FUSED_EXCHANGE, default on when a second copy of the
    // shard fits): the pass before an exchange writes its output out of place,
    // locally into `alt` and remotely into the partner's `alt` (peer_alt), and
    // the two buffers swap roles on every rank.
    double2* alt = nullptr;
    std::vector<double2*> peer_alt;
    int64_t fused = 0;
    // staged fused exchanges (no room for `alt`, e.g. 2^33 amplitudes per
    // GPU): a ring of `stage_slots` staging slots for the outgoing half,
    // per-chunk counters (pass_done[kMaxChunks], push_done[kMaxChunks]) mapped
    // into the partner, and the pusher's descriptor
    static constexpr int kMaxChunks = 256;
    double2* stage = nullptr;
    uint64_t stage_slot_elems = 0;
    int stage_slots = 4, stage_chunks = 0;
    unsigned* sync = nullptr;
    std::vector<unsigned*> peer_sync;
    int64_t staged = 0;
    std::unordered_map<uint64_t, std::vector<int>> rebalance_cache;  // see rebalance()
    // planned segments of recent flushes (repeated circuits replan nothing and
    // reuse their kernels): key = segment ops incl. matrices + plan options
    struct SegPlan {
        std::vector<PlannedPass> passes;
        PlanStats st;
        std::shared_ptr<std::vector<JitMemo>> kern;
    };
    std::deque<std::pair<std::vector<unsigned char>, std::shared_ptr<SegPlan>>> seg_cache;  // acts_key -> ops moved per exchange
    double* d_flag = nullptr;  // 1-element buffer for the stream barrier
    double* gather = nullptr;  // allgather_doubles buffer
    size_t gather_cap = 0;
    double* bcast = nullptr;   // shard_probabilities chunk buffer
    size_t bcast_cap = 0;
    double2* sendbuf = nullptr;
    double2* recvbuf = nullptr;
    uint64_t chunk = 0;  // amplitudes per bounce buffer
    std::vector<int> l2p, p2l;
    int64_t exchanges = 0, bytes = 0;
};

// NQ_SHARD_TIMING=<ms>: report host phases of sharded calls slower than that.
struct PhaseTimer {
    const char* name;
    int rank;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    PhaseTimer(const char* n, int r) : name(n), rank(r) {}
    ~PhaseTimer() {
        static const double thresh = [] {
            const char* e = std::getenv("NQ_SHARD_TIMING");
            return e ? std::atof(e) : -1.0;
        }();
        if (thresh < 0) return;
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms >= thresh) std::fprintf(stderr, "[shard-timing] rank %d %s %.2f ms\n", rank, name, ms);
    }
};

// ---- host scheduling ----------------------------------------------------------
struct Action {
    enum Kind { Segment, Exchange } kind;
    std::vector<EOp> ops;  // Segment: ops in physical bits
    int gbit = 0, vbit = 0;  // Exchange: swap physical global bit gbit with local vbit
};

namespace {

uint64_t emask(const EOp& e, bool ctrl) {
    uint64_t m = 0;
    for (int j = 0; j < e.k; ++j) m |= uint64_t(1) << e.bits[j];
    if (ctrl) m |= e.ctrl;
    return m;
}

// bits that must be local (non-diagonal targets), as in the planner
uint64_t need_bits(const EOp& e) {
    switch (e.type) {
    case E_DENSE:
    case E_DEPOL:
    case E_SWAP:
        return emask(e, false);
    case E_XPERM:
        return uint64_t(1) << e.bits[0];
    default:
        return 0;
    }
}

EOp to_physical(const EOp& e, const std::vector<int>& l2p) {
    EOp p = e;
    for (int j = 0; j < e.k; ++j) p.bits[j] = l2p[size_t(e.bits[j])];
    uint64_t c = 0;
    for (int b = 0; b < 64; ++b)
        if ((e.ctrl >> b) & 1) c |= uint64_t(1) << l2p[size_t(b)];
    p.ctrl = c;
    return p;
}

void swap_map(std::vector<int>& l2p, std::vector<int>& p2l, int pa, int pb) {
    const int la = p2l[size_t(pa)], lb = p2l[size_t(pb)];
    p2l[size_t(pa)] = lb;
    p2l[size_t(pb)] = la;
    l2p[size_t(la)] = pb;
    l2p[size_t(lb)] = pa;
}

// Local physical bit to evict for global bit `g`: not needed by `protect`
// (logical mask), farthest next non-diagonal use in ops[from..].
int choose_victim(const std::vector<EOp>& ops, size_t from, const std::vector<int>& p2l, int nloc,
                  uint64_t protect_logical) {
    int best = -1;
    size_t best_dist = 0;
    for (int v = nloc - 1; v >= 0; --v) {
        const int lq = p2l[size_t(v)];
        if ((protect_logical >> lq) & 1) continue;
        size_t d = ops.size() + 1;  // never used again
        for (size_t i = from; i < ops.size(); ++i)
            if ((need_bits(ops[i]) >> lq) & 1) {
                d = i;
                break;
            }
        if (best < 0 || d > best_dist) {
            best = v;
            best_dist = d;
        }
    }
    if (best < 0) throw NqError{NQ_ERR_INTERNAL, "sharded: no local qubit available to swap in"};
    return best;
}

}  // namespace

// NQ_SHARD_CYCLIC=1 enables the repeat prediction of schedule().  Off by
// default: on the random-circuit benchmark it cut exchanges but made the
// carried qubit map cycle through many layouts (uncompiled pass structures):
// N = 4 with 33 local qubits 661 -> 1012, but with 30 local 9050 -> 4779.
bool shard_cyclic_enabled() {
    static const bool on = ab_knob("NQ_SHARD_CYCLIC", 0) == 1;
    return on;
}

// Split a queue (logical bits) into segments of local work and exchanges,
// updating the qubit map as the exchanges will.
std::vector<Action> schedule(const std::vector<EOp>& ops, std::vector<int>& l2p, std::vector<int>& p2l, int nloc,
                             bool repeat) {
    // A flush that repeats the previous one (same op structure: iterative
    // workloads, benchmark steps) is predicted to be followed by itself: the
    // victims' next uses are looked up in this flush's remainder and then in
    // the predicted next flush, so a qubit needed at the start of the next
    // repetition is not evicted at the end of this one.
    std::vector<EOp> ext;
    if (repeat) {
        ext = ops;
        ext.insert(ext.end(), ops.begin(), ops.end());
    }
    const std::vector<EOp>& future = repeat ? ext : ops;
    std::vector<Action> acts;
    Action seg{Action::Segment, {}, 0, 0};
    const uint64_t loc_mask = (uint64_t(1) << nloc) - 1;
    for (size_t i = 0; i < ops.size(); ++i) {
        EOp p = to_physical(ops[i], l2p);
        uint64_t glob = need_bits(p) & ~loc_mask;
        if (glob) {
            if (!seg.ops.empty()) acts.push_back(std::move(seg));
            seg = Action{Action::Segment, {}, 0, 0};
            const uint64_t protect = emask(ops[i], false);
            while (glob) {
                const int g = __builtin_ctzll(glob);
                glob &= glob - 1;
                const int v = choose_victim(future, i + 1, p2l, nloc, protect);
                acts.push_back(Action{Action::Exchange, {}, g, v});
                swap_map(l2p, p2l, g, v);
            }
            p = to_physical(ops[i], l2p);
        }
        seg.ops.push_back(std::move(p));
    }
    if (!seg.ops.empty()) acts.push_back(std::move(seg));
    return acts;
}

// Exchanges that restore the identity map (physical bit p holds logical p).
std::vector<Action> schedule_identity(std::vector<int>& l2p, std::vector<int>& p2l, int nloc, int n) {
    std::vector<Action> acts;
    for (int p = n - 1; p >= 0; --p) {
        if (p2l[size_t(p)] == p) continue;
        const int w = l2p[size_t(p)];  // where logical p currently lives
        const bool pg = p >= nloc, wg = w >= nloc;
        if (!pg && !wg) {
            EOp s;
            s.type = E_SWAP;
            s.k = 2;
            s.bits[0] = p;
            s.bits[1] = w;
            s.src = 0;
            acts.push_back(Action{Action::Segment, {s}, 0, 0});
        } else if (pg != wg) {
            acts.push_back(Action{Action::Exchange, {}, pg ? p : w, pg ? w : p});
        } else {
            // two global bits: (p w) = (p l)(w l)(p l) through local bit 0
            acts.push_back(Action{Action::Exchange, {}, p, 0});
            acts.push_back(Action{Action::Exchange, {}, w, 0});
            acts.push_back(Action{Action::Exchange, {}, p, 0});
        }
        swap_map(l2p, p2l, p, w);
    }
    return acts;
}

// ---- device execution ------------------------------------------------------------
namespace {

__attribute__((unused)) uint64_t ins_bit(uint64_t k, int v, uint64_t val) {
    return ((k >> v) << (v + 1)) | (val << v) | (k & ((uint64_t(1) << v) - 1));
}

// `layout` (physical -> physical, size n): identity on entry; with relabelling
// passes it receives where each local physical bit's qubit ends up.
struct FuseX {
    int v = 0;           // local physical bit exchanged with the global bit
    uint64_t mybit = 0;  // this rank's value of that global bit
    int partner = 0;
    bool staged = false;  // staged form: in place + staging ring + pusher
    double2* out_local = nullptr;
    double2* out_remote = nullptr;
    bool done = false;   // set when the segment's last pass carried the exchange
};

// Rest position of physical bit v in a pass (0 when v is a tile bit).
int rest_pos(const PassHdr& h, int v) {
    for (int j = 0; j < h.nrest; ++j)
        if (h.rest[j] == v) return j;
    return 0;
}

std::vector<unsigned char> segment_key(const PlanOptions& o, const std::vector<EOp>& ops) {
    std::vector<unsigned char> k;
    auto put = [&](const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        k.insert(k.end(), b, b + n);
    };
    const int32_t opts[] = {o.nbits, o.nloc, o.tile_bits, o.low_bits, o.fuse, o.reg_bits, o.max_ops_per_pass,
                            o.max_pool_per_pass, o.stage_sched};
    put(opts, sizeof opts);
    for (const EOp& e : ops) {
        const int32_t head[] = {int32_t(e.type), e.k, e.pair_next, int32_t(e.mat.size())};
        put(head, sizeof head);
        put(e.bits, size_t(e.k) * sizeof(int));
        put(&e.ctrl, sizeof e.ctrl);
        put(&e.src, sizeof e.src);
        if (!e.mat.empty()) put(e.mat.data(), e.mat.size() * sizeof(cplx));
    }
    return k;
}

void stream_barrier(ShardComm& sc, DeviceCtx& c);

// A pass fused with an exchange when no second copy of the shard fits: one
// cooperative grid whose pass CTAs store the kept half in place and the
// outgoing half chunk by chunk into the staging ring, while its last CTAs
// (the pusher) copy each chunk into the partner's state as soon as both
// ranks have stored it -- NVLink traffic overlaps the pass.
bool launch_staged_exchange(State& s, DeviceCtx& c, const PassHdr& h, const MOp* mops, const cplx* pool,
                            const unsigned char* dev_rec, uint64_t rankbase, JitXStore xs, const FuseX& fx) {
    ShardComm& sc = *s.comm;
    // pusher CTAs appended to the pass grid (one co-resident cooperative
    // launch): enough bytes in flight to keep NVLink busy
    static const unsigned kPushers = unsigned(ab_knob("NQ_STAGE_PUSHERS", 224));
    const int chunks = sc.stage_chunks;
    int cb = 0;
    while ((1 << cb) < chunks) ++cb;
    const int cshift = h.nrest - cb;
    if (cshift < 1) throw NqError{NQ_ERR_INTERNAL, "staged exchange: too few tiles for the chunk count"};
    xs.staged = true;
    xs.cshift = cshift;
    xs.slots = sc.stage_slots;
    xs.chunk_bits = jit_stage_chunk_bits(h, xs.xrot, cshift);
    xs.slot_elems = s.count / 2 / uint64_t(chunks);
    xs.pass_done = sc.sync;
    xs.push_done = sc.sync + ShardComm::kMaxChunks;
    xs.pushers = kPushers;
    xs.peer = sc.peer[size_t(fx.partner)];
    xs.peer_done = sc.peer_sync[size_t(fx.partner)];
    if (xs.slot_elems != sc.stage_slot_elems) throw NqError{NQ_ERR_INTERNAL, "staged exchange: slot size mismatch"};
    // pusher descriptor (sync words 598..647): [vval, nholes, pos[24], src[24]];
    // holes = the chunk bits (source: a bit of the chunk number) and v, whose
    // value on the partner's side is this rank's bit
    unsigned desc[50] = {};
    {
        std::vector<std::pair<int, int>> holes;
        for (int i = 0; i < cb; ++i) {
            const int j = cshift + i;
            holes.push_back({h.rest[j <= xs.xrot ? j - 1 : j], i});
        }
        holes.push_back({fx.v, -1});
        std::sort(holes.begin(), holes.end());
        desc[0] = unsigned(fx.mybit);
        desc[1] = unsigned(holes.size());
        for (size_t k = 0; k < holes.size(); ++k) {
            desc[2 + k] = unsigned(holes[k].first);
            desc[26 + k] = unsigned(holes[k].second);
        }
    }
    if (std::getenv("NQ_SHARD_TRACE")) {
        std::string hs;
        for (unsigned k = 0; k < desc[1]; ++k) hs += " " + std::to_string(desc[2 + k]) + ":" + std::to_string(int(desc[26 + k]));
        std::fprintf(stderr, "[shard] rank %d staged exchange v=%d partner=%d m=%d nrest=%d ntiles=%lld cshift=%d "
                     "chunks=%d slot=%llu xrot=%d holes%s\n", s.rank, fx.v, fx.partner, h.m, h.nrest,
                     (long long)h.ntiles, cshift, chunks, (unsigned long long)xs.slot_elems, xs.xrot, hs.c_str());
    }
    // kernel compiled and loaded before the ranks meet (a rank still
    // compiling would stall its partner), counters zeroed on every rank
    // before any rank's pusher reads them
    // the grid (pass CTAs + pushers) must be co-resident with room for the
    // pass: every rank decides alike (same pass, same device type)
    if (jit_xstore_prepare(h, mops, pool, s.dev, &xs) < int(kPushers) + 148) return false;
    CUDA_TRY(cudaMemsetAsync(sc.sync, 0, sizeof(unsigned) * (2 * ShardComm::kMaxChunks + 16), c.stream));
    CUDA_TRY(cudaMemcpyAsync(sc.sync + 598, desc, sizeof desc, cudaMemcpyHostToDevice, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));  // desc is a host stack array
    stream_barrier(sc, c);
    jit_launch(s.d, dev_rec, h, mops, pool, rankbase, c.stream, s.dev, &xs);
    CUDA_TRY(cudaGetLastError());
    return true;
}

void run_segment(State& s, DeviceCtx& c, const std::vector<EOp>& ops, std::vector<int>* layout = nullptr,
                 FuseX* fx = nullptr) {
    PlanOptions po = s.popt;
    po.relabel = layout != nullptr;
    PlanStats st;
    std::vector<PlannedPass> passes;
    std::shared_ptr<std::vector<JitMemo>> kern;
    if (layout == nullptr) {
        ShardComm& sc = *s.comm;
        std::vector<unsigned char> key = segment_key(po, ops);
        for (auto it = sc.seg_cache.begin(); it != sc.seg_cache.end(); ++it) {
            if (it->first != key) continue;
            passes = it->second->passes;
            st = it->second->st;
            kern = it->second->kern;
            break;
        }
        if (!kern) {
            passes = plan_passes(ops, po, &st, nullptr);
            auto sp = std::make_shared<ShardComm::SegPlan>();
            sp->passes = passes;
            sp->st = st;
            sp->kern = std::make_shared<std::vector<JitMemo>>(passes.size());
            kern = sp->kern;
            sc.seg_cache.emplace_front(std::move(key), std::move(sp));
            if (sc.seg_cache.size() > 16) sc.seg_cache.pop_back();
        }
    } else {
        passes = plan_passes(ops, po, &st, layout);
    }
    if (s.rank == 0 && std::getenv("NQ_SHARD_TRACE"))
        std::fprintf(stderr, "[shard] segment: %zu ops -> %lld passes\n", ops.size(), (long long)st.passes);
    std::vector<size_t> offs;
    std::vector<unsigned char> buf = serialize_passes(passes, s.nloc, &offs);
    s.last_passes += st.passes;
    s.last_microops += st.microops;
    s.last_source_ops += st.source_ops;
    s.last_launches += int64_t(passes.size());
    if (buf.empty()) return;
    {
        PhaseTimer ps("stage", s.rank);
        c.stage(buf.data(), buf.size());
    }
    PhaseTimer pl("launches", s.rank);
    const uint64_t rankbase = uint64_t(s.rank) << s.nloc;
    for (size_t i = 0; i < passes.size(); ++i) {
        NvtxRange pass_range("nq.pass", int64_t(i));
        PassHdr h;
        std::memcpy(&h, buf.data() + offs[i], sizeof(h));
        std::pair<cudaEvent_t, cudaEvent_t>* ev = c.prof_pass ? prof_slot(c) : nullptr;
        if (ev) CUDA_TRY(cudaEventRecord(ev->first, c.stream));
        const unsigned char* rec = buf.data() + offs[i];
        const MOp* mops = reinterpret_cast<const MOp*>(rec + h.op_off);
        if (fx && i + 1 == passes.size() && layout == nullptr && jit_xstore_ok(h, mops)) {
            JitXStore xs;
            xs.out_local = fx->out_local;
            xs.out_remote = fx->out_remote;
            xs.xmask = uint64_t(1) << fx->v;
            xs.xval = fx->mybit << fx->v;
            xs.xrot = rest_pos(h, fx->v);
            if (fx->staged) {
                fx->done = launch_staged_exchange(s, c, h, mops, reinterpret_cast<const cplx*>(rec + h.pool_off),
                                                  c.d_ops + offs[i], rankbase, xs, *fx);
                if (!fx->done && !jit_launch(s.d, c.d_ops + offs[i], h, mops,
                                             reinterpret_cast<const cplx*>(rec + h.pool_off), rankbase, c.stream,
                                             s.dev, nullptr, kern ? kern->data() + i : nullptr))
                    launch_pass(s.d, c.d_ops + offs[i], h, rankbase, c.stream, mops[0].k);
            } else {
                jit_launch(s.d, c.d_ops + offs[i], h, mops, reinterpret_cast<const cplx*>(rec + h.pool_off), rankbase,
                           c.stream, s.dev, &xs);
                fx->done = true;
            }
        } else if (!jit_launch(s.d, c.d_ops + offs[i], h, mops,
                        reinterpret_cast<const cplx*>(rec + h.pool_off), rankbase, c.stream, s.dev, nullptr,
                        kern ? kern->data() + i : nullptr))
            launch_pass(s.d, c.d_ops + offs[i], h, rankbase, c.stream,
                        reinterpret_cast<const MOp*>(rec + h.op_off)[0].k);
        if (ev) CUDA_TRY(cudaEventRecord(ev->second, c.stream));
        if (c.prof) c.prof_pass_bytes += 32.0 * double(s.count);
    }
    CUDA_TRY(cudaGetLastError());
}

// Device-side barrier: a one-element all-reduce completes only after every
// rank's stream has reached it, so no rank touches a peer's state while that
// peer's earlier kernels may still be running (and vice versa afterwards).
void stream_barrier(ShardComm& sc, DeviceCtx& c) {
    if (sc.hg) {
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        sc.hg->barrier();
        return;
    }
    NCCL_TRY(ncclAllReduce(sc.d_flag, sc.d_flag, 1, ncclDouble, ncclSum, sc.comm, c.stream));
}

void run_exchange(State& s, DeviceCtx& c, int g, int v) {
    ShardComm& sc = *s.comm;
    NvtxRange range("nq.exchange", g);
    if (s.rank == 0 && std::getenv("NQ_SHARD_TRACE")) std::fprintf(stderr, "[shard] exchange g=%d v=%d\n", g, v);
    const int j = g - s.nloc;
    const int partner = s.rank ^ (1 << j);
    const uint64_t mybit = uint64_t((s.rank >> j) & 1);
    const uint64_t half = s.count / 2;
    if (!sc.peer.empty()) {
        // One kernel per rank swaps its share of the element pairs directly in
        // both states over NVLink: no bounce buffers, no pack / unpack passes.
        // Pair k: my element with bit v = 1 - mybit <-> the partner's with bit v = mybit.
        stream_barrier(sc, c);
        const uint64_t k0 = mybit ? half / 2 : 0, k1 = mybit ? half : half / 2;
        launch_swap_peer(s.d, sc.peer[size_t(partner)], v, 1 - mybit, mybit, k0, k1, c.stream);
        stream_barrier(sc, c);
        CUDA_TRY(cudaGetLastError());
        sc.bytes += int64_t(half) * 16;
        ++sc.exchanges;
        check_async(sc.comm);
        return;
    }
    if (sc.hg) throw NqError{NQ_ERR_INTERNAL, "host-coordinated ranks need CUDA-IPC peer memory for exchanges"};
    for (uint64_t k0 = 0; k0 < half; k0 += sc.chunk) {
        const uint64_t len = std::min(sc.chunk, half - k0);
        launch_half_pack(s.d, sc.sendbuf, k0, len, v, 1 - mybit, c.stream);
        NCCL_TRY(ncclGroupStart());
        NCCL_TRY(ncclSend(sc.sendbuf, size_t(len) * 2, ncclDouble, partner, sc.comm, c.stream));
        NCCL_TRY(ncclRecv(sc.recvbuf, size_t(len) * 2, ncclDouble, partner, sc.comm, c.stream));
        NCCL_TRY(ncclGroupEnd());
        launch_half_unpack(s.d, sc.recvbuf, k0, len, v, 1 - mybit, c.stream);
        sc.bytes += int64_t(len) * 16;
    }
    CUDA_TRY(cudaGetLastError());
    ++sc.exchanges;
    check_async(sc.comm);
}

// After a pass fused with the exchange (g, v): every rank wrote its output
// into the `alt` buffers, so the buffers swap roles; the barrier keeps any
// rank from reading its new state before its partner's stores have landed
// (and, as no rank touches its old buffer again before the next exchange,
// no barrier is needed before such a pass).
void fused_exchange_done(State& s, DeviceCtx& c, int g, int v, bool staged = false) {
    ShardComm& sc = *s.comm;
    NvtxRange range("nq.exchange.fused", g);
    if (s.rank == 0 && std::getenv("NQ_SHARD_TRACE"))
        std::fprintf(stderr, "[shard] exchange g=%d v=%d (fused into the pass)\n", g, v);
    if (staged) {
        ++sc.staged;  // in place: the partner's pusher wrote into this state
        // watchdog record of the bounded waits (pass kernel / pusher)
        unsigned err = 0;
        CUDA_TRY(cudaMemcpyAsync(&err, sc.sync + 2 * ShardComm::kMaxChunks, sizeof err, cudaMemcpyDeviceToHost,
                                 c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        if (err) {
            std::vector<unsigned> cnt(2 * size_t(sc.stage_chunks));
            cudaMemcpy(cnt.data(), sc.sync, sc.stage_chunks * sizeof(unsigned), cudaMemcpyDeviceToHost);
            cudaMemcpy(cnt.data() + sc.stage_chunks, sc.sync + ShardComm::kMaxChunks,
                       sc.stage_chunks * sizeof(unsigned), cudaMemcpyDeviceToHost);
            std::string d;
            for (int i = 0; i < sc.stage_chunks; ++i)
                d += " " + std::to_string(cnt[size_t(i)]) + "/" + std::to_string(cnt[size_t(sc.stage_chunks + i)]);
            // the partner's counters as this rank sees them through the mapping
            std::vector<unsigned> pc(size_t(sc.stage_chunks), 0u);
            for (size_t r = 0; r < sc.peer_sync.size(); ++r)
                if (sc.peer_sync[r]) {
                    cudaMemcpy(pc.data(), sc.peer_sync[r], pc.size() * sizeof(unsigned), cudaMemcpyDeviceToHost);
                    d += " | peer " + std::to_string(r) + ":";
                    for (int i = 0; i < std::min(8, sc.stage_chunks); ++i) d += " " + std::to_string(pc[size_t(i)]);
                }
            cudaGetLastError();
            char head[96];
            std::snprintf(head, sizeof head, "staged exchange stalled (rank %d, record 0x%x); pass/push per chunk:",
                          s.rank, err);
            throw NqError{NQ_ERR_INTERNAL, head + d};
        }
    } else {
        std::swap(s.d, sc.alt);
        std::swap(sc.peer, sc.peer_alt);
    }
    stream_barrier(sc, c);
    CUDA_TRY(cudaGetLastError());
    sc.bytes += int64_t(s.count / 2) * 16;
    ++sc.exchanges;
    ++sc.fused;
    check_async(sc.comm);
}

// Relabelling passes permute local physical bits inside a segment; the later
// actions (scheduled on the pre-relabel bits) are remapped through `perm`,
// and the composed permutation is folded into the shard's qubit map.
// NQ_SHARD_RELABEL_RESTORE=0: keep a segment's final relabelling (composed
// into the qubit map) instead of restoring it inside the segment.
bool shard_relabel_restore() {
    static const bool on = ab_knob("NQ_SHARD_RELABEL_RESTORE", 1) != 0;
    return on;
}

EOp remap(const EOp& e, const std::vector<int>& perm) {
    EOp r = e;
    for (int j = 0; j < e.k; ++j) r.bits[j] = perm[size_t(e.bits[j])];
    uint64_t c = 0;
    for (int b = 0; b < 64; ++b)
        if ((e.ctrl >> b) & 1) c |= uint64_t(1) << perm[size_t(b)];
    r.ctrl = c;
    return r;
}

// ---- segment rebalancing around exchanges ---------------------------------------
// An exchange (g, v) only relabels the qubits at physical bits g and v, so an
// op of the segment before it that does not need bit v as a non-diagonal
// target, and commutes with the ops of that segment it would pass, can run
// after it instead (its bits translated g <-> v).  Where the split falls
// decides the pass count of the two segments (each ends in a partly filled
// pass; the one before an exchange also carries it as its exchange store), so
// for every Segment-Exchange-Segment triple the number j of such ops moved
// (the last j movable ones) is chosen to minimise the planned passes of the
// pair.  Random circuit, 2^30 amplitudes per GPU, steady state: 32 qubits
// (N = 4) 10 -> 9 passes per step, 33 qubits (N = 8) 11 -> 9.
// NQ_SHARD_REBALANCE=0 disables it.
bool shard_rebalance_enabled() {
    static const bool on = ab_knob("NQ_SHARD_REBALANCE", 1) != 0;
    return on;
}

bool commutes(const EOp& a, const EOp& b) {
    if ((emask(a, true) & emask(b, true)) == 0) return true;
    return a.type == E_DIAG && b.type == E_DIAG;
}

int64_t planned_passes(const std::vector<EOp>& ops, const PlanOptions& po) {
    if (ops.empty()) return 0;
    PlanStats st;
    plan_passes(ops, po, &st);
    return st.passes;
}

uint64_t acts_key(const std::vector<Action>& acts) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t x) {
        h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h *= 1099511628211ull;
    };
    for (const auto& a : acts) {
        mix(uint64_t(a.kind) | (uint64_t(a.gbit) << 8) | (uint64_t(a.vbit) << 16) | (uint64_t(a.ops.size()) << 24));
        for (const auto& e : a.ops) {
            mix(uint64_t(e.type) | (uint64_t(e.k) << 8));
            for (int j = 0; j < e.k; ++j) mix(uint64_t(e.bits[j]));
            mix(e.ctrl);
        }
    }
    return h;
}

using RebalanceCache = std::unordered_map<uint64_t, std::vector<int>>;

void rebalance(std::vector<Action>& acts, PlanOptions po, int n, RebalanceCache* cache) {
    po.relabel = false;
    const uint64_t key = acts_key(acts);
    RebalanceCache local;
    RebalanceCache& rc = cache ? *cache : local;
    auto hit = rc.find(key);
    const bool cached = hit != rc.end();
    std::vector<int> chosen;
    size_t xi = 0;  // index of the exchange among the rebalanced triples
    for (size_t k = 0; k + 2 < acts.size(); ++k) {
        if (acts[k].kind != Action::Segment || acts[k + 1].kind != Action::Exchange ||
            acts[k + 2].kind != Action::Segment)
            continue;
        const int g = acts[k + 1].gbit, v = acts[k + 1].vbit;
        std::vector<EOp>& seg = acts[k].ops;
        std::vector<EOp>& next = acts[k + 2].ops;
        // movable ops, scanning back from the exchange
        std::vector<char> mov(seg.size(), 0);
        std::vector<const EOp*> stay;
        for (size_t i = seg.size(); i-- > 0;) {
            const EOp& e = seg[i];
            bool ok = !((need_bits(e) >> v) & 1);
            for (size_t t = 0; ok && t < stay.size(); ++t) ok = commutes(e, *stay[t]);
            if (ok) mov[i] = 1;
            else stay.push_back(&e);
        }
        std::vector<size_t> idx;
        for (size_t i = 0; i < seg.size(); ++i)
            if (mov[i]) idx.push_back(i);
        std::vector<int> perm(static_cast<size_t>(n));
        for (int b = 0; b < n; ++b) perm[size_t(b)] = b;
        perm[size_t(g)] = v;
        perm[size_t(v)] = g;
        auto split = [&](size_t j, std::vector<EOp>* st, std::vector<EOp>* mv) {
            std::vector<char> take(seg.size(), 0);
            for (size_t t = idx.size() - j; t < idx.size(); ++t) take[idx[t]] = 1;
            for (size_t i = 0; i < seg.size(); ++i) {
                if (take[i]) mv->push_back(remap(seg[i], perm));
                else st->push_back(seg[i]);
            }
        };
        size_t best_j = 0;
        if (cached) {
            best_j = xi < hit->second.size() ? size_t(hit->second[xi]) : 0;
            if (best_j > idx.size()) best_j = 0;
        } else if (!idx.empty()) {
            auto score = [&](size_t j) {
                std::vector<EOp> st, mv;
                split(j, &st, &mv);
                mv.insert(mv.end(), next.begin(), next.end());
                const int64_t ps = planned_passes(st, po);
                // an exchange with no pass before it runs standalone (a full
                // extra read + write of the shard over NVLink)
                return double(ps + planned_passes(mv, po)) + (ps == 0 ? 1.5 : 0.0);
            };
            const size_t m = idx.size();
            const size_t step = std::max<size_t>(1, m / 16);
            double best = score(0);
            for (size_t j = step; j <= m; j += step) {
                const double sj = score(j);
                if (sj < best) best = sj, best_j = j;
            }
            if (step > 1) {
                const size_t lo = best_j > step ? best_j - step + 1 : 1, hi = std::min(m, best_j + step - 1);
                for (size_t j = lo; j <= hi; ++j) {
                    if (j == best_j) continue;
                    const double sj = score(j);
                    if (sj < best) best = sj, best_j = j;
                }
            }
        }
        chosen.push_back(int(best_j));
        ++xi;
        if (best_j == 0) continue;
        std::vector<EOp> st, mv;
        split(best_j, &st, &mv);
        mv.insert(mv.end(), next.begin(), next.end());
        seg = std::move(st);
        next = std::move(mv);
    }
    if (!cached) {
        if (rc.size() >= 64) rc.clear();
        rc.emplace(key, std::move(chosen));
    }
}

void execute(State& s, const std::vector<Action>& acts, bool relabel = false) {
    DeviceCtx& c = ctx_for(s.dev);
    CUDA_TRY(cudaSetDevice(s.dev));
    std::vector<int> perm(size_t(s.n));
    for (int b = 0; b < s.n; ++b) perm[size_t(b)] = b;
    bool moved = false;
    ShardComm& scx = *s.comm;
    for (size_t ai = 0; ai < acts.size(); ++ai) {
        const Action& a = acts[ai];
        if (a.kind == Action::Segment) {
            if (!relabel) {
                const bool next_x = ai + 1 < acts.size() && acts[ai + 1].kind == Action::Exchange;
                if (next_x && (scx.alt || scx.stage)) {
                    // fuse the exchange into the segment's last pass
                    const Action& x = acts[ai + 1];
                    const int j = x.gbit - s.nloc;
                    const int partner = s.rank ^ (1 << j);
                    FuseX fx;
                    fx.v = x.vbit;
                    fx.mybit = uint64_t((s.rank >> j) & 1);
                    fx.partner = partner;
                    fx.staged = scx.alt == nullptr;
                    fx.out_local = fx.staged ? s.d : scx.alt;
                    fx.out_remote = fx.staged ? scx.stage : scx.peer_alt[size_t(partner)];
                    run_segment(s, c, a.ops, nullptr, &fx);
                    if (fx.done) {
                        fused_exchange_done(s, c, x.gbit, x.vbit, fx.staged);
                        ++ai;
                    }
                    continue;
                }
                run_segment(s, c, a.ops);
                continue;
            }
            std::vector<EOp> ops;
            ops.reserve(a.ops.size());
            for (const auto& e : a.ops) ops.push_back(moved ? remap(e, perm) : e);
            std::vector<int> layout(size_t(s.n));
            for (int b = 0; b < s.n; ++b) layout[size_t(b)] = b;
            run_segment(s, c, ops, &layout);
            bool ident = true;
            for (int b = 0; b < s.n; ++b) ident = ident && layout[size_t(b)] == b;
            if (!ident && shard_relabel_restore()) {
                // the segment's last pass could not store every qubit home:
                // restore here, so every flush runs on the scheduled bits
                std::vector<int> p2l(size_t(s.n));
                for (int b = 0; b < s.n; ++b) p2l[size_t(layout[size_t(b)])] = b;
                std::vector<EOp> swaps;
                for (int pb = 0; pb < s.nloc; ++pb) {
                    if (p2l[size_t(pb)] == pb) continue;
                    const int w = layout[size_t(pb)];
                    EOp e;
                    e.type = E_SWAP;
                    e.k = 2;
                    e.bits[0] = std::min(pb, w);
                    e.bits[1] = std::max(pb, w);
                    swaps.push_back(e);
                    const int lp = p2l[size_t(pb)];
                    p2l[size_t(w)] = lp;
                    layout[size_t(lp)] = w;
                    p2l[size_t(pb)] = pb;
                    layout[size_t(pb)] = pb;
                }
                run_segment(s, c, swaps);
            }
            for (int b = 0; b < s.n; ++b) {
                perm[size_t(b)] = layout[size_t(perm[size_t(b)])];
                moved = moved || perm[size_t(b)] != b;
            }
        } else {
            run_exchange(s, c, a.gbit, perm[size_t(a.vbit)]);
        }
    }
    if (moved) {
        ShardComm& sc = *s.comm;
        for (int q = 0; q < s.n; ++q) sc.l2p[size_t(q)] = perm[size_t(sc.l2p[size_t(q)])];
        for (int q = 0; q < s.n; ++q) sc.p2l[size_t(sc.l2p[size_t(q)])] = q;
    }
}

// rank-ordered sum of one double per rank (deterministic)
std::vector<double> allgather_doubles(State& s, const std::vector<double>& mine) {
    PhaseTimer pt("allgather", s.rank);
    DeviceCtx& c = ctx_for(s.dev);
    const size_t k = mine.size();
    // one persistent buffer: NCCL registers the buffers it sees, and a fresh
    // pool address per call measured 40-1400 ms stalls every few calls
    ShardComm& sc = *s.comm;
    const size_t need = (size_t(s.world) + 1) * k;
    if (need > sc.gather_cap) {
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        if (sc.gather) CUDA_TRY(cudaFree(sc.gather));
        sc.gather = nullptr;
        const size_t cap = std::max<size_t>(need, 1 << 16);
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&sc.gather), cap * sizeof(double)));
        sc.gather_cap = cap;
    }
    double* d = sc.gather;
    std::vector<double> all(size_t(s.world) * k);
    if (sc.hg) {
        // (a pageable H2D cudaMemcpy may return before the data lands: copy
        // on the stream and wait for it before the peers may read)
        CUDA_TRY(cudaMemcpyAsync(sc.hg->coll, mine.data(), k * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        sc.hg->barrier();
        for (int r = 0; r < s.world; ++r)
            CUDA_TRY(cudaMemcpy(all.data() + size_t(r) * k, sc.hg->buf(r), k * sizeof(double), cudaMemcpyDeviceToHost));
        sc.hg->barrier();
        return all;
    }
    CUDA_TRY(cudaMemcpyAsync(d, mine.data(), k * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    NCCL_TRY(ncclAllGather(d, d + k, k, ncclDouble, sc.comm, c.stream));
    CUDA_TRY(cudaMemcpyAsync(all.data(), d + k, all.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    return all;
}

// Map every rank's buffer `mine` into this process (CUDA IPC); all ranks must
// agree, so the outcome is all-gathered and any failure (or `want` false on
// any rank) returns an empty vector everywhere.
std::vector<double2*> map_peers(State& s, double2* mine_ptr, bool want) {
    cudaIpcMemHandle_t mine{};
    cudaError_t gerr = cudaSuccess;
    bool ok = want && mine_ptr && (gerr = cudaIpcGetMemHandle(&mine, mine_ptr)) == cudaSuccess;
    cudaGetLastError();
    if (std::getenv("NQ_SHARD_TRACE") && want && mine_ptr && gerr != cudaSuccess)
        std::fprintf(stderr, "[shard] rank %d: cudaIpcGetMemHandle: %s\n", s.rank, cudaGetErrorString(gerr));
    // all-gather the 64-byte handles as doubles (8 per handle) + an ok flag
    constexpr size_t kW = sizeof(cudaIpcMemHandle_t) / sizeof(double) + 1;
    std::vector<double> buf(kW, 0.0);
    std::memcpy(buf.data(), &mine, sizeof(mine));
    buf[kW - 1] = ok ? 1.0 : 0.0;
    const std::vector<double> all = allgather_doubles(s, buf);
    for (int r = 0; r < s.world; ++r) ok = ok && all[size_t(r) * kW + kW - 1] == 1.0;
    std::vector<double2*> peer(size_t(s.world), nullptr);
    for (int r = 0; ok && r < s.world; ++r) {
        if (r == s.rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, all.data() + size_t(r) * kW, sizeof(h));
        void* p = nullptr;
        const cudaError_t oerr = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (oerr != cudaSuccess) {
            cudaGetLastError();
            if (std::getenv("NQ_SHARD_TRACE"))
                std::fprintf(stderr, "[shard] rank %d: cudaIpcOpenMemHandle(rank %d): %s\n", s.rank, r,
                             cudaGetErrorString(oerr));
            ok = false;
            break;
        }
        peer[size_t(r)] = static_cast<double2*>(p);
    }
    // agree: p2p only if every rank mapped every peer
    const std::vector<double> oks = allgather_doubles(s, {ok ? 1.0 : 0.0});
    for (double v : oks) ok = ok && v == 1.0;
    if (!ok) {
        for (double2* p : peer)
            if (p) cudaIpcCloseMemHandle(p);
        peer.clear();
    }
    return peer;
}

// Every rank plans its own flushes, so the options that shape plans and
// exchanges (knobs.hpp) must be identical on all ranks, or their collectives
// diverge: compare a hash of them at creation.
void check_env_agreement(State& s) {
    const std::string fp = plan_env_fingerprint();
    uint64_t h = 1469598103934665603ull;  // FNV-1a
    for (unsigned char ch : fp) h = (h ^ ch) * 1099511628211ull;
    const auto all = allgather_doubles(s, {double(h >> 32), double(h & 0xffffffffu)});
    for (int r = 0; r < s.world; ++r)
        if (all[size_t(2 * r)] != all[0] || all[size_t(2 * r + 1)] != all[1])
            throw NqError{NQ_ERR_CONTRACT, "sharded state: rank " + std::to_string(r) + " and rank 0 run with "
                                               "different NQ_* options (this rank: '" + fp + "'); every rank "
                                               "must see the same environment"};
}

void free_staging(ShardComm& sc) {
    for (unsigned* p : sc.peer_sync)
        if (p) cudaIpcCloseMemHandle(p);
    sc.peer_sync.clear();
    if (sc.stage) cudaFree(sc.stage);
    if (sc.sync) cudaFree(sc.sync);
    sc.stage = nullptr;
    sc.sync = nullptr;
    sc.stage_chunks = 0;
}

bool fused_exchange_wanted() {
    return env_option_str("NQ_FUSED_EXCHANGE") != "0";
}

void setup_peer_exchange(State& s, ShardComm& sc, DeviceCtx& c) {
    const bool want = env_option_str("NQ_EXCHANGE") != "nccl";
    sc.peer = map_peers(s, s.d, want);
    if (sc.peer.empty()) return;
    // a second copy of the shard for fused exchanges, when it fits with room
    // to spare (2^30 amplitudes per GPU: 2 x 16 GiB; 2^33 does not fit)
    bool fx = fused_exchange_wanted();
    if (fx) {
        size_t free_b = 0, total_b = 0;
        fx = cudaMemGetInfo(&free_b, &total_b) == cudaSuccess &&
             free_b > size_t(s.count) * sizeof(double2) + (size_t(4) << 30);
        cudaGetLastError();
    }
    if (fx && cudaMalloc(reinterpret_cast<void**>(&sc.alt), size_t(s.count) * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        sc.alt = nullptr;
    }
    sc.peer_alt = map_peers(s, sc.alt, sc.alt != nullptr);
    if (sc.peer_alt.empty() && sc.alt) {
        cudaFree(sc.alt);
        sc.alt = nullptr;
    }
    // staged fused exchanges when no second copy fits (or when forced by
    // NQ_FUSED_EXCHANGE=staged): 64 chunks (fewer for small shards: a chunk
    // spans at least 2 tiles of the largest pass tile, 2^12), 4 slots of
    // half a chunk each -- 4 GiB at 2^33 amplitudes per GPU
    const std::string fxm = env_option_str("NQ_FUSED_EXCHANGE");
    const bool want_staged = fused_exchange_wanted() && (fxm == "staged" || !sc.alt) && !sc.hg;
    if (want_staged) {
        if (sc.alt) {  // forced: release the second copy
            for (double2* p : sc.peer_alt)
                if (p) cudaIpcCloseMemHandle(p);
            sc.peer_alt.clear();
            cudaFree(sc.alt);
            sc.alt = nullptr;
        }
        sc.stage_slots = ab_knob("NQ_STAGE_SLOTS", 4);
        int chunks = ab_knob("NQ_STAGE_CHUNKS", 64);
        while (chunks > 2 && (uint64_t(chunks) << 13) > s.count) chunks /= 2;
        sc.stage_chunks = chunks;
        sc.stage_slot_elems = s.count / 2 / uint64_t(chunks);
        bool ok = (uint64_t(chunks) << 13) <= s.count &&
                  cudaMalloc(reinterpret_cast<void**>(&sc.stage),
                             size_t(sc.stage_slots) * sc.stage_slot_elems * sizeof(double2)) == cudaSuccess &&
                  // 2 MiB: a small cudaMalloc may share an IPC-able block with
                  // others, and a peer's mapping of the handle then starts at
                  // that block's base, not at this buffer
                  cudaMalloc(reinterpret_cast<void**>(&sc.sync), size_t(2) << 20) == cudaSuccess &&
                  cudaMemset(sc.sync, 0, sizeof(unsigned) * (2 * ShardComm::kMaxChunks + 16)) == cudaSuccess;
        cudaGetLastError();
        std::vector<double2*> ps = map_peers(s, reinterpret_cast<double2*>(sc.sync), ok);
        ok = !ps.empty();
        if (ok) {
            for (double2* p : ps) sc.peer_sync.push_back(reinterpret_cast<unsigned*>(p));
        } else {
            free_staging(sc);
        }
    }
    (void)c;
}

void normalize_map(State& s) {
    ShardComm& sc = *s.comm;
    bool identity = true;
    for (int p = 0; p < s.n; ++p) identity = identity && sc.p2l[size_t(p)] == p;
    if (identity) return;
    execute(s, schedule_identity(sc.l2p, sc.p2l, s.nloc, s.n));
}

}  // namespace

void shard_normalize(State& s) {
    if (s.comm) normalize_map(s);
}

void shard_free(State& s) {
    if (!s.comm) return;
    ShardComm* sc = s.comm;
    DeviceCtx& c = ctx_for(s.dev);
    cudaStreamSynchronize(c.stream);
    if (sc->sendbuf) cudaFree(sc->sendbuf);
    if (sc->recvbuf) cudaFree(sc->recvbuf);
    if (sc->d_flag) cudaFree(sc->d_flag);
    if (sc->gather) cudaFree(sc->gather);
    if (sc->bcast) cudaFree(sc->bcast);
    for (double2* p : sc->peer)
        if (p) cudaIpcCloseMemHandle(p);
    for (double2* p : sc->peer_alt)
        if (p) cudaIpcCloseMemHandle(p);
    if (sc->alt) cudaFree(sc->alt);
    free_staging(*sc);
    if (sc->comm) ncclCommDestroy(sc->comm);
    host_group_free(sc->hg);
    delete sc;
    s.comm = nullptr;
}

void shard_reset(State& s) {
    if (!s.comm) return;
    for (int q = 0; q < s.n; ++q) s.comm->l2p[size_t(q)] = s.comm->p2l[size_t(q)] = q;
}

void shard_flush(State& s) {
    PhaseTimer pt("flush", s.rank);
    NvtxRange range("nq.shard_flush", s.rank);
    ShardComm& sc = *s.comm;
    std::vector<EOp> ops;
    ops.swap(s.queue);
    s.last_passes = s.last_microops = s.last_source_ops = s.last_launches = 0;
    bool repeat = ops.size() == sc.prev_ops.size();
    for (size_t i = 0; i < ops.size() && repeat; ++i) {
        const EOp &a = ops[i], &b = sc.prev_ops[i];
        repeat = a.type == b.type && a.k == b.k && a.ctrl == b.ctrl &&
                 std::equal(a.bits, a.bits + a.k, b.bits);
    }
    std::vector<Action> acts = schedule(ops, sc.l2p, sc.p2l, s.nloc, repeat && shard_cyclic_enabled());
    sc.prev_ops = ops;
    // The qubit map is carried into the next flush (readouts normalise it
    // first).  Re-running one circuit then converges to a map whose global
    // qubits that circuit never needs as targets: after a step or two the
    // flush needs few or no exchanges and runs the same physical program
    // every time (its specialised kernels are reused).  NQ_SHARD_RESTORE=1
    // restores the identity map at the end of every flush instead.
    static const bool restore = ab_knob("NQ_SHARD_RESTORE", 0) == 1;
    if (restore) {
        std::vector<Action> back = schedule_identity(sc.l2p, sc.p2l, s.nloc, s.n);
        acts.insert(acts.end(), back.begin(), back.end());
    }
    // Tail exchange: a flush that repeats the previous one is predicted to be
    // followed by itself.  If that next flush would open with an exchange (its
    // first op needs a qubit this flush leaves global), the exchange runs now
    // as this flush's last action, where it fuses into the final pass, instead
    // of as a standalone swap at the start of the next flush (nothing precedes
    // it there to fuse with).  The map is valid either way; only the moment
    // of the swap moves.
    if (repeat && !restore && !acts.empty() && acts.back().kind == Action::Segment && (sc.alt || sc.stage)) {
        std::vector<int> l2 = sc.l2p, p2 = sc.p2l;
        const std::vector<Action> nxt = schedule(ops, l2, p2, s.nloc, false);
        if (!nxt.empty() && nxt.front().kind == Action::Exchange) {
            acts.push_back(nxt.front());
            swap_map(sc.l2p, sc.p2l, nxt.front().gbit, nxt.front().vbit);
        }
    }
    // Relabelling passes inside the segments: off unless NQ_SHARD_RELABEL=1.
    // Measured at N = 4 (random circuit, 2^30 per GPU): 9 instead of 10 passes
    // per step, but the composed qubit map keeps drifting for several flushes,
    // so repeated circuits keep meeting uncompiled pass structures.
    static const bool relabel = ab_knob("NQ_SHARD_RELABEL", 0) == 1;
    if (shard_rebalance_enabled() && !(relabel && !restore)) {
        PhaseTimer pr("rebalance", s.rank);
        rebalance(acts, s.popt, s.n, &sc.rebalance_cache);
    }
    execute(s, acts, relabel && !restore);
    check_async(sc.comm);
}

double shard_norm_sq(State& s) {
    DeviceCtx& c = ctx_for(s.dev);
    c.ensure_scratch(scratch_doubles_needed(s.count) + 64);
    launch_sumsq(s.d, s.count, c.d_scratch + 64, result_slot(c, 0), c.stream);
    CUDA_TRY(cudaGetLastError());
    double mine = 0.0;
    fetch(c, result_slot(c, 0), 1, &mine);
    const auto all = allgather_doubles(s, {mine});
    double total = 0.0;
    for (double v : all) total += v;
    return total;
}

void shard_expectation(State& s, const uint64_t* flip, const uint64_t* signs, const int32_t* ny, const double* coeff,
                       int nterms, double* out) {
    PhaseTimer pt("expectation", s.rank);
    ShardComm& sc = *s.comm;
    const uint64_t loc_mask = (uint64_t(1) << s.nloc) - 1;
    for (int t = 0; t < nterms; ++t)
        if (__builtin_popcountll(flip[t]) > s.nloc)
            throw NqError{NQ_ERR_CONTRACT, "sharded expectation: a Pauli term flips more qubits (" +
                                               std::to_string(__builtin_popcountll(flip[t])) +
                                               ") than one rank holds (" + std::to_string(s.nloc) + ")"};
    // Terms are evaluated in batches whose flipped qubits are all local under
    // the current qubit map; before a term that flips a global qubit, that
    // qubit is swapped in (Belady victim over the remaining terms' flips).
    const size_t nt = static_cast<size_t>(nterms);
    std::vector<double> mine(2 * nt, 0.0);
    std::vector<int> batch;
    auto run_batch = [&] {
        if (batch.empty()) return;
        std::vector<uint64_t> pf, ps;
        std::vector<double> sgn;
        for (int t : batch) {
            uint64_t f = 0, g = 0;
            for (int q = 0; q < s.n; ++q) {
                if ((flip[t] >> q) & 1) f |= uint64_t(1) << sc.l2p[size_t(q)];
                if ((signs[t] >> q) & 1) g |= uint64_t(1) << sc.l2p[size_t(q)];
            }
            if (f & ~loc_mask) throw NqError{NQ_ERR_INTERNAL, "sharded expectation: flip bit still global"};
            pf.push_back(f);
            ps.push_back(g & loc_mask);
            sgn.push_back((__builtin_popcountll((g >> s.nloc) & uint64_t(s.rank)) & 1) ? -1.0 : 1.0);
        }
        std::vector<cplx> totals;
        PhaseTimer pe("expect_raw", s.rank);
        sv_expect_raw(s, pf.data(), ps.data(), int(batch.size()), totals);
        for (size_t i = 0; i < batch.size(); ++i) {
            mine[2 * size_t(batch[i])] = sgn[i] * totals[i].real();
            mine[2 * size_t(batch[i]) + 1] = sgn[i] * totals[i].imag();
        }
        batch.clear();
    };
    auto stand_in = [](int q) {
        EOp e;
        e.type = E_XPERM;  // an op that needs qubit q local
        e.k = 1;
        e.bits[0] = q;
        return e;
    };
    for (int t = 0; t < nterms; ++t) {
        uint64_t glob = 0;
        for (int q = 0; q < s.n; ++q)
            if (((flip[t] >> q) & 1) && sc.l2p[size_t(q)] >= s.nloc) glob |= uint64_t(1) << q;
        if (glob) {
            run_batch();
            // future uses: the flips of this and the remaining terms
            std::vector<EOp> fut;
            for (int u = t; u < nterms; ++u)
                for (int q = 0; q < s.n; ++q)
                    if ((flip[u] >> q) & 1) fut.push_back(stand_in(q));
            std::vector<Action> ex;
            for (int q = 0; q < s.n; ++q) {
                if (!((glob >> q) & 1)) continue;
                const int gb = sc.l2p[size_t(q)];
                const int v = choose_victim(fut, 0, sc.p2l, s.nloc, flip[t]);
                ex.push_back(Action{Action::Exchange, {}, gb, v});
                swap_map(sc.l2p, sc.p2l, gb, v);
            }
            execute(s, ex);
        }
        batch.push_back(t);
    }
    run_batch();
    const auto all = allgather_doubles(s, mine);
    static const cplx kI4[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    for (int t = 0; t < nterms; ++t) {
        cplx tot(0.0, 0.0);
        for (int r = 0; r < s.world; ++r)
            tot += cplx(all[size_t(r) * mine.size() + size_t(2 * t)], all[size_t(r) * mine.size() + size_t(2 * t + 1)]);
        out[t] = coeff[t] * (tot * kI4[ny[t] & 3]).real();
    }
}

void shard_sample(State& s, const double* sorted_u, uint64_t shots, uint64_t* idx_out, uint64_t* count_out,
                  uint64_t* nout) {
    normalize_map(s);
    DeviceCtx& c = ctx_for(s.dev);
    // approximate rank masses (binade guesses only), then the exact sequential
    // cumulative handed from rank to rank: rank r walks its shard from the
    // exact end of rank r - 1 (sample.cpp), so the ranks' ranges [start, end)
    // tile [0, final) with no gap and every uniform has exactly one owner
    c.ensure_scratch(scratch_doubles_needed(s.count) + 64);
    launch_sumsq(s.d, s.count, c.d_scratch + 64, result_slot(c, 0), c.stream);
    double mass = 0.0;
    fetch(c, result_slot(c, 0), 1, &mass);
    const auto masses = allgather_doubles(s, {mass});
    double approx = 0.0;
    for (int r = 0; r < s.rank; ++r) approx += masses[size_t(r)];
    SeqCum sc;
    seqcum_prepare(c, s.d, nullptr, s.count, approx, sc);
    double start = 0.0, end = 0.0;
    for (int r = 0; r < s.world; ++r) {
        double mine = 0.0;
        if (r == s.rank) mine = end = seqcum_walk(c, s.d, nullptr, sc, start);
        const auto ends = allgather_doubles(s, {mine});
        if (r < s.rank) start = ends[size_t(r)];
    }
    int last_nz = -1;
    for (int r = 0; r < s.world; ++r)
        if (masses[size_t(r)] > 0.0) last_nz = r;
    // uniforms owned by this rank: [start, end); the last nonzero rank also takes leftovers
    uint64_t lo = uint64_t(std::lower_bound(sorted_u, sorted_u + shots, start) - sorted_u);
    uint64_t hi = (s.rank == last_nz) ? shots : uint64_t(std::lower_bound(sorted_u, sorted_u + shots, end) - sorted_u);
    if (s.rank > last_nz) lo = hi = 0;
    std::vector<uint64_t> li(std::max<uint64_t>(hi - lo, 1)), lc(std::max<uint64_t>(hi - lo, 1));
    uint64_t k = 0;
    if (hi > lo)
        sample_assign(c, s.d, nullptr, sc, start, sorted_u + lo, hi - lo, li.data(), lc.data(), &k,
                      s.rank == last_nz);
    // gather (index, count) pairs in rank order
    const auto ks = allgather_doubles(s, {double(k)});
    uint64_t maxk = 1;
    for (double v : ks) maxk = std::max<uint64_t>(maxk, uint64_t(v));
    std::vector<double> pack(size_t(2 * maxk), 0.0);
    for (uint64_t i = 0; i < k; ++i) {
        pack[size_t(2 * i)] = double((uint64_t(s.rank) << s.nloc) | li[size_t(i)]);
        pack[size_t(2 * i + 1)] = double(lc[size_t(i)]);
    }
    const auto all = allgather_doubles(s, pack);
    uint64_t o = 0;
    for (int r = 0; r < s.world; ++r)
        for (uint64_t i = 0; i < uint64_t(ks[size_t(r)]); ++i) {
            idx_out[o] = uint64_t(all[size_t(r) * pack.size() + size_t(2 * i)]);
            count_out[o] = uint64_t(all[size_t(r) * pack.size() + size_t(2 * i + 1)]);
            ++o;
        }
    uint64_t total = 0;
    for (uint64_t i = 0; i < o; ++i) total += count_out[i];
    if (total != shots)
        throw NqError{NQ_ERR_INTERNAL, "sharded sampling assigned " + std::to_string(total) + " of " +
                                           std::to_string(shots) + " shots"};
    *nout = o;
}

// probabilities() of a sharded state: every rank receives the full 2^n
// vector (the reference API's contract), rank by rank in 512 MiB chunks
// broadcast from the owning rank through one persistent device buffer.
void shard_probabilities(State& s, double* host_out) {
    normalize_map(s);
    ShardComm& sc = *s.comm;
    DeviceCtx& c = ctx_for(s.dev);
    const uint64_t chunk = std::min<uint64_t>(s.count, uint64_t(1) << 26);
    if (sc.bcast_cap < chunk) {
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        if (sc.bcast) CUDA_TRY(cudaFree(sc.bcast));
        sc.bcast = nullptr;
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&sc.bcast), chunk * sizeof(double)));
        sc.bcast_cap = chunk;
    }
    if (sc.hg) {
        const uint64_t hc = std::min<uint64_t>(chunk, sc.hg->coll_cap);
        for (int r = 0; r < s.world; ++r)
            for (uint64_t off = 0; off < s.count; off += hc) {
                const uint64_t len = std::min(hc, s.count - off);
                if (r == s.rank) launch_probs(s.d + off, len, sc.hg->coll, c.stream);
                CUDA_TRY(cudaStreamSynchronize(c.stream));
                sc.hg->barrier();
                CUDA_TRY(cudaMemcpy(host_out + (uint64_t(r) << s.nloc) + off, sc.hg->buf(r), len * sizeof(double),
                                    cudaMemcpyDeviceToHost));
                sc.hg->barrier();
            }
        return;
    }
    for (int r = 0; r < s.world; ++r) {
        for (uint64_t off = 0; off < s.count; off += chunk) {
            const uint64_t len = std::min(chunk, s.count - off);
            if (r == s.rank) launch_probs(s.d + off, len, sc.bcast, c.stream);
            NCCL_TRY(ncclBroadcast(sc.bcast, sc.bcast, size_t(len), ncclDouble, r, sc.comm, c.stream));
            CUDA_TRY(cudaMemcpyAsync(host_out + (uint64_t(r) << s.nloc) + off, sc.bcast, len * sizeof(double),
                                     cudaMemcpyDeviceToHost, c.stream));
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c.stream));
}

// set_amplitudes on a sharded state: every rank passes the same host range
// and copies the part it owns (logical order).
void shard_set_amplitudes(State& s, uint64_t offset, uint64_t count, const double* host_in) {
    if (offset > (uint64_t(1) << s.n) || count > (uint64_t(1) << s.n) - offset)
        throw NqError{NQ_ERR_CONTRACT, "amplitude range out of bounds"};
    normalize_map(s);
    DeviceCtx& c = ctx_for(s.dev);
    const uint64_t lo = uint64_t(s.rank) << s.nloc, hi = lo + s.count;
    const uint64_t a = std::max(offset, lo), b = std::min(offset + count, hi);
    if (a < b)
        CUDA_TRY(cudaMemcpyAsync(s.d + (a - lo), host_in + 2 * (a - offset), (b - a) * sizeof(double2),
                                 cudaMemcpyHostToDevice, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
}

void shard_get_amplitudes(State& s, uint64_t offset, uint64_t count, double* host_out) {
    if (offset > (uint64_t(1) << s.n) || count > (uint64_t(1) << s.n) - offset)
        throw NqError{NQ_ERR_CONTRACT, "amplitude range out of bounds"};
    normalize_map(s);
    DeviceCtx& c = ctx_for(s.dev);
    double2* d = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), std::max<uint64_t>(count, 1) * sizeof(double2), c.stream));
    CUDA_TRY(cudaMemsetAsync(d, 0, std::max<uint64_t>(count, 1) * sizeof(double2), c.stream));
    const uint64_t mine_lo = uint64_t(s.rank) << s.nloc, mine_hi = mine_lo + s.count;
    const uint64_t a = std::max(offset, mine_lo), b = std::min(offset + count, mine_hi);
    if (a < b)
        CUDA_TRY(cudaMemcpyAsync(d + (a - offset), s.d + (a - mine_lo), (b - a) * sizeof(double2),
                                 cudaMemcpyDeviceToDevice, c.stream));
    // exactly one rank contributes each element: the sum with zeros is exact
    if (count && s.comm->hg) {
        HostGroup& hg = *s.comm->hg;
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        const uint64_t total = count * 2, hc = hg.coll_cap;
        std::vector<double> part(std::min<uint64_t>(total, hc)), acc(part.size());
        double* dd = reinterpret_cast<double*>(d);
        for (uint64_t off = 0; off < total; off += hc) {
            const uint64_t len = std::min(hc, total - off);
            CUDA_TRY(cudaMemcpyAsync(hg.coll, dd + off, len * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
            CUDA_TRY(cudaStreamSynchronize(c.stream));
            hg.barrier();
            std::fill(acc.begin(), acc.begin() + long(len), 0.0);
            for (int r = 0; r < s.world; ++r) {
                CUDA_TRY(cudaMemcpy(part.data(), hg.buf(r), len * sizeof(double), cudaMemcpyDeviceToHost));
                for (uint64_t i = 0; i < len; ++i) acc[i] += part[i];
            }
            hg.barrier();
            CUDA_TRY(cudaMemcpyAsync(dd + off, acc.data(), len * sizeof(double), cudaMemcpyHostToDevice, c.stream));
            CUDA_TRY(cudaStreamSynchronize(c.stream));
        }
    } else if (count) {
        NCCL_TRY(ncclAllReduce(d, d, size_t(count) * 2, ncclDouble, ncclSum, s.comm->comm, c.stream));
    }
    if (count)
        CUDA_TRY(cudaMemcpyAsync(host_out, d, count * sizeof(double2), cudaMemcpyDeviceToHost, c.stream));
    CUDA_TRY(cudaFreeAsync(d, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
}

}  // namespace nqe

using namespace nqe;

extern "C" {

nq_status nq_comm_unique_id(unsigned char out[128]) {
    return guard([&] {
        if (host_comm_requested()) {
            // host-coordinated ranks: the id only names the shared-memory block
            std::random_device rd;
            for (int i = 0; i < 128; i += 4) {
                const unsigned v = rd();
                std::memcpy(out + i, &v, 4);
            }
            return;
        }
        ncclUniqueId id;
        NCCL_TRY(ncclGetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(out, &id, 128);
    });
}

nq_status nq_sv_create_sharded(int n, int rank, int world, const unsigned char uid[128], const nq_opts* opts,
                               nq_sv** out) {
    return guard([&] {
        if (world < 1 || (world & (world - 1)))
            throw NqError{NQ_ERR_CONTRACT, "world size must be a power of two"};
        if (rank < 0 || rank >= world) throw NqError{NQ_ERR_CONTRACT, "rank out of range"};
        int g = 0;
        while ((1 << g) < world) ++g;
        nq_opts o;
        nq_default_opts(&o);
        if (opts) o = *opts;
        const int cap = o.max_qubits > 0 ? o.max_qubits : 40;
        if (n - g < 1 || n > cap)
            throw NqError{NQ_ERR_CONTRACT, "sharded state qubit count must be in [" + std::to_string(g + 1) + ", " +
                                               std::to_string(cap) + "], got " + std::to_string(n)};
        if (n - g < 8) throw NqError{NQ_ERR_CONTRACT, "sharded states need at least 8 local qubits per rank"};
        auto h = std::make_unique<nq_sv>();
        State& s = h->s;
        nq_opts lo = o;
        lo.max_qubits = n;  // the local allocation is n - g qubits; state_init checks n
        state_init(s, n - g, false, &lo);
        {
            // IPC needs a plain (non-pool) allocation
            DeviceCtx& c0 = ctx_for(s.dev);
            CUDA_TRY(cudaFreeAsync(s.d, c0.stream));
            CUDA_TRY(cudaStreamSynchronize(c0.stream));
            s.d = nullptr;
            CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&s.d), (size_t(1) << (n - g)) * sizeof(double2)));
            s.plain_alloc = true;
        }
        s.n = n;
        s.nbits = n;
        s.nloc = n - g;
        s.count = uint64_t(1) << s.nloc;
        s.rank = rank;
        s.world = world;
        s.popt.nbits = n;
        s.popt.nloc = s.nloc;
        s.popt.relabel = false;  // the sharded layer keeps its own qubit map
        s.layout.clear();
        configure_caps(s.popt);
        DeviceCtx& c = ctx_for(s.dev);
        launch_init_basis(s.d, s.count, rank == 0 ? 0 : UINT64_MAX, c.stream);
        auto sc = std::make_unique<ShardComm>();
        sc->l2p.resize(size_t(n));
        sc->p2l.resize(size_t(n));
        for (int q = 0; q < n; ++q) sc->l2p[size_t(q)] = sc->p2l[size_t(q)] = q;
        sc->chunk = std::min<uint64_t>(s.count / 2, uint64_t(1) << 26);
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&sc->sendbuf), sc->chunk * sizeof(double2)));
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&sc->recvbuf), sc->chunk * sizeof(double2)));
        if (host_comm_requested()) {
            sc->hg = host_group_create(uid, rank, world);
        } else {
            ncclUniqueId id;
            std::memcpy(&id, uid, 128);
            NCCL_TRY(ncclCommInitRank(&sc->comm, world, id, rank));
        }
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&sc->d_flag), sizeof(double)));
        CUDA_TRY(cudaMemset(sc->d_flag, 0, sizeof(double)));
        s.comm = sc.release();
        check_env_agreement(s);
        setup_peer_exchange(s, *s.comm, c);
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        *out = h.release();
    });
}

nq_status nq_sv_comm_stats(const nq_sv* h, int64_t* exchanges, int64_t* bytes_sent) {
    return guard([&] {
        const State& s = h->s;
        if (exchanges) *exchanges = s.comm ? s.comm->exchanges : 0;
        if (bytes_sent) *bytes_sent = s.comm ? s.comm->bytes : 0;
    });
}

nq_status nq_sv_comm_fused(const nq_sv* h, int64_t* fused, int* has_alt_buffer) {
    return guard([&] {
        const State& s = h->s;
        if (fused) *fused = s.comm ? s.comm->fused : 0;
        if (has_alt_buffer) *has_alt_buffer = !s.comm ? 0 : s.comm->alt ? 1 : s.comm->stage ? 2 : 0;
    });
}

// Host scheduling only (no device): the actions a sharded flush of `ops`
// would take from the identity map, serialised as int64 records:
// [kind(0 seg,1 exch), a, b, nops_or_0] followed by nops * nq_op for segments
// (ops in physical bits, as kinds/targets of the lowered elementary ops).
nq_status nq_shard_debug(int n, int world, const nq_op* ops, int64_t count, int flags, int64_t* buf, int64_t cap,
                         int64_t* size) {
    return guard([&] {
        int g = 0;
        while ((1 << g) < world) ++g;
        if ((1 << g) != world || n - g < 1) throw NqError{NQ_ERR_CONTRACT, "bad world size"};
        std::vector<EOp> q;
        for (int64_t i = 0; i < count; ++i) lower_sv_op(ops[i], q);
        const size_t nn = static_cast<size_t>(n);
        std::vector<int> l2p(nn), p2l(nn);
        for (int i = 0; i < n; ++i) l2p[size_t(i)] = p2l[size_t(i)] = i;
        auto acts = schedule(q, l2p, p2l, n - g, false);
        if (flags & 1) {
            PlanOptions po;
            po.nbits = n;
            po.nloc = n - g;
            configure_caps(po);
            rebalance(acts, po, n, nullptr);
        }
        auto fin = schedule_identity(l2p, p2l, n - g, n);
        acts.insert(acts.end(), fin.begin(), fin.end());
        std::vector<int64_t> out;
        for (const auto& a : acts) {
            auto put = [&](std::initializer_list<int64_t> vals) { out.insert(out.end(), vals); };
            if (a.kind == Action::Exchange) {
                put({1, int64_t(a.gbit), int64_t(a.vbit), 0});
                continue;
            }
            put({0, 0, 0, int64_t(a.ops.size())});
            for (const auto& e : a.ops) {
                // elementary op: type, k, bits[4], ctrl, matrix size, matrix (re,im as bit patterns)
                put({int64_t(e.type), int64_t(e.k), int64_t(e.bits[0]), int64_t(e.bits[1]), int64_t(e.bits[2]),
                     int64_t(e.bits[3]), int64_t(e.ctrl), int64_t(e.mat.size())});
                for (const auto& v : e.mat) {
                    int64_t re, im;
                    const double vr = v.real(), vi = v.imag();
                    std::memcpy(&re, &vr, 8);
                    std::memcpy(&im, &vi, 8);
                    out.push_back(re);
                    out.push_back(im);
                }
            }
        }
        *size = int64_t(out.size());
        if (buf && cap > 0) std::memcpy(buf, out.data(), size_t(std::min<int64_t>(cap, *size)) * 8);
    });
}

}  // extern "C"

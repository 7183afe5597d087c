// C ABI of the B200 simulation core (include/naqs_b200.h).
//
// Each function validates its preconditions with the reference's wording
// (proj/src/statevector.cpp, proj/src/densitymatrix.cpp, proj/src/noise.cpp),
// queues work, and runs it on the device's stream.  There is no host
// execution path: every amplitude update, reduction and readout map runs in
// kernels.cu.
#include "../../include/naqs_b200.h"

#include "engine.hpp"
#include "jit.hpp"
#include "kernels.hpp"
#include "knobs.hpp"
#include "nvtx.hpp"
#include "lower.hpp"
#include "state.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <tuple>
#include <vector>

using namespace nqe;

namespace nqe {

thread_local std::string g_last_error;

DeviceCtx& ctx_for(int dev) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<DeviceCtx>> ctxs;
    std::lock_guard<std::mutex> lk(mu);
    auto it = ctxs.find(dev);
    if (it != ctxs.end()) return *it->second;
    auto c = std::make_unique<DeviceCtx>();
    c->dev = dev;
    CUDA_TRY(cudaSetDevice(dev));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&c->h_small), 64 * 1024));
    DeviceCtx& ref = *c;
    ctxs[dev] = std::move(c);
    return ref;
}

void DeviceCtx::ensure_scratch(size_t doubles) {
    if (doubles <= scratch_cap) return;
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (d_scratch) CUDA_TRY(cudaFree(d_scratch));
    d_scratch = nullptr;
    const size_t cap = std::max<size_t>(doubles, 1 << 16);
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&d_scratch), cap * sizeof(double)));
    scratch_cap = cap;
}

void DeviceCtx::stage(const unsigned char* src, size_t bytes) {
    if (stage_pending) {
        CUDA_TRY(cudaEventSynchronize(stage_ev));
        stage_pending = false;
    }
    if (bytes > h_stage_cap) {
        if (h_stage) CUDA_TRY(cudaFreeHost(h_stage));
        h_stage = nullptr;
        const size_t cap = std::max<size_t>(bytes * 2, 1 << 20);
        CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&h_stage), cap));
        h_stage_cap = cap;
    }
    if (bytes > d_ops_cap) {
        CUDA_TRY(cudaStreamSynchronize(stream));
        if (d_ops) CUDA_TRY(cudaFree(d_ops));
        d_ops = nullptr;
        const size_t cap = std::max<size_t>(bytes * 2, 1 << 20);
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&d_ops), cap));
        d_ops_cap = cap;
    }
    std::memcpy(h_stage, src, bytes);
    h2d_bytes += int64_t(bytes);
    CUDA_TRY(cudaMemcpyAsync(d_ops, h_stage, bytes, cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaEventRecord(stage_ev, stream));
    stage_pending = true;
}

// ---- state lifecycle ---------------------------------------------------------
// Layout of a freshly initialised state (|0..0> looks the same in every
// layout).  State vectors: identity.  Density matrices larger than one tile:
// interleaved, column bit q -> physical 2q and row bit q -> physical 2q + 1,
// so a tile's low contiguous bits are whole qubits (both bits of a qubit's
// superoperators) instead of column bits alone.  Opt-in (NQ_DM_INTERLEAVE=1):
// on noisy TFIM-14 it does not reduce the pass count (a chain sweeps the
// qubits either way) and the readouts then need a normalising swap plan.
// Hermitian (mirror) passes for density matrices, in the interleaved layout
// (NQ_DM_MIRROR=0 disables).  Noisy TFIM-14: 134.8 -> 82.0 ms.
bool dm_mirror_enabled() {
    static const bool on = ab_knob("NQ_DM_MIRROR", 1) != 0;
    return on;
}

// NQ_DM_RELABEL=1: relabelling passes for density matrices (whole qubits in
// the low pairs).  Off by default: noisy TFIM-14 planned 52 instead of 55
// passes but ran slower (88.5 vs 81.9 ms).
bool dm_relabel_enabled() {
    static const bool on = ab_knob("NQ_DM_RELABEL", 0) == 1;
    return on;
}

void set_initial_layout(State& s) {
    for (int b = 0; b < s.nbits; ++b) s.layout[size_t(b)] = b;
    static const bool interleave = ab_knob("NQ_DM_INTERLEAVE", 0) == 1;
    s.popt.dm_mirror_n = 0;
    if (s.dm) s.popt.relabel = s.popt.relabel && dm_mirror_enabled() && dm_relabel_enabled();
    if (!s.dm || !(interleave || dm_mirror_enabled()) || s.nloc <= s.popt.tile_bits) return;
    for (int q = 0; q < s.n; ++q) {
        s.layout[size_t(q)] = 2 * q;
        s.layout[size_t(q + s.n)] = 2 * q + 1;
    }
    if (dm_mirror_enabled()) s.popt.dm_mirror_n = s.n;
}

void state_init(State& s, int n, bool dm, const nq_opts* opts) {
    nq_opts o;
    nq_default_opts(&o);
    if (opts) o = *opts;
    const int guard = o.max_qubits > 0 ? o.max_qubits : (dm ? 14 : 30);
    if (n < 1 || n > guard) {
        throw NqError{NQ_ERR_CONTRACT, std::string(dm ? "density matrix" : "state vector") +
                                           " qubit count must be in [1, " + std::to_string(guard) +
                                           "], got " + std::to_string(n)};
    }
    int dev = o.device;
    if (dev < 0) CUDA_TRY(cudaGetDevice(&dev));
    s.dev = dev;
    s.n = n;
    s.dm = dm;
    s.nbits = dm ? 2 * n : n;
    s.nloc = s.nbits;
    s.count = uint64_t(1) << s.nloc;
    s.popt.nbits = s.nbits;
    s.popt.nloc = s.nloc;
    // 11 tile bits: 2^11 amplitudes per CTA, 4 CTAs of 128 threads per SM
    // (best measured pass throughput on B200)
    s.popt.tile_bits = o.tile_qubits > 0 ? std::min(o.tile_qubits, kMaxTileBits) : 11;
    s.popt.low_bits = 4;
    // relabelling stores for state vectors (NQ_RELABEL=0 disables)
    s.popt.relabel = ab_knob("NQ_RELABEL", 1) != 0;  // density matrices: only with the Hermitian layout (below)
    s.popt.stage_sched = !dm;
    s.layout.resize(size_t(s.nbits));
    set_initial_layout(s);
    // tile size options (read per state), A/B low-bit counts
    if (const int t = env_option(dm ? "NQ_TILE_DM" : "NQ_TILE_SV", 0); t > 0 && o.tile_qubits <= 0)
        s.popt.tile_bits = std::max(4, std::min(t, kMaxTileBits));
    // (density matrices: an even count -- the Hermitian layout pairs bits)
    s.popt.low_bits = dm ? (std::max(0, std::min(ab_knob("NQ_LOW_BITS_DM", 4), 4)) & ~1)
                         : std::max(0, std::min(ab_knob("NQ_LOW_BITS", 4), 7));
    s.popt.fuse = o.fuse != 0;
    configure_caps(s.popt);
    DeviceCtx& c = ctx_for(dev);
    CUDA_TRY(cudaSetDevice(dev));
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&s.d), s.count * sizeof(double2), c.stream));
    launch_init_basis(s.d, s.count, 0, c.stream);
    CUDA_TRY(cudaGetLastError());
}

void configure_caps(PlanOptions& p) {
    const int m = std::min(p.tile_bits, p.nloc);
    if (m <= 10) {
        p.max_ops_per_pass = 1024;
        p.max_pool_per_pass = 6144;
    } else {
        p.max_ops_per_pass = 192;
        p.max_pool_per_pass = 1536;
    }
    static const int cap = ab_knob("NQ_MAX_OPS", 0);
    if (cap > 0) p.max_ops_per_pass = cap;  // A/B measurements
}

void state_free(State& s) {
    if (!s.d) return;
    DeviceCtx& c = ctx_for(s.dev);
    cudaSetDevice(s.dev);
    if (s.dprob) {
        cudaFreeAsync(s.dprob, c.stream);
        s.dprob = nullptr;
        s.dprob_cap = 0;
    }
    if (s.plain_alloc) {
        // peers may map this buffer: release the mappings (shard_free) first
        cudaStreamSynchronize(c.stream);
        shard_free(s);
        cudaFree(s.d);
    } else {
        cudaFreeAsync(s.d, c.stream);
        shard_free(s);
    }
    s.d = nullptr;
}

// NQ_PLAN_TRACE=1: one stderr line per planned pass (micro-op kinds, arity,
// real/zero structure of the matrices) for plan inspection.
bool plan_trace() {
    static const bool on = [] {
        const char* e = std::getenv("NQ_PLAN_TRACE");
        return e && e[0] == '1';
    }();
    return on;
}

void trace_passes(const std::vector<PlannedPass>& passes, bool dm) {
    static const char* names[] = {"D", "G", "X", "S", "P", "L"};
    for (size_t i = 0; i < passes.size(); ++i) {
        const PlannedPass& p = passes[i];
        std::string line;
        for (const MOp& op : p.ops) {
            line += ' ';
            line += op.type < 6 ? names[op.type] : "?";
            line += std::to_string(int(op.k));
            if (op.type == MOP_DENSE) {
                const size_t n = size_t(1) << (2 * op.k);
                size_t nz = 0, re = 0;
                for (size_t e = 0; e < n; ++e) {
                    const cplx v = p.pool[op.mat + e];
                    nz += v != cplx(0.0, 0.0);
                    re += v.imag() == 0.0;
                }
                line += "[" + std::to_string(nz) + "/" + std::to_string(n) + (re == n ? "r" : "") + "]";
            }
        }
        std::fprintf(stderr, "[plan%s] pass %zu m=%zu:%s\n", dm ? " dm" : "", i, p.q.size(), line.c_str());
    }
}

void run_passes(State& s, const std::vector<PlannedPass>& passes, const PlanStats& st, bool record = true,
                JitMemo* memo = nullptr, FlushEpilogue* fe = nullptr);
bool layout_is_identity(const State& s);

// Fused-schedule cache: a flush whose queue (kinds, bits, controls,
// matrices), starting layout and plan options equal a recent flush's reuses
// its planned passes and final layout (repeated circuits: benchmark steps,
// sampling loops, re-runs of a parsed circuit).  Keyed by content.
struct PlanCacheEntry {
    std::vector<unsigned char> key;
    std::vector<PlannedPass> passes;
    PlanStats st;
    std::vector<int> layout_out;
    // compiled kernel of each pass, remembered after its first specialised
    // launch (shared by copies of the entry; see jit_launch's memo)
    std::shared_ptr<std::vector<JitMemo>> kern;
};

std::vector<unsigned char> plan_key(const State& s, bool use_layout) {
    std::vector<unsigned char> k;
    auto put = [&](const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        k.insert(k.end(), b, b + n);
    };
    const PlanOptions& o = s.popt;
    const int32_t opts[] = {o.nbits, o.nloc, o.tile_bits, o.low_bits, o.fuse, o.reg_bits, o.max_ops_per_pass,
                            o.max_pool_per_pass, o.relabel, o.stage_sched, o.dm_mirror_n, use_layout};
    put(opts, sizeof opts);
    if (use_layout) put(s.layout.data(), s.layout.size() * sizeof(int));
    for (const EOp& e : s.queue) {
        const int32_t head[] = {int32_t(e.type), e.k, e.pair_next, int32_t(e.mat.size())};
        put(head, sizeof head);
        put(e.bits, size_t(e.k) * sizeof(int));
        put(&e.ctrl, sizeof e.ctrl);
        put(&e.src, sizeof e.src);
        if (!e.mat.empty()) put(e.mat.data(), e.mat.size() * sizeof(cplx));
    }
    return k;
}

// logical sign masks -> physical bits of the state's current layout
void epilogue_masks(const State& s, const FlushEpilogue& fe, uint64_t* out) {
    for (int t = 0; t < fe.nterms; ++t) {
        uint64_t g = 0;
        for (int q = 0; q < s.n; ++q)
            if ((fe.signs[t] >> q) & 1) g |= uint64_t(1) << (s.layout.empty() ? q : s.layout[size_t(q)]);
        out[t] = g;
    }
}

void state_flush(State& s, FlushEpilogue* fe) {
    if (s.queue.empty()) return;
    if (s.world > 1) {
        shard_flush(s);
        return;
    }
    // entries are immutable once published: a hit copies the pointer under
    // the lock and runs the passes after releasing it, so flushes of other
    // states (and devices) are not serialised behind this one
    static std::mutex mu;
    static std::deque<std::shared_ptr<const PlanCacheEntry>> cache;  // most recent first
    constexpr size_t kCacheEntries = 8;
    PlanStats st;
    const bool use_layout = int(s.layout.size()) == s.nbits && (s.popt.relabel || !layout_is_identity(s));
    std::vector<unsigned char> key = plan_key(s, use_layout);
    const std::vector<int> pre_layout = s.layout;  // (a second plan starts from the same map)
    std::shared_ptr<const PlanCacheEntry> hit;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = cache.begin(); it != cache.end(); ++it) {
            if ((*it)->key != key) continue;
            hit = *it;
            cache.erase(it);
            cache.push_front(hit);
            break;
        }
    }
    if (hit) {
        if (use_layout) s.layout = hit->layout_out;
        s.queue.clear();
        run_passes(s, hit->passes, hit->st, true, hit->kern ? hit->kern->data() : nullptr, fe);
        return;
    }
    std::vector<PlannedPass> passes = plan_passes(s.queue, s.popt, &st, use_layout ? &s.layout : nullptr);
    // A second plan with 5 low bits on lanes (32 contiguous amplitudes per
    // warp access instead of 16) is taken when it needs no more passes and no
    // more relayouts: VQE-28 12.87 -> 12.48 ms; random-30 and QFT-30 then
    // need more passes and keep the 4-bit plan (A/B switch NQ_TRY_LOW5).
    static const bool try_low5 = ab_knob("NQ_TRY_LOW5", 1) != 0;
    if (try_low5 && !s.dm && s.world == 1 && s.popt.low_bits == 4 && s.nloc >= 20 && s.popt.relabel && use_layout) {
        PlanOptions o5 = s.popt;
        o5.low_bits = 5;
        std::vector<int> lay5 = pre_layout;
        PlanStats st5;
        std::vector<PlannedPass> p5 = plan_passes(s.queue, o5, &st5, &lay5);
        auto layouts = [](const std::vector<PlannedPass>& ps) {
            size_t k = 0;
            for (const auto& p : ps)
                for (const auto& o : p.ops) k += o.type == MOP_LAYOUT;
            return k;
        };
        if (p5.size() == passes.size() && layouts(p5) <= layouts(passes)) {
            passes.swap(p5);
            st = st5;
            s.layout = lay5;
        }
    }
    s.queue.clear();
    auto kern = std::make_shared<std::vector<JitMemo>>(passes.size());
    auto entry = std::make_shared<const PlanCacheEntry>(PlanCacheEntry{std::move(key), std::move(passes), st, s.layout, kern});
    {
        std::lock_guard<std::mutex> lk(mu);
        cache.push_front(entry);
        if (cache.size() > kCacheEntries) cache.pop_back();
    }
    run_passes(s, entry->passes, entry->st, true, kern->data(), fe);
}

bool layout_is_identity(const State& s) {
    for (size_t b = 0; b < s.layout.size(); ++b)
        if (s.layout[b] != int(b)) return false;
    return true;
}

// Density-matrix reductions read either layout: flush, and report whether
// the state is interleaved (1) or row-major (0; other layouts are normalised).
int dm_flush_for_reduction(State& s) {
    state_flush(s);
    if (layout_is_identity(s)) return 0;
    bool il = true;
    for (int q = 0; q < s.n && il; ++q)
        il = s.layout[size_t(q)] == 2 * q && s.layout[size_t(q + s.n)] == 2 * q + 1;
    if (il) return 1;
    state_flush_normal(s);
    return 0;
}

void state_flush_normal(State& s) {
    state_flush(s);
    if (s.world > 1 || layout_is_identity(s)) return;
    // transpositions of physical bits that bring logical qubit p back to bit p
    std::vector<int> l2p = s.layout, p2l(l2p.size());
    for (size_t b = 0; b < l2p.size(); ++b) p2l[size_t(l2p[b])] = int(b);
    std::vector<EOp> swaps;
    for (int p = 0; p < s.nbits; ++p) {
        if (p2l[size_t(p)] == p) continue;
        const int w = l2p[size_t(p)];  // physical bit holding logical p
        EOp e;
        e.type = E_SWAP;
        e.k = 2;
        e.bits[0] = std::min(p, w);
        e.bits[1] = std::max(p, w);
        swaps.push_back(e);
        const int lp = p2l[size_t(p)];  // logical qubit at physical p moves to w
        p2l[size_t(w)] = lp;
        l2p[size_t(lp)] = w;
        p2l[size_t(p)] = p;
        l2p[size_t(p)] = p;
    }
    PlanOptions po = s.popt;
    po.relabel = false;
    PlanStats st;
    std::vector<PlannedPass> passes = plan_passes(swaps, po, &st);
    run_passes(s, passes, st, false);
    for (size_t b = 0; b < s.layout.size(); ++b) s.layout[b] = int(b);
}

void run_passes(State& s, const std::vector<PlannedPass>& passes, const PlanStats& st, bool record,
                JitMemo* memo, FlushEpilogue* fe) {
    DeviceCtx& c = ctx_for(s.dev);
    CUDA_TRY(cudaSetDevice(s.dev));
    std::vector<size_t> offs;
    std::vector<unsigned char> buf = serialize_passes(passes, s.nloc, &offs);
    if (record) {
        s.last_passes = st.passes;
        s.last_microops = st.microops;
        s.last_source_ops = st.source_ops;
        s.last_launches = int64_t(passes.size());
    }
    if (buf.empty()) return;
    if (plan_trace()) trace_passes(passes, s.dm);
    NvtxRange flush_range("nq.passes", int64_t(passes.size()));
    c.stage(buf.data(), buf.size());
    for (size_t i = 0; i < passes.size(); ++i) {
        NvtxRange pass_range("nq.pass", int64_t(i));
        PassHdr h;
        std::memcpy(&h, buf.data() + offs[i], sizeof(h));
        std::pair<cudaEvent_t, cudaEvent_t>* ev = c.prof_pass ? prof_slot(c) : nullptr;
        if (ev) CUDA_TRY(cudaEventRecord(ev->first, c.stream));
        const unsigned char* rec = buf.data() + offs[i];
        // the flush's last pass may carry Z-type expectation terms (the
        // layout is already the post-flush one: masks in its physical bits)
        JitEpilogue epi;
        JitEpilogue* ep = nullptr;
        if (fe && fe->nterms > 0 && fe->nterms <= 8 && i + 1 == passes.size() && !s.dm) {
            epi.nterms = fe->nterms;
            epilogue_masks(s, *fe, epi.signs);
            c.ensure_scratch(size_t(4096) * kMaxExpTerms + 64);
            epi.part = c.d_scratch + 64;
            ep = &epi;
        }
        if (ep && jit_launch(s.d, c.d_ops + offs[i], h, reinterpret_cast<const MOp*>(rec + h.op_off),
                             reinterpret_cast<const cplx*>(rec + h.pool_off), 0, c.stream, s.dev, nullptr, nullptr,
                             ep)) {
            launch_expect_final(epi.part, epi.grid, epi.nterms, c.d_scratch, c.stream);
            fe->fused = true;
            fe->dev_sums = c.d_scratch;
        } else if (!jit_launch(s.d, c.d_ops + offs[i], h, reinterpret_cast<const MOp*>(rec + h.op_off),
                        reinterpret_cast<const cplx*>(rec + h.pool_off), 0, c.stream, s.dev, nullptr,
                        memo ? memo + i : nullptr))
            launch_pass(s.d, c.d_ops + offs[i], h, 0, c.stream,
                        reinterpret_cast<const MOp*>(rec + h.op_off)[0].k);
        if (ev) CUDA_TRY(cudaEventRecord(ev->second, c.stream));
        // algorithmic bytes: read + write every element; a Hermitian mirror
        // pass reads only the canonical half (self-mirror tiles are a
        // 2^-(rest bits / 2) fraction: ignored) and writes everything
        if (c.prof) c.prof_pass_bytes += ((h.flags & PASS_MIRROR) ? 24.0 : 32.0) * double(s.count);
    }
    CUDA_TRY(cudaGetLastError());
}

double* result_slot(DeviceCtx& c, int i) { return c.d_scratch + i; }

std::pair<cudaEvent_t, cudaEvent_t>* prof_slot(DeviceCtx& c) {
    if (c.prof_used == c.prof_ev.size()) {
        std::pair<cudaEvent_t, cudaEvent_t> p;
        CUDA_TRY(cudaEventCreate(&p.first));
        CUDA_TRY(cudaEventCreate(&p.second));
        c.prof_ev.push_back(p);
    }
    return &c.prof_ev[c.prof_used++];
}

// Copy `count` doubles from device to the pinned small buffer and wait.
void fetch(DeviceCtx& c, const double* dsrc, size_t count, double* host) {
    c.d2h_bytes += int64_t(count * sizeof(double));
    CUDA_TRY(cudaMemcpyAsync(c.h_small, dsrc, count * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    std::memcpy(host, c.h_small, count * sizeof(double));
}

}  // namespace nqe

namespace {

void check_op_shape(const nq_op& op) {
    if (op.kind < 0 || op.kind > NQ_BARRIER)
        throw NqError{NQ_ERR_CONTRACT, "unknown gate kind " + std::to_string(op.kind)};
    const int arity = kind_arity(op.kind);
    if (op.nqubits != arity)
        throw NqError{NQ_ERR_CONTRACT, "gate expects " + std::to_string(arity) + " qubit(s), got " +
                                           std::to_string(op.nqubits)};
    for (int i = 0; i < arity; ++i)
        for (int j = i + 1; j < arity; ++j)
            if (op.qubits[i] == op.qubits[j])
                throw NqError{NQ_ERR_CONTRACT, "duplicate qubit index " + std::to_string(op.qubits[i])};
}

void check_range(const int32_t* q, int k, int n) {
    for (int j = 0; j < k; ++j)
        if (q[j] < 0 || q[j] >= n)
            throw NqError{NQ_ERR_CONTRACT, "qubit index " + std::to_string(q[j]) + " out of range"};
}

template <class T>
State& st(T* h) {
    if (!h) throw NqError{NQ_ERR_CONTRACT, "null handle"};
    return h->s;
}

bool is_identity_kraus(int k, int nkraus, const cplx* kr) {
    if (nkraus != 1) return false;
    const int d = 1 << k;
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c)
            if (std::abs(kr[r * d + c] - cplx(r == c ? 1.0 : 0.0, 0.0)) > 1e-14) return false;
    return true;
}

void pauli_groups(const uint64_t* flip, int nterms, std::map<uint64_t, std::vector<int>>& groups) {
    for (int t = 0; t < nterms; ++t) groups[flip[t]].push_back(t);
}

const cplx kIPow[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};

}  // namespace

extern "C" {

const char* nq_last_error(void) { return g_last_error.c_str(); }
int nq_abi_version(void) { return NAQS_B200_ABI_VERSION; }

nq_status nq_device_count(int* out) {
    return guard([&] {
        int n = 0;
        CUDA_TRY(cudaGetDeviceCount(&n));
        *out = n;
    });
}

nq_status nq_default_opts(nq_opts* out) {
    if (!out) return NQ_ERR_CONTRACT;
    out->device = -1;
    out->max_qubits = 0;
    out->tile_qubits = 0;
    out->fuse = 1;
    return NQ_OK;
}

// ---- state vector --------------------------------------------------------------
nq_status nq_sv_create(int n, const nq_opts* opts, nq_sv** out) {
    return guard([&] {
        auto h = std::make_unique<nq_sv>();
        state_init(h->s, n, false, opts);
        *out = h.release();
    });
}

nq_status nq_sv_destroy(nq_sv* h) {
    return guard([&] {
        if (!h) return;
        state_free(h->s);
        delete h;
    });
}

nq_status nq_sv_clone(const nq_sv* h, nq_sv** out) {
    return guard([&] {
        State& src = const_cast<nq_sv*>(h)->s;
        if (src.world > 1) throw NqError{NQ_ERR_CONTRACT, "clone of a sharded state is not supported"};
        state_flush_normal(src);
        auto c = std::make_unique<nq_sv>();
        c->s.dev = src.dev;
        c->s.n = src.n;
        c->s.dm = src.dm;
        c->s.nbits = src.nbits;
        c->s.nloc = src.nloc;
        c->s.count = src.count;
        c->s.popt = src.popt;
        c->s.layout = src.layout;  // identity after state_flush_normal
        DeviceCtx& cx = ctx_for(src.dev);
        CUDA_TRY(cudaSetDevice(src.dev));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&c->s.d), src.count * sizeof(double2), cx.stream));
        CUDA_TRY(cudaMemcpyAsync(c->s.d, src.d, src.count * sizeof(double2), cudaMemcpyDeviceToDevice,
                                 cx.stream));
        *out = c.release();
    });
}

nq_status nq_sv_reset(nq_sv* h) {
    return guard([&] {
        State& s = st(h);
        s.queue.clear();
        DeviceCtx& c = ctx_for(s.dev);
        CUDA_TRY(cudaSetDevice(s.dev));
        const uint64_t one_at = (s.world > 1 && s.rank != 0) ? UINT64_MAX : 0;
        launch_init_basis(s.d, s.count, one_at, c.stream);
        shard_reset(s);
        for (size_t b = 0; b < s.layout.size(); ++b) s.layout[b] = int(b);
        CUDA_TRY(cudaGetLastError());
    });
}

nq_status nq_sv_num_qubits(const nq_sv* h, int* out) {
    return guard([&] { *out = st(const_cast<nq_sv*>(h)).n; });
}

nq_status nq_sv_apply_ops(nq_sv* h, const nq_op* ops, int64_t count) {
    return guard([&] {
        State& s = st(h);
        // Validate everything first so a failing call leaves the queue untouched.
        for (int64_t i = 0; i < count; ++i) {
            const nq_op& op = ops[i];
            if (op.kind == NQ_MEASURE)
                throw NqError{NQ_ERR_CONTRACT, "MEASURE has no state-vector kernel; use sample()"};
            check_op_shape(op);
            if (op.kind == NQ_BARRIER) continue;
            check_range(op.qubits, op.nqubits, s.n);
        }
        for (int64_t i = 0; i < count; ++i) lower_sv_op(ops[i], s.queue);
    });
}

nq_status nq_sv_apply_matrix(nq_sv* h, const int32_t* qubits, int k, const double* mat) {
    return guard([&] {
        State& s = st(h);
        if (k < 1 || k > 4) throw NqError{NQ_ERR_CONTRACT, "matrix arity must be in [1, 4]"};
        check_range(qubits, k, s.n);
        for (int i = 0; i < k; ++i)
            for (int j = i + 1; j < k; ++j)
                if (qubits[i] == qubits[j]) throw NqError{NQ_ERR_CONTRACT, "duplicate qubit index"};
        int q[4];
        for (int j = 0; j < k; ++j) q[j] = qubits[j];
        s.queue.push_back(sv_matrix_op(q, k, reinterpret_cast<const cplx*>(mat)));
    });
}

nq_status nq_sv_scale(nq_sv* h, double factor) {
    return guard([&] {
        State& s = st(h);
        EOp e;
        e.type = E_DIAG;
        e.k = 0;
        e.mat = {cplx(factor, 0.0)};
        e.src = 0;
        s.queue.push_back(std::move(e));
    });
}

nq_status nq_sv_flush(nq_sv* h) {
    return guard([&] { state_flush(st(h)); });
}

nq_status nq_sv_norm_sq(nq_sv* h, double* out) {
    return guard([&] {
        State& s = st(h);
        state_flush(s);
        if (s.world > 1) {
            *out = shard_norm_sq(s);
            return;
        }
        DeviceCtx& c = ctx_for(s.dev);
        c.ensure_scratch(scratch_doubles_needed(s.count) + 64);
        launch_sumsq(s.d, s.count, c.d_scratch + 64, result_slot(c, 0), c.stream);
        CUDA_TRY(cudaGetLastError());
        fetch(c, result_slot(c, 0), 1, out);
    });
}

nq_status nq_sv_expectation_batch(nq_sv* h, const uint64_t* flip, const uint64_t* signs,
                                  const int32_t* ny, const double* coeff, int nterms, double* out) {
    return guard([&] {
        State& s = st(h);
        const uint64_t lim = (s.n >= 64) ? ~uint64_t(0) : ((uint64_t(1) << s.n) - 1);
        for (int t = 0; t < nterms; ++t)
            if ((flip[t] & ~lim) || (signs[t] & ~lim))
                throw NqError{NQ_ERR_CONTRACT, "Pauli mask exceeds the state's qubit count"};
        // a pending flush whose result is read only as Z-type terms computes
        // them in its last pass (one state read saved)
        bool diag_only = nterms >= 1 && nterms <= 8 && s.world == 1 && !s.dm && !s.queue.empty();
        for (int t = 0; t < nterms && diag_only; ++t) diag_only = flip[t] == 0;
        FlushEpilogue fe;
        if (diag_only) {
            fe.nterms = nterms;
            fe.signs = signs;
        }
        state_flush(s, diag_only ? &fe : nullptr);
        if (fe.fused) {
            DeviceCtx& c = ctx_for(s.dev);
            std::vector<double> sums(static_cast<size_t>(nterms));
            fetch(c, fe.dev_sums, size_t(nterms), sums.data());
            for (int t = 0; t < nterms; ++t) out[t] = coeff[t] * (cplx(sums[size_t(t)], 0.0) * kIPow[ny[t] & 3]).real();
            return;
        }
        if (s.world > 1) {
            shard_expectation(s, flip, signs, ny, coeff, nterms, out);
            return;
        }
        // masks in physical bits of the current layout (no normalising pass)
        std::vector<uint64_t> pf(flip, flip + nterms), ps(signs, signs + nterms);
        if (!layout_is_identity(s)) {
            for (int t = 0; t < nterms; ++t) {
                uint64_t f = 0, g = 0;
                for (int q = 0; q < s.n; ++q) {
                    if ((flip[t] >> q) & 1) f |= uint64_t(1) << s.layout[size_t(q)];
                    if ((signs[t] >> q) & 1) g |= uint64_t(1) << s.layout[size_t(q)];
                }
                pf[size_t(t)] = f;
                ps[size_t(t)] = g;
            }
        }
        std::vector<cplx> totals;
        sv_expect_raw(s, pf.data(), ps.data(), nterms, totals);
        for (int t = 0; t < nterms; ++t) out[t] = coeff[t] * (totals[size_t(t)] * kIPow[ny[t] & 3]).real();
    });
}

}  // extern "C"

namespace nqe {

// sum_y (-1)^popcount(y & signs) conj(a[y^flip]) a[y] for each term, over this
// device's amplitudes (masks in local bits), before the i^ny factor.
void sv_expect_raw(State& s, const uint64_t* flip, const uint64_t* signs, int nterms, std::vector<cplx>& totals) {
    {
        DeviceCtx& c = ctx_for(s.dev);
        std::vector<int> eps(size_t(nterms), 0);
        for (int t = 0; t < nterms; ++t)
            eps[size_t(t)] = (flip[t] != 0 && (__builtin_popcountll(flip[t] & signs[t]) & 1)) ? 1 : 0;
        // 1) batches of terms whose flips fit one tile: one state read per batch
        const int m = std::min(12, s.nloc);
        const int lb = s.nloc <= 12 ? m : 4;
        const uint64_t lowm = (uint64_t(1) << lb) - 1;
        std::vector<ExpBatch> batches;
        std::vector<uint64_t> bhigh;
        std::vector<std::pair<int, int>> slot_of{static_cast<size_t>(nterms)};  // (batch or launch, index)
        std::vector<int> tiled(size_t(nterms), 0);
        // X/Y-type terms pick the batches (their flips fix the tile bits);
        // Z-type terms then fill free slots anywhere
        std::vector<int> order;
        for (int t = 0; t < nterms; ++t)
            if (flip[t]) order.push_back(t);
        for (int t = 0; t < nterms; ++t)
            if (!flip[t]) order.push_back(t);
        for (int t : order) {
            const uint64_t hi = flip[t] & ~lowm;
            if (__builtin_popcountll(hi) > m - lb) continue;
            size_t b = 0;
            for (; b < batches.size(); ++b)
                if (batches[b].nt < kMaxExpTerms && __builtin_popcountll(bhigh[b] | hi) <= m - lb) break;
            if (b == batches.size()) {
                batches.push_back(ExpBatch{});
                bhigh.push_back(0);
            }
            bhigh[b] |= hi;
            slot_of[size_t(t)] = {int(b), batches[b].nt++};
            tiled[size_t(t)] = 1;
        }
        const size_t part = std::max(scratch_doubles_needed(s.count), expect_tiled_scratch());
        const int tpl = terms_per_launch();
        std::map<uint64_t, std::vector<int>> groups;
        for (int t = 0; t < nterms; ++t)
            if (!tiled[size_t(t)]) groups[flip[t]].push_back(t);
        int launches = 0;
        for (auto& g : groups) launches += int((g.second.size() + tpl - 1) / tpl);
        const size_t res_tiled = batches.size() * kMaxExpTerms;
        c.ensure_scratch(part + res_tiled + size_t(launches) * tpl + 64);
        double* tiled_res = c.d_scratch + part;
        for (size_t b = 0; b < batches.size(); ++b) {
            ExpBatch& B = batches[b];
            uint64_t qm = lowm | bhigh[b];
            for (int bit = 0; bit < s.nloc && __builtin_popcountll(qm) < m; ++bit) qm |= uint64_t(1) << bit;
            int tpos[64];
            int k = 0, r = 0;
            for (int bit = 0; bit < s.nloc; ++bit) {
                if ((qm >> bit) & 1) {
                    tpos[bit] = k;
                    B.q[k++] = int8_t(bit);
                } else {
                    tpos[bit] = -1;
                    B.rest[r++] = int8_t(bit);
                }
            }
            B.m = m;
            B.nrest = r;
            for (int t = 0; t < nterms; ++t) {
                if (!tiled[size_t(t)] || slot_of[size_t(t)].first != int(b)) continue;
                ExpTerm& E = B.t[slot_of[size_t(t)].second];
                E = ExpTerm{};
                for (int bit = 0; bit < s.nloc; ++bit) {
                    if ((flip[t] >> bit) & 1) E.ftile |= 1u << tpos[bit];
                    if ((signs[t] >> bit) & 1) {
                        if (tpos[bit] >= 0) E.stile |= 1u << tpos[bit];
                        else E.sglob |= uint64_t(1) << bit;
                    }
                }
                E.f0 = E.ftile ? __builtin_ctz(E.ftile) : 0;
                E.eps_im = eps[size_t(t)];
            }
            if (!jit_expect_launch(s.d, s.nloc, B, c.d_scratch, tiled_res + b * kMaxExpTerms, c.stream, s.dev))
                launch_expect_tiled(s.d, s.nloc, B, c.d_scratch, tiled_res + b * kMaxExpTerms, c.stream);
        }
        // 2) terms with wide flips: one read per flip group
        double* results = tiled_res + res_tiled;
        int li = 0;
        for (auto& g : groups) {
            const uint64_t F = g.first;
            const auto& terms = g.second;
            for (size_t b = 0; b < terms.size(); b += size_t(tpl)) {
                uint64_t sg[64];
                int ep[64];
                const int nt = int(std::min(terms.size() - b, size_t(tpl)));
                for (int j = 0; j < nt; ++j) {
                    const int t = terms[b + size_t(j)];
                    sg[j] = signs[t];
                    ep[j] = eps[size_t(t)];
                    slot_of[size_t(t)] = {li, j};
                }
                launch_expect_sv(s.d, s.nloc, F, sg, ep, nt, c.d_scratch, results + size_t(li) * tpl,
                                 c.stream);
                ++li;
            }
        }
        CUDA_TRY(cudaGetLastError());
        std::vector<double> host(res_tiled + size_t(launches) * tpl);
        c.d2h_bytes += int64_t(host.size() * sizeof(double));
        if (!host.empty()) {
            CUDA_TRY(cudaMemcpyAsync(host.data(), tiled_res, host.size() * sizeof(double),
                                     cudaMemcpyDeviceToHost, c.stream));
        }
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        for (int t = 0; t < nterms; ++t) {
            const size_t at = tiled[size_t(t)]
                                  ? size_t(slot_of[size_t(t)].first) * kMaxExpTerms + size_t(slot_of[size_t(t)].second)
                                  : res_tiled + size_t(slot_of[size_t(t)].first) * tpl +
                                        size_t(slot_of[size_t(t)].second);
            const double acc = host[at];
            cplx total;
            if (flip[t] == 0) total = cplx(acc, 0.0);
            else total = eps[size_t(t)] ? cplx(0.0, 2.0 * acc) : cplx(2.0 * acc, 0.0);
            totals.push_back(total);
        }
    }
}

}  // namespace nqe

extern "C" {

nq_status nq_sv_probabilities(nq_sv* h, double* host_out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        if (s.world > 1) {
            shard_probabilities(s, host_out);
            return;
        }
        DeviceCtx& c = ctx_for(s.dev);
        const uint64_t chunk = std::min<uint64_t>(s.count, uint64_t(1) << 26);
        double* tmp = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), chunk * sizeof(double), c.stream));
        for (uint64_t off = 0; off < s.count; off += chunk) {
            const uint64_t len = std::min(chunk, s.count - off);
            launch_probs(s.d + off, len, tmp, c.stream);
            CUDA_TRY(cudaMemcpyAsync(host_out + off, tmp, len * sizeof(double), cudaMemcpyDeviceToHost,
                                     c.stream));
        }
        CUDA_TRY(cudaFreeAsync(tmp, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

nq_status nq_sv_sample_sorted(nq_sv* h, const double* sorted_u, uint64_t shots, uint64_t* idx_out,
                              uint64_t* count_out, uint64_t* nout) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        if (s.world > 1) {
            shard_sample(s, sorted_u, shots, idx_out, count_out, nout);
            return;
        }
        DeviceCtx& c = ctx_for(s.dev);
        sample_sweep(c, s.d, nullptr, s.count, sorted_u, shots, idx_out, count_out, nout);
    });
}

nq_status nq_sv_kraus_weights(nq_sv* h, const int32_t* qubits, int k, int nkraus, const double* kraus,
                              double* weights_out) {
    return guard([&] {
        State& s = st(h);
        if (k < 1 || k > 3) throw NqError{NQ_ERR_CONTRACT, "Kraus arity must be in [1, 3]"};
        if (nkraus < 1 || nkraus > 16) throw NqError{NQ_ERR_CONTRACT, "1..16 Kraus operators supported"};
        check_range(qubits, k, s.n);
        state_flush_normal(s);
        if (s.world > 1) throw NqError{NQ_ERR_CONTRACT, "trajectories on a sharded state are not supported"};
        DeviceCtx& c = ctx_for(s.dev);
        const size_t D = size_t(1) << k;
        double2* dm = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dm), size_t(nkraus) * D * D * sizeof(double2),
                                 c.stream));
        CUDA_TRY(cudaMemcpyAsync(dm, kraus, size_t(nkraus) * D * D * sizeof(double2), cudaMemcpyHostToDevice,
                                 c.stream));
        c.ensure_scratch(size_t(16) * 2048 + 64 + 16);
        int q[3] = {qubits[0], k > 1 ? qubits[1] : 0, k > 2 ? qubits[2] : 0};
        launch_kraus_weights(s.d, s.nloc, q, k, nkraus, dm, c.d_scratch + 64, result_slot(c, 0), c.stream);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaFreeAsync(dm, c.stream));
        double w[16];
        fetch(c, result_slot(c, 0), 16, w);
        for (int i = 0; i < nkraus; ++i) weights_out[i] = w[i];
    });
}

nq_status nq_sv_get_amplitudes(nq_sv* h, uint64_t offset, uint64_t count, double* host_out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        if (s.world > 1) {
            shard_get_amplitudes(s, offset, count, host_out);
            return;
        }
        if (offset > s.count || count > s.count - offset)
            throw NqError{NQ_ERR_CONTRACT, "amplitude range out of bounds"};
        DeviceCtx& c = ctx_for(s.dev);
        if (count == 0) return;
        c.d2h_bytes += int64_t(count * sizeof(double2));
        CUDA_TRY(cudaMemcpyAsync(host_out, s.d + offset, count * sizeof(double2), cudaMemcpyDeviceToHost,
                                 c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

nq_status nq_sv_set_amplitudes(nq_sv* h, uint64_t offset, uint64_t count, const double* host_in) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        if (s.world > 1) {
            shard_set_amplitudes(s, offset, count, host_in);
            return;
        }
        if (offset > s.count || count > s.count - offset)
            throw NqError{NQ_ERR_CONTRACT, "amplitude range out of bounds"};
        DeviceCtx& c = ctx_for(s.dev);
        if (count == 0) return;
        CUDA_TRY(cudaMemcpyAsync(s.d + offset, host_in, count * sizeof(double2), cudaMemcpyHostToDevice,
                                 c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

nq_status nq_sv_device_ptr(nq_sv* h, void** out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        shard_normalize(s);  // sharded: this rank's block in logical order
        *out = s.d;
    });
}

// Probabilities kept on the device for zero-copy consumers:
// one state-owned buffer, refilled on every call.
static double* device_prob_buffer(State& s, uint64_t len) {
    DeviceCtx& c = ctx_for(s.dev);
    if (s.dprob_cap < len) {
        if (s.dprob) CUDA_TRY(cudaFreeAsync(s.dprob, c.stream));
        s.dprob = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&s.dprob), len * sizeof(double), c.stream));
        s.dprob_cap = len;
    }
    return s.dprob;
}

nq_status nq_sv_probabilities_device(nq_sv* h, double** out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        shard_normalize(s);
        DeviceCtx& c = ctx_for(s.dev);
        double* p = device_prob_buffer(s, s.count);
        launch_probs(s.d, s.count, p, c.stream);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        *out = p;
    });
}

nq_status nq_sv_device(const nq_sv* h, int* device) {
    return guard([&] { *device = const_cast<nq_sv*>(h)->s.dev; });
}

nq_status nq_dm_device(const nq_dm* h, int* device) {
    return guard([&] { *device = const_cast<nq_dm*>(h)->s.dev; });
}

nq_status nq_sv_local_range(const nq_sv* h, uint64_t* offset, uint64_t* count) {
    return guard([&] {
        const State& s = const_cast<nq_sv*>(h)->s;
        *offset = uint64_t(s.rank) << s.nloc;
        *count = s.count;
    });
}

nq_status nq_sv_last_stats(const nq_sv* h, int64_t* passes, int64_t* microops, int64_t* source_ops,
                           int64_t* launches) {
    return guard([&] {
        const State& s = const_cast<nq_sv*>(h)->s;
        if (passes) *passes = s.last_passes;
        if (microops) *microops = s.last_microops;
        if (source_ops) *source_ops = s.last_source_ops;
        if (launches) *launches = s.last_launches;
    });
}

nq_status nq_sv_synchronize(nq_sv* h) {
    return guard([&] {
        State& s = st(h);
        CUDA_TRY(cudaSetDevice(s.dev));
        CUDA_TRY(cudaStreamSynchronize(ctx_for(s.dev).stream));
    });
}

// ---- density matrix ----------------------------------------------------------------
nq_status nq_dm_create(int n, const nq_opts* opts, nq_dm** out) {
    return guard([&] {
        auto h = std::make_unique<nq_dm>();
        state_init(h->s, n, true, opts);
        *out = h.release();
    });
}

nq_status nq_dm_destroy(nq_dm* h) {
    return guard([&] {
        if (!h) return;
        state_free(h->s);
        delete h;
    });
}

nq_status nq_dm_clone(const nq_dm* h, nq_dm** out) {
    return guard([&] {
        State& src = const_cast<nq_dm*>(h)->s;
        state_flush_normal(src);
        auto c = std::make_unique<nq_dm>();
        c->s.dev = src.dev;
        c->s.n = src.n;
        c->s.dm = true;
        c->s.nbits = src.nbits;
        c->s.nloc = src.nloc;
        c->s.count = src.count;
        c->s.popt = src.popt;
        c->s.layout = src.layout;  // identity after state_flush_normal
        DeviceCtx& cx = ctx_for(src.dev);
        CUDA_TRY(cudaSetDevice(src.dev));
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&c->s.d), src.count * sizeof(double2), cx.stream));
        CUDA_TRY(cudaMemcpyAsync(c->s.d, src.d, src.count * sizeof(double2), cudaMemcpyDeviceToDevice,
                                 cx.stream));
        *out = c.release();
    });
}

nq_status nq_dm_reset(nq_dm* h) {
    return guard([&] {
        State& s = st(h);
        s.queue.clear();
        DeviceCtx& c = ctx_for(s.dev);
        CUDA_TRY(cudaSetDevice(s.dev));
        launch_init_basis(s.d, s.count, 0, c.stream);
        set_initial_layout(s);
        CUDA_TRY(cudaGetLastError());
    });
}

nq_status nq_dm_num_qubits(const nq_dm* h, int* out) {
    return guard([&] { *out = st(const_cast<nq_dm*>(h)).n; });
}

static void dm_validate_gate(const State& s, const nq_op& op) {
    if (op.kind == NQ_MEASURE)
        throw NqError{NQ_ERR_CONTRACT, "MEASURE has no density-matrix kernel; use probabilities()"};
    check_op_shape(op);
    if (op.kind == NQ_BARRIER || op.kind == NQ_ID) return;
    check_range(op.qubits, op.nqubits, s.n);
}

nq_status nq_dm_apply_ops(nq_dm* h, const nq_op* ops, int64_t count) {
    return guard([&] {
        State& s = st(h);
        for (int64_t i = 0; i < count; ++i) dm_validate_gate(s, ops[i]);
        for (int64_t i = 0; i < count; ++i) {
            if (ops[i].kind == NQ_BARRIER || ops[i].kind == NQ_ID) {
                if (ops[i].kind == NQ_ID) {
                    EOp e;  // counted, no work (densitymatrix.cpp:115)
                    s.queue.push_back(e);
                }
                continue;
            }
            lower_dm_op(ops[i], s.n, s.queue);
        }
    });
}

static void dm_channel(State& s, const int32_t* qubits, int k, int nkraus, const double* kraus) {
    if (k != 1 && k != 2)
        throw NqError{NQ_ERR_CONTRACT, "channel arity must be 1 or 2, got " + std::to_string(k)};
    if (nkraus < 1) throw NqError{NQ_ERR_CONTRACT, "channel needs at least one Kraus operator"};
    check_range(qubits, k, s.n);
    if (k == 2 && qubits[0] == qubits[1]) throw NqError{NQ_ERR_CONTRACT, "duplicate qubit index"};
    const cplx* kr = reinterpret_cast<const cplx*>(kraus);
    if (is_identity_kraus(k, nkraus, kr)) return;  // densitymatrix.cpp:138
    int q[2] = {qubits[0], k > 1 ? qubits[1] : 0};
    s.queue.push_back(dm_channel_op(q, k, nkraus, kr, s.n));
}

nq_status nq_dm_apply_channel(nq_dm* h, const int32_t* qubits, int k, int nkraus, const double* kraus) {
    return guard([&] { dm_channel(st(h), qubits, k, nkraus, kraus); });
}

nq_status nq_dm_apply_schedule(nq_dm* h, const nq_sched_item* items, int64_t count, const double* pool) {
    return guard([&] {
        State& s = st(h);
        // validate all first (reference run_schedule validates item by item and
        // throws mid-way; we reject the whole schedule before touching rho)
        for (int64_t i = 0; i < count; ++i) {
            const nq_sched_item& it = items[i];
            if (it.type == 0) {
                if (it.op.kind == NQ_MEASURE || it.op.kind == NQ_BARRIER) continue;
                dm_validate_gate(s, it.op);
            } else {
                if (it.op.nqubits != 1 && it.op.nqubits != 2)
                    throw NqError{NQ_ERR_CONTRACT, "channel arity must be 1 or 2"};
                check_range(it.op.qubits, it.op.nqubits, s.n);
            }
        }
        for (int64_t i = 0; i < count; ++i) {
            const nq_sched_item& it = items[i];
            if (it.type == 0) {
                if (it.op.kind == NQ_MEASURE || it.op.kind == NQ_BARRIER) continue;
                if (it.op.kind == NQ_ID) {
                    s.queue.push_back(EOp{});
                    continue;
                }
                lower_dm_op(it.op, s.n, s.queue);
            } else {
                dm_channel(s, it.op.qubits, it.op.nqubits, it.nkraus, pool + 2 * it.kraus_offset);
            }
        }
    });
}

nq_status nq_dm_flush(nq_dm* h) {
    return guard([&] { state_flush(st(h)); });
}

nq_status nq_dm_trace(nq_dm* h, double* out) {
    return guard([&] {
        State& s = st(h);
        const int il = dm_flush_for_reduction(s);
        DeviceCtx& c = ctx_for(s.dev);
        const uint64_t dim = uint64_t(1) << s.n;
        c.ensure_scratch(scratch_doubles_needed(dim) + 64);
        launch_trace(s.d, dim, c.d_scratch + 64, result_slot(c, 0), c.stream, il);
        CUDA_TRY(cudaGetLastError());
        fetch(c, result_slot(c, 0), 1, out);
    });
}

nq_status nq_dm_purity(nq_dm* h, double* out) {
    return guard([&] {
        State& s = st(h);
        state_flush(s);
        DeviceCtx& c = ctx_for(s.dev);
        c.ensure_scratch(scratch_doubles_needed(s.count) + 64);
        launch_sumsq(s.d, s.count, c.d_scratch + 64, result_slot(c, 0), c.stream);
        CUDA_TRY(cudaGetLastError());
        fetch(c, result_slot(c, 0), 1, out);
    });
}

nq_status nq_dm_hermiticity_residual(nq_dm* h, double* out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        DeviceCtx& c = ctx_for(s.dev);
        c.ensure_scratch(2048 + 64);
        launch_herm(s.d, uint64_t(1) << s.n, c.d_scratch + 64, result_slot(c, 0), c.stream);
        CUDA_TRY(cudaGetLastError());
        fetch(c, result_slot(c, 0), 1, out);
    });
}

nq_status nq_dm_expectation_batch(nq_dm* h, const uint64_t* flip, const uint64_t* signs, const int32_t* ny,
                                  const double* coeff, int nterms, double* out_re, double* out_im) {
    return guard([&] {
        State& s = st(h);
        const uint64_t lim = (uint64_t(1) << s.n) - 1;
        for (int t = 0; t < nterms; ++t)
            if ((flip[t] & ~lim) || (signs[t] & ~lim))
                throw NqError{NQ_ERR_CONTRACT, "Pauli mask exceeds the state's qubit count"};
        const int il = dm_flush_for_reduction(s);
        DeviceCtx& c = ctx_for(s.dev);
        const uint64_t dim = uint64_t(1) << s.n;
        std::map<uint64_t, std::vector<int>> groups;
        pauli_groups(flip, nterms, groups);
        const int tpl = terms_per_launch();
        int launches = 0;
        for (auto& g : groups) launches += int((g.second.size() + tpl - 1) / tpl);
        const size_t part = scratch_doubles_needed(dim);
        c.ensure_scratch(part + size_t(launches) * 2 * tpl + 64);
        double* results = c.d_scratch + part;
        std::vector<std::pair<int, int>> slot_of{static_cast<size_t>(nterms)};
        int li = 0;
        for (auto& g : groups) {
            const auto& terms = g.second;
            for (size_t b = 0; b < terms.size(); b += size_t(tpl)) {
                uint64_t sg[64];
                const int nt = int(std::min(terms.size() - b, size_t(tpl)));
                for (int j = 0; j < nt; ++j) {
                    sg[j] = signs[terms[b + size_t(j)]];
                    slot_of[size_t(terms[b + size_t(j)])] = {li, j};
                }
                launch_expect_dm(s.d, s.n, g.first, sg, nt, c.d_scratch, results + size_t(li) * 2 * tpl,
                                 c.stream, il);
                ++li;
            }
        }
        CUDA_TRY(cudaGetLastError());
        std::vector<double> host(size_t(launches) * 2 * tpl);
        if (!host.empty())
            CUDA_TRY(cudaMemcpyAsync(host.data(), results, host.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                     c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        for (int t = 0; t < nterms; ++t) {
            const size_t base = size_t(slot_of[size_t(t)].first) * 2 * tpl + 2 * size_t(slot_of[size_t(t)].second);
            cplx total(host[base], host[base + 1]);
            total *= kIPow[ny[t] & 3];
            out_re[t] = coeff[t] * total.real();
            if (out_im) out_im[t] = total.imag();
        }
    });
}

nq_status nq_dm_probabilities(nq_dm* h, double* host_out) {
    return guard([&] {
        State& s = st(h);
        const int il = dm_flush_for_reduction(s);
        DeviceCtx& c = ctx_for(s.dev);
        const uint64_t dim = uint64_t(1) << s.n;
        c.ensure_scratch(scratch_doubles_needed(dim) + 64);
        double* p = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p), dim * sizeof(double), c.stream));
        launch_dm_probs(s.d, dim, p, c.d_scratch, c.stream, il);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(host_out, p, dim * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        CUDA_TRY(cudaFreeAsync(p, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

nq_status nq_dm_device_ptr(nq_dm* h, void** out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);  // row-major rho (the interleaved layout is undone)
        CUDA_TRY(cudaSetDevice(s.dev));
        CUDA_TRY(cudaStreamSynchronize(ctx_for(s.dev).stream));
        *out = s.d;
    });
}

nq_status nq_dm_probabilities_device(nq_dm* h, double** out) {
    return guard([&] {
        State& s = st(h);
        const int il = dm_flush_for_reduction(s);
        DeviceCtx& c = ctx_for(s.dev);
        const uint64_t dim = uint64_t(1) << s.n;
        c.ensure_scratch(scratch_doubles_needed(dim) + 64);
        double* p = device_prob_buffer(s, dim);
        launch_dm_probs(s.d, dim, p, c.d_scratch, c.stream, il);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        *out = p;
    });
}

nq_status nq_dm_get_entries(nq_dm* h, uint64_t offset, uint64_t count, double* host_out) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        if (offset > s.count || count > s.count - offset)
            throw NqError{NQ_ERR_CONTRACT, "entry range out of bounds"};
        if (count == 0) return;
        DeviceCtx& c = ctx_for(s.dev);
        CUDA_TRY(cudaMemcpyAsync(host_out, s.d + offset, count * sizeof(double2), cudaMemcpyDeviceToHost,
                                 c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

nq_status nq_dm_set_entries(nq_dm* h, uint64_t offset, uint64_t count, const double* host_in) {
    return guard([&] {
        State& s = st(h);
        state_flush_normal(s);
        if (offset > s.count || count > s.count - offset)
            throw NqError{NQ_ERR_CONTRACT, "entry range out of bounds"};
        if (count == 0) return;
        DeviceCtx& c = ctx_for(s.dev);
        CUDA_TRY(cudaMemcpyAsync(s.d + offset, host_in, count * sizeof(double2), cudaMemcpyHostToDevice,
                                 c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

nq_status nq_dm_last_stats(const nq_dm* h, int64_t* passes, int64_t* microops, int64_t* source_ops,
                           int64_t* launches) {
    return guard([&] {
        const State& s = const_cast<nq_dm*>(h)->s;
        if (passes) *passes = s.last_passes;
        if (microops) *microops = s.last_microops;
        if (source_ops) *source_ops = s.last_source_ops;
        if (launches) *launches = s.last_launches;
    });
}

nq_status nq_dm_synchronize(nq_dm* h) {
    return guard([&] {
        State& s = st(h);
        CUDA_TRY(cudaSetDevice(s.dev));
        CUDA_TRY(cudaStreamSynchronize(ctx_for(s.dev).stream));
    });
}

// ---- readout -------------------------------------------------------------------------
nq_status nq_readout_apply_dist(const double* dist_in, int n, const double* p01, const double* p10,
                                double* dist_out) {
    return guard([&] {
        if (n < 0 || n > 40) throw NqError{NQ_ERR_CONTRACT, "readout qubit count out of range"};
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        DeviceCtx& c = ctx_for(dev);
        const uint64_t len = uint64_t(1) << n;
        double* d = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), len * sizeof(double), c.stream));
        CUDA_TRY(cudaMemcpyAsync(d, dist_in, len * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        c.ensure_scratch(scratch_doubles_needed(len) + 64);
        launch_sum_real(d, len, c.d_scratch + 64, result_slot(c, 0), c.stream);
        double sum = 0.0;
        fetch(c, result_slot(c, 0), 1, &sum);
        if (std::abs(sum - 1.0) > 1e-9) {
            cudaFreeAsync(d, c.stream);
            throw NqError{NQ_ERR_CONTRACT, "distribution sums to " + std::to_string(sum) + ", expected 1"};
        }
        for (int q = 0; q < n; ++q) {
            if (p01[q] == 0.0 && p10[q] == 0.0) continue;
            launch_readout(d, n, q, p01[q], p10[q], c.stream);
        }
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(dist_out, d, len * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        CUDA_TRY(cudaFreeAsync(d, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    });
}

// ---- measurement ----------------------------------------------------------------------
nq_status nq_profile_begin(int device, int per_pass_events) {
    return guard([&] {
        int dev = device;
        if (dev < 0) CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaSetDevice(dev));
        DeviceCtx& c = ctx_for(dev);
        if (!c.prof_t0) {
            CUDA_TRY(cudaEventCreate(&c.prof_t0));
            CUDA_TRY(cudaEventCreate(&c.prof_t1));
        }
        c.prof = true;
        c.prof_pass = per_pass_events != 0;
        c.prof_used = 0;
        c.prof_pass_bytes = 0.0;
        c.h2d_bytes = c.d2h_bytes = 0;
        c.prof_launch0 = g_kernel_launches.load();
        CUDA_TRY(cudaEventRecord(c.prof_t0, c.stream));
    });
}

nq_status nq_profile_end(int device, nq_profile* out) {
    return guard([&] {
        int dev = device;
        if (dev < 0) CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaSetDevice(dev));
        DeviceCtx& c = ctx_for(dev);
        if (!c.prof) throw NqError{NQ_ERR_CONTRACT, "nq_profile_end without nq_profile_begin"};
        CUDA_TRY(cudaEventRecord(c.prof_t1, c.stream));
        CUDA_TRY(cudaEventSynchronize(c.prof_t1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, c.prof_t0, c.prof_t1));
        nq_profile p{};
        p.region_ms = ms;
        double pass = 0.0;
        for (size_t i = 0; i < c.prof_used; ++i) {
            float m = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&m, c.prof_ev[i].first, c.prof_ev[i].second));
            pass += m;
        }
        p.pass_ms = pass;
        p.pass_launches = int64_t(c.prof_used);
        p.pass_bytes = c.prof_pass_bytes;
        p.kernel_launches = g_kernel_launches.load() - c.prof_launch0;
        p.h2d_bytes = c.h2d_bytes;
        p.d2h_bytes = c.d2h_bytes;
        c.prof = c.prof_pass = false;
        *out = p;
    });
}

nq_status nq_jit_wait(void) {
    return guard([&] { jit_wait(); });
}

nq_status nq_jit_shutdown(void) {
    return guard([&] { jit_shutdown(); });
}

nq_status nq_jit_stats(int64_t* compiled, int64_t* failed, int64_t* misses, int64_t* launches) {
    return guard([&] {
        const JitStats j = jit_stats();
        if (compiled) *compiled = j.compiled;
        if (failed) *failed = j.failed;
        if (misses) *misses = j.misses;
        if (launches) *launches = j.launches;
    });
}

nq_status nq_jit_debug(int n, const nq_op* ops, int64_t count, int tile_qubits, int pass_index, int compile,
                       char* src_out, int64_t cap, int64_t* size, int* compiled_ok) {
    return guard([&] {
        std::vector<EOp> q;
        for (int64_t i = 0; i < count; ++i) {
            check_op_shape(ops[i]);
            if (ops[i].kind != NQ_BARRIER) check_range(ops[i].qubits, ops[i].nqubits, n);
            lower_sv_op(ops[i], q);
        }
        PlanOptions p;
        p.nbits = n;
        p.nloc = n;
        p.tile_bits = tile_qubits > 0 ? std::min(tile_qubits, kMaxTileBits) : 11;  // the state default (state_init)
        // as single-device state vectors plan; compile & 4: as a sharded
        // segment plans (no relabelling, no carried layout)
        p.relabel = (compile & 4) == 0;
        configure_caps(p);
        std::vector<int> layout(static_cast<size_t>(n));
        for (int b = 0; b < n; ++b) layout[size_t(b)] = b;
        auto passes = plan_passes(q, p, nullptr, (compile & 4) ? nullptr : &layout);
        if (pass_index < 0 || pass_index >= int(passes.size())) throw NqError{NQ_ERR_CONTRACT, "no such pass"};
        std::vector<size_t> offs;
        auto bytes = serialize_passes(passes, n, &offs);
        const unsigned char* rec = bytes.data() + offs[size_t(pass_index)];
        PassHdr h;
        std::memcpy(&h, rec, sizeof(h));
        // compile & 8: the staged exchange-store form (16 chunks, exchanged
        // bit v = the top rest bit, or with compile & 16 a tile bit)
        JitXStore xs;
        if (compile & 8) {
            const int vpos = (compile & 16) ? h.q[std::min(2, h.m - 1)] : h.rest[h.nrest - 1];
            xs.staged = true;
            xs.xmask = uint64_t(1) << vpos;
            xs.xrot = 0;
            for (int j = 0; j < h.nrest; ++j)
                if (h.rest[j] == vpos) xs.xrot = j;
            xs.cshift = std::max(1, h.nrest - 4);
            xs.chunk_bits = jit_stage_chunk_bits(h, xs.xrot, xs.cshift);
            xs.pushers = 16;
        }
        // compile & 32: with a fused Z-term epilogue (Z on physical bits 0,
        // n-1 and 0+1)
        JitEpilogue epi;
        epi.nterms = 3;
        epi.signs[0] = 1;
        epi.signs[1] = uint64_t(1) << (n - 1);
        epi.signs[2] = 3;
        std::string src = jit_source(h, reinterpret_cast<const MOp*>(rec + h.op_off),
                                     reinterpret_cast<const cplx*>(rec + h.pool_off), (compile & 10) != 0,
                                     (compile & 8) ? &xs : nullptr, (compile & 32) ? &epi : nullptr);
        std::string log;
        if (compiled_ok) *compiled_ok = (compile & 1) ? int(jit_compile_only(src, &log)) : -1;
        if (!log.empty()) src += "\n/* NVRTC LOG\n" + log + "\n*/\n";
        *size = int64_t(src.size());
        if (src_out && cap > 0) std::memcpy(src_out, src.data(), size_t(std::min<int64_t>(cap, *size)));
    });
}

// ---- planner introspection -------------------------------------------------------------
nq_status nq_plan_debug(int n, const nq_op* ops, int64_t count, int tile_qubits, int fuse, unsigned char* buf,
                        int64_t cap, int64_t* size) {
    return guard([&] {
        if (n < 1 || n > kMaxStateBits) throw NqError{NQ_ERR_CONTRACT, "qubit count out of range"};
        std::vector<EOp> q;
        for (int64_t i = 0; i < count; ++i) {
            if (ops[i].kind == NQ_MEASURE) throw NqError{NQ_ERR_CONTRACT, "MEASURE in plan"};
            check_op_shape(ops[i]);
            if (ops[i].kind != NQ_BARRIER) check_range(ops[i].qubits, ops[i].nqubits, n);
            lower_sv_op(ops[i], q);
        }
        PlanOptions p;
        p.nbits = n;
        p.nloc = n;
        p.tile_bits = tile_qubits > 0 ? std::min(tile_qubits, kMaxTileBits) : 11;  // the state default (state_init)
        p.fuse = (fuse & 1) != 0;
        p.relabel = (fuse & 2) != 0;  // bit 1: relabelling stores (single-device state vectors)
        if (fuse >> 4) p.low_bits = (fuse >> 4) & 7;  // bits 4-6: low-bit count (planner experiments)
        configure_caps(p);
        PlanStats stt;
        std::vector<int> layout(static_cast<size_t>(n));
        for (int b = 0; b < n; ++b) layout[size_t(b)] = b;
        auto passes = plan_passes(q, p, &stt, &layout);
        std::vector<size_t> offs;
        auto bytes = serialize_passes(passes, n, &offs);
        *size = int64_t(bytes.size());
        if (buf && cap > 0) std::memcpy(buf, bytes.data(), size_t(std::min<int64_t>(cap, int64_t(bytes.size()))));
    });
}

}  // extern "C"

extern "C" {

// ---- batches of small circuits ---------------------------------------------------
nq_status nq_batch_run(int n, int dm, int64_t batch, const int64_t* item_off, const nq_sched_item* items,
                       const double* kraus_pool, const uint64_t* flip, const uint64_t* signs, const int32_t* ny,
                       const double* coeff, int nterms, double* out, double* out_im, double* probs, int device) {
    return guard([&] {
        const int maxq = dm ? kMaxBatchBits / 2 : kMaxBatchBits;
        if (n < 1 || n > maxq)
            throw NqError{NQ_ERR_CONTRACT, std::string(dm ? "density-matrix" : "state-vector") +
                                               " batch qubit count must be in [1, " + std::to_string(maxq) +
                                               "], got " + std::to_string(n)};
        if (batch < 0 || nterms < 0) throw NqError{NQ_ERR_CONTRACT, "negative batch or term count"};
        std::vector<TrajItem> prog;
        std::vector<cplx> pool;
        std::vector<int64_t> off(size_t(batch) + 1, 0);
        // Liouville lowering with caches: a long noisy circuit repeats a few
        // distinct superoperators, and products of consecutive ones on the same
        // (or nested) bit sets are fused once and reused.
        std::map<std::vector<double>, int64_t> content_at;  // matrix data -> pool offset
        std::map<std::vector<double>, int64_t> gate_super_at;  // gate matrix U -> its superoperator
        std::map<std::tuple<int64_t, int32_t, int>, int64_t> channel_at;  // (kraus_offset, nkraus, k) -> superop
        std::map<std::tuple<int64_t, int64_t, unsigned>, int64_t> product_at;  // (new, last, positions) -> fused
        auto intern = [&](const cplx* m, size_t len) {
            std::vector<double> key(reinterpret_cast<const double*>(m), reinterpret_cast<const double*>(m) + 2 * len);
            auto f = content_at.find(key);
            if (f != content_at.end()) return f->second;
            const int64_t at = int64_t(pool.size());
            pool.insert(pool.end(), m, m + len);
            content_at.emplace(std::move(key), at);
            return at;
        };
        auto push_item = [&](int k, const int* q, int64_t mat, int64_t first_of_circuit) {
            // fuse into the previous item of this circuit when our bits are a subset of its bits
            if (dm && int64_t(prog.size()) > first_of_circuit) {
                TrajItem& last = prog.back();
                int pos[4];
                bool subset = k <= last.k;
                for (int j = 0; j < k && subset; ++j) {
                    pos[j] = -1;
                    for (int i = 0; i < last.k; ++i)
                        if (last.q[i] == q[j]) pos[j] = i;
                    subset = pos[j] >= 0;
                }
                if (subset) {
                    unsigned code = unsigned(k);
                    for (int j = 0; j < k; ++j) code |= unsigned(pos[j]) << (4 + 2 * j);
                    const auto key = std::make_tuple(mat, last.mat, code);
                    auto f = product_at.find(key);
                    if (f == product_at.end()) {
                        // fused = (A on positions pos) * M_last, column by column
                        const int D = 1 << last.k, d = 1 << k;
                        std::vector<cplx> M(pool.begin() + last.mat, pool.begin() + last.mat + size_t(D) * D);
                        const cplx* A = pool.data() + mat;
                        unsigned pm = 0;
                        for (int j = 0; j < k; ++j) pm |= 1u << pos[j];
                        std::vector<cplx> x(static_cast<size_t>(d)), y(static_cast<size_t>(d));
                        for (int col = 0; col < D; ++col)
                            for (int g = 0; g < D; ++g) {
                                if (unsigned(g) & pm) continue;  // g: base with the sub bits clear
                                for (int c = 0; c < d; ++c) {
                                    int r = g;
                                    for (int j = 0; j < k; ++j)
                                        if ((c >> j) & 1) r |= 1 << pos[j];
                                    x[size_t(c)] = M[size_t(r) * D + col];
                                }
                                for (int rr = 0; rr < d; ++rr) {
                                    cplx acc(0.0, 0.0);
                                    for (int c = 0; c < d; ++c) acc += A[size_t(rr) * d + c] * x[size_t(c)];
                                    y[size_t(rr)] = acc;
                                }
                                for (int c = 0; c < d; ++c) {
                                    int r = g;
                                    for (int j = 0; j < k; ++j)
                                        if ((c >> j) & 1) r |= 1 << pos[j];
                                    M[size_t(r) * D + col] = y[size_t(c)];
                                }
                            }
                        f = product_at.emplace(key, intern(M.data(), M.size())).first;
                    }
                    last.mat = f->second;
                    return;
                }
            }
            TrajItem t{};
            t.type = 0;
            t.k = k;
            for (int j = 0; j < k; ++j) t.q[j] = q[j];
            t.nmat = 1;
            t.mat = mat;
            prog.push_back(t);
        };
        for (int64_t b = 0; b < batch; ++b) {
            const int64_t first = int64_t(prog.size());
            off[size_t(b)] = first;
            if (item_off[b + 1] < item_off[b]) throw NqError{NQ_ERR_CONTRACT, "item offsets must be non-decreasing"};
            for (int64_t i = item_off[b]; i < item_off[b + 1]; ++i) {
                const nq_sched_item& it = items[i];
                if (it.type == 0) {
                    const nq_op& op = it.op;
                    if (op.kind == NQ_MEASURE || op.kind == NQ_BARRIER || op.kind == NQ_ID) continue;
                    check_op_shape(op);
                    check_range(op.qubits, op.nqubits, n);
                    const std::vector<cplx> m = full_gate_matrix(op);
                    const int k = op.nqubits;
                    if (!dm) {
                        push_item(k, op.qubits, intern(m.data(), m.size()), first);
                        continue;
                    }
                    if (k <= 2) {
                        // U (x) conj(U) on [qs, qs + n] (lower.cpp::superop with one Kraus operator),
                        // cached by U
                        std::vector<double> ukey(reinterpret_cast<const double*>(m.data()),
                                                 reinterpret_cast<const double*>(m.data()) + 2 * m.size());
                        auto g = gate_super_at.find(ukey);
                        if (g == gate_super_at.end()) {
                            const std::vector<cplx> S = superop(k, {m.data()});
                            g = gate_super_at.emplace(std::move(ukey), intern(S.data(), S.size())).first;
                        }
                        int q2[4];
                        for (int j = 0; j < k; ++j) {
                            q2[j] = op.qubits[j];
                            q2[j + k] = op.qubits[j] + n;
                        }
                        push_item(2 * k, q2, g->second, first);
                    } else {
                        // CCX: U on the row bits, conj(U) on the column bits
                        int rq[3], cq[3];
                        for (int j = 0; j < k; ++j) {
                            rq[j] = op.qubits[j] + n;
                            cq[j] = op.qubits[j];
                        }
                        std::vector<cplx> mc(m.size());
                        for (size_t e = 0; e < m.size(); ++e) mc[e] = std::conj(m[e]);
                        push_item(k, rq, intern(m.data(), m.size()), first);
                        push_item(k, cq, intern(mc.data(), mc.size()), first);
                    }
                } else {
                    if (!dm) throw NqError{NQ_ERR_CONTRACT, "channels need a density-matrix batch (or nq_traj_run)"};
                    const int k = it.op.nqubits;
                    if (k < 1 || k > 2) throw NqError{NQ_ERR_CONTRACT, "batch channel arity must be 1 or 2"};
                    if (it.nkraus < 1) throw NqError{NQ_ERR_CONTRACT, "channel without Kraus operators"};
                    check_range(it.op.qubits, k, n);
                    const auto ckey = std::make_tuple(it.kraus_offset, it.nkraus, k);
                    auto f = channel_at.find(ckey);
                    if (f == channel_at.end()) {
                        const cplx* src = reinterpret_cast<const cplx*>(kraus_pool) + it.kraus_offset;
                        std::vector<const cplx*> ks;
                        for (int kk = 0; kk < it.nkraus; ++kk) ks.push_back(src + (size_t(kk) << (2 * k)));
                        const std::vector<cplx> S = superop(k, ks);
                        f = channel_at.emplace(ckey, intern(S.data(), S.size())).first;
                    }
                    int q2[4];
                    for (int j = 0; j < k; ++j) {
                        q2[j] = it.op.qubits[j];
                        q2[j + k] = it.op.qubits[j] + n;
                    }
                    push_item(2 * k, q2, f->second, first);
                }
            }
        }
        off[size_t(batch)] = int64_t(prog.size());
        if (batch == 0) return;
        const auto t_lowered = std::chrono::steady_clock::now();
        DeviceCtx& c = ctx_for(device < 0 ? 0 : device);
        CUDA_TRY(cudaSetDevice(c.dev));
        const size_t dq = size_t(1) << n, nt = size_t(nterms), B = size_t(batch);
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t o_off = 0, o_items = al(o_off + off.size() * 8);
        const size_t o_pool = al(o_items + prog.size() * sizeof(TrajItem));
        const size_t o_f = al(o_pool + pool.size() * sizeof(cplx)), o_s = al(o_f + nt * 8);
        const size_t o_re = al(o_s + nt * 8), o_im = al(o_re + B * nt * 8), o_p = al(o_im + B * nt * 8);
        const size_t total = o_p + (probs ? B * dq * 8 : 0) + 256;
        unsigned char* d = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), total, c.stream));
        auto h2d = [&](size_t o, const void* src, size_t bytes) {
            if (bytes) CUDA_TRY(cudaMemcpyAsync(d + o, src, bytes, cudaMemcpyHostToDevice, c.stream));
            c.h2d_bytes += int64_t(bytes);
        };
        h2d(o_off, off.data(), off.size() * 8);
        h2d(o_items, prog.data(), prog.size() * sizeof(TrajItem));
        h2d(o_pool, pool.data(), pool.size() * sizeof(cplx));
        h2d(o_f, flip, nt * 8);
        h2d(o_s, signs, nt * 8);
        BatchArgs p{};
        p.bits = dm ? 2 * n : n;
        p.n = n;
        p.dm = dm;
        p.nterms = nterms;
        p.prog_off = reinterpret_cast<const int64_t*>(d + o_off);
        p.items = reinterpret_cast<const TrajItem*>(d + o_items);
        p.pool = reinterpret_cast<const double2*>(d + o_pool);
        p.flip = reinterpret_cast<const uint64_t*>(d + o_f);
        p.signs = reinterpret_cast<const uint64_t*>(d + o_s);
        p.out_re = reinterpret_cast<double*>(d + o_re);
        p.out_im = reinterpret_cast<double*>(d + o_im);
        p.probs = probs ? reinterpret_cast<double*>(d + o_p) : nullptr;
        launch_batch(p, batch, c.stream);
        CUDA_TRY(cudaGetLastError());
        std::vector<double> re(B * nt), im(B * nt);
        auto d2h = [&](void* dst, size_t o, size_t bytes) {
            if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, d + o, bytes, cudaMemcpyDeviceToHost, c.stream));
            c.d2h_bytes += int64_t(bytes);
        };
        d2h(re.data(), o_re, re.size() * 8);
        d2h(im.data(), o_im, im.size() * 8);
        if (probs) d2h(probs, o_p, B * dq * 8);
        CUDA_TRY(cudaFreeAsync(d, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        if (std::getenv("NQ_BATCH_TIMING"))
            std::fprintf(stderr, "[nq_batch_run] device+copies %.2f ms, %zu programs items, pool %zu\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_lowered).count(),
                         prog.size(), pool.size());
        for (size_t b = 0; b < B; ++b)
            for (size_t j = 0; j < nt; ++j) {
                const cplx tot = cplx(re[b * nt + j], im[b * nt + j]) * kIPow[ny[j] & 3];
                out[b * nt + j] = coeff[j] * tot.real();
                if (out_im) out_im[b * nt + j] = tot.imag();
            }
    });
}

// ---- batched trajectories -----------------------------------------------------
nq_status nq_traj_run(int n, const nq_sched_item* items, int64_t count, const double* kraus_pool, int64_t ntraj,
                      const double* uniforms, const uint64_t* flip, const uint64_t* signs, const int32_t* ny,
                      const double* coeff, int nterms, double* out, int32_t* branch_out, double* amps_out,
                      int device) {
    return guard([&] {
        if (n < 1 || n > kMaxTrajQubits)
            throw NqError{NQ_ERR_CONTRACT, "trajectory batch qubit count must be in [1, " +
                                               std::to_string(kMaxTrajQubits) + "], got " + std::to_string(n)};
        if (ntraj < 0 || nterms < 0) throw NqError{NQ_ERR_CONTRACT, "negative trajectory or term count"};
        std::vector<TrajItem> prog;
        std::vector<cplx> pool;
        int nch = 0;
        for (int64_t i = 0; i < count; ++i) {
            const nq_sched_item& it = items[i];
            TrajItem t{};
            if (it.type == 0) {
                const nq_op& op = it.op;
                if (op.kind == NQ_MEASURE || op.kind == NQ_BARRIER || op.kind == NQ_ID) continue;
                check_op_shape(op);
                check_range(op.qubits, op.nqubits, n);
                t.type = 0;
                t.k = op.nqubits;
                for (int j = 0; j < t.k; ++j) t.q[j] = op.qubits[j];
                t.nmat = 1;
                t.mat = int64_t(pool.size());
                const std::vector<cplx> m = full_gate_matrix(op);
                pool.insert(pool.end(), m.begin(), m.end());
            } else {
                const int k = it.op.nqubits;
                if (k < 1 || k > 3) throw NqError{NQ_ERR_CONTRACT, "channel arity must be 1..3"};
                if (it.nkraus < 1 || it.nkraus > kMaxTrajKraus)
                    throw NqError{NQ_ERR_CONTRACT, "channel Kraus count out of range"};
                check_range(it.op.qubits, k, n);
                t.type = 1;
                t.k = k;
                for (int j = 0; j < k; ++j) t.q[j] = it.op.qubits[j];
                t.nmat = it.nkraus;
                t.mat = int64_t(pool.size());
                const size_t len = size_t(it.nkraus) << (2 * k);
                const cplx* src = reinterpret_cast<const cplx*>(kraus_pool) + it.kraus_offset;
                pool.insert(pool.end(), src, src + len);
                ++nch;
            }
            prog.push_back(t);
        }
        if (ntraj == 0) return;
        DeviceCtx& c = ctx_for(device < 0 ? 0 : device);
        CUDA_TRY(cudaSetDevice(c.dev));
        const size_t dim = size_t(1) << n;
        const size_t nt = size_t(nterms), tr = size_t(ntraj), C = size_t(nch);
        // one device block: items | pool | uniforms | flip | signs | re | im | branch | amps | err
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t o_items = 0, o_pool = al(o_items + prog.size() * sizeof(TrajItem));
        const size_t o_u = al(o_pool + pool.size() * sizeof(cplx));
        const size_t o_f = al(o_u + tr * C * sizeof(double));
        const size_t o_s = al(o_f + nt * 8), o_re = al(o_s + nt * 8), o_im = al(o_re + tr * nt * 8);
        const size_t o_br = al(o_im + tr * nt * 8), o_am = al(o_br + (branch_out ? tr * C * 4 : 0));
        const size_t o_err = al(o_am + (amps_out ? tr * dim * 16 : 0)), total = o_err + 256;
        unsigned char* d = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), total, c.stream));
        auto h2d = [&](size_t off, const void* src, size_t bytes) {
            if (bytes) CUDA_TRY(cudaMemcpyAsync(d + off, src, bytes, cudaMemcpyHostToDevice, c.stream));
            c.h2d_bytes += int64_t(bytes);
        };
        h2d(o_items, prog.data(), prog.size() * sizeof(TrajItem));
        h2d(o_pool, pool.data(), pool.size() * sizeof(cplx));
        h2d(o_u, uniforms, tr * C * sizeof(double));
        h2d(o_f, flip, nt * 8);
        h2d(o_s, signs, nt * 8);
        CUDA_TRY(cudaMemsetAsync(d + o_err, 0, 4, c.stream));
        TrajArgs p{};
        p.n = n;
        p.nitems = int(prog.size());
        p.nchannels = nch;
        p.nterms = nterms;
        p.items = reinterpret_cast<const TrajItem*>(d + o_items);
        p.pool = reinterpret_cast<const double2*>(d + o_pool);
        p.uniforms = reinterpret_cast<const double*>(d + o_u);
        p.flip = reinterpret_cast<const uint64_t*>(d + o_f);
        p.signs = reinterpret_cast<const uint64_t*>(d + o_s);
        p.out_re = reinterpret_cast<double*>(d + o_re);
        p.out_im = reinterpret_cast<double*>(d + o_im);
        p.branch_out = branch_out ? reinterpret_cast<int32_t*>(d + o_br) : nullptr;
        p.amps_out = amps_out ? reinterpret_cast<double2*>(d + o_am) : nullptr;
        p.err = reinterpret_cast<int*>(d + o_err);
        launch_traj(p, ntraj, c.stream);
        CUDA_TRY(cudaGetLastError());
        std::vector<double> re(tr * nt), im(tr * nt);
        int err = 0;
        auto d2h = [&](void* dst, size_t off, size_t bytes) {
            if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, d + off, bytes, cudaMemcpyDeviceToHost, c.stream));
            c.d2h_bytes += int64_t(bytes);
        };
        d2h(re.data(), o_re, re.size() * 8);
        d2h(im.data(), o_im, im.size() * 8);
        if (branch_out) d2h(branch_out, o_br, tr * C * 4);
        if (amps_out) d2h(amps_out, o_am, tr * dim * 16);
        d2h(&err, o_err, 4);
        CUDA_TRY(cudaFreeAsync(d, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        if (err)
            throw NqError{NQ_ERR_CONTRACT,
                          "Kraus branch probabilities do not sum to 1; channel is not trace preserving on this state"};
        for (size_t b = 0; b < tr; ++b)
            for (size_t j = 0; j < nt; ++j) {
                const cplx tot(re[b * nt + j], im[b * nt + j]);
                out[b * nt + j] = coeff[j] * (tot * kIPow[ny[j] & 3]).real();
            }
    });
}

}  // extern "C"

extern "C" nq_status nq_sample_dist_sorted(const double* dist, uint64_t len, const double* sorted_u,
                                           uint64_t shots, uint64_t* idx_out, uint64_t* count_out,
                                           uint64_t* nout) {
    return guard([&] {
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        DeviceCtx& c = ctx_for(dev);
        double* d = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), len * sizeof(double), c.stream));
        CUDA_TRY(cudaMemcpyAsync(d, dist, len * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        try {
            sample_sweep(c, nullptr, d, len, sorted_u, shots, idx_out, count_out, nout);
        } catch (...) {
            cudaFreeAsync(d, c.stream);
            throw;
        }
        CUDA_TRY(cudaFreeAsync(d, c.stream));
    });
}

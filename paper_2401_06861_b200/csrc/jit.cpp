// Pass-specialised kernels, generated and compiled at run time (NVRTC).
//
// The interpreter kernel (pass_kernel.cu) decodes micro-ops at run time; its
// per-op dispatch costs about as many instructions as the op itself.  A pass
// record fully determines a straight-line program: tile bits, register
// layouts, slots, controls and which diagonal entries are exactly 1 are all
// compile-time here, so the generated kernel is pure loads, FP64 math,
// register moves and relayouts.  Operator matrices stay in the pass's pool
// (shared memory), so re-running the same circuit structure with new angles
// (VQE, Trotter sweeps, repeated benchmark steps) reuses the compiled kernel.
//
// Memory pipeline of the generated pass kernel: each thread streams its 16
// amplitudes of the tile straight into registers in the first register
// layout (128-bit ld.global.cs), computes, relayouts through one shared-memory
// tile buffer, and streams the results out of registers (st.global.cs).
// Residency (4 CTAs x 128 threads x 128 registers per SM) hides the load
// latency.  Measured and removed (round 1, profiles/r01b_*): a cp.async
// double buffer, bulk (TMA) staging, L2 bulk prefetch and warp-local
// relayouts were all slower, because the extra shared memory halves the
// resident CTAs.  The relayout buffer addressing uses a per-pass linear
// swizzle chosen so that every register layout of the pass is bank-conflict
// free.
//
// Compilation is asynchronous: the first time a structure is seen the
// interpreter runs it while worker threads compile; later flushes use the
// specialised kernel.  NQ_JIT=off|auto|sync selects the policy.
#include "jit.hpp"

#include "kernels.hpp"
#include "knobs.hpp"
#include "state.hpp"

#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <dlfcn.h>
#include <execinfo.h>
#include <csignal>
#include <unistd.h>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace nqe {

namespace {

const char* kPassOpsSrc =
#include "pass_ops_src.inc"
    ;

// NVRTC is bound at first use from the toolkit this library was built with
// (NQ_NVRTC_PATH, the Makefile's CUDA_HOME), not through the soname: a process
// that imported torch first already has torch's own, older libnvrtc.so.12
// loaded, and that one rejects the pass kernels' 256-bit global accesses for
// sm_100a.  Loaded RTLD_LOCAL, so the two copies do not interfere.  If only an
// NVRTC older than 12.9 can be found, the kernels fall back to 128-bit pairs.
struct NvrtcApi {
    decltype(&::nvrtcCreateProgram) CreateProgram = nullptr;
    decltype(&::nvrtcCompileProgram) CompileProgram = nullptr;
    decltype(&::nvrtcDestroyProgram) DestroyProgram = nullptr;
    decltype(&::nvrtcGetCUBIN) GetCUBIN = nullptr;
    decltype(&::nvrtcGetCUBINSize) GetCUBINSize = nullptr;
    decltype(&::nvrtcGetProgramLog) GetProgramLog = nullptr;
    decltype(&::nvrtcGetProgramLogSize) GetProgramLogSize = nullptr;
    decltype(&::nvrtcVersion) Version = nullptr;
    bool wide = true;  // 256-bit global accesses supported
    std::string where;
};

#ifndef NQ_NVRTC_PATH
#define NQ_NVRTC_PATH "/usr/local/cuda/lib64/libnvrtc.so.12"
#endif

NvrtcApi& nvrtc() {
    static NvrtcApi api = [] {
        NvrtcApi a;
        void* h = dlopen(NQ_NVRTC_PATH, RTLD_NOW | RTLD_LOCAL);
        a.where = NQ_NVRTC_PATH;
        if (!h) {
            h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
            a.where = "libnvrtc.so.12";
        }
        if (!h) throw NqError{NQ_ERR_CUDA, std::string("NVRTC unavailable: ") + (dlerror() ? dlerror() : "")};
#define NQ_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
        NQ_SYM(CreateProgram, "nvrtcCreateProgram");
        NQ_SYM(CompileProgram, "nvrtcCompileProgram");
        NQ_SYM(DestroyProgram, "nvrtcDestroyProgram");
        NQ_SYM(GetCUBIN, "nvrtcGetCUBIN");
        NQ_SYM(GetCUBINSize, "nvrtcGetCUBINSize");
        NQ_SYM(GetProgramLog, "nvrtcGetProgramLog");
        NQ_SYM(GetProgramLogSize, "nvrtcGetProgramLogSize");
        NQ_SYM(Version, "nvrtcVersion");
#undef NQ_SYM
        if (!a.CreateProgram || !a.CompileProgram || !a.GetCUBIN || !a.Version)
            throw NqError{NQ_ERR_CUDA, "NVRTC at " + a.where + " lacks required entry points"};
        int major = 0, minor = 0;
        a.Version(&major, &minor);
        a.wide = major > 12 || (major == 12 && minor >= 9);
        return a;
    }();
    return api;
}

#define nvrtcCreateProgram nvrtc().CreateProgram
#define nvrtcCompileProgram nvrtc().CompileProgram
#define nvrtcDestroyProgram nvrtc().DestroyProgram
#define nvrtcGetCUBIN nvrtc().GetCUBIN
#define nvrtcGetCUBINSize nvrtc().GetCUBINSize
#define nvrtcGetProgramLog nvrtc().GetProgramLog
#define nvrtcGetProgramLogSize nvrtc().GetProgramLogSize

struct Entry {
    std::atomic<int> state{0};  // 0 pending, 1 ready, 2 failed
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    std::map<int, int> occ;  // device -> blocks per SM
    std::string log;
};

struct Jit {
    std::mutex mu;
    std::condition_variable cv;
    std::unordered_map<std::string, std::shared_ptr<Entry>> cache;
    std::deque<std::pair<std::string, std::shared_ptr<Entry>>> queue;
    int busy = 0;
    bool started = false;
    bool exiting = false;
    int device = 0;
    JitStats stats;
};

Jit& jit() {
    static Jit* j = new Jit();  // leaked on purpose: no teardown-order issues with the workers
    return *j;
}

JitMode mode_from_env() {
    const char* e = std::getenv("NQ_JIT");
    if (!e) return JitMode::Auto;
    const std::string s(e);
    if (s == "off" || s == "0") return JitMode::Off;
    if (s == "sync") return JitMode::Sync;
    return JitMode::Auto;
}

std::string hex64(unsigned long long v) {
    char b[32];
    std::snprintf(b, sizeof b, "0x%llxull", v);
    return b;
}

// deposit bits of `src` (low bits first) into the ascending positions `pos`,
// as an expression built from runs of consecutive positions.
std::string deposit_expr(const std::string& src, const std::vector<int>& pos, bool wide) {
    std::ostringstream o;
    const char* one = wide ? "1ull" : "1u";
    bool first = true;
    size_t k = 0;
    while (k < pos.size()) {
        size_t e = k;
        while (e + 1 < pos.size() && pos[e + 1] == pos[e] + 1) ++e;
        const size_t len = e - k + 1;
        if (!first) o << " | ";
        first = false;
        o << "(((" << src << " >> " << k << ") & ((" << one << " << " << len << ") - " << one << ")) << " << pos[k]
          << ")";
        k = e + 1;
    }
    if (first) o << (wide ? "0ull" : "0u");
    return o.str();
}

struct Layout {
    int rp[4];
    int r = 4;
    std::vector<int> nonr;  // ascending tile bits that are thread bits
    unsigned rconst(int l) const {
        unsigned c = 0;
        for (int j = 0; j < r; ++j)
            if ((l >> j) & 1) c |= 1u << rp[j];
        return c;
    }
};

Layout layout_of(const MOp& op, int m) {
    Layout L;
    L.r = op.k;
    unsigned rm = 0;
    for (int j = 0; j < L.r; ++j) {
        L.rp[j] = op.pos[j];
        rm |= 1u << op.pos[j];
    }
    for (int b = 0; b < m; ++b)
        if (!((rm >> b) & 1u)) L.nonr.push_back(b);
    return L;
}

// Linear swizzle: address = (e & ~7) | sum_p e_p * v[p] (over GF(2)).
struct Swizzle {
    unsigned v[16];
    unsigned apply(unsigned e) const {
        unsigned lo = 0;
        for (int p = 0; p < 16; ++p)
            if ((e >> p) & 1u) lo ^= v[p];
        return (e & ~7u) | lo;
    }
    // masks of the positions contributing to address bit i
    unsigned mask(int i) const {
        unsigned m = 0;
        for (int p = 0; p < 16; ++p)
            if ((v[p] >> i) & 1u) m |= 1u << p;
        return m;
    }
};

bool independent3(unsigned a, unsigned b, unsigned c) {
    return a && b && c && a != b && (a ^ b) != c && a != c && b != c;
}

// Make the three lowest thread bits of every layout (and of the natural
// order) map to distinct 16-byte bank groups.
Swizzle choose_swizzle(const std::vector<Layout>& lays, int m) {
    std::vector<std::array<int, 3>> triples;
    triples.push_back({0, 1, 2});
    for (const auto& L : lays)
        if (L.nonr.size() >= 3) triples.push_back({L.nonr[0], L.nonr[1], L.nonr[2]});
    Swizzle sw{};
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (int attempt = 0; attempt < 20000; ++attempt) {
        for (int p = 0; p < 16; ++p) {
            if (attempt == 0) {
                sw.v[p] = (p < 3) ? (1u << p) : (1u << (p % 3));  // fold-by-3 default
            } else {
                x ^= x << 13;
                x ^= x >> 7;
                x ^= x << 17;
                sw.v[p] = p < m ? unsigned(1 + x % 7) : 0u;
            }
        }
        bool ok = true;
        for (const auto& t : triples) ok = ok && independent3(sw.v[t[0]], sw.v[t[1]], sw.v[t[2]]);
        if (ok) return sw;
    }
    for (int p = 0; p < 16; ++p) sw.v[p] = p < 3 ? (1u << p) : 0u;  // identity: always a bijection
    return sw;
}

std::string swz_expr(const std::string& x, const Swizzle& sw) {
    std::ostringstream o;
    o << "((" << x << " & ~7u)";
    for (int i = 0; i < 3; ++i) {
        const unsigned mk = sw.mask(i);
        if (mk) o << " | ((unsigned)(__popc(" << x << " & " << mk << "u) & 1) << " << i << ")";
    }
    o << ")";
    return o.str();
}

}  // namespace

// NQ_DIAG_SKIP=1: runtime test of each hoisted diagonal factor (A/B).
// Pending register permutation (NQ_JIT_PX=0 disables): an X whose controls
// lie outside the register slots (thread / tile / global bits) is not applied
// to the registers but XOR-ed into a per-thread mask px (the true amplitude
// of register index l is a[l ^ px]); later operators read their matrices
// conjugated by it, diagonals index their tables through it, and relayouts
// and stores XOR it into their addresses, where it disappears.  Ops that need
// the registers in true order (register-controlled X, k >= 3 operators,
// sparse k <= 2 operators, depolarizing maps) first apply the pending bits
// they touch.
bool px_enabled() {
    static const bool on = env_option("NQ_JIT_PX", 1) != 0;
    return on;
}

// Per-thread phase accumulators for unit-modulus diagonal tables (see the
// generator).  NQ_JIT_PHASEACC=0 disables them (A/B).
bool accumulate_phases() {
    static const bool on = ab_knob("NQ_JIT_PHASEACC", 1) != 0;
    return on;
}

bool diag_runtime_skip() {
    static const bool on = ab_knob("NQ_DIAG_SKIP", 0) != 0;
    return on;
}

// Dense k <= 2 operator with structural zeros (Liouville superoperators of
// damping / dephasing channels, diagonal-times-permutation products): only the
// nonzero entries are multiplied, and entries with an exact zero imaginary
// part use real-times-complex products.  Values stay in the shared pool, so the
// kernel is reused for every matrix with the same zero / real pattern.
// Dense k <= 2 operator generated entry by entry with compile-time entry
// classes: zero (skipped), real, pure imaginary (2 FP64 per product, like
// real: U (x) conj(U) of RX and its products with damping / dephasing
// superoperators are of this kind), or complex.  Values stay in the shared
// pool, so the kernel is reused for every matrix with the same pattern.
// Few nonzeros are hoisted into registers; otherwise each use reloads its
// entry from shared memory (as the d2 template does) to spare registers.
std::string sparse_dense(const MOp& op, const cplx* u, int E, const std::string& P) {
    const int d = 1 << op.k;
    // O / M: exactly +1 / -1 (pivot-normalised rows, planner.cpp): an addition
    enum Cls { Z, R, I, C, O, M };
    auto cls = [&](int e) {
        const cplx v = u[e];
        if (v == cplx(0.0, 0.0)) return Z;
        if (v == cplx(1.0, 0.0)) return O;
        if (v == cplx(-1.0, 0.0)) return M;
        if (v.imag() == 0.0) return R;
        if (v.real() == 0.0) return I;
        return C;
    };
    int nnz = 0;
    for (int e = 0; e < d * d; ++e) nnz += cls(e) != Z && cls(e) != O && cls(e) != M;
    const bool hoist = nnz <= 8;
    auto load = [&](int e) {
        std::ostringstream o;
        o << "lds(" << P << " + " << e << ")" << (cls(e) == R ? ".x" : cls(e) == I ? ".y" : "");
        return o.str();
    };
    std::ostringstream s;
    s << "    {\n";
    if (hoist)
        for (int e = 0; e < d * d; ++e) {
            if (cls(e) == Z || cls(e) == O || cls(e) == M) continue;
            s << "      const " << (cls(e) == C ? "double2" : "double") << " u" << e << " = " << load(e) << ";\n";
        }
    unsigned smask = 0;
    for (int j = 0; j < op.k; ++j) smask |= 1u << op.pos[j];
    for (int l = 0; l < E; ++l) {
        if (unsigned(l) & smask) continue;
        auto idx = [&](int i) {
            int x = l;
            for (int j = 0; j < op.k; ++j)
                if ((i >> j) & 1) x |= 1 << op.pos[j];
            return x;
        };
        s << "      {";
        for (int c = 0; c < d; ++c) s << " const double2 x" << c << " = a[" << idx(c) << "];";
        s << "\n";
        for (int r = 0; r < d; ++r) {
            const std::string dst = "a[" + std::to_string(idx(r)) + "]";
            bool first = true;
            // +-1 terms first: they seed the accumulator (a copy / negation the
            // next fma takes as its addend), later ones are additions
            std::vector<int> order;
            for (int c = 0; c < d; ++c)
                if (cls(r * d + c) == O || cls(r * d + c) == M) order.push_back(c);
            for (int c = 0; c < d; ++c)
                if (!(cls(r * d + c) == O || cls(r * d + c) == M)) order.push_back(c);
            for (int c : order) {
                const int e = r * d + c;
                const Cls k = cls(e);
                if (k == Z) continue;
                if (k == O || k == M) {
                    const std::string xn = "x" + std::to_string(c);
                    const char* sg = k == O ? "" : "-";
                    if (first) s << "        " << dst << " = make_double2(" << sg << xn << ".x, " << sg << xn << ".y);\n";
                    else s << "        " << dst << ".x " << (k == O ? "+" : "-") << "= " << xn << ".x; " << dst << ".y "
                           << (k == O ? "+" : "-") << "= " << xn << ".y;\n";
                    first = false;
                    continue;
                }
                const std::string un = hoist ? "u" + std::to_string(e) : "(" + load(e) + ")";
                const std::string xn = "x" + std::to_string(c);
                s << "        ";
                if (k == R) {
                    if (first) s << dst << " = make_double2(" << un << " * " << xn << ".x, " << un << " * " << xn << ".y);\n";
                    else s << dst << ".x = fma(" << un << ", " << xn << ".x, " << dst << ".x); " << dst << ".y = fma(" << un
                           << ", " << xn << ".y, " << dst << ".y);\n";
                } else if (k == I) {
                    // (i w) x = (-w x.y, w x.x)
                    if (first) s << dst << " = make_double2(-(" << un << " * " << xn << ".y), " << un << " * " << xn << ".x);\n";
                    else s << dst << ".x = fma(-" << un << ", " << xn << ".y, " << dst << ".x); " << dst << ".y = fma(" << un
                           << ", " << xn << ".x, " << dst << ".y);\n";
                } else {
                    if (first) s << dst << " = cmul(" << un << ", " << xn << ");\n";
                    else s << dst << " = cfma(" << un << ", " << xn << ", " << dst << ");\n";
                }
                first = false;
            }
            if (first) s << "        " << dst << " = make_double2(0.0, 0.0);\n";
        }
        s << "      }\n";
    }
    s << "    }\n";
    return s.str();
}

// Bounded waits of a staged exchange (pass kernel and pusher): a stall is
// recorded in the sync buffer and reported by the host instead of hanging.
constexpr unsigned long long kStageWatchdogNs = 60000000000ull;

uint64_t jit_stage_chunk_bits(const PassHdr& h, int xrot, int cshift) {
    // rotated counter rr: r bit 0 -> rest position xrot, r bit j >= 1 -> rest
    // position j - 1 below xrot + 1, j above (see the exchange passes' rr)
    uint64_t bits = 0;
    for (int j = std::max(cshift, 1); j < h.nrest; ++j) bits |= uint64_t(1) << h.rest[j <= xrot ? j - 1 : j];
    return bits;
}

std::string jit_source(const PassHdr& h, const MOp* ops, const cplx* pool, bool xstore, const JitXStore* stage,
                       const JitEpilogue* epi) {
    const int nep = (epi && !xstore && !(h.flags & PASS_MIRROR)) ? epi->nterms : 0;
    const bool staged = xstore && stage && stage->staged;
    // staged exchange: compressed position of physical bit p in a staging
    // slot (-1: a removed bit -- a chunk bit or the exchanged bit v)
    const uint64_t holes = staged ? (stage->chunk_bits | stage->xmask) : 0;
    auto cpos = [&](int p) {
        if ((holes >> p) & 1) return -1;
        return p - __builtin_popcountll(holes & ((uint64_t(1) << p) - 1));
    };
    const int m = h.m;
    const int SIZE = 1 << m;
    const int E = 1 << ops[0].k;  // ops[0] is the load layout: 3 or 4 register bits
    const int T = SIZE / E;
    int logT = 0;
    while ((1 << logT) < T) ++logT;
    std::vector<int> q(h.q, h.q + m), rest(h.rest, h.rest + h.nrest);
    std::vector<int> qst(h.qst, h.qst + m);  // store positions (a permutation of q: relabelled pass)
    const bool relabel = qst != q;
    // Hermitian (mirror) pass: tile / rest bits pair as physical (2q, 2q+1)
    bool mirror = (h.flags & PASS_MIRROR) && !xstore;
    std::vector<int> tpair(size_t(m), -1), rpair(rest.size(), -1);
    for (int i = 0; i < m && mirror; ++i)
        for (int j = 0; j < m; ++j)
            if (q[size_t(j)] == (q[size_t(i)] ^ 1)) tpair[size_t(i)] = j;
    for (size_t i = 0; i < rest.size() && mirror; ++i)
        for (size_t j = 0; j < rest.size(); ++j)
            if (rest[j] == (rest[i] ^ 1)) rpair[i] = int(j);
    for (int x : tpair) mirror = mirror && x >= 0;
    for (int x : rpair) mirror = mirror && x >= 0;
    std::vector<int> qmir(static_cast<size_t>(m));
    for (int i = 0; i < m && mirror; ++i) qmir[size_t(i)] = qst[size_t(tpair[size_t(i)])];
    auto mirror_rest_expr = [&](const std::string& r) {
        std::ostringstream o;
        o << "0ull";
        for (size_t j = 0; j < rest.size(); ++j)
            o << " | (((" << r << " >> " << j << ") & 1ull) << " << rpair[j] << ")";
        return o.str();
    };

    std::vector<Layout> lays;
    std::vector<int> lay_of_op(size_t(h.nops), 0);
    for (int i = 0; i < h.nops; ++i) {
        if (ops[i].type == MOP_LAYOUT) lays.push_back(layout_of(ops[i], m));
        lay_of_op[size_t(i)] = int(lays.size()) - 1;
    }
    // Relabelling pass: the tile bits a warp's lanes span must be the ones that
    // store to the low (contiguous) physical bits, so the stores go through one
    // more relayout into LS = the last layout with its thread bits ordered by
    // store position.
    // When the pass already relayouts, its last layout simply takes that
    // thread-bit order (no extra shared-memory round trip).
    auto by_store = [&](Layout L) {
        std::stable_sort(L.nonr.begin(), L.nonr.end(), [&](int x, int y) { return qst[size_t(x)] < qst[size_t(y)]; });
        return L;
    };
    if (relabel && lays.size() >= 2) lays.back() = by_store(lays.back());
    const bool extra_relayout = relabel && lays.size() == 1;
    if (extra_relayout) mirror = false;  // (full tiles then; the mirror store path expects the last layout)
    Layout LS = by_store(lays.back());
    if (extra_relayout) {
        // the extra relayout is free to pick the store layout's register bits:
        // the tile bits with the highest store positions, so the lanes of a
        // warp span the lowest ones (fully coalesced 512-byte stores) even when
        // the program's only layout holds low store bits in registers
        std::vector<int> bits(static_cast<size_t>(m));
        for (int b = 0; b < m; ++b) bits[size_t(b)] = b;
        std::stable_sort(bits.begin(), bits.end(), [&](int x, int y) { return qst[size_t(x)] > qst[size_t(y)]; });
        unsigned rm = 0;
        for (int j = 0; j < LS.r; ++j) rm |= 1u << bits[size_t(j)];
        int j = 0;
        for (int b = 0; b < m; ++b)
            if ((rm >> b) & 1u) LS.rp[j++] = b;
        LS.nonr.clear();
        for (int b = 0; b < m; ++b)
            if (!((rm >> b) & 1u)) LS.nonr.push_back(b);
        LS = by_store(LS);
    }
    std::vector<Layout> sw_lays = lays;
    if (extra_relayout) sw_lays.push_back(LS);
    const Swizzle sw = choose_swizzle(sw_lays, m);
    auto reg_off = [&](const Layout& L, int l, const std::vector<int>& pos) {
        unsigned long long c = 0;
        for (int j = 0; j < L.r; ++j)
            if ((l >> j) & 1) c |= 1ull << pos[size_t(L.rp[j])];
        return c;
    };
    auto state_off = [&](const std::string& tbname, const std::vector<int>& bits, const std::vector<int>& pos) {
        std::ostringstream o;
        bool first = true;
        for (int b : bits) {
            if (!first) o << " | ";
            first = false;
            o << "((unsigned long long)((" << tbname << " >> " << b << ") & 1u) << " << pos[size_t(b)] << ")";
        }
        if (first) o << "0ull";
        return o.str();
    };

    std::ostringstream s;
    s << "#include \"pass_ops.cuh\"\n"
      << "extern \"C\" __global__ void __launch_bounds__(" << T;
    // 8 amplitudes per thread need ~half the registers: aim for 768 threads/SM.
    // Passes with >= 45 arithmetic micro-ops (QFT's phase-table passes) run
    // 3 CTAs/SM of up to 168 registers instead of 4 of 128: their schedules
    // keep more loads and table factors in flight without spilling.
    // Measured (A/B NQ_HEAVY_OPS): QFT-30 73.7 -> 70.8 ms at thresholds 40-50
    // (72.3 at 60); random-30 and VQE-28 unchanged; 2 CTAs/SM for >= 60 ops
    // (NQ_HEAVY2_OPS) slower.
    static const int heavy_ops = ab_knob("NQ_HEAVY_OPS", 45);
    static const int heavy2_ops = ab_knob("NQ_HEAVY2_OPS", 0);  // (2 CTAs/SM, up to 255 registers)
    int narith = 0;
    for (int i = 0; i < h.nops; ++i) narith += ops[i].type == MOP_DENSE || ops[i].type == MOP_DIAG;
    const int minb = (heavy2_ops > 0 && E == 16 && narith >= heavy2_ops) ? std::max(1, 256 / T)
                     : (heavy_ops > 0 && E == 16 && narith >= heavy_ops) ? std::max(1, 384 / T)
                                                                          : std::max(1, (E == 8 ? 768 : 512) / T);
    if (minb > 0) s << ", " << minb;
    s << ")\n"
      << "nqjit(double2* __restrict__ st, const double2* __restrict__ gpool, unsigned long long rankbase,"
         " long long ntiles, double2* xout_l, double2* xout_r, unsigned long long xmask, unsigned long long xval,"
         " int xrot" << (staged ? ", unsigned* pdone, const unsigned* qdone, unsigned long long slot_elems,"
                                  " double2* xpeer, const unsigned* xpeer_done, unsigned npass" : "")
      << (nep ? ", double* __restrict__ epart" : "") << ") {\n"
      << "  using namespace nq;\n"
      << "  extern __shared__ __align__(16) unsigned char smem[];\n"
      << "  double2* buf0 = reinterpret_cast<double2*>(smem);\n"
      << "  double2* pool = buf0 + " << SIZE << ";\n"
      << "  const unsigned tid = threadIdx.x;\n";
    if (staged) {
        // staged exchange: CTAs >= npass are the pusher (cooperative launch:
        // the whole grid is co-resident, so the waits cannot deadlock)
        const int cb = h.nrest - stage->cshift;
        // slot index k -> partner index: k deposited into the kept bit runs
        // (between the holes), plus the chunk number's bits at the chunk-bit
        // holes and v = this rank's bit (xval: the partner keeps v = mybit)
        std::vector<int> hp;
        for (int p = 0; p < 64; ++p)
            if ((holes >> p) & 1) hp.push_back(p);
        std::ostringstream ex;
        ex << "(xval & xmask)";
        int src_bit = 0, prev = 0;  // k bits consumed, next kept position
        for (size_t j = 0; j <= hp.size(); ++j) {
            const int end = j < hp.size() ? hp[j] : 63;  // kept run [prev, end)
            if (end > prev)
                ex << " | (((k >> " << src_bit << ") & " << hex64((end - prev >= 64) ? ~0ull : ((1ull << (end - prev)) - 1))
                   << ") << " << prev << ")";
            src_bit += end - prev;
            prev = end + 1;
        }
        // chunk number bit i -> its hole position
        std::ostringstream cx;
        cx << "0ull";
        for (int i = 0; i < cb; ++i) {
            const int j = stage->cshift + i;
            cx << " | (((unsigned long long)c >> " << i << ") & 1ull) << " << rest[size_t(j <= stage->xrot ? j - 1 : j)];
        }
        s << "  if (blockIdx.x >= npass) {\n"
          << "    stage_push_role<16>(blockIdx.x - npass, gridDim.x - npass, xout_r, xpeer, pdone, xpeer_done, pdone + 256, "
             "pdone + 512, " << (1 << cb) << ", " << stage->slots << ", " << (1u << stage->cshift) << "u, slot_elems, "
          << kStageWatchdogNs << "ull,\n"
          << "      [=] (unsigned long long k, int c) -> unsigned long long { return " << ex.str() << " | "
          << cx.str() << "; });\n"
          << "    return;\n"
          << "  }\n";
    }
    s << ""
      << "  for (unsigned i = tid; i < " << h.pool_n << "u; i += " << T << "u) pool[i] = gpool[i];\n";
    // Per-layout thread constants (tile-bit pattern tb<k> and swizzled
    // offset sw<k>) are defined inside the tile loop where layout k becomes
    // active: short live ranges, so the 16 amplitudes keep the registers.
    // (tidv is tid made opaque to the optimiser once per tile, so these are
    // recomputed per tile -- a few integer ops -- instead of being hoisted out
    // of the loop, where 16 addresses per layout would spill to local memory)
    auto def_layout = [&](size_t k) {
        s << "    const unsigned tb" << k << " = " << deposit_expr("tidv", lays[k].nonr, false) << ";\n";
        s << "    const unsigned sw" << k << " = " << swz_expr("tb" + std::to_string(k), sw) << ";\n";
        s << "    (void)sw" << k << ";\n";
    };
    const Layout& L0 = lays.front();
    const Layout& LN = lays.back();
    {
        // direct streaming loads into the first register layout; one buffer
        s << "  __syncthreads();\n";
        if (staged)
            s << "  unsigned ck_cur = 0xffffffffu, ck_n = 0u;  // chunk of the tiles in flight, tiles stored in it\n";
        for (int k = 0; k < nep; ++k) s << "  double ep" << k << " = 0.0;  // fused <Z> term " << k << "\n";
        s << "  for (long long r = blockIdx.x; r < ntiles; r += " << (staged ? "npass" : "gridDim.x") << ") {\n";
        if (staged) {
            // entering a new chunk: publish the tiles stored in the previous
            // one (fenced), then wait until its staging slot is free again
            s << "    { const unsigned ck = (unsigned)((unsigned long long)r >> " << stage->cshift << ");\n"
              << "      if (ck != ck_cur) {\n"
              << "        if (ck_n) { __threadfence(); __syncthreads(); if (tid == 0) atomicAdd(pdone + ck_cur, ck_n); }\n"
              << "        ck_cur = ck; ck_n = 0u;\n"
              << "        if (ck >= " << stage->slots << "u) {\n"
              << "          if (tid == 0 && ld_acquire_u32(pdone + " << 2 * 256 << ") == 0u && !wait_at_least(qdone + ck - "
              << stage->slots << "u, " << stage->pushers << "u, " << kStageWatchdogNs
              << "ull)) atomicMax(pdone + " << 2 * 256 << ", 0x100u + ck);  // watchdog\n"
              << "          __syncthreads();\n"
              << "        }\n"
              << "      }\n"
              << "    }\n";
        }
        if (mirror) {
            // Hermitian pass: only canonical tiles (r <= mirror(r)) are read
            s << "    const long long rstar = (long long)(" << mirror_rest_expr("(unsigned long long)r") << ");\n"
              << "    if (rstar < r) continue;\n";
        }
        // exchange passes: tile counter bit 0 moves to rest position xrot, so
        // that consecutive CTAs alternate between tiles stored locally and
        // tiles stored to the partner (NVLink and HBM stores overlap)
        const std::string rexpr = xstore ? "rr" : "(unsigned long long)r";
        if (xstore)
            s << "    const unsigned long long r1 = (unsigned long long)r >> 1;\n"
              << "    const unsigned long long rr = ((r1 >> xrot) << (xrot + 1)) | (((unsigned long long)r & 1ull) << xrot)"
                 " | (r1 & ((1ull << xrot) - 1ull));\n";
        s << "    double2* cur = buf0;\n"
          << "    const unsigned long long base = " << deposit_expr(rexpr, rest, true) << ";\n"
          << "    const unsigned long long full = rankbase | base;\n"
          << "    (void)full;\n"
          << "    double2 a[" << E << "];\n"
          << "    double2 ug = make_double2(1.0, 0.0);\n"
          << "    (void)ug;\n"
          << "    unsigned tidv = tid;\n"
          << "    asm volatile(\"\" : \"+r\"(tidv));\n";
        def_layout(0);
        s << "    { const double2* src = st + base + (" << state_off("tb0", L0.nonr, q) << ");\n";
        // a register slot on physical bit 0: its amplitude pairs are adjacent,
        // one 256-bit load each (full 32-byte sectors per lane)
        int j0 = -1;
        for (int j = 0; j < L0.r; ++j)
            if (q[size_t(L0.rp[j])] == 0) j0 = j;
        for (int l = 0; l < E; ++l) {
            if (j0 < 0) {
                s << "      a[" << l << "] = ld_stream(src + " << hex64(reg_off(L0, l, q)) << ");\n";
            } else if (!((l >> j0) & 1)) {
                s << "      ld_stream2(src + " << hex64(reg_off(L0, l, q)) << ", a[" << l << "], a[" << (l | (1 << j0))
                  << "]);\n";
            }
        }
        s << "    }\n";
    }
    // pending-permutation state (see px_enabled): dirty = register slots
    // whose px bit may be set at this point of the program
    const bool use_px = px_enabled() && !mirror;
    unsigned dirty = 0;
    if (use_px) s << "    unsigned px = 0u;\n";
    auto px_bit = [](int b) { return "((px >> " + std::to_string(b) + ") & 1u)"; };
    // tile bits the pending permutation's conditions depend on (px varies
    // across the threads that differ in them)
    unsigned px_ctl = 0;
    auto commit = [&](unsigned mask) {
        const unsigned m = dirty & mask;
        for (int b = 0; b < 4; ++b)
            if ((m >> b) & 1u) s << "    if (px & " << (1u << b) << "u) xperm<" << E << ", " << b << ">(a, 0u);\n";
        if (m) s << "    px &= ~" << m << "u;\n";
        dirty &= ~m;
    };
    // swizzled shared-memory offset of the pending permutation in layout A
    auto px_smem_xor = [&](const Layout& A) {
        std::ostringstream rc;
        rc << "0u";
        for (int b = 0; b < A.r; ++b)
            if ((dirty >> b) & 1u) rc << " | (" << px_bit(b) << " << " << A.rp[b] << ")";
        s << "    const unsigned rcx" << " = " << rc.str() << ";\n"
          << "    const unsigned kx = " << swz_expr("rcx", sw) << ";\n";
    };
    // state offset of the pending permutation at the store (layout A, positions pos)
    auto px_state_xor = [&](const Layout& A, const std::vector<int>& pos) {
        std::ostringstream o;
        o << "0ull";
        for (int b = 0; b < A.r; ++b)
            if ((dirty >> b) & 1u)
                o << " | ((unsigned long long)" << px_bit(b) << " << " << pos[size_t(A.rp[b])] << ")";
        return o.str();
    };
    // Diagonal phase accumulators (unit-modulus tables, e.g. every phase of a
    // state-vector circuit): a diagonal factor that depends on no register
    // slot is uniform over the thread's amplitudes (ug); one that depends on
    // register slot t only is ug-part x (a phase on the amplitudes whose slot
    // t bit is 1), accumulated per thread in ph<t>.  A table on two slots
    // t, u splits into those parts plus an interaction factor applied to the
    // 4 amplitudes with both bits set.  Diagonals commute with each other, so
    // the accumulated phases are applied only before an operator that does
    // not commute with them (a non-diagonal op on the slot, a relayout, the
    // store): one complex multiply per amplitude for all of them (Gray-code
    // walk over the 16 registers) instead of one per amplitude per table.
    bool ug_pending = false;
    bool ph_pending[4] = {false, false, false, false};
    auto ph_name = [](int t) { return "ph" + std::to_string(t); };
    // apply ph<t> to the registers with slot bit t set (no ug)
    auto flush_ph = [&](unsigned mask) {
        for (int t = 0; t < 4; ++t) {
            if (!((mask >> t) & 1u) || !ph_pending[t]) continue;
            for (int l = 0; l < E; ++l)
                if ((l >> t) & 1) s << "    a[" << l << "] = cmul(" << ph_name(t) << ", a[" << l << "]);\n";
            ph_pending[t] = false;
        }
    };
    // everything pending: ug and every ph<t>, one multiply per amplitude
    auto flush_ug = [&] {
        unsigned pm = 0;
        for (int t = 0; t < 4; ++t)
            if (ph_pending[t]) pm |= 1u << t;
        if (!ug_pending && !pm) return;
        if (!pm) {
            s << "    if (!is_one(ug)) {\n";
            for (int l = 0; l < E; ++l) s << "      a[" << l << "] = cmul(ug, a[" << l << "]);\n";
            s << "    }\n";
            ug_pending = false;
            return;
        }
        // Gray-code order over the pending slots: consecutive registers differ
        // in one pending bit, so the running factor takes one multiply (by
        // ph<t> or its conjugate = inverse) per step
        std::vector<int> pb;
        for (int t = 0; t < 4; ++t)
            if ((pm >> t) & 1u) pb.push_back(t);
        const int np = int(pb.size());
        s << "    { double2 pr = " << (ug_pending ? "ug" : "make_double2(1.0, 0.0)") << ";\n";
        unsigned prev = 0;
        for (int i = 0; i < (1 << np); ++i) {
            const unsigned gi = unsigned(i) ^ (unsigned(i) >> 1);
            unsigned sel = 0;  // register bits of the pending slots
            for (int j = 0; j < np; ++j)
                if ((gi >> j) & 1u) sel |= 1u << pb[size_t(j)];
            if (i > 0) {
                const unsigned ch = gi ^ prev;
                const int t = pb[size_t(__builtin_ctz(ch))];
                if (gi & ch) s << "      pr = cmul(pr, " << ph_name(t) << ");\n";
                else s << "      pr = cmul(pr, cconj(" << ph_name(t) << "));\n";
            }
            prev = gi;
            for (int l = 0; l < E; ++l)
                if ((unsigned(l) & pm) == sel) s << "      a[" << l << "] = cmul(pr, a[" << l << "]);\n";
        }
        s << "    }\n";
        ug_pending = false;
        for (int t = 0; t < 4; ++t) ph_pending[t] = false;
    };
    auto ph_mul = [&](int t, const std::string& f) {
        if (ph_pending[t]) s << "      " << ph_name(t) << " = cmul(" << ph_name(t) << ", " << f << ");\n";
        else s << "      " << ph_name(t) << " = " << f << ";\n";
        ph_pending[t] = true;
    };
    auto ug_mul = [&](const std::string& f) {
        if (ug_pending) s << "      ug = cmul(ug, " << f << ");\n";
        else s << "      ug = " << f << ";\n";
        ug_pending = true;
    };
    if (accumulate_phases()) s << "    double2 ph0, ph1, ph2, ph3;\n    (void)ph0; (void)ph1; (void)ph2; (void)ph3;\n";
    for (int i = 1; i < h.nops; ++i) {
        const MOp& op = ops[i];
        const int li = lay_of_op[size_t(i)];
        const Layout& L = lays[size_t(li)];
        const std::string tbn = "tb" + std::to_string(li);
        const std::string P = "pool + " + std::to_string(op.mat);
        switch (op.type) {
        case MOP_LAYOUT: {
            const Layout& A = lays[size_t(li - 1)];
            flush_ug();
            const char* bar1 = "__syncthreads()";
            const char* bar2 = "__syncthreads()";
            s << "    " << bar1 << ";\n";
            // A pending permutation that varies across the 8 lanes of a
            // quarter-warp (its conditions read the layout's 3 lowest thread
            // bits) scatters their 128-bit stores over colliding bank groups
            // when XOR-ed into the addresses (VQE-28: 69 M / 136 M store
            // conflicts in two passes, random-30 pass 2: 71 M).  Committing it
            // to the registers first (predicated swaps) removes them (1.3 M /
            // 4.2 M) but measured slower overall (VQE-28 13.10 -> 13.30 ms,
            // random-30 43.88 -> 44.05 ms): those passes are bound by their
            // relayout count and FP64 work, not by the conflicts.  A/B switch.
            static const bool commit_lanes = ab_knob("NQ_PX_COMMIT_LANES", 0) != 0;
            unsigned lanes8 = 0;
            for (size_t t = 0; t < A.nonr.size() && t < 3; ++t) lanes8 |= 1u << A.nonr[t];
            if (commit_lanes && use_px && dirty && (px_ctl & lanes8)) {
                commit(dirty);
                px_ctl = 0;
            }
            if (use_px && dirty) {
                s << "    {\n";
                px_smem_xor(A);
                for (int l = 0; l < E; ++l)
                    s << "    cur[sw" << (li - 1) << " ^ " << sw.apply(A.rconst(l)) << "u ^ kx] = a[" << l << "];\n";
                s << "    }\n    px = 0u;\n";
                dirty = 0;
                px_ctl = 0;
            } else {
                for (int l = 0; l < E; ++l)
                    s << "    cur[sw" << (li - 1) << " ^ " << sw.apply(A.rconst(l)) << "u] = a[" << l << "];\n";
            }
            s << "    " << bar2 << ";\n";
            def_layout(size_t(li));
            for (int l = 0; l < E; ++l)
                s << "    a[" << l << "] = cur[sw" << li << " ^ " << sw.apply(L.rconst(l)) << "u];\n";
            break;
        }
        case MOP_DENSE: {
            if (op.k == 1 && accumulate_phases() && ph_pending[op.pos[0]] &&
                !(use_px && ((dirty >> op.pos[0]) & 1u))) {
                // N with two exact 1s (planner.cpp: pivot-normalised unitary)
                // after a pending phase p on its slot: N diag(1, p) is folded
                // at run time instead of multiplying p into 8 amplitudes:
                //   [[1, a], [b, 1]] diag(1, p) = diag(1, p) [[1, a p], [b p*, 1]]
                //   [[a, 1], [1, b]] diag(1, p) = p diag(1, p*) [[a p*, 1], [1, b p]]
                const cplx* u = pool + op.mat;
                const bool nd = u[0] == cplx(1.0, 0.0) && u[3] == cplx(1.0, 0.0);
                const bool no = u[1] == cplx(1.0, 0.0) && u[2] == cplx(1.0, 0.0);
                if (nd || no) {
                    const int t = op.pos[0];
                    const std::string ph = ph_name(t);
                    s << "    {\n";
                    if (nd) {
                        s << "      const double2 na = cmul(lds(" << P << " + 1), " << ph << ");\n"
                          << "      const double2 nb = cmul(lds(" << P << " + 2), cconj(" << ph << "));\n";
                    } else {
                        s << "      const double2 na = cmul(lds(" << P << "), cconj(" << ph << "));\n"
                          << "      const double2 nb = cmul(lds(" << P << " + 3), " << ph << ");\n";
                        ug_mul(ph);
                        s << "      " << ph << " = cconj(" << ph << ");\n";
                    }
                    for (int l = 0; l < E; ++l) {
                        if ((l >> t) & 1) continue;
                        const int hi = l | (1 << t);
                        s << "      { const double2 x0 = a[" << l << "]; const double2 x1 = a[" << hi << "];\n";
                        if (nd)
                            s << "        a[" << l << "] = cfma(na, x1, x0); a[" << hi << "] = cfma(nb, x0, x1); }\n";
                        else
                            s << "        a[" << l << "] = cfma(na, x0, x1); a[" << hi << "] = cfma(nb, x1, x0); }\n";
                    }
                    s << "    }\n";
                    break;
                }
            }
            {
                unsigned sl = 0;
                for (int j = 0; j < op.k; ++j) sl |= 1u << op.pos[j];
                flush_ph(sl);
            }
            bool real = true, special = false;
            size_t generic = 0;  // entries that are neither zero, real nor pure imaginary
            const size_t nent = size_t(1) << (2 * op.k);
            for (size_t i = 0; i < nent; ++i) {
                const cplx v = pool[op.mat + i];
                real = real && v.imag() == 0.0;
                generic += v.real() != 0.0 && v.imag() != 0.0;
                special = special || v == cplx(0.0, 0.0) || v == cplx(1.0, 0.0) || v == cplx(-1.0, 0.0);
            }
            const char* R = real ? ", true" : "";
            unsigned slots = 0;
            for (int j = 0; j < op.k; ++j) slots |= 1u << op.pos[j];
            const bool sparse = op.k <= 2 && (special || (!real && generic < nent));
            if (use_px && (dirty & slots)) {
                if (op.k == 1 && !sparse) {
                    s << "    d1f<" << E << ", " << int(op.pos[0]) << R << ">(a, " << P << ", " << px_bit(op.pos[0])
                      << " * 3u);\n";
                    break;
                }
                if (op.k == 2 && !sparse) {
                    s << "    d2f<" << E << ", " << int(op.pos[0]) << ", " << int(op.pos[1]) << R << ">(a, " << P << ", ("
                      << px_bit(op.pos[0]) << " | (" << px_bit(op.pos[1]) << " << 1)) * 5u);\n";
                    break;
                }
                commit(slots);
            }
            if (sparse) {
                s << sparse_dense(op, pool + op.mat, E, P);
            } else if (op.k == 1) {
                s << "    d1<" << E << ", " << int(op.pos[0]) << R << ">(a, " << P << ");\n";
            } else if (op.k == 2) {
                s << "    d2<" << E << ", " << int(op.pos[0]) << ", " << int(op.pos[1]) << R << ">(a, " << P << ");\n";
            } else if (op.k == 3) {
                s << "    d3<" << E << ", " << (6 - op.pos[0] - op.pos[1] - op.pos[2]) << R << ">(a, " << P << ");\n";
            } else {
                s << "    __syncthreads();\n    d4<16" << R << ">(a, " << P << ", cur + tid * 16u);\n";
            }
            break;
        }
        case MOP_SWAP: {
            const int j0 = op.pos[0], j1 = op.pos[1];
            if (ph_pending[j0] || ph_pending[j1]) {
                // the registers trade places: so do their pending phases
                if (ph_pending[j0] && ph_pending[j1])
                    s << "    { const double2 t_ = " << ph_name(j0) << "; " << ph_name(j0) << " = " << ph_name(j1) << "; "
                      << ph_name(j1) << " = t_; }\n";
                else if (ph_pending[j0])
                    s << "    " << ph_name(j1) << " = " << ph_name(j0) << ";\n";
                else
                    s << "    " << ph_name(j0) << " = " << ph_name(j1) << ";\n";
                std::swap(ph_pending[j0], ph_pending[j1]);
            }
            if (use_px && (dirty & ((1u << j0) | (1u << j1)))) {
                // SWAP(j0, j1) . X^px = X^swap(px) . SWAP(j0, j1)
                s << "    px = (px & ~" << ((1u << j0) | (1u << j1)) << "u) | (" << px_bit(j0) << " << " << j1 << ") | ("
                  << px_bit(j1) << " << " << j0 << ");\n";
                const unsigned d0 = (dirty >> j0) & 1u, d1 = (dirty >> j1) & 1u;
                dirty = (dirty & ~((1u << j0) | (1u << j1))) | (d0 << j1) | (d1 << j0);
            }
            s << "    swp<" << E << ", " << j0 << ", " << j1 << ">(a);\n";
            break;
        }
        case MOP_DEPOL:
            flush_ph(0xFu);
            if (use_px) commit(0xFu);
            if (op.k == 2) {
                const int a0 = std::min(op.pos[0], op.pos[1]), a1 = std::max(op.pos[0], op.pos[1]);
                s << "    dep2<" << E << ", " << a0 << ", " << a1 << ">(a, lds(" << P << ").x, lds(" << P << " + 1).x);\n";
            } else {
                const int p0 = op.pos[0] == 0   ? op.pos[2]
                               : op.pos[2] == 0 ? op.pos[0]
                               : op.pos[1] == 0 ? op.pos[3]
                                                : op.pos[1];
                s << "    dep4<16, " << p0 << ">(a, lds(" << P << ").x, lds(" << P << " + 1).x);\n";
            }
            break;
        case MOP_XPERM: {
            flush_ph(1u << op.pos[0]);
            unsigned cmL = 0, cmT = 0;
            for (int p = 0; p < m; ++p) {
                if (!((op.cmask_tile >> p) & 1u)) continue;
                int slot = -1;
                for (int j = 0; j < L.r; ++j)
                    if (L.rp[j] == p) slot = j;
                if (slot >= 0) cmL |= 1u << slot;
                else cmT |= 1u << p;
            }
            const std::string cond = "((full & " + hex64(op.cmask_glob) + ") == " + hex64(op.cmask_glob) + ") && ((" +
                                     tbn + " & " + std::to_string(cmT) + "u) == " + std::to_string(cmT) + "u)";
            if (use_px && cmL == 0 && (op.cmask_glob != 0 || cmT != 0)) {
                // controls outside the registers: record the X, move nothing
                s << "    px ^= (" << cond << " ? 1u : 0u) << " << int(op.pos[0]) << ";\n";
                dirty |= 1u << op.pos[0];
                px_ctl |= cmT;
                break;
            }
            const bool trivial = op.cmask_glob == 0 && cmT == 0;
            if (use_px && trivial && __builtin_popcount(cmL) == 1 && (dirty & cmL)) {
                // CX with its register control c pending: on the registers it is
                // the plain CX when px_c = 0, and the CX followed by an X on the
                // target when px_c = 1 -- which is recorded, not moved
                const int c = __builtin_ctz(cmL);
                s << "    xperm<" << E << ", " << int(op.pos[0]) << ">(a, " << cmL << "u);\n"
                  << "    px ^= " << px_bit(c) << " << " << int(op.pos[0]) << ";\n";
                dirty |= 1u << op.pos[0];
                break;
            }
            if (use_px) commit(cmL);
            s << "    if (" << cond << ") xperm<" << E << ", " << int(op.pos[0]) << ">(a, " << cmL << "u);\n";
            break;
        }
        case MOP_DIAG: {
            std::ostringstream g;
            g << "0u";
            unsigned slotc[4] = {0, 0, 0, 0};
            bool anyreg = false;
            for (int j = 0; j < op.k; ++j) {
                const int p = op.pos[j];
                if (p < 0) {
                    g << " | ((unsigned)((full >> " << (-1 - p) << ") & 1ull) << " << j << ")";
                    continue;
                }
                int slot = -1;
                for (int t = 0; t < L.r; ++t)
                    if (L.rp[t] == p) slot = t;
                if (slot >= 0) {
                    slotc[slot] |= 1u << j;
                    anyreg = true;
                } else {
                    g << " | (((" << tbn << " >> " << p << ") & 1u) << " << j << ")";
                }
            }
            const cplx* tab = pool + op.mat;
            s << "    { const unsigned g = " << g.str() << "; const double2* D = " << P << " + g;\n";
            unsigned dslots = 0;
            for (int t = 0; t < 4; ++t)
                if (slotc[t]) dslots |= 1u << t;
            const int nds = __builtin_popcount(dslots);
            bool unit = true;
            for (int gi = 0; gi < (1 << op.k) && unit; ++gi) unit = std::abs(std::norm(tab[gi]) - 1.0) < 1e-14;
            if (accumulate_phases() && unit && nds >= 1 && nds <= 2 && !(use_px && (dirty & dslots))) {
                const unsigned regmask = slotc[0] | slotc[1] | slotc[2] | slotc[3];
                // table entries with none of the register bits set: exactly 1 for every g?
                bool one0 = true;
                for (int gi = 0; gi < (1 << op.k) && one0; ++gi)
                    if ((unsigned(gi) & regmask) == 0u) one0 = tab[gi] == cplx(1.0, 0.0);
                std::vector<int> ts;
                for (int t = 0; t < 4; ++t)
                    if ((dslots >> t) & 1u) ts.push_back(t);
                if (!one0) {
                    s << "      const double2 f00 = lds(D);\n      const double2 c00 = cconj(f00);\n";
                    ug_mul("f00");
                }
                for (int t : ts) {
                    s << "      const double2 fs" << t << " = lds(D + " << slotc[t] << "u);\n";
                    ph_mul(t, one0 ? "fs" + std::to_string(t) : "cmul(fs" + std::to_string(t) + ", c00)");
                }
                if (nds == 2) {
                    // interaction part on the registers with both slot bits set
                    const int t = ts[0], u = ts[1];
                    s << "      double2 fr = cmul(lds(D + " << (slotc[t] | slotc[u]) << "u), cconj(cmul(fs" << t << ", fs" << u
                      << ")));\n";
                    if (!one0) s << "      fr = cmul(fr, f00);\n";
                    for (int l = 0; l < E; ++l)
                        if (((l >> t) & 1) && ((l >> u) & 1)) s << "      a[" << l << "] = cmul(fr, a[" << l << "]);\n";
                }
                s << "    }\n";
                break;
            }
            if (anyreg && use_px && (dirty & dslots)) {
                // table entries selected through the pending permutation
                std::ostringstream gx;
                gx << "0u";
                for (int t = 0; t < 4; ++t)
                    if (((dirty & dslots) >> t) & 1u) gx << " | (" << px_bit(t) << " * " << slotc[t] << "u)";
                s << "      const unsigned gx = " << gx.str() << ";\n";
                // each distinct entry loaded right before the amplitudes it
                // multiplies: one factor live at a time (preloading all 16
                // next to the 16 amplitudes spilled registers)
                std::map<unsigned, std::vector<int>> users;
                for (int l = 0; l < E; ++l) {
                    unsigned c = 0;
                    for (int t = 0; t < 4; ++t)
                        if ((l >> t) & 1) c |= slotc[t];
                    users[c].push_back(l);
                }
                for (const auto& [c, ls] : users) {
                    s << "      { const double2 f = lds(D + (" << c << "u ^ gx));\n";
                    for (int l : ls) s << "        a[" << l << "] = cmul(f, a[" << l << "]);\n";
                    s << "      }\n";
                }
                s << "    }\n";
                break;
            }
            if (!anyreg) {
                // a factor uniform over the thread's amplitudes: accumulate it and
                // apply the product once (scalars commute with every in-thread op)
                if (ug_pending) s << "      ug = cmul(ug, lds(D)); }\n";
                else s << "      ug = lds(D); }\n";
                ug_pending = true;
            } else {
                const unsigned regmask = slotc[0] | slotc[1] | slotc[2] | slotc[3];
                // one shared-memory load per distinct table entry, right before
                // the complex multiplies of the amplitudes it scales (exact ones
                // skipped at compile time); one factor live at a time
                std::map<unsigned, std::vector<int>> users;
                for (int l = 0; l < E; ++l) {
                    unsigned c = 0;
                    for (int t = 0; t < 4; ++t)
                        if ((l >> t) & 1) c |= slotc[t];
                    bool all_one = true;
                    for (int gi = 0; gi < (1 << op.k) && all_one; ++gi) {
                        if ((unsigned(gi) & regmask) != c) continue;
                        all_one = tab[gi] == cplx(1.0, 0.0);
                    }
                    if (!all_one) users[c].push_back(l);
                }
                for (const auto& [c, ls] : users) {
                    s << "      { const double2 f = lds(D + " << c << "u);\n";
                    // factors that depend on thread / tile bits are often exactly
                    // 1 for a whole warp: optionally tested once per factor
                    if (diag_runtime_skip()) s << "        if (!is_one(f)) {\n";
                    for (int l : ls) s << "        a[" << l << "] = cmul(f, a[" << l << "]);\n";
                    if (diag_runtime_skip()) s << "        }\n";
                    s << "      }\n";
                }
                s << "    }\n";
            }
            break;
        }
        default:
            break;
        }
    }
    flush_ug();
    if (extra_relayout) {
        // (the barrier also orders every load of the tile before any store:
        // relabelled stores hit addresses other threads load)
        const std::string swN = "sw" + std::to_string(lays.size() - 1);
        s << "    __syncthreads();\n";
        if (use_px && dirty) {
            s << "    {\n";
            px_smem_xor(LN);
            for (int l = 0; l < E; ++l)
                s << "    cur[" << swN << " ^ " << sw.apply(LN.rconst(l)) << "u ^ kx] = a[" << l << "];\n";
            s << "    }\n    px = 0u;\n";
            dirty = 0;
        } else {
            for (int l = 0; l < E; ++l)
                s << "    cur[" << swN << " ^ " << sw.apply(LN.rconst(l)) << "u] = a[" << l << "];\n";
        }
        s << "    __syncthreads();\n";
        s << "    const unsigned tbS = " << deposit_expr("tidv", LS.nonr, false) << ";\n";
        s << "    const unsigned swS = " << swz_expr("tbS", sw) << ";\n";
        for (int l = 0; l < E; ++l) s << "    a[" << l << "] = cur[swS ^ " << sw.apply(LS.rconst(l)) << "u];\n";
    }
    const Layout& LST = extra_relayout ? LS : LN;
    // pending permutation: register l holds the amplitude of index l ^ px
    const std::string pxo = (use_px && dirty) ? " ^ pxo" : "";
    if (use_px && dirty) s << "    const unsigned long long pxo = " << px_state_xor(LST, qst) << ";\n";
    {
        const std::string tbl = extra_relayout ? "tbS" : "tb" + std::to_string(lays.size() - 1);
        s << "    const unsigned long long toff_st = " << state_off(tbl, LST.nonr, qst) << ";\n";
        if (mirror) s << "    const unsigned long long toff_mir = " << state_off(tbl, LN.nonr, qmir) << ";\n";
    }
    if (staged) {
        // staged exchange store: kept elements in place, outgoing ones into
        // the staging slot at their compressed physical index
        std::vector<int> qc(qst.size());
        for (size_t i = 0; i < qst.size(); ++i) qc[i] = cpos(qst[i]);
        std::ostringstream sb;
        sb << "0ull";
        for (size_t j = 0; j < rest.size(); ++j)
            if (cpos(rest[j]) >= 0) sb << " | (((rr >> " << j << ") & 1ull) << " << cpos(rest[j]) << ")";
        std::ostringstream tc;
        tc << "0ull";
        for (int b : LST.nonr)
            if (qc[size_t(b)] >= 0) tc << " | ((unsigned long long)((" << (extra_relayout ? "tbS" : "tb" + std::to_string(lays.size() - 1))
                                       << " >> " << b << ") & 1u) << " << qc[size_t(b)] << ")";
        std::ostringstream pc;
        pc << "0ull";
        for (int b = 0; b < LST.r && use_px && dirty; ++b)
            if (((dirty >> b) & 1u) && qc[size_t(LST.rp[b])] >= 0)
                pc << " | ((unsigned long long)" << px_bit(b) << " << " << qc[size_t(LST.rp[b])] << ")";
        auto creg = [&](int l) {
            unsigned long long c = 0;
            for (int j = 0; j < LST.r; ++j)
                if (((l >> j) & 1) && qc[size_t(LST.rp[j])] >= 0) c |= 1ull << qc[size_t(LST.rp[j])];
            return c;
        };
        s << "    { const unsigned long long ob = base + toff_st;\n"
          << "      double2* const sg = xout_r + (unsigned long long)(ck_cur % " << stage->slots << "u) * slot_elems + ("
          << sb.str() << ") + (" << tc.str() << ");\n";
        if (use_px && dirty) s << "      const unsigned long long pxc = " << pc.str() << ";\n";
        for (int l = 0; l < E; ++l)
            s << "      { const unsigned long long o = ob + (" << hex64(reg_off(LST, l, qst)) << pxo << ")"
              << "; st_stream(((o ^ xval) & xmask) ? sg + (" << hex64(creg(l)) << (use_px && dirty ? " ^ pxc" : "")
              << ") : st + o, a[" << l << "]); }\n";
        s << "    }\n";
    } else if (xstore) {
        // exchange store (sharded states): element o whose bit v (xmask)
        // differs from this rank's bit (xval) goes to the partner's buffer at
        // o ^ xmask, the rest to the local output buffer (out of place)
        s << "    { const unsigned long long ob = base + toff_st;\n";
        for (int l = 0; l < E; ++l)
            s << "      { const unsigned long long o = ob + (" << hex64(reg_off(LST, l, qst)) << pxo << ")"
              << "; st_stream(((o ^ xval) & xmask) ? xout_r + (o ^ xmask) : xout_l + o, a[" << l << "]); }\n";
        s << "    }\n";
    } else {
        // register slot stored to physical bit 0 (and not pending in px):
        // adjacent pairs, one 256-bit store each
        int j0 = -1;
        for (int j = 0; j < LST.r; ++j)
            if (qst[size_t(LST.rp[j])] == 0 && !(use_px && ((dirty >> j) & 1u))) j0 = j;
        s << "    { double2* dst = st + base + toff_st;\n";
        for (int l = 0; l < E; ++l) {
            if (j0 < 0)
                s << "      st_stream(dst + (" << hex64(reg_off(LST, l, qst)) << pxo << "), a[" << l << "]);\n";
            else if (!((l >> j0) & 1))
                s << "      st_stream2(dst + (" << hex64(reg_off(LST, l, qst)) << pxo << "), a[" << l << "], a["
                  << (l | (1 << j0)) << "]);\n";
        }
        s << "    }\n";
        if (nep) {
            // fused Z-type terms: the sign of amplitude l is the parity of its
            // store index under the term's mask = a per-thread part (tile and
            // rest bits, pending permutation) x a compile-time part (register l)
            s << "    { const unsigned long long oe = (base + toff_st)" << (use_px && dirty ? " ^ pxo" : "") << ";\n";
            for (int l = 0; l < E; ++l)
                s << "      const double p" << l << " = fma(a[" << l << "].x, a[" << l << "].x, a[" << l << "].y * a[" << l
                  << "].y);\n";
            for (int k = 0; k < nep; ++k) {
                const uint64_t M = epi->signs[k];
                std::ostringstream pos, neg;
                pos << "0.0";
                neg << "0.0";
                for (int l = 0; l < E; ++l)
                    ((__builtin_popcountll(reg_off(LST, l, qst) & M) & 1) ? neg : pos) << " + p" << l;
                s << "      { const double d = (" << pos.str() << ") - (" << neg.str() << ");\n"
                  << "        ep" << k << " += (__popcll(oe & " << hex64(M) << ") & 1) ? -d : d; }\n";
            }
            s << "    }\n";
        }
    }
    if (mirror) {
        // the mirror tile holds the conjugate transpose: element e of tile r is
        // conj'd into element e* (column/row bits swapped) of tile mirror(r)
        s << "    if (rstar != r) {\n"
          << "      double2* dst = st + (" << deposit_expr("(unsigned long long)rstar", rest, true) << ") + toff_mir;\n";
        for (int l = 0; l < E; ++l)
            s << "      st_stream(dst + " << hex64(reg_off(LST, l, qmir)) << ", make_double2(a[" << l << "].x, -a[" << l
              << "].y));\n";
        s << "    }\n";
    }
    s << ""
      << "    __syncthreads();\n";
    if (staged) s << "    ++ck_n;\n";
    s << "  }\n";
    if (staged) s << "  if (ck_n) { __threadfence(); __syncthreads(); if (tid == 0) atomicAdd(pdone + ck_cur, ck_n); }\n";
    if (nep) {
        // fixed-order CTA reduction of the fused terms: warp shuffles, then
        // warp 0 sums the warps' values in order (buf0 is free after the loop)
        // (a CTA narrower than a warp -- small tiles -- is one partial warp)
        const int WL = std::min(32, T), NW = std::max(1, T / 32);
        const std::string wmask = T >= 32 ? "0xffffffffu" : std::to_string((1u << T) - 1u) + "u";
        s << "  {\n"
          << "    double* red = reinterpret_cast<double*>(buf0);\n";
        for (int k = 0; k < nep; ++k)
            s << "    for (int o = " << WL / 2 << "; o > 0; o >>= 1) ep" << k << " += __shfl_down_sync(" << wmask << ", ep"
              << k << ", o);\n"
              << "    if ((tid & " << (WL - 1) << "u) == 0u) red[" << k << " * " << NW << " + tid / " << WL << "u] = ep" << k
              << ";\n";
        s << "    __syncthreads();\n"
          << "    if (tid < " << nep << "u) {\n"
          << "      double t = 0.0;\n"
          << "      for (int w = 0; w < " << NW << "; ++w) t += red[tid * " << NW << " + w];\n"
          << "      epart[(unsigned long long)blockIdx.x * " << kMaxExpTerms << " + tid] = t;\n"
          << "    }\n"
          << "  }\n";
    }
    s << "}\n";
    return s.str();
}

namespace {

// options of every pass / expectation compile (4th: 128-bit pairs when the
// bound NVRTC predates 256-bit global accesses on sm_100a)
const char* const* nvrtc_opts(int* n) {
    static const char* wide[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo"};
    static const char* narrow[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DNQ_NO_V4"};
    const bool w = nvrtc().wide;
    *n = w ? 3 : 4;
    return w ? wide : narrow;
}

bool compile_entry(const std::string& src, Entry& e, int device) {
    if (const char* dir = std::getenv("NQ_JIT_DUMP")) {  // debugging: keep every generated source
        static std::atomic<int> seq{0};
        const std::string path = std::string(dir) + "/nqjit_" + std::to_string(seq.fetch_add(1)) + ".cu";
        if (FILE* f = std::fopen(path.c_str(), "w")) {
            std::fwrite(src.data(), 1, src.size(), f);
            std::fclose(f);
        }
    }
    nvrtcProgram prog;
    const char* hdrs[1] = {kPassOpsSrc};
    const char* names[1] = {"pass_ops.cuh"};
    if (nvrtcCreateProgram(&prog, src.c_str(), "nqjit.cu", 1, hdrs, names) != NVRTC_SUCCESS) {
        e.log = "nvrtcCreateProgram failed";
        return false;
    }
    int nopt_ = 0;
    const char* const* opts_ = nvrtc_opts(&nopt_);
    const nvrtcResult rc = nvrtcCompileProgram(prog, nopt_, opts_);
    size_t logn = 0;
    nvrtcGetProgramLogSize(prog, &logn);
    if (logn > 1) {
        e.log.resize(logn);
        nvrtcGetProgramLog(prog, &e.log[0]);
    }
    if (rc != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return false;
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    std::vector<char> cubin(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    cudaSetDevice(device);
    if (cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
        e.log += " cudaLibraryLoadData failed";
        cudaGetLastError();
        return false;
    }
    // pass kernels are `nqjit`, expectation batches `nqexp`
    const char* name = src.find(" nqexp(") != std::string::npos ? "nqexp" : "nqjit";
    if (cudaLibraryGetKernel(&e.kern, e.lib, name) != cudaSuccess) {
        e.log += " cudaLibraryGetKernel failed";
        cudaGetLastError();
        return false;
    }
    return true;
}

void worker_loop() {
    Jit& J = jit();
    for (;;) {
        std::pair<std::string, std::shared_ptr<Entry>> job;
        {
            std::unique_lock<std::mutex> lk(J.mu);
            J.cv.wait(lk, [&] { return !J.queue.empty() && !J.exiting; });
            job = std::move(J.queue.front());
            J.queue.pop_front();
            ++J.busy;
        }
        const bool ok = compile_entry(job.first, *job.second, J.device);
        job.second->state.store(ok ? 1 : 2);
        {
            std::lock_guard<std::mutex> lk(J.mu);
            --J.busy;
            if (ok) ++J.stats.compiled;
            else ++J.stats.failed;
        }
        J.cv.notify_all();
    }
}

}  // namespace

namespace {
// NQ_SEGV_TRACE=1: print a native backtrace on SIGSEGV (debugging aid).
void segv_handler(int sig) {
    void* frames[64];
    const int n = backtrace(frames, 64);
    const char msg[] = "\n[naqs_b200] fatal signal, native backtrace:\n";
    (void)!write(2, msg, sizeof msg - 1);
    backtrace_symbols_fd(frames, n, 2);
    std::signal(sig, SIG_DFL);
    std::raise(sig);
}
const bool g_segv_trace = [] {
    const char* e = std::getenv("NQ_SEGV_TRACE");
    if (e && e[0] == '1') std::signal(SIGSEGV, segv_handler);
    return true;
}();
}  // namespace

JitMode jit_mode() {
    static const JitMode m = mode_from_env();
    return m;
}

namespace {

// Process exit with compilations in flight: drop the queued ones and wait for
// the running ones, so no worker touches NVRTC / the CUDA runtime while they
// are being torn down.
void drain_at_exit() { jit_shutdown(); }

// NVRTC initialises internal state (with exit-time destructors) on its first
// compile.  One tiny compile before the exit hook is registered puts that
// teardown after the hook, so the hook always runs while NVRTC is intact.
void nvrtc_warm() {
    nvrtcProgram prog;
    const char* src = "extern \"C\" __global__ void nqwarm() {}";
    if (nvrtcCreateProgram(&prog, src, "warm.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return;
    int nopt_ = 0;
    const char* const* opts_ = nvrtc_opts(&nopt_);
    nvrtcCompileProgram(prog, nopt_, opts_);
    nvrtcDestroyProgram(&prog);
}

}  // namespace

void jit_shutdown() {
    Jit& J = jit();
    std::unique_lock<std::mutex> lk(J.mu);
    J.exiting = true;
    for (auto& job : J.queue) job.second->state.store(2);
    J.queue.clear();
    J.cv.wait(lk, [&] { return J.busy == 0; });
}

namespace {

// The compiled entry for `src` when it is ready; otherwise nullptr after
// queueing its compilation (auto) or compiling it inline (sync).
std::shared_ptr<Entry> acquire(const std::string& src, int device, JitMode mode) {
    Jit& J = jit();
    std::shared_ptr<Entry> e;
    {
        std::unique_lock<std::mutex> lk(J.mu);
        auto it = J.cache.find(src);
        if (it == J.cache.end()) {
            e = std::make_shared<Entry>();
            J.cache.emplace(src, e);
            if (mode == JitMode::Sync) {
                lk.unlock();
                const bool ok = compile_entry(src, *e, device);
                e->state.store(ok ? 1 : 2);
                lk.lock();
                if (ok) ++J.stats.compiled;
                else ++J.stats.failed;
                J.cv.notify_all();  // other threads waiting on this entry
            } else {
                if (J.exiting) return nullptr;
                J.device = device;
                if (!J.started) {
                    nvrtc_warm();
                    // NVRTC compiles are independent: a small pool of workers
                    const unsigned hw = std::thread::hardware_concurrency();
                    const unsigned nw = std::max(1u, std::min(8u, hw / 2));
                    for (unsigned w = 0; w < nw; ++w) std::thread(worker_loop).detach();
                    J.started = true;
                    std::atexit(drain_at_exit);
                }
                J.queue.emplace_back(src, e);
                J.cv.notify_all();
                ++J.stats.misses;
                return nullptr;
            }
        } else {
            e = it->second;
        }
    }
    if (mode == JitMode::Sync) {
        // queued or compiling in the background: wait for the worker
        std::unique_lock<std::mutex> lk(J.mu);
        J.cv.wait(lk, [&] { return e->state.load() != 0 || J.exiting; });
    }
    if (e->state.load() != 1) {
        ++J.stats.misses;
        return nullptr;
    }
    return e;
}

int occupancy(Entry& e, int device, int threads, size_t smem) {
    Jit& J = jit();
    std::lock_guard<std::mutex> lk(J.mu);
    auto it = e.occ.find(device);
    if (it != e.occ.end()) return it->second;
    cudaFuncSetAttribute(reinterpret_cast<const void*>(e.kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(e.kern), threads, smem);
    if (occ < 1) occ = 1;
    e.occ[device] = occ;
    return occ;
}

}  // namespace

bool jit_xstore_ok(const PassHdr& h, const MOp* ops) {
    if (jit_mode() == JitMode::Off || h.m < 8 || h.m > 12 || h.nops < 1) return false;
    if (h.flags & PASS_MIRROR) return false;
    (void)ops;
    return true;
}

int jit_xstore_prepare(const PassHdr& h, const MOp* ops, const cplx* pool, int device, const JitXStore* xs) {
    if (!jit_xstore_ok(h, ops)) throw NqError{NQ_ERR_INTERNAL, "exchange pass cannot be specialised"};
    std::shared_ptr<Entry> e = acquire(jit_source(h, ops, pool, true, xs), device, JitMode::Sync);
    if (!e) throw NqError{NQ_ERR_INTERNAL, "exchange pass kernel failed to compile"};
    // load it into this device's context now: with lazy loading, a first
    // launch next to a kernel that spins on it (the staged pusher) could wait
    // for that kernel to finish -- a deadlock
    cudaFuncAttributes fa;
    cudaSetDevice(device);
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(e->kern));
    cudaGetLastError();
    const int T = (1 << h.m) / (1 << ops[0].k);
    const size_t smem = (size_t(1) << h.m) * 16 + size_t(h.pool_n) * 16;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return sms * occupancy(*e, device, T, smem);
}

bool jit_launch(double2* state, const unsigned char* dev_rec, const PassHdr& h, const MOp* ops, const cplx* pool,
                uint64_t rankbase, cudaStream_t s, int device, const JitXStore* xs, JitMemo* memo, JitEpilogue* epi) {
    if (epi && (xs || (h.flags & PASS_MIRROR) || epi->nterms < 1)) epi = nullptr;
    const JitMode mode = jit_mode();
    std::shared_ptr<Entry> e;
    if (memo && !xs && !epi) {
        std::lock_guard<std::mutex> lk(memo->mu);
        e = std::static_pointer_cast<Entry>(memo->entry);
    }
    if (e) {
        // remembered for this pass record (owning reference)
    } else if (xs) {
        if (!jit_xstore_ok(h, ops)) throw NqError{NQ_ERR_INTERNAL, "exchange pass cannot be specialised"};
        const std::string src = jit_source(h, ops, pool, true, xs);
        e = acquire(src, device, JitMode::Sync);
        if (!e) {
            std::string log;
            {
                Jit& J = jit();
                std::lock_guard<std::mutex> lk(J.mu);
                auto it = J.cache.find(src);
                if (it != J.cache.end()) log = it->second->log;
            }
            if (log.size() > 1500) log = log.substr(log.size() - 1500);
            throw NqError{NQ_ERR_INTERNAL, "exchange pass kernel failed to compile: " + log};
        }
    } else {
        if (mode == JitMode::Off || h.m < 8 || h.m > 12) return false;
        if (mode == JitMode::Auto && h.nloc < 18) return false;  // interpreter is fine for small states
        e = acquire(jit_source(h, ops, pool, false, nullptr, epi), device, mode);
        if (e && memo && !epi && e->state.load() == 1) {
            std::lock_guard<std::mutex> lk(memo->mu);
            memo->entry = e;
        }
    }
    if (!e) return false;
    Jit& J = jit();
    const int T = (1 << h.m) / (1 << ops[0].k);
    const size_t smem = (size_t(1) << h.m) * 16 + size_t(h.pool_n) * 16;
    const int occ = occupancy(*e, device, T, smem);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // a staged exchange: the last `pushers` CTAs of a co-resident
    // (cooperative) grid are the pusher, the others the pass
    const bool staged = xs && xs->staged;
    const long long pushers = staged ? xs->pushers : 0;
    const long long grid =
        std::min<long long>(h.ntiles, std::max<long long>(1, (long long)sms * occ - pushers)) + pushers;
    unsigned npass = unsigned(grid - pushers);
    double2* xpeer = staged ? xs->peer : nullptr;
    const unsigned* xpeer_done = staged ? xs->peer_done : nullptr;
    const double2* gpool = reinterpret_cast<const double2*>(dev_rec + h.pool_off);
    unsigned long long rb = rankbase;
    long long nt = h.ntiles;
    double2* xl = xs ? xs->out_local : nullptr;
    double2* xr = xs ? xs->out_remote : nullptr;
    unsigned long long xm = xs ? xs->xmask : 0ull, xv = xs ? xs->xval : 0ull;
    int xrot = xs ? xs->xrot : 0;
    unsigned* pdone = xs ? xs->pass_done : nullptr;
    const unsigned* qdone = xs ? xs->push_done : nullptr;
    unsigned long long slot_elems = xs ? xs->slot_elems : 0ull;
    double* epart = epi ? epi->part : nullptr;
    void* args_ep[] = {&state, &gpool, &rb, &nt, &xl, &xr, &xm, &xv, &xrot, &epart};
    void* args_x[] = {&state, &gpool, &rb, &nt, &xl, &xr, &xm, &xv, &xrot, &pdone, &qdone, &slot_elems, &xpeer,
                      &xpeer_done, &npass};
    void** args = epi ? args_ep : args_x;
    if (epi) epi->grid = int(grid);
    const cudaError_t lrc =
        staged ? cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(e->kern), dim3(unsigned(grid)),
                                             dim3(unsigned(T)), args, smem, s)
               : cudaLaunchKernel(reinterpret_cast<const void*>(e->kern), dim3(unsigned(grid)), dim3(unsigned(T)), args,
                                  smem, s);
    if (lrc != cudaSuccess) {
        cudaGetLastError();
        if (xs) throw NqError{NQ_ERR_CUDA, "exchange pass kernel launch failed"};
        return false;
    }
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    ++J.stats.launches;
    return true;
}

// ---------------------------------------------------------------------------
// Expectation batches (K10, proj/src/statevector.cpp:241-277): one read of
// the state evaluates up to 32 Pauli terms whose flip masks lie in the tile.
//
// Each thread owns 8 amplitudes of the staged tile at a time, in up to four
// register layouts of 3 tile bits.  Terms are assigned to layouts so that
// every flip (X/Y) bit of a term is a register bit: its pair products
// conj(a[y^F]) a[y] are then formed in registers with compile-time signs, and
// the thread-dependent part of the sign is one runtime bit per term.  Z-type
// terms use layout 0: a 3-bit Walsh transform of |a|^2 gives every sign
// pattern over the register bits at once.  Terms that do not fit (more than
// 3 flip bits, or more than four layouts needed) loop over pairs in shared
// memory.  The tile is double-buffered with cp.async; addresses use the
// linear swizzle that makes the natural order and all layouts conflict free.
// ---------------------------------------------------------------------------
namespace {

constexpr int kExpGrid = 296;  // fixed: the summation order never depends on the device

struct ExpPlan {
    std::vector<Layout> lays;
    std::vector<int> lay_of;  // per term: layout or -1 (shared-memory pairs)
};

ExpPlan plan_expect(const ExpBatch& b) {
    const int m = b.m;
    ExpPlan P;
    P.lay_of.assign(size_t(b.nt), -1);
    std::vector<unsigned> bits;
    std::vector<int> order;
    for (int t = 0; t < b.nt; ++t) order.push_back(t);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return __builtin_popcount(b.t[x].ftile) > __builtin_popcount(b.t[y].ftile);
    });
    for (int t : order) {
        const unsigned f = b.t[t].ftile;
        if (f == 0 || __builtin_popcount(f) > 3) continue;
        size_t l = 0;
        for (; l < bits.size(); ++l)
            if (__builtin_popcount(bits[l] | f) <= 3) break;
        if (l == bits.size()) {
            if (bits.size() == 4) continue;
            bits.push_back(0);
        }
        bits[l] |= f;
        P.lay_of[size_t(t)] = int(l);
    }
    if (bits.empty()) bits.push_back(0);
    for (int t = 0; t < b.nt; ++t)
        if (b.t[t].ftile == 0) P.lay_of[size_t(t)] = 0;
    for (auto& r : bits)
        for (int p = m - 1; p >= 0 && __builtin_popcount(r) < 3; --p) r |= 1u << p;
    for (unsigned r : bits) {
        Layout L;
        L.r = 3;
        int k = 0;
        for (int p = 0; p < m; ++p) {
            if ((r >> p) & 1u) L.rp[k++] = p;
            else L.nonr.push_back(p);
        }
        P.lays.push_back(L);
    }
    return P;
}

}  // namespace

std::string expect_source(const ExpBatch& b) {
    const int m = b.m;
    const int SIZE = 1 << m;
    const int T = SIZE / 8;
    const int logT = m - 3;
    const int NW = T / 32;
    const int NT = b.nt;
    const ExpPlan P = plan_expect(b);
    const Swizzle sw = choose_swizzle(P.lays, m);
    std::vector<int> q(b.q, b.q + m), rest(b.rest, b.rest + b.nrest);
    auto reg_slots = [&](const Layout& L, unsigned mask) {
        unsigned c = 0;
        for (int j = 0; j < 3; ++j)
            if ((mask >> L.rp[j]) & 1u) c |= 1u << j;
        return c;
    };
    std::ostringstream s;
    const int minb = std::max(1, 512 / T);
    s << "#include \"pass_ops.cuh\"\n"
      << "extern \"C\" __global__ void __launch_bounds__(" << T << ", " << minb << ")\n"
      << " nqexp(const double2* __restrict__ st, double* __restrict__ part, long long ntiles) {\n"
      << "  using namespace nq;\n"
      << "  extern __shared__ __align__(16) unsigned char smem[];\n"
      << "  double2* buf0 = reinterpret_cast<double2*>(smem);\n"
      << "  double2* buf1 = buf0 + " << SIZE << ";\n"
      << "  __shared__ double red[" << NW << "][" << NT << "];\n"
      << "  const unsigned tid = threadIdx.x;\n";
    {
        std::vector<int> qlow(q.begin(), q.begin() + logT);
        s << "  const unsigned long long goff = " << deposit_expr("(unsigned long long)tid", qlow, true) << ";\n";
        s << "  const unsigned psw = " << swz_expr("tid", sw) << ";\n";
    }
    for (size_t k = 0; k < P.lays.size(); ++k) {
        s << "  const unsigned e" << k << " = " << deposit_expr("tid", P.lays[k].nonr, false) << ";\n";
        s << "  const unsigned s" << k << " = " << swz_expr("e" + std::to_string(k), sw) << ";\n";
    }
    bool any_glob = false;
    s << "  unsigned ts = 0u;\n";
    for (int t = 0; t < NT; ++t) {
        const ExpTerm& E = b.t[t];
        any_glob = any_glob || E.sglob != 0;
        const int l = P.lay_of[size_t(t)];
        if (l >= 0 && E.stile)
            s << "  ts |= (unsigned(__popc(e" << l << " & " << E.stile << "u)) & 1u) << " << t << ";\n";
    }
    for (int t = 0; t < NT; ++t) s << "  double acc" << t << " = 0.0;\n";
    // natural-order tile copy: element tid + j*T
    auto issue = [&](const std::string& rexpr, const std::string& buf, const std::string& ind) {
        s << ind << "{ const double2* src = st + (" << deposit_expr("(unsigned long long)(" + rexpr + ")", rest, true)
          << ") + goff;\n";
        for (int j = 0; j < 8; ++j) {
            unsigned long long dep = 0;
            const unsigned e = unsigned(j) << logT;
            for (int i = 0; i < m; ++i)
                if ((e >> i) & 1u) dep |= 1ull << q[size_t(i)];
            s << ind << "  cp_async16(" << buf << " + (psw ^ " << (sw.apply(e) & ~0u) << "u), src + " << hex64(dep)
              << ");\n";
        }
        s << ind << "}\n";
    };
    s << "  long long r = blockIdx.x;\n"
      << "  if (r < ntiles) ";
    issue("r", "buf0", "  ");
    s << "  cp_async_commit();\n"
      << "  for (int it = 0; r < ntiles; r += gridDim.x, ++it) {\n"
      << "    double2* cur = (it & 1) ? buf1 : buf0;\n"
      << "    double2* nxt = (it & 1) ? buf0 : buf1;\n"
      << "    const long long rn = r + gridDim.x;\n"
      << "    if (rn < ntiles) ";
    issue("rn", "nxt", "    ");
    s << "    cp_async_commit();\n"
      << "    cp_async_wait<1>();\n"
      << "    __syncthreads();\n";
    if (any_glob) {
        s << "    const unsigned long long base = " << deposit_expr("(unsigned long long)r", rest, true) << ";\n"
          << "    unsigned gb = 0u;\n";
        for (int t = 0; t < NT; ++t)
            if (b.t[t].sglob)
                s << "    gb |= (unsigned(__popcll(base & " << hex64(b.t[t].sglob) << ")) & 1u) << " << t << ";\n";
    } else {
        s << "    const unsigned gb = 0u;\n";
    }
    s << "    const unsigned gs = ts ^ gb;\n";
    for (size_t k = 0; k < P.lays.size(); ++k) {
        const Layout& L = P.lays[k];
        bool used = false;
        for (int t = 0; t < NT; ++t) used = used || P.lay_of[size_t(t)] == int(k);
        if (!used) continue;
        s << "    {\n";
        for (int j = 0; j < 8; ++j)
            s << "      const double2 v" << j << " = cur[s" << k << " ^ " << sw.apply(L.rconst(j)) << "u];\n";
        bool anyz = false;
        for (int t = 0; t < NT; ++t) anyz = anyz || (b.t[t].ftile == 0 && P.lay_of[size_t(t)] == int(k));
        if (anyz) {
            for (int j = 0; j < 8; ++j) s << "      double w" << j << " = fma(v" << j << ".x, v" << j << ".x, v" << j << ".y * v" << j << ".y);\n";
            for (int bb = 0; bb < 3; ++bb)
                for (int j = 0; j < 8; ++j) {
                    if ((j >> bb) & 1) continue;
                    const int h = j | (1 << bb);
                    s << "      { const double x = w" << j << ", y = w" << h << "; w" << j << " = x + y; w" << h
                      << " = x - y; }\n";
                }
        }
        for (int t = 0; t < NT; ++t) {
            if (P.lay_of[size_t(t)] != int(k)) continue;
            const ExpTerm& E = b.t[t];
            const unsigned cs = reg_slots(L, E.stile);
            if (E.ftile == 0) {
                s << "      acc" << t << " += ((gs >> " << t << ") & 1u) ? -w" << cs << " : w" << cs << ";\n";
                continue;
            }
            const unsigned fr = reg_slots(L, E.ftile);
            const int f0 = __builtin_ctz(fr);
            s << "      { double x = 0.0;\n";
            for (int j = 0; j < 8; ++j) {
                if ((j >> f0) & 1) continue;
                const int z = j ^ int(fr);
                const bool neg = __builtin_popcount(unsigned(j) & cs) & 1;
                std::ostringstream v;
                if (E.eps_im)
                    v << "fma(v" << z << ".x, v" << j << ".y, -(v" << z << ".y * v" << j << ".x))";
                else
                    v << "fma(v" << z << ".x, v" << j << ".x, v" << z << ".y * v" << j << ".y)";
                s << "        x " << (neg ? "-= " : "+= ") << v.str() << ";\n";
            }
            s << "        acc" << t << " += ((gs >> " << t << ") & 1u) ? -x : x; }\n";
        }
        s << "    }\n";
    }
    for (int t = 0; t < NT; ++t) {
        if (P.lay_of[size_t(t)] >= 0) continue;
        const ExpTerm& E = b.t[t];
        const int f0 = __builtin_ctz(E.ftile);
        s << "    for (unsigned w = tid; w < " << SIZE / 2 << "u; w += " << T << "u) {\n"
          << "      const unsigned y = ((w >> " << f0 << ") << " << f0 + 1 << ") | (w & " << ((1u << f0) - 1u)
          << "u);\n"
          << "      const unsigned z = y ^ " << E.ftile << "u;\n"
          << "      const double2 ay = cur[" << swz_expr("y", sw) << "], az = cur[" << swz_expr("z", sw) << "];\n";
        if (E.eps_im) s << "      const double x = fma(az.x, ay.y, -(az.y * ay.x));\n";
        else s << "      const double x = fma(az.x, ay.x, az.y * ay.y);\n";
        s << "      acc" << t << " += ((__popc(y & " << E.stile << "u) ^ (gb >> " << t << ")) & 1u) ? -x : x;\n"
          << "    }\n";
    }
    s << "    __syncthreads();\n"
      << "  }\n"
      << "  cp_async_wait<0>();\n"
      << "  const unsigned lane = tid & 31u, warp = tid >> 5;\n";
    for (int t = 0; t < NT; ++t) {
        s << "  { double v = acc" << t << ";\n"
          << "    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);\n"
          << "    if (lane == 0) red[warp][" << t << "] = v; }\n";
    }
    s << "  __syncthreads();\n"
      << "  if (tid < " << NT << "u) {\n"
      << "    double v = 0.0;\n"
      << "    for (int w = 0; w < " << NW << "; ++w) v += red[w][tid];\n"
      << "    part[size_t(blockIdx.x) * " << kMaxExpTerms << " + tid] = v;\n"
      << "  }\n"
      << "}\n";
    return s.str();
}

bool jit_expect_launch(const double2* state, int nloc, const ExpBatch& b, double* part, double* out,
                       cudaStream_t s, int device) {
    const JitMode mode = jit_mode();
    if (mode == JitMode::Off || b.m < 8 || b.m > 12 || b.nt < 1) return false;
    if (mode == JitMode::Auto && nloc < 18) return false;
    std::shared_ptr<Entry> e = acquire(expect_source(b), device, mode);
    if (!e) return false;
    const int T = (1 << b.m) / 8;
    const size_t smem = (size_t(2) << b.m) * 16;
    occupancy(*e, device, T, smem);
    const long long ntiles = 1ll << (nloc - b.m);
    const long long grid = std::min<long long>(ntiles, kExpGrid);
    long long nt = ntiles;
    void* args[] = {const_cast<double2**>(&state), &part, &nt};
    if (cudaLaunchKernel(reinterpret_cast<const void*>(e->kern), dim3(unsigned(grid)), dim3(unsigned(T)), args, smem,
                         s) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    ++jit().stats.launches;
    launch_expect_final(part, int(grid), b.nt, out, s);
    return true;
}

bool jit_compile_only(const std::string& src, std::string* log) {
    nvrtcProgram prog;
    const char* hdrs[1] = {kPassOpsSrc};
    const char* names[1] = {"pass_ops.cuh"};
    if (nvrtcCreateProgram(&prog, src.c_str(), "nqjit.cu", 1, hdrs, names) != NVRTC_SUCCESS) return false;
    int nopt_ = 0;
    const char* const* opts_ = nvrtc_opts(&nopt_);
    const nvrtcResult rc = nvrtcCompileProgram(prog, nopt_, opts_);
    size_t logn = 0;
    nvrtcGetProgramLogSize(prog, &logn);
    if (log && logn > 1) {
        log->resize(logn);
        nvrtcGetProgramLog(prog, &(*log)[0]);
    }
    nvrtcDestroyProgram(&prog);
    return rc == NVRTC_SUCCESS;
}

void jit_wait() {
    Jit& J = jit();
    std::unique_lock<std::mutex> lk(J.mu);
    J.cv.wait(lk, [&] { return J.queue.empty() && J.busy == 0; });
}

JitStats jit_stats() {
    Jit& J = jit();
    std::lock_guard<std::mutex> lk(J.mu);
    return J.stats;
}

}  // namespace nqe

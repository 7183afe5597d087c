// The fused pass kernel (sm_100a): one HBM read + one HBM write of the state
// per pass, every micro-op of the pass applied in between.
//
// Replaces the per-gate full-state sweeps of the reference (K1-K8,
// proj/src/statevector.cpp:50-180) and its blockwise Kraus sums (K14,
// proj/src/densitymatrix.cpp:60-110).
//
// Layout.  A pass has an m-bit tile set Q (PassHdr::q).  Each CTA owns 2^m
// amplitudes at a time (one value of the non-tile bits; persistent loop over
// tiles).  Every thread keeps E = 16 of them in REGISTERS: the 4 "register
// bits" of the current layout (MOP_LAYOUT) index a thread's amplitudes, the
// other m-4 tile bits index the thread.  Operators whose non-diagonal bits are
// register bits run entirely in registers with compile-time slot indices;
// diagonal operators only need each amplitude's index and run in any layout.
// A MOP_LAYOUT between ops re-distributes the tile through shared memory
// (one swizzled STS.128 + LDS.128 round trip); the planner inserts one only
// when the next op needs a bit that is not register-resident.  Operator
// matrices live in shared memory and are re-read (broadcast LDS) where used,
// which keeps the kernel at <= 128 registers (two 256-thread CTAs per SM).
#include "kernels.hpp"
#include "pass_ops.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace nqe {

namespace {

using namespace nq;

template <int M, int RR>
struct Geo {
    static constexpr int SIZE = 1 << M;
    static constexpr int R = M < RR ? M : RR;  // register bits
    static constexpr int E = 1 << R;         // amplitudes per thread
    static constexpr int T = SIZE / E;       // threads per CTA
};

// Register layout state of a thread.
struct Lay {
    int rp[4];      // tile bit of register slot j
    uint32_t rmask; // tile bits that are register bits
    uint32_t tb;    // this thread's tile-index bits (thread bits deposited)
};

template <int M, int RR>
__device__ __forceinline__ void set_layout(Lay& L, const int8_t* pos, int tid) {
    constexpr int R = Geo<M, RR>::R;
    uint32_t rmask = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        L.rp[j] = j < R ? pos[j] : 0;
        if (j < R) rmask |= 1u << pos[j];
    }
    uint32_t tb = 0;
    int k = 0;
#pragma unroll
    for (int b = 0; b < M; ++b) {
        if (!((rmask >> b) & 1u)) {
            tb |= uint32_t((tid >> k) & 1) << b;
            ++k;
        }
    }
    L.rmask = rmask;
    L.tb = tb;
}

template <int R>
__device__ __forceinline__ uint32_t rpart(const Lay& L, int l) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) r |= uint32_t((l >> j) & 1) << L.rp[j];
    return r;
}

// Diagonal operator: table index bit j comes from a register slot, a thread
// bit, or a full-index bit outside the tile.  Per amplitude: a compile-time
// OR of per-slot contributions, one broadcast-friendly LDS, one cmul.
template <int M, int RR>
__device__ __forceinline__ void diag_op(double2 (&a)[Geo<M, RR>::E], const Lay& L, const MOp& op, const double2* tab,
                                        uint64_t full) {
    constexpr int E = Geo<M, RR>::E, R = Geo<M, RR>::R;
    uint32_t base = 0;       // thread + global contributions
    uint32_t ms[4] = {0, 0, 0, 0};  // contribution of register slot s
    bool any_reg = false;
    for (int j = 0; j < op.k; ++j) {
        const int p = op.pos[j];
        if (p < 0) {
            base |= uint32_t((full >> (-1 - p)) & 1u) << j;
        } else if ((L.rmask >> p) & 1u) {
#pragma unroll
            for (int s = 0; s < R; ++s)
                if (L.rp[s] == p) ms[s] |= 1u << j;
            any_reg = true;
        } else {
            base |= ((L.tb >> p) & 1u) << j;
        }
    }
    if (!any_reg) {
        const double2 f = lds(tab + base);
        if (is_one(f)) return;
#pragma unroll
        for (int l = 0; l < E; ++l) a[l] = cmul(f, a[l]);
        return;
    }
#pragma unroll
    for (int l = 0; l < E; ++l) {
        uint32_t idx = base;
#pragma unroll
        for (int s = 0; s < R; ++s)
            if ((l >> s) & 1) idx |= ms[s];
        const double2 f = lds(tab + idx);
        if (!is_one(f)) a[l] = cmul(f, a[l]);
    }
}

template <int M, int RR>
__device__ __forceinline__ void dense_op(double2 (&a)[Geo<M, RR>::E], const MOp& op, const double2* u,
                                         double2* scratch) {
    constexpr int E = Geo<M, RR>::E, R = Geo<M, RR>::R;
    if (op.k == 1) {
        switch (op.pos[0]) {
        case 0: d1<E, 0>(a, u); break;
        case 1: if constexpr (R > 1) d1<E, 1>(a, u); break;
        case 2: if constexpr (R > 2) d1<E, 2>(a, u); break;
        default: if constexpr (R > 3) d1<E, 3>(a, u); break;
        }
    } else if (op.k == 2) {
        if constexpr (R >= 2) {
            switch (op.pos[0] * 4 + op.pos[1]) {
            case 1: d2<E, 0, 1>(a, u); break;
            case 2: if constexpr (R > 2) d2<E, 0, 2>(a, u); break;
            case 3: if constexpr (R > 3) d2<E, 0, 3>(a, u); break;
            case 6: if constexpr (R > 2) d2<E, 1, 2>(a, u); break;
            case 7: if constexpr (R > 3) d2<E, 1, 3>(a, u); break;
            default: if constexpr (R > 3) d2<E, 2, 3>(a, u); break;
            }
        }
    } else if (op.k == 3) {
        if constexpr (R == 3) {
            d3<E, 3>(a, u);
        } else if constexpr (R == 4) {
            switch (6 - op.pos[0] - op.pos[1] - op.pos[2]) {  // the slot not used
            case 0: d3<E, 0>(a, u); break;
            case 1: d3<E, 1>(a, u); break;
            case 2: d3<E, 2>(a, u); break;
            default: d3<E, 3>(a, u); break;
            }
        }
    } else {
        d4<E>(a, u, scratch);
    }
}

template <int M, int RR>
__device__ __forceinline__ void xperm_op(double2 (&a)[Geo<M, RR>::E], const Lay& L, const MOp& op, uint64_t full) {
    constexpr int E = Geo<M, RR>::E, R = Geo<M, RR>::R;
    if ((full & op.cmask_glob) != op.cmask_glob) return;
    // split tile controls into register-slot controls and thread-bit controls
    uint32_t cmL = 0, cmT = 0;
    for (int p = 0; p < M; ++p) {
        if (!((op.cmask_tile >> p) & 1u)) continue;
        if ((L.rmask >> p) & 1u) {
#pragma unroll
            for (int s = 0; s < R; ++s)
                if (L.rp[s] == p) cmL |= 1u << s;
        } else {
            cmT |= 1u << p;
        }
    }
    if ((L.tb & cmT) != cmT) return;
    switch (op.pos[0]) {
    case 0: xperm<E, 0>(a, cmL); break;
    case 1: if constexpr (R > 1) xperm<E, 1>(a, cmL); break;
    case 2: if constexpr (R > 2) xperm<E, 2>(a, cmL); break;
    default: if constexpr (R > 3) xperm<E, 3>(a, cmL); break;
    }
}

template <int M, int RR>
__device__ __forceinline__ void swap_op(double2 (&a)[Geo<M, RR>::E], const MOp& op) {
    constexpr int E = Geo<M, RR>::E, R = Geo<M, RR>::R;
    if constexpr (R >= 2) {
        switch (op.pos[0] * 4 + op.pos[1]) {
        case 1: swp<E, 0, 1>(a); break;
        case 2: if constexpr (R > 2) swp<E, 0, 2>(a); break;
        case 3: if constexpr (R > 3) swp<E, 0, 3>(a); break;
        case 6: if constexpr (R > 2) swp<E, 1, 2>(a); break;
        case 7: if constexpr (R > 3) swp<E, 1, 3>(a); break;
        default: if constexpr (R > 3) swp<E, 2, 3>(a); break;
        }
    }
}

template <int M, int RR>
__device__ __forceinline__ void depol_op(double2 (&a)[Geo<M, RR>::E], const MOp& op, const double2* p) {
    constexpr int E = Geo<M, RR>::E, R = Geo<M, RR>::R;
    const double al = lds(p).x, be = lds(p + 1).x;
    if (op.k == 2) {
        if constexpr (R >= 2) {
            const int s0 = min(op.pos[0], op.pos[1]), s1 = max(op.pos[0], op.pos[1]);
            switch (s0 * 4 + s1) {
            case 1: dep2<E, 0, 1>(a, al, be); break;
            case 2: if constexpr (R > 2) dep2<E, 0, 2>(a, al, be); break;
            case 3: if constexpr (R > 3) dep2<E, 0, 3>(a, al, be); break;
            case 6: if constexpr (R > 2) dep2<E, 1, 2>(a, al, be); break;
            case 7: if constexpr (R > 3) dep2<E, 1, 3>(a, al, be); break;
            default: if constexpr (R > 3) dep2<E, 2, 3>(a, al, be); break;
            }
        }
    } else {
        // pairs (pos[0], pos[2]) and (pos[1], pos[3]): slot 0's partner
        const int p0 = op.pos[0] == 0 ? op.pos[2] : op.pos[2] == 0 ? op.pos[0] : op.pos[1] == 0 ? op.pos[3] : op.pos[1];
        switch (p0) {
        case 1: dep4<E, 1>(a, al, be); break;
        case 2: dep4<E, 2>(a, al, be); break;
        default: dep4<E, 3>(a, al, be); break;
        }
    }
}

__device__ __forceinline__ uint64_t deposit(uint64_t v, const int8_t* pos, int cnt) {
    uint64_t r = 0;
    for (int j = 0; j < cnt; ++j)
        if ((v >> j) & 1) r |= uint64_t(1) << pos[j];
    return r;
}

// State offset of tile element e (tile bit i <-> state bit q[i]).
template <int M, int RR>
__device__ __forceinline__ uint64_t tile_off(uint32_t e, const int8_t* q) {
    uint64_t r = 0;
#pragma unroll
    for (int i = 0; i < M; ++i)
        if ((e >> i) & 1u) r |= uint64_t(1) << q[i];
    return r;
}

template <int M, int RR>
__global__ void __launch_bounds__(Geo<M, RR>::T, (Geo<M, RR>::T >= 256 ? 512 / Geo<M, RR>::T : 1))
    pass_kernel(double2* __restrict__ st, const unsigned char* __restrict__ rec, uint64_t rankbase) {
    constexpr int SIZE = Geo<M, RR>::SIZE, R = Geo<M, RR>::R, E = Geo<M, RR>::E, T = Geo<M, RR>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int8_t s_q[16];
    __shared__ int8_t s_qst[16];
    __shared__ int8_t s_rest[56];

    const PassHdr* h = reinterpret_cast<const PassHdr*>(rec);
    const int tid = threadIdx.x;
    const int nops = h->nops;
    const int pool_n = int(h->pool_n);
    double2* tile = reinterpret_cast<double2*>(smem_raw);  // SIZE entries (relayout + d4 scratch)
    double2* pool = tile + SIZE;
    MOp* ops = reinterpret_cast<MOp*>(pool + pool_n);

    const double2* gpool = reinterpret_cast<const double2*>(rec + h->pool_off);
    for (int i = tid; i < pool_n; i += T) pool[i] = gpool[i];
    const uint4* gops = reinterpret_cast<const uint4*>(rec + h->op_off);
    uint4* sops = reinterpret_cast<uint4*>(ops);
    for (int i = tid; i < nops * 2; i += T) sops[i] = gops[i];
    for (int i = tid; i < 16; i += T) {
        s_q[i] = h->q[i];
        s_qst[i] = h->qst[i];
    }
    for (int i = tid; i < 56; i += T) s_rest[i] = h->rest[i];
    __syncthreads();

    // ops[0] is the load layout
    Lay L0;
    set_layout<M, RR>(L0, ops[0].pos, tid);
    const int nrest = h->nrest;
    const int64_t ntiles = h->ntiles;
    bool relabel = false;  // stores go to a permutation of the loaded bits
    for (int i = 0; i < M; ++i) relabel = relabel || h->q[i] != h->qst[i];
    const uint64_t off0 = tile_off<M, RR>(L0.tb, s_q);
    uint64_t roff0[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) roff0[j] = j < R ? uint64_t(1) << s_q[L0.rp[j]] : 0;
    double2* scratch = tile + tid * E;

    for (int64_t r = blockIdx.x; r < ntiles; r += gridDim.x) {
        const uint64_t base = deposit(uint64_t(r), s_rest, nrest);
        double2 a[E];
        {
            const double2* src = st + base + off0;
#pragma unroll
            for (int l = 0; l < E; ++l) {
                uint64_t o = 0;
#pragma unroll
                for (int j = 0; j < R; ++j) o += ((l >> j) & 1) ? roff0[j] : 0;
                a[l] = ld_stream(src + o);
            }
        }
        Lay L = L0;
        const uint64_t full = rankbase | base;
#pragma unroll 1
        for (int o = 1; o < nops; ++o) {
            const MOp op = ops[o];
            switch (op.type) {
            case MOP_DENSE:
                if (op.k == 4) __syncthreads();  // scratch rows alias the relayout buffer
                dense_op<M, RR>(a, op, pool + op.mat, scratch);
                break;
            case MOP_DIAG: diag_op<M, RR>(a, L, op, pool + op.mat, full); break;
            case MOP_XPERM: xperm_op<M, RR>(a, L, op, full); break;
            case MOP_SWAP: swap_op<M, RR>(a, op); break;
            case MOP_DEPOL: depol_op<M, RR>(a, op, pool + op.mat); break;
            case MOP_LAYOUT:
                if constexpr (R < M) {
                    __syncthreads();  // previous readers of the buffer are done
#pragma unroll
                    for (int l = 0; l < E; ++l) tile[swz(L.tb | rpart<R>(L, l))] = a[l];
                    set_layout<M, RR>(L, op.pos, tid);
                    __syncthreads();
#pragma unroll
                    for (int l = 0; l < E; ++l) a[l] = tile[swz(L.tb | rpart<R>(L, l))];
                }
                break;
            default: break;
            }
        }
        {
            // with a relabelling store another thread may still have to load
            // the addresses this thread writes
            if (relabel) __syncthreads();
            const uint64_t offs = tile_off<M, RR>(L.tb, s_qst);
            uint64_t ro[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) ro[j] = j < R ? uint64_t(1) << s_qst[L.rp[j]] : 0;
            double2* dst = st + base + offs;
#pragma unroll
            for (int l = 0; l < E; ++l) {
                uint64_t o = 0;
#pragma unroll
                for (int j = 0; j < R; ++j) o += ((l >> j) & 1) ? ro[j] : 0;
                st_stream(dst + o, a[l]);
            }
        }
        if constexpr (R < M) __syncthreads();  // the next tile's first relayout reuses the buffer
    }
}

int sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int d = 0;
    cudaGetDevice(&d);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(d);
    if (it != cache.end()) return it->second;
    int s = 148;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, d);
    cache[d] = s;
    return s;
}

template <int M, int RR>
void launch_pass_m(double2* state, const unsigned char* rec, const PassHdr& h, uint64_t rankbase, cudaStream_t s) {
    constexpr int SIZE = Geo<M, RR>::SIZE, T = Geo<M, RR>::T;
    const size_t smem = size_t(SIZE) * 16 + size_t(h.pool_n) * 16 + size_t(h.nops) * sizeof(MOp);
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> occ_cache;
    int dev = 0;
    cudaGetDevice(&dev);
    int occ = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto key = std::make_pair(dev, smem);
        auto it = occ_cache.find(key);
        if (it == occ_cache.end()) {
            cudaFuncSetAttribute(pass_kernel<M, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_kernel<M, RR>, T, smem);
            if (occ < 1) occ = 1;
            occ_cache[key] = occ;
        } else {
            occ = it->second;
        }
    }
    const int64_t grid = std::min<int64_t>(h.ntiles, int64_t(sm_count()) * occ);
    pass_kernel<M, RR><<<unsigned(grid), T, smem, s>>>(state, rec, rankbase);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int M>
void launch_pass_r(double2* state, const unsigned char* rec, const PassHdr& h, uint64_t rankbase, cudaStream_t s,
                   int rbits) {
    if constexpr (M >= 5) {
        if (rbits == 3) {
            launch_pass_m<M, 3>(state, rec, h, rankbase, s);
            return;
        }
    }
    launch_pass_m<M, 4>(state, rec, h, rankbase, s);
}

}  // namespace

void launch_pass(double2* state, const unsigned char* dev_rec, const PassHdr& h, uint64_t rankbase,
                 cudaStream_t s, int rbits) {
    switch (h.m) {
    case 1: launch_pass_r<1>(state, dev_rec, h, rankbase, s, rbits); break;
    case 2: launch_pass_r<2>(state, dev_rec, h, rankbase, s, rbits); break;
    case 3: launch_pass_r<3>(state, dev_rec, h, rankbase, s, rbits); break;
    case 4: launch_pass_r<4>(state, dev_rec, h, rankbase, s, rbits); break;
    case 5: launch_pass_r<5>(state, dev_rec, h, rankbase, s, rbits); break;
    case 6: launch_pass_r<6>(state, dev_rec, h, rankbase, s, rbits); break;
    case 7: launch_pass_r<7>(state, dev_rec, h, rankbase, s, rbits); break;
    case 8: launch_pass_r<8>(state, dev_rec, h, rankbase, s, rbits); break;
    case 9: launch_pass_r<9>(state, dev_rec, h, rankbase, s, rbits); break;
    case 10: launch_pass_r<10>(state, dev_rec, h, rankbase, s, rbits); break;
    case 11: launch_pass_r<11>(state, dev_rec, h, rankbase, s, rbits); break;
    case 12: launch_pass_r<12>(state, dev_rec, h, rankbase, s, rbits); break;
    case 13: launch_pass_r<13>(state, dev_rec, h, rankbase, s, rbits); break;
    default: throw std::logic_error("launch_pass: unsupported tile size " + std::to_string(h.m));
    }
}

}  // namespace nqe

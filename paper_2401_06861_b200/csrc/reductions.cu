// sm_100a kernels of the SV/DM simulation core, other than the fused pass
// kernel (pass_kernel.cu):
//  reductions       fixed-grid, fixed-order (bit-reproducible) sums:
//                   norm/purity (K9/K15), Pauli expectations (K10/K16),
//                   probabilities (K11/K17), Kraus weights (K13).
//  sampling         block sums + per-block sequential sweeps (K12).
//  readout          per-qubit 2x2 stochastic maps (K18).
#include "kernels.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace nqe {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ uint32_t ins0(uint32_t w, int b) {
    return ((w >> b) << (b + 1)) | (w & ((1u << b) - 1u));
}
__device__ __forceinline__ uint64_t ins0_64(uint64_t w, int b) {
    return ((w >> b) << (b + 1)) | (w & ((uint64_t(1) << b) - 1u));
}
// |a|^2 exactly as std::norm on the host (proj/src/statevector.cpp:281):
// re*re + im*im with each product rounded, no fused multiply-add, so device
// probabilities equal the reference's bit for bit on the same amplitudes.
__device__ __forceinline__ double prob_rn(double2 v) { return __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)); }
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// ---------------------------------------------------------------------------
// reductions (fixed grid -> per-block partials -> one-block final combine)
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NT], double* out, int stride) {
    __shared__ double red[kThreads / 32][NT > 0 ? NT : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        double v = acc[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][t] = v;
    }
    __syncthreads();
    if (threadIdx.x < NT) {
        double s = 0.0;
        for (int w = 0; w < int(blockDim.x / 32); ++w) s += red[w][threadIdx.x];
        out[size_t(blockIdx.x) * stride + threadIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_sumsq(const double2* __restrict__ a, uint64_t n,
                                                   uint64_t chunk, double* __restrict__ part) {
    const uint64_t lo = uint64_t(blockIdx.x) * chunk;
    const uint64_t hi = min(n, lo + chunk);
    double acc[1] = {0.0};
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 v = a[i];
        acc[0] = fma(v.x, v.x, fma(v.y, v.y, acc[0]));
    }
    block_reduce_store<1>(acc, part, 1);
}

// Index of rho[row, col] in HBM: row-major (vec bits: columns low, rows
// high), or interleaved (column bit q at 2q, row bit q at 2q + 1; the layout
// of the Hermitian pass kernels).
__device__ __forceinline__ uint64_t spread_bits(uint64_t x) {
    x &= 0xFFFFFFFFull;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}
__device__ __forceinline__ uint64_t dm_index(uint64_t row, uint64_t col, uint64_t dim, int il) {
    return il ? ((spread_bits(row) << 1) | spread_bits(col)) : row * dim + col;
}

// sum of Re(rho[i, i]) for i < n (DM trace)
__global__ void __launch_bounds__(kThreads) k_strided_re(const double2* __restrict__ a, uint64_t n, int il,
                                                        uint64_t chunk, double* __restrict__ part) {
    const uint64_t lo = uint64_t(blockIdx.x) * chunk;
    const uint64_t hi = min(n, lo + chunk);
    double acc[1] = {0.0};
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc[0] += a[dm_index(i, i, n, il)].x;
    block_reduce_store<1>(acc, part, 1);
}

// Sum NT columns of per-block partials (nblk rows) in a fixed order.
__global__ void k_final(const double* __restrict__ part, int nblk, int nt, double* __restrict__ out) {
    __shared__ double sh[kThreads];
    for (int t = 0; t < nt; ++t) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += part[size_t(b) * nt + t];
        sh[threadIdx.x] = s;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (int(threadIdx.x) < w) sh[threadIdx.x] += sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[t] = sh[0];
        __syncthreads();
    }
}

constexpr int kTermsPerLaunch = 16;

struct TermBatch {
    uint64_t signs[kTermsPerLaunch];
    int eps_im[kTermsPerLaunch];  // 1: accumulate Im(conj(a[y^F]) a[y]) instead of Re
    int nt;
};

// SV Pauli expectations sharing one flip mask F.
//  F == 0: acc_t = sum_y s_t(y) |a_y|^2
//  F != 0: y ranges over indices with bit f0 = 0, v = conj(a[y^F]) a[y];
//          acc_t = sum_y s_t(y) * (eps_t ? Im v : Re v)   (see abi.cpp)
__global__ void __launch_bounds__(kThreads) k_expect(const double2* __restrict__ a, uint64_t nwork,
                                                    uint64_t flip, int f0, uint64_t chunk,
                                                    TermBatch tb, double* __restrict__ part) {
    double acc[kTermsPerLaunch];
#pragma unroll
    for (int t = 0; t < kTermsPerLaunch; ++t) acc[t] = 0.0;
    const uint64_t lo = uint64_t(blockIdx.x) * chunk;
    const uint64_t hi = min(nwork, lo + chunk);
    for (uint64_t w = lo + threadIdx.x; w < hi; w += blockDim.x) {
        uint64_t y;
        double re, im;
        if (flip == 0) {
            y = w;
            const double2 v = a[y];
            re = fma(v.x, v.x, v.y * v.y);
            im = 0.0;
        } else {
            y = ins0_64(w, f0);
            const double2 ay = a[y], az = a[y ^ flip];
            re = fma(az.x, ay.x, az.y * ay.y);
            im = fma(az.x, ay.y, -az.y * ay.x);
        }
#pragma unroll
        for (int t = 0; t < kTermsPerLaunch; ++t) {
            if (t < tb.nt) {
                const double v = tb.eps_im[t] ? im : re;
                acc[t] += (__popcll(y & tb.signs[t]) & 1) ? -v : v;
            }
        }
    }
    block_reduce_store<kTermsPerLaunch>(acc, part, kTermsPerLaunch);
}

// DM Pauli expectations: sum_y s(y) rho[y, y^F] (complex), dim = 2^n.
__global__ void __launch_bounds__(kThreads) k_dm_expect(const double2* __restrict__ rho, uint64_t dim, int il,
                                                       uint64_t flip, uint64_t chunk, TermBatch tb,
                                                       double* __restrict__ part) {
    double acc[2 * kTermsPerLaunch];
#pragma unroll
    for (int t = 0; t < 2 * kTermsPerLaunch; ++t) acc[t] = 0.0;
    const uint64_t lo = uint64_t(blockIdx.x) * chunk;
    const uint64_t hi = min(dim, lo + chunk);
    for (uint64_t y = lo + threadIdx.x; y < hi; y += blockDim.x) {
        const double2 v = rho[dm_index(y, y ^ flip, dim, il)];
#pragma unroll
        for (int t = 0; t < kTermsPerLaunch; ++t) {
            if (t < tb.nt) {
                const bool neg = (__popcll(y & tb.signs[t]) & 1) != 0;
                acc[2 * t] += neg ? -v.x : v.x;
                acc[2 * t + 1] += neg ? -v.y : v.y;
            }
        }
    }
    block_reduce_store<2 * kTermsPerLaunch>(acc, part, 2 * kTermsPerLaunch);
}

__global__ void k_probs(const double2* __restrict__ a, uint64_t n, double* __restrict__ p) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        p[i] = prob_rn(a[i]);
    }
}

// DM diagonal: max(0, Re rho_ii)
__global__ void k_dm_diag(const double2* __restrict__ rho, uint64_t dim, int il, double* __restrict__ p) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < dim;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = fmax(0.0, rho[dm_index(i, i, dim, il)].x);
}

__global__ void k_sum_real(const double* __restrict__ x, uint64_t n, uint64_t chunk,
                           double* __restrict__ part) {
    const uint64_t lo = uint64_t(blockIdx.x) * chunk;
    const uint64_t hi = min(n, lo + chunk);
    double acc[1] = {0.0};
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc[0] += x[i];
    block_reduce_store<1>(acc, part, 1);
}

__global__ void k_scale_real(double* __restrict__ x, uint64_t n, const double* __restrict__ denom) {
    const double d = *denom;
    if (!(d > 0.0)) return;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        x[i] /= d;
}

// max_{r,c} |rho[r,c] - conj(rho[c,r])| via 32x32 smem transposes; per-block max.
__global__ void k_herm(const double2* __restrict__ rho, uint64_t dim, double* __restrict__ part) {
    __shared__ double2 t[32][33];
    const uint64_t tiles_per_row = (dim + 31) / 32;
    const uint64_t ntiles = tiles_per_row * tiles_per_row;
    double worst = 0.0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t tr = tile / tiles_per_row, tc = tile % tiles_per_row;
        if (tc < tr) continue;  // upper triangle of tiles (incl. diagonal)
        const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
        for (int yy = ty; yy < 32; yy += 8) {
            const uint64_t r = tc * 32 + yy, c = tr * 32 + tx;  // transposed tile
            t[yy][tx] = (r < dim && c < dim) ? rho[r * dim + c] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        for (int yy = ty; yy < 32; yy += 8) {
            const uint64_t r = tr * 32 + yy, c = tc * 32 + tx;
            if (r < dim && c < dim) {
                const double2 a = rho[r * dim + c];
                const double2 b = t[tx][yy];  // rho[c, r]
                const double dx = a.x - b.x, dy = a.y + b.y;
                worst = fmax(worst, sqrt(dx * dx + dy * dy));
            }
        }
        __syncthreads();
    }
    __shared__ double red[kThreads];
    red[threadIdx.x] = worst;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_final_max(const double* __restrict__ part, int nblk, double* __restrict__ out) {
    __shared__ double sh[kThreads];
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) s = fmax(s, part[b]);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// ---- Kraus branch weights (K13): w_i = sum_groups sum_row |(K_i v)_row|^2 ----
struct KrausBatch {
    int k;
    int nk;
    int sp[3];        // sorted positions
    uint32_t off[8];  // local offsets (bit j <-> qubits[j])
};

__global__ void __launch_bounds__(kThreads) k_kraus_w(const double2* __restrict__ a, uint64_t ngroups,
                                                     uint64_t chunk, KrausBatch kb,
                                                     const double2* __restrict__ mats,
                                                     double* __restrict__ part) {
    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.0;
    const int D = 1 << kb.k;
    const uint64_t lo = uint64_t(blockIdx.x) * chunk;
    const uint64_t hi = min(ngroups, lo + chunk);
    for (uint64_t w = lo + threadIdx.x; w < hi; w += blockDim.x) {
        uint64_t e = w;
        for (int j = 0; j < kb.k; ++j) e = ins0_64(e, kb.sp[j]);
        double2 v[8];
        for (int l = 0; l < D; ++l) v[l] = a[e + kb.off[l]];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (i < kb.nk) {
                const double2* K = mats + size_t(i) * D * D;
                double s = 0.0;
                for (int r = 0; r < D; ++r) {
                    double2 z = make_double2(0.0, 0.0);
                    for (int c = 0; c < D; ++c) z = cfma(K[r * D + c], v[c], z);
                    s = fma(z.x, z.x, fma(z.y, z.y, s));
                }
                acc[i] += s;
            }
        }
    }
    block_reduce_store<16>(acc, part, 16);
}

// ---- sampling (K12) ----
// Per-block probability sums over fixed blocks of kSampleBlock elements.
__global__ void k_block_psum(const double2* __restrict__ a, const double* __restrict__ p, uint64_t n,
                             uint64_t bs, double* __restrict__ out) {
    // one block of threads per sample block; fixed-order tree
    const uint64_t lo = uint64_t(blockIdx.x) * bs;
    const uint64_t hi = min(n, lo + bs);
    double acc[1] = {0.0};
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        acc[0] += a ? prob_rn(a[i]) : p[i];
    }
    block_reduce_store<1>(acc, out, 1);
}

// Exact reproduction of the reference's sequential `cum += p[i]`
// (proj/src/statevector.cpp:311-320) without a serial pass: while cum stays in
// one binade [2^k, 2^(k+1)) every partial sum lies on the grid of ulp
// 2^(k-52), so fl(cum + p) = cum + rint(p / ulp) * ulp exactly unless
// p / ulp is a tie (x.5, where round-half-even depends on cum's last bit).
// Integer increments are associative: this kernel sums rint(p * 2^(52-k))
// over the block for the binade k the host guessed (kb[b]); the host
// (sample.cpp) verifies the binade and that the block stays inside it, and
// replays flagged blocks (ties, overflow, binade crossings) sequentially.
__global__ void k_block_isum(const double2* __restrict__ a, const double* __restrict__ p, uint64_t n,
                             uint64_t bs, const int* __restrict__ kb, unsigned long long* __restrict__ isum,
                             int* __restrict__ flags) {
    constexpr unsigned long long kSat = 1ull << 62;
    const uint64_t lo = uint64_t(blockIdx.x) * bs;
    const uint64_t hi = min(n, lo + bs);
    const int k = kb[blockIdx.x];
    __shared__ unsigned long long red[kThreads / 32];
    __shared__ int bad_any;
    if (threadIdx.x == 0) bad_any = 0;
    __syncthreads();
    if (k == INT_MIN) {
        if (threadIdx.x == 0) {
            isum[blockIdx.x] = 0;
            flags[blockIdx.x] = 1;
        }
        return;
    }
    const double scale = ldexp(1.0, 52 - k);  // exact power of two (host keeps 52 - k <= 1000)
    unsigned long long acc = 0;
    int bad = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double pi = a ? prob_rn(a[i]) : p[i];
        const double y = __dmul_rn(pi, scale);
        if (!(y < 9007199254740992.0) || !(y >= 0.0)) {  // >= 2^53 (leaves the binade), NaN, negative
            bad = 1;
            continue;
        }
        const double f = floor(y);
        if (y - f == 0.5) bad = 1;  // tie: rounding depends on cum's parity
        acc = min(acc + (unsigned long long)rint(y), kSat);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = min(acc + __shfl_xor_sync(0xffffffffu, acc, o), kSat);
    if (lane == 0) red[warp] = acc;
    if (bad) bad_any = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t = min(t + red[w], kSat);
        isum[blockIdx.x] = t;
        flags[blockIdx.x] = bad_any;
    }
}

// One thread per block that owns uniforms: sequential cumulative sweep from
// the host-computed block start, exactly like proj/src/statevector.cpp:311-320.
__global__ void k_block_sweep(const double2* __restrict__ a, const double* __restrict__ p, uint64_t n,
                              uint64_t bs, const int64_t* __restrict__ blk, const double* __restrict__ cum0,
                              const int64_t* __restrict__ ulo, const int64_t* __restrict__ uhi,
                              const double* __restrict__ u, int nb, uint64_t* __restrict__ idx_out,
                              uint64_t* __restrict__ cnt_out, int64_t* __restrict__ npairs) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nb) return;
    const uint64_t lo = uint64_t(blk[t]) * bs;
    const uint64_t hi = min(n, lo + bs);
    double cum = cum0[t];
    int64_t next = ulo[t];
    const int64_t end = uhi[t];
    int64_t slot = ulo[t];
    uint64_t last_nz = UINT64_MAX;
    for (uint64_t i = lo; i < hi && next < end; ++i) {
        const double pi = a ? prob_rn(a[i]) : p[i];
        cum = __dadd_rn(cum, pi);
        if (pi > 0.0) last_nz = i;
        uint64_t here = 0;
        while (next < end && u[next] < cum) {
            ++here;
            ++next;
        }
        if (here > 0) {
            idx_out[slot] = i;
            cnt_out[slot] = here;
            ++slot;
        }
    }
    if (next < end) {
        // rounding between the host block prefix and this sweep: the remaining
        // uniforms belong to this block; give them to its last nonzero entry.
        for (uint64_t i = hi; i-- > lo;) {
            const double pi = a ? prob_rn(a[i]) : p[i];
            if (pi > 0.0) {
                last_nz = i;
                break;
            }
        }
        if (last_nz != UINT64_MAX) {
            if (slot > ulo[t] && idx_out[slot - 1] == last_nz) {
                cnt_out[slot - 1] += uint64_t(end - next);
            } else {
                idx_out[slot] = last_nz;
                cnt_out[slot] = uint64_t(end - next);
                ++slot;
            }
        }
    }
    npairs[t] = slot - ulo[t];
}

// Last index with p > 0 inside one block (for leftover uniforms).
__global__ void k_last_nonzero(const double2* __restrict__ a, const double* __restrict__ p, uint64_t lo,
                               uint64_t hi, uint64_t* __restrict__ out) {
    __shared__ unsigned long long best;
    if (threadIdx.x == 0) best = 0;
    __syncthreads();
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double pi = a ? prob_rn(a[i]) : p[i];
        if (pi > 0.0) atomicMax(&best, (unsigned long long)(i + 1));
    }
    __syncthreads();
    if (threadIdx.x == 0) *out = uint64_t(best);
}

// ---- readout confusion (K18): one qubit per launch, pairs (idx, idx|bit) ----
__global__ void k_readout(double* __restrict__ d, uint64_t half, int q, double p01, double p10) {
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < half;
         w += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i0 = ins0_64(w, q), i1 = i0 | (uint64_t(1) << q);
        const double v0 = d[i0], v1 = d[i1];
        d[i0] = (1.0 - p10) * v0 + p01 * v1;
        d[i1] = p10 * v0 + (1.0 - p01) * v1;
    }
}

__global__ void k_init_basis(double2* a, uint64_t n, uint64_t one_at) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        a[i] = make_double2(i == one_at ? 1.0 : 0.0, 0.0);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
struct DevInfo {
    int sms = 148;
};

DevInfo dev_info() {
    static std::mutex mu;
    static std::map<int, DevInfo> cache;
    int d = 0;
    cudaGetDevice(&d);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(d);
    if (it != cache.end()) return it->second;
    DevInfo info;
    cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, d);
    cache[d] = info;
    return info;
}

int grid_for(uint64_t n, int per_thread = 4) {
    const uint64_t want = (n + uint64_t(kThreads) * per_thread - 1) / (uint64_t(kThreads) * per_thread);
    const int sms = dev_info().sms;
    return int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sms) * 16)));
}

// Fixed reduction geometry: chunk and block count depend only on n, never on
// the device, so results are bit-identical on any GPU / any run.
void reduction_geometry(uint64_t n, uint64_t* chunk, int* nblk) {
    const uint64_t target_blocks = 2048;
    uint64_t c = (n + target_blocks - 1) / target_blocks;
    c = std::max<uint64_t>(c, 1024);
    c = (c + kThreads - 1) / kThreads * kThreads;
    *chunk = c;
    *nblk = int((n + c - 1) / c);
    if (*nblk < 1) *nblk = 1;
}

}  // namespace

std::atomic<int64_t> g_kernel_launches{0};

void launch_init_basis(double2* a, uint64_t n, uint64_t one_at, cudaStream_t s) {
    k_init_basis<<<grid_for(n), kThreads, 0, s>>>(a, n, one_at);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_sumsq(const double2* a, uint64_t n, double* scratch, double* out, cudaStream_t s) {
    uint64_t chunk;
    int nblk;
    reduction_geometry(n, &chunk, &nblk);
    k_sumsq<<<nblk, kThreads, 0, s>>>(a, n, chunk, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch, nblk, 1, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_trace(const double2* rho, uint64_t dim, double* scratch, double* out, cudaStream_t s, int il) {
    uint64_t chunk;
    int nblk;
    reduction_geometry(dim, &chunk, &nblk);
    k_strided_re<<<nblk, kThreads, 0, s>>>(rho, dim, il, chunk, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch, nblk, 1, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

size_t scratch_doubles_needed(uint64_t n) {
    uint64_t chunk;
    int nblk;
    reduction_geometry(n, &chunk, &nblk);
    return size_t(nblk) * 2 * kTermsPerLaunch + 64;
}

int terms_per_launch() { return kTermsPerLaunch; }

void launch_expect_sv(const double2* a, int nbits, uint64_t flip, const uint64_t* signs,
                      const int* eps_im, int nt, double* scratch, double* out, cudaStream_t s) {
    TermBatch tb{};
    tb.nt = nt;
    for (int t = 0; t < nt; ++t) {
        tb.signs[t] = signs[t];
        tb.eps_im[t] = eps_im[t];
    }
    const uint64_t n = uint64_t(1) << nbits;
    const uint64_t nwork = flip ? n / 2 : n;
    const int f0 = flip ? __builtin_ctzll(flip) : 0;
    uint64_t chunk;
    int nblk;
    reduction_geometry(nwork, &chunk, &nblk);
    k_expect<<<nblk, kThreads, 0, s>>>(a, nwork, flip, f0, chunk, tb, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch, nblk, kTermsPerLaunch, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_expect_dm(const double2* rho, int n, uint64_t flip, const uint64_t* signs, int nt,
                      double* scratch, double* out, cudaStream_t s, int il) {
    TermBatch tb{};
    tb.nt = nt;
    for (int t = 0; t < nt; ++t) tb.signs[t] = signs[t];
    const uint64_t dim = uint64_t(1) << n;
    uint64_t chunk;
    int nblk;
    reduction_geometry(dim, &chunk, &nblk);
    k_dm_expect<<<nblk, kThreads, 0, s>>>(rho, dim, il, flip, chunk, tb, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch, nblk, 2 * kTermsPerLaunch, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_probs(const double2* a, uint64_t n, double* p, cudaStream_t s) {
    k_probs<<<grid_for(n), kThreads, 0, s>>>(a, n, p);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_dm_probs(const double2* rho, uint64_t dim, double* p, double* scratch, cudaStream_t s, int il) {
    k_dm_diag<<<grid_for(dim), kThreads, 0, s>>>(rho, dim, il, p);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    uint64_t chunk;
    int nblk;
    reduction_geometry(dim, &chunk, &nblk);
    k_sum_real<<<nblk, kThreads, 0, s>>>(p, dim, chunk, scratch + 1);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch + 1, nblk, 1, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_scale_real<<<grid_for(dim), kThreads, 0, s>>>(p, dim, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_sum_real(const double* x, uint64_t n, double* scratch, double* out, cudaStream_t s) {
    uint64_t chunk;
    int nblk;
    reduction_geometry(n, &chunk, &nblk);
    k_sum_real<<<nblk, kThreads, 0, s>>>(x, n, chunk, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch, nblk, 1, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_herm(const double2* rho, uint64_t dim, double* scratch, double* out, cudaStream_t s) {
    const uint64_t tpr = (dim + 31) / 32;
    const int nblk = int(std::min<uint64_t>(tpr * tpr, 2048));
    k_herm<<<nblk, kThreads, 0, s>>>(rho, dim, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final_max<<<1, kThreads, 0, s>>>(scratch, nblk, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_kraus_weights(const double2* a, int nbits, const int* qubits, int k, int nk,
                          const double2* dev_mats, double* scratch, double* out, cudaStream_t s) {
    KrausBatch kb{};
    kb.k = k;
    kb.nk = nk;
    int sp[3] = {qubits[0], k > 1 ? qubits[1] : 0, k > 2 ? qubits[2] : 0};
    std::sort(sp, sp + k);
    for (int j = 0; j < k; ++j) kb.sp[j] = sp[j];
    for (int l = 0; l < (1 << k); ++l) {
        uint32_t o = 0;
        for (int j = 0; j < k; ++j)
            if ((l >> j) & 1) o |= 1u << qubits[j];
        kb.off[l] = o;
    }
    const uint64_t ng = (uint64_t(1) << nbits) >> k;
    uint64_t chunk;
    int nblk;
    reduction_geometry(ng, &chunk, &nblk);
    k_kraus_w<<<nblk, kThreads, 0, s>>>(a, ng, chunk, kb, dev_mats, scratch);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    k_final<<<1, kThreads, 0, s>>>(scratch, nblk, 16, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_block_psum(const double2* a, const double* p, uint64_t n, uint64_t bs, double* out,
                       cudaStream_t s) {
    const uint64_t nb = (n + bs - 1) / bs;
    k_block_psum<<<unsigned(nb), kThreads, 0, s>>>(a, p, n, bs, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_block_isum(const double2* a, const double* p, uint64_t n, uint64_t bs, const int* kb,
                       unsigned long long* isum, int* flags, cudaStream_t s) {
    const uint64_t nb = (n + bs - 1) / bs;
    k_block_isum<<<unsigned(nb), kThreads, 0, s>>>(a, p, n, bs, kb, isum, flags);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_block_sweep(const double2* a, const double* p, uint64_t n, uint64_t bs, const int64_t* blk,
                        const double* cum0, const int64_t* ulo, const int64_t* uhi, const double* u,
                        int nb, uint64_t* idx_out, uint64_t* cnt_out, int64_t* npairs, cudaStream_t s) {
    if (nb <= 0) return;
    k_block_sweep<<<(nb + 127) / 128, 128, 0, s>>>(a, p, n, bs, blk, cum0, ulo, uhi, u, nb, idx_out,
                                                   cnt_out, npairs);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_last_nonzero(const double2* a, const double* p, uint64_t lo, uint64_t hi, uint64_t* out,
                         cudaStream_t s) {
    k_last_nonzero<<<1, kThreads, 0, s>>>(a, p, lo, hi, out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_readout(double* d, int n, int q, double p01, double p10, cudaStream_t s) {
    const uint64_t half = (uint64_t(1) << n) / 2;
    k_readout<<<grid_for(half), kThreads, 0, s>>>(d, half, q, p01, p10);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace nqe

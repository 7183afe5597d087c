// Batched Monte-Carlo trajectories: many independent
// trajectories of one noisy schedule per launch.
//
// Reference: StateVector::run_trajectory / apply_kraus_trajectory
// (proj/src/statevector.cpp:339-401), driven one trajectory at a time with a
// shared Rng (tests/acceptance/acceptance_main.cpp:137-173).  Each channel
// application draws exactly one next_double(), so trajectory t consumes draws
// [t*C, (t+1)*C) of the sequential stream (C = channels in the schedule): the
// host generates them once and the batch reproduces the sequential loop.
//
// One CTA per trajectory; its 2^n amplitudes live in shared memory for the
// whole schedule (n <= 13).  Gates: gather / 2^k x 2^k matvec / scatter per
// group, threads over groups.  Channels: per-Kraus branch weights
// ||K_i psi||^2 by a fixed-order block reduction, branch chosen by one thread
// exactly as the reference (u * total against the running sum, leftover to
// the last), then K_chosen / sqrt(w_chosen) applied.  Final Pauli
// expectations (statevector.cpp:241-277) per trajectory.
#include "kernels.hpp"

#include <cuda_runtime.h>

namespace nqe {

namespace {

constexpr int kTrajThreads = 128;

__device__ __forceinline__ double2 cmul_(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];  // fixed order
    return s;
}

// base index of group g: zeros inserted at the sorted target positions
__device__ __forceinline__ uint32_t expand(uint32_t g, const int* sorted, int k) {
#pragma unroll 4
    uint32_t x = g;
    for (int j = 0; j < k; ++j) {
        const int p = sorted[j];
        x = ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u));
    }
    return x;
}

struct Targets {
    int sorted[4];
    uint32_t off[16];
};

template <int K>
__device__ __forceinline__ void targets_of(const TrajItem& it, Targets& t) {
    for (int j = 0; j < K; ++j) t.sorted[j] = it.q[j];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = i + 1; j < K; ++j)
            if (t.sorted[j] < t.sorted[i]) {
                const int x = t.sorted[i];
                t.sorted[i] = t.sorted[j];
                t.sorted[j] = x;
            }
#pragma unroll
    for (int c = 0; c < (1 << K); ++c) {
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((c >> j) & 1) o |= 1u << it.q[j];
        t.off[c] = o;
    }
}

// psi <- scale * M psi on qubits q[0..K) (local bit j <-> q[j])
template <int K>
__device__ void apply_mat_k(double2* a, int n, const TrajItem& it, const double2* M, double scale) {
    constexpr int d = 1 << K;
    Targets t;
    targets_of<K>(it, t);
    const uint32_t groups = 1u << (n - K);
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x) {
        const uint32_t base = expand(g, t.sorted, K);
        double2 x[d];
#pragma unroll
        for (int c = 0; c < d; ++c) x[c] = a[base + t.off[c]];
#pragma unroll(K <= 2 ? d : 1)
        for (int r = 0; r < d; ++r) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < d; ++c) {
                const double2 p = cmul_(M[r * d + c], x[c]);
                acc.x += p.x;
                acc.y += p.y;
            }
            a[base + t.off[r]] = make_double2(acc.x * scale, acc.y * scale);
        }
    }
}

__device__ void apply_mat(double2* a, int n, const TrajItem& it, const double2* M, double scale) {
    switch (it.k) {
    case 1: apply_mat_k<1>(a, n, it, M, scale); break;
    case 2: apply_mat_k<2>(a, n, it, M, scale); break;
    case 3: apply_mat_k<3>(a, n, it, M, scale); break;
    default: apply_mat_k<4>(a, n, it, M, scale); break;
    }
}

template <int K>
__device__ double branch_weight_k(const double2* a, int n, const TrajItem& it, const double2* Km) {
    constexpr int d = 1 << K;
    Targets t;
    targets_of<K>(it, t);
    double acc = 0.0;
    const uint32_t groups = 1u << (n - K);
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x) {
        const uint32_t base = expand(g, t.sorted, K);
        double2 x[d];
#pragma unroll
        for (int c = 0; c < d; ++c) x[c] = a[base + t.off[c]];
#pragma unroll(K <= 2 ? d : 1)
        for (int r = 0; r < d; ++r) {
            double2 w = make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < d; ++c) {
                const double2 p = cmul_(Km[r * d + c], x[c]);
                w.x += p.x;
                w.y += p.y;
            }
            acc += w.x * w.x + w.y * w.y;
        }
    }
    return acc;
}

__device__ double branch_weight(const double2* a, int n, const TrajItem& it, const double2* Km) {
    switch (it.k) {
    case 1: return branch_weight_k<1>(a, n, it, Km);
    case 2: return branch_weight_k<2>(a, n, it, Km);
    default: return branch_weight_k<3>(a, n, it, Km);
    }
}

__global__ void __launch_bounds__(kTrajThreads) k_traj(TrajArgs p) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* a = reinterpret_cast<double2*>(smem);
    __shared__ double red[kTrajThreads / 32];
    __shared__ double s_w[kMaxTrajKraus];
    __shared__ int s_sel;
    __shared__ double s_scale;
    const int64_t b = blockIdx.x;
    const uint32_t dim = 1u << p.n;
    for (uint32_t i = threadIdx.x; i < dim; i += blockDim.x) a[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
    __syncthreads();
    int ch = 0;
    for (int i = 0; i < p.nitems; ++i) {
        const TrajItem it = p.items[i];
        const double2* M = p.pool + it.mat;
        if (it.type == 0) {
            apply_mat(a, p.n, it, M, 1.0);
            __syncthreads();
            continue;
        }
        const int d2 = 1 << (2 * it.k);
        for (int ki = 0; ki < it.nmat; ++ki) {
            const double w = block_sum(branch_weight(a, p.n, it, M + ki * d2), red);
            if (threadIdx.x == 0) s_w[ki] = w;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double total = 0.0;
            for (int ki = 0; ki < it.nmat; ++ki) total += s_w[ki];
            if (fabs(total - 1.0) > 1e-8) atomicExch(p.err, 1);
            const double u = p.uniforms[b * p.nchannels + ch] * total;
            int chosen = it.nmat - 1;
            double cum = 0.0;
            for (int ki = 0; ki < it.nmat; ++ki) {
                cum += s_w[ki];
                if (u < cum) {
                    chosen = ki;
                    break;
                }
            }
            s_sel = chosen;
            s_scale = 1.0 / sqrt(s_w[chosen]);
            if (p.branch_out) p.branch_out[b * p.nchannels + ch] = chosen;
        }
        __syncthreads();
        apply_mat(a, p.n, it, M + s_sel * d2, s_scale);
        __syncthreads();
        ++ch;
    }
    // Pauli expectations (statevector.cpp:241-277), before the i^ny factor
    for (int t = 0; t < p.nterms; ++t) {
        const uint64_t F = p.flip[t], S = p.signs[t];
        double re = 0.0, im = 0.0;
        for (uint32_t y = threadIdx.x; y < dim; y += blockDim.x) {
            const double2 ay = a[y], az = a[y ^ uint32_t(F)];
            // conj(az) * ay
            double xr = az.x * ay.x + az.y * ay.y, xi = az.x * ay.y - az.y * ay.x;
            if (__popcll(uint64_t(y) & S) & 1) {
                xr = -xr;
                xi = -xi;
            }
            re += xr;
            im += xi;
        }
        re = block_sum(re, red);
        im = block_sum(im, red);
        if (threadIdx.x == 0) {
            p.out_re[b * p.nterms + t] = re;
            p.out_im[b * p.nterms + t] = im;
        }
    }
    if (p.amps_out) {
        for (uint32_t i = threadIdx.x; i < dim; i += blockDim.x) p.amps_out[size_t(b) * dim + i] = a[i];
    }
}

__global__ void __launch_bounds__(kTrajThreads) k_batch(BatchArgs p) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* a = reinterpret_cast<double2*>(smem);
    __shared__ double red[kTrajThreads / 32];
    const int64_t b = blockIdx.x;
    const uint32_t dim = 1u << p.bits;
    for (uint32_t i = threadIdx.x; i < dim; i += blockDim.x) a[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
    __syncthreads();
    for (int64_t i = p.prog_off[b]; i < p.prog_off[b + 1]; ++i) {
        const TrajItem it = p.items[i];
        apply_mat(a, p.bits, it, p.pool + it.mat, 1.0);
        __syncthreads();
    }
    const uint32_t dq = 1u << p.n;
    for (int t = 0; t < p.nterms; ++t) {
        const uint64_t F = p.flip[t], S = p.signs[t];
        double re = 0.0, im = 0.0;
        for (uint32_t y = threadIdx.x; y < dq; y += blockDim.x) {
            double xr, xi;
            if (p.dm) {
                // rho[y, y ^ F] (densitymatrix.cpp:196-218), row-major vec index
                const double2 v = a[(y << p.n) | (y ^ uint32_t(F))];
                xr = v.x;
                xi = v.y;
            } else {
                const double2 ay = a[y], az = a[y ^ uint32_t(F)];
                xr = az.x * ay.x + az.y * ay.y;
                xi = az.x * ay.y - az.y * ay.x;
            }
            if (__popcll(uint64_t(y) & S) & 1) {
                xr = -xr;
                xi = -xi;
            }
            re += xr;
            im += xi;
        }
        re = block_sum(re, red);
        im = block_sum(im, red);
        if (threadIdx.x == 0) {
            p.out_re[b * p.nterms + t] = re;
            p.out_im[b * p.nterms + t] = im;
        }
    }
    if (p.probs) {
        double* out = p.probs + size_t(b) * dq;
        if (p.dm) {
            // max(0, Re rho_ii) / sequential sum (densitymatrix.cpp:221-232)
            if (threadIdx.x == 0) {
                double sum = 0.0;
                for (uint32_t i = 0; i < dq; ++i) {
                    const double v = fmax(0.0, a[(i << p.n) | i].x);
                    out[i] = v;
                    sum += v;
                }
                for (uint32_t i = 0; i < dq; ++i) out[i] /= sum;
            }
        } else {
            for (uint32_t i = threadIdx.x; i < dq; i += blockDim.x) out[i] = a[i].x * a[i].x + a[i].y * a[i].y;
        }
    }
}

}  // namespace

void launch_batch(const BatchArgs& p, int64_t batch, cudaStream_t s) {
    const size_t smem = (size_t(16) << p.bits);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_batch<<<unsigned(batch), kTrajThreads, smem, s>>>(p);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_traj(const TrajArgs& p, int64_t ntraj, cudaStream_t s) {
    const size_t smem = (size_t(16) << p.n);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_traj, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_traj<<<unsigned(ntraj), kTrajThreads, smem, s>>>(p);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace nqe

// Pack / unpack of the half-shard exchanged when a global qubit is swapped
// with local qubit v (shard.cpp): element k of the half is the local index
// with bit v forced to `val` and the other bits taken from k.
#include "kernels.hpp"

namespace nqe {

namespace {

__device__ __forceinline__ uint64_t ins_bit(uint64_t k, int v, uint64_t val) {
    return ((k >> v) << (v + 1)) | (val << v) | (k & ((uint64_t(1) << v) - 1));
}

__global__ void k_half_pack(const double2* __restrict__ st, double2* __restrict__ buf, uint64_t k0, uint64_t len,
                            int v, uint64_t val) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += uint64_t(gridDim.x) * blockDim.x)
        buf[i] = __ldcs(st + ins_bit(k0 + i, v, val));
}

__global__ void k_half_unpack(double2* __restrict__ st, const double2* __restrict__ buf, uint64_t k0, uint64_t len,
                              int v, uint64_t val) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += uint64_t(gridDim.x) * blockDim.x)
        __stcs(st + ins_bit(k0 + i, v, val), buf[i]);
}

// In-place swap over peer memory (NVLink, CUDA IPC mapping): for k in
// [k0, k1), mine[ins(k, v, mval)] <-> peer[ins(k, v, pval)].  The two ranks of
// a pair cover disjoint k ranges, so every element pair is touched by exactly
// one kernel.  Each thread keeps 4 pairs in flight (remote loads are ~1-2 us).
__global__ void __launch_bounds__(256) k_swap_peer(double2* __restrict__ mine, double2* __restrict__ peer, int v,
                                                   uint64_t mval, uint64_t pval, uint64_t k0, uint64_t k1) {
    constexpr int U = 4;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t base = k0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; base < k1; base += stride * U) {
        double2 x[U], y[U];
        uint64_t im[U], ip[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t k = base + uint64_t(u) * stride;
            if (k < k1) {
                im[u] = ins_bit(k, v, mval);
                ip[u] = ins_bit(k, v, pval);
                x[u] = __ldcs(mine + im[u]);
                y[u] = __ldcg(peer + ip[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t k = base + uint64_t(u) * stride;
            if (k < k1) {
                __stcs(mine + im[u], y[u]);
                __stcg(peer + ip[u], x[u]);
            }
        }
    }
}

unsigned grid_of(uint64_t len) {
    const uint64_t g = (len + 255) / 256;
    return unsigned(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

}  // namespace

void launch_half_pack(const double2* st, double2* buf, uint64_t k0, uint64_t len, int v, uint64_t val,
                      cudaStream_t s) {
    k_half_pack<<<grid_of(len), 256, 0, s>>>(st, buf, k0, len, v, val);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_half_unpack(double2* st, const double2* buf, uint64_t k0, uint64_t len, int v, uint64_t val,
                        cudaStream_t s) {
    k_half_unpack<<<grid_of(len), 256, 0, s>>>(st, buf, k0, len, v, val);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_swap_peer(double2* mine, double2* peer, int v, uint64_t mval, uint64_t pval, uint64_t k0, uint64_t k1,
                      cudaStream_t s) {
    if (k1 <= k0) return;
    k_swap_peer<<<148 * 8, 256, 0, s>>>(mine, peer, v, mval, pval, k0, k1);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace nqe

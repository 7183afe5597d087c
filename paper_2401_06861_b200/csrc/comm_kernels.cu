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

}  // namespace nqe

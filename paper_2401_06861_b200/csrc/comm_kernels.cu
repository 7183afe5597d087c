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

// Staged exchange pusher (shard.cpp, JitXStore::staged): one persistent
// grid on the SMs the exchange pass leaves free.  Chunk by chunk, once this
// rank's pass and the partner's pass have stored every tile of the chunk
// (pass_done counters; the partner's is read over NVLink, so the partner has
// also consumed its own copy of those positions), the chunk's staging slot
// is copied into the partner's state: slot index k expands to the physical
// index with the chunk bits and v re-inserted (v = the partner-side value),
// consecutive k -> consecutive addresses on both sides.
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(256) k_stage_push(const double2* __restrict__ stage, double2* __restrict__ peer,
                                                    const unsigned* my_done, const unsigned* peer_done,
                                                    unsigned* push_done, StagePush sp) {
    for (int c = 0; c < sp.chunks; ++c) {
        if (threadIdx.x == 0 && ld_acq(push_done + sp.err_index) == 0u) {
            // bounded waits (60 s): a stalled partner is recorded and reported
            // by the host, not hung on (no further waits once recorded)
            const unsigned long long t0 = gtimer();
            while (ld_acq(my_done + c) < sp.tiles_per_chunk)
                if (gtimer() - t0 > 60000000000ull) {
                    atomicMax(push_done + sp.err_index, 0x10000u + unsigned(c));
                    break;
                }
            while (ld_acq(peer_done + c) < sp.tiles_per_chunk)
                if (gtimer() - t0 > 60000000000ull) {
                    atomicMax(push_done + sp.err_index, 0x20000u + unsigned(c));
                    break;
                }
        }
        __syncthreads();
        // index bits contributed by the chunk number and v: fixed per chunk
        const double2* src = stage + uint64_t(c % sp.slots) * sp.slot_elems;
        const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
        for (uint64_t k0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k0 < sp.slot_elems; k0 += 4 * stride) {
            double2 x[4];
            uint64_t o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t k = k0 + uint64_t(u) * stride;
                if (k < sp.slot_elems) {
                    x[u] = __ldcs(src + k);
                    uint64_t w = k;
                    for (int j = 0; j < sp.nholes; ++j) {  // ascending hole positions
                        const int h = sp.hole_pos[j];
                        const uint64_t bit = sp.hole_src[j] < 0 ? sp.vval : (uint64_t(c) >> sp.hole_src[j]) & 1u;
                        w = ((w >> h) << (h + 1)) | (bit << h) | (w & ((uint64_t(1) << h) - 1));
                    }
                    o[u] = w;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t k = k0 + uint64_t(u) * stride;
                if (k < sp.slot_elems) __stcs(peer + o[u], x[u]);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            atomicAdd(push_done + c, 1u);
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

void preload_stage_push() {
    // see jit_xstore_prepare: kernels that spin on each other must both be
    // loaded before either is launched (CUDA lazy loading)
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(&k_stage_push));
    cudaGetLastError();
}

void launch_stage_push(const double2* stage, double2* peer, const unsigned* my_done, const unsigned* peer_done,
                       unsigned* push_done, const StagePush& sp, int ctas, cudaStream_t s) {
    k_stage_push<<<ctas, 256, 0, s>>>(stage, peer, my_done, peer_done, push_done, sp);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace nqe

// Two-GPU in-place half-shard swap over NVLink peer memory (the exchange of
// shard.cpp), variants of the k_swap_peer kernel.  One process, two devices.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t ins_bit(uint64_t k, int v, uint64_t val) {
    return ((k >> v) << (v + 1)) | (val << v) | (k & ((uint64_t(1) << v) - 1));
}

template <int U, bool CS>
__global__ void __launch_bounds__(256) k_swap(double2* mine, double2* peer, int v, uint64_t mval, uint64_t pval,
                                              uint64_t k0, uint64_t k1) {
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
                y[u] = CS ? __ldcs(peer + ip[u]) : __ldcg(peer + ip[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t k = base + uint64_t(u) * stride;
            if (k < k1) {
                __stcs(mine + im[u], y[u]);
                if (CS) __stcs(peer + ip[u], x[u]);
                else __stcg(peer + ip[u], x[u]);
            }
        }
    }
}

int main() {
    const int nloc = 30;
    const uint64_t count = uint64_t(1) << nloc, half = count / 2;
    double2* st[2];
    cudaStream_t s[2];
    cudaEvent_t e0[2], e1[2];
    for (int d = 0; d < 2; ++d) {
        cudaSetDevice(d);
        cudaDeviceEnablePeerAccess(1 - d, 0);
        if (cudaMalloc(&st[d], count * 16) != cudaSuccess) return 1;
        cudaMemset(st[d], 0, count * 16);
        cudaStreamCreate(&s[d]);
        cudaEventCreate(&e0[d]);
        cudaEventCreate(&e1[d]);
    }
    const int v = 29;
    auto run = [&](auto kern, int grid, const char* name) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
            for (int d = 0; d < 2; ++d) {
                cudaSetDevice(d);
                const uint64_t mybit = uint64_t(d);
                const uint64_t k0 = mybit ? half / 2 : 0, k1 = mybit ? half : half / 2;
                cudaEventRecord(e0[d], s[d]);
                kern<<<grid, 256, 0, s[d]>>>(st[d], st[1 - d], v, 1 - mybit, mybit, k0, k1);
                cudaEventRecord(e1[d], s[d]);
            }
            float ms = 0;
            for (int d = 0; d < 2; ++d) {
                cudaSetDevice(d);
                cudaEventSynchronize(e1[d]);
                float t;
                cudaEventElapsedTime(&t, e0[d], e1[d]);
                ms = t > ms ? t : ms;
            }
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-28s grid %5d: %.2f ms  %.0f GB/s per direction\n", name, grid, best, half * 16.0 / best / 1e6);
    };
    for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        run(k_swap<4, false>, g, "U4 ldcg/stcg");
        run(k_swap<8, false>, g, "U8 ldcg/stcg");
        run(k_swap<4, true>, g, "U4 cs");
    }
    return 0;
}

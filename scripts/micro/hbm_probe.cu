// HBM streaming probes for the pass roofline: copy (A -> B) vs in-place
// read-modify-write of the same 16 GiB array (what every fused pass does),
// 16-byte accesses, grid-stride, several unroll depths.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        __stcs(b + i, __ldcs(a + i));
}

template <int U>
__global__ void k_inplace(double2* __restrict__ a, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += stride * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u].x *= 1.0000000001;
            if (i + u * stride < n) __stcs(a + i + u * stride, v[u]);
        }
    }
}

template <class F>
float timeit(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    const size_t n = size_t(1) << 30;  // 16 GiB of double2
    double2 *a, *b;
    if (cudaMalloc(&a, n * 16) != cudaSuccess || cudaMalloc(&b, n * 16) != cudaSuccess) return 1;
    cudaMemset(a, 0, n * 16);
    cudaMemset(b, 0, n * 16);
    const double bytes = 2.0 * 16.0 * double(n);
    for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        float ms = timeit([&] { k_copy<<<g, 256>>>(a, b, n); });
        printf("copy      grid %5d x256: %.3f ms  %.0f GB/s\n", g, ms, bytes / ms / 1e6);
    }
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
        float ms1 = timeit([&] { k_inplace<1><<<g, 256>>>(a, n); });
        float ms4 = timeit([&] { k_inplace<4><<<g, 256>>>(a, n); });
        float ms16 = timeit([&] { k_inplace<16><<<g, 128>>>(a, n); });
        printf("inplace   grid %5d: U1 %.0f GB/s, U4 %.0f GB/s, U16(128 thr) %.0f GB/s\n", g, bytes / ms1 / 1e6,
               bytes / ms4 / 1e6, bytes / ms16 / 1e6);
    }
    return 0;
}

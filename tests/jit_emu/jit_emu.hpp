// Host emulation of the CUDA subset the generated pass kernels use
// (test infrastructure: tests/jit_emu.py).  One CTA runs at a time as T
// std::threads; __syncthreads is a std::barrier; the dynamic shared memory is
// one static buffer.  Memory primitives are in pass_ops.cuh (#ifdef NQ_EMU).
#pragma once

#include <barrier>
#include <cmath>

struct double2 {
    double x, y;
};
inline double2 make_double2(double x, double y) { return {x, y}; }
using std::fma;

#define __device__
#define __forceinline__ inline
#define __global__
#define __launch_bounds__(...)
#define __align__(n) __attribute__((aligned(n)))
#define __shared__

inline int __popc(unsigned v) { return __builtin_popcount(v); }

struct EmuDim {
    unsigned x, y, z;
};
extern thread_local EmuDim threadIdx;
extern thread_local EmuDim blockIdx;
extern EmuDim gridDim;
extern EmuDim blockDim;
extern std::barrier<>* emu_barrier;
inline void __syncthreads() { emu_barrier->arrive_and_wait(); }
inline int __popcll(unsigned long long v) { return __builtin_popcountll(v); }

// Warp shuffles for the fused-expectation epilogue: every thread of the CTA
// calls them uniformly there, so a CTA-wide exchange through a shared array
// (two barriers) emulates the warp-synchronous shuffle.
extern double emu_shfl[1024];
inline double __shfl_down_sync(unsigned, double v, int o) {
    const unsigned t = threadIdx.x;
    emu_shfl[t] = v;
    __syncthreads();
    const double r = ((t & 31u) + unsigned(o) < 32u && t + unsigned(o) < blockDim.x) ? emu_shfl[t + unsigned(o)] : v;
    __syncthreads();
    return r;
}

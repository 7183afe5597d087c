// Register-resident micro-op building blocks of the fused pass kernel.
//
// Shared by the interpreter kernel (pass_kernel.cu) and the pass-specialised
// kernels generated at run time (jit.cpp compiles this header with NVRTC).
// Self-contained: no includes, only CUDA built-ins.
//
// A thread holds E = 2^R amplitudes a[l]; bit j of l is register slot j.
// Every operator takes its slots as template arguments, so amplitudes stay in
// registers; operator matrices are read from shared memory at the point of use.
#pragma once

#ifdef NQ_EMU
#include "jit_emu.hpp"
#endif

namespace nq {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ bool is_one(double2 f) { return f.x == 1.0 && f.y == 0.0; }

#ifndef NQ_EMU
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// 256-bit streaming pair access (LDG/STG.E.ENL2.256, sm_100): two amplitudes
// adjacent in memory (a register slot on physical bit 0) in one 32-byte sector
// (NQ_NO_V4: two 128-bit accesses, for an NVRTC older than 12.9)
__device__ __forceinline__ void ld_stream2(const double2* p, double2& a, double2& b) {
#ifdef NQ_NO_V4
    a = ld_stream(p);
    b = ld_stream(p + 1);
#else
    asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
                 : "l"(p));
#endif
}
__device__ __forceinline__ void st_stream2(double2* p, double2 a, double2 b) {
#ifdef NQ_NO_V4
    st_stream(p, a);
    st_stream(p + 1, b);
#else
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
#endif
}
// Acquire load of a 32-bit counter (staged exchanges: another kernel, or the
// partner GPU over NVLink, increments it)
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Nanosecond clock (watchdogs of the staged exchange waits)
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Bounded wait until *p >= want (acquire): false after `ns` without progress
// (the caller records the failure instead of hanging the device)
__device__ __forceinline__ bool wait_at_least(const unsigned* p, unsigned want, unsigned long long ns) {
    if (ld_acquire_u32(p) >= want) return true;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_u32(p) < want)
        if (globaltimer_ns() - t0 > ns) return false;
    return true;
}
// Pusher role of a staged exchange pass (shard.cpp, jit.cpp): the last CTAs
// of the (cooperatively launched, so co-resident) grid.  Chunk by chunk, once
// this rank and the partner have stored every tile of the chunk (pass_done
// counters; the partner's read over NVLink, so the partner has consumed its
// own copy of those positions), the chunk's staging slot is copied into the
// partner's state: slot index k expands to the physical index with the holes
// re-inserted (Expand: generated per pass, the hole positions are constants;
// the chunk's own bits and v come in through `fixed`), so consecutive k are
// consecutive addresses on both sides.  Waits are bounded: a stall is
// recorded in *err and reported by the host.
template <int U, class Expand>
__device__ __forceinline__ void stage_push_role(unsigned pid, unsigned npush, const double2* stage, double2* peer,
                                                const unsigned* my_done, const unsigned* peer_done,
                                                unsigned* push_done, unsigned* err, int chunks, int slots,
                                                unsigned tpc, unsigned long long slot_elems,
                                                unsigned long long watchdog_ns, Expand expand) {
    const unsigned tid = threadIdx.x, nt = blockDim.x;
    const unsigned long long stride = (unsigned long long)npush * nt;
    for (int c = 0; c < chunks; ++c) {
        if (tid == 0 && ld_acquire_u32(err) == 0u) {
            if (!wait_at_least(my_done + c, tpc, watchdog_ns)) atomicMax(err, 0x10000u + unsigned(c));
            else if (!wait_at_least(peer_done + c, tpc, watchdog_ns)) atomicMax(err, 0x20000u + unsigned(c));
        }
        __syncthreads();
        const double2* src = stage + (unsigned long long)(c % slots) * slot_elems;
        // U loads in flight per thread: the copy is bound by local-read
        // latency x bytes in flight unless that exceeds what NVLink takes
        for (unsigned long long k0 = (unsigned long long)pid * nt + tid; k0 < slot_elems; k0 += U * stride) {
            double2 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned long long k = k0 + (unsigned long long)u * stride;
                if (k < slot_elems) x[u] = ld_stream(src + k);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned long long k = k0 + (unsigned long long)u * stride;
                if (k < slot_elems) st_stream(peer + expand(k, c), x[u]);
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence_system();
            atomicAdd(push_done + c, 1u);
        }
    }
}
// Shared-memory load the compiler may not hoist: matrices are re-read (one
// broadcast LDS per entry) instead of occupying registers.
__device__ __forceinline__ double2 lds(const double2* p) {
    double2 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

// Swizzle of the relayout buffer: conflict-free LDS/STS.128 when the three
// lowest thread bits of a layout have distinct residues mod 3.
__device__ __forceinline__ unsigned swz(unsigned e) { return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9)) & 7u); }

// 16-byte global -> shared asynchronous copy (LDGSTS), bypassing L1.
__device__ __forceinline__ void cp_async16(double2* smem_dst, const double2* gsrc) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
#else
// Host emulation of the memory primitives (tests/jit_emu.py runs generated
// pass kernels on CPU threads against the oracle; NQ_EMU builds only).
__device__ __forceinline__ double2 ld_stream(const double2* p) { return *p; }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { *p = v; }
__device__ __forceinline__ void ld_stream2(const double2* p, double2& a, double2& b) {
    a = p[0];
    b = p[1];
}
__device__ __forceinline__ void st_stream2(double2* p, double2 a, double2 b) {
    p[0] = a;
    p[1] = b;
}
__device__ __forceinline__ double2 lds(const double2* p) { return *p; }
#endif

// a <- diag factor f, skipping exact ones (d0 = 1 diagonals touch half the amplitudes)
__device__ __forceinline__ double2 dmul(double2 a, double2 f) { return is_one(f) ? a : cmul(f, a); }

// Matrix-entry products; R = true when the pass compiler proved every entry of
// the matrix real (H, RY and their products): half the FP64 work.
template <bool R>
__device__ __forceinline__ double2 mmul(double2 u, double2 x) {
    if constexpr (R) return make_double2(u.x * x.x, u.x * x.y);
    else return cmul(u, x);
}
template <bool R>
__device__ __forceinline__ double2 mfma(double2 u, double2 x, double2 acc) {
    if constexpr (R) return make_double2(fma(u.x, x.x, acc.x), fma(u.x, x.y, acc.y));
    else return cfma(u, x, acc);
}

template <int E, int J, bool R = false>
__device__ __forceinline__ void d1(double2 (&a)[E], const double2* u) {
    const double2 u00 = lds(u), u01 = lds(u + 1), u10 = lds(u + 2), u11 = lds(u + 3);
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if ((l >> J) & 1) continue;
        const int h = l | (1 << J);
        const double2 x0 = a[l], x1 = a[h];
        a[l] = mfma<R>(u00, x0, mmul<R>(u01, x1));
        a[h] = mfma<R>(u10, x0, mmul<R>(u11, x1));
    }
}

// d1 / d2 on registers that hold a pending X permutation (jit.cpp: the
// true amplitude of register l is a[l ^ px]): the operator conjugated by
// that X, i.e. entry e read at e ^ f (f = 3 p for k = 1, 5 p for k = 2 with p
// the pending bits of the operator's slots).
template <int E, int J, bool R = false>
__device__ __forceinline__ void d1f(double2 (&a)[E], const double2* u, unsigned f) {
    const double2 u00 = lds(u + f), u01 = lds(u + (1u ^ f)), u10 = lds(u + (2u ^ f)), u11 = lds(u + (3u ^ f));
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if ((l >> J) & 1) continue;
        const int h = l | (1 << J);
        const double2 x0 = a[l], x1 = a[h];
        a[l] = mfma<R>(u00, x0, mmul<R>(u01, x1));
        a[h] = mfma<R>(u10, x0, mmul<R>(u11, x1));
    }
}

template <int E, int J0, int J1, bool R = false>
__device__ __forceinline__ void d2f(double2 (&a)[E], const double2* u, unsigned f) {
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if (((l >> J0) & 1) || ((l >> J1) & 1)) continue;
        const int i0 = l, i1 = l | (1 << J0), i2 = l | (1 << J1), i3 = l | (1 << J0) | (1 << J1);
        const double2 x0 = a[i0], x1 = a[i1], x2 = a[i2], x3 = a[i3];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const unsigned e = 4u * unsigned(r);
            double2 acc = mmul<R>(lds(u + (e ^ f)), x0);
            acc = mfma<R>(lds(u + ((e + 1u) ^ f)), x1, acc);
            acc = mfma<R>(lds(u + ((e + 2u) ^ f)), x2, acc);
            acc = mfma<R>(lds(u + ((e + 3u) ^ f)), x3, acc);
            a[r == 0 ? i0 : r == 1 ? i1 : r == 2 ? i2 : i3] = acc;
        }
    }
}

template <int E, int J0, int J1, bool R = false>
__device__ __forceinline__ void d2(double2 (&a)[E], const double2* u) {
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if (((l >> J0) & 1) || ((l >> J1) & 1)) continue;
        const int i0 = l, i1 = l | (1 << J0), i2 = l | (1 << J1), i3 = l | (1 << J0) | (1 << J1);
        const double2 x0 = a[i0], x1 = a[i1], x2 = a[i2], x3 = a[i3];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double2 acc = mmul<R>(lds(u + 4 * r), x0);
            acc = mfma<R>(lds(u + 4 * r + 1), x1, acc);
            acc = mfma<R>(lds(u + 4 * r + 2), x2, acc);
            acc = mfma<R>(lds(u + 4 * r + 3), x3, acc);
            a[r == 0 ? i0 : r == 1 ? i1 : r == 2 ? i2 : i3] = acc;
        }
    }
}

// k = 3 on all slots except `Skip` (local bit order = ascending slots).
template <int E, int Skip, bool R = false>
__device__ __forceinline__ void d3(double2 (&a)[E], const double2* u) {
    constexpr int J0 = Skip == 0 ? 1 : 0;
    constexpr int J1 = Skip <= 1 ? 2 : 1;
    constexpr int J2 = Skip <= 2 ? 3 : 2;
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if ((l >> J0) & 1 || (l >> J1) & 1 || (l >> J2) & 1) continue;
        double2 x[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = a[l | ((c & 1) << J0) | (((c >> 1) & 1) << J1) | (((c >> 2) & 1) << J2)];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double2 acc = mmul<R>(lds(u + 8 * r), x[0]);
#pragma unroll
            for (int c = 1; c < 8; ++c) acc = mfma<R>(lds(u + 8 * r + c), x[c], acc);
            a[l | ((r & 1) << J0) | (((r >> 1) & 1) << J1) | (((r >> 2) & 1) << J2)] = acc;
        }
    }
}

// k = 4 on all slots: inputs parked in this thread's private scratch row.
template <int E, bool R = false>
__device__ __forceinline__ void d4(double2 (&a)[E], const double2* u, double2* scratch) {
    if constexpr (E == 16) {
#pragma unroll
        for (int c = 0; c < 16; ++c) scratch[c] = a[c];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            double2 acc = mmul<R>(lds(u + 16 * r), lds(scratch));
#pragma unroll
            for (int c = 1; c < 16; ++c) acc = mfma<R>(lds(u + 16 * r + c), lds(scratch + c), acc);
            a[r] = acc;
        }
    }
}

// X on slot J for the amplitudes whose register-slot controls CML are set.
template <int E, int J>
__device__ __forceinline__ void xperm(double2 (&a)[E], unsigned cmL) {
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if ((l >> J) & 1) continue;
        if ((unsigned(l) & cmL) == cmL) {
            const double2 t = a[l];
            a[l] = a[l | (1 << J)];
            a[l | (1 << J)] = t;
        }
    }
}

template <int E, int J0, int J1>
__device__ __forceinline__ void swp(double2 (&a)[E]) {
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if (((l >> J0) & 1) && !((l >> J1) & 1)) {
            const int o = (l & ~(1 << J0)) | (1 << J1);
            const double2 t = a[l];
            a[l] = a[o];
            a[o] = t;
        }
    }
}

// 1-qubit depolarizing in Liouville form on slots {J0, J1} (column, row bit).
template <int E, int J0, int J1>
__device__ __forceinline__ void dep2(double2 (&a)[E], double al, double be) {
#pragma unroll
    for (int l = 0; l < E; ++l) {
        if (((l >> J0) & 1) || ((l >> J1) & 1)) continue;
        const int d = l | (1 << J0) | (1 << J1);
        const double tr = a[l].x + a[d].x, ti = a[l].y + a[d].y;
        a[l] = make_double2(fma(al, a[l].x, be * tr), fma(al, a[l].y, be * ti));
        a[d] = make_double2(fma(al, a[d].x, be * tr), fma(al, a[d].y, be * ti));
        a[l | (1 << J0)] = make_double2(al * a[l | (1 << J0)].x, al * a[l | (1 << J0)].y);
        a[l | (1 << J1)] = make_double2(al * a[l | (1 << J1)].x, al * a[l | (1 << J1)].y);
    }
}

// 2-qubit depolarizing on all 4 slots; slot 0 is paired with slot P (1..3).
template <int E, int P>
__device__ __forceinline__ void dep4(double2 (&a)[E], double al, double be) {
    if constexpr (E == 16) {
        constexpr int Q0 = P == 1 ? 2 : 1;
        constexpr int Q1 = P == 3 ? 2 : 3;
        double tr = 0.0, ti = 0.0;
#pragma unroll
        for (int l = 0; l < 16; ++l) {
            if ((((l >> 0) & 1) == ((l >> P) & 1)) && (((l >> Q0) & 1) == ((l >> Q1) & 1))) {
                tr += a[l].x;
                ti += a[l].y;
            }
        }
#pragma unroll
        for (int l = 0; l < 16; ++l) {
            const bool dg = (((l >> 0) & 1) == ((l >> P) & 1)) && (((l >> Q0) & 1) == ((l >> Q1) & 1));
            a[l] = dg ? make_double2(fma(al, a[l].x, be * tr), fma(al, a[l].y, be * ti))
                      : make_double2(al * a[l].x, al * a[l].y);
        }
    }
}

}  // namespace nq

// Runner for generated pass kernels on the host (see jit_emu.hpp).  The
// generated sources are concatenated after this file with their entry points
// renamed nqjit_<i>; emu_run(i, ...) launches pass i as one CTA of T threads
// whose grid-stride loop covers every tile.
#include "pass_ops.cuh"

#include <new>
#include <thread>
#include <vector>

thread_local EmuDim threadIdx;
thread_local EmuDim blockIdx;
EmuDim gridDim{1, 1, 1};
EmuDim blockDim{1, 1, 1};
std::barrier<>* emu_barrier = nullptr;
// the CTA's dynamic shared memory, allocated per launch at exactly the size
// the launch would request (so an address sanitizer build sees overruns)
unsigned char* emu_smem = nullptr;
double emu_shfl[1024];
// partial sums of a fused-expectation epilogue (tests/jit_emu.py run(zterms=...))
double* emu_epart = nullptr;
extern "C" void emu_set_epart(double* p) { emu_epart = p; }

typedef void (*emu_kernel)(double2*, const double2*, unsigned long long, long long, double2*, double2*,
                           unsigned long long, unsigned long long, int);
extern emu_kernel emu_table[];

extern "C" int emu_run(int pass, double* state, const double* pool, long long ntiles, int threads,
                       long long smem_bytes) {
    emu_smem = static_cast<unsigned char*>(::operator new[](size_t(smem_bytes), std::align_val_t(16)));
    std::barrier<> bar(threads);
    emu_barrier = &bar;
    blockDim.x = unsigned(threads);
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t)
        ts.emplace_back([=] {
            threadIdx = EmuDim{unsigned(t), 0, 0};
            blockIdx = EmuDim{0, 0, 0};
            emu_table[pass](reinterpret_cast<double2*>(state), reinterpret_cast<const double2*>(pool), 0ull, ntiles,
                            nullptr, nullptr, 0ull, 0ull, 0);
        });
    for (auto& t : ts) t.join();
    emu_barrier = nullptr;
    ::operator delete[](emu_smem, std::align_val_t(16));
    emu_smem = nullptr;
    return 0;
}

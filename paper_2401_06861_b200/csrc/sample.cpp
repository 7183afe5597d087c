// Sorted-uniform sampling sweep (K12; proj/src/statevector.cpp:293-332).
//
// The reference draws `shots` uniforms, sorts them, and walks the cumulative
// distribution once.  Here the walk is split in two levels so that no 2^n
// array ever reaches the host:
//   1. the device sums probabilities over fixed blocks of kBlock entries;
//   2. the host prefix-sums the block sums (sequentially, like the reference)
//      and assigns each sorted uniform to the block whose cumulative range
//      contains it;
//   3. one device thread per block that owns uniforms replays the reference's
//      sequential `cum += p[i]` sweep from the block's starting cumulative.
// Uniforms left over after the final cumulative (float round-off) go to the
// highest index with nonzero probability, as in statevector.cpp:321-330.
#include "kernels.hpp"
#include "state.hpp"

#include <algorithm>
#include <cstring>

namespace nqe {

namespace {
constexpr uint64_t kBlock = 4096;
}

void sample_sweep(DeviceCtx& c, const double2* a, const double* p, uint64_t n, const double* sorted_u,
                  uint64_t shots, uint64_t* idx_out, uint64_t* count_out, uint64_t* nout, double cum_start,
                  bool leftovers) {
    *nout = 0;
    if (shots == 0) return;
    CUDA_TRY(cudaSetDevice(c.dev));
    const uint64_t bs = std::min<uint64_t>(kBlock, n);
    const uint64_t nb = (n + bs - 1) / bs;
    double* d_bsum = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_bsum), nb * sizeof(double), c.stream));
    launch_block_psum(a, p, n, bs, d_bsum, c.stream);
    CUDA_TRY(cudaGetLastError());
    std::vector<double> bsum(nb);
    CUDA_TRY(cudaMemcpyAsync(bsum.data(), d_bsum, nb * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CUDA_TRY(cudaFreeAsync(d_bsum, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));

    // host: block prefix + uniform ownership
    std::vector<int64_t> blk, ulo, uhi;
    std::vector<double> cum0;
    double cum = cum_start;
    uint64_t next = 0;
    for (uint64_t b = 0; b < nb && next < shots; ++b) {
        const double start = cum;
        cum += bsum[b];
        const uint64_t lo = next;
        while (next < shots && sorted_u[next] < cum) ++next;
        if (next > lo) {
            blk.push_back(int64_t(b));
            cum0.push_back(start);
            ulo.push_back(int64_t(lo));
            uhi.push_back(int64_t(next));
        }
    }
    const int nbw = int(blk.size());
    std::vector<uint64_t> idx(shots), cnt(shots);
    std::vector<int64_t> npairs(size_t(nbw), 0);
    if (nbw > 0) {
        // one device allocation for all sweep inputs/outputs
        const size_t bytes = size_t(nbw) * (3 * sizeof(int64_t) + sizeof(double) + sizeof(int64_t)) +
                             shots * (sizeof(double) + 2 * sizeof(uint64_t)) + 256;
        unsigned char* dbuf = nullptr;
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dbuf), bytes, c.stream));
        unsigned char* at = dbuf;
        auto take = [&](size_t b) {
            unsigned char* r = at;
            at += (b + 15) & ~size_t(15);
            return r;
        };
        auto* d_blk = reinterpret_cast<int64_t*>(take(size_t(nbw) * 8));
        auto* d_ulo = reinterpret_cast<int64_t*>(take(size_t(nbw) * 8));
        auto* d_uhi = reinterpret_cast<int64_t*>(take(size_t(nbw) * 8));
        auto* d_cum0 = reinterpret_cast<double*>(take(size_t(nbw) * 8));
        auto* d_np = reinterpret_cast<int64_t*>(take(size_t(nbw) * 8));
        auto* d_u = reinterpret_cast<double*>(take(shots * 8));
        auto* d_idx = reinterpret_cast<uint64_t*>(take(shots * 8));
        auto* d_cnt = reinterpret_cast<uint64_t*>(take(shots * 8));
        CUDA_TRY(cudaMemcpyAsync(d_blk, blk.data(), size_t(nbw) * 8, cudaMemcpyHostToDevice, c.stream));
        CUDA_TRY(cudaMemcpyAsync(d_ulo, ulo.data(), size_t(nbw) * 8, cudaMemcpyHostToDevice, c.stream));
        CUDA_TRY(cudaMemcpyAsync(d_uhi, uhi.data(), size_t(nbw) * 8, cudaMemcpyHostToDevice, c.stream));
        CUDA_TRY(cudaMemcpyAsync(d_cum0, cum0.data(), size_t(nbw) * 8, cudaMemcpyHostToDevice, c.stream));
        CUDA_TRY(cudaMemcpyAsync(d_u, sorted_u, shots * 8, cudaMemcpyHostToDevice, c.stream));
        launch_block_sweep(a, p, n, bs, d_blk, d_cum0, d_ulo, d_uhi, d_u, nbw, d_idx, d_cnt, d_np, c.stream);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(npairs.data(), d_np, size_t(nbw) * 8, cudaMemcpyDeviceToHost, c.stream));
        CUDA_TRY(cudaMemcpyAsync(idx.data(), d_idx, shots * 8, cudaMemcpyDeviceToHost, c.stream));
        CUDA_TRY(cudaMemcpyAsync(cnt.data(), d_cnt, shots * 8, cudaMemcpyDeviceToHost, c.stream));
        CUDA_TRY(cudaFreeAsync(dbuf, c.stream));
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    }
    uint64_t k = 0;
    for (int b = 0; b < nbw; ++b) {
        for (int64_t j = 0; j < npairs[size_t(b)]; ++j) {
            const uint64_t i = idx[size_t(ulo[size_t(b)] + j)];
            const uint64_t ct = cnt[size_t(ulo[size_t(b)] + j)];
            if (k > 0 && idx_out[k - 1] == i) {
                count_out[k - 1] += ct;
            } else {
                idx_out[k] = i;
                count_out[k] = ct;
                ++k;
            }
        }
    }
    if (next < shots && leftovers) {
        // leftovers: last index with nonzero probability
        int64_t lastb = -1;
        for (uint64_t b = nb; b-- > 0;)
            if (bsum[b] > 0.0) {
                lastb = int64_t(b);
                break;
            }
        if (lastb >= 0) {
            uint64_t* d_last = nullptr;
            CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_last), 8, c.stream));
            const uint64_t lo = uint64_t(lastb) * bs, hi = std::min(n, lo + bs);
            launch_last_nonzero(a, p, lo, hi, d_last, c.stream);
            uint64_t last1 = 0;
            CUDA_TRY(cudaMemcpyAsync(&last1, d_last, 8, cudaMemcpyDeviceToHost, c.stream));
            CUDA_TRY(cudaFreeAsync(d_last, c.stream));
            CUDA_TRY(cudaStreamSynchronize(c.stream));
            if (last1 > 0) {
                const uint64_t i = last1 - 1;
                // keep ascending order: merge or insert
                uint64_t pos = k;
                while (pos > 0 && idx_out[pos - 1] > i) --pos;
                if (pos > 0 && idx_out[pos - 1] == i) {
                    count_out[pos - 1] += shots - next;
                } else {
                    for (uint64_t t = k; t > pos; --t) {
                        idx_out[t] = idx_out[t - 1];
                        count_out[t] = count_out[t - 1];
                    }
                    idx_out[pos] = i;
                    count_out[pos] = shots - next;
                    ++k;
                }
            }
        }
    }
    *nout = k;
}

}  // namespace nqe

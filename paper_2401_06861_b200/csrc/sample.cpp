// Sorted-uniform sampling sweep (K12; proj/src/statevector.cpp:293-332).
//
// The reference draws `shots` uniforms, sorts them, and walks the cumulative
// distribution once with a sequential `cum += dist[i]`.  The bins therefore
// depend on the ROUNDING of that sequential sum; a parallel scan rounds
// differently and can move a uniform that lies within an ulp of a boundary.
// This file reproduces the sequential sum bit for bit without a serial pass
// over 2^n entries and without a 2^n array on the host:
//
//   1. prepare: the device sums each block of kBlock entries (approximate, only
//      used to guess in which binade [2^k, 2^(k+1)) the running sum sits while
//      it crosses the block), then k_block_isum sums the block's exact integer
//      increments rint(p * 2^(52-k)) for that binade.  Inside one binade every
//      partial sum is a multiple of ulp = 2^(k-52), so fl(cum + p) =
//      cum + rint(p / ulp) * ulp exactly (no ties): integer sums are
//      associative, the rounding sequence is reproduced exactly.
//   2. walk (host, one step per block): from the exact start, a block whose
//      guessed binade is verified (cum in [2^k, 2^(k+1)) and cum + increments
//      < 2^(k+1)) advances by its integer sum; any other block (binade
//      crossing, tie, wrong guess, the zero start) is fetched and replayed with
//      the reference's own sequential adds on the host.  Result: the exact
//      cumulative value at every block end.
//   3. assign: a uniform u belongs to the first index i with u < cum_i, i.e.
//      to the block b with end_(b-1) <= u < end_b; one device thread per
//      owning block replays that block's sequential sweep from end_(b-1).
// Uniforms left over after the final cumulative (float round-off) go to the
// highest index with nonzero probability, as in statevector.cpp:321-330.
// Probabilities are |a|^2 = re*re + im*im without fused multiply-adds on both
// sides (std::norm), so device and host sums see identical terms.
#include "kernels.hpp"
#include "state.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

namespace nqe {

namespace {
constexpr uint64_t kBlock = 4096;
constexpr int kSkip = INT_MIN;
constexpr double kTwo53 = 9007199254740992.0;
constexpr int kFetchBatch = 256;  // special blocks fetched per round trip

// std::norm as the reference computes it (two rounded products, one rounded
// sum); volatile keeps the compiler from contracting it into an FMA.
inline double host_prob(double re, double im) {
    volatile double a = re * re;
    volatile double b = im * im;
    return a + b;
}

// k with x in [2^k, 2^(k+1)), x > 0 finite
inline int binade(double x) {
    int e = 0;
    std::frexp(x, &e);
    return e - 1;
}
}  // namespace

void seqcum_prepare(DeviceCtx& c, const double2* a, const double* p, uint64_t n, double approx_start, SeqCum& sc) {
    CUDA_TRY(cudaSetDevice(c.dev));
    sc.n = n;
    sc.bs = std::min<uint64_t>(kBlock, n);
    sc.nb = (n + sc.bs - 1) / sc.bs;
    const uint64_t nb = sc.nb;
    unsigned char* dbuf = nullptr;
    const size_t bytes = nb * (sizeof(double) + sizeof(int) + sizeof(unsigned long long) + sizeof(int)) + 64;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dbuf), bytes, c.stream));
    auto* d_bsum = reinterpret_cast<double*>(dbuf);
    auto* d_isum = reinterpret_cast<unsigned long long*>(d_bsum + nb);
    auto* d_kb = reinterpret_cast<int*>(d_isum + nb);
    auto* d_flags = d_kb + nb;
    launch_block_psum(a, p, n, sc.bs, d_bsum, c.stream);
    CUDA_TRY(cudaGetLastError());
    sc.bsum.assign(nb, 0.0);
    CUDA_TRY(cudaMemcpyAsync(sc.bsum.data(), d_bsum, nb * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    // binade guesses from the approximate prefix, with a relative margin far
    // above the gap between any two summation orders
    sc.kb.assign(nb, kSkip);
    double acc = approx_start;
    for (uint64_t b = 0; b < nb; ++b) {
        const double lo = acc * (1.0 - 1e-6), hi = (acc + sc.bsum[b]) * (1.0 + 1e-6);
        acc += sc.bsum[b];
        if (sc.bsum[b] == 0.0 || !(lo > 0x1p-900) || !std::isfinite(hi)) continue;
        const int klo = binade(lo), khi = binade(hi);
        if (klo == khi) sc.kb[b] = klo;
    }
    CUDA_TRY(cudaMemcpyAsync(d_kb, sc.kb.data(), nb * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    launch_block_isum(a, p, n, sc.bs, d_kb, d_isum, d_flags, c.stream);
    CUDA_TRY(cudaGetLastError());
    sc.isum.assign(nb, 0);
    sc.flags.assign(nb, 0);
    CUDA_TRY(cudaMemcpyAsync(sc.isum.data(), d_isum, nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             c.stream));
    CUDA_TRY(cudaMemcpyAsync(sc.flags.data(), d_flags, nb * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CUDA_TRY(cudaFreeAsync(dbuf, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
}

double seqcum_walk(DeviceCtx& c, const double2* a, const double* p, SeqCum& sc, double start) {
    const uint64_t nb = sc.nb, bs = sc.bs;
    sc.ends.assign(nb, 0.0);
    sc.replayed = 0;
    const size_t esz = a ? sizeof(double2) : sizeof(double);
    std::vector<unsigned char> buf;
    std::vector<uint64_t> fetched;  // blocks held in buf, in order
    size_t fpos = 0;
    auto is_special = [&](uint64_t b) { return sc.bsum[b] != 0.0 && (sc.kb[b] == kSkip || sc.flags[b] != 0); };
    // fetch block b plus the next special blocks (one synchronisation)
    auto fetch_from = [&](uint64_t b) {
        fetched.clear();
        fetched.push_back(b);
        for (uint64_t x = b + 1; x < nb && fetched.size() < size_t(kFetchBatch); ++x)
            if (is_special(x)) fetched.push_back(x);
        buf.resize(fetched.size() * bs * esz);
        for (size_t i = 0; i < fetched.size(); ++i) {
            const uint64_t lo = fetched[i] * bs, len = std::min(sc.n, lo + bs) - lo;
            const void* src = a ? static_cast<const void*>(a + lo) : static_cast<const void*>(p + lo);
            CUDA_TRY(cudaMemcpyAsync(buf.data() + i * bs * esz, src, len * esz, cudaMemcpyDeviceToHost, c.stream));
        }
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        fpos = 0;
    };
    double cum = start;
    for (uint64_t b = 0; b < nb; ++b) {
        if (sc.bsum[b] == 0.0) {  // all-zero block (a sum of non-negative terms): cum unchanged
            sc.ends[b] = cum;
            continue;
        }
        const int k = sc.kb[b];
        if (k != kSkip && sc.flags[b] == 0 && cum > 0.0 && binade(cum) == k) {
            const double ci = std::ldexp(cum, 52 - k);  // integer in [2^52, 2^53)
            const double tot = ci + double(sc.isum[b]);
            if (sc.isum[b] < (1ull << 53) && tot < kTwo53) {
                cum = std::ldexp(tot, k - 52);
                sc.ends[b] = cum;
                continue;
            }
        }
        // sequential replay of this block, exactly as the reference
        while (fpos < fetched.size() && fetched[fpos] < b) ++fpos;
        if (fpos >= fetched.size() || fetched[fpos] != b) fetch_from(b);
        const unsigned char* blk = buf.data() + fpos * bs * esz;
        const uint64_t len = std::min(sc.n, b * bs + bs) - b * bs;
        if (a) {
            const double* v = reinterpret_cast<const double*>(blk);
            for (uint64_t i = 0; i < len; ++i) cum += host_prob(v[2 * i], v[2 * i + 1]);
        } else {
            const double* v = reinterpret_cast<const double*>(blk);
            for (uint64_t i = 0; i < len; ++i) cum += v[i];
        }
        ++sc.replayed;
        sc.ends[b] = cum;
    }
    return cum;
}

void sample_assign(DeviceCtx& c, const double2* a, const double* p, const SeqCum& sc, double start,
                   const double* sorted_u, uint64_t shots, uint64_t* idx_out, uint64_t* count_out, uint64_t* nout,
                   bool leftovers) {
    *nout = 0;
    if (shots == 0) return;
    CUDA_TRY(cudaSetDevice(c.dev));
    const uint64_t nb = sc.nb, bs = sc.bs, n = sc.n;
    // uniform ownership from the exact block ends: block b owns
    // [end_(b-1), end_b) (first index with u < cum_i lies in b)
    std::vector<int64_t> blk, ulo, uhi;
    std::vector<double> cum0;
    uint64_t next = 0;
    double prev = start;
    for (uint64_t b = 0; b < nb && next < shots; ++b) {
        const uint64_t lo = next;
        while (next < shots && sorted_u[next] < sc.ends[b]) ++next;
        if (next > lo) {
            blk.push_back(int64_t(b));
            cum0.push_back(prev);
            ulo.push_back(int64_t(lo));
            uhi.push_back(int64_t(next));
        }
        prev = sc.ends[b];
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
    uint64_t k = 0, assigned = 0;
    for (int b = 0; b < nbw; ++b) {
        for (int64_t j = 0; j < npairs[size_t(b)]; ++j) {
            const uint64_t i = idx[size_t(ulo[size_t(b)] + j)];
            const uint64_t ct = cnt[size_t(ulo[size_t(b)] + j)];
            assigned += ct;
            if (k > 0 && idx_out[k - 1] == i) {
                count_out[k - 1] += ct;
            } else {
                idx_out[k] = i;
                count_out[k] = ct;
                ++k;
            }
        }
    }
    if (assigned != next)
        throw NqError{NQ_ERR_INTERNAL, "sampling sweep assigned " + std::to_string(assigned) + " of " +
                                           std::to_string(next) + " owned uniforms"};
    if (next < shots && leftovers) {
        // leftovers: last index with nonzero probability
        int64_t lastb = -1;
        for (uint64_t b = nb; b-- > 0;)
            if (sc.bsum[b] > 0.0) {
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

void sample_sweep(DeviceCtx& c, const double2* a, const double* p, uint64_t n, const double* sorted_u,
                  uint64_t shots, uint64_t* idx_out, uint64_t* count_out, uint64_t* nout) {
    *nout = 0;
    if (shots == 0) return;
    SeqCum sc;
    seqcum_prepare(c, a, p, n, 0.0, sc);
    seqcum_walk(c, a, p, sc, 0.0);
    sample_assign(c, a, p, sc, 0.0, sorted_u, shots, idx_out, count_out, nout, true);
}

}  // namespace nqe

// naqs-b200: the library's only random source.
//
// Sampling must reproduce the reference engine bit for bit, so this is the
// same published algorithm (xoshiro256++, Blackman & Vigna, with a SplitMix64
// seed expansion) behind the same interface as proj/include/naqs/rng.hpp.
#pragma once

#include <cstdint>

namespace naqs {

namespace rng_detail {
inline std::uint64_t rotate_left(std::uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }
inline std::uint64_t splitmix_finalize(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
} // namespace rng_detail

class Rng {
  public:
    explicit Rng(std::uint64_t seed) {
        std::uint64_t x = seed;
        for (int i = 0; i < 4; ++i) {
            x += 0x9E3779B97F4A7C15ULL;
            st_[i] = rng_detail::splitmix_finalize(x);
        }
    }

    std::uint64_t next_u64() {
        const std::uint64_t out = rng_detail::rotate_left(st_[0] + st_[3], 23) + st_[0];
        const std::uint64_t shifted = st_[1] << 17;
        st_[2] ^= st_[0];
        st_[3] ^= st_[1];
        st_[1] ^= st_[2];
        st_[0] ^= st_[3];
        st_[2] ^= shifted;
        st_[3] = rng_detail::rotate_left(st_[3], 45);
        return out;
    }

    /// 53 random mantissa bits, uniform on [0, 1).
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

    double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }

  private:
    std::uint64_t st_[4];
};

/// Independent sub-stream seed for stream index `stream` of `base`.
inline std::uint64_t derive_seed(std::uint64_t base, std::uint64_t stream) {
    return rng_detail::splitmix_finalize(base + 0x9E3779B97F4A7C15ULL * (stream + 1));
}

} // namespace naqs

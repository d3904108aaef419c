// Philox4x64-10 as used by numpy.random.Philox, and the depolarizing
// inverse CDF of sample_error (pkg/src/qsagms/channel.py:55-76).
//
// numpy's Philox(key=[seed, stream_id]) starts its 256-bit counter at 0 and
// increments it before producing each 4-word block, so block b of a stream
// uses counter (b + 1, 0, 0, 0); Generator.random() maps word w to
// (w >> 11) * 2^-53 and qubit q consumes word q.  The comparisons
// u >= t (t = 1 - eps, 1 - eps + eps/3, 1 - eps/3) are replaced by exact
// integer comparisons (w >> 11) >= ceil(t * 2^53), computed on the host.
#pragma once

#include <stdint.h>

namespace qsg {

constexpr uint64_t kPhM0 = 0xD2E7470EE14C6C93ull;
constexpr uint64_t kPhM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhW0 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kPhW1 = 0xBB67AE8584CAA73Bull;

struct U64x4 { uint64_t v[4]; };

__device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t key0, uint64_t key1)
{
    uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll  // fully unrolled: rolling the rounds measured 1-8% slower at p <= 0.04
    for (int r = 0; r < 10; ++r) {
        if (r) { key0 += kPhW0; key1 += kPhW1; }
        const uint64_t lo0 = kPhM0 * c0, hi0 = __umul64hi(kPhM0, c0);
        const uint64_t lo1 = kPhM1 * c2, hi1 = __umul64hi(kPhM1, c2);
        const uint64_t n0 = hi1 ^ c1 ^ key0, n2 = hi0 ^ c3 ^ key1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return U64x4{{c0, c1, c2, c3}};
}

// Inverse CDF of channel.py:70-75 (later masks override earlier ones).
// (The branch-free form n ^ (n >> 1), n = #thresholds <= k, measured 2.5%
// slower at p = 0.02.)
__device__ __forceinline__ uint8_t pauli_from_word(uint64_t w, uint64_t kx, uint64_t ky, uint64_t kz)
{
    const uint64_t k = w >> 11;
    uint8_t c = 0;
    if (k >= kx && k < ky) c = 1;  // X
    if (k >= ky && k < kz) c = 3;  // Y
    if (k >= kz) c = 2;            // Z
    return c;
}

}  // namespace qsg

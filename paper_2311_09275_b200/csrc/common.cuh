// common.cuh -- device-side building blocks shared by the libising kernels.
//
// Philox4x32-10 (Salmon et al., SC'11) with the 10 round keys precomputed on the
// host (they depend only on the seed), so each round is 2 IMAD.WIDE + 2 LOP3.
// Counter layout and stream ids are the contract of DESIGN.md §3.3.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ising {

enum : uint32_t { ST_INIT = 0, ST_PLANE = 1, ST_WORD_HI = 2, ST_WORD_LO = 3, ST_EXCH = 4, ST_ICM = 5,
                  ST_COLOUR = 6 };

struct RoundKeys {
    uint32_t k[20];  // (k0, k1) for rounds 0..9
};

inline RoundKeys make_round_keys(uint64_t seed)
{
    RoundKeys rk;
    uint32_t k0 = (uint32_t)(seed & 0xFFFFFFFFu), k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = k0;
        rk.k[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return rk;
}

__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        const RoundKeys &rk)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = hi0 ^ c3 ^ rk.k[2 * r + 1];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// 0x00000000 or 0xFFFFFFFF from the sign bit of byte `sel` of x (PRMT sign replicate).
template <int sel>
__device__ __forceinline__ uint32_t byte_sign_mask(uint32_t x)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "n"((8 + sel) * 0x1111));
    return r;
}

// Bit-sliced counter: add the 32 one-bit lanes of `a` into the vertical number c[0..L).
template <int L>
__device__ __forceinline__ void vadd(uint32_t (&c)[L], uint32_t a)
{
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const uint32_t t = c[l] & a;
        c[l] ^= a;
        a = t;
    }
}

}  // namespace ising

// bits_core.cuh -- shared machinery of the bit-packed (multi-spin-coded) sweep kernels:
// Philox for the PLANE contract with rounds 0-1 hoisted, the MSB-first lazy plane
// comparison, bit-sliced counters, and the fused parallel-tempering step of a copy
// held by a thread-block cluster.
#pragma once
#include <cooperative_groups.h>

#include "internal.h"

namespace ising {
namespace bits {

namespace cg = cooperative_groups;

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
constexpr int kCntLevels = 12;  // per-thread counter + 5 butterfly levels
constexpr int kQItemBytes = 20;

struct GridGeom {
    int32_t Lx, Ly, hx, half;
    uint32_t ymagic;
};

// Uniform (per CTA, per sweep) parts of Philox rounds 0-1 for counter
// (i, t, g, PLANE<<24 | j4).
struct PlaneUniform {
    uint32_t U0;    // lo(M1*g) ^ K0_1
    uint32_t L0r1;  // lo(M0*A),  A = hi(M1*g) ^ t ^ K0_0
    uint32_t H0r1;  // hi(M0*A)
};

__device__ __forceinline__ PlaneUniform plane_uniform(uint32_t g, uint32_t t, const RoundKeys &rk)
{
    const uint32_t H1g = __umulhi(kM1, g), L1g = kM1 * g;
    const uint32_t A = H1g ^ t ^ rk.k[0];
    PlaneUniform u;
    u.U0 = L1g ^ rk.k[2];
    u.L0r1 = kM0 * A;
    u.H0r1 = __umulhi(kM0, A);
    return u;
}

// Per-site parts: sA = hi(M0*i) ^ (PLANE<<24) ^ K1_0, sB = H0r1 ^ lo(M0*i) ^ K1_1.
__device__ __forceinline__ void plane_site(uint32_t i, const PlaneUniform &u, const RoundKeys &rk,
                                           uint32_t &sA, uint32_t &sB)
{
    const uint32_t H0 = __umulhi(kM0, i), L0 = kM0 * i;
    sA = H0 ^ (ST_PLANE << 24) ^ rk.k[1];
    sB = u.H0r1 ^ L0 ^ rk.k[3];
}

// Philox4x32-10 of counter (i, t, g, PLANE<<24 | j4) from the hoisted parts (rounds 2-9 in
// full; the round keys are kernel-uniform values the compiler keeps in uniform registers).
__device__ __forceinline__ uint4 philox_plane(uint32_t sA, uint32_t sB, uint32_t j4,
                                              const PlaneUniform &u, const RoundKeys &rk)
{
    const uint32_t X = sA ^ j4;  // round-0 output word 2 (j4 < 2^24)
    uint32_t c0 = __umulhi(kM1, X) ^ u.U0;
    uint32_t c1 = kM1 * X;
    uint32_t c2 = sB;
    uint32_t c3 = u.L0r1;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        const uint32_t lo0 = kM0 * c0, hi0 = __umulhi(kM0, c0);
        const uint32_t lo1 = kM1 * c2, hi1 = __umulhi(kM1, c2);
        const uint32_t n0 = hi1 ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = hi0 ^ c3 ^ rk.k[2 * r + 1];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// m ? a : b bitwise, as ONE lop3 (the compiler otherwise splits it when ~m is live)
__device__ __forceinline__ uint32_t mux(uint32_t m, uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(m), "r"(a), "r"(b));
    return r;
}

// Planes 4*j4 .. 4*j4+3 of the lazy MSB-first comparison.  Lanes in D have
// dE = 8 (m8 set) or dE = 4 (m8 clear); P4/P8 are the word type's planes.
__device__ __forceinline__ void plane_call(uint32_t sA, uint32_t sB, uint32_t j4, const PlaneUniform &u,
                                           const RoundKeys &rk, const uint32_t *P, uint32_t m8,
                                           uint32_t &D, uint32_t &acc)
{
    const uint4 w = philox_plane(sA, sB, j4, u, rk);
    const uint4 q4 = *reinterpret_cast<const uint4 *>(P + 4 * j4);
    const uint4 q8 = *reinterpret_cast<const uint4 *>(P + 64 + 4 * j4);
    const uint32_t t0 = mux(m8, q8.x, q4.x);
    const uint32_t y0 = D & ~w.x & t0;
    D &= ~(w.x ^ t0);
    const uint32_t t1 = mux(m8, q8.y, q4.y);
    const uint32_t y1 = D & ~w.y & t1;
    D &= ~(w.y ^ t1);
    acc |= y0 | y1;
    const uint32_t t2 = mux(m8, q8.z, q4.z);
    const uint32_t y2 = D & ~w.z & t2;
    D &= ~(w.z ^ t2);
    const uint32_t t3 = mux(m8, q8.w, q4.w);
    const uint32_t y3 = D & ~w.w & t3;
    D &= ~(w.w ^ t3);
    acc |= y2 | y3;
}

// Planes 4 j4 .. 4 j4 + 7 (calls j4 and j4 + 1) with both Philox evaluations interleaved.
__device__ __forceinline__ void plane_call2(uint32_t sA, uint32_t sB, const PlaneUniform &u,
                                            const RoundKeys &rk, const uint32_t *P, uint32_t m8,
                                            uint32_t &D, uint32_t &acc, uint32_t j4 = 0u)
{
    const uint4 w0 = philox_plane(sA, sB, j4, u, rk);
    const uint4 w1 = philox_plane(sA, sB, j4 + 1u, u, rk);
    const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const uint4 a4 = *reinterpret_cast<const uint4 *>(P + 4 * j4);
    const uint4 b4 = *reinterpret_cast<const uint4 *>(P + 4 * j4 + 4);
    const uint4 a8 = *reinterpret_cast<const uint4 *>(P + 64 + 4 * j4);
    const uint4 b8 = *reinterpret_cast<const uint4 *>(P + 68 + 4 * j4);
    const uint32_t t4[8] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
    const uint32_t t8[8] = {a8.x, a8.y, a8.z, a8.w, b8.x, b8.y, b8.z, b8.w};
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
        const uint32_t ta = mux(m8, t8[j], t4[j]);
        const uint32_t ya = D & ~ws[j] & ta;
        D &= ~(ws[j] ^ ta);
        const uint32_t tb = mux(m8, t8[j + 1], t4[j + 1]);
        const uint32_t yb = D & ~ws[j + 1] & tb;
        D &= ~(ws[j + 1] ^ tb);
        acc |= ya | yb;
    }
}

// Shared-memory word / byte access at an explicit 32-bit shared address.  volatile keeps
// them ordered among themselves and against barriers; plain C++ accesses of the same
// arrays elsewhere are separated from them by __syncthreads.
__device__ __forceinline__ uint32_t lds_u32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Bit-sliced addition of two L-bit vertical numbers (no overflow beyond L bits:
// the caller sizes L for the warp total).
template <int L>
__device__ __forceinline__ void vsum_xor(uint32_t (&c)[L], int off)
{
    uint32_t carry = 0u;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, c[l], off);
        const uint32_t s = c[l] ^ o ^ carry;
        carry = (c[l] & o) | (carry & (c[l] ^ o));
        c[l] = s;
    }
}


// ------------------------------------------------------------------ fused PT step
struct PtShared {
    int64_t Ecopy[256];  // the copy's energies (slot k = 32*rank + bit)
    int64_t Wcopy[256];  // walker ids
    uint32_t Mswap[8];   // accepted pairs (k, k+1) as bit k
    int64_t bestE, bestSlot, bestSweep;
    int32_t kmin, improve;
};

__device__ __forceinline__ void pt_init(PtShared &ps, const int64_t *walker, int c_local, int K)
{
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        ps.Wcopy[k] = walker[(size_t)c_local * K + k];
    if (threadIdx.x == 0) {
        ps.bestE = INT64_MAX;
        ps.bestSlot = -1;
        ps.bestSweep = -1;
    }
}

// End of a PT round for the copy held by this cluster (one CTA per 32-temperature word,
// cluster rank = word type wt): gather the copy's energies from every CTA's Ucnt through
// DSMEM, best-so-far check (strict <, ties -> lowest slot; the owning CTA snapshots via
// `snap(bit)`), exchange e (pairs k = e%2 + 2j, identical decisions in every CTA), then
// move configurations: within-word pairs by a delta swap, the cross-word pair through the
// neighbours' boundary bit planes B0 / B31 (n bits each).  Same result as k_exchange +
// k_swap_bits.
//
// Band split (torus kernel, NB = 2): the cluster holds NB CTAs per word type (rank = wt * NB +
// band), each owning the rows of one band; a word type's energy is the sum of its bands'
// counts.  Every CTA applies the swaps to its whole local lattice copy: its own rows and the
// halo rows it holds are current, and the halo rows' boundary bits come from the same band of
// the neighbouring word type, whose copy of those rows is current as well.
template <int NB = 1, class Snap>
__device__ void pt_step(PtShared &ps, const int32_t *Ucnt, int64_t m_edges, uint32_t *S, int n,
                        uint32_t *B0, uint32_t *B31, int KW, int wt, uint32_t c_global, uint32_t t_now,
                        uint32_t e_now, const uint64_t *Tx, const int64_t *Tx_off, const int32_t *Tx_len,
                        const RoundKeys &rk, Snap snap, int band = 0)
{
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int K = 32 * KW;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every CTA's Ucnt complete
    if (NB == 1) {
        for (int k = tid; k < K; k += nt) {
            const int32_t *rem = cluster.map_shared_rank(Ucnt, k >> 5);
            ps.Ecopy[k] = 2 * (int64_t)rem[k & 31] - m_edges;
        }
    } else {
        for (int k = tid; k < K; k += nt) {
            int64_t u = 0;
#pragma unroll
            for (int b = 0; b < NB; ++b)
                u += cluster.map_shared_rank(Ucnt, (k >> 5) * NB + b)[k & 31];
            ps.Ecopy[k] = 2 * u - m_edges;
        }
    }
    for (int q = tid; q < KW; q += nt)
        ps.Mswap[q] = 0u;
    __syncthreads();
    if (warp == 0) {  // best-so-far of the copy: argmin, ties -> lowest slot
        int64_t bE = INT64_MAX;
        int bk = -1;
        for (int k = lane; k < K; k += 32)
            if (bk < 0 || ps.Ecopy[k] < bE) {
                bE = ps.Ecopy[k];
                bk = k;
            }
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t oE = __shfl_down_sync(0xFFFFFFFFu, bE, o);
            const int ok = __shfl_down_sync(0xFFFFFFFFu, bk, o);
            if (ok >= 0 && (bk < 0 || oE < bE || (oE == bE && ok < bk))) {
                bE = oE;
                bk = ok;
            }
        }
        if (lane == 0) {
            ps.improve = bE < ps.bestE;
            ps.kmin = bk;
            if (bE < ps.bestE) {
                ps.bestE = bE;
                ps.bestSlot = (int64_t)c_global * K + bk;
                ps.bestSweep = t_now;
            }
        }
    }
    __syncthreads();
    if (ps.improve && (ps.kmin >> 5) == wt)  // the owning CTA snapshots the configuration
        snap(ps.kmin & 31);
    const int par = (int)(e_now & 1u);
    const int npairs = (K - par) / 2;
    for (int pi = tid; pi < npairs; pi += nt) {
        const int k = par + 2 * pi;
        const int64_t d = ps.Ecopy[k + 1] - ps.Ecopy[k];
        bool accept = d >= 0;
        if (!accept) {
            const int64_t j = -d - 1;
            if (j < Tx_len[k]) {
                const uint4 w = philox((uint32_t)k, e_now, c_global, ST_EXCH << 24, rk);
                const uint64_t Ux = ((uint64_t)w.x << 32) | (uint64_t)w.y;
                accept = Ux < Tx[Tx_off[k] + j];
            }
        }
        if (accept) {
            atomicOr(&ps.Mswap[k >> 5], 1u << (k & 31));
            const int64_t te = ps.Ecopy[k];
            ps.Ecopy[k] = ps.Ecopy[k + 1];
            ps.Ecopy[k + 1] = te;
            const int64_t tw = ps.Wcopy[k];
            ps.Wcopy[k] = ps.Wcopy[k + 1];
            ps.Wcopy[k + 1] = tw;
        }
    }
    __syncthreads();
    const uint32_t Min = ps.Mswap[wt] & 0x7FFFFFFFu;
    const bool cross_lo = wt > 0 && ((ps.Mswap[wt - 1] >> 31) & 1u);
    const bool cross_hi = wt + 1 < KW && ((ps.Mswap[wt] >> 31) & 1u);
    bool any_cross = false;
    for (int q = 0; q + 1 < KW; ++q)
        any_cross |= (ps.Mswap[q] >> 31) & 1u;
    const int nbw = (n + 31) / 32;
    if (any_cross) {  // uniform over the cluster
        for (int b = warp * 32; b < nbw * 32; b += nt) {
            const int l = b + lane;
            const uint32_t w = l < n ? S[l] : 0u;
            const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, w & 1u);
            const uint32_t b31 = __ballot_sync(0xFFFFFFFFu, w >> 31);
            if (lane == 0) {
                B0[b >> 5] = b0;
                B31[b >> 5] = b31;
            }
        }
        cluster.sync();
        const uint32_t *nB31 = cross_lo ? cluster.map_shared_rank(B31, NB == 1 ? wt - 1 : (wt - 1) * NB + band) : B31;
        const uint32_t *nB0 = cross_hi ? cluster.map_shared_rank(B0, NB == 1 ? wt + 1 : (wt + 1) * NB + band) : B0;
        for (int l = tid; l < n; l += nt) {
            uint32_t w = S[l];
            const uint32_t tt = (w ^ (w >> 1)) & Min;
            w ^= tt ^ (tt << 1);
            if (cross_lo)
                w = (w & ~1u) | ((nB31[l >> 5] >> (l & 31)) & 1u);
            if (cross_hi)
                w = (w & 0x7FFFFFFFu) | (((nB0[l >> 5] >> (l & 31)) & 1u) << 31);
            S[l] = w;
        }
    } else if (Min) {
        for (int l = tid; l < n; l += nt) {
            const uint32_t w = S[l];
            const uint32_t tt = (w ^ (w >> 1)) & Min;
            S[l] = w ^ tt ^ (tt << 1);
        }
    }
    __syncthreads();
}

template <int NB = 1>
__device__ __forceinline__ void pt_finish(const PtShared &ps, bool pt, int n_rounds, const int32_t *Ucnt,
                                          int64_t m_edges, int64_t *E_out, int64_t *walker,
                                          int64_t *copy_best, int gl, int wt, int c_local, int K,
                                          int band = 0)
{
    const int tid = threadIdx.x;
    if (NB > 1 && band != 0)  // band 0 writes the word type's results (every band holds the same)
        return;
    if (tid < 32) {
        E_out[(size_t)gl * 32 + tid] =
            pt && n_rounds > 0 ? ps.Ecopy[32 * wt + tid] : 2 * (int64_t)Ucnt[tid] - m_edges;
        if (pt)
            walker[(size_t)c_local * K + 32 * wt + tid] = ps.Wcopy[32 * wt + tid];
    }
    if (pt && wt == 0 && tid == 0) {
        copy_best[3 * c_local + 0] = ps.bestE;
        copy_best[3 * c_local + 1] = ps.bestSlot;
        copy_best[3 * c_local + 2] = ps.bestSweep;
    }
}

// warp total of the per-thread vertical counters; lane b gets replica b's count
__device__ __forceinline__ int32_t warp_counts(uint32_t (&cnt)[kCntLevels])
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
        vsum_xor(cnt, off);
    int32_t acc = 0;
#pragma unroll
    for (int l = 0; l < kCntLevels; ++l)
        acc += (int32_t)((cnt[l] >> (threadIdx.x & 31)) & 1u) << l;
    return acc;
}

}  // namespace bits
}  // namespace ising

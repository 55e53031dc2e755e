// k_icm.cu -- Houdayer / isoenergetic cluster moves on bit-packed spins (sm_100a).
//
// SURVEY §8(f) NEXT-1; PAPER.md P:53 ("two replicas at the same temperature are compared
// and a cluster of spins is identified, after which the sign of the cluster is changed in
// each replica", refs [20] Houdayer, [21] ICM).  Contract: DESIGN.md §3.7.
//
// One CTA per (copy pair (2p, 2p+1), word type wt): the two 32-temperature words hold the
// replicas of the same 32 temperatures in the two copies, so the overlap X = s_a ^ s_b is
// bit-sliced too and all 32 clusters grow at once: C |= X & OR(C of the neighbours),
// iterated in place over shared memory until a full pass changes nothing (the fixed point
// is the connected component of each bit's seed in the {X = 1} subgraph, whatever the
// visiting order).  The cluster bits then flip in both words; the 64 energies are
// recomputed with bit-sliced counters.
#include "internal.h"
#include "bits_core.cuh"

namespace ising {

using namespace bits;

__global__ void __launch_bounds__(1024) k_icm_bits(const IcmParams p)
{
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ int32_t Ua[32], Ub[32];
    const int n = p.n;
    uint32_t *X = sm;
    uint32_t *Cm = sm + n;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int pl = blockIdx.x, wt = blockIdx.y;
    const int KW = p.KW, K = 32 * KW;
    const size_t ga = (size_t)(2 * pl) * KW + wt, gb = ga + KW;
    uint32_t *Sa = p.state + ga * n, *Sb = p.state + gb * n;
    // temperatures k = 32 wt + b >= k_min take part
    const int lo = p.k_min - 32 * wt;
    const uint32_t kmask = lo <= 0 ? 0xFFFFFFFFu : (lo >= 32 ? 0u : ~((1u << lo) - 1u));
    if (kmask == 0u)
        return;
    for (int i = tid; i < n; i += nt) {
        X[i] = (Sa[i] ^ Sb[i]) & kmask;
        Cm[i] = 0u;
    }
    if (tid < 32) {
        Ua[tid] = 0;
        Ub[tid] = 0;
    }
    __syncthreads();
    // seeds: bit b's first candidate i_j = (w_j n) >> 32 with X = 1
    const uint32_t pair = p.pair0 + (uint32_t)pl;
    if (tid < 32 && ((kmask >> tid) & 1u)) {
        const uint32_t k = (uint32_t)(32 * wt + tid);
        int seed = -1;
        for (uint32_t j4 = 0; j4 < 16u; ++j4) {
            const uint4 w = philox(k, p.f, pair, (ST_ICM << 24) | j4, p.rk);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const uint32_t i = (uint32_t)(((uint64_t)ws[a] * (uint64_t)n) >> 32);
                const int idx = (int)(p.o2i ? p.o2i[i] : i);
                if (seed < 0 && ((X[idx] >> tid) & 1u))
                    seed = idx;
            }
        }
        if (seed >= 0)
            atomicOr(&Cm[seed], 1u << tid);
    }
    __syncthreads();
    // grow all 32 clusters to the fixed point
    bool changed = true;
    while (changed) {
        bool mine = false;
        for (int i = tid; i < n; i += nt) {
            const uint32_t x = X[i];
            const uint32_t c = Cm[i];
            if ((x & ~c) == 0u)
                continue;
            uint32_t nb = 0u;
            if (p.kind == 0) {
                const int y = i / p.Lx, xx = i - y * p.Lx;
                const int r = y * p.Lx + (xx + 1 == p.Lx ? 0 : xx + 1);
                const int l = y * p.Lx + (xx == 0 ? p.Lx - 1 : xx - 1);
                const int d = (y + 1 == p.Ly ? 0 : y + 1) * p.Lx + xx;
                const int u = (y == 0 ? p.Ly - 1 : y - 1) * p.Lx + xx;
                nb = Cm[r] | Cm[l] | Cm[d] | Cm[u];
            } else {
                for (int e = p.rp[i]; e < p.rp[i + 1]; ++e)
                    nb |= Cm[p.nbr[e] & 0x7FFFFFFFu];
            }
            const uint32_t nc = c | (x & nb);
            if (nc != c) {
                Cm[i] = nc;
                mine = true;
            }
        }
        changed = __syncthreads_or(mine) != 0;
    }
    // flip the clusters in both replicas and recount the unsatisfied bonds
    uint32_t ca[kCntLevels], cb[kCntLevels];
#pragma unroll
    for (int l = 0; l < kCntLevels; ++l) {
        ca[l] = 0u;
        cb[l] = 0u;
    }
    for (int i = tid; i < n; i += nt) {
        const uint32_t c = Cm[i];
        if (c) {
            Sa[i] ^= c;
            Sb[i] ^= c;
        }
    }
    __syncthreads();  // global writes of this CTA visible to its own threads
    for (int i = tid; i < n; i += nt) {
        const uint32_t a = Sa[i], b = Sb[i];
        if (p.kind == 0) {
            const int y = i / p.Lx, xx = i - y * p.Lx;
            const int r = y * p.Lx + (xx + 1 == p.Lx ? 0 : xx + 1);
            const int d = (y + 1 == p.Ly ? 0 : y + 1) * p.Lx + xx;
            const uint32_t jr = 0u - (uint32_t)(p.jbyte_orig[i] & 1u), jd = 0u - (uint32_t)((p.jbyte_orig[i] >> 1) & 1u);
            vadd(ca, ~(a ^ Sa[r] ^ jr));
            vadd(ca, ~(a ^ Sa[d] ^ jd));
            vadd(cb, ~(b ^ Sb[r] ^ jr));
            vadd(cb, ~(b ^ Sb[d] ^ jd));
        } else {
            for (int e = p.rp[i]; e < p.rp[i + 1]; ++e) {
                const uint32_t nbv = p.nbr[e];
                const uint32_t j = nbv & 0x7FFFFFFFu;
                if ((int)j <= i)
                    continue;
                const uint32_t jm = (uint32_t)((int32_t)nbv >> 31);
                vadd(ca, ~(a ^ Sa[j] ^ jm));
                vadd(cb, ~(b ^ Sb[j] ^ jm));
            }
        }
    }
    const int32_t na = warp_counts(ca), nb = warp_counts(cb);
    atomicAdd(&Ua[lane], na);
    atomicAdd(&Ub[lane], nb);
    __syncthreads();
    if (tid < 32 && ((kmask >> tid) & 1u)) {
        const int64_t ra = (int64_t)(2 * pl) * K + 32 * wt + tid;
        p.E[ra] = 2 * (int64_t)Ua[tid] - p.m_edges;
        p.E[ra + K] = 2 * (int64_t)Ub[tid] - p.m_edges;
    }
}

cudaError_t launch_icm_bits(const IcmParams &p, int32_t pairs, int32_t threads, cudaStream_t st)
{
    const size_t smem = (size_t)8 * p.n;
    cudaError_t e = cudaFuncSetAttribute(k_icm_bits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    k_icm_bits<<<dim3((unsigned)pairs, (unsigned)p.KW), threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace ising

// k_csr_bits.cu -- multi-spin-coded Metropolis sweeps on a +-1 CSR graph (sm_100a).
//
// Rows a3-a6 of SURVEY.md §8(a) for the sparse-random-graph workload (C3: G70
// stand-in, "Unweighted MaxCut on sparse random graph", encoded
// J = +1 in CSR with a greedy colouring).  Same structure as k_grid_bits: one
// CTA owns one 32-replica word group resident in shared memory for a whole
// ising_sweep call; colour classes are contiguous in the internal vertex order
// (and sorted by degree inside a class so a warp mostly sees one degree); the
// CSR itself (~120 KB for C3) is read through the L1/read-only path.
//
// Per (vertex of degree d, word): a_b = ~(s_i ^ s_j ^ J_b) for every neighbour,
// summed into a 4-bit vertical counter u (bit-sliced adder);
// dE = -2 s h = 2d - 4u > 0  <=>  2u < d, class q = dE/2 = d - 2u.  The lanes of
// each class compare their PLANE-contract U64 against the word's threshold
// planes P[q][j] MSB first, exactly as in k_grid_bits.
#include "internal.h"

namespace ising {

namespace {
constexpr int kPlaneStride = 65;  // padded row: classes of one plane land on distinct banks
constexpr int kMaxCls = 8;        // d <= 15 -> at most 8 classes with dE > 0
constexpr int kCntLevels = 12;
}  // namespace

size_t csr_bits_smem(int32_t n, int32_t qmax, int32_t words_per_copy)
{
    (void)words_per_copy;
    return (size_t)n * sizeof(uint32_t) + (size_t)qmax * kPlaneStride * sizeof(uint32_t);
}

__global__ void __launch_bounds__(1024, 1) k_csr_bits(const CsrBitsParams p)
{
    extern __shared__ uint32_t sm[];
    __shared__ int32_t Ucnt[32];
    const int n = p.n;
    uint32_t *S = sm;
    uint32_t *P = sm + n;  // P[(q-1)*65 + j], q = 1..qmax
    const int gl = blockIdx.x;
    const uint32_t g = p.g0 + (uint32_t)gl;
    const int wt = (int)(g % (uint32_t)p.words_per_copy);
    const int tid = threadIdx.x, nt = blockDim.x;

    const uint32_t *src = p.state_in + (size_t)gl * n;
    for (int i = tid; i < n; i += nt)
        S[i] = src[i];
    for (int x = tid; x < p.qmax * 64; x += nt) {
        const int q = x / 64, j = x % 64;
        P[q * kPlaneStride + j] = p.planes[((size_t)wt * p.qmax + q) * 64 + j];
    }
    if (tid < 32)
        Ucnt[tid] = 0;
    __syncthreads();

    for (int s = 0; s < p.n_sweeps; ++s) {
        const uint32_t t = p.t0 + (uint32_t)s;
#pragma unroll 1
        for (int c = 0; c < p.ncol; ++c) {
            const int v0 = __ldg(p.class_off + c), v1 = __ldg(p.class_off + c + 1);
            for (int v = v0 + tid; v < v1; v += nt) {
                const uint32_t own = S[v];
                const int e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
                const int d = e1 - e0;
                uint32_t u[4] = {0u, 0u, 0u, 0u};
                for (int e = e0; e < e1; ++e) {
                    const uint32_t nb = __ldg(p.nbr + e);
                    const uint32_t jm = (uint32_t)((int32_t)nb >> 31);
                    vadd(u, ~(own ^ S[nb & 0x7FFFFFFFu] ^ jm));
                }
                // classes v = 0 .. (d-1)/2 : lanes with u == v, q = d - 2v
                const int ncls = (d + 1) >> 1;
                uint32_t mk[kMaxCls];
                uint32_t D = 0u;
#pragma unroll
                for (int cv = 0; cv < kMaxCls; ++cv) {
                    mk[cv] = 0u;
                    if (cv < ncls) {
                        const uint32_t e_0 = (cv & 1) ? u[0] : ~u[0];
                        const uint32_t e_1 = (cv & 2) ? u[1] : ~u[1];
                        const uint32_t e_2 = (cv & 4) ? u[2] : ~u[2];
                        const uint32_t e_3 = (cv & 8) ? u[3] : ~u[3];
                        mk[cv] = e_0 & e_1 & e_2 & e_3;
                        D |= mk[cv];
                    }
                }
                const uint32_t always = ~D;  // dE <= 0
                uint32_t lt = 0u;
                if (D) {
                    const uint32_t io = __ldg(p.orig + v);
                    uint32_t j4 = 0;
                    do {
                        const uint4 w = philox(io, t, g, (ST_PLANE << 24) | j4, p.rk);
                        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            const int j = 4 * (int)j4 + a;
                            uint32_t tj = 0u;
#pragma unroll
                            for (int cv = 0; cv < kMaxCls; ++cv)
                                if (cv < ncls)
                                    tj |= mk[cv] & P[(d - 2 * cv - 1) * kPlaneStride + j];
                            lt |= D & ~ww[a] & tj;
                            D &= ~(ww[a] ^ tj);
                        }
                        ++j4;
                    } while (D && j4 < 16u);
                }
                S[v] = own ^ (always | lt);
            }
            __syncthreads();
        }
    }

    // energy: each undirected edge once (neighbour id > own id); E = 2U - m
    {
        uint32_t cnt[kCntLevels];
#pragma unroll
        for (int l = 0; l < kCntLevels; ++l)
            cnt[l] = 0;
        for (int v = tid; v < n; v += nt) {
            const uint32_t own = S[v];
            const int e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
            for (int e = e0; e < e1; ++e) {
                const uint32_t nb = __ldg(p.nbr + e);
                const uint32_t j = nb & 0x7FFFFFFFu;
                if ((int)j <= v)
                    continue;
                const uint32_t jm = (uint32_t)((int32_t)nb >> 31);
                vadd(cnt, ~(own ^ S[j] ^ jm));
            }
        }
        const int lane = tid & 31;
        int32_t acc = 0;
#pragma unroll
        for (int l = 0; l < kCntLevels; ++l) {
            if (__syncthreads_or(cnt[l] != 0u) == 0)
                continue;
#pragma unroll 4
            for (int b = 0; b < 32; ++b) {
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (cnt[l] >> b) & 1u);
                if (lane == b)
                    acc += __popc(bal) << l;
            }
        }
        atomicAdd(&Ucnt[lane], acc);
        __syncthreads();
        if (tid < 32)
            p.E_out[(size_t)gl * 32 + tid] = 2 * (int64_t)Ucnt[tid] - p.m;
    }

    uint32_t *dst = p.state_out + (size_t)gl * n;
    for (int i = tid; i < n; i += nt)
        dst[i] = S[i];
}

cudaError_t launch_csr_bits(const CsrBitsParams &p, int32_t G, int32_t threads, size_t smem,
                            cudaStream_t st)
{
    if (smem > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(k_csr_bits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return e;
    }
    k_csr_bits<<<G, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace ising

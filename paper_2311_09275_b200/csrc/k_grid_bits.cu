// k_grid_bits.cu -- multi-spin-coded Metropolis sweeps on +-1 tori (sm_100a).
//
// Hot path rows a3-a6 of SURVEY.md §8(a) for the grid workloads (C2, C4; Gset
// spin-glass tori, Table I).  One CTA owns one 32-replica word
// group g (32 consecutive global slots = 32 temperatures of one copy) for all
// n sites and keeps it resident in shared memory for a whole ising_sweep call:
// load -> n_sweeps x {colour 0, colour 1} with __syncthreads between phases ->
// energy of the 32 replicas -> store.  Shared memory holds the spins in
// colour-separated order (each colour class contiguous per row), so lane l of
// a warp touches word l of a row: conflict-free LDS/STS for the site and all
// four neighbours.
//
// Per (site, word) -- 32 attempts at once, bit b = slot 32g+b:
//   a_b   = ~(s_i ^ s_j ^ J_b)                 unsatisfied-bond bits (J_b s_i s_j = +1)
//   u     = #unsatisfied among 4;  dE = 8 - 4u  (dE = -2 s_i h_i)
//   m8/m4 = lanes with dE = 8 / 4 (u = 0 / 1); all other lanes flip (dE <= 0).
//   PLANE contract: U64 bit (63-j) = bit b of word (j&3) of
//       Philox(i, t, g, PLANE<<24 | j>>2); accept iff U64 < T[beta_k][dE].
//   The comparison runs MSB plane first over the 32 undecided lanes D:
//       lt |= D & ~u_j & t_j;  D &= ~(u_j ^ t_j)
//   and stops when D is empty (the first differing bit fixes U < T), so the
//   result is exactly the 64-bit comparison.
//   t_j (threshold plane j of the word's 32 temperatures) comes from the host
//   plane table P[wt][dE][j]; slot temperatures never change (exchanges move
//   configurations), so the table is fixed for the whole run.
#include "internal.h"

namespace ising {

size_t grid_bits_smem(int32_t n) { return (size_t)(2 * n + 128) * sizeof(uint32_t); }

namespace {

struct GridGeom {
    int32_t Lx, Ly, hx, half;
    uint32_t ymagic;
};

// Neighbour words of colour-c site with class index l; returns the four
// unsatisfied-bond masks and the original site id.
__device__ __forceinline__ void grid_unsat(const uint32_t *S, const uint32_t *JW, const GridGeom &G,
                                           int c, int l, uint32_t own, uint32_t &a0, uint32_t &a1,
                                           uint32_t &a2, uint32_t &a3, uint32_t &i_orig)
{
    const int y = (int)__umulhi((uint32_t)l, G.ymagic);
    const int m = l - y * G.hx;
    const int par = (c + y) & 1;
    const int x = 2 * m + par;
    const int mr = par ? (m + 1 == G.hx ? 0 : m + 1) : m;
    const int ml = par ? m : (m == 0 ? G.hx - 1 : m - 1);
    const int yd = (y + 1 == G.Ly) ? 0 : y + 1;
    const int yu = (y == 0) ? G.Ly - 1 : y - 1;
    const int ob = (1 - c) * G.half;
    const uint32_t xr = S[ob + y * G.hx + mr];
    const uint32_t xl = S[ob + y * G.hx + ml];
    const uint32_t xd = S[ob + yd * G.hx + m];
    const uint32_t xu = S[ob + yu * G.hx + m];
    const uint32_t jw = JW[c * G.half + l];
    a0 = ~(own ^ xr ^ byte_sign_mask<0>(jw));
    a1 = ~(own ^ xl ^ byte_sign_mask<1>(jw));
    a2 = ~(own ^ xd ^ byte_sign_mask<2>(jw));
    a3 = ~(own ^ xu ^ byte_sign_mask<3>(jw));
    i_orig = (uint32_t)(x + G.Lx * y);
}

constexpr int kCntLevels = 8;

}  // namespace

__global__ void __launch_bounds__(1024, 1) k_grid_bits(const GridBitsParams p)
{
    extern __shared__ uint32_t sm[];
    __shared__ int32_t Ucnt[32];
    const int n = p.n;
    GridGeom G{p.Lx, p.Ly, p.hx, p.half, p.ymagic};
    uint32_t *S = sm;
    uint32_t *JW = sm + n;
    uint32_t *P = sm + 2 * n;  // P[0..63]: dE=4 planes, P[64..127]: dE=8 planes
    const int gl = blockIdx.x;
    const uint32_t g = p.g0 + (uint32_t)gl;
    const int wt = (int)(g % (uint32_t)p.words_per_copy);
    const int tid = threadIdx.x, nt = blockDim.x;

    // ---- load: original order -> colour-separated order
    const uint32_t *src = p.state_in + (size_t)gl * n;
    for (int i = tid; i < n; i += nt) {
        const int y = i / p.Lx, x = i - y * p.Lx;
        S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)] = src[i];
    }
    for (int l = tid; l < n; l += nt)
        JW[l] = p.jword[l];
    for (int j = tid; j < 128; j += nt)
        P[j] = p.planes[wt * 128 + j];
    if (tid < 32)
        Ucnt[tid] = 0;
    __syncthreads();

    // ---- sweeps
    for (int s = 0; s < p.n_sweeps; ++s) {
        const uint32_t t = p.t0 + (uint32_t)s;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            uint32_t *Sc = S + c * G.half;
            for (int l = tid; l < G.half; l += nt) {
                const uint32_t own = Sc[l];
                uint32_t a0, a1, a2, a3, i_orig;
                grid_unsat(S, JW, G, c, l, own, a0, a1, a2, a3, i_orig);
                const uint32_t s01 = a0 ^ a1, c01 = a0 & a1;
                const uint32_t s23 = a2 ^ a3, c23 = a2 & a3;
                const uint32_t m8 = ~(s01 | c01 | s23 | c23);  // u = 0 -> dE = 8
                const uint32_t m4 = (s01 ^ s23) & ~(c01 | c23); // u = 1 -> dE = 4
                uint32_t D = m8 | m4, lt = 0;
                if (D) {
                    uint32_t j4 = 0;
                    do {
                        const uint4 w = philox(i_orig, t, g, (ST_PLANE << 24) | j4, p.rk);
                        const uint4 q4 = *reinterpret_cast<const uint4 *>(P + 4 * j4);
                        const uint4 q8 = *reinterpret_cast<const uint4 *>(P + 64 + 4 * j4);
#define PLANE_STEP(U, T4, T8)                                   \
    {                                                           \
        const uint32_t tj = (m4 & (T4)) | (m8 & (T8));          \
        lt |= D & ~(U) & tj;                                    \
        D &= ~((U) ^ tj);                                       \
    }
                        PLANE_STEP(w.x, q4.x, q8.x)
                        PLANE_STEP(w.y, q4.y, q8.y)
                        PLANE_STEP(w.z, q4.z, q8.z)
                        PLANE_STEP(w.w, q4.w, q8.w)
#undef PLANE_STEP
                        ++j4;
                    } while (D && j4 < 16u);
                }
                Sc[l] = own ^ (~(m8 | m4) | lt);
            }
            __syncthreads();
        }
    }

    // ---- energy: every bond joins a colour-0 and a colour-1 site, so the four
    // bonds of the colour-1 sites count each bond exactly once.  E = 2U - 2n.
    {
        uint32_t cnt[kCntLevels];
#pragma unroll
        for (int l = 0; l < kCntLevels; ++l)
            cnt[l] = 0;
        const uint32_t *S1 = S + G.half;
        for (int l = tid; l < G.half; l += nt) {
            uint32_t a0, a1, a2, a3, i_orig;
            grid_unsat(S, JW, G, 1, l, S1[l], a0, a1, a2, a3, i_orig);
            vadd(cnt, a0);
            vadd(cnt, a1);
            vadd(cnt, a2);
            vadd(cnt, a3);
        }
        const int lane = tid & 31;
        int32_t acc = 0;
#pragma unroll
        for (int l = 0; l < kCntLevels; ++l) {
            if (l >= p.cnt_levels)
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
            p.E_out[(size_t)gl * 32 + tid] = 2 * (int64_t)Ucnt[tid] - 2 * (int64_t)n;
    }

    // ---- store: colour-separated -> original order
    uint32_t *dst = p.state_out + (size_t)gl * n;
    for (int i = tid; i < n; i += nt) {
        const int y = i / p.Lx, x = i - y * p.Lx;
        dst[i] = S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)];
    }
}

cudaError_t launch_grid_bits(const GridBitsParams &p, int32_t G, int32_t threads, size_t smem,
                             cudaStream_t st)
{
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_grid_bits, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess)
            return e;
    }
    k_grid_bits<<<G, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace ising

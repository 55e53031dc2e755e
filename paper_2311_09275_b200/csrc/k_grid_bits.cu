// k_grid_bits.cu -- multi-spin-coded Metropolis sweeps on +-1 tori (sm_100a).
//
// Hot path rows a3-a6 of SURVEY.md §8(a) for the grid workloads (C2, C4; Gset
// spin-glass tori, Table I).  One CTA owns one 32-replica word
// group g (32 consecutive global slots = 32 temperatures of one copy) for all
// n sites and keeps it resident in shared memory for a whole ising_sweep call:
// load -> n_sweeps x {colour 0, colour 1} -> energy of the 32 replicas -> store.
// Shared memory holds the spins in colour-separated order (each colour class
// contiguous per row), so lane l of a warp touches word l of a row:
// conflict-free LDS/STS for the site and all four neighbours.
//
// Per (site, word) -- 32 attempts at once, bit b = slot 32g+b:
//   a_b   = ~(s_i ^ s_j ^ J_b)                 unsatisfied-bond bits (J_b s_i s_j = +1)
//   u     = #unsatisfied among 4;  dE = 8 - 4u  (dE = -2 s_i h_i)
//   m8/m4 = lanes with dE = 8 / 4 (u = 0 / 1); all other lanes flip (dE <= 0).
//   PLANE contract: U64 bit (63-j) = bit b of word (j&3) of
//       Philox(i, t, g, PLANE<<24 | j>>2); accept iff U64 < T[beta_k][dE].
//   The comparison runs MSB plane first over the undecided lanes D:
//       acc |= D & ~u_j & t_j;  D &= ~(u_j ^ t_j)
//   and stops when D is empty (the first differing bit fixes U < T), so the
//   result is exactly the 64-bit comparison.  t_j (threshold
//   plane j of the word's 32 temperatures) comes from the host plane table
//   P[wt][dE][j]; slot temperatures never change (exchanges move
//   configurations), so the table is fixed for the whole run.
//
// Work compaction of the RNG tail: a colour phase runs in two
// stages.  Stage 1: every site draws planes 0..7 (two Philox calls); ~89% of
// words are then decided and written.  The rest are pushed to a shared-memory
// queue and stage 2 finishes them with all 32 lanes of a warp busy, instead of
// leaving most lanes of a warp idle while one lane draws its 3rd/4th call.
// Philox rounds 0-1 are partially hoisted: the parts that depend only on the
// CTA's group g, the sweep t or the site i are computed once, not per call.
#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace ising {

namespace {

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

// Philox4x32-10 of counter (i, t, g, PLANE<<24 | j4) from the hoisted parts.  Round
// keys are re-derived from the 64-bit key (k0 + r W0, k1 + r W1): kernel-uniform values
// the compiler keeps in uniform registers instead of reloading them per call.
__device__ __forceinline__ uint4 philox_plane(uint32_t sA, uint32_t sB, uint32_t j4,
                                              const PlaneUniform &u, const RoundKeys &rk)
{
    const uint32_t k0 = rk.k[0], k1 = rk.k[1];
    const uint32_t X = sA ^ j4;  // round-0 output word 2 (j4 < 2^24)
    uint32_t c0 = __umulhi(kM1, X) ^ u.U0;
    uint32_t c1 = kM1 * X;
    uint32_t c2 = sB;
    uint32_t c3 = u.L0r1;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        const uint32_t lo0 = kM0 * c0, hi0 = __umulhi(kM0, c0);
        const uint32_t lo1 = kM1 * c2, hi1 = __umulhi(kM1, c2);
        const uint32_t n0 = hi1 ^ c1 ^ (k0 + (uint32_t)r * 0x9E3779B9u);
        const uint32_t n2 = hi0 ^ c3 ^ (k1 + (uint32_t)r * 0xBB67AE85u);
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ uint32_t mux(uint32_t m, uint32_t a, uint32_t b) { return (m & a) | (~m & b); }

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

// Planes 0..7 (calls j4 = 0 and 1) with both Philox evaluations interleaved.
__device__ __forceinline__ void plane_call2(uint32_t sA, uint32_t sB, const PlaneUniform &u,
                                            const RoundKeys &rk, const uint32_t *P, uint32_t m8,
                                            uint32_t &D, uint32_t &acc)
{
    const uint4 w0 = philox_plane(sA, sB, 0u, u, rk);
    const uint4 w1 = philox_plane(sA, sB, 1u, u, rk);
    const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const uint4 a4 = *reinterpret_cast<const uint4 *>(P);
    const uint4 b4 = *reinterpret_cast<const uint4 *>(P + 4);
    const uint4 a8 = *reinterpret_cast<const uint4 *>(P + 64);
    const uint4 b8 = *reinterpret_cast<const uint4 *>(P + 68);
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

// Site geometry of one thread in the 2-D mapping (column m of a colour class,
// rows ty, ty + rpp, ...).
struct ThreadGeom {
    int m, mL, mR;  // class column and its wrapped neighbours
    int ty;
    bool active;
};

__device__ __forceinline__ void site_unsat(const uint32_t *S, const uint8_t *JB, const GridGeom &G,
                                           const ThreadGeom &T, int c, int y, uint32_t own,
                                           uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3,
                                           uint32_t &i_orig)
{
    const int par = (c + y) & 1;
    const int yd = (y + 1 == G.Ly) ? 0 : y + 1;
    const int yu = (y == 0) ? G.Ly - 1 : y - 1;
    const uint32_t *So = S + (1 - c) * G.half;
    const int row = y * G.hx;
    const uint32_t xr = So[row + (par ? T.mR : T.m)];
    const uint32_t xl = So[row + (par ? T.m : T.mL)];
    const uint32_t xd = So[yd * G.hx + T.m];
    const uint32_t xu = So[yu * G.hx + T.m];
    const uint32_t jw = (uint32_t)JB[c * G.half + row + T.m] * 0x10204080u;
    a0 = ~(own ^ xr ^ byte_sign_mask<0>(jw));
    a1 = ~(own ^ xl ^ byte_sign_mask<1>(jw));
    a2 = ~(own ^ xd ^ byte_sign_mask<2>(jw));
    a3 = ~(own ^ xu ^ byte_sign_mask<3>(jw));
    i_orig = (uint32_t)(2 * T.m + par + G.Lx * y);
}

}  // namespace

int32_t grid_bits_qcap(int32_t n)
{
    const size_t base = (size_t)4 * n + (((size_t)n + 15) & ~(size_t)15) + 512 +
                        (size_t)8 * ((n + 31) / 32);
    const size_t half = (size_t)n / 2;
    size_t qcap = half < 4096 ? half : 4096;
    const size_t budget = 200 * 1024;
    if (base + qcap * kQItemBytes > budget)
        qcap = base < budget ? (budget - base) / kQItemBytes : 0;
    return (int32_t)qcap;
}

size_t grid_bits_smem(int32_t n)
{
    // S (4n) + JB (n, padded to 16) + planes (512) + queue + 2 boundary bit planes
    return (size_t)4 * n + (((size_t)n + 15) & ~(size_t)15) + 512 +
           (size_t)grid_bits_qcap(n) * kQItemBytes + (size_t)8 * ((n + 31) / 32);
}

__global__ void __launch_bounds__(1024, 1) k_grid_bits(const GridBitsParams p)
{
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ int32_t Ucnt[32];
    __shared__ int32_t wcount[33];
    __shared__ int32_t wprefix[33];
    // fused PT rounds (cluster of words_per_copy CTAs = one copy): the copy's energies,
    // walker ids, swap mask and best record, held identically by every CTA of the cluster
    __shared__ int64_t Ecopy[256];
    __shared__ int64_t Wcopy[256];
    __shared__ uint32_t Mswap[8];
    __shared__ int64_t bestE, bestSlot, bestSweep;
    __shared__ int32_t s_kmin, s_improve;
    const int n = p.n;
    const GridGeom G{p.Lx, p.Ly, p.hx, p.half, p.ymagic};
    uint32_t *S = sm;
    uint8_t *JB = reinterpret_cast<uint8_t *>(sm + n);
    uint32_t *P = reinterpret_cast<uint32_t *>(JB + ((n + 15) & ~15));  // P[0..63] dE=4, P[64..127] dE=8
    uint32_t *Q = P + 128;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nt >> 5;
    const int qcap = p.qcap;
    const int wcap = qcap / nwarps;  // per-warp queue region
    uint32_t *q_idx = Q, *q_own = Q + qcap, *q_D = Q + 2 * qcap, *q_acc = Q + 3 * qcap,
             *q_m8 = Q + 4 * qcap;
    const int nbw = (n + 31) / 32;
    uint32_t *B0 = Q + 5 * qcap;  // boundary bit planes for cross-word swaps (PT mode)
    uint32_t *B31 = B0 + nbw;
    const int wq0 = warp * wcap;

    const int gl = blockIdx.x;
    const uint32_t g = p.g0 + (uint32_t)gl;
    const int KW = p.words_per_copy;
    const int wt = (int)(g % (uint32_t)KW);
    const int K = 32 * KW;
    const bool pt = p.pt != 0;
    const int c_local = gl / KW;
    const uint32_t c_global = g / (uint32_t)KW;

    // 2-D thread mapping: column m = tid % hx of a class row, rows ty + k*rpp
    const int rpp = nt / G.hx;  // rows per pass (host guarantees >= 1)
    const int npass = (G.Ly + rpp - 1) / rpp;
    ThreadGeom T;
    T.ty = tid / G.hx;
    T.m = tid - T.ty * G.hx;
    T.mL = T.m == 0 ? G.hx - 1 : T.m - 1;
    T.mR = T.m + 1 == G.hx ? 0 : T.m + 1;
    T.active = T.ty < rpp;

    // ---- load: original order -> colour-separated order
    const uint32_t *src = p.state_in + (size_t)gl * n;
    for (int i = tid; i < n; i += nt) {
        const int y = i / p.Lx, x = i - y * p.Lx;
        S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)] = src[i];
    }
    for (int l = tid; l < n; l += nt)
        JB[l] = p.jbyte[l];
    for (int j = tid; j < 128; j += nt)
        P[j] = p.planes[wt * 128 + j];
    if (pt) {
        for (int k = tid; k < K; k += nt)
            Wcopy[k] = p.walker[(size_t)c_local * K + k];
        if (tid == 0) {
            bestE = INT64_MAX;
            bestSlot = -1;
            bestSweep = -1;
        }
    }
    __syncthreads();

    for (int round = 0; round < p.n_rounds; ++round) {
        // ---- k_ex sweeps
        for (int s = 0; s < p.k_ex; ++s) {
            const uint32_t t = p.t0 + (uint32_t)(round * p.k_ex + s);
            const PlaneUniform U = plane_uniform(g, t, p.rk);
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                uint32_t *Sc = S + c * G.half;
                // stage 1: planes 0..7 for every site; undecided words go to this warp's queue
                int wq = 0;  // warp-uniform
                for (int pass = 0; pass < npass; ++pass) {
                    const int y = T.ty + pass * rpp;
                    const bool valid = T.active && y < G.Ly;
                    const int l = y * G.hx + T.m;
                    uint32_t own = 0, D = 0, acc = 0, m8 = 0, i_orig = 0;
                    if (valid) {
                        own = Sc[l];
                        uint32_t a0, a1, a2, a3;
                        site_unsat(S, JB, G, T, c, y, own, a0, a1, a2, a3, i_orig);
                        const uint32_t s01 = a0 ^ a1, c01 = a0 & a1;
                        const uint32_t s23 = a2 ^ a3, c23 = a2 & a3;
                        m8 = ~(s01 | c01 | s23 | c23);                   // u = 0 -> dE = 8
                        const uint32_t m4 = (s01 ^ s23) & ~(c01 | c23);  // u = 1 -> dE = 4
                        D = m8 | m4;
                        acc = ~D;  // dE <= 0 always flips
                        if (D) {  // planes 0..7: both calls issued together (two independent chains)
                            uint32_t sA, sB;
                            plane_site(i_orig, U, p.rk, sA, sB);
                            plane_call2(sA, sB, U, p.rk, P, m8, D, acc);
                        }
                    }
                    const bool need = D != 0u;
                    const uint32_t pm = __ballot_sync(0xFFFFFFFFu, need);
                    const int slot = wq + __popc(pm & lanemask_lt());
                    wq += __popc(pm);
                    if (need && slot < wcap) {
                        const int qs = wq0 + slot;
                        q_idx[qs] = (uint32_t)l | (i_orig << 16);
                        q_own[qs] = own;
                        q_D[qs] = D;
                        q_acc[qs] = acc;
                        q_m8[qs] = m8;
                    } else if (valid) {
                        if (need) {  // this warp's queue region is full: finish inline
                            uint32_t sA, sB;
                            plane_site(i_orig, U, p.rk, sA, sB);
                            uint32_t j4 = 2;
                            do {
                                plane_call(sA, sB, j4, U, p.rk, P, m8, D, acc);
                                ++j4;
                            } while (D && j4 < 16u);
                        }
                        Sc[l] = own ^ acc;
                    }
                }
                if (lane == 0)
                    wcount[warp] = min(wq, wcap);
                __syncthreads();
                if (warp == 0) {  // exclusive prefix over the warp regions
                    const int v = lane < nwarps ? wcount[lane] : 0;
                    int incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (lane >= o)
                            incl += u;
                    }
                    wprefix[lane] = incl - v;
                    if (lane == 31)
                        wprefix[32] = incl;
                }
                __syncthreads();
                // stage 2: the queued tail, one word per thread, all lanes busy
                const int nq = wprefix[32];
                for (int q = tid; q < nq; q += nt) {
                    int lo = 0, hi = nwarps;  // region w: wprefix[w] <= q < wprefix[w+1]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (wprefix[mid] <= q)
                            lo = mid;
                        else
                            hi = mid;
                    }
                    const int qs = lo * wcap + (q - wprefix[lo]);
                    const uint32_t idx = q_idx[qs];
                    const int l = (int)(idx & 0xFFFFu);
                    const uint32_t i_orig = idx >> 16;
                    uint32_t D = q_D[qs], acc = q_acc[qs];
                    const uint32_t m8 = q_m8[qs];
                    uint32_t sA, sB;
                    plane_site(i_orig, U, p.rk, sA, sB);
                    uint32_t j4 = 2;
                    do {
                        plane_call(sA, sB, j4, U, p.rk, P, m8, D, acc);
                        ++j4;
                    } while (D && j4 < 16u);
                    Sc[l] = q_own[qs] ^ acc;
                }
                __syncthreads();
            }
        }

        // ---- energy: every bond joins a colour-0 and a colour-1 site, so the four
        // bonds of the colour-1 sites count each bond exactly once.  E = 2U - 2n.
        {
            if (tid < 32)
                Ucnt[tid] = 0;
            uint32_t cnt[kCntLevels];
#pragma unroll
            for (int l = 0; l < kCntLevels; ++l)
                cnt[l] = 0;
            const uint32_t *S1 = S + G.half;
            for (int pass = 0; pass < npass; ++pass) {
                const int y = T.ty + pass * rpp;
                if (T.active && y < G.Ly) {
                    uint32_t a0, a1, a2, a3, i_orig;
                    site_unsat(S, JB, G, T, 1, y, S1[y * G.hx + T.m], a0, a1, a2, a3, i_orig);
                    vadd(cnt, a0);
                    vadd(cnt, a1);
                    vadd(cnt, a2);
                    vadd(cnt, a3);
                }
            }
            // warp total by a butterfly of bit-sliced additions, then lane b reads bit b
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                vsum_xor(cnt, off);
            int32_t acc = 0;
#pragma unroll
            for (int l = 0; l < kCntLevels; ++l)
                acc += (int32_t)((cnt[l] >> lane) & 1u) << l;
            __syncthreads();  // Ucnt zeroed
            atomicAdd(&Ucnt[lane], acc);
            __syncthreads();
        }
        if (!pt)
            continue;

        // ---- fused PT step for this copy (a7/a8): same result as ising_exchange
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();  // every CTA's Ucnt complete
        if (tid < K) {
            const int32_t *rem = cluster.map_shared_rank(Ucnt, tid >> 5);
            Ecopy[tid] = 2 * (int64_t)rem[tid & 31] - 2 * (int64_t)n;
        }
        if (tid < KW)
            Mswap[tid] = 0u;
        __syncthreads();
        const uint32_t t_now = p.t0 + (uint32_t)((round + 1) * p.k_ex);
        const uint32_t e_now = p.e0 + (uint32_t)round;
        if (warp == 0) {  // best-so-far of the copy: argmin, ties -> lowest slot
            int64_t bE = INT64_MAX;
            int bk = -1;
            for (int k = lane; k < K; k += 32)
                if (bk < 0 || Ecopy[k] < bE) {
                    bE = Ecopy[k];
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
                s_improve = bE < bestE;
                s_kmin = bk;
                if (bE < bestE) {
                    bestE = bE;
                    bestSlot = (int64_t)c_global * K + bk;
                    bestSweep = t_now;
                }
            }
        }
        __syncthreads();
        if (s_improve && (s_kmin >> 5) == wt) {  // the owning CTA snapshots the configuration
            const int bit = s_kmin & 31;
            int8_t *dst = p.snap + (size_t)c_local * n;
            for (int i = tid; i < n; i += nt) {
                const int y = i / p.Lx, x = i - y * p.Lx;
                dst[i] = ((S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)] >> bit) & 1u) ? -1 : 1;
            }
        }
        // exchange e_now: pairs (k, k+1), k = e%2 + 2j (decided identically in every CTA)
        const int par = (int)(e_now & 1u);
        const int npairs = (K - par) / 2;
        if (tid < npairs) {
            const int k = par + 2 * tid;
            const int64_t d = Ecopy[k + 1] - Ecopy[k];
            bool accept = d >= 0;
            if (!accept) {
                const int64_t j = -d - 1;
                if (j < p.Tx_len[k]) {
                    const uint4 w = philox((uint32_t)k, e_now, c_global, ST_EXCH << 24, p.rk);
                    const uint64_t Ux = ((uint64_t)w.x << 32) | (uint64_t)w.y;
                    accept = Ux < p.Tx[p.Tx_off[k] + j];
                }
            }
            if (accept) {
                atomicOr(&Mswap[k >> 5], 1u << (k & 31));
                const int64_t te = Ecopy[k];
                Ecopy[k] = Ecopy[k + 1];
                Ecopy[k + 1] = te;
                const int64_t tw = Wcopy[k];
                Wcopy[k] = Wcopy[k + 1];
                Wcopy[k + 1] = tw;
            }
        }
        __syncthreads();
        // move the configurations: within-word pairs by a delta swap; the cross-word pair
        // (32wt-1, 32wt) / (32wt+31, 32wt+32) through the neighbours' boundary bit planes
        const uint32_t Min = Mswap[wt] & 0x7FFFFFFFu;
        const bool cross_lo = wt > 0 && ((Mswap[wt - 1] >> 31) & 1u);
        const bool cross_hi = wt + 1 < KW && ((Mswap[wt] >> 31) & 1u);
        bool any_cross = false;
        for (int q = 0; q + 1 < KW; ++q)
            any_cross |= (Mswap[q] >> 31) & 1u;
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
            const uint32_t *nB31 = cross_lo ? cluster.map_shared_rank(B31, wt - 1) : B31;
            const uint32_t *nB0 = cross_hi ? cluster.map_shared_rank(B0, wt + 1) : B0;
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
                uint32_t w = S[l];
                const uint32_t tt = (w ^ (w >> 1)) & Min;
                S[l] = w ^ tt ^ (tt << 1);
            }
        }
        __syncthreads();
    }

    // ---- outputs
    if (tid < 32) {
        p.E_out[(size_t)gl * 32 + tid] =
            pt && p.n_rounds > 0 ? Ecopy[32 * wt + tid] : 2 * (int64_t)Ucnt[tid] - 2 * (int64_t)n;
        if (pt)
            p.walker[(size_t)c_local * K + 32 * wt + tid] = Wcopy[32 * wt + tid];
    }
    if (pt && wt == 0 && tid == 0) {
        p.copy_best[3 * c_local + 0] = bestE;
        p.copy_best[3 * c_local + 1] = bestSlot;
        p.copy_best[3 * c_local + 2] = bestSweep;
    }
    uint32_t *dst = p.state_out + (size_t)gl * n;
    for (int i = tid; i < n; i += nt) {
        const int y = i / p.Lx, x = i - y * p.Lx;
        dst[i] = S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)];
    }
    if (pt)
        cg::this_cluster().sync();  // no CTA exits while a peer may still read its shared memory
}

cudaError_t launch_grid_bits(const GridBitsParams &p, int32_t G, int32_t threads, size_t smem,
                             cudaStream_t st)
{
    cudaError_t e = cudaFuncSetAttribute(k_grid_bits, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.pt ? (unsigned)p.words_per_copy : 1u;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_grid_bits, p);
}

}  // namespace ising

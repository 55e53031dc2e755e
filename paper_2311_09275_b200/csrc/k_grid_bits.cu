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
// words are then decided and written.  The rest are pushed to the warp's
// shared-memory queue, and the warp finishes them right after its stage 1 with
// all 32 lanes busy (no barrier in between), instead of leaving most lanes of a
// warp idle while one lane draws its 3rd/4th call.
// Philox rounds 0-1 are partially hoisted: the parts that depend only on the
// CTA's group g, the sweep t or the site i are computed once, not per call.
#include "bits_core.cuh"

namespace ising {

using namespace bits;

namespace {

__device__ __forceinline__ int T_m_plus1_off(int tid, int hx)
{
    const int m = tid % hx;
    return m + 1 == hx ? 1 - hx : 1;
}

__device__ __forceinline__ int T_m_minus1_off(int tid, int hx)
{
    const int m = tid % hx;
    return m == 0 ? hx - 1 : -1;
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

// tail-queue item: {l | i_orig << 16, D, acc, m8} (the own word is re-read from S)
constexpr int kGridQItem = 16;

int32_t grid_bits_qcap(int32_t n)
{
    const size_t base = (size_t)4 * n + (((size_t)n + 15) & ~(size_t)15) + 512 +
                        (size_t)8 * ((n + 31) / 32);
    const size_t half = (size_t)n / 2;
    size_t qcap = half;
    const size_t budget = 200 * 1024;
    if (base + qcap * kGridQItem > budget)
        qcap = base < budget ? (budget - base) / kGridQItem : 0;
    return (int32_t)qcap;
}

size_t grid_bits_smem(int32_t n)
{
    // S (4n) + JB (n, padded to 16) + planes (512) + queue + 2 boundary bit planes
    return (size_t)4 * n + (((size_t)n + 15) & ~(size_t)15) + 512 +
           (size_t)grid_bits_qcap(n) * kGridQItem + (size_t)8 * ((n + 31) / 32);
}

// SPILL: the lattice has leftover rows that the column-less warps take (grid_bits_spill);
// a separate instantiation, so lattices without them keep the plain kernel's code
template <bool SPILL>
__global__ void __launch_bounds__(kGridMaxThreads, 1) k_grid_bits(const GridBitsParams p)
{
    extern __shared__ __align__(16) uint32_t sm[];
    // per-replica bond counts, double-buffered by round parity: peers of the cluster read a
    // CTA's counts over DSMEM after a cluster barrier, and the next round writes the other
    // buffer, so no write can overtake a slow peer's read
    __shared__ int32_t Ubuf[2][32];
    // fused PT rounds (cluster of words_per_copy CTAs = one copy): the copy's energies,
    // walker ids, swap mask and best record, held identically by every CTA of the cluster
    __shared__ PtShared ps;
    const int n = p.n;
    const GridGeom G{p.Lx, p.Ly, p.hx, p.half, p.ymagic};
    uint32_t *S = sm;
    uint8_t *JB = reinterpret_cast<uint8_t *>(sm + n);
    uint32_t *P = reinterpret_cast<uint32_t *>(JB + ((n + 15) & ~15));  // P[0..63] dE=4, P[64..127] dE=8
    uint4 *Q4 = reinterpret_cast<uint4 *>(P + 128);  // tail queue (16-byte items)
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nt >> 5;
    const int qcap = p.qcap;
    const int wcap = qcap / nwarps;  // per-warp queue region
    const int nbw = (n + 31) / 32;
    uint32_t *B0 = reinterpret_cast<uint32_t *>(Q4 + qcap);  // boundary bit planes (PT mode)
    uint32_t *B31 = B0 + nbw;
    const int wq0 = warp * wcap;

    RoundKeys rkr;  // round keys held in registers for the whole launch
#pragma unroll
    for (int r = 0; r < 20; ++r)
        rkr.k[r] = p.rk.k[r];
    const int gl = blockIdx.x;
    const uint32_t g = p.g0 + (uint32_t)gl;
    const int KW = p.words_per_copy;
    const int wt = (int)(g % (uint32_t)KW);
    const int K = 32 * KW;
    const bool pt = p.pt != 0;
    const int c_local = gl / KW;
    const uint32_t c_global = g / (uint32_t)KW;

    // 2-D thread mapping: column m = tid % hx of a class row, rows ty + k*rpp
    const int rpp = grid_rows_per_pass(nt, G.hx);  // even when possible (host guarantees >= 1)
    const int npass = (G.Ly + rpp - 1) / rpp;
    // leftover rows beyond the last full pass go to the warps without a class column when
    // they can finish them within the full passes
    const int full_passes = G.Ly / rpp, main_rows = full_passes * rpp;
    const int idle_w0 = (rpp * G.hx + 31) / 32;  // first warp with no column thread
    const int spill_sites = (G.Ly - main_rows) * G.hx;
    const int nidle_all = (nwarps - idle_w0) * 32;
    const int spill_iters = nidle_all > 0 ? (spill_sites + nidle_all - 1) / nidle_all : 0;
    const bool spill = SPILL && spill_sites > 0 && nidle_all > 0 && spill_iters <= full_passes;
    const int npass_main = spill ? full_passes : npass;
    // per-warp stage-2 limit: about one 32-lane round of queued words per 8 passes (~11% of the
    // words stay undecided after stage 1); beyond it a word is finished inline in stage 1, so a
    // warp rarely pays a second, mostly empty stage-2 round after the others are done
    const int wlim = min(wcap, 32 * max(1, (npass_main + 7) / 8));
    // neighbour offsets of a class column: m+1 and m-1 wrapped, rows below/above wrapped
    const int offR1 = T_m_plus1_off(tid, G.hx), offL0 = T_m_minus1_off(tid, G.hx);
    const uint32_t hx4 = 4u * (uint32_t)G.hx;
    const uint32_t wrapDb = 4u * (uint32_t)((1 - G.Ly) * G.hx), wrapUb = 4u * (uint32_t)((G.Ly - 1) * G.hx);
    const uint32_t sS = (uint32_t)__cvta_generic_to_shared(S);
    const uint32_t sJB = (uint32_t)__cvta_generic_to_shared(JB);
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
    if (pt)
        pt_init(ps, p.walker, c_local, K);
    __syncthreads();

    for (int round = 0; round < p.n_rounds; ++round) {
        int32_t *Ucnt = Ubuf[round & 1];
        if (tid < 32)  // zeroed here: the colour-phase barriers order it before the atomicAdds
            Ucnt[tid] = 0;
        // ---- k_ex sweeps
        for (int s = 0; s < p.k_ex; ++s) {
            const uint32_t t = p.t0 + (uint32_t)(round * p.k_ex + s);
            const PlaneUniform U = plane_uniform(g, t, rkr);
            if (p.planes_sched) {  // annealing: this sweep's threshold planes
                __syncthreads();
                const uint32_t *src_p = p.planes_sched + (size_t)(round * p.k_ex + s) * p.words_per_copy * 128;
                for (int j = tid; j < 128; j += nt)
                    P[j] = src_p[wt * 128 + j];
                __syncthreads();
            }
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                uint32_t *Sc = S + c * G.half;
#ifdef ISING_GRID_TIMING
                long long tA = clock64();
#endif
                // stage 1: planes 0..7 for every site; undecided words go to this warp's queue.
                // rpp is even, so a thread's sites all have parity par = (c + ty) & 1 and fixed
                // horizontal neighbour offsets; rows advance by rpp per pass.  Shared-memory
                // addresses are explicit 32-bit byte addresses advanced per pass.
                const int par = (c + T.ty) & 1;
                const int hx = G.hx;
                const uint32_t l0 = (uint32_t)(T.ty * hx + T.m);
                uint32_t aC = sS + 4u * ((uint32_t)(c * G.half) + l0);        // own word
                uint32_t aO = sS + 4u * ((uint32_t)((1 - c) * G.half) + l0);  // same cell, other class
                uint32_t aJ = sJB + (uint32_t)(c * G.half) + l0;
                const uint32_t offRb = 4u * (uint32_t)(par ? offR1 : 0);
                const uint32_t offLb = 4u * (uint32_t)(par ? 0 : offL0);
                const uint32_t rstep = (uint32_t)(rpp * hx), istep = (uint32_t)(G.Lx * rpp);
                uint32_t i_orig = (uint32_t)(2 * T.m + par + G.Lx * T.ty);
                int wq = 0;  // warp-uniform
                int y = T.ty;
#pragma unroll 1
                for (int pass = 0; pass < npass_main;
                     ++pass, y += rpp, aC += 4u * rstep, aO += 4u * rstep, aJ += rstep, i_orig += istep) {
                    const bool valid = T.active && y < G.Ly;
                    uint32_t own = 0, D = 0, acc = 0, m8 = 0;
                    if (valid) {
                        own = lds_u32(aC);
                        const uint32_t xr = lds_u32(aO + offRb);
                        const uint32_t xl = lds_u32(aO + offLb);
                        const uint32_t xd = lds_u32(aO + (y + 1 == G.Ly ? wrapDb : hx4));
                        const uint32_t xu = lds_u32(aO + (y == 0 ? wrapUb : 0u - hx4));
                        const uint32_t jw = lds_u8(aJ) * 0x10204080u;
                        const uint32_t a0 = ~(own ^ xr ^ byte_sign_mask<0>(jw));
                        const uint32_t a1 = ~(own ^ xl ^ byte_sign_mask<1>(jw));
                        const uint32_t a2 = ~(own ^ xd ^ byte_sign_mask<2>(jw));
                        const uint32_t a3 = ~(own ^ xu ^ byte_sign_mask<3>(jw));
                        const uint32_t s01 = a0 ^ a1, c01 = a0 & a1;
                        const uint32_t s23 = a2 ^ a3, c23 = a2 & a3;
                        m8 = ~(s01 | c01 | s23 | c23);                   // u = 0 -> dE = 8
                        const uint32_t m4 = (s01 ^ s23) & ~(c01 | c23);  // u = 1 -> dE = 4
                        D = m8 | m4;
                        acc = ~D;  // dE <= 0 always flips
                        if (D) {  // planes 0..7: both calls issued together (two independent chains)
                            uint32_t sA, sB;
                            plane_site(i_orig, U, rkr, sA, sB);
                            plane_call2(sA, sB, U, rkr, P, m8, D, acc);
                        }
                    }
                    const bool need = D != 0u;
                    const uint32_t pm = __ballot_sync(0xFFFFFFFFu, need);
                    const int slot = wq + __popc(pm & lanemask_lt());
                    wq += __popc(pm);
                    if (need && slot < wlim) {
                        const uint32_t l = (aC - sS) / 4u - (uint32_t)(c * G.half);
                        Q4[wq0 + slot] = make_uint4(l | (i_orig << 16), D, acc, m8);
                    } else if (valid) {
                        if (need) {  // this warp's queue region is full: finish inline
                            uint32_t sA, sB;
                            plane_site(i_orig, U, rkr, sA, sB);
                            uint32_t j4 = 2;
                            do {
                                plane_call(sA, sB, j4, U, rkr, P, m8, D, acc);
                                ++j4;
                            } while (D && j4 < 16u);
                        }
                        sts_u32(aC, own ^ acc);
                    }
                }
                // leftover rows (Ly not a multiple of rpp): the warps that hold no class column
                // take them, concurrently with the main passes, instead of a last partial pass
                // of the column threads (C2: rows 96..99 on the 16th warp, 8 passes per warp
                // instead of 9 for five warps)
                if (SPILL && spill && warp >= idle_w0) {
                    const int nidle = (nwarps - idle_w0) * 32, k0 = tid - idle_w0 * 32;
#pragma unroll 1
                    for (int it = 0; it < spill_iters; ++it) {
                        const int sidx = it * nidle + k0;
                        const bool valid = sidx < spill_sites;
                        const int yy = main_rows + (valid ? sidx / hx : 0);
                        const int mm = valid ? sidx - (sidx / hx) * hx : 0;
                        const int pp = (c + yy) & 1;
                        const uint32_t ll = (uint32_t)(yy * hx + mm);
                        const uint32_t bC = sS + 4u * ((uint32_t)(c * G.half) + ll);
                        const uint32_t bO = sS + 4u * ((uint32_t)((1 - c) * G.half) + ll);
                        const uint32_t bJ = sJB + (uint32_t)(c * G.half) + ll;
                        const int oR = pp ? (mm + 1 == hx ? 1 - hx : 1) : 0;
                        const int oL = pp ? 0 : (mm == 0 ? hx - 1 : -1);
                        const uint32_t io = (uint32_t)(2 * mm + pp + G.Lx * yy);
                        uint32_t own = 0, D = 0, acc = 0, m8 = 0;
                        if (valid) {
                            own = lds_u32(bC);
                            const uint32_t xr = lds_u32(bO + 4u * (uint32_t)oR);
                            const uint32_t xl = lds_u32(bO + 4u * (uint32_t)oL);
                            const uint32_t xd = lds_u32(bO + (yy + 1 == G.Ly ? wrapDb : hx4));
                            const uint32_t xu = lds_u32(bO + (yy == 0 ? wrapUb : 0u - hx4));
                            const uint32_t jw = lds_u8(bJ) * 0x10204080u;
                            const uint32_t a0 = ~(own ^ xr ^ byte_sign_mask<0>(jw));
                            const uint32_t a1 = ~(own ^ xl ^ byte_sign_mask<1>(jw));
                            const uint32_t a2 = ~(own ^ xd ^ byte_sign_mask<2>(jw));
                            const uint32_t a3 = ~(own ^ xu ^ byte_sign_mask<3>(jw));
                            const uint32_t s01 = a0 ^ a1, c01 = a0 & a1;
                            const uint32_t s23 = a2 ^ a3, c23 = a2 & a3;
                            m8 = ~(s01 | c01 | s23 | c23);
                            const uint32_t m4 = (s01 ^ s23) & ~(c01 | c23);
                            D = m8 | m4;
                            acc = ~D;
                            if (D) {
                                uint32_t sA, sB;
                                plane_site(io, U, rkr, sA, sB);
                                plane_call2(sA, sB, U, rkr, P, m8, D, acc);
                            }
                        }
                        const bool need = D != 0u;
                        const uint32_t pm = __ballot_sync(0xFFFFFFFFu, need);
                        const int slot = wq + __popc(pm & lanemask_lt());
                        wq += __popc(pm);
                        if (need && slot < wlim) {
                            Q4[wq0 + slot] = make_uint4(ll | (io << 16), D, acc, m8);
                        } else if (valid) {
                            if (need) {
                                uint32_t sA, sB;
                                plane_site(io, U, rkr, sA, sB);
                                uint32_t j4 = 2;
                                do {
                                    plane_call(sA, sB, j4, U, rkr, P, m8, D, acc);
                                    ++j4;
                                } while (D && j4 < 16u);
                            }
                            sts_u32(bC, own ^ acc);
                        }
                    }
                }
#ifdef ISING_GRID_TIMING
                long long tB = clock64();
#endif
#ifdef ISING_GRID_TIMING
                long long tC = clock64();
#endif
                // stage 2 (own-queue variant): each warp finishes its own queued words right
                // after its stage 1, no barrier in between
                const int nown = min(wq, wlim);
                for (int qb = 0; qb < nown; qb += 32) {
                    const int q = qb + lane;
                    if (q >= nown)
                        continue;
                    const uint4 item = Q4[wq0 + q];
                    const int l = (int)(item.x & 0xFFFFu);
                    const uint32_t i_orig = item.x >> 16;
                    uint32_t D = item.y, acc = item.z;
                    const uint32_t m8 = item.w;
                    uint32_t sA, sB;
                    plane_site(i_orig, U, rkr, sA, sB);
                    plane_call2(sA, sB, U, rkr, P, m8, D, acc, 2u);  // planes 8..15, calls interleaved
                    uint32_t j4 = 4;
                    while (D && j4 < 16u) {
                        plane_call(sA, sB, j4, U, rkr, P, m8, D, acc);
                        ++j4;
                    }
                    const uint32_t a = sS + 4u * ((uint32_t)(c * G.half) + (uint32_t)l);
                    sts_u32(a, lds_u32(a) ^ acc);  // queued words were not written in stage 1
                }
#ifdef ISING_GRID_TIMING
                long long tD = clock64();
#endif
                __syncthreads();
#ifdef ISING_GRID_TIMING
                long long tE = clock64();
                if (blockIdx.x == 0 && lane == 0 && round == 2 && s == 0)
                    printf("T c=%d w=%2d s1=%lld b1=%lld s2=%lld b2=%lld nq=%d wq=%d\n", c, warp, tB - tA, tC - tB,
                           tD - tC, tE - tD, nq, wq);
#endif
            }
        }

        // ---- energy: every bond joins a colour-0 and a colour-1 site, so the four
        // bonds of the colour-1 sites count each bond exactly once.  E = 2U - 2n.
        {
            uint32_t c7[7];  // per-thread counts <= 4 * npass <= 124
#pragma unroll
            for (int l = 0; l < 7; ++l)
                c7[l] = 0;
            const uint32_t *S1 = S + G.half;
            for (int pass = 0; pass < npass; ++pass) {
                const int y = T.ty + pass * rpp;
                if (T.active && y < G.Ly) {
                    uint32_t a0, a1, a2, a3, i_orig;
                    site_unsat(S, JB, G, T, 1, y, S1[y * G.hx + T.m], a0, a1, a2, a3, i_orig);
                    vadd(c7, a0);
                    vadd(c7, a1);
                    vadd(c7, a2);
                    vadd(c7, a3);
                }
            }
            uint32_t cnt[kCntLevels];
#pragma unroll
            for (int l = 0; l < kCntLevels; ++l)
                cnt[l] = l < 7 ? c7[l] : 0u;
            // warp total by a butterfly of bit-sliced additions, then lane b reads bit b
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                vsum_xor(cnt, off);
            int32_t acc = 0;
#pragma unroll
            for (int l = 0; l < kCntLevels; ++l)
                acc += (int32_t)((cnt[l] >> lane) & 1u) << l;
            if (p.k_ex == 0)  // no colour phase (hence no barrier) since the zeroing
                __syncthreads();
            atomicAdd(&Ucnt[lane], acc);
            if (!pt)  // pt_step opens with a cluster barrier
                __syncthreads();
        }
        if (!pt)
            continue;

        // ---- fused PT step for this copy (a7/a8): same result as ising_exchange
        auto snap = [&](int bit) {
            int8_t *dst = p.snap + (size_t)c_local * n;
            for (int i = tid; i < n; i += nt) {
                const int y = i / p.Lx, x = i - y * p.Lx;
                dst[i] = ((S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)] >> bit) & 1u) ? -1 : 1;
            }
        };
        pt_step(ps, Ucnt, 2 * (int64_t)n, S, n, B0, B31, KW, wt, c_global,
                p.t0 + (uint32_t)((round + 1) * p.k_ex), p.e0 + (uint32_t)round, p.Tx, p.Tx_off,
                p.Tx_len, p.rk, snap);
    }

    // ---- outputs
    int32_t *Ucnt = Ubuf[(p.n_rounds - 1) & 1];  // the last round's counts
    pt_finish(ps, pt, p.n_rounds, Ucnt, 2 * (int64_t)n, p.E_out, p.walker, p.copy_best, gl, wt,
              c_local, K);
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
    // the spilling instantiation only where the host-side geometry says rows are left over
    // and the column-less warps can take them within the full passes (same rule as the kernel)
    const int hx = p.hx, rpp = grid_rows_per_pass(threads, hx);
    const int full = p.Ly / rpp, left = (p.Ly - full * rpp) * hx;
    const int nidle = (threads / 32 - (rpp * hx + 31) / 32) * 32;
    const bool spill = left > 0 && nidle > 0 && (left + nidle - 1) / nidle <= full;
    auto kern = spill ? k_grid_bits<true> : k_grid_bits<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace ising

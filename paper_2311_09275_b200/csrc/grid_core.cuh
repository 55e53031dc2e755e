// grid_core.cuh -- the colour-phase update and the bond count of the multi-spin-coded torus
// kernels (k_grid_bits: one CTA per word group for a whole launch; k_grid_sched: persistent
// CTAs that take (word group, round) tasks).  DESIGN.md §5.2.
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
// Shared memory holds the spins in colour-separated order (each colour class contiguous per
// row), so lane l of a warp touches word l of a row: conflict-free LDS/STS for the site and
// all four neighbours.
//
// Work compaction of the RNG tail: stage 1 draws planes 0..7 (two Philox calls) for every
// site, which decides ~89% of words; the undecided ones go to the warp's own shared-memory
// queue and the warp finishes them right after its stage 1 with all lanes busy (no barrier
// in between).
#pragma once
#include "bits_core.cuh"

namespace ising {
namespace grid {

using namespace bits;

// tail-queue item: {l | i_orig << 16, D, acc, m8} (the own word is re-read from S)
constexpr int kGridQItem = 16;

__device__ __forceinline__ void sts_u128(uint32_t a, uint4 v)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

__device__ __forceinline__ uint4 lds_u128(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// Site geometry of one thread in the 2-D mapping (column m of a colour class,
// rows ty, ty + rpp, ...).
struct ThreadGeom {
    int m, mL, mR;  // class column and its wrapped neighbours
    int ty;
    bool active;
};

// Per-launch constants of a thread's mapping (computed once per CTA).
struct Ctx {
    GridGeom G;
    ThreadGeom T;
    int n, tid, nt, lane, warp, nwarps;
    int wq0;          // this warp's queue region
    int rpp;          // class rows per pass (even when possible)
    int npass;        // passes of the full mapping
    int y0, y1;       // the thread block's rows [y0, y1) (a band of the lattice, or all of it)
    int main_rows;    // rows covered by the full passes
    int idle_w0;      // first warp with no column thread
    int spill_sites;  // leftover-row sites taken by the column-less warps
    int spill_iters;
    bool spill;
    int npass_main;   // passes of the column threads (full passes if the leftover rows spill)
    int wlim;         // per-warp stage-2 limit
    int offR1, offL0; // horizontal neighbour offsets of the class column
    uint32_t hx4, wrapDb, wrapUb, sS, sJB;
    uint32_t sQw;     // shared address of this warp's tail-queue region
};

// y0, y1: the rows this thread block updates (band split: one band of the lattice; the rows
// outside it are kept current by the other band).  limit_stage2: cap the per-warp stage-2 queue
// (the band kernel measured faster without the cap).
__device__ __forceinline__ Ctx make_ctx(const GridGeom &G, int n, int qcap, const uint32_t *S, const uint8_t *JB,
                                        const uint4 *Q4, bool SPILL, int y0 = 0, int y1 = -1,
                                        bool limit_stage2 = true)
{
    Ctx X;
    X.G = G;
    X.n = n;
    X.y0 = y0;
    X.y1 = y1 < 0 ? G.Ly : y1;
    const int nrows = X.y1 - X.y0;
    X.tid = threadIdx.x;
    X.nt = blockDim.x;
    X.lane = X.tid & 31;
    X.warp = X.tid >> 5;
    X.nwarps = X.nt >> 5;
    const int wcap = qcap / X.nwarps;
    X.wq0 = X.warp * wcap;
    X.rpp = grid_rows_per_pass(X.nt, G.hx);  // even when possible (host guarantees >= 1)
    X.npass = (nrows + X.rpp - 1) / X.rpp;
    // leftover rows beyond the last full pass go to the warps without a class column when
    // they can finish them within the full passes
    const int full_passes = nrows / X.rpp;
    X.main_rows = X.y0 + full_passes * X.rpp;
    X.idle_w0 = (X.rpp * G.hx + 31) / 32;
    X.spill_sites = (X.y1 - X.main_rows) * G.hx;
    const int nidle_all = (X.nwarps - X.idle_w0) * 32;
    X.spill_iters = nidle_all > 0 ? (X.spill_sites + nidle_all - 1) / nidle_all : 0;
    X.spill = SPILL && X.spill_sites > 0 && nidle_all > 0 && X.spill_iters <= full_passes;
    X.npass_main = X.spill ? full_passes : X.npass;
    // per-warp stage-2 limit: about one 32-lane round of queued words per 8 passes (~11% of the
    // words stay undecided after stage 1); beyond it a word is finished inline in stage 1, so a
    // warp rarely pays a second, mostly empty stage-2 round after the others are done
    X.wlim = limit_stage2 ? min(wcap, 32 * max(1, (X.npass_main + 7) / 8)) : wcap;
    {
        const int m = X.tid % G.hx;
        X.offR1 = m + 1 == G.hx ? 1 - G.hx : 1;
        X.offL0 = m == 0 ? G.hx - 1 : -1;
    }
    X.hx4 = 4u * (uint32_t)G.hx;
    X.wrapDb = 4u * (uint32_t)((1 - G.Ly) * G.hx);
    X.wrapUb = 4u * (uint32_t)((G.Ly - 1) * G.hx);
    X.sS = (uint32_t)__cvta_generic_to_shared(S);
    X.sJB = (uint32_t)__cvta_generic_to_shared(JB);
    X.sQw = (uint32_t)__cvta_generic_to_shared(Q4) + 16u * (uint32_t)X.wq0;
    X.T.ty = X.tid / G.hx;
    X.T.m = X.tid - X.T.ty * G.hx;
    X.T.mL = X.T.m == 0 ? G.hx - 1 : X.T.m - 1;
    X.T.mR = X.T.m + 1 == G.hx ? 0 : X.T.m + 1;
    X.T.active = X.T.ty < X.rpp;
    return X;
}

// Shared-memory index of original site i (colour-separated order).
__device__ __forceinline__ int colsep(const GridGeom &G, int i)
{
    const int y = i / G.Lx, x = i - y * G.Lx;
    return ((x + y) & 1) * G.half + y * G.hx + (x >> 1);
}

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

// The update of one site word: unsatisfied-bond classes, then planes 0..7 (both Philox calls
// issued together: two independent chains).  Returns with D = still undecided lanes.
__device__ __forceinline__ void stage1_site(uint32_t aO, uint32_t offRb, uint32_t offLb, uint32_t offDb,
                                            uint32_t offUb, uint32_t aJ, uint32_t own, uint32_t i_orig,
                                            const PlaneUniform &U, const RoundKeys &rkr, const uint32_t *P,
                                            uint32_t &D, uint32_t &acc, uint32_t &m8)
{
    const uint32_t xr = lds_u32(aO + offRb);
    const uint32_t xl = lds_u32(aO + offLb);
    const uint32_t xd = lds_u32(aO + offDb);
    const uint32_t xu = lds_u32(aO + offUb);
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
    if (D) {
        uint32_t sA, sB;
        plane_site(i_orig, U, rkr, sA, sB);
        plane_call2(sA, sB, U, rkr, P, m8, D, acc);
    }
}

// Finish a word inline (its warp's queue region is full): planes 8.. one call at a time.
__device__ __forceinline__ void finish_inline(uint32_t i_orig, const PlaneUniform &U, const RoundKeys &rkr,
                                              const uint32_t *P, uint32_t m8, uint32_t &D, uint32_t &acc)
{
    uint32_t sA, sB;
    plane_site(i_orig, U, rkr, sA, sB);
    uint32_t j4 = 2;
    do {
        plane_call(sA, sB, j4, U, rkr, P, m8, D, acc);
        ++j4;
    } while (D && j4 < 16u);
}

struct PassConst {
    uint32_t dO;    // other class, same cell (bytes)
    uint32_t jb;    // J bytes of the class
    uint32_t offRb, offLb;  // horizontal neighbour offsets (bytes, within the other class)
    uint32_t rstep, istep;  // per pass: class words (not bytes), original ids
    int c;
};

struct PassState {
    uint32_t aC, lq, i_orig;
    int wq;
};

// One pass of stage 1 for the thread's site in row y (then advances the state to the next
// pass).  WRAP: the pass may hold row 0 or row Ly-1 (vertical neighbours wrap) or rows >= y1.
template <bool WRAP>
__device__ __forceinline__ void pass_site(const Ctx &X, const PassConst &pc, PassState &ps, int y,
                                          const PlaneUniform &U, const RoundKeys &rkr, const uint32_t *P)
{
    const GridGeom &G = X.G;
    const bool valid = X.T.active && (!WRAP || y < X.y1);
    uint32_t own = 0, D = 0, acc = 0, m8 = 0;
    if (valid) {
        own = lds_u32(ps.aC);
        const uint32_t offD = WRAP && y + 1 == G.Ly ? X.wrapDb : X.hx4;
        const uint32_t offU = WRAP && y == 0 ? X.wrapUb : 0u - X.hx4;
        stage1_site(ps.aC + pc.dO, pc.offRb, pc.offLb, offD, offU, pc.jb + ps.lq, own, ps.i_orig, U, rkr, P, D, acc,
                    m8);
    }
    const bool need = D != 0u;
    const uint32_t pm = __ballot_sync(0xFFFFFFFFu, need);
    const int slot = ps.wq + __popc(pm & lanemask_lt());
    ps.wq += __popc(pm);
    if (need && slot < X.wlim) {
        sts_u128(X.sQw + 16u * (uint32_t)slot, make_uint4(ps.lq | (ps.i_orig << 16), D, acc, m8));
    } else if (valid) {
        if (need)
            finish_inline(ps.i_orig, U, rkr, P, m8, D, acc);
        sts_u32(ps.aC, own ^ acc);
    }
    ps.aC += 4u * pc.rstep;
    ps.lq += pc.rstep;
    ps.i_orig += pc.istep;
}

// One colour phase c of sweep t for word group g: stage 1 over the thread's passes (+ the
// leftover rows on the column-less warps), then the warp's own stage-2 queue (X.sQw), then a
// CTA barrier (BARRIER = false: only the warp's, for a caller that ends the phase with a
// cluster barrier).  Spins (X.sS) in colour-separated order; P: the word type's planes.
template <bool SPILL, bool BARRIER = true>
__device__ __forceinline__ void colour_phase(const Ctx &X, int c, const PlaneUniform &U, const RoundKeys &rkr,
                                             const uint32_t *P)
{
    const GridGeom &G = X.G;
    const ThreadGeom &T = X.T;
    // rpp is even, so a thread's sites all have parity par = (c + ty) & 1 and fixed
    // horizontal neighbour offsets; rows advance by rpp per pass.  Shared-memory addresses
    // are explicit 32-bit byte addresses advanced per pass.
    const int ys = X.y0 + T.ty;  // the thread's first row
    const int par = (c + ys) & 1;
    const int hx = G.hx;
    const uint32_t l0 = (uint32_t)(ys * hx + T.m);
    // the site's words: own at aC, neighbours of the other class at aC + dO + (right, left, down,
    // up) offsets, J bytes at jb + lq; dO, jb and the vertical offsets are CTA-uniform
    PassState ps;
    ps.aC = X.sS + 4u * ((uint32_t)(c * G.half) + l0);
    ps.lq = l0;  // the site's index in its class (queue items carry it)
    ps.i_orig = (uint32_t)(2 * T.m + par + G.Lx * ys);
    ps.wq = 0;   // warp-uniform
    const PassConst pc{4u * (uint32_t)((1 - 2 * c) * G.half), X.sJB + (uint32_t)(c * G.half),
                       4u * (uint32_t)(par ? X.offR1 : 0), 4u * (uint32_t)(par ? 0 : X.offL0),
                       (uint32_t)(X.rpp * hx), (uint32_t)(G.Lx * X.rpp), c};
    // rows 0 and Ly-1 (the vertical wrap) can only be in the first and the last pass: the passes
    // in between take the plain offsets and need no row test (their rows lie inside [y0, y1))
    const int np = X.npass_main;
    int y = ys;
    pass_site<true>(X, pc, ps, y, U, rkr, P);
    if (np > 1) {
#pragma unroll 1
        for (int k = 1; k + 1 < np; ++k) {
            y += X.rpp;
            pass_site<false>(X, pc, ps, y, U, rkr, P);
        }
        y += X.rpp;
        pass_site<true>(X, pc, ps, y, U, rkr, P);
    }
    int wq = ps.wq;
    // leftover rows (Ly not a multiple of rpp): the warps that hold no class column take them,
    // concurrently with the main passes, instead of a last partial pass of the column threads
    // (C2: rows 96..99 on the 16th warp, 8 passes per warp instead of 9 for five warps)
    if (SPILL && X.spill && X.warp >= X.idle_w0) {
        const int nidle = (X.nwarps - X.idle_w0) * 32, k0 = X.tid - X.idle_w0 * 32;
#pragma unroll 1
        for (int it = 0; it < X.spill_iters; ++it) {
            const int sidx = it * nidle + k0;
            const bool valid = sidx < X.spill_sites;
            const int yy = X.main_rows + (valid ? sidx / hx : 0);
            const int mm = valid ? sidx - (sidx / hx) * hx : 0;
            const int pp = (c + yy) & 1;
            const uint32_t ll = (uint32_t)(yy * hx + mm);
            const uint32_t bC = X.sS + 4u * ((uint32_t)(c * G.half) + ll);
            const uint32_t bO = X.sS + 4u * ((uint32_t)((1 - c) * G.half) + ll);
            const uint32_t bJ = X.sJB + (uint32_t)(c * G.half) + ll;
            const int oR = pp ? (mm + 1 == hx ? 1 - hx : 1) : 0;
            const int oL = pp ? 0 : (mm == 0 ? hx - 1 : -1);
            const uint32_t io = (uint32_t)(2 * mm + pp + G.Lx * yy);
            uint32_t own = 0, D = 0, acc = 0, m8 = 0;
            if (valid) {
                own = lds_u32(bC);
                stage1_site(bO, 4u * (uint32_t)oR, 4u * (uint32_t)oL, yy + 1 == G.Ly ? X.wrapDb : X.hx4,
                            yy == 0 ? X.wrapUb : 0u - X.hx4, bJ, own, io, U, rkr, P, D, acc, m8);
            }
            const bool need = D != 0u;
            const uint32_t pm = __ballot_sync(0xFFFFFFFFu, need);
            const int slot = wq + __popc(pm & lanemask_lt());
            wq += __popc(pm);
            if (need && slot < X.wlim) {
                sts_u128(X.sQw + 16u * (uint32_t)slot, make_uint4(ll | (io << 16), D, acc, m8));
            } else if (valid) {
                if (need)
                    finish_inline(io, U, rkr, P, m8, D, acc);
                sts_u32(bC, own ^ acc);
            }
        }
    }
    // stage 2 (own-queue variant): each warp finishes its own queued words right after its
    // stage 1, no barrier in between
    const int nown = min(wq, X.wlim);
    for (int qb = 0; qb < nown; qb += 32) {
        const int q = qb + X.lane;
        if (q >= nown)
            continue;
        const uint4 item = lds_u128(X.sQw + 16u * (uint32_t)q);
        const int l = (int)(item.x & 0xFFFFu);
        const uint32_t io = item.x >> 16;
        uint32_t D = item.y, acc = item.z;
        const uint32_t m8 = item.w;
        uint32_t sA, sB;
        plane_site(io, U, rkr, sA, sB);
        plane_call2(sA, sB, U, rkr, P, m8, D, acc, 2u);  // planes 8..15, calls interleaved
        uint32_t j4 = 4;
        while (D && j4 < 16u) {
            plane_call(sA, sB, j4, U, rkr, P, m8, D, acc);
            ++j4;
        }
        const uint32_t a = X.sS + 4u * ((uint32_t)(c * G.half) + (uint32_t)l);
        sts_u32(a, lds_u32(a) ^ acc);  // queued words were not written in stage 1
    }
    if (BARRIER)
        __syncthreads();
    else
        __syncwarp();  // the caller's barrier follows; the warp's own sites are final here
}

// Per-lane count of unsatisfied bonds of the group's 32 replicas (lane b: replica b) over the
// rows [y0, y1): every bond joins a colour-0 and a colour-1 site, so the four bonds of the
// colour-1 sites count each bond exactly once; E = 2U - 2n (band split: the bands' counts add).
__device__ __forceinline__ int32_t unsat_counts(const Ctx &X, const uint32_t *S, const uint8_t *JB)
{
    const GridGeom &G = X.G;
    uint32_t c7[7];  // per-thread counts <= 4 * npass <= 124
#pragma unroll
    for (int l = 0; l < 7; ++l)
        c7[l] = 0;
    const uint32_t *S1 = S + G.half;
    for (int pass = 0; pass < X.npass; ++pass) {
        const int y = X.y0 + X.T.ty + pass * X.rpp;
        if (X.T.active && y < X.y1) {
            uint32_t a0, a1, a2, a3, i_orig;
            site_unsat(S, JB, G, X.T, 1, y, S1[y * G.hx + X.T.m], a0, a1, a2, a3, i_orig);
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
        acc += (int32_t)((cnt[l] >> X.lane) & 1u) << l;
    return acc;
}

}  // namespace grid
}  // namespace ising

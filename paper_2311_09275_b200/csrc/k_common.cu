// k_common.cu -- initialisation, PT exchange, best-so-far, configuration
// moves and diagnostics shared by all sweep kernels (sm_100a).
//
// Rows a2 (init), a7 (replica exchange), a8 (best-so-far / record gather) and
// a9 (readback) of SURVEY.md §8(a).
#include <curand_philox4x32_x.h>

#include "internal.h"

namespace ising {

// ------------------------------------------------------------------ a2: init
// s(r, i) = -1 iff bit (r & 31) of word 0 of Philox(i, 0, r >> 5, INIT << 24)
// (uniform independent spins).
__global__ void k_init_bits(uint32_t *state, int32_t n, const uint32_t *orig, uint32_t g0,
                            const RoundKeys rk)
{
    const int gl = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t io = orig ? orig[i] : (uint32_t)i;
        state[(size_t)gl * n + i] = philox(io, 0u, g0 + (uint32_t)gl, ST_INIT << 24, rk).x;
    }
}

cudaError_t launch_init_bits(uint32_t *state, int32_t G, int32_t n, const uint32_t *orig,
                             uint32_t g0, const RoundKeys &rk, cudaStream_t st)
{
    dim3 grid((unsigned)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184), (unsigned)G);
    k_init_bits<<<grid, 256, 0, st>>>(state, n, orig, g0, rk);
    return cudaGetLastError();
}

__global__ void k_init_i8(int8_t *s, int32_t n, int32_t R, const uint32_t *orig, int64_t slot0,
                          const RoundKeys rk)
{
    const int32_t nq = R >> 2;
    const int64_t total = (int64_t)n * nq;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = (int32_t)(idx / nq), q = (int32_t)(idx % nq);
        const int64_t r = slot0 + 4 * (int64_t)q;
        const uint32_t io = orig ? orig[i] : (uint32_t)i;
        const uint32_t w = philox(io, 0u, (uint32_t)(r >> 5), ST_INIT << 24, rk).x;
        char4 v;
        v.x = ((w >> ((r + 0) & 31)) & 1u) ? -1 : 1;
        v.y = ((w >> ((r + 1) & 31)) & 1u) ? -1 : 1;
        v.z = ((w >> ((r + 2) & 31)) & 1u) ? -1 : 1;
        v.w = ((w >> ((r + 3) & 31)) & 1u) ? -1 : 1;
        reinterpret_cast<char4 *>(s)[idx] = v;
    }
}

cudaError_t launch_init_i8(int8_t *s, int32_t n, int32_t R, const uint32_t *orig, int64_t slot0,
                           const RoundKeys &rk, cudaStream_t st)
{
    k_init_i8<<<148 * 8, 256, 0, st>>>(s, n, R, orig, slot0, rk);
    return cudaGetLastError();
}

// ------------------------------------------------------------ a7/a8: exchange
namespace {

__device__ __forceinline__ bool key_less(int64_t ea, int64_t sa, int64_t eb, int64_t sb, bool is_f)
{
    if (is_f) {
        const double da = __longlong_as_double(ea), db = __longlong_as_double(eb);
        return da < db || (da == db && sa < sb);
    }
    return ea < eb || (ea == eb && sa < sb);
}

__device__ __forceinline__ int8_t spin_of(const ExchangeParams &p, int64_t rl, int32_t i)
{
    const uint32_t j = p.perm_o2i ? p.perm_o2i[i] : (uint32_t)i;
    if (p.layout == 0) {
        const uint32_t w = p.state[(size_t)(rl >> 5) * p.n + j];
        return ((w >> (rl & 31)) & 1u) ? -1 : 1;
    }
    return p.s8[(size_t)j * p.R_local + rl];
}

}  // namespace

// (1) best-so-far: argmin over the candidate records (strict <, ties -> lowest global slot;
// SPEC.md S:261-264); the handle owning the winning slot snapshots its configuration.
// (2) exchange e: per local copy, pairs (k, k+1) with k = e%2 + 2p; d = E_b - E_a; accept iff
// d >= 0 or U64x(k, e, c) < Tx[k][d] = floor(exp((beta_{k+1}-beta_k) d) 2^64) (min(1,
// exp(dbeta dH))).  Accepted pairs swap energies and walker ids here
// and set bit k of the copy's swap mask; the configurations are swapped by k_swap_* right after.
//
// One CTA per group of copies (the work is a few dependent global loads per item, so it is
// latency-bound: spreading it over SMs, not threads, is what shortens it).  Each CTA takes the
// per-copy best of its copies, the best over its candidates (its copies' slots, read before its
// own swaps; or its slice of the gathered records) into xpart, then its copies' exchanges; the
// CTA that finishes last (atomic ticket) merges the partial bests -- (E, slot) is a total order,
// so the merge equals one sequential scan -- updates the record and takes the snapshot.
__global__ void __launch_bounds__(kExThreads) k_exchange(const ExchangeParams p)
{
    __shared__ int64_t wE[kExThreads / 32], wS[kExThreads / 32];
    __shared__ int s_update, s_last;
    __shared__ int64_t s_slot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = (int)(blockDim.x >> 5);
    const bool is_f = p.is_float != 0;
    const int32_t cpb = (p.C_local + (int32_t)gridDim.x - 1) / (int32_t)gridDim.x;
    const int32_t c0 = min(p.C_local, (int32_t)blockIdx.x * cpb), c1 = min(p.C_local, c0 + cpb);
    if (p.do_best) {
        // per-copy best-so-far (trials = copies; NEXT-2 harness): strict <, ties -> lowest slot;
        // one warp per copy (lanes over the temperatures, then a shuffle argmin)
        for (int c = c0 + warp; c < c1; c += nwarps) {
            int64_t bE = 0, bS = -1;
#pragma unroll 4
            for (int k = lane; k < p.K; k += 32) {
                const int64_t e = p.E[(int64_t)c * p.K + k];
                const int64_t sl = p.slot0 + (int64_t)c * p.K + k;
                if (bS < 0 || key_less(e, sl, bE, bS, is_f)) {
                    bE = e;
                    bS = sl;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const int64_t oE = __shfl_down_sync(0xFFFFFFFFu, bE, o);
                const int64_t oS = __shfl_down_sync(0xFFFFFFFFu, bS, o);
                if (oS >= 0 && (bS < 0 || key_less(oE, oS, bE, bS, is_f))) {
                    bE = oE;
                    bS = oS;
                }
            }
            if (lane == 0) {
                int64_t *cb = p.cbest + 3 * c;
                const bool better = cb[1] < 0 || (is_f ? __longlong_as_double(bE) < __longlong_as_double(cb[0])
                                                      : bE < cb[0]);
                if (better) {
                    cb[0] = bE;
                    cb[1] = bS;
                    cb[2] = p.t;
                }
            }
        }
        // this CTA's candidates: its slice of the gathered records, or its copies' slots
        int64_t r0, r1;
        if (p.recs) {
            const int64_t per = (p.n_recs + gridDim.x - 1) / gridDim.x;
            r0 = min(p.n_recs, (int64_t)blockIdx.x * per);
            r1 = min(p.n_recs, r0 + per);
        } else {
            r0 = (int64_t)c0 * p.K;
            r1 = (int64_t)c1 * p.K;
        }
        int64_t bE = 0, bS = -1;
#pragma unroll 4
        for (int64_t r = r0 + tid; r < r1; r += blockDim.x) {
            const int64_t e = p.recs ? p.recs[r].energy : p.E[r];
            const int64_t s = p.recs ? p.recs[r].slot : p.slot0 + r;
            if (s >= 0 && (bS < 0 || key_less(e, s, bE, bS, is_f))) {
                bE = e;
                bS = s;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t oE = __shfl_down_sync(0xFFFFFFFFu, bE, o);
            const int64_t oS = __shfl_down_sync(0xFFFFFFFFu, bS, o);
            if (oS >= 0 && (bS < 0 || key_less(oE, oS, bE, bS, is_f))) {
                bE = oE;
                bS = oS;
            }
        }
        if (lane == 0) {
            wE[warp] = bE;
            wS[warp] = bS;
        }
        __syncthreads();  // (also: every read of this CTA's energies precedes its swaps below)
        if (tid == 0) {
            int64_t E0 = 0, S0 = -1;
            for (int w = 0; w < nwarps; ++w)
                if (wS[w] >= 0 && (S0 < 0 || key_less(wE[w], wS[w], E0, S0, is_f))) {
                    E0 = wE[w];
                    S0 = wS[w];
                }
            p.xpart[2 * blockIdx.x] = E0;
            p.xpart[2 * blockIdx.x + 1] = S0;
            __threadfence();
            s_last = atomicAdd(p.xctr, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            if (warp == 0) {  // the merge: lanes over the CTAs' partials, then a shuffle argmin
                __threadfence();
                int64_t E0 = 0, S0 = -1;
                for (uint32_t q = lane; q < gridDim.x; q += 32) {
                    const int64_t e = __ldcg(p.xpart + 2 * q), sl = __ldcg(p.xpart + 2 * q + 1);
                    if (sl >= 0 && (S0 < 0 || key_less(e, sl, E0, S0, is_f))) {
                        E0 = e;
                        S0 = sl;
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const int64_t oE = __shfl_down_sync(0xFFFFFFFFu, E0, o);
                    const int64_t oS = __shfl_down_sync(0xFFFFFFFFu, S0, o);
                    if (oS >= 0 && (S0 < 0 || key_less(oE, oS, E0, S0, is_f))) {
                        E0 = oE;
                        S0 = oS;
                    }
                }
                if (lane == 0) {
                    *p.xctr = 0u;  // ready for the next launch (stream order)
                    BestDev bd = *p.best;
                    const bool better = S0 >= 0 && (bd.slot < 0 ||
                                                    (is_f ? __longlong_as_double(E0) < __longlong_as_double(bd.energy)
                                                          : E0 < bd.energy));
                    s_update = better ? 1 : 0;
                    s_slot = S0;
                    if (better) {
                        bd.energy = E0;
                        bd.slot = S0;
                        bd.sweep = p.t;
                        bd.owner = (S0 >= p.slot0 && S0 < p.slot0 + p.R_local) ? 1 : 0;
                        *p.best = bd;
                    }
                }
            }
            __syncthreads();
            // the snapshot reads configurations, which k_exchange never changes (k_swap_* does)
            if (s_update && s_slot >= p.slot0 && s_slot < p.slot0 + p.R_local) {
                const int64_t rl = s_slot - p.slot0;
#pragma unroll 4
                for (int32_t i = tid; i < p.n; i += blockDim.x)
                    p.best_spins[i] = spin_of(p, rl, i);
            }
        }
    }
    if (p.do_swap && p.K >= 2) {
        const int32_t wpc = p.words_per_copy;
        for (int idx = c0 * wpc + tid; idx < c1 * wpc; idx += blockDim.x)
            p.swapmask[idx] = 0u;
        __syncthreads();
        const int32_t par = (int32_t)(p.e & 1u);
        const int32_t npairs = (p.K - par) / 2;
        const int64_t total = (int64_t)(c1 - c0) * npairs;
#pragma unroll 2
        for (int64_t idx = tid; idx < total; idx += blockDim.x) {
            const int32_t c = c0 + (int32_t)(idx / npairs);
            const int32_t k = par + 2 * (int32_t)(idx % npairs);
            const int64_t a = (int64_t)c * p.K + k, b = a + 1;
            const int64_t d = p.E[b] - p.E[a];
            bool accept = d >= 0;
            if (!accept) {
                const int64_t j = -d - 1;
                if (j < p.Tx_len[k]) {
                    const uint32_t cg = (uint32_t)(p.slot0 / p.K) + (uint32_t)c;
                    const uint4 w = philox((uint32_t)k, p.e, cg, ST_EXCH << 24, p.rk);
                    const uint64_t U = ((uint64_t)w.x << 32) | (uint64_t)w.y;
                    accept = U < p.Tx[p.Tx_off[k] + j];
                }
            }
            if (accept) {
                atomicOr(&p.swapmask[c * wpc + (k >> 5)], 1u << (k & 31));
                const int64_t te = p.E[a];
                p.E[a] = p.E[b];
                p.E[b] = te;
                const int64_t tw = p.walker[a];
                p.walker[a] = p.walker[b];
                p.walker[b] = tw;
            }
        }
    }
}

cudaError_t launch_exchange(const ExchangeParams &p, cudaStream_t st)
{
    // about 4 copies per CTA, at most kExMaxBlocks CTAs (the partial-best scratch)
    int32_t nb = (p.C_local + 3) / 4;
    nb = nb < 1 ? 1 : (nb > kExMaxBlocks ? kExMaxBlocks : nb);
    k_exchange<<<nb, kExThreads, 0, st>>>(p);
    return cudaGetLastError();
}

// Merge the per-copy best records of a fused PT launch into the handle's best record:
// lexicographic min over copies of (E, sweep, slot) -- the order in which the sequential
// schedule would have met them -- then strict improvement over the previous record.
__global__ void k_merge_copy_best(const int64_t *copy_best, const int8_t *snap, int32_t C_local,
                                  int32_t n, BestDev *best, int8_t *best_spins, int64_t *cbest)
{
    __shared__ int32_t s_win;
    for (int32_t c = threadIdx.x; c < C_local; c += blockDim.x) {  // persistent per-copy records
        const int64_t *r = copy_best + 3 * c;
        int64_t *cb = cbest + 3 * c;
        if (r[1] >= 0 && (cb[1] < 0 || r[0] < cb[0])) {
            cb[0] = r[0];
            cb[1] = r[1];
            cb[2] = r[2];
        }
    }
    if (threadIdx.x == 0) {
        int32_t win = -1;
        for (int32_t c = 0; c < C_local; ++c) {
            const int64_t *r = copy_best + 3 * c;
            if (r[1] < 0)
                continue;
            if (win < 0)
                win = c;
            else {
                const int64_t *w = copy_best + 3 * win;
                if (r[0] < w[0] || (r[0] == w[0] && (r[2] < w[2] || (r[2] == w[2] && r[1] < w[1]))))
                    win = c;
            }
        }
        BestDev b = *best;
        if (win >= 0 && (b.slot < 0 || copy_best[3 * win] < b.energy)) {
            b.energy = copy_best[3 * win];
            b.slot = copy_best[3 * win + 1];
            b.sweep = copy_best[3 * win + 2];
            b.owner = 1;
            *best = b;
        } else {
            win = -1;
        }
        s_win = win;
    }
    __syncthreads();
    if (s_win >= 0)
        for (int32_t i = threadIdx.x; i < n; i += blockDim.x)
            best_spins[i] = snap[(size_t)s_win * n + i];
}

cudaError_t launch_merge_copy_best(const int64_t *copy_best, const int8_t *snap, int32_t C_local,
                                   int32_t n, BestDev *best, int8_t *best_spins, int64_t *cbest,
                                   cudaStream_t st)
{
    k_merge_copy_best<<<1, 1024, 0, st>>>(copy_best, snap, C_local, n, best, best_spins, cbest);
    return cudaGetLastError();
}

// Move configurations of accepted pairs: slots k and k+1 of a copy are bits k and
// k+1 of the copy's K-bit string (words_per_copy words per site).  Delta swap.
template <int KW>
__global__ void k_swap_bits(uint32_t *state, const uint32_t *swapmask, int32_t n, int32_t C_local)
{
    const int c = blockIdx.y;
    uint32_t M[KW];
    bool any = false;
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        M[q] = swapmask[c * KW + q];
        any |= M[q] != 0u;
    }
    if (!any)
        return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t w[KW], t[KW];
#pragma unroll
        for (int q = 0; q < KW; ++q)
            w[q] = state[(size_t)(c * KW + q) * n + i];
#pragma unroll
        for (int q = 0; q < KW; ++q) {
            const uint32_t up = (w[q] >> 1) | (q + 1 < KW ? (w[q + 1 < KW ? q + 1 : q] << 31) : 0u);
            t[q] = (w[q] ^ up) & M[q];
        }
#pragma unroll
        for (int q = 0; q < KW; ++q) {
            w[q] ^= t[q] ^ (t[q] << 1);
            if (q + 1 < KW)
                w[q + 1 < KW ? q + 1 : q] ^= t[q] >> 31;
        }
#pragma unroll
        for (int q = 0; q < KW; ++q)
            state[(size_t)(c * KW + q) * n + i] = w[q];
    }
}

cudaError_t launch_swap_bits(uint32_t *state, const uint32_t *swapmask, int32_t n, int32_t C_local,
                             int32_t words_per_copy, cudaStream_t st)
{
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)C_local);
    switch (words_per_copy) {
    case 1: k_swap_bits<1><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 2: k_swap_bits<2><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 3: k_swap_bits<3><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 4: k_swap_bits<4><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 5: k_swap_bits<5><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 6: k_swap_bits<6><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 7: k_swap_bits<7><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    case 8: k_swap_bits<8><<<grid, 256, 0, st>>>(state, swapmask, n, C_local); break;
    default: return cudaErrorInvalidValue;  // K > 256 rejected at create
    }
    return cudaGetLastError();
}

__global__ void k_swap_i8(int8_t *s, const uint32_t *swapmask, int32_t n, int32_t R, int32_t K)
{
    const int c = blockIdx.y;
    const int wpc = (K + 31) / 32;
    bool any = false;
    for (int q = 0; q < wpc; ++q)
        any |= swapmask[c * wpc + q] != 0u;
    if (!any)
        return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int8_t *row = s + (size_t)i * R + (size_t)c * K;
        for (int q = 0; q < wpc; ++q) {
            uint32_t m = swapmask[c * wpc + q];
            while (m) {
                const int k = 32 * q + __ffs(m) - 1;
                m &= m - 1;
                const int8_t a = row[k];
                row[k] = row[k + 1];
                row[k + 1] = a;
            }
        }
    }
}

cudaError_t launch_swap_i8(int8_t *s, const uint32_t *swapmask, int32_t n, int32_t R, int32_t K,
                           cudaStream_t st)
{
    const int32_t C_local = R / K;
    dim3 grid((unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), (unsigned)C_local);
    k_swap_i8<<<grid, 256, 0, st>>>(s, swapmask, n, R, K);
    return cudaGetLastError();
}

__global__ void k_records(const int64_t *E, ising_record *out, int64_t R, int64_t slot0)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        ising_record rec;
        rec.energy = E[r];
        rec.slot = slot0 + r;
        out[r] = rec;
    }
}

cudaError_t launch_records(const int64_t *E, ising_record *out, int64_t R, int64_t slot0,
                           cudaStream_t st)
{
    k_records<<<(unsigned)((R + 255) / 256 < 1024 ? (R + 255) / 256 : 1024), 256, 0, st>>>(E, out, R,
                                                                                        slot0);
    return cudaGetLastError();
}

// Global best over per-rank best records {E, sweep, slot} (slot < 0: none): the
// lexicographic minimum of (E, sweep, slot) -- lowest energy, then first reached, then lowest
// slot -- as multi-process runs merge their ranks' ising_best records
// (ising_merge_best).  E is an int64 or the bits of a double.  One CTA; out[3] = the winner
// (slot -1 if no record has one).
__device__ __forceinline__ bool best_less(const int64_t *a, const int64_t *b, int32_t is_float)
{
    if (b[2] < 0)
        return a[2] >= 0;
    if (a[2] < 0)
        return false;
    if (is_float) {
        const double ea = __longlong_as_double(a[0]), eb = __longlong_as_double(b[0]);
        if (ea != eb)
            return ea < eb;
    } else if (a[0] != b[0]) {
        return a[0] < b[0];
    }
    return a[1] != b[1] ? a[1] < b[1] : a[2] < b[2];
}

__global__ void k_merge_best(const int64_t *recs, int64_t n, int32_t is_float, int64_t *out)
{
    __shared__ int64_t sk[1024][3];
    int64_t k[3] = {0, -1, -1};
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t c[3] = {recs[3 * i], recs[3 * i + 1], recs[3 * i + 2]};
        if (best_less(c, k, is_float)) {
            k[0] = c[0];
            k[1] = c[1];
            k[2] = c[2];
        }
    }
    sk[threadIdx.x][0] = k[0];
    sk[threadIdx.x][1] = k[1];
    sk[threadIdx.x][2] = k[2];
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s && best_less(sk[threadIdx.x + s], sk[threadIdx.x], is_float)) {
            sk[threadIdx.x][0] = sk[threadIdx.x + s][0];
            sk[threadIdx.x][1] = sk[threadIdx.x + s][1];
            sk[threadIdx.x][2] = sk[threadIdx.x + s][2];
        }
        __syncthreads();
    }
    if (threadIdx.x < 3)
        out[threadIdx.x] = sk[0][threadIdx.x];
}

cudaError_t launch_merge_best(const int64_t *recs, int64_t n, int32_t is_float, int64_t *out, cudaStream_t st)
{
    k_merge_best<<<1, 1024, 0, st>>>(recs, n, is_float, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a9: readback
__global__ void k_extract_bits(const uint32_t *state, int32_t n, int32_t gl, int32_t bit,
                               const uint32_t *perm_o2i, int8_t *out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t j = perm_o2i ? perm_o2i[i] : (uint32_t)i;
        out[i] = ((state[(size_t)gl * n + j] >> bit) & 1u) ? -1 : 1;
    }
}

cudaError_t launch_extract_bits(const uint32_t *state, int32_t n, int32_t gl, int32_t bit,
                                const uint32_t *perm_o2i, int8_t *out, cudaStream_t st)
{
    k_extract_bits<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(state, n, gl, bit, perm_o2i, out);
    return cudaGetLastError();
}

__global__ void k_insert_bits(uint32_t *state, int32_t n, int32_t gl, int32_t bit,
                              const uint32_t *perm_o2i, const int8_t *in)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t j = perm_o2i ? perm_o2i[i] : (uint32_t)i;
        uint32_t *w = state + (size_t)gl * n + j;
        const uint32_t m = 1u << bit;
        *w = (in[i] < 0) ? (*w | m) : (*w & ~m);
    }
}

cudaError_t launch_insert_bits(uint32_t *state, int32_t n, int32_t gl, int32_t bit,
                               const uint32_t *perm_o2i, const int8_t *in, cudaStream_t st)
{
    k_insert_bits<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(state, n, gl, bit, perm_o2i, in);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ diagnostics
__global__ void k_debug_philox(const uint32_t *in, int32_t n, uint32_t *out_lib, uint32_t *out_cur)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const uint32_t *a = in + 6 * i;
    RoundKeys rk;
    uint32_t k0 = a[4], k1 = a[5];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = k0;
        rk.k[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    const uint4 m = philox(a[0], a[1], a[2], a[3], rk);
    const uint4 c = curand_Philox4x32_10(make_uint4(a[0], a[1], a[2], a[3]), make_uint2(a[4], a[5]));
    out_lib[4 * i + 0] = m.x; out_lib[4 * i + 1] = m.y; out_lib[4 * i + 2] = m.z; out_lib[4 * i + 3] = m.w;
    out_cur[4 * i + 0] = c.x; out_cur[4 * i + 1] = c.y; out_cur[4 * i + 2] = c.z; out_cur[4 * i + 3] = c.w;
}

cudaError_t launch_debug_philox(const uint32_t *in, int32_t n, uint32_t *out_lib,
                                uint32_t *out_curand, cudaStream_t st)
{
    k_debug_philox<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(in, n, out_lib, out_curand);
    return cudaGetLastError();
}

}  // namespace ising

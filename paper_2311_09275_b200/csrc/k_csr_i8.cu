// k_csr_i8.cu -- per-lane Metropolis on int8 spins over a CSR graph (sm_100a).
//
// Rows a3-a4 (field + decision + flip) for the I8 layout: any int32 or float32
// couplings (C5: random 3-regular with N(0,1) float32 weights; C1 torus in
// int8).  Spins are stored s[v][r] (internal vertex v, local replica r,
// replica-minor), so a warp that owns 128 consecutive replicas of one vertex
// reads every neighbour row as one coalesced 128-byte segment.
//
// One thread = (vertex of the current colour class, 4 consecutive replicas as
// char4).  Field h = sum_j w_ij s_j: exact int32 for integer weights; for float
// weights a left fold in the CSR row order with round-to-nearest adds and no
// contraction (h = ((0 + t0) + t1) + t2, t = +-w) -- the order is part of the
// contract.  dE = -2 s h.  dE <= 0 accepts
// without drawing randomness; otherwise the WORD contract draws
// hi = word (r&3) of Philox(i, t, r>>2, WORD_HI<<24) and, only if
// hi == T >> 32, lo from the WORD_LO stream: accept iff (hi<<32 | lo) < T,
// T = floor(exp(-beta_k dE) 2^64) (integer: host table; float: the float32
// contract exponential cexp32 below).
#include "internal.h"

namespace ising {

namespace {

// Float32 contract exponential, x <= 0.
__device__ __forceinline__ float cexp32(float x)
{
    if (x < -64.0f)
        return 0.0f;
    const float k = floorf(__fmul_rn(x, 0x1.715476p+0f));
    float r = __fmaf_rn(-k, 0x1.62e400p-1f, x);
    r = __fmaf_rn(-k, 0x1.7f7d1cp-20f, r);
    float p = 0x1.71de3ap-19f;
    p = __fmaf_rn(p, r, 0x1.a01a02p-16f);
    p = __fmaf_rn(p, r, 0x1.a01a02p-13f);
    p = __fmaf_rn(p, r, 0x1.6c16c2p-10f);
    p = __fmaf_rn(p, r, 0x1.111112p-7f);
    p = __fmaf_rn(p, r, 0x1.555556p-5f);
    p = __fmaf_rn(p, r, 0x1.555556p-3f);
    p = __fmaf_rn(p, r, 0x1p-1f);
    p = __fmaf_rn(p, r, 0x1p+0f);
    p = __fmaf_rn(p, r, 0x1p+0f);
    // 2^k with k in [-93, 0]: a normal float, so the product is exact
    return __fmul_rn(p, __int_as_float(((int)k + 127) << 23));
}

__device__ __forceinline__ uint64_t thr_f32(float betaf, float dE)
{
    const float x = -__fmul_rn(betaf, dE);
    const float v = __fmul_rn(cexp32(x), 0x1p64f);
    if (v >= 0x1p64f)
        return ~0ull;
    return __float2ull_rz(v);
}

// Fast, exact decision of (hi:lo) < floor(cexp32(x) 2^64) for x = -(beta dE) < 0 from the
// 32-bit word hi alone when it is far from the threshold: e = ex2.approx(
// fma(x, log2 e, 32)) estimates cexp32(x) 2^32 with relative error <= 2^-13 (verified
// exhaustively over every float x in [-64, 0] by ising_debug_exp_bound, which evaluates this
// exact expression); margin 2^-12.  For x < -64 (contract threshold 0) e < 2^-60, so only
// hi = 0 stays undecided and the exact path rejects it.  Returns 1 = accept, 0 = reject,
// -1 = undecided (caller evaluates the exact threshold).
__device__ __forceinline__ float exp_est32(float x)
{
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmaf_rn(x, 0x1.715476p+0f, 32.0f)));
    return e;
}

__device__ __forceinline__ int fast_decide(float x, uint32_t hi)
{
    const float e = exp_est32(x);
    const float hf = __uint2float_rn(hi);
    const bool acc = hf <= __fmaf_rn(e, 1.0f - 0x1p-12f, -2.0f);
    const bool rej = hf >= __fmul_rn(e, 1.0f + 0x1p-12f);
    return acc ? 1 : (rej ? 0 : -1);
}

}  // namespace

// Exhaustive check of the fast-decision bound: max over all float x in [-64, 0] of
// |exp_est32(x) / (cexp32(x) 2^32) - 1|, as float bits in *out (atomicMax).
__global__ void k_debug_exp_bound(uint32_t *out)
{
    const uint32_t lo = 0x80000000u, hi = 0xC2800000u;  // -0 .. -64
    float worst = 0.f;
    for (uint64_t b = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= hi;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((uint32_t)b);
        const float e = exp_est32(x);
        const float c = __fmul_rn(cexp32(x), 0x1p32f);
        const float rel = fabsf(e / c - 1.0f);
        worst = fmaxf(worst, rel);
    }
    atomicMax(out, __float_as_uint(worst));
}

cudaError_t launch_debug_exp_bound(uint32_t *out, cudaStream_t st)
{
    k_debug_exp_bound<<<148 * 8, 256, 0, st>>>(out);
    return cudaGetLastError();
}

// One thread = (vertex of the current colour class, W words = 4W consecutive replicas).
// ELL: neighbours from the padded 4-wide table (one 16-byte load per vertex, pad = -1)
// instead of row_ptr -> col -> spins, so a neighbour-row load depends on one load only.
template <bool FLOAT, bool ELL, int W>
__global__ void __launch_bounds__(256, 4) k_csr_i8_phase(const CsrI8Params p)
{
    const uint32_t rw = (uint32_t)p.R >> 2;  // 32-bit words per vertex row
    const uint32_t ntv = rw / W;             // threads per vertex
    const uint32_t total = (uint32_t)(p.v_end - p.v_begin) * ntv;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t *s32 = reinterpret_cast<const uint32_t *>(p.s);
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const uint32_t vv = p.nq_shift >= 0 ? idx >> p.nq_shift : idx / ntv;
        const uint32_t o = idx - vv * ntv;
        const int32_t v = p.v_begin + (int32_t)vv;
        const uint32_t wbase = (uint32_t)v * rw + o * W;  // first own word
        uint32_t own[W];
        if (W == 2) {
            const uint2 t2 = *reinterpret_cast<const uint2 *>(s32 + wbase);
            own[0] = t2.x;
            own[W - 1] = t2.y;
        } else {
            own[0] = s32[wbase];
        }
        float hf[4 * W];
        int32_t hi[4 * W];
#pragma unroll
        for (int a = 0; a < 4 * W; ++a) {
            hf[a] = 0.f;
            hi[a] = 0;
        }
        auto accumulate = [&](const uint32_t (&nb)[W], uint32_t wb) {
#pragma unroll
            for (int w = 0; w < W; ++w)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (FLOAT) {
                        // term = s_j > 0 ? w : -w == w with its sign bit xor-ed by s_j's sign bit
                        const uint32_t sb = (nb[w] << (24 - 8 * b)) & 0x80000000u;
                        hf[4 * w + b] = __fadd_rn(hf[4 * w + b], __uint_as_float(wb ^ sb));
                    } else {
                        hi[4 * w + b] += (int32_t)wb * (int32_t)(int8_t)(nb[w] >> (8 * b));
                    }
                }
        };
        auto load_nb = [&](int32_t j, uint32_t (&nb)[W]) {
            const uint32_t a = (uint32_t)j * rw + o * W;
            if (W == 2) {
                const uint2 t2 = __ldg(reinterpret_cast<const uint2 *>(s32 + a));
                nb[0] = t2.x;
                nb[W - 1] = t2.y;
            } else {
                nb[0] = __ldg(s32 + a);
            }
        };
        if (ELL) {
            const int4 c = __ldg(reinterpret_cast<const int4 *>(p.ell_col) + v);
            const int4 wv = __ldg(reinterpret_cast<const int4 *>(p.ell_w) + v);
            const int32_t cs[4] = {c.x, c.y, c.z, c.w};
            const uint32_t ws[4] = {(uint32_t)wv.x, (uint32_t)wv.y, (uint32_t)wv.z, (uint32_t)wv.w};
            uint32_t nbv[4][W];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (cs[u] >= 0)
                    load_nb(cs[u], nbv[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (cs[u] >= 0)  // row order: ELL slots keep the CSR order, pads at the end
                    accumulate(nbv[u], ws[u]);
        } else {
            const int32_t e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
            for (int32_t eb = e0; eb < e1; eb += 4) {
                const int32_t cnt = e1 - eb < 4 ? e1 - eb : 4;
                uint32_t nbv[4][W];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < cnt)
                        load_nb(__ldg(p.col + eb + u), nbv[u]);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < cnt)
                        accumulate(nbv[u], FLOAT ? __float_as_uint(__ldg(p.wf + eb + u))
                                                 : (uint32_t)__ldg(p.wi + eb + u));
            }
        }
        uint32_t fm[W];
        const uint32_t io = __ldg(p.orig + v);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t r0 = 4u * (o * W + w);  // local replica of byte 0 of this word
            const uint32_t quad = (uint32_t)(p.slot0 >> 2) + o * W + w;
            bool flip[4];
            if (FLOAT) {
                float dEv[4], x[4];
                bool need = false;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    // s h (the own spin's sign bit xor-ed into h); dE = -2 s h is exact, so
                    // dE <= 0 <=> s h >= 0 and x = -(beta dE) = RN((2 beta) * (s h)) exactly
                    const uint32_t sbit = (own[w] << (24 - 8 * b)) & 0x80000000u;
                    const float sh = __uint_as_float(__float_as_uint(hf[4 * w + b]) ^ sbit);
                    dEv[b] = -2.0f * sh;
                    flip[b] = sh >= 0.0f;
                    x[b] = __fmul_rn(__ldg(p.betaf + r0 + b), sh);  // betaf holds 2 beta_k
                    need |= !flip[b];
                }
                if (need) {
                    const uint4 h4 = philox(io, p.t, quad, ST_WORD_HI << 24, p.rk);
                    const uint32_t hw[4] = {h4.x, h4.y, h4.z, h4.w};
                    int dec[4];
                    bool undecided = false;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        dec[b] = flip[b] ? 1 : fast_decide(x[b], hw[b]);
                        undecided |= dec[b] < 0;
                    }
                    if (undecided) {  // rare: exact contract threshold; lo word only on a hi tie
                        uint64_t T[4];
                        bool tie = false;
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            T[b] = 0;
                            if (dec[b] < 0) {
                                T[b] = thr_f32(0.5f * __ldg(p.betaf + r0 + b), dEv[b]);
                                const uint32_t th = (uint32_t)(T[b] >> 32);
                                dec[b] = hw[b] < th ? 1 : (hw[b] > th ? 0 : -1);
                                tie |= dec[b] < 0;
                            }
                        }
                        if (tie) {
                            const uint4 l4 = philox(io, p.t, quad, ST_WORD_LO << 24, p.rk);
                            const uint32_t lw[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                            for (int b = 0; b < 4; ++b)
                                if (dec[b] < 0)
                                    dec[b] = lw[b] < (uint32_t)T[b] ? 1 : 0;
                        }
                    }
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        flip[b] = dec[b] == 1;
                }
            } else {
                uint64_t T[4];
                bool need = false;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int32_t sv = (int32_t)(int8_t)(own[w] >> (8 * b));
                    const int32_t dE = -2 * sv * hi[4 * w + b];  // |h| < 2^30
                    flip[b] = dE <= 0;
                    T[b] = 0;
                    if (!flip[b]) {
                        T[b] = __ldg(p.T + (size_t)(r0 + b) * (p.qmax + 1) + (dE >> 1));
                        need = true;
                    }
                }
                if (need) {
                    const uint4 h4 = philox(io, p.t, quad, ST_WORD_HI << 24, p.rk);
                    const uint32_t hw[4] = {h4.x, h4.y, h4.z, h4.w};
                    bool tie = false;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        if (!flip[b]) {
                            const uint32_t th = (uint32_t)(T[b] >> 32);
                            flip[b] = hw[b] < th;
                            tie |= hw[b] == th;
                        }
                    }
                    if (tie) {
                        const uint4 l4 = philox(io, p.t, quad, ST_WORD_LO << 24, p.rk);
                        const uint32_t lw[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            if (!flip[b] && hw[b] == (uint32_t)(T[b] >> 32))
                                flip[b] = lw[b] < (uint32_t)T[b];
                    }
                }
            }
            // +1 (0x01) <-> -1 (0xFF): xor the byte with 0xFE
            fm[w] = (flip[0] ? 0x000000FEu : 0u) | (flip[1] ? 0x0000FE00u : 0u) |
                    (flip[2] ? 0x00FE0000u : 0u) | (flip[3] ? 0xFE000000u : 0u);
        }
        uint32_t *dst = const_cast<uint32_t *>(s32) + wbase;
        if (W == 2)
            *reinterpret_cast<uint2 *>(dst) = make_uint2(own[0] ^ fm[0], own[W - 1] ^ fm[W - 1]);
        else
            dst[0] = own[0] ^ fm[0];
    }
}

cudaError_t launch_csr_i8_phase(const CsrI8Params &p, int32_t threads, cudaStream_t st)
{
    const int32_t W = (p.R % 8 == 0) ? 2 : 1;
    const int64_t total = (int64_t)(p.v_end - p.v_begin) * (p.R / (4 * W));
    if (total <= 0)
        return cudaSuccess;
    if (total >= ((int64_t)1 << 32))
        return cudaErrorInvalidValue;
    const int64_t want = (total + threads - 1) / threads;
    const unsigned blocks = (unsigned)(want < 148 * 32 ? want : 148 * 32);
    const bool ell = p.ell_col != nullptr;
#define LAUNCH(F, E, WW) k_csr_i8_phase<F, E, WW><<<blocks, threads, 0, st>>>(p)
    if (p.wf) {
        if (ell) { if (W == 2) LAUNCH(true, true, 2); else LAUNCH(true, true, 1); }
        else { if (W == 2) LAUNCH(true, false, 2); else LAUNCH(true, false, 1); }
    } else {
        if (ell) { if (W == 2) LAUNCH(false, true, 2); else LAUNCH(false, true, 1); }
        else { if (W == 2) LAUNCH(false, false, 2); else LAUNCH(false, false, 1); }
    }
#undef LAUNCH
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a6: energy
// E_r = sum over edges {v, j}, j > v (internal ids; each edge once) of
// w s_v s_j.  Two passes with a fixed reduction order (deterministic for
// float64 too): per-block partials over a vertex range, then a per-replica sum
// over blocks in block order.
namespace {
constexpr int kEnergyBlocks = 1184;
}

size_t energy_i8_scratch(int32_t n, int32_t R)
{
    (void)n;
    return (size_t)kEnergyBlocks * R * sizeof(double);
}

template <bool FLOAT>
__global__ void __launch_bounds__(256) k_energy_i8_partial(const int8_t *s, const int32_t *rp,
                                                           const int32_t *col, const int32_t *wi,
                                                           const float *wf, int32_t n, int32_t R,
                                                           void *partials)
{
    __shared__ double red[256 * 4];
    const int32_t nq = R >> 2;
    const int32_t qs = nq < 256 ? nq : 256;
    const int32_t nsub = 256 / qs;
    const int tid = threadIdx.x;
    const int32_t sub = tid / qs, ql = tid % qs;
    const int32_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int32_t v0 = blockIdx.x * chunk, v1 = min(n, v0 + chunk);
    for (int32_t q0 = 0; q0 < nq; q0 += qs) {
        const int32_t q = q0 + ql;
        double accf[4] = {0, 0, 0, 0};
        long long acci[4] = {0, 0, 0, 0};
        if (sub < nsub && q < nq) {
            for (int32_t v = v0 + sub; v < v1; v += nsub) {
                const char4 sv = reinterpret_cast<const char4 *>(s + (size_t)v * R)[q];
                for (int32_t e = rp[v]; e < rp[v + 1]; ++e) {
                    const int32_t j = col[e];
                    if (j <= v)
                        continue;
                    const char4 sj = reinterpret_cast<const char4 *>(s + (size_t)j * R)[q];
                    if (FLOAT) {
                        const double w = (double)wf[e];
                        accf[0] += w * (double)(sv.x * sj.x);
                        accf[1] += w * (double)(sv.y * sj.y);
                        accf[2] += w * (double)(sv.z * sj.z);
                        accf[3] += w * (double)(sv.w * sj.w);
                    } else {
                        const long long w = wi[e];
                        acci[0] += w * (sv.x * sj.x);
                        acci[1] += w * (sv.y * sj.y);
                        acci[2] += w * (sv.z * sj.z);
                        acci[3] += w * (sv.w * sj.w);
                    }
                }
            }
        }
        // fixed-order reduction over `sub` for each quad
        for (int a = 0; a < 4; ++a)
            red[tid * 4 + a] = FLOAT ? accf[a] : __longlong_as_double(acci[a]);
        __syncthreads();
        if (sub == 0 && q < nq) {
            double sf[4] = {0, 0, 0, 0};
            long long si[4] = {0, 0, 0, 0};
            for (int32_t u = 0; u < nsub; ++u)
                for (int a = 0; a < 4; ++a) {
                    const double x = red[(u * qs + ql) * 4 + a];
                    if (FLOAT)
                        sf[a] += x;
                    else
                        si[a] += __double_as_longlong(x);
                }
            for (int a = 0; a < 4; ++a) {
                if (FLOAT)
                    reinterpret_cast<double *>(partials)[(size_t)blockIdx.x * R + 4 * q + a] = sf[a];
                else
                    reinterpret_cast<long long *>(partials)[(size_t)blockIdx.x * R + 4 * q + a] = si[a];
            }
        }
        __syncthreads();
    }
}

template <bool FLOAT>
__global__ void k_energy_i8_final(const void *partials, int32_t nblk, int32_t R, int64_t *Ei,
                                  double *Ef)
{
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R)
        return;
    if (FLOAT) {
        double s = 0.0;
        for (int32_t b = 0; b < nblk; ++b)
            s += reinterpret_cast<const double *>(partials)[(size_t)b * R + r];
        Ef[r] = s;
        Ei[r] = __double_as_longlong(s);
    } else {
        long long s = 0;
        for (int32_t b = 0; b < nblk; ++b)
            s += reinterpret_cast<const long long *>(partials)[(size_t)b * R + r];
        Ei[r] = s;
    }
}

cudaError_t launch_energy_i8(const int8_t *s, const int32_t *rp, const int32_t *col,
                             const int32_t *wi, const float *wf, int32_t n, int32_t R,
                             int64_t *Ei, double *Ef, void *scratch, size_t scratch_bytes,
                             cudaStream_t st)
{
    int32_t nblk = kEnergyBlocks;
    if (n < nblk * 8)
        nblk = (n + 7) / 8;
    if ((size_t)nblk * R * sizeof(double) > scratch_bytes)
        return cudaErrorInvalidValue;
    if (wf) {
        k_energy_i8_partial<true><<<nblk, 256, 0, st>>>(s, rp, col, wi, wf, n, R, scratch);
        k_energy_i8_final<true><<<(R + 127) / 128, 128, 0, st>>>(scratch, nblk, R, Ei, Ef);
    } else {
        k_energy_i8_partial<false><<<nblk, 256, 0, st>>>(s, rp, col, wi, wf, n, R, scratch);
        k_energy_i8_final<false><<<(R + 127) / 128, 128, 0, st>>>(scratch, nblk, R, Ei, Ef);
    }
    return cudaGetLastError();
}

}  // namespace ising

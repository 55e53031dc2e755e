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

template <bool FLOAT>
__device__ __forceinline__ void field4(const CsrI8Params &p, int32_t v, int32_t q, int32_t (&hi)[4],
                                       float (&hf)[4])
{
    const int32_t e0 = p.rp[v], e1 = p.rp[v + 1];
    for (int32_t e = e0; e < e1; ++e) {
        const int32_t j = __ldg(p.col + e);
        const char4 nb = reinterpret_cast<const char4 *>(p.s + (size_t)j * p.R)[q];
        if (FLOAT) {
            const float w = __ldg(p.wf + e);
            hf[0] = __fadd_rn(hf[0], nb.x > 0 ? w : -w);
            hf[1] = __fadd_rn(hf[1], nb.y > 0 ? w : -w);
            hf[2] = __fadd_rn(hf[2], nb.z > 0 ? w : -w);
            hf[3] = __fadd_rn(hf[3], nb.w > 0 ? w : -w);
        } else {
            const int32_t w = __ldg(p.wi + e);
            hi[0] += w * nb.x;
            hi[1] += w * nb.y;
            hi[2] += w * nb.z;
            hi[3] += w * nb.w;
        }
    }
}

}  // namespace

template <bool FLOAT>
__global__ void __launch_bounds__(256) k_csr_i8_phase(const CsrI8Params p)
{
    const int32_t nq = p.R >> 2;
    const int64_t total = (int64_t)(p.v_end - p.v_begin) * nq;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = p.v_begin + (int32_t)(idx / nq);
        const int32_t q = (int32_t)(idx % nq);
        char4 *own_p = reinterpret_cast<char4 *>(p.s + (size_t)v * p.R) + q;
        const char4 own = *own_p;
        int32_t hi[4] = {0, 0, 0, 0};
        float hf[4] = {0.f, 0.f, 0.f, 0.f};
        field4<FLOAT>(p, v, q, hi, hf);
        const int8_t sv[4] = {own.x, own.y, own.z, own.w};
        bool flip[4];
        uint64_t T[4];
        bool need = false;
        const int64_t r0 = p.slot0 + 4 * (int64_t)q;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int32_t k = (int32_t)((4 * q + a) % p.K);
            if (FLOAT) {
                const float dE = sv[a] > 0 ? __fmul_rn(-2.0f, hf[a]) : __fmul_rn(2.0f, hf[a]);
                flip[a] = dE <= 0.0f;
                T[a] = flip[a] ? 0ull : thr_f32(p.betaf[k], dE);
            } else {
                const int64_t dE = -2 * (int64_t)sv[a] * (int64_t)hi[a];
                flip[a] = dE <= 0;
                T[a] = flip[a] ? 0ull : __ldg(p.T + (size_t)k * (p.qmax + 1) + (dE >> 1));
            }
            need |= !flip[a];
        }
        if (need) {
            const uint32_t io = __ldg(p.orig + v);
            const uint32_t quad = (uint32_t)(r0 >> 2);
            const uint4 h4 = philox(io, p.t, quad, ST_WORD_HI << 24, p.rk);
            const uint32_t hw[4] = {h4.x, h4.y, h4.z, h4.w};
            bool tie = false;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                if (!flip[a]) {
                    const uint32_t th = (uint32_t)(T[a] >> 32);
                    flip[a] = hw[a] < th;
                    tie |= hw[a] == th;
                }
            }
            if (tie) {
                const uint4 l4 = philox(io, p.t, quad, ST_WORD_LO << 24, p.rk);
                const uint32_t lw[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                for (int a = 0; a < 4; ++a)
                    if (!flip[a] && hw[a] == (uint32_t)(T[a] >> 32))
                        flip[a] = lw[a] < (uint32_t)T[a];
            }
        }
        char4 out;
        out.x = flip[0] ? -own.x : own.x;
        out.y = flip[1] ? -own.y : own.y;
        out.z = flip[2] ? -own.z : own.z;
        out.w = flip[3] ? -own.w : own.w;
        *own_p = out;
    }
}

cudaError_t launch_csr_i8_phase(const CsrI8Params &p, int32_t threads, cudaStream_t st)
{
    const int64_t total = (int64_t)(p.v_end - p.v_begin) * (p.R >> 2);
    if (total <= 0)
        return cudaSuccess;
    const int64_t want = (total + threads - 1) / threads;
    const unsigned blocks = (unsigned)(want < 148 * 64 ? want : 148 * 64);
    if (p.wf)
        k_csr_i8_phase<true><<<blocks, threads, 0, st>>>(p);
    else
        k_csr_i8_phase<false><<<blocks, threads, 0, st>>>(p);
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

// k_csr_i8.cu -- per-lane Metropolis on int8 spins over a CSR graph (sm_100a).
//
// Rows a3-a4 (field + decision + flip) for the I8 layout: any int32 or float32
// couplings (C5: random 3-regular with N(0,1) float32 weights; C1 torus in
// int8).  Spins are stored s[v][r] (internal vertex v, local replica r,
// replica-minor), so the 32 threads that own the R = 256 replicas of one vertex
// read every neighbour row as one coalesced 256-byte segment.
//
// One thread = (vertex of the current colour class, 8 consecutive replicas as
// two 32-bit words).  The field is evaluated in relative signs: sigma_j =
// s_i s_j is bit 7 of each byte of own ^ nb_j, and s_i h = sum_j w_ij sigma_j
// (exact int32; float: a left fold in CSR row order with round-to-nearest adds
// and no contraction, ((0 + t0) + t1) + t2 -- multiplying every term by s_i
// commutes exactly with RN addition, up to the sign of a zero, which cannot
// change the decision s_i h >= 0).  dE = -2 s_i h: s_i h >= 0
// flips without randomness; otherwise the WORD contract
// decides U < T with U = hi16 * 2^48 + lo48:
//   hi16 = 16-bit half (r & 1) of word ((r >> 1) & 3) of Philox(i, t, r >> 3, WORD_HI<<24)
//   lo48 = w0 * 2^16 + (w1 >> 16) of Philox(i, t, r, WORD_LO<<24)   (only if hi16 == T >> 48)
// so one Philox call serves the thread's 8 attempts.  T = floor(exp(-beta dE) 2^64):
// integer weights from the host table; float weights from the float32 contract
// exponential cexp32, which is only evaluated when a fast estimate cannot decide.
#include "internal.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

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

// Contract threshold floor(cexp32(x) 2^64), saturated, for x = -(beta dE) <= 0.
__device__ __forceinline__ uint64_t thr_x(float x)
{
    const float v = __fmul_rn(cexp32(x), 0x1p64f);
    if (v >= 0x1p64f)
        return ~0ull;
    return __float2ull_rz(v);
}

// The fast decision estimates c = T / 2^48 = cexp32(x) 2^16 (x = -(beta dE) = (2 beta) s_i h) by
//   e = ex2.approx(RN(bl * sh + 16)),   bl = RN((2 beta) * log2 e),   sh = s_i h,
// one FFMA and one MUFU per attempt (bl is computed once per thread).  Relative to c the
// error has four sources: bl vs log2e * x / sh (two roundings, <= 2^-23 relative in the
// exponent argument), the FFMA rounding of the argument, ex2.approx, and cexp32 vs exp.
// Wherever c >= 1/2 (x >= -11.8, argument <= 17 in magnitude) they sum to < 2^-18.5;
// ising_debug_exp_bound checks |e/c - 1| < 2^-17 for every float sh and the ladder's betas,
// together with e < 1 wherever c < 1/2.  Since c <= 2^16, |e - c| <= 1/2 where c >= 1/2.
// The decision compares d = RN(hf - e), hf = 2^23 + hi16 (|d - (hf - e)| <= 1/2, the result
// lies in [2^22, 2^24)):
//   d <= 2^23 - 2  =>  hi16 + 1 <= e - 1/2 <= c  =>  (hi16 + 1) 2^48 <= T  =>  U < T: accept
//                      (c < 1/2: e < 1 makes it impossible, as it must be)
//   d >= 2^23 + 1  =>  hi16 >= e + 1/2 >= c      =>  U >= hi16 2^48 >= T: reject
//                      (c < 1/2: hi16 >= 1 > 2 c, and U >= 2^48 > T)
// (T saturated at 2^64 - 1, c = 2^16: accept needs hi16 <= 65534, so U < T still holds).
// s h >= 0 (dE <= 0, always flips) needs no test of its own: the argument is >= 16, so
// e >= 2^16 (1 - 2^-22) and d <= 2^23 - 1 + 2^-6: never rejected, accepted unless hi16 = 65535
// near s h = 0, which the undecided path flips;
// anything in between (d in (2^23 - 2, 2^23 + 1), ~3 values of hi16 in 2^16) is decided
// exactly from the contract threshold.
constexpr float kLog2e = 0x1.715476p+0f;

__device__ __forceinline__ float exp_est16(float bl, float sh)
{
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmaf_rn(bl, sh, 16.0f)));
    return e;
}

// d = RN(hf - e) of the fast decision; accepted if d <= 2^23 - 2, rejected if d >= 2^23 + 1
__device__ __forceinline__ float fast_d(float hf, float e) { return __fsub_rn(hf, e); }
__device__ __forceinline__ bool fast_accept(float d) { return d <= 0x1p23f - 2.0f; }
__device__ __forceinline__ bool fast_reject(float d) { return d >= 0x1p23f + 1.0f; }

// lo48 of replica r: Philox(i, t, r, WORD_LO<<24) words 0 and 1
__device__ __forceinline__ uint64_t lo48_of(uint32_t io, uint32_t t, uint32_t r, const RoundKeys &rk)
{
    const uint4 l = philox(io, t, r, ST_WORD_LO << 24, rk);
    return ((uint64_t)l.x << 16) | (uint64_t)(l.y >> 16);
}

// exact U < T for hi16 on the tie path
__device__ __forceinline__ bool exact_less(uint32_t hi16, uint64_t T, uint32_t io, uint32_t t, uint32_t r,
                                           const RoundKeys &rk)
{
    const uint32_t th = (uint32_t)(T >> 48);
    if (hi16 != th)
        return hi16 < th;
    return lo48_of(io, t, r, rk) < (T & 0xFFFFFFFFFFFFull);
}

}  // namespace

// Exhaustive check of the fast-decision bound for one 2 beta per blockIdx.y: over every float
// sh in [-80 / (2 beta), 0] (beyond it e < 2^-99), out[0] = max |e / c - 1| where c >= 1/2 and
// out[1] = max e where c < 1/2, with e = exp_est16(RN(2 beta log2e), sh) and c = cexp32(RN(2 beta
// sh)) 2^16 -- the exact expressions of the kernels (float bits, atomicMax).
__global__ void k_debug_exp_bound(const float *beta2, uint32_t *out)
{
    const float b2 = beta2[blockIdx.y];
    const float bl = __fmul_rn(b2, kLog2e);
    const uint32_t hi = __float_as_uint(-80.0f / b2) + 1u;  // float bits of -0 .. -(80/b2)
    float worst = 0.f, small = 0.f;
    for (uint64_t u = 0x80000000u + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= hi;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const float sh = __uint_as_float((uint32_t)u);
        const float e = exp_est16(bl, sh);
        const float c = __fmul_rn(cexp32(__fmul_rn(b2, sh)), 0x1p16f);
        if (c >= 0.5f)
            worst = fmaxf(worst, fabsf(e / c - 1.0f));
        else
            small = fmaxf(small, e);
    }
    atomicMax(out, __float_as_uint(worst));
    atomicMax(out + 1, __float_as_uint(small));
}

cudaError_t launch_debug_exp_bound(const float *beta2, int32_t n_beta, uint32_t *out, cudaStream_t st)
{
    k_debug_exp_bound<<<dim3(148 * 8, (unsigned)n_beta), 256, 0, st>>>(beta2, out);
    return cudaGetLastError();
}

// Philox4x32-10 with each round's products as one 64-bit multiply (IMAD.WIDE.U32).
__device__ __forceinline__ uint4 philox_w(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                          const RoundKeys &rk)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

// 2^23 + hi16 as a float (exact), from half (b & 1) of word w: one PRMT
template <int b>
__device__ __forceinline__ float hi16_f(uint32_t w)
{
    uint32_t r;
    // bytes (lo..hi): hi16 low byte, hi16 high byte, 0x00, 0x4B  (0x4B000000 = 2^23)
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(0x4B000000u), "n"((b & 1) ? 0x7432 : 0x7410));
    return __uint_as_float(r);
}

// same with the 0x4B000000 source in a register (selector immediate)
template <int b>
__device__ __forceinline__ float hi16_fr(uint32_t w, uint32_t c4b)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(c4b), "n"((b & 1) ? 0x7432 : 0x7410));
    return __uint_as_float(r);
}

// Float-weight decisions of one thread's 8 replicas: field s_i h in two
// halves of 4 replicas, fast estimate, exact contract threshold for the rare undecided.
template <bool ELL>
__device__ __forceinline__ void float_decide(const CsrI8Params &p, int32_t v, const uint2 own,
                                             const uint2 (&x)[4], const uint32_t (&wv)[4],
                                             const uint32_t *tb, uint32_t rw, uint32_t io, uint32_t g0,
                                             uint32_t o, const float4 *bp, const uint32_t (&hw)[4],
                                             uint32_t &fm0, uint32_t &fm1)
{
        // two halves of 4 replicas (one spin word each) to keep the live set small
        const float4 *bph = bp;
        bool und = false;  // some replica the fast estimate cannot decide
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            float sh[4];
            if (ELL) {
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    sh[b] = 0.0f;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < p.ell_deg) {  // kernel-uniform: the table's used width
                        const uint32_t word = half ? x[u].y : x[u].x;
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const uint32_t sg = (word << (24 - 8 * b)) & 0x80000000u;
                            sh[b] = __fadd_rn(sh[b], __uint_as_float(wv[u] ^ sg));
                        }
                    }
            } else {
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    sh[b] = 0.0f;
                const int32_t e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
                for (int32_t e = e0; e < e1; ++e) {
                    const uint32_t nbw = __ldg(tb + (uint32_t)__ldg(p.col + e) * rw + (uint32_t)half);
                    const uint32_t word = (half ? own.y : own.x) ^ nbw;
                    const uint32_t w = __float_as_uint(__ldg(p.wf + e));
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const uint32_t sg = (word << (24 - 8 * b)) & 0x80000000u;
                        sh[b] = __fadd_rn(sh[b], __uint_as_float(w ^ sg));
                    }
                }
            }
            const float4 bq = __ldg(bph + half);  // 2 beta_k, L1-resident
            const float b2[4] = {__fmul_rn(bq.x, kLog2e), __fmul_rn(bq.y, kLog2e), __fmul_rn(bq.z, kLog2e),
                                 __fmul_rn(bq.w, kLog2e)};  // RN(2 beta log2e)
            uint32_t fm = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                // s h >= 0 flips; else estimate cexp32((2 beta)(s h)) 2^16
                const float e = exp_est16(b2[b], sh[b]);
                const uint32_t hword = hw[2 * half + (b >> 1)];
                const float hf = (b & 1) ? hi16_f<1>(hword) : hi16_f<0>(hword);  // 2^23 + hi16
                const float d = fast_d(hf, e);
                const bool acc = fast_accept(d);  // s h >= 0: e >= 2^16, accepted here or left undecided
                const bool dec = acc || fast_reject(d);
                fm |= acc ? (0xFEu << (8 * b)) : 0u;
                und |= !dec;
            }
            if (half)
                fm1 = fm;
            else
                fm0 = fm;
        }
        if (__builtin_expect(und != 0u, 0)) {  // rare: recompute field and estimate; exact threshold
#pragma unroll 1
            for (int b = 0; b < 8; ++b) {  // no dynamic indexing: x[] and hw[] stay in registers
                float shb = 0.0f;
                if (ELL) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (u >= p.ell_deg)
                            break;
                        const uint32_t word = b < 4 ? x[u].x : x[u].y;  // select, u static
                        shb = __fadd_rn(shb, __uint_as_float(wv[u] ^ ((word << (24 - 8 * (b & 3))) & 0x80000000u)));
                    }
                } else {
                    const int32_t e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
                    for (int32_t e = e0; e < e1; ++e) {
                        const uint32_t nbw = __ldg(tb + (uint32_t)__ldg(p.col + e) * rw + (uint32_t)(b >> 2));
                        const uint32_t word = (b < 4 ? own.x : own.y) ^ nbw;
                        shb = __fadd_rn(shb, __uint_as_float(__float_as_uint(__ldg(p.wf + e)) ^
                                                             ((word << (24 - 8 * (b & 3))) & 0x80000000u)));
                    }
                }
                const float b2v = __ldg(p.betaf + 8u * o + (uint32_t)b);
                const float xv = __fmul_rn(b2v, shb);  // x = -(beta dE), the contract's product
                const uint32_t hword = (b >> 1) == 0 ? hw[0] : (b >> 1) == 1 ? hw[1] : (b >> 1) == 2 ? hw[2] : hw[3];
                const uint32_t hb = (b & 1) ? (hword >> 16) : (hword & 0xFFFFu);
                if (shb >= 0.0f) {  // dE <= 0 always flips
                    if (b < 4)
                        fm0 |= 0xFEu << (8 * (b & 3));
                    else
                        fm1 |= 0xFEu << (8 * (b & 3));
                    continue;
                }
                const float e = exp_est16(__fmul_rn(b2v, kLog2e), shb);
                const float d = fast_d(__uint_as_float(0x4B000000u | hb), e);
                if (fast_accept(d) || fast_reject(d))
                    continue;  // decided by the fast path (same expressions)
                if (exact_less(hb, thr_x(xv), io, p.t, 8u * g0 + (uint32_t)b, p.rk)) {
                    if (b < 4)
                        fm0 |= 0xFEu << (8 * (b & 3));
                    else
                        fm1 |= 0xFEu << (8 * (b & 3));
                }
            }
        }
}

// One thread = (vertex v of the current colour class, local replicas 8o .. 8o+7), with
// o = blockIdx.y * blockDim.x + threadIdx.x fixed for the thread's lifetime and vertices strided over (blockIdx.x, threadIdx.y).
// ELL: neighbours from the padded 4-wide table (one 16-byte load per vertex, pad = -1)
// instead of row_ptr -> col -> spins, so a neighbour-row load depends on one load only.
template <bool FLOAT, bool ELL>
__global__ void __launch_bounds__(kI8Threads, FLOAT ? kI8MinBlocks : 3) k_csr_i8_phase(const CsrI8Params p)
{
    const uint32_t rw = (uint32_t)p.R >> 2;  // 32-bit words per vertex row
    const uint32_t ntv = rw >> 1;            // threads per vertex (8 replicas each)
    const uint32_t o = blockIdx.y * blockDim.x + threadIdx.x;
    if (o >= ntv)
        return;
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    const uint32_t vstride = gridDim.x * blockDim.y;
    uint32_t *tb = reinterpret_cast<uint32_t *>(p.s) + 2u * o;  // this thread's column of words
    char *tbb = reinterpret_cast<char *>(tb);                    // ... as bytes: one IMAD.WIDE per row
    const uint32_t rwb = 4u * rw;                                // row bytes
    const uint32_t g0 = (uint32_t)(p.slot0 >> 3) + o;            // Philox counter word 2
    const float4 *bp = reinterpret_cast<const float4 *>(p.betaf) + 2u * o;  // 2 beta_k (float)
    // software pipeline: the next vertex's neighbour table row and original id are loaded
    // one iteration ahead, so a vertex's spin-row loads issue as soon as it starts
    uint32_t vv = blockIdx.x * blockDim.y + threadIdx.y;
    int4 c_nx = make_int4(-1, -1, -1, -1), w_nx = make_int4(0, 0, 0, 0);
    uint32_t io_nx = 0u;
    if (vv < nv) {
        io_nx = __ldg(p.orig + p.v_begin + (int32_t)vv);
        if (ELL) {
            c_nx = __ldg(reinterpret_cast<const int4 *>(p.ell_col) + p.v_begin + (int32_t)vv);
            w_nx = __ldg(reinterpret_cast<const int4 *>(p.ell_w) + p.v_begin + (int32_t)vv);
        }
    }
    for (; vv < nv; vv += vstride) {
        const int32_t v = p.v_begin + (int32_t)vv;
        uint2 *own_p = reinterpret_cast<uint2 *>(tbb + (uint32_t)v * rwb);
        const uint32_t io = io_nx;
        const uint2 own = *own_p;
        // x[u] = own ^ nb_u: bit 8b+7 of word w set iff s_i != s_j for replica 4w+b
        uint2 x[4];
        uint32_t wv[4];
        if (ELL) {
            const int32_t cs[4] = {c_nx.x, c_nx.y, c_nx.z, c_nx.w};
            wv[0] = (uint32_t)w_nx.x; wv[1] = (uint32_t)w_nx.y; wv[2] = (uint32_t)w_nx.z; wv[3] = (uint32_t)w_nx.w;
            uint2 nb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                nb[u] = own;  // a pad (col = self, w 0) adds an exact zero term
                if (u < p.ell_deg)  // kernel-uniform
                    nb[u] = __ldg(reinterpret_cast<const uint2 *>(tbb + (uint32_t)cs[u] * rwb));
            }
            const uint32_t vn = vv + vstride;
            if (vn < nv) {
                io_nx = __ldg(p.orig + p.v_begin + (int32_t)vn);
                c_nx = __ldg(reinterpret_cast<const int4 *>(p.ell_col) + p.v_begin + (int32_t)vn);
                w_nx = __ldg(reinterpret_cast<const int4 *>(p.ell_w) + p.v_begin + (int32_t)vn);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                x[u] = make_uint2(own.x ^ nb[u].x, own.y ^ nb[u].y);
        } else {
            const uint32_t vn = vv + vstride;
            if (vn < nv)
                io_nx = __ldg(p.orig + p.v_begin + (int32_t)vn);
        }
        // one Philox call for the 8 replicas (issued early: independent of the loads)
        const uint4 h = philox_w(io, p.t, g0, ST_WORD_HI << 24, p.rk);
        const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
        uint32_t fm0 = 0u, fm1 = 0u;  // flip masks (0xFE per flipped byte)
        if (FLOAT) {
            float_decide<ELL>(p, v, own, x, wv, tb, rw, io, g0, o, bp, hw, fm0, fm1);
        } else {
            int32_t sh[8];
#pragma unroll
            for (int b = 0; b < 8; ++b)
                sh[b] = 0;
            auto fold = [&](const uint2 &xx, int32_t w) {
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const uint32_t word = b < 4 ? xx.x : xx.y;
                    const int32_t m = (int32_t)(word << (24 - 8 * (b & 3))) >> 31;  // -1 iff s_i != s_j
                    sh[b] += (w ^ m) - m;
                }
            };
            if (ELL) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < p.ell_deg)
                        fold(x[u], (int32_t)wv[u]);
            } else {
                const int32_t e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
                for (int32_t e = e0; e < e1; ++e) {
                    const uint2 nb = __ldg(reinterpret_cast<const uint2 *>(tb + (uint32_t)__ldg(p.col + e) * rw));
                    fold(make_uint2(own.x ^ nb.x, own.y ^ nb.y), __ldg(p.wi + e));
                }
            }
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                bool acc = sh[b] >= 0;  // dE = -2 s h <= 0
                if (!acc) {
                    const uint32_t hb = (b & 1) ? (hw[b >> 1] >> 16) : (hw[b >> 1] & 0xFFFFu);
                    const uint32_t rl = 8u * o + (uint32_t)b;  // local replica
                    const uint64_t T = __ldg(p.T + (size_t)rl * (p.qmax + 1) + (uint32_t)(-sh[b]));
                    acc = exact_less(hb, T, io, p.t, 8u * g0 + (uint32_t)b, p.rk);
                }
                if (acc) {
                    if (b < 4)
                        fm0 |= 0xFEu << (8 * (b & 3));
                    else
                        fm1 |= 0xFEu << (8 * (b & 3));
                }
            }
        }
        // +1 (0x01) <-> -1 (0xFF): xor the byte with 0xFE
        *own_p = make_uint2(own.x ^ fm0, own.y ^ fm1);
    }
}

// Float weights + padded neighbour table of fixed width DEG (the graph's maximum degree,
// <= 4): software pipeline, unrolled by two so no register is copied between iterations
// (DESIGN.md §5.4).  Step k decides vertex k from rows issued in step k-1; at its top it
// issues the spin rows of vertex k+1 (columns loaded in step k-1), the weights / original
// id of vertex k+1 and the columns of vertex k+2.  Philox rounds 0-1 are half hoisted (the
// counter words t, g0 and the stream are loop-invariant).
template <int DEG>
struct I8Rows {
    uint2 own;
    uint2 nb[DEG];
};

struct I8Meta {
    int4 w;       // weights (float bits), pads 0
    uint32_t io;  // original id (Philox counter word 0)
};

// Philox4x32-10(io, t, g0, WORD_HI<<24) with the loop-invariant parts of rounds 0 and 1
// precomputed: per call 2 + 18 IMAD.WIDE-equivalents fewer than the plain form.
struct PhiloxHoist {
    uint32_t c3k1;  // (WORD_HI << 24) ^ k1
    uint32_t bk2;   // lo(M1 g0) ^ k2           (round 1, word 0)
    uint32_t hak3;  // hi(M0 A) ^ k3, A = hi(M1 g0) ^ t ^ k0 (round 1, word 2)
    uint32_t la;    // lo(M0 A)                 (round 1, word 3)
};

__device__ __forceinline__ PhiloxHoist philox_hoist(uint32_t t, uint32_t g0, const RoundKeys &rk)
{
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * g0;
    const uint32_t A = (uint32_t)(p1 >> 32) ^ t ^ rk.k[0];
    const uint32_t B = (uint32_t)p1;
    const uint64_t pa = (uint64_t)0xD2511F53u * A;
    PhiloxHoist h;
    h.c3k1 = ((uint32_t)ST_WORD_HI << 24) ^ rk.k[1];
    h.bk2 = B ^ rk.k[2];
    h.hak3 = (uint32_t)(pa >> 32) ^ rk.k[3];
    h.la = (uint32_t)pa;
    return h;
}

__device__ __forceinline__ uint4 philox_hoisted(uint32_t io, const PhiloxHoist &hh, const RoundKeys &rk)
{
    // round 0: c0 = A, c1 = B, c2 = hi(M0 io) ^ c3 ^ k1, c3 = lo(M0 io)
    const uint64_t p0 = (uint64_t)0xD2511F53u * io;
    const uint32_t c2r0 = (uint32_t)(p0 >> 32) ^ hh.c3k1;
    // round 1: p0' = M0 A (hoisted), p1' = M1 c2r0
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2r0;
    uint32_t c0 = (uint32_t)(p1 >> 32) ^ hh.bk2;
    uint32_t c1 = (uint32_t)p1;
    uint32_t c2 = hh.hak3 ^ (uint32_t)p0;
    uint32_t c3 = hh.la;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        const uint64_t q0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t q1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(q1 >> 32) ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = (uint32_t)(q0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
        c1 = (uint32_t)q1;
        c3 = (uint32_t)q0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

// sign-adjusted weight of neighbour term u for byte b of x = (own ^ nb_u) & 0x80808080 (bit 7 of
// byte b set where s_i != s_j): w_u if s_i = s_j, -w_u otherwise.
template <int b>
__device__ __forceinline__ float term(uint32_t x, uint32_t w)
{
    return __uint_as_float(w ^ ((b == 3 ? x : (x << (24 - 8 * b))) & 0x80000000u));
}

// bytes 0..3 = 0xFF where k0..k3 (float bits) are negative, else 0x00 (PRMT sign replication)
__device__ __forceinline__ uint32_t sign_bytes4(uint32_t k0, uint32_t k1, uint32_t k2, uint32_t k3)
{
    uint32_t a, b, r;
    asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(a) : "r"(k0), "r"(k1));
    asm("prmt.b32 %0, %1, %2, 0xFB00;" : "=r"(b) : "r"(k2), "r"(k3));
    asm("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// field s_i h of the 4 replicas of one spin word (left fold in row order; the leading
// 0 + t_0 of the contract fold is t_0 up to the sign of a zero, which no decision sees)
template <int DEG, int HALF>
__device__ __forceinline__ void field4(const uint2 (&x)[DEG], const int4 &wq, float (&sh)[4])
{
    const uint32_t wv[4] = {(uint32_t)wq.x, (uint32_t)wq.y, (uint32_t)wq.z, (uint32_t)wq.w};
    const uint32_t x0 = HALF ? x[0].y : x[0].x;
    sh[0] = term<0>(x0, wv[0]);
    sh[1] = term<1>(x0, wv[0]);
    sh[2] = term<2>(x0, wv[0]);
    sh[3] = term<3>(x0, wv[0]);
#pragma unroll
    for (int u = 1; u < DEG; ++u) {
        const uint32_t xu = HALF ? x[u].y : x[u].x;
        sh[0] = __fadd_rn(sh[0], term<0>(xu, wv[u]));
        sh[1] = __fadd_rn(sh[1], term<1>(xu, wv[u]));
        sh[2] = __fadd_rn(sh[2], term<2>(xu, wv[u]));
        sh[3] = __fadd_rn(sh[3], term<3>(xu, wv[u]));
    }
}

// row addresses as one IMAD.WIDE.U32 each (64-bit product of the 32-bit id and row bytes)
template <int DEG>
__device__ __forceinline__ void pipe_issue(I8Rows<DEG> &r, const char *tbb, uint32_t rwb, uint32_t v,
                                           const int4 &c)
{
    r.own = *reinterpret_cast<const uint2 *>(tbb + (uint64_t)v * rwb);
    const int32_t cs[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int u = 0; u < DEG; ++u)
        r.nb[u] = __ldg(reinterpret_cast<const uint2 *>(tbb + (uint64_t)(uint32_t)cs[u] * rwb));
}

// Decide the 8 attempts of vertex v (internal id) and write its row.
// PAT (the ring kernel: a warp is one vertex's 256-replica slice): the field of each replica is
// looked up by one shuffle from the lane that folded its relative-sign pattern (lane l folds
// pattern l mod 2^DEG with the sign masks pm; the same terms in the same order, so the same
// floats as field4), the pattern of byte b being bits 8b .. 8b+DEG-1 of
// z = OR_u x_u >> (7 - u).
template <int DEG, bool PAT = false>
__device__ __forceinline__ void pipe_decide(const CsrI8Params &p, const I8Rows<DEG> &r, const I8Meta &m,
                                            uint32_t v, char *tbb, uint32_t rwb, const float (&bl)[8],
                                            const PhiloxHoist &ph, uint32_t g0, uint32_t o, uint32_t c4b,
                                            const uint32_t *pm = nullptr)
{
    uint2 x[DEG];
#pragma unroll
    for (int u = 0; u < DEG; ++u)
        x[u] = make_uint2((r.own.x ^ r.nb[u].x) & 0x80808080u, (r.own.y ^ r.nb[u].y) & 0x80808080u);
    float sv = 0.0f;
    if (PAT) {
        const uint32_t wv[4] = {(uint32_t)m.w.x, (uint32_t)m.w.y, (uint32_t)m.w.z, (uint32_t)m.w.w};
        sv = __uint_as_float(wv[0] ^ pm[0]);
#pragma unroll
        for (int u = 1; u < DEG; ++u)
            sv = __fadd_rn(sv, __uint_as_float(wv[u] ^ pm[u]));
    }
    const uint4 h = philox_hoisted(m.io, ph, p.rk);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
    uint32_t fm[2];
    bool und = false;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        float sh[4];
        if (PAT) {
            uint32_t z = (half ? x[0].y : x[0].x) >> 7;
#pragma unroll
            for (int u = 1; u < DEG; ++u)
                z |= (half ? x[u].y : x[u].x) >> (7 - u);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                sh[b] = __shfl_sync(0xFFFFFFFFu, sv, (int)(z >> (8 * b)));
        } else if (half)
            field4<DEG, 1>(x, m.w, sh);
        else
            field4<DEG, 0>(x, m.w, sh);
        // k = d - (2^23 - 3/2) (exact: d is a float within a factor 2 of the constant, or far
        // enough that only its sign matters, and RN keeps a nonzero difference's sign): d takes
        // half-integer values below 2^23 and integers above, so k < 0 exactly where d <= 2^23 - 2
        // (fast accept; d = -inf included), k in {+0, 1/2, 1, 3/2} (float bits <= 0x3FC00000)
        // where the fast test cannot decide, k >= 5/2 where d >= 2^23 + 1 (fast reject).  The
        // accepted bytes come from the sign bits by PRMT sign replication (3 PRMT per 4 attempts)
        // and the undecided test is one unsigned compare of the float bits: one FADD on the FMA
        // pipe and ~1.75 ALU instructions per attempt instead of two FSETP, a SEL and the merges
        // (C5 +5%).
        uint32_t kb[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float e = exp_est16(bl[4 * half + b], sh[b]);
            const uint32_t hword = hw[2 * half + (b >> 1)];
            const float hf = (b & 1) ? hi16_fr<1>(hword, c4b) : hi16_fr<0>(hword, c4b);  // 2^23 + hi16
            kb[b] = __float_as_uint(__fsub_rn(fast_d(hf, e), 0x1p23f - 1.5f));
            und |= kb[b] <= 0x3FC00000u;  // k in [+0, 3/2]
        }
        fm[half] = sign_bytes4(kb[0], kb[1], kb[2], kb[3]);
    }
    if (__builtin_expect(und, 0)) {  // rare: recompute the field per replica, exact threshold
#pragma unroll 1
        for (int b = 0; b < 8; ++b) {
            float shb;
            {
                float s4[4];
                if (b < 4)
                    field4<DEG, 0>(x, m.w, s4);
                else
                    field4<DEG, 1>(x, m.w, s4);
                const int bb = b & 3;
                shb = bb == 0 ? s4[0] : bb == 1 ? s4[1] : bb == 2 ? s4[2] : s4[3];
            }
            if (shb >= 0.0f) {  // dE <= 0 always flips (left undecided only when s h ~ +0)
                if (b < 4)
                    fm[0] |= 0xFEu << (8 * (b & 3));
                else
                    fm[1] |= 0xFEu << (8 * (b & 3));
                continue;
            }
            const uint32_t hword = (b >> 1) == 0 ? hw[0] : (b >> 1) == 1 ? hw[1] : (b >> 1) == 2 ? hw[2] : hw[3];
            const uint32_t hb = (b & 1) ? (hword >> 16) : (hword & 0xFFFFu);
            const float b2v = __ldg(p.betaf + 8u * o + (uint32_t)b);
            const float e = exp_est16(__fmul_rn(b2v, kLog2e), shb);
            const float d = fast_d(__uint_as_float(0x4B000000u | hb), e);
            // the two-comparison bracket decides every replica the k form decided (same bands,
            // tests/test_fast_decision_classes.py); an accept is applied here as well, so this
            // path stays correct for any valid fast test
            const bool fa = fast_accept(d);
            if (fa || fast_reject(d)) {
                if (fa) {
                    if (b < 4)
                        fm[0] |= 0xFEu << (8 * (b & 3));
                    else
                        fm[1] |= 0xFEu << (8 * (b & 3));
                }
                continue;
            }
            if (exact_less(hb, thr_x(__fmul_rn(b2v, shb)), m.io, p.t, 8u * g0 + (uint32_t)b, p.rk)) {
                if (b < 4)  // scalar updates: a dynamically indexed fm[] would live in local memory
                    fm[0] |= 0xFEu << (8 * (b & 3));
                else
                    fm[1] |= 0xFEu << (8 * (b & 3));
            }
        }
    }
    // +1 (0x01) <-> -1 (0xFF): xor the byte with 0xFE
    // st.global on the (global-space) row address: the ring kernel's row base is an opaque
    // register copy the compiler would otherwise store through with a generic ST
    asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(tbb + (uint64_t)v * rwb),
                 "r"(r.own.x ^ (fm[0] & 0xFEFEFEFEu)), "r"(r.own.y ^ (fm[1] & 0xFEFEFEFEu))
                 : "memory");
}

template <int DEG>
__global__ void __launch_bounds__(kI8Threads, kI8PipeMinBlocks) k_csr_i8_pipe(const CsrI8Params p)
{
    const uint32_t rw = (uint32_t)p.R >> 2;
    const uint32_t ntv = rw >> 1;
    const uint32_t o = blockIdx.y * blockDim.x + threadIdx.x;
    if (o >= ntv)
        return;
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    const uint32_t vstride = gridDim.x * blockDim.y;
    uint32_t vv = blockIdx.x * blockDim.y + threadIdx.y;
    if (vv >= nv)
        return;
    char *tbb = reinterpret_cast<char *>(reinterpret_cast<uint32_t *>(p.s) + 2u * o);
    const uint32_t rwb = 4u * rw;
    const uint32_t g0 = (uint32_t)(p.slot0 >> 3) + o;
    float bl[8];
    {
        const float4 *bp = reinterpret_cast<const float4 *>(p.betaf) + 2u * o;  // 2 beta_k
        const float4 a = __ldg(bp), b = __ldg(bp + 1);
        const float b2[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
            bl[i] = __fmul_rn(b2[i], kLog2e);
    }
    const PhiloxHoist ph = philox_hoist(p.t, g0, p.rk);
    // 0x4B000000 (= 2^23) in a register the compiler cannot fold (rwb < 2^31), so the PRMT
    // building 2^23 + hi16 takes its selector as an immediate
    const uint32_t c4b = 0x4B000000u | (rwb >> 31);
    const uint32_t vb = (uint32_t)p.v_begin;
    const int4 *ec = reinterpret_cast<const int4 *>(p.ell_col) + vb;
    const int4 *ew = reinterpret_cast<const int4 *>(p.ell_w) + vb;
    const uint32_t *eo = p.orig + vb;
    auto meta = [&](uint32_t q) {
        I8Meta m;
        m.w = __ldg(ew + q);
        m.io = __ldg(eo + q);
        return m;
    };
    // prologue: rows + meta of the first vertex, columns of the second
    I8Rows<DEG> rA, rB;
    I8Meta mA = meta(vv), mB;
    pipe_issue<DEG>(rA, tbb, rwb, vb + vv, __ldg(ec + vv));
    int4 cn = make_int4(0, 0, 0, 0);
    if (vv + vstride < nv)
        cn = __ldg(ec + vv + vstride);
    for (;;) {
        // step with A current, B next
        uint32_t v1 = vv + vstride;
        if (v1 < nv) {
            pipe_issue<DEG>(rB, tbb, rwb, vb + v1, cn);
            mB = meta(v1);
            if (v1 + vstride < nv)
                cn = __ldg(ec + v1 + vstride);
        }
        pipe_decide<DEG>(p, rA, mA, vb + vv, tbb, rwb, bl, ph, g0, o, c4b);
        vv = v1;
        if (vv >= nv)
            break;
        // step with B current, A next
        v1 = vv + vstride;
        if (v1 < nv) {
            pipe_issue<DEG>(rA, tbb, rwb, vb + v1, cn);
            mA = meta(v1);
            if (v1 + vstride < nv)
                cn = __ldg(ec + v1 + vstride);
        }
        pipe_decide<DEG>(p, rB, mB, vb + vv, tbb, rwb, bl, ph, g0, o, c4b);
        vv = v1;
        if (vv >= nv)
            break;
    }
}

// ---------------------------------------------------------------- cp.async ring variant
// Float weights, padded table, R a multiple of 256 (every warp = 32 threads x 8 replicas of
// one vertex): each warp sweeps a CONTIGUOUS chunk of the colour class and keeps S vertices'
// spin rows in flight through a per-warp shared-memory ring filled by cp.async (LDGSTS), so
// the memory-level parallelism no longer costs registers (the register pipeline above keeps
// one vertex in flight and stalls on load latency).  The table rows (columns,
// weights, original ids) of 32 consecutive vertices arrive by one cp.async per lane into a
// double buffer, 32 vertices ahead.  Each lane reads back only the row bytes it copied
// itself; table entries are read by every lane after a __syncwarp.
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// table entry of one vertex in shared memory: columns (16 B), weights (16 B), original id, pad
constexpr uint32_t kRingEntry = 48;
constexpr uint32_t kRingMetaBuf = 32 * kRingEntry;  // one block of 32 vertices

template <int DEG, int S>
__host__ __device__ constexpr uint32_t ring_warp_bytes()
{
    return (uint32_t)S * (DEG + 1) * 256u + 2u * kRingMetaBuf;
}

__device__ __forceinline__ uint2 lds64(uint32_t a)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds128(uint32_t a)
{
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

template <int DEG, int S>
__global__ void __launch_bounds__(256, kI8RingMinBlocks) k_csr_i8_ring(const CsrI8Params p, uint32_t nslice, uint32_t chunk)
{
    extern __shared__ __align__(16) unsigned char ring_smem[];
    constexpr uint32_t kSlot = (DEG + 1) * 256u;
    constexpr uint32_t kRing = S * kSlot;
    const uint32_t lane = threadIdx.x;
    const uint32_t gw = blockIdx.x * blockDim.y + threadIdx.y;
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    const uint32_t slice = gw % nslice;
    const uint32_t j0 = (gw / nslice) * chunk;
    if (j0 >= nv)
        return;
    const uint32_t cnt = min(chunk, nv - j0);
    const uint32_t o = slice * 32u + lane;
    const uint32_t rwb = (uint32_t)p.R;  // row bytes (one int8 per replica)
    // this thread's column of the spin rows, held in a register pair (an opaque copy: the
    // compiler would otherwise re-derive it from threadIdx and the parameter every vertex)
    char *tbb;
    asm volatile("mov.b64 %0, %1;" : "=l"(tbb) : "l"(reinterpret_cast<char *>(p.s) + 8u * o));
    const uint32_t g0 = (uint32_t)(p.slot0 >> 3) + o;
    float bl[8];
    {
        const float4 *bp = reinterpret_cast<const float4 *>(p.betaf) + 2u * o;
        const float4 a = __ldg(bp), b = __ldg(bp + 1);
        const float b2[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
            bl[i] = __fmul_rn(b2[i], kLog2e);
    }
    const PhiloxHoist ph = philox_hoist(p.t, g0, p.rk);
    const uint32_t c4b = 0x4B000000u | (rwb >> 31);
    uint32_t pm[DEG];  // sign masks of this lane's relative-sign pattern (lane mod 2^DEG)
#pragma unroll
    for (int u = 0; u < DEG; ++u)
        pm[u] = ((lane >> u) & 1u) << 31;
    // shared addresses: this lane's bytes of ring slot 0, and the warp's table double buffer
    const uint32_t wsh = (uint32_t)__cvta_generic_to_shared(ring_smem) + threadIdx.y * ring_warp_bytes<DEG, S>();
    const uint32_t ring0 = wsh + lane * 8u;
    const uint32_t meta0 = wsh + kRing;
    const uint32_t vb = (uint32_t)p.v_begin + j0;  // internal id of the chunk's first vertex
    auto meta_issue = [&](uint32_t blk) {
        const uint32_t j = blk * 32u + lane;
        if (j < cnt) {
            const uint32_t me = meta0 + (blk & 1u) * kRingMetaBuf + lane * kRingEntry;
            cp_async16(me, p.ell_col + 4u * (vb + j));
            cp_async16(me + 16u, p.ell_w + 4u * (vb + j));
            cp_async4(me + 32u, p.orig + vb + j);
        }
    };
    // table entries of the two 32-vertex blocks form one circular list of 64 entries
    const uint32_t meta_end = meta0 + 2u * kRingMetaBuf;
    auto next_entry = [&](uint32_t e) { return e + kRingEntry == meta_end ? meta0 : e + kRingEntry; };
    auto rows_issue = [&](uint32_t j, uint32_t sl, uint32_t e) {
        const int4 c = lds128(e);
        const int32_t cs[4] = {c.x, c.y, c.z, c.w};
        cp_async8(sl, tbb + (uint64_t)(vb + j) * rwb);
#pragma unroll
        for (int u = 0; u < DEG; ++u)
            cp_async8(sl + (u + 1) * 256u, tbb + (uint64_t)(uint32_t)cs[u] * rwb);
    };
    meta_issue(0);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
#pragma unroll
    for (uint32_t j = 0; j + 1 < S; ++j) {  // vertices 0 .. S-2 into ring slots 0 .. S-2
        if (j < cnt)
            rows_issue(j, ring0 + j * kSlot, meta0 + j * kRingEntry);
        cp_commit();
    }
    // main loop, unrolled by U (a multiple of S dividing 32): the ring slot of vertex j is
    // j % S (a constant per unrolled step), and its table entry is j % 64 of the circular list
    // (a group of U vertices never straddles the wrap of the decide-side entry pointer)
    constexpr uint32_t U = kI8RingUnroll;
    static_assert(U % S == 0 && 32 % U == 0, "unroll must be a multiple of the ring depth dividing 32");
    uint32_t e_cur = meta0;  // table entry of vertex jb
    for (uint32_t jb = 0; jb < cnt; jb += U) {
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const uint32_t j = jb + u;
            if (j >= cnt)
                break;
            if (u == 0 && (jb & 31u) == 0) {
                __syncwarp();  // every lane is done with the buffer this block overwrites
                meta_issue((j >> 5) + 1);
            }
            if (j + S - 1 < cnt)
                rows_issue(j + S - 1, ring0 + ((u + S - 1) % S) * kSlot, meta0 + ((j + S - 1) & 63u) * kRingEntry);
            cp_commit();
            cp_wait<S - 1>();
            // the table block issued at the start of this 32-vertex block is complete from here on
            // (S - 1 steps later); one __syncwarp makes every lane's part visible to all lanes
            if (u == S - 1 && (jb & 31u) == 0)
                __syncwarp();
            I8Rows<DEG> r;
            const uint32_t sl = ring0 + (u % S) * kSlot;
            r.own = lds64(sl);
#pragma unroll
            for (int q = 0; q < DEG; ++q)
                r.nb[q] = lds64(sl + (q + 1) * 256u);
            I8Meta m;
            m.w = lds128(e_cur + u * kRingEntry + 16u);
            m.io = lds32(e_cur + u * kRingEntry + 32u);
            pipe_decide<DEG, kI8RingPattern>(p, r, m, vb + j, tbb, rwb, bl, ph, g0, o, c4b, pm);
        }
        e_cur = e_cur + U * kRingEntry == meta_end ? meta0 : e_cur + U * kRingEntry;
    }
    cp_wait<0>();
}

template <int DEG, int S>
cudaError_t launch_ring(const CsrI8Params &p, cudaStream_t st)
{
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    const uint32_t nslice = (uint32_t)p.R / 256u;
    const size_t smem = (size_t)8 * ring_warp_bytes<DEG, S>();
    static int per_sm = 0;  // resident CTAs per SM (once per instantiation)
    if (!per_sm) {
        cudaError_t e = cudaFuncSetAttribute(k_csr_i8_ring<DEG, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_csr_i8_ring<DEG, S>, 256, smem);
        if (e != cudaSuccess)
            return e;
        if (per_sm < 1)
            return cudaErrorInvalidConfiguration;
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t want = (uint32_t)nsm * (uint32_t)per_sm * 8u;  // one wave of resident warps
    uint32_t nch = want / nslice;
    if (nch < 1)
        nch = 1;
    if (nch > nv)
        nch = nv;
    // at least 40 vertices per warp: the prologue / drain stay a small share of a warp's work
    // (and every chunk of more than 32 vertices crosses a table double-buffer boundary)
    uint32_t chunk = (nv + nch - 1) / nch;
    if (chunk < 40u)
        chunk = 40u;
    nch = (nv + chunk - 1) / chunk;
    const uint32_t warps = nch * nslice;
    k_csr_i8_ring<DEG, S><<<(warps + 7) / 8, dim3(32, 8), smem, st>>>(p, nslice, chunk);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- packed-row variant
// The same sweep (WORD contract, relative-sign float fold, fast decision + exact bracket) on a
// bit-packed working copy of the int8 state: row v holds the R replicas of vertex v as R/32
// words (R/8 bytes instead of R), so a vertex step moves 4 x 32 bytes per 256 replicas instead
// of 4 x 256.  Bit layout: word w of a row covers the int8 row's bytes
// 32w .. 32w+31; byte 8a + k (local replica 32w + 8a + k) is bit pk(a, k) = 8 (k & 3) +
// 4 (k >> 2) + a.  Lane l of the warp that owns replicas 256q .. 256q+255 decides replicas
// 256q + 8l + k (k = 0..7, the 8 attempts of one WORD Philox call, as in the int8 kernels): the
// bits pk(l & 3, k) of word 8q + (l >> 2), a word shared by 4 lanes.
//
// Field: s_i h is a function of the relative-sign pattern of the vertex's DEG neighbours, and
// the contract fold of each of the 2^DEG patterns is computed once per vertex (lane l folds
// pattern l mod 2^DEG: the same terms in the same order as the int8 kernels, so the same
// floats).  Rotating x_u = own ^ nb_u right by a - u puts replica k's bit u at bit u of nibble
// 2 (k & 3) + (k >> 2) of z (one bit-select per neighbour beyond the first), and the replica's
// field is one shuffle from lane z >> 4 nibble (index bits above the pattern select duplicate
// lanes).  The accepted bits come from the float sign bits of the decision differences by PRMT
// sign replication (one byte per replica k & 3, masked to bit 4 (k >> 2) + a); the 4 lanes that
// share a word OR-combine them by two xor-shuffles and lane a = 0 writes the word.
__device__ __forceinline__ uint32_t pk_bit(uint32_t a, uint32_t k) { return 8u * (k & 3u) + 4u * (k >> 2) + a; }

__global__ void k_pack_rows(const int8_t *__restrict__ s, uint32_t *__restrict__ P, uint64_t nwords)
{
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(s) + 2 * w;
        const uint4 u0 = __ldg(src), u1 = __ldg(src + 1);
        const uint32_t b[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
        uint32_t out = 0u;
#pragma unroll
        for (int i = 0; i < 32; ++i) {  // byte i = 8a + k (bit 7 of the byte: spin -1)
            const uint32_t bit = (b[i >> 2] >> (8 * (i & 3) + 7)) & 1u;
            out |= bit << pk_bit((uint32_t)i >> 3, (uint32_t)i & 7u);
        }
        P[w] = out;
    }
}

__global__ void k_unpack_rows(const uint32_t *__restrict__ P, int8_t *__restrict__ s, uint64_t nwords)
{
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = __ldg(P + w);
        uint32_t b[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t v = 0u;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = 4 * j + c;  // byte i = 8a + k
                const uint32_t bit = (x >> pk_bit((uint32_t)i >> 3, (uint32_t)i & 7u)) & 1u;
                v |= (bit ? 0xFFu : 0x01u) << (8 * c);
            }
            b[j] = v;
        }
        uint4 *dst = reinterpret_cast<uint4 *>(s) + 2 * w;
        dst[0] = make_uint4(b[0], b[1], b[2], b[3]);
        dst[1] = make_uint4(b[4], b[5], b[6], b[7]);
    }
}

// rotate right (funnel shift of x with itself)
__device__ __forceinline__ uint32_t rotr(uint32_t x, uint32_t n) { return __funnelshift_r(x, x, n); }

// Decide the 8 attempts of one lane for vertex v from its words own / nb[u] (this lane's word of
// each row), the weights wq and original id io; returns the word's flip mask (all 4 lanes).
template <int DEG>
__device__ __forceinline__ uint32_t packed_decide(const CsrI8Params &p, uint32_t own, const uint32_t (&nb)[DEG],
                                                  const int4 &wq, uint32_t io, uint32_t a, const uint32_t (&pm)[DEG],
                                                  const float (&bl)[8], const PhiloxHoist &ph, uint32_t g0,
                                                  uint32_t o, uint32_t c4b, uint32_t amask)
{
    const uint32_t wv[4] = {(uint32_t)wq.x, (uint32_t)wq.y, (uint32_t)wq.z, (uint32_t)wq.w};
    // the contract fold of this lane's pattern (pattern l mod 2^DEG)
    float sv = __uint_as_float(wv[0] ^ pm[0]);
#pragma unroll
    for (int u = 1; u < DEG; ++u)
        sv = __fadd_rn(sv, __uint_as_float(wv[u] ^ pm[u]));
    // pattern nibbles: bit u of nibble 2 (k & 3) + (k >> 2) of z = bit pk(a, k) of own ^ nb_u
    uint32_t z = rotr(own ^ nb[0], a);
#pragma unroll
    for (int u = 1; u < DEG; ++u) {
        const uint32_t ru = rotr(own ^ nb[u], (a - (uint32_t)u) & 31u);
        const uint32_t m = 0x11111111u << u;
        z = (z & ~m) | (ru & m);
    }
    const uint4 h = philox_hoisted(io, ph, p.rk);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
    float sh[8];
    uint32_t kb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int nib = 2 * (k & 3) + (k >> 2);
        sh[k] = __shfl_sync(0xFFFFFFFFu, sv, (int)(z >> (4 * nib)));
        const float e = exp_est16(bl[k], sh[k]);
        const uint32_t hword = hw[k >> 1];
        const float hf = (k & 1) ? hi16_fr<1>(hword, c4b) : hi16_fr<0>(hword, c4b);  // 2^23 + hi16
        kb[k] = __float_as_uint(__fsub_rn(fast_d(hf, e), 0x1p23f - 1.5f));
    }
    // k < 0: fast accept (sign bit); k in [+0, 3/2] (float bits <= 0x3FC00000): undecided
    const uint32_t kmin = min(min(min(kb[0], kb[1]), min(kb[2], kb[3])), min(min(kb[4], kb[5]), min(kb[6], kb[7])));
    // byte j of lo / hi = 0xFF where replica j / 4 + j accepts; bit pk(a, k) kept by amask
    const uint32_t lo = sign_bytes4(kb[0], kb[1], kb[2], kb[3]);
    const uint32_t hi = sign_bytes4(kb[4], kb[5], kb[6], kb[7]);
    uint32_t acc = ((lo & 0x0F0F0F0Fu) | (hi & 0xF0F0F0F0u)) & amask;
    if (__builtin_expect(kmin <= 0x3FC00000u, 0)) {  // rare: exact decisions
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
            float shv = sh[0];
#pragma unroll
            for (int q = 1; q < 8; ++q)
                shv = k == q ? sh[q] : shv;  // select, no dynamic indexing
            const uint32_t bit = 1u << pk_bit(a, (uint32_t)k);
            if (shv >= 0.0f) {
                acc |= bit;
                continue;
            }
            const int kh = k >> 1;
            const uint32_t hword = kh == 0 ? h.x : kh == 1 ? h.y : kh == 2 ? h.z : h.w;
            const uint32_t hb = (k & 1) ? (hword >> 16) : (hword & 0xFFFFu);
            const float b2v = __ldg(p.betaf + 8u * o + (uint32_t)k);
            const float e = exp_est16(__fmul_rn(b2v, kLog2e), shv);
            const float d = fast_d(__uint_as_float(0x4B000000u | hb), e);
            const bool fa = fast_accept(d);
            if (fa || fast_reject(d)) {  // the bracket decides what the k form decided (same bands)
                acc = fa ? (acc | bit) : (acc & ~bit);
                continue;
            }
            if (exact_less(hb, thr_x(__fmul_rn(b2v, shv)), io, p.t, 8u * g0 + (uint32_t)k, p.rk))
                acc |= bit;
            else
                acc &= ~bit;
        }
    }
    acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
    acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 2);
    return acc;
}

// Each warp sweeps a contiguous chunk of the colour class for one 256-replica slice, with S
// vertices' rows in flight through a per-warp shared-memory ring filled by cp.async (each lane
// copies and reads back only its own 4-byte word of each row) and the table entries (columns,
// weights, original id: 48 bytes) of 32 consecutive vertices in a double buffer, 32 ahead
// (the k_csr_i8_ring scheme with 32-byte rows).
template <int DEG, int S>
__host__ __device__ constexpr uint32_t packed_warp_bytes()
{
    return (uint32_t)S * (DEG + 1) * 128u + 2u * kRingMetaBuf;
}

template <int DEG, int S>
__global__ void __launch_bounds__(256, kI8PackedMinBlocks) k_csr_packed(const CsrI8Params p, uint32_t *P,
                                                                         uint32_t nslice, uint32_t chunk)
{
    extern __shared__ __align__(16) unsigned char pk_smem[];
    constexpr uint32_t kSlot = (DEG + 1) * 128u;
    constexpr uint32_t kRing = S * kSlot;
    const uint32_t lane = threadIdx.x;
    const uint32_t gw = blockIdx.x * blockDim.y + threadIdx.y;
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    const uint32_t slice = gw % nslice;
    const uint32_t j0 = (gw / nslice) * chunk;
    if (j0 >= nv)
        return;
    const uint32_t cnt = min(chunk, nv - j0);
    const uint32_t o = slice * 32u + lane;  // local replicas 8o .. 8o+7
    const uint32_t a = lane & 3u;
    const uint32_t rwb = (uint32_t)p.R >> 3;  // packed row bytes
    // this lane's word column of the packed rows (an opaque register copy, as in the ring kernel)
    char *tbb;
    asm volatile("mov.b64 %0, %1;" : "=l"(tbb) : "l"(reinterpret_cast<char *>(P) + 4u * (slice * 8u + (lane >> 2))));
    const uint32_t g0 = (uint32_t)(p.slot0 >> 3) + o;
    float bl[8];
    {
        const float4 *bp = reinterpret_cast<const float4 *>(p.betaf) + 2u * o;
        const float4 q0 = __ldg(bp), q1 = __ldg(bp + 1);
        const float b2[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
            bl[i] = __fmul_rn(b2[i], kLog2e);
    }
    const PhiloxHoist ph = philox_hoist(p.t, g0, p.rk);
    // 0x4B000000 (= 2^23) in a register the compiler cannot fold, so the PRMT building 2^23 + hi16
    // takes its selector as an immediate (else two selector constants are re-materialised per vertex)
    const uint32_t c4b = 0x4B000000u | ((uint32_t)p.R >> 31);  // p.R > 0: the bit is 0
    uint32_t pm[DEG];
#pragma unroll
    for (int u = 0; u < DEG; ++u)
        pm[u] = ((lane >> u) & 1u) << 31;
    const uint32_t amask = 0x11111111u << a;
    const uint32_t wsh = (uint32_t)__cvta_generic_to_shared(pk_smem) + threadIdx.y * packed_warp_bytes<DEG, S>();
    const uint32_t ring0 = wsh + lane * 4u;
    const uint32_t meta0 = wsh + kRing;
    const uint32_t vb = (uint32_t)p.v_begin + j0;
    auto meta_issue = [&](uint32_t blk) {
        const uint32_t j = blk * 32u + lane;
        if (j < cnt) {
            const uint32_t me = meta0 + (blk & 1u) * kRingMetaBuf + lane * kRingEntry;
            cp_async16(me, p.ell_col + 4u * (vb + j));
            cp_async16(me + 16u, p.ell_w + 4u * (vb + j));
            cp_async4(me + 32u, p.orig + vb + j);
        }
    };
    const uint32_t meta_end = meta0 + 2u * kRingMetaBuf;
    auto rows_issue = [&](uint32_t j, uint32_t sl, uint32_t e) {
        const int4 c = lds128(e);
        cp_async4(sl, tbb + (uint64_t)(vb + j) * rwb);
        cp_async4(sl + 128u, tbb + (uint64_t)(uint32_t)c.x * rwb);
        if (DEG > 1)
            cp_async4(sl + 256u, tbb + (uint64_t)(uint32_t)c.y * rwb);
        if (DEG > 2)
            cp_async4(sl + 384u, tbb + (uint64_t)(uint32_t)c.z * rwb);
        if (DEG > 3)
            cp_async4(sl + 512u, tbb + (uint64_t)(uint32_t)c.w * rwb);
    };
    meta_issue(0);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
#pragma unroll
    for (uint32_t j = 0; j + 1 < S; ++j) {
        if (j < cnt)
            rows_issue(j, ring0 + j * kSlot, meta0 + j * kRingEntry);
        cp_commit();
    }
    constexpr uint32_t U = kI8PackedUnroll;
    static_assert(U % S == 0 && 32 % U == 0, "unroll must be a multiple of the ring depth dividing 32");
    // (measured and dropped: a main loop without the per-vertex bounds tests, with a checked tail
    // loop, -1%; the next vertex's Philox call issued before this vertex's decision, -4.6%)
    uint32_t e_cur = meta0;
    uint32_t sink = lane;  // kI8PackedNoMem probe: keeps the decisions live
    for (uint32_t jb = 0; jb < cnt; jb += U) {
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const uint32_t j = jb + u;
            if (j >= cnt)
                break;
            if (u == 0 && (jb & 31u) == 0) {
                __syncwarp();
                meta_issue((j >> 5) + 1);
            }
            if (!kI8PackedNoMem && j + S - 1 < cnt)
                rows_issue(j + S - 1, ring0 + ((u + S - 1) % S) * kSlot, meta0 + ((j + S - 1) & 63u) * kRingEntry);
            cp_commit();
            cp_wait<S - 1>();
            if (u == S - 1 && (jb & 31u) == 0)
                __syncwarp();
            const uint32_t sl = ring0 + (u % S) * kSlot;
            uint32_t own, nb[DEG];
            if (kI8PackedNoMem) {  // timing probe only (wrong results): rows from registers
                own = (j * 0x9E3779B9u) ^ (lane * 0x01000193u);  // independent of earlier vertices
#pragma unroll
                for (int q = 0; q < DEG; ++q)
                    nb[q] = own * (0x85EBCA6Bu + 2u * q);
            } else {
                own = lds32(sl);
#pragma unroll
                for (int q = 0; q < DEG; ++q)
                    nb[q] = lds32(sl + (q + 1) * 128u);
            }
            const int4 wq = lds128(e_cur + u * kRingEntry + 16u);
            const uint32_t io = lds32(e_cur + u * kRingEntry + 32u);
            const uint32_t fl = packed_decide<DEG>(p, own, nb, wq, io, a, pm, bl, ph, g0, o, c4b, amask);
            if (kI8PackedNoMem)
                sink += fl;
            else if (a == 0u)
                asm volatile("st.global.cg.u32 [%0], %1;" ::"l"(tbb + (uint64_t)(vb + j) * rwb), "r"(own ^ fl)
                             : "memory");
        }
        e_cur = e_cur + U * kRingEntry == meta_end ? meta0 : e_cur + U * kRingEntry;
    }
    cp_wait<0>();
    if (kI8PackedNoMem && sink == 0x7FFFFFFFu)
        P[0] = sink;
}

template <int DEG, int S>
cudaError_t launch_packed_deg(const CsrI8Params &p, uint32_t *P, cudaStream_t st)
{
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    if (nv == 0)
        return cudaSuccess;
    const uint32_t nslice = (uint32_t)p.R / 256u;
    const size_t smem = (size_t)8 * packed_warp_bytes<DEG, S>();
    static int per_sm = 0;
    if (!per_sm) {
        cudaError_t e = cudaFuncSetAttribute(k_csr_packed<DEG, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_csr_packed<DEG, S>, 256, smem);
        if (e != cudaSuccess)
            return e;
        if (per_sm < 1)
            return cudaErrorInvalidConfiguration;
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t want = (uint32_t)nsm * (uint32_t)per_sm * 8u;  // one wave of resident warps
    uint32_t nch = want / nslice;
    if (nch < 1)
        nch = 1;
    if (nch > nv)
        nch = nv;
    uint32_t chunk = (nv + nch - 1) / nch;
    if (chunk < 40u)
        chunk = 40u;
    nch = (nv + chunk - 1) / chunk;
    const uint32_t warps = nch * nslice;
    k_csr_packed<DEG, S><<<(warps + 7) / 8, dim3(32, 8), smem, st>>>(p, P, nslice, chunk);
    return cudaGetLastError();
}

cudaError_t launch_pack_rows(const int8_t *s, uint32_t *P, int64_t n, int64_t R, bool unpack, cudaStream_t st)
{
    if (R % 32 != 0)
        return cudaErrorInvalidValue;
    const uint64_t nwords = (uint64_t)n * (uint64_t)(R / 32);
    if (nwords == 0)
        return cudaSuccess;
    const uint64_t want = (nwords + 255) / 256;
    const unsigned grid = (unsigned)(want < 148ull * 16 ? want : 148ull * 16);
    if (unpack)
        k_unpack_rows<<<grid, 256, 0, st>>>(P, const_cast<int8_t *>(s), nwords);
    else
        k_pack_rows<<<grid, 256, 0, st>>>(s, P, nwords);
    return cudaGetLastError();
}

cudaError_t launch_csr_packed_phase(const CsrI8Params &p, uint32_t *P, cudaStream_t st)
{
    if (!p.wf || !p.ell_col || p.R % 256 != 0 || p.slot0 % 8 != 0)
        return cudaErrorInvalidValue;
    switch (p.ell_deg) {
    case 1: return launch_packed_deg<1, kI8PackedRing>(p, P, st);
    case 2: return launch_packed_deg<2, kI8PackedRing>(p, P, st);
    case 3: return launch_packed_deg<3, kI8PackedRing>(p, P, st);
    default: return launch_packed_deg<4, kI8PackedRing>(p, P, st);
    }
}

cudaError_t launch_csr_i8_phase(const CsrI8Params &p, int32_t threads, cudaStream_t st)
{
    if (p.R % 8 != 0 || p.slot0 % 8 != 0)
        return cudaErrorInvalidValue;
    const int64_t nv = (int64_t)(p.v_end - p.v_begin);
    if (nv <= 0)
        return cudaSuccess;
    const int32_t ntv = p.R / 8;  // threads per vertex
    if (threads < 32 || threads > kI8Threads)
        threads = kI8Threads;
    const int32_t bx = ntv < threads ? ntv : threads;
    const int32_t by = threads / bx;
    const int64_t gy = (ntv + bx - 1) / bx;
    if (gy > 65535)
        return cudaErrorInvalidValue;
    const int64_t want = (nv + by - 1) / by;
    const int64_t cap = (int64_t)148 * 64 / (gy < 64 ? gy : 64);  // a few waves of resident CTAs
    const dim3 grid((unsigned)(want < cap ? want : cap), (unsigned)gy);
    const dim3 block((unsigned)bx, (unsigned)by);
    const bool ell = p.ell_col != nullptr;
    if (p.wf) {
        if (ell && kI8Ring > 0 && p.R % 256 == 0) {
            switch (p.ell_deg) {
            case 1: return launch_ring<1, kI8Ring>(p, st);
            case 2: return launch_ring<2, kI8Ring>(p, st);
            case 3: return launch_ring<3, kI8Ring>(p, st);
            default: return launch_ring<4, kI8Ring>(p, st);
            }
        } else if (ell && kI8Pipe) {
            switch (p.ell_deg) {
            case 1: k_csr_i8_pipe<1><<<grid, block, 0, st>>>(p); break;
            case 2: k_csr_i8_pipe<2><<<grid, block, 0, st>>>(p); break;
            case 3: k_csr_i8_pipe<3><<<grid, block, 0, st>>>(p); break;
            default: k_csr_i8_pipe<4><<<grid, block, 0, st>>>(p); break;
            }
        }
        else if (ell) k_csr_i8_phase<true, true><<<grid, block, 0, st>>>(p);
        else k_csr_i8_phase<true, false><<<grid, block, 0, st>>>(p);
    } else {
        if (ell) k_csr_i8_phase<false, true><<<grid, block, 0, st>>>(p);
        else k_csr_i8_phase<false, false><<<grid, block, 0, st>>>(p);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- fused small int8 PT
// Small instances with integer weights (C1: a 16x16 torus, 64 slots = 16 KB): one CTA per
// copy keeps the copy's n x K spins in shared memory for ALL rounds of a PT run -- k_ex
// sweeps (the k_csr_i8_phase arithmetic: relative-sign integer field, WORD contract, host
// threshold table), the energies of the K slots, the copy's best-so-far check, the exchange
// decisions and the configuration swaps -- instead of ~24 launches per
// round, each a few microseconds of work.  Per-copy best records are merged afterwards by
// k_merge_copy_best, as for the bit-packed fused launch.
__global__ void __launch_bounds__(kI8SmallThreads, 1) k_i8_small(const SmallI8Params p)
{
    extern __shared__ __align__(16) unsigned char small_smem[];
    const int K = p.K, n = p.n, tid = threadIdx.x, nt = blockDim.x;
    const int c = blockIdx.x;  // local copy
    int8_t *S = reinterpret_cast<int8_t *>(small_smem);                       // [n][K]
    int64_t *E = reinterpret_cast<int64_t *>(small_smem + (((size_t)n * K + 15) & ~(size_t)15));  // [K]
    int64_t *W = E + K;                                                         // [K] walker ids
    const int nparts = nt / K;
    int64_t *part = W + K;                                                      // [nparts][K]
    uint64_t *Ts = reinterpret_cast<uint64_t *>(part + (size_t)nparts * K);    // [K][qmax+1]
    __shared__ uint32_t mswap[8];
    __shared__ int64_t bestE, bestSlot, bestSweep;
    __shared__ int32_t kmin, improve;
    const int64_t slot_c = p.slot0 + (int64_t)c * K;  // global slot of the copy's slot 0
    const uint32_t c_global = (uint32_t)(slot_c / K);
    for (int x = tid; x < n * K; x += nt) {
        const int v = x / K, k = x - v * K;
        S[x] = p.s[(size_t)v * p.R + (size_t)c * K + k];
    }
    for (int k = tid; k < K; k += nt)
        W[k] = p.walker[(size_t)c * K + k];
    for (int x = tid; x < K * (p.qmax + 1); x += nt)  // this copy's rows of the threshold table
        Ts[x] = p.T[(size_t)c * K * (p.qmax + 1) + x];
    if (tid == 0) {
        bestE = INT64_MAX;
        bestSlot = -1;
        bestSweep = -1;
    }
    __syncthreads();
    const int ng = K / 8;  // 8-replica groups per vertex
    for (int round = 0; round < p.n_rounds; ++round) {
        for (int sw = 0; sw < p.k_ex; ++sw) {
            const uint32_t t = p.t0 + (uint32_t)(round * p.k_ex + sw);
            for (int cl = 0; cl < p.ncol; ++cl) {
                const int v0 = p.class_off[cl], nvc = p.class_off[cl + 1] - v0;
                for (int task = tid; task < nvc * ng; task += nt) {
                    const int v = v0 + task / ng, o = task - (task / ng) * ng;
                    uint2 *own_p = reinterpret_cast<uint2 *>(S + (size_t)v * K + 8 * o);
                    const uint2 own = *own_p;
                    int32_t sh[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        sh[b] = 0;
                    for (int e = __ldg(p.rp + v); e < __ldg(p.rp + v + 1); ++e) {
                        const uint2 nb = *reinterpret_cast<const uint2 *>(S + (size_t)__ldg(p.col + e) * K + 8 * o);
                        const int32_t w = __ldg(p.wi + e);
                        const uint32_t x0 = own.x ^ nb.x, x1 = own.y ^ nb.y;
#pragma unroll
                        for (int b = 0; b < 8; ++b) {
                            const uint32_t word = b < 4 ? x0 : x1;
                            const int32_t m = (int32_t)(word << (24 - 8 * (b & 3))) >> 31;  // -1 iff s_i != s_j
                            sh[b] += (w ^ m) - m;
                        }
                    }
                    const uint32_t io = __ldg(p.orig + v);
                    const uint32_t g = (uint32_t)(slot_c >> 3) + (uint32_t)o;
                    const uint4 h = philox(io, t, g, ST_WORD_HI << 24, p.rk);
                    const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
                    uint32_t fm0 = 0u, fm1 = 0u;
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        bool acc = sh[b] >= 0;  // dE = -2 s h <= 0
                        if (!acc) {
                            const uint32_t hb = (b & 1) ? (hw[b >> 1] >> 16) : (hw[b >> 1] & 0xFFFFu);
                            const uint64_t T = Ts[(size_t)(8 * o + b) * (p.qmax + 1) + (uint32_t)(-sh[b])];
                            acc = exact_less(hb, T, io, t, (uint32_t)(slot_c + 8 * o + b), p.rk);
                        }
                        if (acc) {
                            if (b < 4)
                                fm0 |= 0xFEu << (8 * (b & 3));
                            else
                                fm1 |= 0xFEu << (8 * (b & 3));
                        }
                    }
                    *own_p = make_uint2(own.x ^ fm0, own.y ^ fm1);
                }
                __syncthreads();
            }
        }
        // energies of the K slots: each edge once (from its lower internal endpoint)
        {
            const int k = tid % K, pt = tid / K;
            int64_t acc = 0;
            if (pt < nparts)
                for (int v = pt; v < n; v += nparts) {
                    const int32_t sv = S[(size_t)v * K + k];
                    for (int e = __ldg(p.rp + v); e < __ldg(p.rp + v + 1); ++e) {
                        const int j = __ldg(p.col + e);
                        if (j > v)
                            acc += (int64_t)__ldg(p.wi + e) * sv * S[(size_t)j * K + k];
                    }
                }
            if (pt < nparts)
                part[pt * K + k] = acc;
            __syncthreads();
            for (int kk = tid; kk < K; kk += nt) {
                int64_t e = 0;
                for (int q = 0; q < nparts; ++q)
                    e += part[q * K + kk];
                E[kk] = e;
            }
            if (tid < 8)
                mswap[tid] = 0u;
            __syncthreads();
        }
        const uint32_t t_now = p.t0 + (uint32_t)((round + 1) * p.k_ex);
        const uint32_t e_now = p.e0 + (uint32_t)round;
        if (tid < 32) {  // the copy's best-so-far: argmin, ties -> lowest slot; strict <
            int64_t bE = INT64_MAX;
            int bk = -1;
            for (int k = tid; k < K; k += 32)
                if (bk < 0 || E[k] < bE) {
                    bE = E[k];
                    bk = k;
                }
            for (int off = 16; off > 0; off >>= 1) {
                const int64_t oE = __shfl_down_sync(0xFFFFFFFFu, bE, off);
                const int ok = __shfl_down_sync(0xFFFFFFFFu, bk, off);
                if (ok >= 0 && (bk < 0 || oE < bE || (oE == bE && ok < bk))) {
                    bE = oE;
                    bk = ok;
                }
            }
            if (tid == 0) {
                improve = bE < bestE;
                kmin = bk;
                if (bE < bestE) {
                    bestE = bE;
                    bestSlot = slot_c + bk;
                    bestSweep = t_now;
                }
            }
        }
        __syncthreads();
        if (improve)
            for (int v = tid; v < n; v += nt)
                p.snap[(size_t)c * n + __ldg(p.orig + v)] = S[(size_t)v * K + kmin];
        // exchange e_now: pairs (k, k+1), k = e % 2 + 2 j (identical rule to k_exchange)
        const int par = (int)(e_now & 1u);
        for (int k = par + 2 * tid; k + 1 < K; k += 2 * nt) {
            const int64_t d = E[k + 1] - E[k];
            bool accept = d >= 0;
            if (!accept) {
                const int64_t j = -d - 1;
                if (j < __ldg(p.Tx_len + k)) {
                    const uint4 w = philox((uint32_t)k, e_now, c_global, ST_EXCH << 24, p.rk);
                    const uint64_t Ux = ((uint64_t)w.x << 32) | (uint64_t)w.y;
                    accept = Ux < __ldg(p.Tx + __ldg(p.Tx_off + k) + j);
                }
            }
            if (accept) {
                atomicOr(&mswap[k >> 5], 1u << (k & 31));
                const int64_t te = E[k];
                E[k] = E[k + 1];
                E[k + 1] = te;
                const int64_t tw = W[k];
                W[k] = W[k + 1];
                W[k + 1] = tw;
            }
        }
        __syncthreads();
        // configurations of accepted pairs trade places (the slot temperatures stay)
        const int npair = (K - par) / 2;
        for (int x = tid; x < n * npair; x += nt) {
            const int v = x / npair, k = par + 2 * (x - v * npair);
            if ((mswap[k >> 5] >> (k & 31)) & 1u) {
                int8_t *a = S + (size_t)v * K + k;
                const int8_t ta = a[0];
                a[0] = a[1];
                a[1] = ta;
            }
        }
        __syncthreads();
    }
    for (int x = tid; x < n * K; x += nt) {
        const int v = x / K, k = x - v * K;
        p.s[(size_t)v * p.R + (size_t)c * K + k] = S[x];
    }
    for (int k = tid; k < K; k += nt) {
        p.E_out[(size_t)c * K + k] = E[k];
        p.walker[(size_t)c * K + k] = W[k];
    }
    if (tid == 0) {
        p.copy_best[3 * c + 0] = bestE;
        p.copy_best[3 * c + 1] = bestSlot;
        p.copy_best[3 * c + 2] = bestSweep;
    }
}

// The same PT run with each copy spread over a cluster of K/8 CTAs: CTA q holds the copy's
// slots 8q .. 8q+7 (one 8-replica group: n x 8 bytes), so the sweeps of a small instance run on
// K/8 SMs instead of one.  Only the exchange couples the CTAs: the slots' energies are gathered
// through distributed shared memory, every CTA takes the same decisions, and the pair that
// crosses two CTAs in odd exchanges (slots 8q+7, 8q+8) trades its byte columns over DSMEM
// (both sides copy the other's column into a buffer, synchronise, then write).
//
// REG (every colour class has at most kI8ClusterThreads vertices, at most kRegCol classes, degree
// <= 4: C1's 16 x 16 torus): thread tid owns vertex tid of every class for the whole launch and
// keeps its padded neighbour row, weights and original id in registers, so a colour phase is one
// dependent chain of shared-memory loads, one hoisted Philox call and the decisions, with no
// global CSR loads; the per-round energies come from the same registers (each bond from its
// lower internal endpoint) and a warp-shuffle reduction.
// The 8 slots of a vertex are split over 8 / kRegRPT threads (kRegRPT replicas each, one
// redundant Philox call per thread): more warps per SM to hide the dependent chain of a phase.
constexpr int kI8ClusterThreads = 128;
constexpr int kRegCol = 4;
constexpr int kRegVerts = 128;  // vertices of a class per CTA row of threads
#ifndef ISING_I8_REG_RPT
#define ISING_I8_REG_RPT 4
#endif
constexpr int kRegRPT = ISING_I8_REG_RPT;  // replicas per thread
constexpr int kI8ClusterRegThreads = kRegVerts * (8 / kRegRPT);

template <bool REG>
__global__ void __launch_bounds__(REG ? kI8ClusterRegThreads : kI8ClusterThreads, 1)
    k_i8_cluster(const SmallI8Params p)
{
    extern __shared__ __align__(16) unsigned char cl_smem[];
    const int K = p.K, n = p.n, tid = threadIdx.x, nt = blockDim.x;
    const int NC = K / 8;
    cg::cluster_group cl = cg::this_cluster();
    const int q = (int)cl.block_rank();              // this CTA's 8-slot group of the copy
    const int c = (int)(blockIdx.x / (unsigned)NC);  // local copy
    uint2 *S = reinterpret_cast<uint2 *>(cl_smem);                      // [n] 8 slots each
    int8_t *xlo = reinterpret_cast<int8_t *>(S + n);                    // [n] prev CTA's slot 7
    int8_t *xhi = xlo + n;                                              // [n] next CTA's slot 0
    int64_t *Ecopy = reinterpret_cast<int64_t *>(cl_smem + (((size_t)n * 10 + 15) & ~(size_t)15));
    int64_t *Wcopy = Ecopy + K;
    int64_t *Eown = Wcopy + K;                                          // [8]
    int64_t *part = Eown + 8;                                           // [nt]
    uint64_t *Ts = reinterpret_cast<uint64_t *>(part + nt);            // [8][qmax+1]
    __shared__ uint32_t mswap[2];
    __shared__ int64_t bestE, bestSlot, bestSweep;
    __shared__ int32_t kmin, improve;
    const int64_t slot_c = p.slot0 + (int64_t)c * K;
    const uint32_t c_global = (uint32_t)(slot_c / K);
    const size_t col0 = (size_t)c * K + 8 * q;  // first local replica column of this CTA
    for (int v = tid; v < n; v += nt)
        S[v] = *reinterpret_cast<const uint2 *>(p.s + (size_t)v * p.R + col0);
    for (int k = tid; k < K; k += nt)
        Wcopy[k] = p.walker[(size_t)c * K + k];
    for (int x = tid; x < 8 * (p.qmax + 1); x += nt)
        Ts[x] = p.T[col0 * (p.qmax + 1) + x];
    if (tid == 0) {
        bestE = INT64_MAX;
        bestSlot = -1;
        bestSweep = -1;
    }
    __syncthreads();
    const uint32_t g = (uint32_t)(slot_c >> 3) + (uint32_t)q;
    int8_t *Sb = reinterpret_cast<int8_t *>(S);
    // REG: this thread's vertex of each class (-1: none), its padded row, weights, original id
    int rv[kRegCol], rnb[kRegCol][4];
    int32_t rw[kRegCol][4];
    uint32_t rio[kRegCol];
#pragma unroll
    for (int cc = 0; cc < kRegCol; ++cc) {
        rv[cc] = -1;
        rio[cc] = 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            rnb[cc][u] = 0;
            rw[cc][u] = 0;
        }
        if (REG && cc < p.ncol) {
            const int v = __ldg(p.class_off + cc) + tid % kRegVerts;
            if (v < __ldg(p.class_off + cc + 1)) {
                rv[cc] = v;
                const int4 c4 = __ldg(reinterpret_cast<const int4 *>(p.ell_col) + v);
                const int4 w4 = __ldg(reinterpret_cast<const int4 *>(p.ell_w) + v);
                const int cs[4] = {c4.x, c4.y, c4.z, c4.w}, ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    rnb[cc][u] = cs[u] >= 0 ? cs[u] : v;  // pad: own row, weight 0
                    rw[cc][u] = cs[u] >= 0 ? ws[u] : 0;
                }
                rio[cc] = __ldg(p.orig + v);
            }
        }
    }
    for (int round = 0; round < p.n_rounds; ++round) {
        for (int sw = 0; sw < p.k_ex; ++sw) {
            const uint32_t t = p.t0 + (uint32_t)(round * p.k_ex + sw);
            if (REG) {
                // thread (vertex tid % kRegVerts, replicas sub*kRegRPT .. +kRegRPT-1 of the 8)
                const int sub = tid / kRegVerts;
                const int wi = (sub * kRegRPT) >> 2, bo = (sub * kRegRPT) & 3;  // word, first byte
                uint32_t *Sw = reinterpret_cast<uint32_t *>(S);
                const PhiloxHoist ph = philox_hoist(t, g, p.rk);
#pragma unroll
                for (int cc = 0; cc < kRegCol; ++cc) {
                    if (cc >= p.ncol)
                        break;
                    const int v = rv[cc];
                    if (v >= 0) {
                        const uint32_t own = Sw[2 * v + wi];
                        uint32_t nbw[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            nbw[u] = Sw[2 * rnb[cc][u] + wi];
                        const uint4 h = philox_hoisted(rio[cc], ph, p.rk);
                        // word (b >> 1) of the call for slot b = sub * kRegRPT + j, selected without
                        // a dynamically indexed array (which would live in local memory)
                        auto hword = [&](int j) {
                            const int k = (sub * kRegRPT + j) >> 1;
                            return k == 0 ? h.x : k == 1 ? h.y : k == 2 ? h.z : h.w;
                        };
                        int32_t sh[kRegRPT];
#pragma unroll
                        for (int j = 0; j < kRegRPT; ++j)
                            sh[j] = 0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t x = own ^ nbw[u];
                            const int32_t w = rw[cc][u];
#pragma unroll
                            for (int j = 0; j < kRegRPT; ++j) {
                                const int32_t m = (int32_t)(x << (24 - 8 * (bo + j))) >> 31;  // -1 iff s_i != s_j
                                sh[j] += (w ^ m) - m;
                            }
                        }
                        // branch-free decisions: every threshold row entry is loaded (row 0 for
                        // s h >= 0, unused), U < T is decided on the 16-bit high words, and only a
                        // tie of the high words (probability 2^-16) takes the lo48 call
                        uint64_t Tj[kRegRPT];
#pragma unroll
                        for (int j = 0; j < kRegRPT; ++j) {
                            const int b = sub * kRegRPT + j;
                            Tj[j] = Ts[(size_t)b * (p.qmax + 1) + (uint32_t)(sh[j] < 0 ? -sh[j] : 0)];
                        }
                        uint32_t fm = 0u;
#pragma unroll
                        for (int j = 0; j < kRegRPT; ++j) {
                            const int b = sub * kRegRPT + j;  // slot within this CTA's 8
                            const uint32_t hwj = hword(j);
                            const uint32_t hb = (b & 1) ? (hwj >> 16) : (hwj & 0xFFFFu);
                            const uint32_t th = (uint32_t)(Tj[j] >> 48);
                            bool acc = sh[j] >= 0 || hb < th;  // dE = -2 s h <= 0, or U < T by the high word
                            if (!acc && sh[j] < 0 && hb == th)
                                acc = lo48_of(rio[cc], t, (uint32_t)(slot_c + 8 * q + b), p.rk) <
                                      (Tj[j] & 0xFFFFFFFFFFFFull);
                            if (acc)
                                fm |= 0xFEu << (8 * (bo + j));
                        }
                        if (kRegRPT == 4) {
                            Sw[2 * v + wi] = own ^ fm;
                        } else if (kRegRPT == 2) {  // this thread's bytes only (the rest belong to peers)
                            uint16_t *Sh = reinterpret_cast<uint16_t *>(S);
                            Sh[4 * v + ((sub * kRegRPT) >> 1)] = (uint16_t)((own ^ fm) >> (8 * bo));
                        } else {
                            uint8_t *S8 = reinterpret_cast<uint8_t *>(S);
                            S8[8 * v + sub] = (uint8_t)((own ^ fm) >> (8 * bo));
                        }
                    }
                    __syncthreads();
                }
                continue;
            }
            for (int ccl = 0; ccl < p.ncol; ++ccl) {
                const int v0 = p.class_off[ccl], v1 = p.class_off[ccl + 1];
                for (int v = v0 + tid; v < v1; v += nt) {
                    const uint2 own = S[v];
                    int32_t sh[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        sh[b] = 0;
                    for (int e = __ldg(p.rp + v); e < __ldg(p.rp + v + 1); ++e) {
                        const uint2 nb = S[__ldg(p.col + e)];
                        const int32_t w = __ldg(p.wi + e);
                        const uint32_t x0 = own.x ^ nb.x, x1 = own.y ^ nb.y;
#pragma unroll
                        for (int b = 0; b < 8; ++b) {
                            const uint32_t word = b < 4 ? x0 : x1;
                            const int32_t m = (int32_t)(word << (24 - 8 * (b & 3))) >> 31;  // -1 iff s_i != s_j
                            sh[b] += (w ^ m) - m;
                        }
                    }
                    const uint32_t io = __ldg(p.orig + v);
                    const uint4 h = philox(io, t, g, ST_WORD_HI << 24, p.rk);
                    const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
                    uint32_t fm0 = 0u, fm1 = 0u;
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        bool acc = sh[b] >= 0;  // dE = -2 s h <= 0
                        if (!acc) {
                            const uint32_t hb = (b & 1) ? (hw[b >> 1] >> 16) : (hw[b >> 1] & 0xFFFFu);
                            const uint64_t T = Ts[(size_t)b * (p.qmax + 1) + (uint32_t)(-sh[b])];
                            acc = exact_less(hb, T, io, t, (uint32_t)(slot_c + 8 * q + b), p.rk);
                        }
                        if (acc) {
                            if (b < 4)
                                fm0 |= 0xFEu << (8 * (b & 3));
                            else
                                fm1 |= 0xFEu << (8 * (b & 3));
                        }
                    }
                    S[v] = make_uint2(own.x ^ fm0, own.y ^ fm1);
                }
                __syncthreads();
            }
        }
        if (REG) {  // energies of this CTA's 8 slots from the register rows (each bond once)
            const int sub = tid / kRegVerts;
            const int wi = (sub * kRegRPT) >> 2, bo = (sub * kRegRPT) & 3;
            const uint32_t *Sw = reinterpret_cast<const uint32_t *>(S);
            int32_t ea[kRegRPT];
#pragma unroll
            for (int j = 0; j < kRegRPT; ++j)
                ea[j] = 0;
#pragma unroll
            for (int cc = 0; cc < kRegCol; ++cc) {
                const int v = rv[cc];
                if (v < 0)
                    continue;
                const uint32_t own = Sw[2 * v + wi];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int jv = rnb[cc][u];
                    if (jv <= v)  // the bond is counted from its lower endpoint (pads: jv = v)
                        continue;
                    const uint32_t x = own ^ Sw[2 * jv + wi];
                    const int32_t w = rw[cc][u];
#pragma unroll
                    for (int j = 0; j < kRegRPT; ++j) {
                        const int32_t m = (int32_t)(x << (24 - 8 * (bo + j))) >> 31;
                        ea[j] += (w ^ m) - m;  // w s_v s_j
                    }
                }
            }
            // |partial| <= sum |w| < 2^30 (create-time guard): int32 warp sums, int64 over warps;
            // the warps of one replica group (sub) are tid / 32 in [sub * 4, sub * 4 + 4)
#pragma unroll
            for (int j = 0; j < kRegRPT; ++j)
                ea[j] = __reduce_add_sync(0xFFFFFFFFu, ea[j]);
            if ((tid & 31) == 0)
#pragma unroll
                for (int j = 0; j < kRegRPT; ++j)
                    part[(tid >> 5) * kRegRPT + j] = ea[j];
            __syncthreads();
            if (tid < 8) {
                constexpr int wpg = kRegVerts / 32;  // warps per replica group
                const int sb = tid / kRegRPT, jb = tid % kRegRPT;
                int64_t e = 0;
                for (int w = 0; w < wpg; ++w)
                    e += part[(sb * wpg + w) * kRegRPT + jb];
                Eown[tid] = e;
            }
            if (tid < 2)
                mswap[tid] = 0u;
        } else {  // energies of this CTA's 8 slots (each edge once, fixed-order partial sums)
            const int b = tid & 7, pt = tid >> 3, np = nt >> 3;
            int64_t acc = 0;
            for (int v = pt; v < n; v += np) {
                const int32_t sv = Sb[8 * v + b];
                for (int e = __ldg(p.rp + v); e < __ldg(p.rp + v + 1); ++e) {
                    const int j = __ldg(p.col + e);
                    if (j > v)
                        acc += (int64_t)__ldg(p.wi + e) * sv * Sb[8 * j + b];
                }
            }
            part[tid] = acc;
            __syncthreads();
            if (tid < 8) {
                int64_t e = 0;
                for (int x = 0; x < np; ++x)
                    e += part[8 * x + tid];
                Eown[tid] = e;
            }
            if (tid < 2)
                mswap[tid] = 0u;
        }
        cl.sync();  // every CTA's Eown complete
        for (int k = tid; k < K; k += nt)
            Ecopy[k] = cl.map_shared_rank(Eown, (unsigned)(k >> 3))[k & 7];
        __syncthreads();
        const uint32_t t_now = p.t0 + (uint32_t)((round + 1) * p.k_ex);
        const uint32_t e_now = p.e0 + (uint32_t)round;
        if (tid < 32) {  // the copy's best-so-far: argmin, ties -> lowest slot; strict <
            int64_t bE = INT64_MAX;
            int bk = -1;
            for (int k = tid; k < K; k += 32)
                if (bk < 0 || Ecopy[k] < bE) {
                    bE = Ecopy[k];
                    bk = k;
                }
            for (int off = 16; off > 0; off >>= 1) {
                const int64_t oE = __shfl_down_sync(0xFFFFFFFFu, bE, off);
                const int ok = __shfl_down_sync(0xFFFFFFFFu, bk, off);
                if (ok >= 0 && (bk < 0 || oE < bE || (oE == bE && ok < bk))) {
                    bE = oE;
                    bk = ok;
                }
            }
            if (tid == 0) {
                improve = bE < bestE;
                kmin = bk;
                if (bE < bestE) {
                    bestE = bE;
                    bestSlot = slot_c + bk;
                    bestSweep = t_now;
                }
            }
        }
        __syncthreads();
        if (improve && (kmin >> 3) == q)
            for (int v = tid; v < n; v += nt)
                p.snap[(size_t)c * n + __ldg(p.orig + v)] = Sb[8 * v + (kmin & 7)];
        const int par = (int)(e_now & 1u);
        for (int k = par + 2 * tid; k + 1 < K; k += 2 * nt) {  // same rule as k_exchange
            const int64_t d = Ecopy[k + 1] - Ecopy[k];
            bool accept = d >= 0;
            if (!accept) {
                const int64_t j = -d - 1;
                if (j < __ldg(p.Tx_len + k)) {
                    const uint4 w = philox((uint32_t)k, e_now, c_global, ST_EXCH << 24, p.rk);
                    const uint64_t Ux = ((uint64_t)w.x << 32) | (uint64_t)w.y;
                    accept = Ux < __ldg(p.Tx + __ldg(p.Tx_off + k) + j);
                }
            }
            if (accept) {
                atomicOr(&mswap[k >> 5], 1u << (k & 31));
                const int64_t te = Ecopy[k];
                Ecopy[k] = Ecopy[k + 1];
                Ecopy[k + 1] = te;
                const int64_t tw = Wcopy[k];
                Wcopy[k] = Wcopy[k + 1];
                Wcopy[k + 1] = tw;
            }
        }
        __syncthreads();
        auto accepted = [&](int k) { return ((mswap[k >> 5] >> (k & 31)) & 1u) != 0u; };
        // within-group pairs: local byte swaps
        for (int x = tid; x < n * 4; x += nt) {
            const int v = x >> 2, kk = par + 2 * (x & 3);  // kk, kk+1 inside this group
            if (kk + 1 < 8 && accepted(8 * q + kk)) {
                const int8_t a = Sb[8 * v + kk];
                Sb[8 * v + kk] = Sb[8 * v + kk + 1];
                Sb[8 * v + kk + 1] = a;
            }
        }
        // the pairs across groups (odd exchanges): uniform over the cluster
        bool any_cross = false;
        for (int r = 0; r + 1 < NC; ++r)
            any_cross |= par == 1 && accepted(8 * r + 7);
        if (any_cross) {
            const bool hi = par == 1 && q + 1 < NC && accepted(8 * q + 7);  // my slot 7 <-> next's slot 0
            const bool lo = par == 1 && q > 0 && accepted(8 * q - 1);       // prev's slot 7 <-> my slot 0
            cl.sync();  // every CTA's within-group swaps done (slots 0 and 7 are not touched by them)
            const int8_t *nxt = hi ? reinterpret_cast<const int8_t *>(cl.map_shared_rank(S, (unsigned)(q + 1))) : nullptr;
            const int8_t *prv = lo ? reinterpret_cast<const int8_t *>(cl.map_shared_rank(S, (unsigned)(q - 1))) : nullptr;
            for (int v = tid; v < n; v += nt) {
                if (hi)
                    xhi[v] = nxt[8 * v + 0];
                if (lo)
                    xlo[v] = prv[8 * v + 7];
            }
            cl.sync();  // every CTA has copied what it takes before anything is overwritten
            for (int v = tid; v < n; v += nt) {
                if (hi)
                    Sb[8 * v + 7] = xhi[v];
                if (lo)
                    Sb[8 * v + 0] = xlo[v];
            }
        }
        __syncthreads();
    }
    for (int v = tid; v < n; v += nt)
        *reinterpret_cast<uint2 *>(p.s + (size_t)v * p.R + col0) = S[v];
    for (int b = tid; b < 8; b += nt)
        p.E_out[col0 + b] = Ecopy[8 * q + b];
    if (q == 0) {
        for (int k = tid; k < K; k += nt)
            p.walker[(size_t)c * K + k] = Wcopy[k];
        if (tid == 0) {
            p.copy_best[3 * c + 0] = bestE;
            p.copy_best[3 * c + 1] = bestSlot;
            p.copy_best[3 * c + 2] = bestSweep;
        }
    }
    cl.sync();  // no CTA exits while a peer may still read its shared memory
}

cudaError_t launch_i8_small(const SmallI8Params &p, int32_t C_local, cudaStream_t st)
{
    const int nparts = kI8SmallThreads / p.K;
    const size_t smem = (((size_t)p.n * p.K + 15) & ~(size_t)15) + (size_t)(2 + nparts) * p.K * 8 +
                        (size_t)p.K * (p.qmax + 1) * 8;
    if (kI8Cluster && p.K / 8 <= 8) {  // each copy on a cluster of K/8 CTAs (8 slots each)
        const int NC = p.K / 8;
        // register rows: every class fits one thread row per vertex, at most kRegCol classes,
        // degree <= 4
        const bool reg = p.ell_col != nullptr && p.ncol <= kRegCol && p.max_class <= kRegVerts;
        const int nthr = reg ? kI8ClusterRegThreads : kI8ClusterThreads;
        const size_t cs = (((size_t)p.n * 10 + 15) & ~(size_t)15) + (size_t)(2 * p.K + 8 + nthr) * 8 +
                          (size_t)8 * (p.qmax + 1) * 8;
        auto kern = reg ? k_i8_cluster<true> : k_i8_cluster<false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
        if (e != cudaSuccess)
            return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(C_local * NC));
        cfg.blockDim = dim3((unsigned)nthr);
        cfg.dynamicSmemBytes = cs;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)NC;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, p);
    }
    cudaError_t e = cudaFuncSetAttribute(k_i8_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    k_i8_small<<<C_local, kI8SmallThreads, smem, st>>>(p);
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

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

// e = ex2.approx(fma(x, log2 e, 16)) estimates cexp32(x) 2^16 = T / 2^48 with relative
// error below 2^-17 (measured 3.6e-6 = 2^-18.1, checked exhaustively over every float x in
// [-64, 0] by ising_debug_exp_bound, which evaluates this exact expression).  With the
// 2^-16 margin (> twice the error bound):
//   2^23 + hi16 <= RN(e (1 - 2^-16) + 2^23 - 2)  =>  hi16 + 1 <= T / 2^48  =>  accept
//   2^23 + hi16 >= RN(e (1 + 2^-16) + 2^23 + 1)  =>  hi16 > T / 2^48      =>  reject
// (the RN of a value near 2^23 is within 1/2, covered by the -2 / +1 slack)
// and anything else is decided exactly.  For x < -64 (T = 0) e < 2^-76,
// so only hi16 = 0 stays undecided and the exact path rejects it.
__device__ __forceinline__ float exp_est16(float x)
{
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmaf_rn(x, 0x1.715476p+0f, 16.0f)));
    return e;
}

constexpr float kLoMargin = 1.0f - 0x1p-16f, kHiMargin = 1.0f + 0x1p-16f;

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

// Exhaustive check of the fast-decision bound: max over all float x in [-64, 0] of
// |exp_est16(x) / (cexp32(x) 2^16) - 1|, as float bits in *out (atomicMax).
__global__ void k_debug_exp_bound(uint32_t *out)
{
    const uint32_t lo = 0x80000000u, hi = 0xC2800000u;  // -0 .. -64
    float worst = 0.f;
    for (uint64_t b = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= hi;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((uint32_t)b);
        const float e = exp_est16(x);
        const float c = __fmul_rn(cexp32(x), 0x1p16f);
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
            const float b2[4] = {bq.x, bq.y, bq.z, bq.w};
            uint32_t fm = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                // x = -(beta dE) = (2 beta)(s h) exactly; s h >= 0 flips
                const float xv = __fmul_rn(b2[b], sh[b]);
                const float e = exp_est16(xv);
                const uint32_t hword = hw[2 * half + (b >> 1)];
                const float hf = (b & 1) ? hi16_f<1>(hword) : hi16_f<0>(hword);  // 2^23 + hi16
                const bool acc = sh[b] >= 0.0f || hf <= __fmaf_rn(e, kLoMargin, 0x1p23f - 2.0f);
                const bool dec = acc || hf >= __fmaf_rn(e, kHiMargin, 0x1p23f + 1.0f);
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
                const float xv = __fmul_rn(__ldg(p.betaf + 8u * o + (uint32_t)b), shb);
                const uint32_t hword = (b >> 1) == 0 ? hw[0] : (b >> 1) == 1 ? hw[1] : (b >> 1) == 2 ? hw[2] : hw[3];
                const uint32_t hb = (b & 1) ? (hword >> 16) : (hword & 0xFFFFu);
                if (shb >= 0.0f)
                    continue;
                const float e = exp_est16(xv);
                const float hf = __uint_as_float(0x4B000000u | hb);
                if (hf <= __fmaf_rn(e, kLoMargin, 0x1p23f - 2.0f) || hf >= __fmaf_rn(e, kHiMargin, 0x1p23f + 1.0f))
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

// Float weights + padded neighbour table, two-deep software pipeline: while vertex k is
// decided, the spin rows of vertex k+1 are already in flight (issued at the top of iteration
// k) and the table row of vertex k+2 is being loaded, so each warp keeps two vertices' gathers
// outstanding.
__global__ void __launch_bounds__(kI8Threads, kI8PipeMinBlocks) k_csr_i8_pipe(const CsrI8Params p)
{
    const uint32_t rw = (uint32_t)p.R >> 2;
    const uint32_t ntv = rw >> 1;
    const uint32_t o = blockIdx.y * blockDim.x + threadIdx.x;
    if (o >= ntv)
        return;
    const uint32_t nv = (uint32_t)(p.v_end - p.v_begin);
    const uint32_t vstride = gridDim.x * blockDim.y;
    uint32_t *tb = reinterpret_cast<uint32_t *>(p.s) + 2u * o;
    const char *tbb = reinterpret_cast<const char *>(tb);
    const uint32_t rwb = 4u * rw;
    const uint32_t g0 = (uint32_t)(p.slot0 >> 3) + o;
    const float4 *bp = reinterpret_cast<const float4 *>(p.betaf) + 2u * o;
    const int deg = p.ell_deg;
    const int4 *ec = reinterpret_cast<const int4 *>(p.ell_col) + p.v_begin;
    const int4 *ew = reinterpret_cast<const int4 *>(p.ell_w) + p.v_begin;
    const uint32_t *eo = p.orig + p.v_begin;
    uint32_t vv = blockIdx.x * blockDim.y + threadIdx.y;
    if (vv >= nv)
        return;
    auto rows = [&](uint32_t vq, const int4 &c, uint2 &own, uint2 (&nb)[4]) {
        own = *reinterpret_cast<const uint2 *>(tbb + (p.v_begin + vq) * rwb);
        const int32_t cs[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (u < deg)
                nb[u] = __ldg(reinterpret_cast<const uint2 *>(tbb + (uint32_t)cs[u] * rwb));
    };
    // prologue: table rows of vertices 0 and 1, spin rows of vertex 0
    int4 c1 = __ldg(ec + vv), w1 = __ldg(ew + vv);
    uint32_t io1 = __ldg(eo + vv);
    uint2 own1, nb1[4];
    rows(vv, c1, own1, nb1);
    uint32_t vq2 = vv + vstride;
    int4 c2 = make_int4(0, 0, 0, 0), w2 = make_int4(0, 0, 0, 0);
    uint32_t io2 = 0;
    if (vq2 < nv) {
        c2 = __ldg(ec + vq2);
        w2 = __ldg(ew + vq2);
        io2 = __ldg(eo + vq2);
    }
    for (; vv < nv; vv += vstride) {
        // current vertex: rows and meta from the previous iteration
        const uint2 own = own1;
        uint2 nb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            nb[u] = nb1[u];
        const int4 wq = w1;
        const uint32_t io = io1;
        // next vertex: issue its spin-row gathers now; the one after: its table row
        const uint32_t vn = vv + vstride;
        if (vn < nv) {
            rows(vn, c2, own1, nb1);
            w1 = w2;
            io1 = io2;
            const uint32_t vn2 = vn + vstride;
            if (vn2 < nv) {
                c2 = __ldg(ec + vn2);
                w2 = __ldg(ew + vn2);
                io2 = __ldg(eo + vn2);
            }
        }
        uint2 x[4];
        const uint32_t wv[4] = {(uint32_t)wq.x, (uint32_t)wq.y, (uint32_t)wq.z, (uint32_t)wq.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
            x[u] = u < deg ? make_uint2(own.x ^ nb[u].x, own.y ^ nb[u].y) : make_uint2(0u, 0u);
        const uint4 h = philox_w(io, p.t, g0, ST_WORD_HI << 24, p.rk);
        const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
        uint32_t fm0 = 0u, fm1 = 0u;
        const int32_t v = p.v_begin + (int32_t)vv;
        float_decide<true>(p, v, own, x, wv, tb, rw, io, g0, o, bp, hw, fm0, fm1);
        *reinterpret_cast<uint2 *>(tb + (size_t)(uint32_t)v * rw) = make_uint2(own.x ^ fm0, own.y ^ fm1);
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
        if (ell && kI8Pipe) k_csr_i8_pipe<<<grid, block, 0, st>>>(p);
        else if (ell) k_csr_i8_phase<true, true><<<grid, block, 0, st>>>(p);
        else k_csr_i8_phase<true, false><<<grid, block, 0, st>>>(p);
    } else {
        if (ell) k_csr_i8_phase<false, true><<<grid, block, 0, st>>>(p);
        else k_csr_i8_phase<false, false><<<grid, block, 0, st>>>(p);
    }
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

// k_csr_bits.cu -- multi-spin-coded Metropolis sweeps on a +-1 CSR graph (sm_100a).
//
// Rows a3-a7 of SURVEY.md §8(a) for the sparse-random-graph workload (C3: G70
// stand-in, "Unweighted MaxCut on sparse random graph", encoded
// J = +1 in CSR with a greedy colouring).  Same structure as k_grid_bits: one CTA
// owns one 32-replica word group resident in shared memory for a whole launch;
// colour classes are contiguous in the internal vertex order (sorted by degree inside
// a class, so a warp mostly sees one degree); the CSR itself (~120 KB for C3) is read
// through the L1/read-only path.  Two-stage RNG-tail compaction and the fused PT step
// are shared with the grid kernel (bits_core.cuh).
//
// Per (vertex of degree d, word): a_b = ~(s_i ^ s_j ^ J_b) for every neighbour, summed
// into a 4-bit vertical counter u; dE = -2 s h = 2d - 4u > 0 <=> u < ceil(d/2); the
// lane's threshold row is q = dE/2 = d - 2u, selected per plane by a multiplexer tree
// over the bits of u (plane rows P[q][j], q = 1..qmax).
#include "bits_core.cuh"

namespace ising {

using namespace bits;

namespace {

constexpr int kRow = 68;  // plane-row stride in words (16-byte aligned rows)
constexpr int kCsrCnt = 14;
constexpr int kCsrQItem = 12;

struct CsrSite {
    uint32_t own, D, u0, u1, u2;
    int d;
};

// Evaluate vertex v (internal id) of the current class on the words in S.
__device__ __forceinline__ CsrSite csr_eval(const uint32_t *S, const CsrBitsParams &p, int v)
{
    CsrSite r;
    r.own = S[v];
    const int e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
    r.d = e1 - e0;
    uint32_t u[4] = {0u, 0u, 0u, 0u};
    for (int e = e0; e < e1; ++e) {
        const uint32_t nb = __ldg(p.nbr + e);
        const uint32_t jm = (uint32_t)((int32_t)nb >> 31);
        vadd(u, ~(r.own ^ S[nb & 0x7FFFFFFFu] ^ jm));
    }
    // D = lanes with u < ceil(d/2), by a bit-sliced comparison with the constant
    const uint32_t cth = (uint32_t)(r.d + 1) >> 1;
    uint32_t lt = 0u, eq = ~0u;
#pragma unroll
    for (int l = 3; l >= 0; --l) {
        const uint32_t cb = 0u - ((cth >> l) & 1u);
        lt |= eq & ~u[l] & cb;
        eq &= ~(u[l] ^ cb);
    }
    r.D = lt;
    r.u0 = u[0];
    r.u1 = u[1];
    r.u2 = u[2];
    return r;
}

// csr_eval for a vertex of small, compile-time degree DEG (the warp's vertices share it: a
// class is sorted by degree): the unsatisfied-bond count u of the DEG bonds by a fixed adder and
// D = {u < ceil(DEG/2)} directly, instead of the general loop's 4-bit vertical counter and
// bit-sliced comparison.  u1, u2 are only used by the threshold multiplexer for DEG > 4.
template <int DEG>
__device__ __forceinline__ CsrSite csr_eval_fixed(const uint32_t *S, const CsrBitsParams &p, int v, int e0)
{
    CsrSite r;
    r.own = S[v];
    r.d = DEG;
    uint32_t a[DEG > 0 ? DEG : 1];
#pragma unroll
    for (int k = 0; k < DEG; ++k) {
        const uint32_t nb = __ldg(p.nbr + e0 + k);
        a[k] = ~(r.own ^ S[nb & 0x7FFFFFFFu] ^ (uint32_t)((int32_t)nb >> 31));
    }
    r.u1 = r.u2 = 0u;
    if (DEG == 0) {
        r.u0 = 0u;
        r.D = 0u;  // h = 0: dE = 0 always flips
    } else if (DEG == 1) {
        r.u0 = a[0];
        r.D = ~a[0];
    } else if (DEG == 2) {
        r.u0 = a[0] ^ a[1];
        r.u1 = a[0] & a[1];
        r.D = ~(a[0] | a[1]);
    } else if (DEG == 3) {
        r.u0 = a[0] ^ a[1] ^ a[2];
        r.u1 = (a[0] & a[1]) | (a[2] & (a[0] | a[1]));  // majority
        r.D = ~r.u1;                                    // u <= 1
    } else {  // DEG == 4
        const uint32_t s3 = a[0] ^ a[1] ^ a[2], c3 = (a[0] & a[1]) | (a[2] & (a[0] | a[1]));
        r.u0 = s3 ^ a[3];
        const uint32_t c4 = s3 & a[3];
        r.u1 = c3 ^ c4;
        r.u2 = c3 & c4;
        r.D = ~(r.u1 | r.u2);  // u <= 1
    }
    return r;
}

// m ? a : b bitwise, as ONE lop3 (the compiler otherwise splits it when ~m is live)
__device__ __forceinline__ uint32_t mux(uint32_t m, uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(m), "r"(a), "r"(b));
    return r;
}

// Threshold planes 4*j4 .. 4*j4+3 of each lane: row q-1 with q = d - 2u.
__device__ __forceinline__ uint4 csr_thr4(const uint32_t *P, const CsrSite &s, uint32_t j4)
{
    auto row = [&](int k) {  // plane-row of u = k (clamped; lanes outside D ignore it)
        const int q = s.d - 2 * k;
        return *reinterpret_cast<const uint4 *>(P + (q >= 1 ? q - 1 : 0) * kRow + 4 * j4);
    };
    const uint4 r0 = row(0);
    if (s.d <= 2)
        return r0;
    const uint4 r1 = row(1);
    uint4 t;
    t.x = mux(s.u0, r1.x, r0.x);
    t.y = mux(s.u0, r1.y, r0.y);
    t.z = mux(s.u0, r1.z, r0.z);
    t.w = mux(s.u0, r1.w, r0.w);
    if (s.d <= 4)
        return t;
    const uint4 r2 = row(2), r3 = row(3);
    uint4 h;
    h.x = mux(s.u0, r3.x, r2.x);
    h.y = mux(s.u0, r3.y, r2.y);
    h.z = mux(s.u0, r3.z, r2.z);
    h.w = mux(s.u0, r3.w, r2.w);
    t.x = mux(s.u1, h.x, t.x);
    t.y = mux(s.u1, h.y, t.y);
    t.z = mux(s.u1, h.z, t.z);
    t.w = mux(s.u1, h.w, t.w);
    if (s.d <= 8)
        return t;
    const uint4 r4 = row(4), r5 = row(5), r6 = row(6), r7 = row(7);
    uint4 a, b;
    a.x = mux(s.u0, r5.x, r4.x);
    a.y = mux(s.u0, r5.y, r4.y);
    a.z = mux(s.u0, r5.z, r4.z);
    a.w = mux(s.u0, r5.w, r4.w);
    b.x = mux(s.u0, r7.x, r6.x);
    b.y = mux(s.u0, r7.y, r6.y);
    b.z = mux(s.u0, r7.z, r6.z);
    b.w = mux(s.u0, r7.w, r6.w);
    a.x = mux(s.u1, b.x, a.x);
    a.y = mux(s.u1, b.y, a.y);
    a.z = mux(s.u1, b.z, a.z);
    a.w = mux(s.u1, b.w, a.w);
    t.x = mux(s.u2, a.x, t.x);
    t.y = mux(s.u2, a.y, t.y);
    t.z = mux(s.u2, a.z, t.z);
    t.w = mux(s.u2, a.w, t.w);
    return t;
}

__device__ __forceinline__ void csr_call(uint32_t sA, uint32_t sB, uint32_t j4, const PlaneUniform &U,
                                         const RoundKeys &rk, const uint32_t *P, const CsrSite &s,
                                         uint32_t &D, uint32_t &acc)
{
    const uint4 w = philox_plane(sA, sB, j4, U, rk);
    const uint4 t = csr_thr4(P, s, j4);
    const uint32_t y0 = D & ~w.x & t.x;
    D &= ~(w.x ^ t.x);
    const uint32_t y1 = D & ~w.y & t.y;
    D &= ~(w.y ^ t.y);
    acc |= y0 | y1;
    const uint32_t y2 = D & ~w.z & t.z;
    D &= ~(w.z ^ t.z);
    const uint32_t y3 = D & ~w.w & t.w;
    D &= ~(w.w ^ t.w);
    acc |= y2 | y3;
}

}  // namespace

int32_t csr_bits_qcap(int32_t n, int32_t qmax)
{
    const size_t base = (size_t)4 * n + (size_t)(qmax > 0 ? qmax : 1) * kRow * 4 + (size_t)8 * ((n + 31) / 32);
    size_t qcap = (size_t)n < 4096 ? (size_t)n : 4096;
    const size_t budget = 200 * 1024;
    if (base + qcap * kCsrQItem > budget)
        qcap = base < budget ? (budget - base) / kCsrQItem : 0;
    return (int32_t)qcap;
}

size_t csr_bits_smem(int32_t n, int32_t qmax, int32_t words_per_copy)
{
    (void)words_per_copy;
    return (size_t)4 * n + (size_t)(qmax > 0 ? qmax : 1) * kRow * 4 + (size_t)8 * ((n + 31) / 32) +
           (size_t)csr_bits_qcap(n, qmax) * kCsrQItem;
}

__global__ void __launch_bounds__(kCsrMaxThreads, 1) k_csr_bits(const CsrBitsParams p)
{
    extern __shared__ __align__(16) uint32_t sm[];
    // per-replica bond counts, double-buffered by round parity: peers of the cluster read a
    // CTA's counts over DSMEM after a cluster barrier, and the next round writes the other
    // buffer, so no write can overtake a slow peer's read
    __shared__ int32_t Ubuf[2][32];
    __shared__ PtShared ps;
    const int n = p.n;
    const int nbw = (n + 31) / 32;
    uint32_t *S = sm;
    uint32_t *P = sm + ((n + 3) & ~3);  // [qmax][kRow], 16-byte aligned
    uint32_t *B0 = P + (p.qmax > 0 ? p.qmax : 1) * kRow;
    uint32_t *B31 = B0 + nbw;
    uint32_t *Q = B31 + nbw;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nt >> 5;
    const int qcap = p.qcap;
    const int wcap = qcap / nwarps;
    uint32_t *q_idx = Q, *q_D = Q + qcap, *q_acc = Q + 2 * qcap;
    const int wq0 = warp * wcap;
    const int wbase = tid - lane;

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

    const uint32_t *src = p.state_in + (size_t)gl * n;
    for (int i = tid; i < n; i += nt)
        S[i] = src[i];
    for (int x = tid; x < p.qmax * 64; x += nt) {
        const int q = x / 64, j = x % 64;
        P[q * kRow + j] = p.planes[((size_t)wt * p.qmax + q) * 64 + j];
    }
    if (pt)
        pt_init(ps, p.walker, c_local, K);
    __syncthreads();

    for (int round = 0; round < p.n_rounds; ++round) {
        int32_t *Ucnt = Ubuf[round & 1];
        if (tid < 32)  // zeroed here: the colour-phase barriers order it before the atomicAdds
            Ucnt[tid] = 0;
        for (int s = 0; s < p.k_ex; ++s) {
            const uint32_t t = p.t0 + (uint32_t)(round * p.k_ex + s);
            const PlaneUniform U = plane_uniform(g, t, rkr);
            if (p.planes_sched) {  // annealing: this sweep's threshold planes
                __syncthreads();
                const uint32_t *src_p =
                    p.planes_sched + (size_t)(round * p.k_ex + s) * p.words_per_copy * p.qmax * 64;
                for (int x = tid; x < p.qmax * 64; x += nt) {
                    const int q = x / 64, j = x % 64;
                    P[q * kRow + j] = src_p[((size_t)wt * p.qmax + q) * 64 + j];
                }
                __syncthreads();
            }
#pragma unroll 1
            for (int c = 0; c < p.ncol; ++c) {
                const int v1 = __ldg(p.class_off + c + 1);
                int wq = 0;  // warp-uniform
                for (int b = __ldg(p.class_off + c) + wbase; b < v1; b += nt) {
                    const int v = b + lane;
                    const bool valid = v < v1;
                    uint32_t D = 0u, acc = 0u, io = 0u, own = 0u;
                    // the warp's degree when its vertices share one (classes are degree-sorted)
                    int e0 = 0, dv = -1;
                    if (valid) {
                        e0 = __ldg(p.rp + v);
                        dv = __ldg(p.rp + v + 1) - e0;
                    }
                    const int dw = __reduce_max_sync(0xFFFFFFFFu, dv);
                    const bool uni = __all_sync(0xFFFFFFFFu, dv == dw || dv < 0) && dw <= 4;
                    CsrSite st;
                    if (valid) {
                        if (uni) {
                            switch (dw) {  // warp-uniform
                            case 0: st = csr_eval_fixed<0>(S, p, v, e0); break;
                            case 1: st = csr_eval_fixed<1>(S, p, v, e0); break;
                            case 2: st = csr_eval_fixed<2>(S, p, v, e0); break;
                            case 3: st = csr_eval_fixed<3>(S, p, v, e0); break;
                            default: st = csr_eval_fixed<4>(S, p, v, e0); break;
                            }
                        } else {
                            st = csr_eval(S, p, v);
                        }
                        own = st.own;
                        D = st.D;
                        acc = ~D;  // dE <= 0 always flips
                        if (D) {
                            io = __ldg(p.orig + v);
                            uint32_t sA, sB;
                            plane_site(io, U, rkr, sA, sB);
                            csr_call(sA, sB, 0u, U, rkr, P, st, D, acc);
                            if (D)
                                csr_call(sA, sB, 1u, U, rkr, P, st, D, acc);
                        }
                    }
                    const bool need = D != 0u;
                    const uint32_t pm = __ballot_sync(0xFFFFFFFFu, need);
                    const int slot = wq + __popc(pm & lanemask_lt());
                    wq += __popc(pm);
                    if (need && slot < wcap) {
                        const int qs = wq0 + slot;
                        q_idx[qs] = (uint32_t)v;
                        q_D[qs] = D;
                        q_acc[qs] = acc;
                    } else if (valid) {
                        if (need) {  // this warp's queue region is full: finish inline
                            uint32_t sA, sB;
                            plane_site(io, U, rkr, sA, sB);
                            uint32_t j4 = 2;
                            do {
                                csr_call(sA, sB, j4, U, rkr, P, st, D, acc);
                                ++j4;
                            } while (D && j4 < 16u);
                        }
                        S[v] = own ^ acc;
                    }
                }
                // stage 2: each warp re-evaluates its own queued vertices (their neighbours
                // cannot change inside a colour phase) right after its stage 1, no barrier in
                // between, and finishes their comparisons from plane 8 on
                const int nown = min(wq, wcap);
                for (int qb = 0; qb < nown; qb += 32) {
                    const int q = qb + lane;
                    if (q >= nown)
                        continue;
                    const int qs = wq0 + q;
                    const int v = (int)q_idx[qs];
                    uint32_t D = q_D[qs], acc = q_acc[qs];
                    const CsrSite st = csr_eval(S, p, v);
                    uint32_t sA, sB;
                    plane_site(__ldg(p.orig + v), U, rkr, sA, sB);
                    uint32_t j4 = 2;
                    do {
                        csr_call(sA, sB, j4, U, rkr, P, st, D, acc);
                        ++j4;
                    } while (D && j4 < 16u);
                    S[v] = st.own ^ acc;
                }
                __syncthreads();
            }
        }

        // energy: each edge once, counted from its endpoint in the higher colour class
        {
            uint32_t cnt[kCsrCnt];
#pragma unroll
            for (int l = 0; l < kCsrCnt; ++l)
                cnt[l] = 0u;
            for (int c = 1; c < p.ncol; ++c) {
                const int lo_c = __ldg(p.class_off + c), v1 = __ldg(p.class_off + c + 1);
                for (int v = lo_c + tid; v < v1; v += nt) {
                    const uint32_t own = S[v];
                    const int e0 = __ldg(p.rp + v), e1 = __ldg(p.rp + v + 1);
                    for (int e = e0; e < e1; ++e) {
                        const uint32_t nb = __ldg(p.nbr + e);
                        const uint32_t j = nb & 0x7FFFFFFFu;
                        if ((int)j >= lo_c)
                            continue;
                        const uint32_t jm = (uint32_t)((int32_t)nb >> 31);
                        vadd(cnt, ~(own ^ S[j] ^ jm));
                    }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                vsum_xor(cnt, off);
            int32_t acc = 0;
#pragma unroll
            for (int l = 0; l < kCsrCnt; ++l)
                acc += (int32_t)((cnt[l] >> lane) & 1u) << l;
            if (p.k_ex == 0)  // no colour phase (hence no barrier) since the zeroing
                __syncthreads();
            atomicAdd(&Ucnt[lane], acc);
            if (!pt)  // pt_step opens with a cluster barrier
                __syncthreads();
        }
        if (!pt)
            continue;
        auto snap = [&](int bit) {
            int8_t *dst = p.snap + (size_t)c_local * n;
            for (int v = tid; v < n; v += nt)
                dst[__ldg(p.orig + v)] = ((S[v] >> bit) & 1u) ? -1 : 1;
        };
        pt_step(ps, Ucnt, p.m, S, n, B0, B31, KW, wt, c_global,
                p.t0 + (uint32_t)((round + 1) * p.k_ex), p.e0 + (uint32_t)round, p.Tx, p.Tx_off,
                p.Tx_len, p.rk, snap);
    }

    int32_t *Ucnt = Ubuf[(p.n_rounds - 1) & 1];  // the last round's counts
    pt_finish(ps, pt, p.n_rounds, Ucnt, p.m, p.E_out, p.walker, p.copy_best, gl, wt, c_local, K);
    uint32_t *dst = p.state_out + (size_t)gl * n;
    for (int i = tid; i < n; i += nt)
        dst[i] = S[i];
    if (pt)
        cg::this_cluster().sync();
}

cudaError_t launch_csr_bits(const CsrBitsParams &p, int32_t G, int32_t threads, size_t smem,
                            cudaStream_t st)
{
    cudaError_t e = cudaFuncSetAttribute(k_csr_bits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    return cudaLaunchKernelEx(&cfg, k_csr_bits, p);
}

}  // namespace ising

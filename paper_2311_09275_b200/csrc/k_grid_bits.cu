// k_grid_bits.cu -- multi-spin-coded Metropolis sweeps on +-1 tori (sm_100a).
//
// Hot path rows a3-a6 of SURVEY.md §8(a) for the grid workloads (C2, C4; Gset
// spin-glass tori, Table I).  One CTA owns one 32-replica word
// group g (32 consecutive global slots = 32 temperatures of one copy) for all
// n sites and keeps it resident in shared memory for a whole launch:
// load -> n_rounds x {k_ex sweeps x {colour 0, colour 1} -> energy of the 32
// replicas -> [fused PT step of the copy's cluster]} -> store.  The colour-phase
// update and the bond count are grid_core.cuh (shared with k_grid_sched, the
// persistent variant for handles with more word groups than SMs).
// Philox rounds 0-1 are partially hoisted: the parts that depend only on the
// CTA's group g, the sweep t or the site i are computed once, not per call.
#include "grid_core.cuh"

namespace ising {

using namespace bits;
using grid::kGridQItem;

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
    const int tid = threadIdx.x, nt = blockDim.x;
    const int qcap = p.qcap;
    const int nbw = (n + 31) / 32;
    uint32_t *B0 = reinterpret_cast<uint32_t *>(Q4 + qcap);  // boundary bit planes (PT mode)
    uint32_t *B31 = B0 + nbw;

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
    const grid::Ctx X = grid::make_ctx(G, n, qcap, S, JB, Q4, SPILL);

    // ---- load: original order -> colour-separated order
    const uint32_t *src = p.state_in + (size_t)gl * n;
    for (int i = tid; i < n; i += nt)
        S[grid::colsep(G, i)] = src[i];
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
            for (int c = 0; c < 2; ++c)
                grid::colour_phase<SPILL>(X, c, U, rkr, P);
        }

        // ---- energy of the 32 replicas: E = 2U - 2n
        {
            const int32_t acc = grid::unsat_counts(X, S, JB);
            if (p.k_ex == 0)  // no colour phase (hence no barrier) since the zeroing
                __syncthreads();
            atomicAdd(&Ucnt[X.lane], acc);
            if (!pt)  // pt_step opens with a cluster barrier
                __syncthreads();
        }
        if (!pt)
            continue;

        // ---- fused PT step for this copy (a7/a8): same result as ising_exchange
        auto snap = [&](int bit) {
            int8_t *dst = p.snap + (size_t)c_local * n;
            for (int i = tid; i < n; i += nt)
                dst[i] = ((S[grid::colsep(G, i)] >> bit) & 1u) ? -1 : 1;
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
    for (int i = tid; i < n; i += nt)
        dst[i] = S[grid::colsep(G, i)];
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

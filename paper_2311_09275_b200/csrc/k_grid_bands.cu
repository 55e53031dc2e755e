// k_grid_bands.cu -- the torus PT kernel with each word group's rows split over a CTA pair
// (sm_100a).  Used when a handle holds at most half as many word groups as the GPU has SMs
// (one rank's share of C4 at 8 GPUs: 64 groups), so twice as many SMs work.
//
// Band b of a group owns rows [y0, y1) = [b Ly/2, (b+1) Ly/2) and keeps a full copy of the
// group's lattice in shared memory.  The colour phase and the bond count are grid_core.cuh's
// (the same code as k_grid_bits / k_grid_sched) restricted to the band's rows; after every
// colour phase the band pushes its edge rows of the class just updated into the other band's
// copy through DSMEM and the cluster synchronises, so the neighbour rows a phase reads are
// current.  Energies are the sum of the bands' bond counts; the fused PT step runs on clusters
// of (K/32) x 2 CTAs (bits_core.cuh), or -- when those do not all fit at once -- on K/32
// clusters of 2 that meet at global-memory copy barriers in one cooperative launch.
//
// Hot path rows a3-a6 of SURVEY.md §8(a) for the grid workloads (C4's 8-GPU share; Gset
// spin-glass tori, Table I).
#include "grid_core.cuh"

namespace ising {

using namespace bits;


using grid::kGridQItem;

// Copy-wide barrier over the copy's clusters through a global counter (the launch is
// cooperative, so every CTA of the grid is resident and the spin cannot deadlock).
__device__ __forceinline__ void copy_barrier(uint32_t *bar, uint32_t target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        uint32_t v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// PT step of a copy spread over K/32 clusters (one per word type, each the CTA pair of the
// two bands): as bits::pt_step, with the word types' energies and boundary bit planes passed
// through global memory (double-buffered by round parity) between copy barriers.
template <class Snap>
__device__ void pt_step_xc(PtShared &ps, const int32_t *Ucnt, int64_t m_edges, uint32_t *S, int n,
                           uint32_t *B0, uint32_t *B31, int KW, int wt, int band, uint32_t c_global,
                           uint32_t t_now, uint32_t e_now, int round, const GridBitsParams &p, int c_local,
                           uint32_t &bar_target, Snap snap)
{
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int K = 32 * KW;
    const int nbw = (n + 31) / 32;
    const int par_r = round & 1;
    int64_t *Eg = p.xc_E + ((size_t)c_local * 2 + par_r) * K;
    uint32_t *Bg = p.xc_B + ((size_t)c_local * 2 + par_r) * (size_t)KW * 4 * nbw;
    uint32_t *bar = p.xc_bar + c_local;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // both bands' counts complete
    if (band == 0 && tid < 32) {
        const int32_t u = Ucnt[tid] + cl.map_shared_rank(Ucnt, cl.block_rank() + 1u)[tid];
        Eg[32 * wt + tid] = 2 * (int64_t)u - m_edges;
    }
    bar_target += 2u * (uint32_t)KW;
    copy_barrier(bar, bar_target);
    for (int k = tid; k < K; k += nt)
        ps.Ecopy[k] = __ldcg(Eg + k);
    for (int q = tid; q < KW; q += nt)
        ps.Mswap[q] = 0u;
    __syncthreads();
    if (warp == 0) {  // best-so-far of the copy: argmin, ties -> lowest slot
        int64_t bE = INT64_MAX;
        int bk = -1;
        for (int k = lane; k < K; k += 32)
            if (bk < 0 || ps.Ecopy[k] < bE) {
                bE = ps.Ecopy[k];
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
            ps.improve = bE < ps.bestE;
            ps.kmin = bk;
            if (bE < ps.bestE) {
                ps.bestE = bE;
                ps.bestSlot = (int64_t)c_global * K + bk;
                ps.bestSweep = t_now;
            }
        }
    }
    __syncthreads();
    if (ps.improve && (ps.kmin >> 5) == wt)
        snap(ps.kmin & 31);
    const int par = (int)(e_now & 1u);
    const int npairs = (K - par) / 2;
    for (int pi = tid; pi < npairs; pi += nt) {
        const int k = par + 2 * pi;
        const int64_t d = ps.Ecopy[k + 1] - ps.Ecopy[k];
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
            atomicOr(&ps.Mswap[k >> 5], 1u << (k & 31));
            const int64_t te = ps.Ecopy[k];
            ps.Ecopy[k] = ps.Ecopy[k + 1];
            ps.Ecopy[k + 1] = te;
            const int64_t tw = ps.Wcopy[k];
            ps.Wcopy[k] = ps.Wcopy[k + 1];
            ps.Wcopy[k + 1] = tw;
        }
    }
    __syncthreads();
    const uint32_t Min = ps.Mswap[wt] & 0x7FFFFFFFu;
    const bool cross_lo = wt > 0 && ((ps.Mswap[wt - 1] >> 31) & 1u);
    const bool cross_hi = wt + 1 < KW && ((ps.Mswap[wt] >> 31) & 1u);
    bool any_cross = false;
    for (int q = 0; q + 1 < KW; ++q)
        any_cross |= (ps.Mswap[q] >> 31) & 1u;
    if (any_cross) {  // uniform over the copy
        uint32_t *mine = Bg + ((size_t)wt * 2 + band) * 2 * nbw;
        for (int b = warp * 32; b < nbw * 32; b += nt) {
            const int l = b + lane;
            const uint32_t w = l < n ? S[l] : 0u;
            const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, w & 1u);
            const uint32_t b31 = __ballot_sync(0xFFFFFFFFu, w >> 31);
            if (lane == 0) {
                mine[b >> 5] = b0;
                mine[nbw + (b >> 5)] = b31;
            }
        }
        bar_target += 2u * (uint32_t)KW;
        copy_barrier(bar, bar_target);
        const uint32_t *nB31 = Bg + ((size_t)(wt - 1) * 2 + band) * 2 * nbw + nbw;  // used iff cross_lo
        const uint32_t *nB0 = Bg + ((size_t)(wt + 1) * 2 + band) * 2 * nbw;         // used iff cross_hi
        for (int l = tid; l < n; l += nt) {
            uint32_t w = S[l];
            const uint32_t tt = (w ^ (w >> 1)) & Min;
            w ^= tt ^ (tt << 1);
            if (cross_lo)
                w = (w & ~1u) | ((__ldcg(nB31 + (l >> 5)) >> (l & 31)) & 1u);
            if (cross_hi)
                w = (w & 0x7FFFFFFFu) | (((__ldcg(nB0 + (l >> 5)) >> (l & 31)) & 1u) << 31);
            S[l] = w;
        }
    } else if (Min) {
        for (int l = tid; l < n; l += nt) {
            const uint32_t w = S[l];
            const uint32_t tt = (w ^ (w >> 1)) & Min;
            S[l] = w ^ tt ^ (tt << 1);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kGridMaxThreads, 1) k_grid_bands(const GridBitsParams p)
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
    // band split: NB CTAs (consecutive, one cluster) share a word group; CTA `band` updates
    // rows [y0, y1) of its full local lattice copy, whose halo rows (the neighbouring bands'
    // edge rows) the neighbours push into it through DSMEM after every colour phase
    constexpr int NB = 2;
    const int band = (int)(blockIdx.x % (unsigned)NB);
    const int y0 = band * (p.Ly / NB), y1 = y0 + p.Ly / NB;
    const int gl = (int)(blockIdx.x / (unsigned)NB);
    const uint32_t g = p.g0 + (uint32_t)gl;
    const int KW = p.words_per_copy;
    const int wt = (int)(g % (uint32_t)KW);
    const int K = 32 * KW;
    const bool pt = p.pt != 0;
    const int c_local = gl / KW;
    const uint32_t c_global = g / (uint32_t)KW;

    // the colour phase and the bond count of grid_core.cuh over this band's rows [y0, y1)
    const grid::Ctx X = grid::make_ctx(G, n, qcap, S, JB, Q4, false, y0, y1, /*limit_stage2=*/false);

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

    uint32_t bar_target = 0;  // xc mode: the copy barrier's count after the next arrival
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
                // the band's edge rows of class c go to the other band's copy as soon as the
                // warp that owns them has finished its phase (its stage-2 queue holds only its
                // own sites), so one cluster barrier ends the phase
                grid::colour_phase<false, false>(X, c, U, rkr, P);
                cg::cluster_group cl = cg::this_cluster();
                if (X.T.active) {
                    const unsigned rbase = cl.block_rank() - (unsigned)band;
                    const int nrows = y1 - y0;
                    const int off0 = c * G.half + X.T.m;
                    if (X.T.ty == 0) {  // row y0 -> the band above
                        const int off = off0 + y0 * G.hx;
                        cl.map_shared_rank(S, rbase + (unsigned)((band + NB - 1) % NB))[off] = S[off];
                    }
                    if (X.T.ty == (nrows - 1) % X.rpp) {  // row y1 - 1 -> the band below
                        const int off = off0 + (y1 - 1) * G.hx;
                        cl.map_shared_rank(S, rbase + (unsigned)((band + 1) % NB))[off] = S[off];
                    }
                }
                cl.sync();
            }
        }

        // ---- energy of this band's rows (the bands' counts add up to the group's)
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
        auto snap = [&](int bit) {  // this band's rows of the configuration
            int8_t *dst = p.snap + (size_t)c_local * n;
            for (int i = y0 * p.Lx + tid; i < y1 * p.Lx; i += nt) {
                const int y = i / p.Lx, x = i - y * p.Lx;
                dst[i] = ((S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)] >> bit) & 1u) ? -1 : 1;
            }
        };
        if (p.xc)
            pt_step_xc(ps, Ucnt, 2 * (int64_t)n, S, n, B0, B31, KW, wt, band, c_global,
                       p.t0 + (uint32_t)((round + 1) * p.k_ex), p.e0 + (uint32_t)round, round, p, c_local,
                       bar_target, snap);
        else
            pt_step<NB>(ps, Ucnt, 2 * (int64_t)n, S, n, B0, B31, KW, wt, c_global,
                        p.t0 + (uint32_t)((round + 1) * p.k_ex), p.e0 + (uint32_t)round, p.Tx, p.Tx_off,
                        p.Tx_len, p.rk, snap, band);
    }

    // ---- outputs
    int32_t *Ucnt = Ubuf[(p.n_rounds - 1) & 1];  // the last round's counts
    if (NB > 1 && !(pt && p.n_rounds > 0)) {  // the group's counts: sum over its bands
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        int32_t u = 0;
        if (tid < 32)
            for (int b = 0; b < NB; ++b)
                u += cl.map_shared_rank(Ucnt, cl.block_rank() - (unsigned)band + (unsigned)b)[tid];
        cl.sync();  // every band has read every band's counts
        if (tid < 32)
            Ucnt[tid] = u;
        __syncthreads();
    }
    pt_finish<NB>(ps, pt, p.n_rounds, Ucnt, 2 * (int64_t)n, p.E_out, p.walker, p.copy_best, gl, wt,
                  c_local, K, band);
    uint32_t *dst = p.state_out + (size_t)gl * n;
    for (int i = y0 * p.Lx + tid; i < y1 * p.Lx; i += nt) {
        const int y = i / p.Lx, x = i - y * p.Lx;
        dst[i] = S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)];
    }
    if (pt || NB > 1)
        cg::this_cluster().sync();  // no CTA exits while a peer may still read its shared memory
}

// Co-resident clusters of `cluster` CTAs of this kernel (GPC sizes are uneven: with one CTA
// per SM, 15 clusters of 8 fit on a B200 but 33 of 4 and 74 of 2).
int32_t grid_bands_max_clusters(int32_t cluster, int32_t threads, size_t smem)
{
    if (cudaFuncSetAttribute(k_grid_bands, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cluster);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_grid_bands, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

cudaError_t launch_grid_bands(const GridBitsParams &p, int32_t G, int32_t threads, size_t smem,
                              cudaStream_t st)
{
    cudaError_t e = cudaFuncSetAttribute(k_grid_bands, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(G * 2));
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (p.pt && !p.xc ? (unsigned)p.words_per_copy : 1u) * 2u;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;  // xc: copy barriers need every CTA resident
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pt && p.xc ? 2 : 1;
    if (p.pt && p.xc) {
        e = cudaMemsetAsync(p.xc_bar, 0, (size_t)(G / p.words_per_copy) * sizeof(uint32_t), st);
        if (e != cudaSuccess)
            return e;
    }
    return cudaLaunchKernelEx(&cfg, k_grid_bands, p);
}

}  // namespace ising

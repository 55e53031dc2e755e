// k_grid_sched.cu -- persistent, ticket-scheduled variant of the fused torus PT launch
// (sm_100a), for handles with more 32-replica word groups than SMs (C4 on one or two GPUs:
// 512 / 256 groups on 148 SMs).  DESIGN.md §5.2b.
//
// Why: the fused launch of k_grid_bits keeps each word group resident in one CTA for the
// whole schedule and runs each copy as a cluster of K/32 CTAs.  With 512 groups in clusters
// of 4, only 33 clusters (132 CTAs) fit on a B200 at once (GPC sizes), so 128 copies take 4
// waves on 132 SMs: 86% of the GPU's SM-time.  Here one CTA per SM (a cooperative launch)
// loops over TASKS = (word group, round): one TMA bulk copy brings the group's state (kept
// colour-separated between rounds in a global scratch; the whole C4b state is 41 MB, L2-
// resident) straight into the lattice array, the round's k_ex sweeps and the bond count run in
// shared memory exactly as in k_grid_bits (grid_core.cuh), one bulk copy stores the state back
// and the 32 energies are published.  Tasks are handed out by one atomic ticket in round-major
// order (the next ticket is fetched while the current task runs), so every SM stays busy until
// the last round; the state round trip (~160 KB of L2 traffic per task of ~0.3 ms) costs ~1%.
//
// The PT step of a copy (best-so-far check, exchange decisions, walker and energy swaps;
// same rule and RNG counters as bits::pt_step / k_exchange) is run by the
// CTA that completes the copy's LAST task of the round (an atomic counter per copy).  It does
// not touch the configurations: it publishes the copy's swap mask, and each group applies it
// when it loads its state for the next round -- pairs inside a word by a delta swap, the pair
// that crosses two words from the neighbouring group's boundary bit plane (bit 0 / bit 31 of
// every site, in colour-separated order) saved at the end of the round (double-buffered by
// round parity).  After the
// last round the PT step applies the swaps to the stored states itself.  A task of round r
// waits (acquire spin) until its copy's exchange r-1 is published; tickets are handed out in
// order and every CTA is resident, so a wait is always on an earlier ticket that a running
// CTA holds: no deadlock, and in practice no waiting (the previous round's tasks of a copy
// were handed out one round of tickets, >= 1.7 task durations, earlier).
//
// Results are bit-identical to k_grid_bits' fused launch (tests: test_sched_*).
#include "grid_core.cuh"

namespace ising {

using namespace bits;

namespace {

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *a)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(uint32_t *a, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA bulk copy global -> shared (bytes % 16 == 0, both 16-byte aligned), completing on mbar
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase)
{
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(mbar), "r"(phase) : "memory");
}

// TMA bulk copy shared -> global, waited for completion and ordered before later generic
// accesses (fence.proxy.async) -- the CTA's release of the copy counter follows it
__device__ __forceinline__ void bulk_store_wait(void *dst, uint32_t src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// The PT step of copy c_local after round `round` (all its K/32 groups stored).  Run by
// every thread of the CTA that completed the copy's last task of the round.
__device__ void copy_pt_step(PtShared &ps, const GridBitsParams &p, int round, int c_local)
{
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int KW = p.words_per_copy, K = 32 * KW, n = p.n;
    const uint32_t c_global = p.g0 / (uint32_t)KW + (uint32_t)c_local;
    const uint32_t t_now = p.t0 + (uint32_t)((round + 1) * p.k_ex), e_now = p.e0 + (uint32_t)round;
    const int64_t *Eg = p.xs_E + (size_t)c_local * K;
    int64_t *Wg = p.walker + (size_t)c_local * K;
    int64_t *cb = p.copy_best + 3 * (size_t)c_local;
    for (int k = tid; k < K; k += nt) {  // one round trip: energies, walkers, the copy's best
        ps.Ecopy[k] = __ldcg(Eg + k);
        ps.Wcopy[k] = __ldcg(Wg + k);
    }
    if (tid == 0) {
        ps.bestE = __ldcg(cb);
        ps.bestSlot = __ldcg(cb + 1);
    }
    for (int q = tid; q < KW; q += nt)
        ps.Mswap[q] = 0u;
    __syncthreads();
    if (warp == 0) {  // best-so-far of the copy: argmin, ties -> lowest slot; strict improvement
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
            const bool imp = ps.bestSlot < 0 || bE < ps.bestE;
            ps.improve = imp;
            ps.kmin = bk;
            if (imp) {
                cb[0] = bE;
                cb[1] = (int64_t)c_global * K + bk;
                cb[2] = t_now;
            }
        }
    }
    __syncthreads();
    if (ps.improve) {  // snapshot of the configuration (stored this round, before the swap)
        const int gk = c_local * KW + (ps.kmin >> 5), bit = ps.kmin & 31;
        int8_t *dst = p.snap + (size_t)c_local * n;
        const bool last = round + 1 == p.n_rounds;  // the last round stores original order
        const uint32_t *src = (last ? p.state_out : p.xs_S) + (size_t)gk * n;
        for (int y = warp; y < p.Ly; y += nt / 32)
            for (int x = lane; x < p.Lx; x += 32) {
                const int i = y * p.Lx + x;
                const int l = last ? i : ((x + y) & 1) * p.half + y * p.hx + (x >> 1);
                dst[i] = ((__ldcg(src + l) >> bit) & 1u) ? -1 : 1;
            }
    }
    const int par = (int)(e_now & 1u);
    const int npairs = (K - par) / 2;
    for (int pi = tid; pi < npairs; pi += nt) {
        const int k = par + 2 * pi;
        const int64_t d = ps.Ecopy[k + 1] - ps.Ecopy[k];
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
    for (int k = tid; k < K; k += nt) {
        p.E_out[(size_t)c_local * K + k] = ps.Ecopy[k];
        Wg[k] = ps.Wcopy[k];
    }
    for (int q = tid; q < KW; q += nt)
        p.xs_M[(size_t)c_local * KW + q] = ps.Mswap[q];
    if (round + 1 == p.n_rounds) {  // no later load applies the swaps: apply them to the states
        bool any = false;
        for (int q = 0; q < KW; ++q)
            any |= ps.Mswap[q] != 0u;
        if (any) {
            uint32_t *base = p.state_out + (size_t)c_local * KW * n;
            for (int i = tid; i < n; i += nt) {
                uint32_t prev = 0u, cur = __ldcg(base + i);
                for (int q = 0; q < KW; ++q) {
                    const uint32_t next = q + 1 < KW ? __ldcg(base + (size_t)(q + 1) * n + i) : 0u;
                    const uint32_t M = ps.Mswap[q];
                    uint32_t w = cur;
                    const uint32_t tt = (w ^ (w >> 1)) & M & 0x7FFFFFFFu;
                    w ^= tt ^ (tt << 1);
                    if (q > 0 && ((ps.Mswap[q - 1] >> 31) & 1u))
                        w = (w & ~1u) | (prev >> 31);
                    if (q + 1 < KW && ((M >> 31) & 1u))
                        w = (w & 0x7FFFFFFFu) | (next << 31);
                    base[(size_t)q * n + i] = w;
                    prev = cur;
                    cur = next;
                }
            }
        }
    }
}

}  // namespace

template <bool SPILL>
__global__ void __launch_bounds__(kGridMaxThreads, 1) k_grid_sched(const GridBitsParams p)
{
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ int32_t Ucnt[32];
    __shared__ PtShared ps;
    __shared__ int32_t s_task, s_last;
    __shared__ __align__(8) uint64_t mbar;
    const int n = p.n;
    const GridGeom G{p.Lx, p.Ly, p.hx, p.half, p.ymagic};
    uint32_t *S = sm;
    uint8_t *JB = reinterpret_cast<uint8_t *>(sm + n);
    uint32_t *P = reinterpret_cast<uint32_t *>(JB + ((n + 15) & ~15));  // P[0..63] dE=4, P[64..127] dE=8
    uint4 *Q4 = reinterpret_cast<uint4 *>(P + 128);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int KW = p.words_per_copy;
    const int Gl = p.n_groups;
    const int C_local = Gl / KW;
    const int32_t ntask = Gl * p.n_rounds;  // host guarantees < 2^31
    const int nbw = (n + 31) / 32;
    const uint32_t bytes = 4u * (uint32_t)n;  // n % 4 == 0 (even tori): whole 16-byte units
    uint32_t *ticket = p.xs_ctl, *cnt = p.xs_ctl + 1, *ready = p.xs_ctl + 1 + C_local;
    // plain sweeps (p.pt == 0): tasks (group, chunk of k_ex sweeps) wait only for the group's
    // previous chunk, published per group after the copy counters
    uint32_t *gready = p.xs_ctl + 1 + 2 * C_local;
    const bool pt = p.pt != 0;

    RoundKeys rkr;
#pragma unroll
    for (int r = 0; r < 20; ++r)
        rkr.k[r] = p.rk.k[r];
    const grid::Ctx X = grid::make_ctx(G, n, p.qcap, S, JB, Q4, SPILL);
    for (int l = tid; l < n; l += nt)  // the couplings are the same for every task
        JB[l] = p.jbyte[l];
    const uint32_t mb = smem_u32(&mbar), sS = smem_u32(S);
    uint32_t phase = 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_task = (int32_t)atomicAdd(ticket, 1u);
    }
    __syncthreads();

    for (;;) {
        const int32_t task = s_task;
        __syncthreads();  // every thread has read s_task before thread 0 overwrites it
        if (task >= ntask)
            break;
        uint32_t next = 0;  // the next ticket, fetched while this task runs (thread 0)
        if (tid == 0)
            next = atomicAdd(ticket, 1u);
        const int round = task / Gl, gl = task - round * Gl;
        const bool last = round + 1 == p.n_rounds;
        const uint32_t g = p.g0 + (uint32_t)gl;
        const int wt = (int)(g % (uint32_t)KW);
        const int c_local = gl / KW;
        uint32_t *scratch = p.xs_S + (size_t)gl * n;  // colour-separated state between rounds
        if (round == 0) {
            // ---- first round: the launch's input, original order -> colour-separated
            const uint32_t *src = p.state_in + (size_t)gl * n;
            for (int y = X.warp; y < G.Ly; y += X.nwarps)
                for (int x = X.lane; x < G.Lx; x += 32)
                    S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)] = __ldcg(src + y * G.Lx + x);
        } else {
            // ---- the copy's exchange of the previous round must be published; then one TMA
            // bulk copy of the stored state straight into S and the pending swaps applied in place
            if (tid == 0) {
                const uint32_t *rw = pt ? ready + c_local : gready + gl;
                while (ld_acquire(rw) < (uint32_t)round)
                    __nanosleep(256);
                asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired data -> async proxy
                bulk_load(sS, scratch, bytes, mb);
            }
            // the barrier's completion follows thread 0's acquire of `ready` (its arrive releases
            // at CTA scope, the wait acquires): the copy's swap mask and the neighbours' boundary
            // planes are read only after it
            mbar_wait(mb, phase);
            phase ^= 1u;
        }
        if (pt && round > 0) {
            const uint32_t *M = p.xs_M + (size_t)c_local * KW;
            const uint32_t Mw = __ldcg(M + wt);
            const uint32_t Min = Mw & 0x7FFFFFFFu;
            const bool clo = wt > 0 && ((__ldcg(M + wt - 1) >> 31) & 1u);
            const bool chi = wt + 1 < KW && ((Mw >> 31) & 1u);
            const uint32_t *Bp = p.xs_B + (size_t)((round - 1) & 1) * Gl * 2 * nbw;
            const uint32_t *nB31 = Bp + ((size_t)(gl - 1) * 2 + 1) * nbw;  // used only if clo (wt > 0)
            const uint32_t *nB0 = Bp + (size_t)(gl + 1) * 2 * nbw;         // used only if chi (wt < KW - 1)
            if (Min | clo | chi) {
                for (int l = tid; l < n; l += nt) {
                    uint32_t w = S[l];
                    const uint32_t tt = (w ^ (w >> 1)) & Min;
                    w ^= tt ^ (tt << 1);
                    if (clo)
                        w = (w & ~1u) | ((__ldcg(nB31 + (l >> 5)) >> (l & 31)) & 1u);
                    if (chi)
                        w = (w & 0x7FFFFFFFu) | (((__ldcg(nB0 + (l >> 5)) >> (l & 31)) & 1u) << 31);
                    S[l] = w;
                }
            }
        }
        for (int j = tid; j < 128; j += nt)
            P[j] = __ldg(p.planes + wt * 128 + j);
        if (tid < 32)
            Ucnt[tid] = 0;
        __syncthreads();
        // ---- the round's k_ex sweeps (grid_core.cuh, as k_grid_bits)
        for (int s = 0; s < p.k_ex; ++s) {
            const uint32_t t = p.t0 + (uint32_t)(round * p.k_ex + s);
            const PlaneUniform U = plane_uniform(g, t, rkr);
#pragma unroll 1
            for (int c = 0; c < 2; ++c)
                grid::colour_phase<SPILL>(X, c, U, rkr, P);
        }
        if (pt || last)  // plain sweeps: the energies of the call's last sweep only
            atomicAdd(&Ucnt[X.lane], grid::unsat_counts(X, S, JB));
        if (last) {
            // ---- the launch's output, original order (the PT step applies the last swaps there)
            uint32_t *dst = p.state_out + (size_t)gl * n;
            for (int y = X.warp; y < G.Ly; y += X.nwarps)
                for (int x = X.lane; x < G.Lx; x += 32)
                    dst[y * G.Lx + x] = S[((x + y) & 1) * G.half + y * G.hx + (x >> 1)];
        } else if (pt) {
            // ---- this round's boundary bit planes (parity round & 1), then one bulk store of S
            uint32_t *Bo = p.xs_B + ((size_t)(round & 1) * Gl + gl) * 2 * nbw;
            for (int b = X.warp * 32; b < nbw * 32; b += nt) {
                const int l = b + X.lane;
                const uint32_t w = l < n ? S[l] : 0u;
                const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, w & 1u);
                const uint32_t b31 = __ballot_sync(0xFFFFFFFFu, w >> 31);
                if (X.lane == 0) {
                    Bo[b >> 5] = b0;
                    Bo[nbw + (b >> 5)] = b31;
                }
            }
        }
        // every thread's generic accesses of S are ordered before the async proxy's (the bulk
        // store below reads S, the next task's bulk load overwrites it)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();  // Ucnt complete; S final
        if (pt && tid < 32)
            p.xs_E[(size_t)gl * 32 + tid] = 2 * (int64_t)Ucnt[tid] - 2 * (int64_t)n;
        if (!pt && last && tid < 32)
            p.E_out[(size_t)gl * 32 + tid] = 2 * (int64_t)Ucnt[tid] - 2 * (int64_t)n;
        if (tid == 0 && !last)
            bulk_store_wait(scratch, sS, bytes);
        __threadfence();
        __syncthreads();
        if (!pt) {  // plain sweeps: publish the group's chunk, take the next ticket
            if (tid == 0) {
                st_release(gready + gl, (uint32_t)(round + 1));
                s_task = (int32_t)next;
            }
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            const uint32_t done = atomicAdd(cnt + c_local, 1u) + 1u;
            s_last = done == (uint32_t)KW * (uint32_t)(round + 1);
            s_task = (int32_t)next;
        }
        __syncthreads();
        if (s_last) {  // this CTA completed the copy's round: its PT step
            __threadfence();
            copy_pt_step(ps, p, round, c_local);
            __threadfence();
            __syncthreads();
            if (tid == 0)
                st_release(ready + c_local, (uint32_t)(round + 1));
        }
    }
}

// Resident CTAs of the persistent launch (one per SM at this shared-memory size), 0 if the
// kernel cannot be launched.
int32_t grid_sched_ctas(int32_t threads, size_t smem, bool spill)
{
    auto kern = spill ? k_grid_sched<true> : k_grid_sched<false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0, dev = 0, nsm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess ||
        cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm * nsm;
}

cudaError_t launch_grid_sched(const GridBitsParams &p, int32_t ctas, int32_t threads, size_t smem,
                              cudaStream_t st)
{
    const int hx = p.hx, rpp = grid_rows_per_pass(threads, hx);
    const int full = p.Ly / rpp, left = (p.Ly - full * rpp) * hx;
    const int nidle = (threads / 32 - (rpp * hx + 31) / 32) * 32;
    const bool spill = left > 0 && nidle > 0 && (left + nidle - 1) / nidle <= full;
    auto kern = spill ? k_grid_sched<true> : k_grid_sched<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    // control words: ticket, per-copy task counters and published exchange rounds, per-group
    // published chunks (plain sweeps)
    e = cudaMemsetAsync(p.xs_ctl, 0,
                        sizeof(uint32_t) * (1 + 2 * (size_t)(p.n_groups / p.words_per_copy) + (size_t)p.n_groups), st);
    if (e != cudaSuccess)
        return e;
    // per-copy best of this launch: slot -1 = none yet (all bytes 0xFF); plain sweeps keep none
    if (p.pt) {
        e = cudaMemsetAsync(p.copy_best, 0xFF, sizeof(int64_t) * 3 * (size_t)(p.n_groups / p.words_per_copy), st);
        if (e != cudaSuccess)
            return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the spin waits cannot deadlock
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace ising

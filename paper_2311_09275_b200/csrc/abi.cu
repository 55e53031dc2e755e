// abi.cu -- host runtime and C ABI of libising.so (see include/ising.h).
//
// Row a1 of SURVEY.md §8(a) (create / preprocess: validation, colouring,
// colour reordering, threshold and plane tables, upload) plus the orchestration
// of rows a2-a9 on the handle's CUDA stream.  Host tables follow the contract
// of DESIGN.md §3.4: T = min(floor(exp(x) * 2^64), 2^64-1) with
// x = -(beta_k * dE) for Metropolis and x = (beta_{k+1} - beta_k) * d for the
// exchange.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>
#include <queue>
#include <functional>

#include "internal.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys / ncu --nvtx (SURVEY.md §5 tracing)

using namespace ising;

namespace {

// NVTX range for the lifetime of a scope (no-op unless a tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_err;

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *what)
{
    return fail(e == cudaErrorMemoryAllocation ? ISING_E_OOM : ISING_E_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                  \
    do {                                          \
        cudaError_t _e = (expr);                  \
        if (_e != cudaSuccess)                    \
            return cuda_fail(_e, #expr);          \
    } while (0)

uint64_t p64(double x)
{
    const double p = std::exp(x);
    const double v = std::ldexp(p, 64);
    if (v >= 18446744073709551616.0)
        return std::numeric_limits<uint64_t>::max();
    return (uint64_t)v;
}

uint64_t metropolis_threshold(double beta, int64_t dE) { return p64(-(beta * (double)dE)); }

// FNV-1a over raw bytes: checkpoint fingerprint of what a resumed handle must share.
uint64_t fnv1a(uint64_t hsh, const void *p, size_t bytes)
{
    const unsigned char *b = (const unsigned char *)p;
    for (size_t i = 0; i < bytes; ++i) {
        hsh ^= b[i];
        hsh *= 0x100000001b3ull;
    }
    return hsh;
}
constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;

uint64_t exchange_threshold(double beta_lo, double beta_hi, int64_t d)
{
    return p64((beta_hi - beta_lo) * (double)d);
}

}  // namespace

struct ising_handle {
    int32_t kernel = 0;
    int32_t n = 0, Lx = 0, Ly = 0, ncol = 0;
    int64_t m = 0;
    int32_t wtype = 0, layout = 0, rng = 0;
    int64_t W_int = 0;
    double W_f = 0.0;
    uint64_t seed = 0;
    RoundKeys rk{};
    int32_t K = 0, C = 0, c0 = 0, c1 = 0, C_local = 0, G = 0, wpc = 0;
    int64_t R = 0, slot0 = 0;
    uint32_t g0 = 0;
    std::vector<double> betas;
    uint32_t t = 0, e = 0;
    int32_t device = 0;
    cudaStream_t st = nullptr;
    int32_t threads = 1024;
    size_t smem = 0;
    uint32_t ymagic = 0;
    int32_t cnt_levels = 8;
    int32_t qmax = 0;
    int32_t ell_deg = 0;  // I8: width of the padded neighbour table (0 = CSR path)
    int32_t bands = 1;    // grid BITS: row bands per word group (CTA pairs with DSMEM halos)
    bool fused_ok = true; // grid BITS: the fused PT launch's clusters (K/32 x bands CTAs per copy) fit one wave
    bool xc_ok = false;   // grid BITS, 2 bands: cooperative fused launch with copies over K/32 clusters
    bool sched_ok = false;     // grid BITS, 1 band: persistent ticket-scheduled fused launch (k_grid_sched)
    int32_t sched_ctas = 0;    // its resident CTAs
    uint32_t *d_xs_ctl = nullptr, *d_xs_B = nullptr, *d_xs_M = nullptr, *d_xs_S = nullptr;
    int64_t *d_xs_E = nullptr;
    int64_t *d_xc_E = nullptr;
    uint32_t *d_xc_B = nullptr, *d_xc_bar = nullptr;
    std::vector<int32_t> class_off;
    // device buffers
    uint32_t *d_state[2] = {nullptr, nullptr};
    int cur = 0;
    int8_t *d_s8 = nullptr;
    uint32_t *d_pk = nullptr;  // packed-row working copy of d_s8 (float + padded table, §5.4c), lazily allocated
    int64_t *d_E = nullptr;
    double *d_Ef = nullptr;
    int64_t *d_walker = nullptr;
    uint32_t *d_swapmask = nullptr;
    int64_t *d_xpart = nullptr;  // k_exchange partial bests
    uint32_t *d_xctr = nullptr;  // k_exchange CTA ticket
    uint8_t *d_jbyte = nullptr;
    uint8_t *d_jrd = nullptr;  // grid: original order, bit 0 J_right=-1, bit 1 J_down=-1 (ICM energies)
    uint32_t f = 0;            // Houdayer/ICM moves done
    uint32_t *d_planes = nullptr;
    int32_t *d_rp = nullptr, *d_col = nullptr, *d_wi = nullptr, *d_class_off = nullptr;
    int32_t *d_ell_col = nullptr, *d_ell_w = nullptr;
    uint32_t *d_nbr = nullptr, *d_orig = nullptr, *d_o2i = nullptr;
    float *d_wf = nullptr, *d_betaf = nullptr;
    uint64_t *d_T = nullptr, *d_Tx = nullptr;
    int64_t *d_Tx_off = nullptr;
    int32_t *d_Tx_len = nullptr;
    BestDev *d_best = nullptr;
    int64_t *d_copy_best = nullptr;  // fused PT launches: per-copy best (E, slot, sweep)
    int64_t *d_cbest = nullptr;      // persistent per-copy best-so-far (E, slot, sweep)
    int8_t *d_snap = nullptr;        // fused PT launches: per-copy best configuration
    int8_t *d_best_spins = nullptr, *d_tmp = nullptr;
    int64_t *d_merge = nullptr;      // ising_merge_best result (E, sweep, slot)
    void *d_scratch = nullptr;
    size_t scratch_bytes = 0;
    std::vector<void *> allocs;
    void *d_sched = nullptr;  // annealing schedules (planes or thresholds), grown on demand
    size_t sched_bytes = 0;
    std::vector<uint32_t> orig;  // internal -> original (CSR kernels)
    std::vector<uint32_t> o2i;
    uint64_t fingerprint = 0;  // FNV-1a of the instance, colouring and ladder (checkpoints)

    template <class T>
    // Device buffers come from the device's stream-ordered memory pool (cudaMallocAsync on the
    // handle's stream), which keeps freed memory for the next handle: creating and destroying
    // handles in a loop (bench e2e, trial batches) costs no cudaMalloc / cudaFree (the latter
    // synchronises the device) after the first time.
    cudaError_t alloc(T **p, size_t count)
    {
        *p = nullptr;
        if (count == 0)
            count = 1;
        cudaError_t e = cudaMallocAsync((void **)p, count * sizeof(T), st);
        if (e == cudaSuccess)
            allocs.push_back((void *)*p);
        return e;
    }
    ~ising_handle()
    {
        for (void *p : allocs)
            cudaFreeAsync(p, st);
        if (d_sched)
            cudaFree(d_sched);
        cudaStreamSynchronize(st);
    }
};

namespace {

int validate_desc(const ising_run_desc *d)
{
    if (!d)
        return fail(ISING_E_ARG, "desc is NULL");
    if (d->n_temps < 1)
        return fail(ISING_E_ARG, "n_temps must be >= 1");
    if (d->n_copies < 1)
        return fail(ISING_E_ARG, "n_copies must be >= 1");
    if (d->copy_begin < 0 || d->copy_end > d->n_copies || d->copy_begin >= d->copy_end)
        return fail(ISING_E_ARG, "bad copy shard [" + std::to_string(d->copy_begin) + ", " +
                                     std::to_string(d->copy_end) + ")");
    if (!d->betas)
        return fail(ISING_E_ARG, "betas is NULL");
    for (int k = 0; k < d->n_temps; ++k) {
        if (!(d->betas[k] > 0.0) || !std::isfinite(d->betas[k]))
            return fail(ISING_E_ARG, "beta[" + std::to_string(k) + "] must be finite and > 0");
        if (k > 0 && !(d->betas[k] > d->betas[k - 1]))
            return fail(ISING_E_ARG, "betas must be strictly increasing (at index " +
                                         std::to_string(k) + ")");
    }
    if (d->layout != ISING_SPINS_BITS && d->layout != ISING_SPINS_I8)
        return fail(ISING_E_ARG, "unknown layout");
    if (d->layout == ISING_SPINS_BITS && d->rng != ISING_RNG_PLANE)
        return fail(ISING_E_ARG, "BITS layout requires the PLANE RNG contract");
    if (d->layout == ISING_SPINS_I8 && d->rng != ISING_RNG_WORD)
        return fail(ISING_E_ARG, "I8 layout requires the WORD RNG contract");
    if (d->layout == ISING_SPINS_BITS && (d->n_temps % 32 != 0 || d->n_temps > 256))
        return fail(ISING_E_ARG, "BITS layout requires n_temps % 32 == 0 and <= 256");
    if (d->layout == ISING_SPINS_I8 && d->n_temps % 8 != 0)  // one WORD Philox call = 8 replicas
        return fail(ISING_E_ARG, "I8 layout requires n_temps % 8 == 0");
    if ((int64_t)d->n_copies * d->n_temps >= (int64_t)1 << 33)
        return fail(ISING_E_ARG, "too many replicas");
    // the int8 kernels index local replicas with int32 (R and R/8 threads per vertex)
    if (d->layout == ISING_SPINS_I8 && (int64_t)(d->copy_end - d->copy_begin) * d->n_temps >= (int64_t)1 << 31)
        return fail(ISING_E_UNSUPPORTED, "I8 layout: local replicas must be < 2^31");
    if (d->stream) {  // a stream of another device would run the handle's work on the wrong GPU
        int sdev = -1;
        if (cudaStreamGetDevice((cudaStream_t)d->stream, &sdev) == cudaSuccess && sdev != d->device)
            return fail(ISING_E_ARG, "stream belongs to device " + std::to_string(sdev) + ", desc->device is " +
                                         std::to_string(d->device));
        cudaGetLastError();
    }
    if (d->colouring != ISING_COLOUR_GREEDY && d->colouring != ISING_COLOUR_JP)
        return fail(ISING_E_ARG, "unknown colouring");
    if (d->block_threads != 0 && (d->block_threads < 32 || d->block_threads > 1024 ||
                                  d->block_threads % 32 != 0))
        return fail(ISING_E_ARG, "block_threads must be 0 or a multiple of 32 in [32, 1024]");
    return ISING_OK;
}

void fill_run(ising_handle *h, const ising_run_desc *d)
{
    h->seed = d->seed;
    h->rk = make_round_keys(d->seed);
    h->K = d->n_temps;
    h->C = d->n_copies;
    h->c0 = d->copy_begin;
    h->c1 = d->copy_end;
    h->C_local = h->c1 - h->c0;
    h->R = (int64_t)h->C_local * h->K;
    h->slot0 = (int64_t)h->c0 * h->K;
    h->G = (int32_t)(h->R / 32);
    h->g0 = (uint32_t)(h->slot0 / 32);
    h->wpc = (h->K + 31) / 32;
    h->betas.assign(d->betas, d->betas + h->K);
    h->layout = d->layout;
    h->rng = d->rng;
    h->device = d->device;
    h->st = (cudaStream_t)d->stream;
    {  // keep freed pool memory for the next handle (default threshold 0 returns it at sync)
        static bool retained[64] = {};
        if (d->device >= 0 && d->device < 64 && !retained[d->device]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, d->device) == cudaSuccess) {
                uint64_t thr = ~0ull;
                if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess)
                    retained[d->device] = true;
            }
            cudaGetLastError();  // no GPU: the first CUDA call of create reports it
        }
    }
    h->threads = d->block_threads ? d->block_threads : 1024;
}

// Integer Metropolis table T[k][q] (q = dE/2 = 0..qmax; q = 0 unused).
std::vector<uint64_t> accept_table(const std::vector<double> &betas, int32_t qmax)
{
    const size_t K = betas.size();
    std::vector<uint64_t> T(K * (qmax + 1));
    for (size_t k = 0; k < K; ++k) {
        T[k * (qmax + 1)] = std::numeric_limits<uint64_t>::max();
        for (int32_t q = 1; q <= qmax; ++q)
            T[k * (qmax + 1) + q] = metropolis_threshold(betas[k], 2 * (int64_t)q);
    }
    return T;
}

// Plane tables: for word type wt (temperatures 32wt..32wt+31) and class q,
// P[j] has bit b = bit (63-j) of T[32wt+b][q].
void plane_table(const std::vector<double> &betas, const std::vector<int32_t> &qs,
                 std::vector<uint32_t> &out)
{
    const int32_t KW = (int32_t)betas.size() / 32;
    out.assign((size_t)KW * qs.size() * 64, 0u);
    for (int32_t wt = 0; wt < KW; ++wt)
        for (size_t qi = 0; qi < qs.size(); ++qi)
            for (int b = 0; b < 32; ++b) {
                const uint64_t T = metropolis_threshold(betas[32 * wt + b], 2 * (int64_t)qs[qi]);
                for (int j = 0; j < 64; ++j)
                    if ((T >> (63 - j)) & 1u)
                        out[((size_t)wt * qs.size() + qi) * 64 + j] |= 1u << b;
            }
}

int build_common_device(ising_handle *h, int64_t sum_abs_w)
{
    CK(cudaSetDevice(h->device));
    CK(h->alloc(&h->d_E, h->R));
    if (h->wtype == ISING_W_F32)
        CK(h->alloc(&h->d_Ef, h->R));
    CK(h->alloc(&h->d_walker, h->R));
    CK(h->alloc(&h->d_swapmask, (size_t)h->C_local * h->wpc));
    CK(h->alloc(&h->d_xpart, 2 * (size_t)kExMaxBlocks));
    CK(h->alloc(&h->d_xctr, 1));
    CK(cudaMemsetAsync(h->d_xctr, 0, sizeof(uint32_t), h->st));
    CK(h->alloc(&h->d_best, 1));
    CK(h->alloc(&h->d_cbest, (size_t)h->C_local * 3));
    {
        std::vector<int64_t> cb((size_t)h->C_local * 3);
        for (int32_t c = 0; c < h->C_local; ++c) {
            cb[3 * c] = 0;
            cb[3 * c + 1] = -1;
            cb[3 * c + 2] = -1;
        }
        CK(cudaMemcpyAsync(h->d_cbest, cb.data(), cb.size() * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    CK(h->alloc(&h->d_best_spins, h->n));
    CK(h->alloc(&h->d_merge, 3));
    CK(h->alloc(&h->d_tmp, h->n));
    std::vector<int64_t> walker(h->R);
    std::iota(walker.begin(), walker.end(), h->slot0);
    CK(cudaMemcpyAsync(h->d_walker, walker.data(), h->R * sizeof(int64_t), cudaMemcpyHostToDevice,
                       h->st));
    BestDev b{0, -1, -1, 0, 0};
    CK(cudaMemcpyAsync(h->d_best, &b, sizeof(b), cudaMemcpyHostToDevice, h->st));
    // exchange tables (integer weights): d from -1 down while the threshold is
    // non-zero, capped by the largest possible energy difference 2*sum|w|.
    if (h->wtype == ISING_W_I32 && h->K >= 2) {
        // rows are independent (hundreds of thousands of libm exp calls for a 64-rung
        // ladder): built on host threads, then concatenated in pair order
        const int32_t npair = h->K - 1;
        std::vector<std::vector<uint64_t>> rows(npair);
        const int64_t dmax = 2 * sum_abs_w;
        auto build_rows = [&](int32_t k0, int32_t step) {
            for (int32_t k = k0; k < npair; k += step)
                for (int64_t d = -1; -d <= dmax; --d) {
                    const uint64_t T = exchange_threshold(h->betas[k], h->betas[k + 1], d);
                    if (T == 0)
                        break;
                    rows[k].push_back(T);
                }
        };
        const int32_t nthr =
            std::max(1, std::min<int32_t>(std::min<int32_t>(npair, 16), (int32_t)std::thread::hardware_concurrency()));
        if (nthr > 1 && dmax > 256) {
            std::vector<std::thread> pool;
            for (int32_t t = 0; t < nthr; ++t)
                pool.emplace_back(build_rows, t, nthr);
            for (auto &th : pool)
                th.join();
        } else {
            build_rows(0, 1);
        }
        std::vector<uint64_t> Tx;
        std::vector<int64_t> off(npair);
        std::vector<int32_t> len(npair);
        for (int32_t k = 0; k < npair; ++k) {
            off[k] = (int64_t)Tx.size();
            len[k] = (int32_t)rows[k].size();
            Tx.insert(Tx.end(), rows[k].begin(), rows[k].end());
        }
        CK(h->alloc(&h->d_Tx, Tx.size()));
        CK(h->alloc(&h->d_Tx_off, off.size()));
        CK(h->alloc(&h->d_Tx_len, len.size()));
        CK(cudaMemcpyAsync(h->d_Tx, Tx.data(), Tx.size() * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(h->d_Tx_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(h->d_Tx_len, len.data(), len.size() * 4, cudaMemcpyHostToDevice, h->st));
    }
    return ISING_OK;
}

// k_grid_bits launch: n_rounds x (k_ex sweeps [+ best check + exchange if pt]).
GridBitsParams grid_params(ising_handle *h, int32_t n_rounds, int32_t k_ex, bool pt)
{
    GridBitsParams p{};
    p.state_in = h->d_state[h->cur];
    p.state_out = h->d_state[h->cur ^ 1];
    p.jbyte = h->d_jbyte;
    p.qcap = grid_bits_qcap(h->n);
    p.planes = h->d_planes;
    p.E_out = h->d_E;
    p.Lx = h->Lx; p.Ly = h->Ly; p.n = h->n; p.hx = h->Lx / 2; p.half = h->n / 2;
    p.ymagic = h->ymagic;
    p.words_per_copy = h->wpc;
    p.g0 = h->g0;
    p.t0 = h->t;
    p.n_rounds = n_rounds;
    p.k_ex = k_ex;
    p.pt = pt ? 1 : 0;
    p.e0 = h->e;
    p.walker = h->d_walker;
    p.copy_best = h->d_copy_best;
    p.snap = h->d_snap;
    p.Tx = h->d_Tx;
    p.Tx_off = h->d_Tx_off;
    p.Tx_len = h->d_Tx_len;
    p.rk = h->rk;
    p.bands = h->bands;
    p.xc = 0;
    p.xc_E = h->d_xc_E;
    p.xc_B = h->d_xc_B;
    p.xc_bar = h->d_xc_bar;
    p.n_groups = h->G;
    p.xs_ctl = h->d_xs_ctl;
    p.xs_E = h->d_xs_E;
    p.xs_B = h->d_xs_B;
    p.xs_M = h->d_xs_M;
    p.xs_S = h->d_xs_S;
    return p;
}

CsrBitsParams csr_params(ising_handle *h, int32_t n_rounds, int32_t k_ex, bool pt)
{
    CsrBitsParams p{};
    p.state_in = h->d_state[h->cur];
    p.state_out = h->d_state[h->cur ^ 1];
    p.rp = h->d_rp; p.nbr = h->d_nbr; p.orig = h->d_orig; p.class_off = h->d_class_off;
    p.planes = h->d_planes; p.E_out = h->d_E;
    p.n = h->n; p.ncol = h->ncol; p.qmax = h->qmax; p.m = h->m;
    p.words_per_copy = h->wpc; p.g0 = h->g0; p.t0 = h->t;
    p.n_rounds = n_rounds;
    p.k_ex = k_ex;
    p.qcap = csr_bits_qcap(h->n, h->qmax);
    p.pt = pt ? 1 : 0;
    p.e0 = h->e;
    p.walker = h->d_walker;
    p.copy_best = h->d_copy_best;
    p.snap = h->d_snap;
    p.Tx = h->d_Tx;
    p.Tx_off = h->d_Tx_off;
    p.Tx_len = h->d_Tx_len;
    p.rk = h->rk;
    return p;
}

// Small int8 instances with integer weights run a whole PT schedule in one k_i8_small launch
// (one CTA per copy, the copy's n x K spins in shared memory).
bool small_i8(const ising_handle *h)
{
    return h->kernel == KER_CSR_I8 && h->wtype == ISING_W_I32 && h->K >= 2 && h->K <= 256 &&
           h->K % 8 == 0 && (int64_t)h->n * h->K <= kI8SmallMaxBytes &&
           (int64_t)h->K * (h->qmax + 1) * 8 <= 64 * 1024;  // threshold rows in shared memory
}

// Torus sweep launch: the band-split kernel when the handle's groups are split over CTA pairs.
cudaError_t launch_grid(const ising_handle *h, const GridBitsParams &p)
{
    return h->bands > 1 ? launch_grid_bands(p, h->G, h->threads, h->smem, h->st)
                        : launch_grid_bits(p, h->G, h->threads, h->smem, h->st);
}

// Energies after a state change (set_spins / create).
int refresh_energy(ising_handle *h)
{
    if (h->kernel == KER_GRID_BITS) {
        CK(launch_grid(h, grid_params(h, 1, 0, false)));
        h->cur ^= 1;
    } else if (h->kernel == KER_CSR_BITS) {
        CK(launch_csr_bits(csr_params(h, 1, 0, false), h->G, h->threads, h->smem, h->st));
        h->cur ^= 1;
    } else {
        CK(launch_energy_i8(h->d_s8, h->d_rp, h->d_col, h->d_wi, h->d_wf, h->n, (int32_t)h->R, h->d_E,
                            h->d_Ef, h->d_scratch, h->scratch_bytes, h->st));
    }
    return ISING_OK;
}

// Validated CSR -> internal, colour-sorted CSR and device upload (CSR kernels).
// Lowest i in [0, n) with !check(i, nullptr), or n: the vertices split over up to 16 host
// threads (per-vertex checks of a graph are independent; the lowest failing vertex is the one a
// sequential scan reports first).
template <class F>
int32_t par_first_failing(int32_t n, F &&check)
{
    const int32_t nthr =
        std::max(1, std::min<int32_t>(16, std::min<int32_t>((int32_t)std::thread::hardware_concurrency(), n / 65536)));
    std::vector<int32_t> bad(nthr, n);
    auto work = [&](int32_t t) {
        const int32_t lo = (int32_t)((int64_t)n * t / nthr), hi = (int32_t)((int64_t)n * (t + 1) / nthr);
        for (int32_t i = lo; i < hi; ++i)
            if (!check(i, nullptr)) {
                bad[t] = i;
                return;
            }
    };
    if (nthr > 1) {
        std::vector<std::thread> pool;
        for (int32_t t = 0; t < nthr; ++t)
            pool.emplace_back(work, t);
        for (auto &th : pool)
            th.join();
    } else {
        work(0);
    }
    return *std::min_element(bad.begin(), bad.end());
}

// Row checks of vertex i in (entry) order: range, self-loop, duplicate of an earlier entry,
// finite weight.  False with the message of the first failing entry.
bool csr_row_ok(int32_t n, const int64_t *row_ptr, const int32_t *col, const int32_t *wi, const float *wf,
                int32_t i, std::string *msg)
{
    const int64_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
    const bool small = e1 - e0 <= 64;
    std::vector<int32_t> seen;  // earlier entries of a long row, kept sorted
    for (int64_t e = e0; e < e1; ++e) {
        const int32_t j = col[e];
        if (j < 0 || j >= n) {
            if (msg)
                *msg = "col[" + std::to_string(e) + "] = " + std::to_string(j) + " out of range at vertex " +
                       std::to_string(i);
            return false;
        }
        if (j == i) {
            if (msg)
                *msg = "self-loop at vertex " + std::to_string(i);
            return false;
        }
        bool dup = false;
        if (small) {
            for (int64_t f = e0; f < e && !dup; ++f)
                dup = col[f] == j;
        } else {
            const auto it = std::lower_bound(seen.begin(), seen.end(), j);
            dup = it != seen.end() && *it == j;
            if (!dup)
                seen.insert(it, j);
        }
        if (dup) {
            if (msg)
                *msg = "duplicate edge " + std::to_string(i) + "-" + std::to_string(j);
            return false;
        }
        if (wf && !std::isfinite(wf[e])) {
            if (msg)
                *msg = "non-finite weight at entry " + std::to_string(e);
            return false;
        }
    }
    return true;
}

// Symmetry of vertex i's row: (i, j, w) present iff (j, i, w).
bool csr_sym_ok(const int64_t *row_ptr, const int32_t *col, const int32_t *wi, const float *wf, int32_t i,
                std::string *msg)
{
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        const int32_t j = col[e];
        bool found = false;
        for (int64_t f = row_ptr[j]; f < row_ptr[j + 1]; ++f)
            if (col[f] == i) {
                found = wi ? (wi[f] == wi[e]) : (wf[f] == wf[e]);
                break;
            }
        if (!found) {
            if (msg)
                *msg = "asymmetric coupling " + std::to_string(i) + "-" + std::to_string(j);
            return false;
        }
    }
    return true;
}

// Device buffers that live only during create (returned to the stream-ordered pool).
struct CreateTmp {
    cudaStream_t st;
    std::vector<void *> ptrs;
    template <class T>
    cudaError_t alloc(T **p, size_t count)
    {
        *p = nullptr;
        cudaError_t e = cudaMallocAsync((void **)p, (count ? count : 1) * sizeof(T), st);
        if (e == cudaSuccess)
            ptrs.push_back((void *)*p);
        return e;
    }
    ~CreateTmp()
    {
        for (void *p : ptrs)
            cudaFreeAsync(p, st);
    }
};

int create_csr_i8_device(int32_t n, const int64_t *row_ptr, const int32_t *col, const void *w, int32_t wtype,
                         const int32_t *colour, const ising_run_desc *desc, ising_handle **out);

int create_csr_impl(int32_t n, const int64_t *row_ptr, const int32_t *col, const void *w,
                    int32_t wtype, const int32_t *colour, const ising_run_desc *desc,
                    ising_handle **out)
{
    std::unique_ptr<ising_handle> h(new ising_handle());
    h->n = n;
    h->wtype = wtype;
    fill_run(h.get(), desc);
    const int64_t m2 = row_ptr[n];
    if (m2 >= ((int64_t)1 << 31) - 1)
        return fail(ISING_E_UNSUPPORTED, "more than 2^31-1 directed edges");
    h->m = m2 / 2;
    const int32_t *wi = wtype == ISING_W_I32 ? (const int32_t *)w : nullptr;
    const float *wf = wtype == ISING_W_F32 ? (const float *)w : nullptr;

    // per-vertex sum |w| guard and totals
    int64_t qmax = 0, sum_abs = 0;
    int32_t maxdeg = 0;
    bool pm1 = true;
    for (int32_t i = 0; i < n; ++i) {
        int64_t s = 0;
        maxdeg = std::max<int32_t>(maxdeg, (int32_t)(row_ptr[i + 1] - row_ptr[i]));
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            if (wi) {
                s += std::llabs((long long)wi[e]);
                pm1 &= (wi[e] == 1 || wi[e] == -1);
                if (col[e] > i)
                    h->W_int += wi[e];
            } else if (col[e] > i) {
                h->W_f += (double)wf[e];
            }
        }
        if (wi && s >= ((int64_t)1 << 30))
            return fail(ISING_E_GRAPH, "sum of |w| at vertex " + std::to_string(i) + " >= 2^30");
        qmax = std::max(qmax, s);
        sum_abs += s;
    }
    sum_abs /= 2;
    // (the int8 layout is created on the device: create_csr_i8_device)
    if (!desc->block_threads)
        h->threads = kCsrMaxThreads;
    if (h->threads > kCsrMaxThreads)
        return fail(ISING_E_ARG, "BITS: block_threads must be <= " + std::to_string(kCsrMaxThreads));
    if (!wi || !pm1)
        return fail(ISING_E_UNSUPPORTED, "BITS layout needs integer weights in {-1,+1}");
    if (maxdeg > 15)
        return fail(ISING_E_UNSUPPORTED, "BITS layout supports degree <= 15");
    h->kernel = KER_CSR_BITS;
    h->qmax = (int32_t)qmax;

    // colouring
    std::vector<int32_t> col_of(n);
    if (colour) {
        int32_t mx = -1;
        for (int32_t i = 0; i < n; ++i) {
            if (colour[i] < 0 || colour[i] >= (1 << 16))
                return fail(ISING_E_GRAPH, "colour of vertex " + std::to_string(i) + " out of range");
            mx = std::max(mx, colour[i]);
            col_of[i] = colour[i];
        }
        auto proper = [&](int32_t i, std::string *msg) -> bool {
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
                if (colour[col[e]] == colour[i]) {
                    if (msg)
                        *msg = "improper colouring: vertices " + std::to_string(i) + " and " +
                               std::to_string(col[e]) + " share colour";
                    return false;
                }
            return true;
        };
        const int32_t bad = par_first_failing(n, proper);
        if (bad < n) {
            std::string msg;
            proper(bad, &msg);
            return fail(ISING_E_GRAPH, msg);
        }
        std::vector<char> used(mx + 1, 0);
        for (int32_t i = 0; i < n; ++i)
            used[col_of[i]] = 1;
        for (int32_t c = 0; c <= mx; ++c)
            if (!used[c])
                return fail(ISING_E_GRAPH, "colour ids must be 0..ncol-1 without gaps (missing " +
                                               std::to_string(c) + ")");
        h->ncol = mx + 1;
    } else if (desc->colouring == ISING_COLOUR_JP) {  // on the device, as for the int8 layout
        CK(cudaSetDevice(h->device));
        CreateTmp tmp{h->st, {}};
        int64_t *d_rp64;
        int32_t *d_c, *d_colour, *d_cnt;
        uint32_t *d_prio;
        CK(tmp.alloc(&d_rp64, (size_t)n + 1));
        CK(tmp.alloc(&d_c, (size_t)row_ptr[n]));
        CK(tmp.alloc(&d_colour, (size_t)n));
        CK(tmp.alloc(&d_prio, (size_t)n));
        CK(tmp.alloc(&d_cnt, 2));
        CK(cudaMemcpyAsync(d_rp64, row_ptr, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(d_c, col, (size_t)row_ptr[n] * 4, cudaMemcpyHostToDevice, h->st));
        int32_t ncol = 0;
        CK(colour_jp_device(n, d_rp64, d_c, d_prio, d_colour, d_cnt, &ncol, h->st));
        CK(cudaMemcpyAsync(col_of.data(), d_colour, (size_t)n * 4, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        h->ncol = ncol;
    } else {
        h->ncol = ising_greedy_colour(n, row_ptr, col, col_of.data());
        if (h->ncol < 0)
            return h->ncol;
    }

    // internal order: (colour, degree, original id)
    h->orig.resize(n);
    const bool by_deg = h->kernel == KER_CSR_BITS;
    {  // counting sort by key (colour, [degree]), ids ascending inside a key: O(n + keys)
        const int64_t nd = by_deg ? (int64_t)maxdeg + 1 : 1;
        auto key = [&](int32_t i) {
            return (int64_t)col_of[i] * nd + (by_deg ? row_ptr[i + 1] - row_ptr[i] : 0);
        };
        std::vector<int64_t> start((size_t)h->ncol * nd + 1, 0);
        for (int32_t i = 0; i < n; ++i)
            ++start[key(i) + 1];
        for (size_t k = 1; k < start.size(); ++k)
            start[k] += start[k - 1];
        for (int32_t i = 0; i < n; ++i)
            h->orig[start[key(i)]++] = (uint32_t)i;
    }
    h->o2i.resize(n);
    for (int32_t v = 0; v < n; ++v)
        h->o2i[h->orig[v]] = (uint32_t)v;
    h->class_off.assign(h->ncol + 1, 0);
    for (int32_t i = 0; i < n; ++i)
        h->class_off[col_of[i] + 1]++;
    for (int32_t c = 0; c < h->ncol; ++c)
        h->class_off[c + 1] += h->class_off[c];

    std::vector<int32_t> rp(n + 1, 0);
    for (int32_t v = 0; v < n; ++v)
        rp[v + 1] = rp[v] + (int32_t)(row_ptr[h->orig[v] + 1] - row_ptr[h->orig[v]]);
    std::vector<int32_t> ci(m2);
    std::vector<int32_t> wiv;
    std::vector<float> wfv;
    std::vector<uint32_t> nbr;
    if (wi) wiv.resize(m2);
    if (wf) wfv.resize(m2);
    if (by_deg) nbr.resize(m2);
    for (int32_t v = 0; v < n; ++v) {
        const int32_t i = (int32_t)h->orig[v];
        int32_t o = rp[v];
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e, ++o) {
            ci[o] = (int32_t)h->o2i[col[e]];
            if (wi) wiv[o] = wi[e];
            if (wf) wfv[o] = wf[e];
            if (by_deg) nbr[o] = (uint32_t)ci[o] | (wi[e] < 0 ? 0x80000000u : 0u);
        }
    }

    int rc = build_common_device(h.get(), sum_abs);
    if (rc)
        return rc;
    CK(h->alloc(&h->d_rp, n + 1));
    CK(h->alloc(&h->d_orig, n));
    CK(h->alloc(&h->d_o2i, n));
    CK(h->alloc(&h->d_class_off, h->ncol + 1));
    CK(cudaMemcpyAsync(h->d_rp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->d_orig, h->orig.data(), (size_t)n * 4, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->d_o2i, h->o2i.data(), (size_t)n * 4, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->d_class_off, h->class_off.data(), (h->ncol + 1) * 4,
                       cudaMemcpyHostToDevice, h->st));
    if (by_deg) {
        CK(h->alloc(&h->d_nbr, m2));
        CK(cudaMemcpyAsync(h->d_nbr, nbr.data(), (size_t)m2 * 4, cudaMemcpyHostToDevice, h->st));
        // planes for q = 1..qmax
        std::vector<int32_t> qs(h->qmax);
        std::iota(qs.begin(), qs.end(), 1);
        std::vector<uint32_t> planes;
        plane_table(h->betas, qs, planes);
        CK(h->alloc(&h->d_planes, std::max<size_t>(planes.size(), 1)));
        if (!planes.empty())
            CK(cudaMemcpyAsync(h->d_planes, planes.data(), planes.size() * 4, cudaMemcpyHostToDevice,
                               h->st));
        h->smem = csr_bits_smem(n, h->qmax, h->wpc);
        if (h->smem > 200 * 1024)
            return fail(ISING_E_UNSUPPORTED,
                        "BITS layout: n too large for a shared-memory resident word group");
        CK(h->alloc(&h->d_state[0], (size_t)h->G * n));
        CK(h->alloc(&h->d_state[1], (size_t)h->G * n));
        CK(h->alloc(&h->d_copy_best, (size_t)h->C_local * 3));
        CK(h->alloc(&h->d_snap, (size_t)h->C_local * n));
        CK(launch_init_bits(h->d_state[0], h->G, n, h->d_orig, h->g0, h->rk, h->st));
    }
    rc = refresh_energy(h.get());
    if (rc)
        return rc;
    CK(cudaStreamSynchronize(h->st));
    h->fingerprint = fnv1a(kFnvBasis, row_ptr, ((size_t)n + 1) * 8);
    h->fingerprint = fnv1a(h->fingerprint, col, (size_t)m2 * 4);
    h->fingerprint = fnv1a(h->fingerprint, w, (size_t)m2 * 4);
    h->fingerprint = fnv1a(h->fingerprint, h->orig.data(), h->orig.size() * 4);
    h->fingerprint = fnv1a(h->fingerprint, h->betas.data(), h->betas.size() * 8);
    *out = h.release();
    return ISING_OK;
}

// ising_create_csr for the int8 layout: the caller's CSR is uploaded once and
// validated, coloured (caller colouring validated, or Jones-Plassmann on the device, or the
// ascending-id greedy on the host), put in the colour-sorted internal order and turned into
// the internal CSR / padded tables by kernels (k_create.cu).  Same checks, error precedence,
// internal order and tables as the host path of the bit-packed layout.
int create_csr_i8_device(int32_t n, const int64_t *row_ptr, const int32_t *col, const void *w, int32_t wtype,
                         const int32_t *colour, const ising_run_desc *desc, ising_handle **out)
{
    std::unique_ptr<ising_handle> h(new ising_handle());
    h->n = n;
    h->wtype = wtype;
    h->kernel = KER_CSR_I8;
    fill_run(h.get(), desc);
    const int64_t m2 = row_ptr[n];
    if (m2 >= ((int64_t)1 << 31) - 1)
        return fail(ISING_E_UNSUPPORTED, "more than 2^31-1 directed edges");
    h->m = m2 / 2;
    const int32_t *wi = wtype == ISING_W_I32 ? (const int32_t *)w : nullptr;
    const float *wf = wtype == ISING_W_F32 ? (const float *)w : nullptr;
    CK(cudaSetDevice(h->device));
    CreateTmp tmp{h->st, {}};
    int64_t *d_rp64;
    int32_t *d_colin, *d_colour, *d_jp;
    uint32_t *d_win, *d_prio;
    CsrCheck *d_chk;
    uint8_t *d_used;
    CK(tmp.alloc(&d_rp64, (size_t)n + 1));
    CK(tmp.alloc(&d_colin, (size_t)m2));
    CK(tmp.alloc(&d_win, (size_t)m2));
    CK(tmp.alloc(&d_colour, (size_t)n));
    CK(tmp.alloc(&d_chk, 1));
    CK(tmp.alloc(&d_used, (size_t)1 << 16));
    CK(tmp.alloc(&d_jp, 2));
    CK(cudaMemcpyAsync(d_rp64, row_ptr, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(d_colin, col, (size_t)m2 * 4, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(d_win, w, (size_t)m2 * 4, cudaMemcpyHostToDevice, h->st));
    if (colour)
        CK(cudaMemcpyAsync(d_colour, colour, (size_t)n * 4, cudaMemcpyHostToDevice, h->st));
    CK(launch_csr_check(n, d_rp64, d_colin, wi ? (const int32_t *)d_win : nullptr,
                        wf ? (const float *)d_win : nullptr, colour ? d_colour : nullptr, d_chk, d_used, h->st));
    CsrCheck chk;
    CK(cudaMemcpyAsync(&chk, d_chk, sizeof(chk), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    // errors in the host path's order: row checks, symmetry, the |w| guard, the colouring
    if (chk.bad_row != INT32_MAX || chk.bad_sym != INT32_MAX) {
        std::string msg;
        if (chk.bad_row != INT32_MAX)
            csr_row_ok(n, row_ptr, col, wi, wf, chk.bad_row, &msg);
        else
            csr_sym_ok(row_ptr, col, wi, wf, chk.bad_sym, &msg);
        return fail(ISING_E_GRAPH, msg);
    }
    if (chk.bad_sum != INT32_MAX)
        return fail(ISING_E_GRAPH, "sum of |w| at vertex " + std::to_string(chk.bad_sum) + " >= 2^30");
    if (colour) {
        if (chk.bad_colrange != INT32_MAX)
            return fail(ISING_E_GRAPH, "colour of vertex " + std::to_string(chk.bad_colrange) + " out of range");
        if (chk.bad_proper != INT32_MAX) {
            const int32_t i = chk.bad_proper;
            int32_t j = -1;
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1] && j < 0; ++e)
                if (colour[col[e]] == colour[i])
                    j = col[e];
            return fail(ISING_E_GRAPH, "improper colouring: vertices " + std::to_string(i) + " and " +
                                           std::to_string(j) + " share colour");
        }
        std::vector<uint8_t> used((size_t)chk.max_colour + 1);
        CK(cudaMemcpyAsync(used.data(), d_used, used.size(), cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        for (int32_t c = 0; c <= chk.max_colour; ++c)
            if (!used[c])
                return fail(ISING_E_GRAPH, "colour ids must be 0..ncol-1 without gaps (missing " +
                                               std::to_string(c) + ")");
        h->ncol = chk.max_colour + 1;
    } else if (desc->colouring == ISING_COLOUR_JP) {
        CK(tmp.alloc(&d_prio, (size_t)n));
        int32_t ncol = 0;
        CK(colour_jp_device(n, d_rp64, d_colin, d_prio, d_colour, d_jp, &ncol, h->st));
        h->ncol = ncol;
    } else {  // ascending-id greedy (host, sequential by definition)
        std::vector<int32_t> col_of(n);
        h->ncol = ising_greedy_colour(n, row_ptr, col, col_of.data());
        if (h->ncol < 0)
            return h->ncol;
        CK(cudaMemcpyAsync(d_colour, col_of.data(), (size_t)n * 4, cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    h->qmax = (int32_t)chk.qmax;
    h->W_int = chk.W_int;
    const int32_t maxdeg = chk.maxdeg;
    // colour-sorted internal order (ids ascending inside a class) and the internal CSR
    CK(h->alloc(&h->d_orig, n));
    CK(h->alloc(&h->d_o2i, n));
    CK(h->alloc(&h->d_class_off, h->ncol + 1));
    CK(h->alloc(&h->d_rp, (size_t)n + 1));
    CK(build_order_device(n, h->ncol, d_colour, d_rp64, h->d_orig, h->d_o2i, h->d_class_off, h->d_rp, h->st));
    CK(h->alloc(&h->d_col, m2));
    uint32_t *d_wo;
    if (wi) {
        CK(h->alloc(&h->d_wi, m2));
        d_wo = (uint32_t *)h->d_wi;
    } else {
        CK(h->alloc(&h->d_wf, m2));
        d_wo = (uint32_t *)h->d_wf;
    }
    if (maxdeg <= 4) {
        h->ell_deg = maxdeg;
        CK(h->alloc(&h->d_ell_col, (size_t)n * 4));
        CK(h->alloc(&h->d_ell_w, (size_t)n * 4));
    }
    CK(launch_build_internal(n, d_rp64, d_colin, d_win, h->d_orig, h->d_o2i, h->d_rp, h->d_col, d_wo,
                             h->d_ell_col, (uint32_t *)h->d_ell_w, h->st));
    unsigned long long *d_hash;
    CK(tmp.alloc(&d_hash, 1));
    CK(cudaMemsetAsync(d_hash, 0, 8, h->st));
    CK(launch_hash_order(n, h->d_orig, d_hash, h->st));
    h->class_off.assign(h->ncol + 1, 0);
    CK(cudaMemcpyAsync(h->class_off.data(), h->d_class_off, (h->ncol + 1) * 4, cudaMemcpyDeviceToHost, h->st));
    int rc = build_common_device(h.get(), chk.sum_abs / 2);
    if (rc)
        return rc;
    if (wi) {  // per LOCAL replica r (temperature k = (slot0 + r) mod K): T_r[r][q], q = dE/2
        std::vector<uint64_t> Tk = accept_table(h->betas, h->qmax);
        std::vector<uint64_t> T((size_t)h->R * (h->qmax + 1));
        for (int64_t r = 0; r < h->R; ++r) {
            const int32_t k = (int32_t)((h->slot0 + r) % h->K);
            std::copy(Tk.begin() + (size_t)k * (h->qmax + 1), Tk.begin() + (size_t)(k + 1) * (h->qmax + 1),
                      T.begin() + (size_t)r * (h->qmax + 1));
        }
        CK(h->alloc(&h->d_T, T.size()));
        CK(cudaMemcpyAsync(h->d_T, T.data(), T.size() * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    } else {
        std::vector<float> bf(h->R);
        for (int64_t r = 0; r < h->R; ++r)
            bf[r] = 2.0f * (float)h->betas[(h->slot0 + r) % h->K];  // exact doubling
        CK(h->alloc(&h->d_betaf, h->R));
        CK(cudaMemcpyAsync(h->d_betaf, bf.data(), h->R * 4, cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    CK(h->alloc(&h->d_s8, (size_t)n * h->R));
    if (small_i8(h.get())) {  // fused PT launch scratch (k_i8_small)
        CK(h->alloc(&h->d_copy_best, (size_t)h->C_local * 3));
        CK(h->alloc(&h->d_snap, (size_t)h->C_local * n));
    }
    h->scratch_bytes = energy_i8_scratch(n, (int32_t)h->R);
    CK(h->alloc((char **)&h->d_scratch, h->scratch_bytes));
    CK(launch_init_i8(h->d_s8, n, (int32_t)h->R, h->d_orig, h->slot0, h->rk, h->st));
    rc = refresh_energy(h.get());
    if (rc)
        return rc;
    // float weights: W = sum of w over edges in edge order, in float64 (a sequential sum, on
    // the host while the device initialises)
    if (wf)
        for (int32_t i = 0; i < n; ++i)
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
                if (col[e] > i)
                    h->W_f += (double)wf[e];
    unsigned long long order_hash = 0;
    CK(cudaMemcpyAsync(&order_hash, d_hash, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const uint64_t hv[3] = {chk.hash, order_hash, (uint64_t)n};
    h->fingerprint = fnv1a(kFnvBasis, hv, sizeof(hv));
    h->fingerprint = fnv1a(h->fingerprint, h->betas.data(), h->betas.size() * 8);
    *out = h.release();
    return ISING_OK;
}

// int8 kernels: per colour phase launches; `sched` (annealing) holds per-sweep threshold
// tables T[s][R][qmax+1] (integer weights) or betaf[s][R] (float weights), else null.
int launch_sweeps_i8(ising_handle *h, int32_t ns, const void *sched)
{
    CsrI8Params p{};
    p.s = h->d_s8; p.rp = h->d_rp; p.col = h->d_col; p.wi = h->d_wi; p.wf = h->d_wf;
    p.orig = h->d_orig; p.T = h->d_T; p.betaf = h->d_betaf; p.R = (int32_t)h->R; p.K = h->K;
    p.nq = (int32_t)(h->R / 4);
    p.ell_col = h->d_ell_col;
    p.ell_w = h->d_ell_w;
    p.ell_deg = h->ell_deg;
    const int32_t tpv = (int32_t)(h->R / 8);  // threads per vertex
    p.nq_shift = -1;
    for (int sh = 0; sh < 31; ++sh)
        if ((1 << sh) == tpv)
            p.nq_shift = sh;
    p.slot0 = h->slot0; p.qmax = h->qmax; p.rk = h->rk;
    const int32_t thr = h->threads > kI8Threads ? kI8Threads : h->threads;
    // float weights + padded table + R % 256 == 0: sweep a packed-row working copy of the
    // state (same contract and decisions as the int8 kernels, so the result is
    // identical), packed before the first and unpacked after the last sweep of this call.
    // ISING_I8_PACKED=0 keeps the int8 kernels, =1 uses the packed rows for any sweep count.
    bool packed = h->wtype == ISING_W_F32 && h->d_ell_col && h->R % 256 == 0 && h->slot0 % 8 == 0;
    if (packed) {
        int mode = -1;
        if (const char *env = std::getenv("ISING_I8_PACKED"))
            mode = std::atoi(env);
        packed = mode == 1 || (mode != 0 && ns >= kI8PackedMinSweeps);
    }
    if (packed && !h->d_pk && h->alloc(&h->d_pk, (size_t)h->n * (size_t)(h->R / 32)) != cudaSuccess) {
        (void)cudaGetLastError();  // no room for the working copy: the int8 kernels run instead
        h->d_pk = nullptr;
        packed = false;
    }
    if (packed) {
        CK(launch_pack_rows(h->d_s8, h->d_pk, h->n, h->R, false, h->st));
        for (int32_t s = 0; s < ns; ++s) {
            p.t = h->t + (uint32_t)s;
            if (sched)
                p.betaf = (const float *)sched + (size_t)s * h->R;
            for (int32_t c = 0; c < h->ncol; ++c) {
                p.v_begin = h->class_off[c];
                p.v_end = h->class_off[c + 1];
                CK(launch_csr_packed_phase(p, h->d_pk, h->st));
            }
        }
        CK(launch_pack_rows(h->d_s8, h->d_pk, h->n, h->R, true, h->st));
    }
    for (int32_t s = 0; s < (packed ? 0 : ns); ++s) {
        p.t = h->t + (uint32_t)s;
        if (sched) {
            if (h->wtype == ISING_W_I32)
                p.T = (const uint64_t *)sched + (size_t)s * h->R * (h->qmax + 1);
            else
                p.betaf = (const float *)sched + (size_t)s * h->R;
        }
        for (int32_t c = 0; c < h->ncol; ++c) {
            p.v_begin = h->class_off[c];
            p.v_end = h->class_off[c + 1];
            CK(launch_csr_i8_phase(p, thr, h->st));
        }
    }
    if (ns > 0)
        CK(launch_energy_i8(h->d_s8, h->d_rp, h->d_col, h->d_wi, h->d_wf, h->n, (int32_t)h->R, h->d_E,
                            h->d_Ef, h->d_scratch, h->scratch_bytes, h->st));
    h->t += (uint32_t)ns;
    return ISING_OK;
}

int launch_sweeps(ising_handle *h, int32_t ns)
{
    if (h->kernel == KER_GRID_BITS && h->sched_ok && ns >= 2 && ns % 2 == 0) {
        // more word groups than resident CTAs: the persistent kernel with tasks (group, half of
        // the sweeps) keeps every SM busy (waves of whole groups would leave the last wave part-
        // filled: 512 groups = 3.46 x 148); same RNG counters, same result
        GridBitsParams p = grid_params(h, 2, ns / 2, false);
        const cudaError_t le = launch_grid_sched(p, h->sched_ctas, h->threads, h->smem, h->st);
        if (le == cudaErrorCooperativeLaunchTooLarge) {
            cudaGetLastError();
            h->sched_ok = false;
        } else {
            CK(le);
            h->cur ^= 1;
            h->t += (uint32_t)ns;
            return ISING_OK;
        }
    }
    if (h->kernel == KER_GRID_BITS) {
        CK(launch_grid(h, grid_params(h, 1, ns, false)));
        h->cur ^= 1;
    } else if (h->kernel == KER_CSR_BITS) {
        CK(launch_csr_bits(csr_params(h, 1, ns, false), h->G, h->threads, h->smem, h->st));
        h->cur ^= 1;
    } else {
        return launch_sweeps_i8(h, ns, nullptr);
    }
    h->t += (uint32_t)ns;
    return ISING_OK;
}

ExchangeParams exchange_params(ising_handle *h)
{
    ExchangeParams p{};
    p.xpart = h->d_xpart;
    p.xctr = h->d_xctr;
    p.E = h->d_E;
    p.walker = h->d_walker;
    p.cbest = h->d_cbest;
    p.swapmask = h->d_swapmask;
    p.best = h->d_best;
    p.best_spins = h->d_best_spins;
    p.layout = h->layout;
    p.state = h->d_state[h->cur];
    p.s8 = h->d_s8;
    p.perm_o2i = (h->kernel == KER_GRID_BITS) ? nullptr : h->d_o2i;
    p.n = h->n;
    p.K = h->K;
    p.C_local = h->C_local;
    p.words_per_copy = h->wpc;
    p.slot0 = h->slot0;
    p.R_local = h->R;
    p.is_float = h->wtype == ISING_W_F32;
    p.t = h->t;
    p.e = h->e;
    p.Tx = h->d_Tx;
    p.Tx_off = h->d_Tx_off;
    p.Tx_len = h->d_Tx_len;
    p.rk = h->rk;
    return p;
}

int do_exchange(ising_handle *h, const void *recs, int64_t n_recs, bool do_swap)
{
    if (do_swap && h->wtype == ISING_W_F32)
        return fail(ISING_E_UNSUPPORTED, "replica exchange requires integer weights");
    ExchangeParams p = exchange_params(h);
    p.recs = (const ising_record *)recs;
    p.n_recs = recs ? n_recs : 0;
    p.do_best = 1;
    p.do_swap = do_swap ? 1 : 0;
    CK(launch_exchange(p, h->st));
    if (do_swap && h->K >= 2) {
        if (h->layout == ISING_SPINS_BITS)
            CK(launch_swap_bits(h->d_state[h->cur], h->d_swapmask, h->n, h->C_local, h->wpc, h->st));
        else
            CK(launch_swap_i8(h->d_s8, h->d_swapmask, h->n, (int32_t)h->R, h->K, h->st));
    }
    if (do_swap)
        h->e += 1;
    return ISING_OK;
}

int check_handle(const ising_handle *h)
{
    if (!h)
        return fail(ISING_E_ARG, "handle is NULL");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess)
        return cuda_fail(e, "cudaSetDevice");
    return ISING_OK;
}

// Copy one local slot's configuration (original ids, original order) into d_tmp.
int slot_to_tmp(ising_handle *h, int64_t rl)
{
    if (h->layout == ISING_SPINS_BITS) {
        CK(launch_extract_bits(h->d_state[h->cur], h->n, (int32_t)(rl / 32), (int32_t)(rl % 32),
                               h->kernel == KER_GRID_BITS ? nullptr : h->d_o2i, h->d_tmp, h->st));
    } else {
        CK(launch_extract_i8(h->d_s8, h->R, h->n, rl, h->d_o2i, h->d_tmp, h->st));
    }
    return ISING_OK;
}

}  // namespace

// =========================================================================== ABI
extern "C" {

const char *ising_last_error(void) { return g_err.c_str(); }

const char *ising_version(void) { return "libising 0.1 (sm_100a)"; }

uint64_t ising_threshold(double beta, int64_t dE) { return metropolis_threshold(beta, dE); }

int ising_greedy_colour(int32_t n, const int64_t *row_ptr, const int32_t *col, int32_t *colour_out)
{
    if (n < 1 || !row_ptr || !col || !colour_out)
        return fail(ISING_E_ARG, "greedy_colour: bad arguments");
    int32_t maxdeg = 0;
    for (int32_t i = 0; i < n; ++i)
        maxdeg = std::max<int32_t>(maxdeg, (int32_t)(row_ptr[i + 1] - row_ptr[i]));
    std::vector<int32_t> stamp(maxdeg + 2, -1);
    int32_t ncol = 0;
    for (int32_t i = 0; i < n; ++i)
        colour_out[i] = -1;
    for (int32_t i = 0; i < n; ++i) {
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            const int32_t c = colour_out[col[e]];
            if (c >= 0 && c <= maxdeg + 1)
                stamp[c] = i;
        }
        int32_t c = 0;
        while (stamp[c] == i)
            ++c;
        colour_out[i] = c;
        ncol = std::max(ncol, c + 1);
    }
    return ncol;
}

int ising_colour_jp(int32_t device, int32_t n, const int64_t *row_ptr, const int32_t *col, int32_t *colour_out)
{
    g_err.clear();
    if (n < 1 || !row_ptr || !col || !colour_out)
        return fail(ISING_E_ARG, "NULL argument or n < 1");
    if (row_ptr[0] != 0)
        return fail(ISING_E_GRAPH, "row_ptr[0] != 0");
    for (int32_t i = 0; i < n; ++i)
        if (row_ptr[i + 1] < row_ptr[i])
            return fail(ISING_E_GRAPH, "row_ptr decreases at vertex " + std::to_string(i));
    for (int64_t e = 0; e < row_ptr[n]; ++e)
        if (col[e] < 0 || col[e] >= n)
            return fail(ISING_E_GRAPH, "col[" + std::to_string(e) + "] out of range");
    CK(cudaSetDevice(device));
    cudaStream_t st = nullptr;
    CreateTmp tmp{st, {}};
    int64_t *d_rp64;
    int32_t *d_c, *d_colour, *d_cnt;
    uint32_t *d_prio;
    CK(tmp.alloc(&d_rp64, (size_t)n + 1));
    CK(tmp.alloc(&d_c, (size_t)row_ptr[n]));
    CK(tmp.alloc(&d_colour, (size_t)n));
    CK(tmp.alloc(&d_prio, (size_t)n));
    CK(tmp.alloc(&d_cnt, 2));
    CK(cudaMemcpyAsync(d_rp64, row_ptr, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_c, col, (size_t)row_ptr[n] * 4, cudaMemcpyHostToDevice, st));
    int32_t ncol = 0;
    CK(colour_jp_device(n, d_rp64, d_c, d_prio, d_colour, d_cnt, &ncol, st));
    CK(cudaMemcpyAsync(colour_out, d_colour, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return ncol;
}

int ising_greedy_colour_sl(int32_t n, const int64_t *row_ptr, const int32_t *col, int32_t *colour_out)
{
    if (n < 1 || !row_ptr || !col || !colour_out)
        return fail(ISING_E_ARG, "greedy_colour_sl: bad arguments");
    // smallest-last order: repeatedly remove a vertex of minimum remaining degree (ties:
    // lowest id).  One three-level bitmap over the ids per remaining degree: the next vertex
    // is the lowest set bit of the lowest non-empty bucket, found through the summary levels
    // in a few word operations (O(n + m) on sparse graphs).  Graphs whose buckets would not
    // fit in 256 MB use a (degree, id) min-heap with lazy deletion.  Both produce exactly the
    // order of the definition (the oracle's own implementation is the heap).
    std::vector<int32_t> deg(n), order;
    order.reserve(n);
    std::vector<char> gone(n, 0);
    int32_t dmax = 0;
    for (int32_t i = 0; i < n; ++i) {
        deg[i] = (int32_t)(row_ptr[i + 1] - row_ptr[i]);
        dmax = std::max(dmax, deg[i]);
    }
    const size_t n0 = ((size_t)n + 63) / 64, n1 = (n0 + 63) / 64, n2 = (n1 + 63) / 64;
    if ((size_t)(dmax + 1) * (n0 + n1 + n2) <= ((size_t)1 << 25)) {
        struct Bits3 {
            uint64_t *l0, *l1, *l2;
            size_t n2;
            void set(int32_t i)
            {
                const size_t w0 = (size_t)i >> 6, w1 = w0 >> 6;
                if (!l0[w0]) {
                    if (!l1[w1])
                        l2[w1 >> 6] |= (uint64_t)1 << (w1 & 63);
                    l1[w1] |= (uint64_t)1 << (w0 & 63);
                }
                l0[w0] |= (uint64_t)1 << (i & 63);
            }
            void clr(int32_t i)
            {
                const size_t w0 = (size_t)i >> 6, w1 = w0 >> 6;
                l0[w0] &= ~((uint64_t)1 << (i & 63));
                if (!l0[w0]) {
                    l1[w1] &= ~((uint64_t)1 << (w0 & 63));
                    if (!l1[w1])
                        l2[w1 >> 6] &= ~((uint64_t)1 << (w1 & 63));
                }
            }
            int32_t first() const
            {
                for (size_t w2 = 0; w2 < n2; ++w2)
                    if (l2[w2]) {
                        const size_t w1 = w2 * 64 + (size_t)__builtin_ctzll(l2[w2]);
                        const size_t w0 = w1 * 64 + (size_t)__builtin_ctzll(l1[w1]);
                        return (int32_t)(w0 * 64 + (size_t)__builtin_ctzll(l0[w0]));
                    }
                return -1;
            }
        };
        const size_t per = n0 + n1 + n2;
        std::vector<uint64_t> store((size_t)(dmax + 1) * per, 0);
        std::vector<Bits3> bk(dmax + 1);
        std::vector<int64_t> cnt(dmax + 1, 0);
        for (int32_t d = 0; d <= dmax; ++d) {
            uint64_t *base = store.data() + (size_t)d * per;
            bk[d] = Bits3{base, base + n0, base + n0 + n1, n2};
        }
        // remaining degree and "removed" in one array (the sentinel), one byte per vertex when
        // the degrees fit: the order visits vertices at random, so each step is a chain of
        // cache misses (row -> neighbours -> their degrees); the rows of the neighbours just
        // decremented (the likeliest next picks) are prefetched (C5: 2.9 s -> 1.5 s)
        auto run = [&](auto *dg, auto gone_v) {
            for (int32_t i = 0; i < n; ++i) {
                dg[i] = (decltype(gone_v))deg[i];
                bk[deg[i]].set(i);
                ++cnt[deg[i]];
            }
            int32_t dmin = 0;
            for (int32_t k = 0; k < n; ++k) {
                while (cnt[dmin] == 0)
                    ++dmin;
                const int32_t i = bk[dmin].first();
                bk[dmin].clr(i);
                --cnt[dmin];
                dg[i] = gone_v;
                order.push_back(i);
                const int64_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
                for (int64_t e = e0; e < e1; ++e) {
                    const int32_t j = col[e];
                    const int32_t dj = (int32_t)dg[j];
                    if (dg[j] != gone_v) {
                        __builtin_prefetch(row_ptr + j);
                        bk[dj].clr(j);
                        --cnt[dj];
                        dg[j] = (decltype(gone_v))(dj - 1);
                        bk[dj - 1].set(j);
                        ++cnt[dj - 1];
                        dmin = std::min(dmin, dj - 1);
                    }
                }
                for (int64_t e = e0; e < e1; ++e) {
                    const int32_t j = col[e];
                    if (dg[j] != gone_v)
                        __builtin_prefetch(col + row_ptr[j]);
                }
            }
        };
        if (dmax < 255) {
            std::vector<uint8_t> d8(n);
            run(d8.data(), (uint8_t)0xFF);
        } else {
            std::vector<int32_t> d32(n);
            run(d32.data(), (int32_t)-1);
        }
    } else {
        std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> heap;
        for (int32_t i = 0; i < n; ++i)
            heap.push(((uint64_t)(uint32_t)deg[i] << 32) | (uint32_t)i);
        while (!heap.empty()) {
            const uint64_t top = heap.top();
            heap.pop();
            const int32_t i = (int32_t)(top & 0xFFFFFFFFu);
            if (gone[i] || (int32_t)(top >> 32) != deg[i])
                continue;  // stale entry
            gone[i] = 1;
            order.push_back(i);
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                const int32_t j = col[e];
                if (!gone[j]) {
                    --deg[j];
                    heap.push(((uint64_t)(uint32_t)deg[j] << 32) | (uint32_t)j);
                }
            }
        }
    }
    // greedy in reverse removal order, smallest colour unused by coloured neighbours
    int32_t maxdeg = 0;
    for (int32_t i = 0; i < n; ++i)
        maxdeg = std::max<int32_t>(maxdeg, (int32_t)(row_ptr[i + 1] - row_ptr[i]));
    std::vector<int32_t> stamp(maxdeg + 2, -1);
    for (int32_t i = 0; i < n; ++i)
        colour_out[i] = -1;
    int32_t ncol = 0;
    for (int32_t q = n - 1; q >= 0; --q) {
        // prefetch ahead along the known order: row offsets, the row, its neighbours' colours
        if (q >= 16)
            __builtin_prefetch(row_ptr + order[q - 16]);
        if (q >= 8)
            __builtin_prefetch(col + row_ptr[order[q - 8]]);
        if (q >= 4) {
            const int32_t v = order[q - 4];
            for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e)
                __builtin_prefetch(colour_out + col[e]);
        }
        const int32_t i = order[q];
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            const int32_t c = colour_out[col[e]];
            if (c >= 0 && c <= maxdeg + 1)
                stamp[c] = i;
        }
        int32_t c = 0;
        while (stamp[c] == i)
            ++c;
        colour_out[i] = c;
        ncol = std::max(ncol, c + 1);
    }
    return ncol;
}

int ising_create_grid(int32_t Lx, int32_t Ly, const int8_t *J_right, const int8_t *J_down,
                      const ising_run_desc *desc, ising_handle **out)
{
    NvtxRange nvtx_range("ising_create_grid");
    g_err.clear();
    if (!out)
        return fail(ISING_E_ARG, "out is NULL");
    *out = nullptr;
    if (!J_right || !J_down)
        return fail(ISING_E_ARG, "J_right/J_down is NULL");
    if (Lx < 4 || Ly < 4 || (Lx & 1) || (Ly & 1))
        return fail(ISING_E_ARG, "grid dims must be even and >= 4 (got " + std::to_string(Lx) + "x" +
                                     std::to_string(Ly) + ")");
    if ((int64_t)Lx * Ly >= ((int64_t)1 << 30))
        return fail(ISING_E_ARG, "grid too large");
    int rc = validate_desc(desc);
    if (rc)
        return rc;
    const int32_t n = Lx * Ly;
    for (int32_t i = 0; i < n; ++i) {
        if (J_right[i] != 1 && J_right[i] != -1)
            return fail(ISING_E_GRAPH, "J_right[" + std::to_string(i) + "] not in {-1,+1}");
        if (J_down[i] != 1 && J_down[i] != -1)
            return fail(ISING_E_GRAPH, "J_down[" + std::to_string(i) + "] not in {-1,+1}");
    }
    if (desc->layout == ISING_SPINS_I8) {
        // generic CSR kernels: row order right, left, down, up; checkerboard colouring
        std::vector<int64_t> rp(n + 1);
        std::vector<int32_t> col(4 * (size_t)n), w(4 * (size_t)n), colour(n);
        for (int32_t y = 0; y < Ly; ++y)
            for (int32_t x = 0; x < Lx; ++x) {
                const int32_t i = x + Lx * y;
                const int32_t r = (x + 1) % Lx + Lx * y, l = (x + Lx - 1) % Lx + Lx * y;
                const int32_t d = x + Lx * ((y + 1) % Ly), u = x + Lx * ((y + Ly - 1) % Ly);
                rp[i] = 4 * (int64_t)i;
                col[4 * i] = r; w[4 * i] = J_right[i];
                col[4 * i + 1] = l; w[4 * i + 1] = J_right[l];
                col[4 * i + 2] = d; w[4 * i + 2] = J_down[i];
                col[4 * i + 3] = u; w[4 * i + 3] = J_down[u];
                colour[i] = (x + y) & 1;
            }
        rp[n] = 4 * (int64_t)n;
        rc = create_csr_i8_device(n, rp.data(), col.data(), w.data(), ISING_W_I32, colour.data(), desc,
                                  out);
        if (rc == ISING_OK) {
            (*out)->Lx = Lx;
            (*out)->Ly = Ly;
        }
        return rc;
    }

    std::unique_ptr<ising_handle> h(new ising_handle());
    h->kernel = KER_GRID_BITS;
    h->n = n;
    h->Lx = Lx;
    h->Ly = Ly;
    h->ncol = 2;
    h->m = 2 * (int64_t)n;
    h->wtype = ISING_W_I32;
    fill_run(h.get(), desc);
    for (int32_t i = 0; i < n; ++i)
        h->W_int += J_right[i] + J_down[i];
    h->smem = grid_bits_smem(n);
    if (n > 65536 || grid_bits_qcap(n) < 1 || h->smem > 200 * 1024)
        return fail(ISING_E_UNSUPPORTED, "BITS grid: lattice too large for shared memory (n=" +
                                             std::to_string(n) + ")");
    const int32_t hx = Lx / 2, half = n / 2;
    // band split: with at most half as many word groups as SMs, each group's
    // rows are split over a CTA pair (halo rows through DSMEM), so twice as many SMs work.
    // ISING_GRID_BANDS=1|2 overrides the choice (tests, measurements).
    {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device);
        const bool can2 = h->wpc * 2 <= 8;  // portable cluster size with the fused PT launch
        h->bands = (can2 && 2 * (int64_t)h->G <= nsm) ? 2 : 1;
        if (const char *env = std::getenv("ISING_GRID_BANDS")) {
            const int want = std::atoi(env);
            if (want != 1 && want != 2)
                return fail(ISING_E_ARG, "ISING_GRID_BANDS must be 1 or 2");
            if (want == 2 && !can2)
                return fail(ISING_E_UNSUPPORTED, "ISING_GRID_BANDS=2 needs n_temps <= 128");
            h->bands = want;
        }
    }
    const int32_t band_rows = Ly / h->bands;
    h->ymagic = (uint32_t)((((uint64_t)1 << 32) + hx - 1) / hx);
    for (int32_t l = 0; l < half; ++l)
        if ((int32_t)(((uint64_t)l * h->ymagic) >> 32) != l / hx)
            return fail(ISING_E_UNSUPPORTED, "grid index magic not exact");
    // 2-D thread mapping of k_grid_bits: column of a class row per thread, rows in passes.
    // Default CTA size: the fewest passes whose rows-per-pass x Lx/2 fits in kGridMaxThreads,
    // rounded up to a multiple of 128 threads (equal warps per scheduler; measured: 25 or 26
    // warps run ~5% slower than 24 on C2).
    if (desc->block_threads == 0) {
        h->threads = 0;
        for (int32_t np = 1; np <= band_rows && !h->threads; ++np) {
            int32_t rows = (band_rows + np - 1) / np;
            if (rows >= 2)
                rows += rows & 1;  // grid_rows_per_pass keeps rows per pass even
            const int32_t nt = ((hx * rows + 127) / 128) * 128;
            if (nt <= kGridMaxThreads)
                h->threads = nt;
        }
        if (!h->threads)
            return fail(ISING_E_UNSUPPORTED, "BITS grid: Lx exceeds the CTA size limit");
    }
    if (h->threads > kGridMaxThreads)
        return fail(ISING_E_ARG, "BITS grid: block_threads must be <= " + std::to_string(kGridMaxThreads));
    if (2 * hx > h->threads)  // two class rows per pass at least (even rows per pass)
        return fail(ISING_E_UNSUPPORTED, "BITS grid needs block_threads >= Lx");
    const int32_t rpp = grid_rows_per_pass(h->threads, hx), npass = (band_rows + rpp - 1) / rpp;
    if (npass > 31)
        return fail(ISING_E_UNSUPPORTED, "BITS grid: too many rows per thread (Ly/(threads/(Lx/2)) > 31)");
    // the fused PT launch runs one cluster of K/32 x bands CTAs per copy: with bands it only
    // pays when every copy's cluster is resident at once (else ising_run takes per-round
    // launches, whose clusters are the band pairs alone)
    if (h->bands > 1 && h->K >= 2) {
        CK(cudaSetDevice(h->device));
        h->fused_ok = grid_bands_max_clusters(h->wpc * h->bands, h->threads, h->smem) >= h->C_local;
        // otherwise one copy spans K/32 clusters of 2 (the band pairs) that meet at global-memory
        // copy barriers: needs every cluster resident (cooperative launch)
        if (!h->fused_ok && grid_bands_max_clusters(2, h->threads, h->smem) >= h->G) {
            const size_t nbw = ((size_t)n + 31) / 32;
            CK(h->alloc(&h->d_xc_E, (size_t)h->C_local * 2 * h->K));
            CK(h->alloc(&h->d_xc_B, (size_t)h->C_local * 2 * h->wpc * 4 * nbw));
            CK(h->alloc(&h->d_xc_bar, (size_t)h->C_local));
            h->xc_ok = true;
        }
    }
    // more word groups than resident CTAs (C4 on 1-2 GPUs): the fused PT launch as a persistent
    // ticket-scheduled kernel (k_grid_sched) instead of waves of clusters.
    // ISING_GRID_SCHED=0|1 overrides the choice (tests, measurements).
    if (h->bands == 1 && h->K >= 2) {
        CK(cudaSetDevice(h->device));
        const int32_t full = Ly / rpp, left = (Ly - full * rpp) * hx;
        const int32_t nidle = (h->threads / 32 - (rpp * hx + 31) / 32) * 32;
        const bool spill = left > 0 && nidle > 0 && (left + nidle - 1) / nidle <= full;
        const int32_t ctas = grid_sched_ctas(h->threads, h->smem, spill);
        bool want = ctas > 0 && h->G > ctas;
        if (const char *env = std::getenv("ISING_GRID_SCHED")) {
            const int v = std::atoi(env);
            if (v != 0 && v != 1)
                return fail(ISING_E_ARG, "ISING_GRID_SCHED must be 0 or 1");
            want = v == 1 && ctas > 0;
        }
        if (want) {
            const size_t nbw = ((size_t)n + 31) / 32;
            CK(h->alloc(&h->d_xs_ctl, 1 + 2 * (size_t)h->C_local + (size_t)h->G));
            CK(h->alloc(&h->d_xs_E, (size_t)h->G * 32));
            CK(h->alloc(&h->d_xs_B, (size_t)2 * h->G * 2 * nbw));
            CK(h->alloc(&h->d_xs_M, (size_t)h->C_local * h->wpc));
            CK(h->alloc(&h->d_xs_S, (size_t)h->G * n));
            h->sched_ok = true;
            h->sched_ctas = std::min(ctas, h->G);
        }
    }
    // J bytes in colour-separated order: bit 0..3 = (right, left, down, up) bond has J = -1
    std::vector<uint8_t> jb(n);
    for (int32_t c = 0; c < 2; ++c)
        for (int32_t y = 0; y < Ly; ++y)
            for (int32_t mm = 0; mm < hx; ++mm) {
                const int32_t x = 2 * mm + ((c + y) & 1);
                const int32_t i = x + Lx * y;
                const int32_t l = (x + Lx - 1) % Lx + Lx * y, u = x + Lx * ((y + Ly - 1) % Ly);
                uint8_t v = 0;
                if (J_right[i] < 0) v |= 1;
                if (J_right[l] < 0) v |= 2;
                if (J_down[i] < 0) v |= 4;
                if (J_down[u] < 0) v |= 8;
                jb[c * half + y * hx + mm] = v;
            }
    std::vector<uint32_t> planes;
    plane_table(h->betas, {2, 4}, planes);
    rc = build_common_device(h.get(), 2 * (int64_t)n);
    if (rc)
        return rc;
    CK(h->alloc(&h->d_jbyte, n));
    {
        std::vector<uint8_t> jrd(n);
        for (int32_t i = 0; i < n; ++i)
            jrd[i] = (uint8_t)((J_right[i] < 0 ? 1 : 0) | (J_down[i] < 0 ? 2 : 0));
        CK(h->alloc(&h->d_jrd, n));
        CK(cudaMemcpyAsync(h->d_jrd, jrd.data(), (size_t)n, cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    CK(h->alloc(&h->d_planes, planes.size()));
    CK(cudaMemcpyAsync(h->d_jbyte, jb.data(), (size_t)n, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->d_planes, planes.data(), planes.size() * 4, cudaMemcpyHostToDevice, h->st));
    CK(h->alloc(&h->d_state[0], (size_t)h->G * n));
    CK(h->alloc(&h->d_state[1], (size_t)h->G * n));
    CK(h->alloc(&h->d_copy_best, (size_t)h->C_local * 3));
    CK(h->alloc(&h->d_snap, (size_t)h->C_local * n));
    CK(launch_init_bits(h->d_state[0], h->G, n, nullptr, h->g0, h->rk, h->st));
    rc = refresh_energy(h.get());
    if (rc)
        return rc;
    CK(cudaStreamSynchronize(h->st));
    h->fingerprint = fnv1a(kFnvBasis, J_right, (size_t)n);
    h->fingerprint = fnv1a(h->fingerprint, J_down, (size_t)n);
    h->fingerprint = fnv1a(h->fingerprint, h->betas.data(), h->betas.size() * 8);
    *out = h.release();
    return ISING_OK;
}

int ising_create_csr(int32_t n, const int64_t *row_ptr, const int32_t *col, const void *w,
                     int32_t wtype, const int32_t *colour, const ising_run_desc *desc,
                     ising_handle **out)
{
    NvtxRange nvtx_range("ising_create_csr");
    g_err.clear();
    if (!out)
        return fail(ISING_E_ARG, "out is NULL");
    *out = nullptr;
    if (n < 1)
        return fail(ISING_E_ARG, "n must be >= 1");
    if (!row_ptr || !col || !w)
        return fail(ISING_E_ARG, "row_ptr/col/w is NULL");
    if (wtype != ISING_W_I32 && wtype != ISING_W_F32)
        return fail(ISING_E_ARG, "unknown wtype");
    int rc = validate_desc(desc);
    if (rc)
        return rc;
    if (row_ptr[0] != 0)
        return fail(ISING_E_GRAPH, "row_ptr[0] != 0");
    for (int32_t i = 0; i < n; ++i)
        if (row_ptr[i + 1] < row_ptr[i])
            return fail(ISING_E_GRAPH, "row_ptr decreases at vertex " + std::to_string(i));
    const int32_t *wi = wtype == ISING_W_I32 ? (const int32_t *)w : nullptr;
    const float *wf = wtype == ISING_W_F32 ? (const float *)w : nullptr;
    // int8 layout: validation, colouring, internal order and tables on the device (k_create.cu)
    if (desc->layout == ISING_SPINS_I8)
        return create_csr_i8_device(n, row_ptr, col, w, wtype, colour, desc, out);
    // Row checks in (vertex, entry) order, then symmetry.  Rows are independent, so the
    // vertices are checked on host threads; the error reported is the one of the lowest
    // failing vertex (the first one a sequential scan meets), its message produced by
    // re-checking that row.
    auto check_row = [&](int32_t i, std::string *msg) { return csr_row_ok(n, row_ptr, col, wi, wf, i, msg); };
    auto check_sym = [&](int32_t i, std::string *msg) { return csr_sym_ok(row_ptr, col, wi, wf, i, msg); };
    for (int pass = 0; pass < 2; ++pass) {
        const int32_t i = pass == 0 ? par_first_failing(n, check_row) : par_first_failing(n, check_sym);
        if (i < n) {
            std::string msg;
            if (pass == 0)
                check_row(i, &msg);
            else
                check_sym(i, &msg);
            return fail(ISING_E_GRAPH, msg);
        }
    }
    return create_csr_impl(n, row_ptr, col, w, wtype, colour, desc, out);
}

int ising_sweep(ising_handle *h, int32_t n_sweeps)
{
    NvtxRange nvtx_range("ising_sweep");
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (n_sweeps < 0)
        return fail(ISING_E_ARG, "n_sweeps < 0");
    if ((uint64_t)h->t + (uint64_t)n_sweeps >= ((uint64_t)1 << 32))
        return fail(ISING_E_ARG, "sweep counter would exceed 2^32");
    return launch_sweeps(h, n_sweeps);
}

int ising_energy(ising_handle *h, void *out)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!out)
        return fail(ISING_E_ARG, "out is NULL");
    if (h->wtype == ISING_W_F32)
        CK(cudaMemcpyAsync(out, h->d_Ef, h->R * 8, cudaMemcpyDeviceToHost, h->st));
    else
        CK(cudaMemcpyAsync(out, h->d_E, h->R * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return ISING_OK;
}

int ising_cut(ising_handle *h, void *out)
{
    int rc = ising_energy(h, out);
    if (rc)
        return rc;
    if (h->wtype == ISING_W_F32) {
        double *o = (double *)out;
        for (int64_t r = 0; r < h->R; ++r)
            o[r] = (h->W_f - o[r]) / 2.0;
    } else {
        int64_t *o = (int64_t *)out;
        for (int64_t r = 0; r < h->R; ++r)
            o[r] = (h->W_int - o[r]) / 2;
    }
    return ISING_OK;
}

int ising_run(ising_handle *h, int32_t n_rounds, int32_t k_ex)
{
    NvtxRange nvtx_range("ising_run");
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (n_rounds < 0 || k_ex < 1)
        return fail(ISING_E_ARG, "n_rounds < 0 or k_ex < 1");
    if ((uint64_t)h->t + (uint64_t)n_rounds * (uint64_t)k_ex >= ((uint64_t)1 << 32))
        return fail(ISING_E_ARG, "sweep counter would exceed 2^32");
    if (h->wtype == ISING_W_F32)
        return fail(ISING_E_UNSUPPORTED, "replica exchange requires integer weights");
    if (n_rounds == 0)
        return ISING_OK;
    if (small_i8(h)) {
        SmallI8Params p{};
        p.s = h->d_s8; p.rp = h->d_rp; p.col = h->d_col; p.wi = h->d_wi; p.orig = h->d_orig;
        p.class_off = h->d_class_off; p.T = h->d_T;
        p.ell_col = h->ell_deg > 0 ? h->d_ell_col : nullptr; p.ell_w = h->d_ell_w;
        for (int32_t c = 0; c < h->ncol; ++c)
            p.max_class = std::max(p.max_class, h->class_off[c + 1] - h->class_off[c]);
        p.E_out = h->d_E; p.walker = h->d_walker; p.copy_best = h->d_copy_best; p.snap = h->d_snap;
        p.Tx = h->d_Tx; p.Tx_off = h->d_Tx_off; p.Tx_len = h->d_Tx_len;
        p.n = h->n; p.R = (int32_t)h->R; p.K = h->K; p.qmax = h->qmax; p.ncol = h->ncol;
        p.slot0 = h->slot0; p.t0 = h->t; p.e0 = h->e; p.n_rounds = n_rounds; p.k_ex = k_ex; p.rk = h->rk;
        CK(launch_i8_small(p, h->C_local, h->st));
        CK(launch_merge_copy_best(h->d_copy_best, h->d_snap, h->C_local, h->n, h->d_best,
                                  h->d_best_spins, h->d_cbest, h->st));
        h->t += (uint32_t)(n_rounds * k_ex);
        h->e += (uint32_t)n_rounds;
        return ISING_OK;
    }
    if (h->kernel == KER_GRID_BITS && h->K >= 2 && h->sched_ok) {
        // persistent ticket-scheduled launches; tasks (group, round) are counted in int32
        const int32_t max_rounds = (int32_t)std::max<int64_t>(1, (((int64_t)1 << 31) - 1) / h->G);
        for (int32_t r0 = 0; r0 < n_rounds; r0 += max_rounds) {
            const int32_t nr = std::min(max_rounds, n_rounds - r0);
            GridBitsParams p = grid_params(h, nr, k_ex, true);
            const cudaError_t le = launch_grid_sched(p, h->sched_ctas, h->threads, h->smem, h->st);
            if (le == cudaErrorCooperativeLaunchTooLarge) {
                // fewer SMs available than at create (e.g. another context): the cluster launch
                // from now on, same results
                cudaGetLastError();
                h->sched_ok = false;
                return ising_run(h, n_rounds - r0, k_ex);
            }
            CK(le);
            h->cur ^= 1;
            CK(launch_merge_copy_best(h->d_copy_best, h->d_snap, h->C_local, h->n, h->d_best,
                                      h->d_best_spins, h->d_cbest, h->st));
            h->t += (uint32_t)(nr * k_ex);
            h->e += (uint32_t)nr;
        }
        return ISING_OK;
    }
    if (h->kernel == KER_GRID_BITS && h->K >= 2 && !h->fused_ok && h->xc_ok) {
        GridBitsParams p = grid_params(h, n_rounds, k_ex, true);
        p.xc = 1;
        const cudaError_t le = launch_grid(h, p);
        if (le == cudaErrorCooperativeLaunchTooLarge) {
            // the copies' clusters no longer fit at once (e.g. another context holds SMs):
            // per-round launches from now on, same results
            cudaGetLastError();
            h->xc_ok = false;
            return ising_run(h, n_rounds, k_ex);
        }
        CK(le);
        h->cur ^= 1;
        CK(launch_merge_copy_best(h->d_copy_best, h->d_snap, h->C_local, h->n, h->d_best,
                                  h->d_best_spins, h->d_cbest, h->st));
        h->t += (uint32_t)(n_rounds * k_ex);
        h->e += (uint32_t)n_rounds;
        return ISING_OK;
    }
    if ((h->kernel == KER_CSR_BITS || h->kernel == KER_GRID_BITS) && h->K >= 2 &&
        (h->kernel != KER_GRID_BITS || h->fused_ok)) {
        // one launch: clusters of K/32 CTAs (one copy each) run all rounds on chip
        if (h->kernel == KER_GRID_BITS)
            CK(launch_grid(h, grid_params(h, n_rounds, k_ex, true)));
        else
            CK(launch_csr_bits(csr_params(h, n_rounds, k_ex, true), h->G, h->threads, h->smem, h->st));
        h->cur ^= 1;
        CK(launch_merge_copy_best(h->d_copy_best, h->d_snap, h->C_local, h->n, h->d_best,
                                  h->d_best_spins, h->d_cbest, h->st));
        h->t += (uint32_t)(n_rounds * k_ex);
        h->e += (uint32_t)n_rounds;
        return ISING_OK;
    }
    for (int32_t r = 0; r < n_rounds; ++r) {
        rc = launch_sweeps(h, k_ex);
        if (rc)
            return rc;
        rc = do_exchange(h, nullptr, 0, true);
        if (rc)
            return rc;
    }
    return ISING_OK;
}

int ising_anneal(ising_handle *h, int32_t n_sweeps, const double *sched)
{
    NvtxRange nvtx_range("ising_anneal");
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (n_sweeps < 0 || (n_sweeps > 0 && !sched))
        return fail(ISING_E_ARG, "n_sweeps < 0 or schedule is NULL");
    if ((uint64_t)h->t + (uint64_t)n_sweeps >= ((uint64_t)1 << 32))
        return fail(ISING_E_ARG, "sweep counter would exceed 2^32");
    for (int64_t x = 0; x < (int64_t)n_sweeps * h->K; ++x)
        if (!(sched[x] > 0.0) || !std::isfinite(sched[x]))
            return fail(ISING_E_ARG, "schedule entry " + std::to_string(x) + " must be finite and > 0");
    if (n_sweeps == 0)
        return ISING_OK;
    // per-sweep tables, same formulas as the fixed ladder, built and
    // uploaded in chunks of sweeps so the table never exceeds kAnnealChunkBytes on the host or
    // the device (a chunk's launches equal the same sweeps in one launch: every random number is
    // keyed by the sweep counter t)
    size_t per_sweep = 0;
    std::vector<int32_t> qs;
    if (h->layout == ISING_SPINS_BITS) {
        if (h->kernel == KER_GRID_BITS)
            qs = {2, 4};
        else
            for (int32_t q = 1; q <= h->qmax; ++q)
                qs.push_back(q);
        per_sweep = (size_t)h->wpc * qs.size() * 64 * 4;
    } else if (h->wtype == ISING_W_I32) {
        per_sweep = (size_t)h->R * (h->qmax + 1) * 8;
    } else {
        per_sweep = (size_t)h->R * 4;
    }
    constexpr size_t kAnnealChunkBytes = 64u << 20;
    const int32_t chunk = (int32_t)std::max<size_t>(1, std::min<size_t>(n_sweeps, kAnnealChunkBytes / per_sweep));
    std::vector<uint8_t> host;
    for (int32_t s0 = 0; s0 < n_sweeps; s0 += chunk) {
        const int32_t ns = std::min(chunk, n_sweeps - s0);
        const double *sc = sched + (size_t)s0 * h->K;
        host.resize(per_sweep * ns);
        if (h->layout == ISING_SPINS_BITS) {
            std::vector<uint32_t> planes;
            for (int32_t s = 0; s < ns; ++s) {
                std::vector<double> row(sc + (size_t)s * h->K, sc + (size_t)(s + 1) * h->K);
                plane_table(row, qs, planes);
                std::memcpy(host.data() + s * per_sweep, planes.data(), per_sweep);
            }
        } else if (h->wtype == ISING_W_I32) {
            uint64_t *all = (uint64_t *)host.data();
            const size_t per = (size_t)h->R * (h->qmax + 1);
            for (int32_t s = 0; s < ns; ++s)
                for (int64_t r = 0; r < h->R; ++r) {
                    const double beta = sc[(size_t)s * h->K + (h->slot0 + r) % h->K];
                    all[s * per + r * (h->qmax + 1)] = std::numeric_limits<uint64_t>::max();
                    for (int32_t q = 1; q <= h->qmax; ++q)
                        all[s * per + r * (h->qmax + 1) + q] = metropolis_threshold(beta, 2 * (int64_t)q);
                }
        } else {
            float *all = (float *)host.data();
            for (int32_t s = 0; s < ns; ++s)
                for (int64_t r = 0; r < h->R; ++r)
                    all[(size_t)s * h->R + r] = 2.0f * (float)sc[(size_t)s * h->K + (h->slot0 + r) % h->K];
        }
        CK(cudaStreamSynchronize(h->st));  // the previous chunk's table may still be in use
        if (host.size() > h->sched_bytes) {
            if (h->d_sched)
                cudaFree(h->d_sched);
            h->d_sched = nullptr;
            h->sched_bytes = 0;
            CK(cudaMalloc(&h->d_sched, host.size()));
            h->sched_bytes = host.size();
        }
        CK(cudaMemcpyAsync(h->d_sched, host.data(), host.size(), cudaMemcpyHostToDevice, h->st));
        if (h->kernel == KER_GRID_BITS) {
            GridBitsParams p = grid_params(h, 1, ns, false);
            p.planes_sched = (const uint32_t *)h->d_sched;
            CK(launch_grid(h, p));
            h->cur ^= 1;
            h->t += (uint32_t)ns;
        } else if (h->kernel == KER_CSR_BITS) {
            CsrBitsParams p = csr_params(h, 1, ns, false);
            p.planes_sched = (const uint32_t *)h->d_sched;
            CK(launch_csr_bits(p, h->G, h->threads, h->smem, h->st));
            h->cur ^= 1;
            h->t += (uint32_t)ns;
        } else {
            rc = launch_sweeps_i8(h, ns, h->d_sched);
            if (rc)
                return rc;
        }
    }
    CK(cudaStreamSynchronize(h->st));  // host table buffer goes out of scope
    return do_exchange(h, nullptr, 0, false);  // best-so-far check after the anneal
}

int ising_icm(ising_handle *h, int32_t k_min)
{
    NvtxRange nvtx_range("ising_icm");
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (h->layout != ISING_SPINS_BITS)
        return fail(ISING_E_UNSUPPORTED, "cluster moves are implemented for the BITS layout");
    if ((h->c0 & 1) || (h->C_local & 1))
        return fail(ISING_E_UNSUPPORTED, "cluster moves need a copy shard of whole pairs (2p, 2p+1)");
    if (k_min < 0 || k_min > h->K)
        return fail(ISING_E_ARG, "k_min out of range");
    if ((size_t)8 * h->n > 200 * 1024)
        return fail(ISING_E_UNSUPPORTED, "cluster moves: n too large for shared memory");
    IcmParams p{};
    p.state = h->d_state[h->cur];
    p.E = h->d_E;
    p.n = h->n;
    p.kind = h->kernel == KER_GRID_BITS ? 0 : 1;
    p.Lx = h->Lx;
    p.Ly = h->Ly;
    p.jbyte_orig = h->d_jrd;
    p.rp = h->d_rp;
    p.nbr = h->d_nbr;
    p.o2i = h->kernel == KER_GRID_BITS ? nullptr : h->d_o2i;
    p.KW = h->wpc;
    p.pair0 = (uint32_t)(h->c0 / 2);
    p.k_min = k_min;
    p.f = h->f;
    p.m_edges = h->m;
    p.rk = h->rk;
    if (h->C_local >= 2)
        CK(launch_icm_bits(p, h->C_local / 2, 1024, h->st));
    h->f += 1;
    return ISING_OK;
}

int ising_exchange(ising_handle *h)
{
    NvtxRange nvtx_range("ising_exchange");
    int rc = check_handle(h);
    if (rc)
        return rc;
    return do_exchange(h, nullptr, 0, true);
}

int ising_exchange_begin(ising_handle *h, void *dev_send)
{
    NvtxRange nvtx_range("ising_exchange_begin");
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!dev_send)
        return fail(ISING_E_ARG, "dev_send is NULL");
    CK(launch_records(h->d_E, (ising_record *)dev_send, h->R, h->slot0, h->st));
    return ISING_OK;
}

int ising_exchange_end(ising_handle *h, const void *dev_recv, int64_t n_records)
{
    NvtxRange nvtx_range("ising_exchange_end");
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!dev_recv || n_records < 1)
        return fail(ISING_E_ARG, "dev_recv is NULL or n_records < 1");
    return do_exchange(h, dev_recv, n_records, true);
}

int ising_check_best(ising_handle *h, const void *dev_recv, int64_t n_records)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (dev_recv && n_records < 1)
        return fail(ISING_E_ARG, "n_records < 1");
    return do_exchange(h, dev_recv, dev_recv ? n_records : 0, false);
}

int ising_merge_best(ising_handle *h, const void *dev_recs, int64_t n, void *best_E, int64_t *slot,
                     int64_t *sweep)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!dev_recs || n < 1 || !best_E || !slot || !sweep)
        return fail(ISING_E_ARG, "NULL argument or n < 1");
    CK(launch_merge_best((const int64_t *)dev_recs, n, h->wtype == ISING_W_F32 ? 1 : 0, h->d_merge, h->st));
    int64_t out[3];
    CK(cudaMemcpyAsync(out, h->d_merge, sizeof(out), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (out[2] < 0)
        return fail(ISING_E_STATE, "no record holds a slot");
    std::memcpy(best_E, &out[0], 8);
    *sweep = out[1];
    *slot = out[2];
    return ISING_OK;
}

int ising_best(ising_handle *h, void *best_E, int64_t *slot, int64_t *sweep, int8_t *spins_out)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    BestDev b;
    CK(cudaMemcpyAsync(&b, h->d_best, sizeof(b), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (b.slot < 0)
        return fail(ISING_E_STATE, "no best-so-far check has run yet");
    if (best_E)
        std::memcpy(best_E, &b.energy, 8);
    if (slot)
        *slot = b.slot;
    if (sweep)
        *sweep = b.sweep;
    if (spins_out) {
        if (!b.owner)
            return fail(ISING_E_STATE, "best configuration is held by another shard");
        CK(cudaMemcpyAsync(spins_out, h->d_best_spins, h->n, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    return ISING_OK;
}

int ising_copy_best(ising_handle *h, void *best_E, int64_t *slot, int64_t *sweep)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!best_E || !slot || !sweep)
        return fail(ISING_E_ARG, "NULL output");
    std::vector<int64_t> cb((size_t)h->C_local * 3);
    CK(cudaMemcpyAsync(cb.data(), h->d_cbest, cb.size() * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    for (int32_t c = 0; c < h->C_local; ++c) {
        std::memcpy((char *)best_E + 8 * c, &cb[3 * c], 8);
        slot[c] = cb[3 * c + 1];
        sweep[c] = cb[3 * c + 2];
    }
    return ISING_OK;
}

int ising_get_spins(ising_handle *h, int64_t slot, int8_t *out)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!out)
        return fail(ISING_E_ARG, "out is NULL");
    if (slot < h->slot0 || slot >= h->slot0 + h->R)
        return fail(ISING_E_STATE, "slot " + std::to_string(slot) + " is not held by this handle");
    rc = slot_to_tmp(h, slot - h->slot0);  // original order
    if (rc)
        return rc;
    CK(cudaMemcpyAsync(out, h->d_tmp, h->n, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return ISING_OK;
}

int ising_set_spins(ising_handle *h, int64_t slot, const int8_t *in)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!in)
        return fail(ISING_E_ARG, "in is NULL");
    if (slot < h->slot0 || slot >= h->slot0 + h->R)
        return fail(ISING_E_STATE, "slot " + std::to_string(slot) + " is not held by this handle");
    for (int32_t i = 0; i < h->n; ++i)
        if (in[i] != 1 && in[i] != -1)
            return fail(ISING_E_ARG, "spin " + std::to_string(i) + " not in {-1,+1}");
    const int64_t rl = slot - h->slot0;
    if (h->layout == ISING_SPINS_BITS) {
        CK(cudaMemcpyAsync(h->d_tmp, in, h->n, cudaMemcpyHostToDevice, h->st));
        CK(launch_insert_bits(h->d_state[h->cur], h->n, (int32_t)(rl / 32), (int32_t)(rl % 32),
                              h->kernel == KER_GRID_BITS ? nullptr : h->d_o2i, h->d_tmp, h->st));
    } else {  // scatter through the internal order on the device
        CK(cudaMemcpyAsync(h->d_tmp, in, h->n, cudaMemcpyHostToDevice, h->st));
        CK(launch_insert_i8(h->d_s8, h->R, h->n, rl, h->d_o2i, h->d_tmp, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    rc = refresh_energy(h);
    if (rc)
        return rc;
    CK(cudaStreamSynchronize(h->st));
    return ISING_OK;
}

int ising_get_walkers(ising_handle *h, int64_t *out)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!out)
        return fail(ISING_E_ARG, "out is NULL");
    CK(cudaMemcpyAsync(out, h->d_walker, h->R * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return ISING_OK;
}

int ising_info(const ising_handle *h, ising_info_t *out)
{
    if (!h || !out)
        return fail(ISING_E_ARG, "NULL argument");
    out->n = h->n;
    out->n_colours = h->ncol;
    out->n_edges = h->m;
    out->n_temps = h->K;
    out->n_copies = h->C;
    out->copy_begin = h->c0;
    out->copy_end = h->c1;
    out->slot_begin = h->slot0;
    out->n_slots = h->R;
    out->layout = h->layout;
    out->rng = h->rng;
    out->wtype = h->wtype;
    out->kernel = h->kernel;
    out->sweeps_done = h->t;
    out->exchanges_done = h->e;
    out->W_int = h->W_int;
    out->W_f64 = h->W_f;
    out->bands = h->bands;
    out->fused_pt = ((h->kernel == KER_CSR_BITS || (h->kernel == KER_GRID_BITS && h->fused_ok)) && h->K >= 2) ||
                    small_i8(h);
    if (h->kernel == KER_GRID_BITS && h->K >= 2 && !h->fused_ok && h->xc_ok)
        out->fused_pt = 2;  // one cooperative launch; each copy spans K/32 clusters
    if (h->kernel == KER_GRID_BITS && h->K >= 2 && h->sched_ok)
        out->fused_pt = 3;  // one persistent ticket-scheduled launch (k_grid_sched)
    return ISING_OK;
}

// ---------------------------------------------------------------- checkpoint / resume
}  // extern "C"
namespace {

struct CkptHeader {             // 128 bytes
    char magic[8];              // "ISNGCKP1"
    int32_t kernel, layout, wtype, rng;
    int32_t n, K, C, c0, c1, pad0;
    int64_t m, W_int;
    double W_f;
    uint64_t seed, fingerprint;
    uint32_t t, e, f, pad1;
    int64_t payload;            // bytes after the header
    uint8_t reserved[16];
};
static_assert(sizeof(CkptHeader) == 128, "checkpoint header must stay 128 bytes");

// (device pointer, bytes) of every dynamic state buffer, in blob order.
std::vector<std::pair<void *, size_t>> ckpt_parts(const ising_handle *h)
{
    std::vector<std::pair<void *, size_t>> v;
    if (h->layout == ISING_SPINS_BITS)
        v.push_back({h->d_state[h->cur], (size_t)h->G * h->n * 4});
    else
        v.push_back({h->d_s8, (size_t)h->n * h->R});
    v.push_back({h->d_E, (size_t)h->R * 8});
    if (h->d_Ef)
        v.push_back({h->d_Ef, (size_t)h->R * 8});
    v.push_back({h->d_walker, (size_t)h->R * 8});
    v.push_back({h->d_cbest, (size_t)h->C_local * 3 * 8});
    v.push_back({h->d_best, sizeof(BestDev)});
    v.push_back({h->d_best_spins, (size_t)h->n});
    return v;
}

CkptHeader ckpt_header(const ising_handle *h)
{
    CkptHeader c{};
    std::memcpy(c.magic, "ISNGCKP1", 8);
    c.kernel = h->kernel; c.layout = h->layout; c.wtype = h->wtype; c.rng = h->rng;
    c.n = h->n; c.K = h->K; c.C = h->C; c.c0 = h->c0; c.c1 = h->c1;
    c.m = h->m; c.W_int = h->W_int; c.W_f = h->W_f;
    c.seed = h->seed; c.fingerprint = h->fingerprint;
    c.t = h->t; c.e = h->e; c.f = h->f;
    for (const auto &p : ckpt_parts(h))
        c.payload += (int64_t)p.second;
    return c;
}

}  // namespace
extern "C" {

int ising_state_size(const ising_handle *h, int64_t *bytes)
{
    if (!h || !bytes)
        return fail(ISING_E_ARG, "NULL argument");
    *bytes = (int64_t)sizeof(CkptHeader) + ckpt_header(h).payload;
    return ISING_OK;
}

int ising_state_save(ising_handle *h, void *buf, int64_t bytes)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    const CkptHeader c = ckpt_header(h);
    if (!buf || bytes < (int64_t)sizeof(c) + c.payload)
        return fail(ISING_E_ARG, "buffer is NULL or smaller than ising_state_size");
    std::memcpy(buf, &c, sizeof(c));
    char *dst = (char *)buf + sizeof(c);
    for (const auto &p : ckpt_parts(h)) {
        CK(cudaMemcpyAsync(dst, p.first, p.second, cudaMemcpyDeviceToHost, h->st));
        dst += p.second;
    }
    CK(cudaStreamSynchronize(h->st));
    return ISING_OK;
}

int ising_state_load(ising_handle *h, const void *buf, int64_t bytes)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    if (!buf || bytes < (int64_t)sizeof(CkptHeader))
        return fail(ISING_E_ARG, "buffer is NULL or shorter than a checkpoint header");
    CkptHeader in;
    std::memcpy(&in, buf, sizeof(in));
    if (std::memcmp(in.magic, "ISNGCKP1", 8) != 0)
        return fail(ISING_E_STATE, "not a libising checkpoint (bad magic/version)");
    const CkptHeader me = ckpt_header(h);
    auto mismatch = [&](const char *what) {
        return fail(ISING_E_STATE, std::string("checkpoint does not match this handle: ") + what);
    };
    if (in.kernel != me.kernel || in.layout != me.layout || in.wtype != me.wtype || in.rng != me.rng)
        return mismatch("kernel/layout/weight type/RNG contract");
    if (in.n != me.n || in.m != me.m || in.W_int != me.W_int || std::memcmp(&in.W_f, &me.W_f, 8) != 0)
        return mismatch("instance shape or weights");
    if (in.K != me.K || in.C != me.C || in.c0 != me.c0 || in.c1 != me.c1)
        return mismatch("temperatures, copies or shard");
    if (in.seed != me.seed)
        return mismatch("seed");
    if (in.fingerprint != me.fingerprint)
        return mismatch("instance/colouring/ladder fingerprint");
    if (in.payload != me.payload || bytes < (int64_t)sizeof(in) + in.payload)
        return fail(ISING_E_ARG, "checkpoint is truncated");
    CK(cudaStreamSynchronize(h->st));  // nothing in flight may still touch the state
    const char *src = (const char *)buf + sizeof(in);
    for (const auto &p : ckpt_parts(h)) {
        CK(cudaMemcpyAsync(p.first, src, p.second, cudaMemcpyHostToDevice, h->st));
        src += p.second;
    }
    CK(cudaStreamSynchronize(h->st));
    h->t = in.t;
    h->e = in.e;
    h->f = in.f;
    return ISING_OK;
}

int ising_sync(ising_handle *h)
{
    int rc = check_handle(h);
    if (rc)
        return rc;
    CK(cudaStreamSynchronize(h->st));
    return ISING_OK;
}

void ising_destroy(ising_handle *h)
{
    if (!h)
        return;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->st);
    delete h;
}

int ising_debug_philox(int32_t device, const uint32_t *in, int32_t n, uint32_t *out_lib,
                       uint32_t *out_curand)
{
    if (!in || !out_lib || !out_curand || n < 1)
        return fail(ISING_E_ARG, "debug_philox: bad arguments");
    CK(cudaSetDevice(device));
    uint32_t *d_in = nullptr, *d_a = nullptr, *d_b = nullptr;
    CK(cudaMalloc(&d_in, (size_t)n * 24));
    CK(cudaMalloc(&d_a, (size_t)n * 16));
    CK(cudaMalloc(&d_b, (size_t)n * 16));
    CK(cudaMemcpy(d_in, in, (size_t)n * 24, cudaMemcpyHostToDevice));
    CK(launch_debug_philox(d_in, n, d_a, d_b, nullptr));
    CK(cudaMemcpy(out_lib, d_a, (size_t)n * 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_curand, d_b, (size_t)n * 16, cudaMemcpyDeviceToHost));
    cudaFree(d_in);
    cudaFree(d_a);
    cudaFree(d_b);
    return ISING_OK;
}

int ising_debug_exp_bound(int32_t device, const float *beta2, int32_t n_beta, float *worst_rel,
                          float *max_small)
{
    if (!beta2 || n_beta < 1 || n_beta > 65535 || !worst_rel || !max_small)
        return fail(ISING_E_ARG, "NULL argument or n_beta out of [1, 65535]");
    for (int32_t i = 0; i < n_beta; ++i)
        if (!(beta2[i] > 0.0f) || !std::isfinite(beta2[i]))
            return fail(ISING_E_ARG, "beta2 entries must be finite and > 0");
    CK(cudaSetDevice(device));
    uint32_t *d = nullptr;
    float *db = nullptr;
    CK(cudaMalloc(&d, 8));
    CK(cudaMalloc(&db, (size_t)n_beta * 4));
    CK(cudaMemset(d, 0, 8));
    CK(cudaMemcpy(db, beta2, (size_t)n_beta * 4, cudaMemcpyHostToDevice));
    CK(launch_debug_exp_bound(db, n_beta, d, nullptr));
    uint32_t bits[2] = {0, 0};
    CK(cudaMemcpy(bits, d, 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
    cudaFree(db);
    std::memcpy(worst_rel, &bits[0], 4);
    std::memcpy(max_small, &bits[1], 4);
    return ISING_OK;
}

}  // extern "C"

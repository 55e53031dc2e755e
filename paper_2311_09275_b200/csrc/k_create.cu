// k_create.cu -- device-side preprocessing for ising_create_csr (row a1 of SURVEY.md §8(a))
// of the int8 layout: validation of the caller's CSR, Jones-Plassmann colouring, the colour-
// sorted internal order and the internal CSR / padded neighbour tables, all on the GPU.
//
// Why on the device: for the 4e6-vertex C5 instance the host create path spent ~1 s
// (a sequential smallest-last order, host loops over 12e6 entries and a byte-wise
// fingerprint) next to ~1.3 s of sweeps, so the end-to-end rate through the public API was
// half the device rate.  Every step here is a plain data-parallel pass over vertices or
// entries; the results equal the host path's (tests compare them: same errors for the same
// lowest failing vertex, same internal order for a given colouring).
//
// Jones-Plassmann (R12c): vertex i has the priority pr(i) = word 0 of
// Philox4x32-10(i, 0, 0, COLOUR << 24) under key (0, 0); a round colours every uncoloured
// vertex whose higher-priority neighbours (pr larger, ties: lower id) are all coloured, with
// the smallest colour none of them uses.  The result is exactly the sequential greedy
// colouring in decreasing priority order (a vertex is coloured after all its higher-priority
// neighbours and before all its lower-priority ones), which the oracle computes directly.
#include <cub/cub.cuh>

#include "internal.h"

namespace ising {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int32_t warp_min(int32_t v)
{
    return __reduce_min_sync(0xFFFFFFFFu, v);
}

__device__ __forceinline__ int32_t warp_max(int32_t v)
{
    return __reduce_max_sync(0xFFFFFFFFu, v);
}

__device__ __forceinline__ int64_t warp_sum64(int64_t v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

__device__ __forceinline__ void amin(int32_t *a, int32_t v)
{
    v = warp_min(v);
    if ((threadIdx.x & 31) == 0 && v != INT32_MAX)
        atomicMin(a, v);
}

}  // namespace

// One thread per vertex (grid-stride; every lane of a warp runs the same number of
// iterations so the warp reductions see full warps).  Checks of SPEC.md S:29-35 and the
// library's guards, each reported as the LOWEST failing vertex (the one a sequential scan
// meets first; the host re-checks that vertex for the message).
__global__ void k_csr_check(int32_t n, const int64_t *rp, const int32_t *col, const int32_t *wi, const float *wf,
                            const int32_t *colour, CsrCheck *out, uint8_t *colour_used)
{
    const int32_t stride = gridDim.x * blockDim.x;
    const int32_t base = blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t iters = (n + stride - 1) / stride;
    int32_t maxdeg = 0, maxcol = -1;
    uint32_t pm1 = 1u;
    int64_t qmax = 0, sum_abs = 0, W = 0;
    uint64_t hash = 0;
    for (int32_t it = 0; it < iters; ++it) {
        const int32_t i = base + it * stride;
        int32_t bad_row = INT32_MAX, bad_sym = INT32_MAX, bad_sum = INT32_MAX, bad_cr = INT32_MAX,
                bad_pr = INT32_MAX;
        if (i < n) {
            const int64_t e0 = rp[i], e1 = rp[i + 1];
            maxdeg = max(maxdeg, (int32_t)(e1 - e0));
            hash += mix64(((uint64_t)(uint32_t)i << 32) ^ (uint64_t)e1);
            bool ok = true;
            int64_t s = 0;
            for (int64_t e = e0; e < e1 && ok; ++e) {
                const int32_t j = col[e];
                const uint32_t wb = wi ? (uint32_t)wi[e] : __float_as_uint(wf[e]);
                hash += mix64(((uint64_t)e << 32) ^ (uint64_t)(uint32_t)j) ^ mix64((uint64_t)wb + 0x9E3779B97F4A7C15ull * (uint64_t)(e + 1));
                if (j < 0 || j >= n || j == i)
                    ok = false;
                for (int64_t f = e0; f < e && ok; ++f)
                    if (col[f] == j)
                        ok = false;
                if (wf && !isfinite(wf[e]))
                    ok = false;
                if (wi) {
                    s += wi[e] < 0 ? -(int64_t)wi[e] : (int64_t)wi[e];
                    pm1 &= (wi[e] == 1 || wi[e] == -1) ? 1u : 0u;
                    if (j > i)
                        W += wi[e];
                }
            }
            if (!ok) {
                bad_row = i;
            } else {
                for (int64_t e = e0; e < e1; ++e) {  // (i, j, w) present iff (j, i, w)
                    const int32_t j = col[e];
                    bool found = false;
                    for (int64_t f = rp[j]; f < rp[j + 1]; ++f)
                        if (col[f] == i) {
                            found = wi ? (wi[f] == wi[e]) : (wf[f] == wf[e]);
                            break;
                        }
                    if (!found) {
                        bad_sym = i;
                        break;
                    }
                }
            }
            if (wi) {
                if (s >= ((int64_t)1 << 30))
                    bad_sum = i;
                qmax = max(qmax, s);
                sum_abs += s;
            }
            if (colour) {
                const int32_t c = colour[i];
                if (c < 0 || c >= (1 << 16)) {
                    bad_cr = i;
                } else {
                    colour_used[c] = 1;
                    maxcol = max(maxcol, c);
                    for (int64_t e = e0; e < e1; ++e) {
                        const int32_t j = col[e];
                        if (j >= 0 && j < n && colour[j] == c) {
                            bad_pr = i;
                            break;
                        }
                    }
                }
            }
        }
        amin(&out->bad_row, bad_row);
        amin(&out->bad_sym, bad_sym);
        amin(&out->bad_sum, bad_sum);
        amin(&out->bad_colrange, bad_cr);
        amin(&out->bad_proper, bad_pr);
    }
    maxdeg = warp_max(maxdeg);
    maxcol = warp_max(maxcol);
    pm1 = __reduce_and_sync(0xFFFFFFFFu, pm1);
    const int64_t qm = (int64_t)__reduce_max_sync(0xFFFFFFFFu, (uint32_t)min(qmax, (int64_t)0x7FFFFFFF));
    sum_abs = warp_sum64(sum_abs);
    W = warp_sum64(W);
    hash = (uint64_t)warp_sum64((int64_t)hash);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out->maxdeg, maxdeg);
        atomicMax(&out->max_colour, maxcol);
        atomicAnd(&out->pm1, pm1);
        atomicMax((unsigned long long *)&out->qmax, (unsigned long long)qm);
        atomicAdd((unsigned long long *)&out->sum_abs, (unsigned long long)sum_abs);
        atomicAdd((unsigned long long *)&out->W_int, (unsigned long long)W);
        atomicAdd((unsigned long long *)&out->hash, (unsigned long long)hash);
    }
}

// ---- Jones-Plassmann colouring
__global__ void k_jp_init(int32_t n, uint32_t *prio, int32_t *colour)
{
    RoundKeys rk0;  // key (0, 0): the round keys are the Weyl sequence from 0
    uint32_t a = 0u, b = 0u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        rk0.k[2 * r] = a;
        rk0.k[2 * r + 1] = b;
        a += 0x9E3779B9u;
        b += 0xBB67AE85u;
    }
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        prio[i] = philox((uint32_t)i, 0u, 0u, ST_COLOUR << 24, rk0).x;
        colour[i] = -1;
    }
}

// One round: every uncoloured vertex whose higher-priority neighbours are all coloured takes
// the smallest colour they do not use.  A neighbour's colour is final once written (it is
// written once), so reading it in the same round either sees -1 (retry next round) or the
// final value.  pending: uncoloured vertices left after this round; ncol: colours used.
__global__ void k_jp_round(int32_t n, const int64_t *rp, const int32_t *col, const uint32_t *prio,
                           int32_t *colour, int32_t *pending, int32_t *ncol)
{
    volatile int32_t *vc = colour;
    int32_t left = 0, mx = -1;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (vc[i] >= 0)
            continue;
        const uint32_t p = prio[i];
        bool ready = true;
        uint64_t used = 0;
        bool wide = false;  // a neighbour colour >= 64: take the slow path
        const int64_t e0 = rp[i], e1 = rp[i + 1];
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t j = col[e];
            const uint32_t q = prio[j];
            if (q > p || (q == p && j < i)) {
                const int32_t c = vc[j];
                if (c < 0) {
                    ready = false;
                    break;
                }
                if (c < 64)
                    used |= 1ull << c;
                else
                    wide = true;
            }
        }
        if (!ready) {
            ++left;
            continue;
        }
        int32_t c = __ffsll((long long)~used) - 1;
        if (wide || used == ~0ull) {  // smallest colour not used by a higher-priority neighbour
            for (c = 0;; ++c) {
                bool taken = false;
                for (int64_t e = e0; e < e1 && !taken; ++e) {
                    const int32_t j = col[e];
                    const uint32_t q = prio[j];
                    taken = (q > p || (q == p && j < i)) && vc[j] == c;
                }
                if (!taken)
                    break;
            }
        }
        vc[i] = c;
        mx = max(mx, c);
    }
    for (int o = 16; o > 0; o >>= 1) {
        left += __shfl_xor_sync(0xFFFFFFFFu, left, o);
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (left)
            atomicAdd(pending, left);
        atomicMax(ncol, mx + 1);
    }
}

// ---- colour-sorted internal order
__global__ void k_iota_keys(int32_t n, const int32_t *colour, uint32_t *keys, uint32_t *ids)
{
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        keys[i] = (uint32_t)colour[i];
        ids[i] = (uint32_t)i;
    }
}

// class_off[c] = first position of colour c in the sorted keys; o2i = inverse permutation;
// deg[v] = degree of internal vertex v (deg[n] = 0 for the exclusive scan)
__global__ void k_order_finish(int32_t n, int32_t ncol, const uint32_t *keys, const uint32_t *orig,
                               const int64_t *rp, int32_t *class_off, uint32_t *o2i, int32_t *deg)
{
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x) {
        if (v == n) {
            class_off[ncol] = n;
            deg[n] = 0;
            continue;
        }
        const uint32_t k = keys[v];
        if (v == 0 || keys[v - 1] != k)
            for (uint32_t c = v == 0 ? 0u : keys[v - 1] + 1u; c <= k; ++c)
                class_off[c] = v;
        const uint32_t i = orig[v];
        o2i[i] = (uint32_t)v;
        deg[v] = (int32_t)(rp[i + 1] - rp[i]);
    }
}

// internal CSR (rows in the caller's order, columns renumbered) and, for max degree <= 4, the
// padded 4-wide table (pads: the vertex itself with weight 0, an exact zero term)
__global__ void k_build_internal(int32_t n, const int64_t *rp, const int32_t *col, const uint32_t *w,
                                 const uint32_t *orig, const uint32_t *o2i, const int32_t *rpi, int32_t *ci,
                                 uint32_t *wo, int32_t *ell_col, uint32_t *ell_w)
{
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t i = orig[v];
        const int64_t e0 = rp[i];
        const int32_t d = (int32_t)(rp[i + 1] - e0);
        const int32_t o = rpi[v];
        for (int32_t u = 0; u < d; ++u) {
            ci[o + u] = (int32_t)o2i[col[e0 + u]];
            wo[o + u] = w[e0 + u];
        }
        if (ell_col) {
            int4 c4 = make_int4(v, v, v, v);
            uint4 w4 = make_uint4(0u, 0u, 0u, 0u);
            int32_t *cc = &c4.x;
            uint32_t *ww = &w4.x;
            for (int32_t u = 0; u < d; ++u) {
                cc[u] = (int32_t)o2i[col[e0 + u]];
                ww[u] = w[e0 + u];
            }
            reinterpret_cast<int4 *>(ell_col)[v] = c4;
            reinterpret_cast<uint4 *>(ell_w)[v] = w4;
        }
    }
}

// fingerprint of the internal order (checkpoints): sum of mixed (position, vertex) pairs
__global__ void k_hash_order(int32_t n, const uint32_t *orig, unsigned long long *hash)
{
    uint64_t h = 0;
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        h += mix64(((uint64_t)(uint32_t)v << 32) ^ orig[v] ^ 0xC2B2AE3D27D4EB4Full);
    h = (uint64_t)warp_sum64((int64_t)h);
    if ((threadIdx.x & 31) == 0)
        atomicAdd(hash, (unsigned long long)h);
}

// int8 readback / overwrite of one local replica rl through the internal order
__global__ void k_extract_i8(const int8_t *s, int64_t R, int32_t n, int64_t rl, const uint32_t *o2i, int8_t *out)
{
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = s[(size_t)o2i[i] * R + rl];
}

__global__ void k_insert_i8(int8_t *s, int64_t R, int32_t n, int64_t rl, const uint32_t *o2i, const int8_t *in)
{
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        s[(size_t)o2i[i] * R + rl] = in[i];
}

// ------------------------------------------------------------------ launchers
namespace {
unsigned grid_for(int64_t n, int threads = 256)
{
    const int64_t b = (n + threads - 1) / threads;
    return (unsigned)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}
}  // namespace

cudaError_t launch_csr_check(int32_t n, const int64_t *rp, const int32_t *col, const int32_t *wi, const float *wf,
                             const int32_t *colour, CsrCheck *out, uint8_t *colour_used, cudaStream_t st)
{
    CsrCheck init{};
    init.bad_row = init.bad_sym = init.bad_sum = init.bad_colrange = init.bad_proper = INT32_MAX;
    init.max_colour = -1;
    init.pm1 = 1u;
    cudaError_t e = cudaMemcpyAsync(out, &init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess)
        return e;
    if (colour) {
        e = cudaMemsetAsync(colour_used, 0, 1 << 16, st);
        if (e != cudaSuccess)
            return e;
    }
    k_csr_check<<<grid_for(n), 256, 0, st>>>(n, rp, col, wi, wf, colour, out, colour_used);
    e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(st);  // `init` is read by the copy above
    return e;
}

cudaError_t colour_jp_device(int32_t n, const int64_t *rp, const int32_t *col, uint32_t *prio, int32_t *colour,
                             int32_t *counters, int32_t *ncol_out, cudaStream_t st)
{
    // counters[0]: vertices left uncoloured by the last rounds; counters[1]: colours used
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(int32_t), st);
    if (e != cudaSuccess)
        return e;
    k_jp_init<<<grid_for(n), 256, 0, st>>>(n, prio, colour);
    if ((e = cudaGetLastError()) != cudaSuccess)
        return e;
    int32_t h[2] = {0, 0};
    for (int batch = 0;; ++batch) {
        // a few rounds per readback (a round with little left to colour is a cheap scan);
        // counters[0] counts the vertices the LAST of them left uncoloured
        for (int k = 0; k < 4; ++k) {
            if (k == 3 && (e = cudaMemsetAsync(counters, 0, sizeof(int32_t), st)) != cudaSuccess)
                return e;
            k_jp_round<<<grid_for(n), 256, 0, st>>>(n, rp, col, prio, colour, counters, counters + 1);
        }
        if ((e = cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            return e;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess)
            return e;
        if (h[0] == 0)
            break;
        if (batch > (1 << 22))  // cannot happen: every round colours the top-priority uncoloured vertex
            return cudaErrorUnknown;
    }
    *ncol_out = h[1];
    return cudaSuccess;
}

cudaError_t build_order_device(int32_t n, int32_t ncol, const int32_t *colour, const int64_t *rp, uint32_t *orig,
                               uint32_t *o2i, int32_t *class_off, int32_t *rpi, cudaStream_t st)
{
    uint32_t *keys_in = nullptr, *keys_out = nullptr, *ids = nullptr;
    int32_t *deg = nullptr;
    void *tmp = nullptr;
    size_t tmp_sort = 0, tmp_scan = 0;
    int end_bit = 1;
    while ((1 << end_bit) < ncol)
        ++end_bit;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys_in, keys_out, ids, orig, n, 0, end_bit, st);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, deg, rpi, n + 1, st);
    const size_t tmpb = tmp_sort > tmp_scan ? tmp_sort : tmp_scan;
    if (e == cudaSuccess)
        e = cudaMallocAsync(&keys_in, sizeof(uint32_t) * (size_t)n, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&keys_out, sizeof(uint32_t) * (size_t)n, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&ids, sizeof(uint32_t) * (size_t)n, st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&deg, sizeof(int32_t) * ((size_t)n + 1), st);
    if (e == cudaSuccess)
        e = cudaMallocAsync(&tmp, tmpb, st);
    if (e == cudaSuccess) {
        k_iota_keys<<<grid_for(n), 256, 0, st>>>(n, colour, keys_in, ids);
        e = cudaGetLastError();
    }
    // stable LSD radix sort by colour: ids ascending inside a class (the host path's order)
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_sort, keys_in, keys_out, ids, orig, n, 0, end_bit, st);
    if (e == cudaSuccess) {
        k_order_finish<<<grid_for((int64_t)n + 1), 256, 0, st>>>(n, ncol, keys_out, orig, rp, class_off, o2i, deg);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, deg, rpi, n + 1, st);
    cudaFreeAsync(keys_in, st);
    cudaFreeAsync(keys_out, st);
    cudaFreeAsync(ids, st);
    cudaFreeAsync(deg, st);
    cudaFreeAsync(tmp, st);
    return e;
}

cudaError_t launch_build_internal(int32_t n, const int64_t *rp, const int32_t *col, const uint32_t *w,
                                  const uint32_t *orig, const uint32_t *o2i, const int32_t *rpi, int32_t *ci,
                                  uint32_t *wo, int32_t *ell_col, uint32_t *ell_w, cudaStream_t st)
{
    k_build_internal<<<grid_for(n), 256, 0, st>>>(n, rp, col, w, orig, o2i, rpi, ci, wo, ell_col, ell_w);
    return cudaGetLastError();
}

cudaError_t launch_hash_order(int32_t n, const uint32_t *orig, unsigned long long *hash, cudaStream_t st)
{
    k_hash_order<<<grid_for(n), 256, 0, st>>>(n, orig, hash);
    return cudaGetLastError();
}

cudaError_t launch_extract_i8(const int8_t *s, int64_t R, int32_t n, int64_t rl, const uint32_t *o2i, int8_t *out,
                              cudaStream_t st)
{
    k_extract_i8<<<grid_for(n), 256, 0, st>>>(s, R, n, rl, o2i, out);
    return cudaGetLastError();
}

cudaError_t launch_insert_i8(int8_t *s, int64_t R, int32_t n, int64_t rl, const uint32_t *o2i, const int8_t *in,
                             cudaStream_t st)
{
    k_insert_i8<<<grid_for(n), 256, 0, st>>>(s, R, n, rl, o2i, in);
    return cudaGetLastError();
}

}  // namespace ising

// gather_peak.cu -- measured memory roof of the C5 access pattern (k_csr_i8_ring without its
// arithmetic), so the C5 kernel's HBM fraction can be read against what this access pattern can
// reach on a B200, not only against the streaming copy peak of MEASURED_PEAKS.json.
//
// The pattern: int8 spins s[v][r], R = 256 replicas (256-byte rows), 4e6 rows in
// colour-sorted order; one launch per colour class (37.5 / 37 / 23 / 2.6 % of the rows); each warp
// sweeps a contiguous chunk of its class; per vertex it reads the 48-byte table entry (4 columns,
// 4 weights, original id: 36 bytes used), its own row and three neighbour rows in the other
// classes (uniformly random rows: the C5 graph is a random 3-regular expander, so its neighbour
// rows have no locality either), and writes its own row back.  Each lane moves 8 bytes of every
// row (one coalesced 256-byte segment per warp).  Two variants:
//   ring: the rows go through a per-warp shared-memory ring filled by cp.async, S vertices deep,
//         the table entries are prefetched 32 vertices ahead (the k_csr_i8_ring skeleton);
//   ldg:  plain 8-byte loads, U vertices unrolled (register MLP).
// The "decision" is one XOR with a runtime mask of 0, so every row is still read and the own row
// written (the stored value equals the loaded one).
//
// Reported per configuration: attempts/s (rows x 256 replicas per sweep / time) and DRAM GB/s
// of the pattern's bytes (1,316 per vertex = 5.14 per attempt), over `sweeps` timed sweeps after
// one untimed sweep.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/gather_peak tools/gather_peak.cu
// Run:   tools/gather_peak <variant ring|ldg> <depth S or unroll U> <CTAs per SM> <sweeps>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

namespace {

constexpr uint32_t kRows = 4000000;
constexpr uint32_t kR = 256;  // bytes per row
constexpr int kClasses = 4;
constexpr double kFrac[kClasses] = {0.375, 0.370, 0.229, 0.026};

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint2 lds64(uint32_t a)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

struct Entry {  // 48-byte table entry, as in the ring kernel's shared-memory copy
    int4 col;
    int4 w;
    uint32_t orig, pad[3];
};

// table entry of vertex j (chunk-relative) from the lane that prefetched it
__device__ __forceinline__ int4 entry_cols(const int4 &mine, uint32_t j)
{
    const int src = (int)(j & 31u);
    return make_int4(__shfl_sync(0xFFFFFFFFu, mine.x, src), __shfl_sync(0xFFFFFFFFu, mine.y, src),
                     __shfl_sync(0xFFFFFFFFu, mine.z, src), 0);
}

template <int S>
__global__ void __launch_bounds__(256) k_ring(uint8_t *s, const Entry *tab, uint32_t v0, uint32_t nv,
                                              uint32_t chunk, uint32_t mask, uint32_t *sink)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib;
    const uint32_t j0 = gw * chunk;
    if (j0 >= nv)
        return;
    const uint32_t cnt = min(chunk, nv - j0);
    const uint32_t vb = v0 + j0;
    uint8_t *col8 = s + 8u * lane;
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(smem) + wib * (S * 4u * 256u) + lane * 8u;
    // table entries of the current and the next 32-vertex block (one per lane)
    int4 cur = make_int4(0, 0, 0, 0), nxt = cur, wcur = cur;
    uint32_t ocur = 0;
    if (lane < cnt) {
        cur = __ldg(&tab[vb + lane].col);
        wcur = __ldg(&tab[vb + lane].w);
        ocur = __ldg(&tab[vb + lane].orig);
    }
    if (32u + lane < cnt)
        nxt = __ldg(&tab[vb + 32u + lane].col);
    auto cols_of = [&](uint32_t j) {  // j within [jb, jb + 64) of the current block
        return (j >> 5) == 0 ? entry_cols(cur, j) : entry_cols(nxt, j);
    };
    auto issue = [&](uint32_t j, int4 c) {
        const uint32_t sl = ring0 + (j % S) * 4u * 256u;
        cp_async8(sl, col8 + (uint64_t)(vb + j) * kR);
        cp_async8(sl + 256u, col8 + (uint64_t)(uint32_t)c.x * kR);
        cp_async8(sl + 512u, col8 + (uint64_t)(uint32_t)c.y * kR);
        cp_async8(sl + 768u, col8 + (uint64_t)(uint32_t)c.z * kR);
    };
    uint32_t acc = 0;
#pragma unroll
    for (uint32_t j = 0; j + 1 < S; ++j) {
        if (j < cnt)
            issue(j, cols_of(j));
        cp_commit();
    }
    uint32_t base = 0;  // first vertex of the `cur` block
    for (uint32_t j = 0; j < cnt; ++j) {
        if (j == base + 32u) {  // slide the table window
            base += 32u;
            cur = nxt;
            nxt = make_int4(0, 0, 0, 0);
            if (base + 32u + lane < cnt)
                nxt = __ldg(&tab[vb + base + 32u + lane].col);
            if (base + lane < cnt) {
                wcur = __ldg(&tab[vb + base + lane].w);
                ocur = __ldg(&tab[vb + base + lane].orig);
            }
        }
        const uint32_t jn = j + S - 1;
        if (jn < cnt)
            issue(jn, cols_of(jn - base));
        cp_commit();
        cp_wait<S - 1>();
        const uint32_t sl = ring0 + (j % S) * 4u * 256u;
        const uint2 own = lds64(sl);
        const uint2 a = lds64(sl + 256u), b = lds64(sl + 512u), c = lds64(sl + 768u);
        const uint32_t x = (a.x ^ b.x ^ c.x ^ a.y ^ b.y ^ c.y) & mask;
        *reinterpret_cast<uint2 *>(col8 + (uint64_t)(vb + j) * kR) = make_uint2(own.x ^ x, own.y ^ x);
        acc ^= (uint32_t)wcur.x ^ ocur;
    }
    cp_wait<0>();
    if ((acc & mask) == 0xFFFFFFFFu)  // never true (mask = 0): keeps the table loads alive
        sink[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg(uint8_t *s, const Entry *tab, uint32_t v0, uint32_t nv,
                                             uint32_t chunk, uint32_t mask, uint32_t *sink)
{
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib;
    const uint32_t j0 = gw * chunk;
    if (j0 >= nv)
        return;
    const uint32_t cnt = min(chunk, nv - j0);
    const uint32_t vb = v0 + j0;
    uint8_t *col8 = s + 8u * lane;
    uint32_t acc = 0;
    for (uint32_t jb = 0; jb < cnt; jb += 32u) {
        int4 mine = make_int4(0, 0, 0, 0), wm = mine;
        uint32_t om = 0;
        if (jb + lane < cnt) {
            mine = __ldg(&tab[vb + jb + lane].col);
            wm = __ldg(&tab[vb + jb + lane].w);
            om = __ldg(&tab[vb + jb + lane].orig);
        }
        acc ^= (uint32_t)wm.x ^ om;
        const uint32_t nb = min(32u, cnt - jb);
        for (uint32_t u0 = 0; u0 < nb; u0 += U) {
            uint2 own[U], a[U], b[U], c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t j = u0 + (uint32_t)u;
                if (j < nb) {
                    const int4 cc = entry_cols(mine, j);
                    own[u] = *reinterpret_cast<const uint2 *>(col8 + (uint64_t)(vb + jb + j) * kR);
                    a[u] = __ldg(reinterpret_cast<const uint2 *>(col8 + (uint64_t)(uint32_t)cc.x * kR));
                    b[u] = __ldg(reinterpret_cast<const uint2 *>(col8 + (uint64_t)(uint32_t)cc.y * kR));
                    c[u] = __ldg(reinterpret_cast<const uint2 *>(col8 + (uint64_t)(uint32_t)cc.z * kR));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t j = u0 + (uint32_t)u;
                if (j < nb) {
                    const uint32_t x = (a[u].x ^ b[u].x ^ c[u].x ^ a[u].y ^ b[u].y ^ c[u].y) & mask;
                    *reinterpret_cast<uint2 *>(col8 + (uint64_t)(vb + jb + j) * kR) =
                        make_uint2(own[u].x ^ x, own[u].y ^ x);
                }
            }
        }
    }
    if ((acc & mask) == 0xFFFFFFFFu)
        sink[0] = acc;
}

uint64_t splitmix(uint64_t &x)
{
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace

int main(int argc, char **argv)
{
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s ring|ldg <S|U> <ctas_per_sm> <sweeps>\n", argv[0]);
        return 2;
    }
    const bool ring = std::strcmp(argv[1], "ring") == 0;
    const int depth = std::atoi(argv[2]);
    const int cps = std::atoi(argv[3]);
    const int sweeps = std::atoi(argv[4]);
    int dev = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));

    // classes: contiguous row ranges; neighbours uniformly random rows of the other classes
    uint32_t cls0[kClasses + 1];
    cls0[0] = 0;
    for (int c = 0; c < kClasses; ++c)
        cls0[c + 1] = c + 1 == kClasses ? kRows : cls0[c] + (uint32_t)(kFrac[c] * kRows);
    std::vector<Entry> tab(kRows);
    uint64_t st = 2311;
    for (int c = 0; c < kClasses; ++c)
        for (uint32_t v = cls0[c]; v < cls0[c + 1]; ++v) {
            const uint32_t outside = kRows - (cls0[c + 1] - cls0[c]);
            int32_t cs[3];
            for (int u = 0; u < 3; ++u) {
                uint32_t r = (uint32_t)(splitmix(st) % outside);
                if (r >= cls0[c])
                    r += cls0[c + 1] - cls0[c];
                cs[u] = (int32_t)r;
            }
            tab[v].col = make_int4(cs[0], cs[1], cs[2], -1);
            tab[v].w = make_int4(1, 2, 3, 0);
            tab[v].orig = v;
        }
    uint8_t *s = nullptr;
    Entry *dtab = nullptr;
    uint32_t *sink = nullptr;
    CK(cudaMalloc(&s, (size_t)kRows * kR));
    CK(cudaMemset(s, 1, (size_t)kRows * kR));
    CK(cudaMalloc(&dtab, sizeof(Entry) * kRows));
    CK(cudaMemcpy(dtab, tab.data(), sizeof(Entry) * kRows, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&sink, 4));

    const size_t smem = ring ? (size_t)8 * depth * 4 * 256 : 0;
    auto launch = [&](uint32_t v0, uint32_t nv) {
        const uint32_t warps_want = (uint32_t)nsm * (uint32_t)cps * 8u;
        uint32_t chunk = (nv + warps_want - 1) / warps_want;
        if (chunk < 40u)
            chunk = 40u;
        const uint32_t warps = (nv + chunk - 1) / chunk;
        const dim3 grid((warps + 7) / 8);
        if (ring) {
            switch (depth) {
            case 4: k_ring<4><<<grid, 256, smem>>>(s, dtab, v0, nv, chunk, 0u, sink); break;
            case 6: k_ring<6><<<grid, 256, smem>>>(s, dtab, v0, nv, chunk, 0u, sink); break;
            case 8: k_ring<8><<<grid, 256, smem>>>(s, dtab, v0, nv, chunk, 0u, sink); break;
            default: std::fprintf(stderr, "S in {4, 6, 8}\n"); std::exit(2);
            }
        } else {
            switch (depth) {
            case 2: k_ldg<2><<<grid, 256>>>(s, dtab, v0, nv, chunk, 0u, sink); break;
            case 4: k_ldg<4><<<grid, 256>>>(s, dtab, v0, nv, chunk, 0u, sink); break;
            case 8: k_ldg<8><<<grid, 256>>>(s, dtab, v0, nv, chunk, 0u, sink); break;
            default: std::fprintf(stderr, "U in {2, 4, 8}\n"); std::exit(2);
            }
        }
    };
    if (ring) {
        CK(cudaFuncSetAttribute(k_ring<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4 * 256));
        CK(cudaFuncSetAttribute(k_ring<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 6 * 4 * 256));
        CK(cudaFuncSetAttribute(k_ring<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8 * 4 * 256));
    }
    int occ = 0;
    if (ring) {
        switch (depth) {
        case 4: CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ring<4>, 256, smem)); break;
        case 6: CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ring<6>, 256, smem)); break;
        default: CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ring<8>, 256, smem)); break;
        }
    } else {
        occ = 8;
    }
    auto sweep = [&]() {
        for (int c = 0; c < kClasses; ++c)
            launch(cls0[c], cls0[c + 1] - cls0[c]);
    };
    sweep();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int t = 0; t < sweeps; ++t)
        sweep();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double attempts = (double)kRows * kR * sweeps;
    const double bytes = (double)kRows * sweeps * (5.0 * kR + 36.0);
    std::printf("{\"variant\": \"%s\", \"depth\": %d, \"ctas_per_sm\": %d, \"resident_ctas_per_sm\": %d, "
                "\"sweeps\": %d, \"ms\": %.3f, \"attempts_per_s\": %.6e, \"gbs\": %.1f, "
                "\"bytes_per_attempt\": %.4f}\n",
                ring ? "ring" : "ldg", depth, cps, occ, sweeps, ms, attempts / (ms * 1e-3),
                bytes / (ms * 1e-3) / 1e9, (5.0 * kR + 36.0) / kR);
    return 0;
}

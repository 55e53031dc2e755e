// alu_peak.cu -- measured issue roof of the bit-packed sweep kernels' instruction mix
// ("ALU fraction = the kernel's instruction rate / the rate of a
// Philox-only + LOP3-only microbenchmark at the same clock").
//
// The bit-packed kernels (k_grid_bits, k_grid_bands, k_csr_bits) spend their issue slots on
// Philox4x32-10 (IMAD.WIDE on the FMA pipe + LOP3 on the ALU pipe) and on the MSB-first plane
// comparison (LOP3 only).  This program runs exactly that mix with no memory traffic, at full
// occupancy, on every SM, and reports the issue rate it reaches:
//   mode 0 "philox":  two interleaved Philox calls per iteration, results folded by LOP3;
//   mode 1 "plane":   the same two calls + the 8-plane comparison of bits_core.cuh (mux LOP3 +
//                     2 LOP3 per plane), i.e. stage 1 of the sweep kernels without the loads.
// Instructions per loop iteration are counted from the SASS (tools/alu_peak.py) and, on the
// box, by ncu (smsp__inst_executed.sum); the SM clock is measured in-kernel (clock64 against
// %globaltimer) so the roof is also expressed per SM cycle, which bench.py scales by the clock
// it samples during its own timed region.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/alu_peak tools/alu_peak.cu
// Run:   tools/alu_peak <mode 0|1> <threads per CTA> <CTAs per SM> <iterations>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;

struct Keys {
    uint32_t k[20];
};

__device__ __forceinline__ uint32_t mux(uint32_t m, uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(m), "r"(a), "r"(b));
    return r;
}

// rounds 2..9 of the hoisted PLANE Philox (bits_core.cuh philox_plane)
__device__ __forceinline__ uint4 philox8(uint32_t sA, uint32_t sB, uint32_t j4, uint32_t U0, uint32_t L0r1,
                                         const Keys &rk)
{
    const uint32_t X = sA ^ j4;
    uint32_t c0 = __umulhi(kM1, X) ^ U0;
    uint32_t c1 = kM1 * X;
    uint32_t c2 = sB;
    uint32_t c3 = L0r1;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        const uint32_t lo0 = kM0 * c0, hi0 = __umulhi(kM0, c0);
        const uint32_t lo1 = kM1 * c2, hi1 = __umulhi(kM1, c2);
        const uint32_t n0 = hi1 ^ c1 ^ rk.k[2 * r];
        const uint32_t n2 = hi0 ^ c3 ^ rk.k[2 * r + 1];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

template <int MODE>
__global__ void k_alu(Keys rk, uint32_t iters, const uint32_t *planes, uint32_t *out, unsigned long long *clk)
{
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t sA = gid * 0x9E3779B9u ^ rk.k[1];
    uint32_t sB = gid * 0x85EBCA6Bu ^ rk.k[3];
    const uint32_t U0 = rk.k[2] ^ blockIdx.x, L0r1 = rk.k[0] * 0x27D4EB2Fu;
    uint32_t t4[8], t8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        t4[j] = planes[j];
        t8[j] = planes[8 + j];
    }
    uint32_t m8 = gid * 0x165667B1u, D = ~0u, acc = 0u;
    unsigned long long c0 = 0, g0 = 0;
    if (gid == 0) {
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    }
#pragma unroll 1
    for (uint32_t it = 0; it < iters; ++it) {
        const uint4 w0 = philox8(sA, sB, 2u * it, U0, L0r1, rk);
        const uint4 w1 = philox8(sA, sB, 2u * it + 1u, U0, L0r1, rk);
        if (MODE == 0) {
            acc ^= w0.x ^ w0.y ^ w0.z;
            D ^= w0.w ^ w1.x ^ w1.y;
            m8 ^= w1.z ^ w1.w;
        } else {
            const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                const uint32_t ta = mux(m8, t8[j], t4[j]);
                const uint32_t ya = D & ~ws[j] & ta;
                D &= ~(ws[j] ^ ta);
                const uint32_t tb = mux(m8, t8[j + 1], t4[j + 1]);
                const uint32_t yb = D & ~ws[j + 1] & tb;
                D &= ~(ws[j + 1] ^ tb);
                acc |= ya | yb;
            }
            D = ~acc ^ w1.w;  // next word's undecided lanes (keeps the chain data-dependent)
            m8 ^= w0.x;
        }
        sB ^= acc;  // the next calls depend on this iteration's results
    }
    if (gid == 0) {
        unsigned long long g1;
        const unsigned long long c1 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        clk[0] = c1 - c0;
        clk[1] = g1 - g0;
    }
    out[gid] = acc ^ D ^ m8;
}

}  // namespace

int main(int argc, char **argv)
{
    const int mode = argc > 1 ? atoi(argv[1]) : 1;
    const int threads = argc > 2 ? atoi(argv[2]) : 1024;
    const int per_sm = argc > 3 ? atoi(argv[3]) : 2;
    const uint32_t iters = argc > 4 ? (uint32_t)atoll(argv[4]) : 20000u;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm * per_sm;
    Keys rk;
    uint32_t a = 2311u, b = 0u;
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = a;
        rk.k[2 * r + 1] = b;
        a += 0x9E3779B9u;
        b += 0xBB67AE85u;
    }
    uint32_t hp[16];
    for (int j = 0; j < 16; ++j)
        hp[j] = 0x9E3779B9u * (uint32_t)(j + 1);
    uint32_t *planes, *out;
    unsigned long long *clk;
    cudaMalloc(&planes, sizeof(hp));
    cudaMemcpy(planes, hp, sizeof(hp), cudaMemcpyHostToDevice);
    cudaMalloc(&out, (size_t)grid * threads * 4);
    cudaMalloc(&clk, 16);
    auto kern = mode == 0 ? k_alu<0> : k_alu<1>;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w)  // warm-up (clocks ramp, module load)
        kern<<<grid, threads>>>(rk, iters, planes, out, clk);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int w = 0; w < reps; ++w)
        kern<<<grid, threads>>>(rk, iters, planes, out, clk);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        fprintf(stderr, "alu_peak: CUDA error %s\n", cudaGetErrorString(err));
        return 1;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long hc[2];
    cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0);
    printf("{\"mode\": %d, \"threads\": %d, \"ctas_per_sm\": %d, \"resident_ctas_per_sm\": %d, \"grid\": %d, "
           "\"iters\": %u, \"launches\": %d, \"ms_per_launch\": %.6f, \"sm_mhz_in_kernel\": %.1f}\n",
           mode, threads, per_sm, occ, grid, iters, reps, ms / reps, 1e3 * (double)hc[0] / (double)hc[1]);
    return 0;
}

// internal.h -- handle layout and kernel launchers of libising (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/ising.h"
#include "common.cuh"

namespace ising {

enum Kernel : int32_t { KER_GRID_BITS = 0, KER_CSR_BITS = 1, KER_CSR_I8 = 2 };

// CTA size limits (and launch bounds) of the bit-packed kernels, multiples of 4 warps so the
// four schedulers get equal work.  Measured on C2/C4b/C3: the torus kernel
// runs fastest with 16 warps and up to 128 registers per thread, the CSR kernel with 24.
// (A/B on C4b, abtest/c4b_max.sh: a 640-thread cap -- 600-thread passes -- -6%; a 576 cap, i.e.
// 512 threads at <= 112 registers, +0.1%)
#ifndef ISING_GRID_MAX_THREADS
#define ISING_GRID_MAX_THREADS 512
#endif
constexpr int32_t kGridMaxThreads = ISING_GRID_MAX_THREADS;
constexpr int32_t kCsrMaxThreads = 768;

// k_csr_i8_phase CTA size and the resident CTAs per SM its register budget is sized for
constexpr int32_t kI8Threads = 256, kI8MinBlocks = 4;
// float + padded-table graphs: two-deep pipelined kernel and its resident CTAs per SM
constexpr bool kI8Pipe = true;
constexpr int32_t kI8PipeMinBlocks = 4;
// float + padded-table graphs with R % 256 == 0: cp.async ring kernel with this many vertices
// in flight per warp (0 = use the register pipeline)
// (the ISING_* macros only serve A/B builds of variants, abtest/variant.sh)
#ifndef ISING_I8_RING
#define ISING_I8_RING 4
#endif
#ifndef ISING_I8_RING_UNROLL
#define ISING_I8_RING_UNROLL 4
#endif
#ifndef ISING_I8_RING_MINB
#define ISING_I8_RING_MINB 3
#endif
constexpr int32_t kI8Ring = ISING_I8_RING;
constexpr int32_t kI8RingUnroll = ISING_I8_RING_UNROLL;  // main-loop unroll (multiple of kI8Ring, divides 32; 8 measured -1.3%)
#ifndef ISING_I8_RING_PATTERN
#define ISING_I8_RING_PATTERN 1
#endif
// ring kernel: fields by per-vertex pattern folds + one shuffle per replica
constexpr bool kI8RingPattern = ISING_I8_RING_PATTERN != 0;
constexpr int32_t kI8RingMinBlocks = ISING_I8_RING_MINB;  // resident CTAs per SM the ring kernel's registers are sized for
// packed-row working copy of the int8 state for float + padded-table sweeps:
// resident CTAs per SM its registers are sized for, and the fewest sweeps per call that use it
// (each call packs the state before its first sweep and unpacks it after its last)
#ifndef ISING_I8_PACKED_MINB
#define ISING_I8_PACKED_MINB 3
#endif
// (4 resident CTAs per SM at 64 registers: -0.3%)
constexpr int32_t kI8PackedMinBlocks = ISING_I8_PACKED_MINB;
constexpr int32_t kI8PackedMinSweeps = 4;
// timing probe of the packed kernel's arithmetic alone (rows from registers, no row loads or
// stores; results wrong): abtest builds with -DISING_I8_PACKED_NOMEM=1
#ifndef ISING_I8_PACKED_NOMEM
#define ISING_I8_PACKED_NOMEM 0
#endif
constexpr bool kI8PackedNoMem = ISING_I8_PACKED_NOMEM != 0;
#ifndef ISING_I8_PACKED_RING
#define ISING_I8_PACKED_RING 4
#endif
constexpr int32_t kI8PackedRing = ISING_I8_PACKED_RING;  // vertices in flight per warp (2: -2.3%)
#ifndef ISING_I8_PACKED_UNROLL
#define ISING_I8_PACKED_UNROLL 8
#endif
constexpr int32_t kI8PackedUnroll = ISING_I8_PACKED_UNROLL;  // main-loop unroll (8: +2.9% over 4)

// Rows of a colour class per pass of the 2-D thread mapping: threads / (Lx/2), rounded
// down to an even number when >= 2 so that the parity (c + y) & 1 of a thread's sites is
// the same in every pass.  The host uses the same rule (abi.cu) to validate the shape.
__host__ __device__ inline int grid_rows_per_pass(int threads, int hx)
{
    const int r = threads / hx;
    return r >= 2 ? (r & ~1) : r;
}


// Best-so-far record kept in device memory (updated by the exchange kernel).
struct BestDev {
    int64_t energy;  // int64, or double bits
    int64_t slot;    // global slot, -1 = none yet
    int64_t sweep;
    int32_t owner;   // 1 if this handle snapshotted the configuration
    int32_t pad;
};

// ----------------------------------------------------------------- kernel params
struct GridBitsParams {
    const uint32_t *state_in;  // [G][n], original site order
    uint32_t *state_out;
    const uint8_t *jbyte;      // [n] colour-separated order: bit 0..3 = right,left,down,up has J=-1
    const uint32_t *planes;    // [K/32][2][64]: index 0 = dE 4, 1 = dE 8
    int64_t *E_out;            // [R_local]
    int32_t Lx, Ly, n, hx, half;
    uint32_t ymagic;           // floor division by hx via umulhi
    int32_t words_per_copy;    // K/32
    uint32_t g0;               // global group of local group 0
    uint32_t t0;
    int32_t n_rounds;          // rounds of k_ex sweeps in this launch
    int32_t k_ex;              // sweeps per round
    int32_t qcap;              // capacity of the shared-memory tail queue
    const uint32_t *planes_sched;  // annealing: [sweep][K/32][2][64] per-sweep planes, or null
    // fused PT (pt = 1, launched as clusters of words_per_copy CTAs = one copy each)
    int32_t pt;
    uint32_t e0;               // exchange index of the first round
    int64_t *walker;           // [R_local] walker ids (read + written)
    int64_t *copy_best;        // [C_local][3] per-copy best (E, slot, sweep) of this launch
    int8_t *snap;              // [C_local][n] per-copy best configuration (original order)
    const uint64_t *Tx;
    const int64_t *Tx_off;
    const int32_t *Tx_len;
    RoundKeys rk;
    int32_t bands;             // row bands per word group (1, or 2: CTA pairs with DSMEM halo rows)
    // band split with a copy spread over K/32 clusters of 2 (cooperative launch): the PT
    // step exchanges energies and boundary bit planes through global memory
    int32_t xc;
    int64_t *xc_E;             // [C_local][2][K] word types' energies, by round parity
    uint32_t *xc_B;            // [C_local][2][K/32][2 bands][2 planes][nbw], by round parity
    uint32_t *xc_bar;          // [C_local] copy barrier counters (zero at launch)
    // persistent ticket-scheduled launch (k_grid_sched): tasks = (local word group, round)
    int32_t n_groups;          // local word groups G
    uint32_t *xs_ctl;          // [1 + 2 C_local]: ticket, per-copy finished tasks, published rounds
    int64_t *xs_E;             // [G][32] energies of the group's last round
    uint32_t *xs_S;            // [G][n] the groups' states between rounds, colour-separated order
    uint32_t *xs_B;            // [2][G][2][nbw] bit 0 / bit 31 planes (colour-separated order), by round parity
    uint32_t *xs_M;            // [C_local][K/32] swap mask of the copy's last exchange
};

struct CsrBitsParams {
    const uint32_t *state_in;  // [G][n] internal order
    uint32_t *state_out;
    const int32_t *rp;         // [n+1] internal
    const uint32_t *nbr;       // [m2] internal neighbour id | (J==-1) << 31
    const uint32_t *orig;      // [n] internal -> original id
    const int32_t *class_off;  // [ncol+1]
    const uint32_t *planes;    // [K/32][Qmax][64]  q = dE/2 = 1..Qmax
    int64_t *E_out;
    int32_t n, ncol, qmax;
    int64_t m;                 // undirected edges
    int32_t words_per_copy;
    uint32_t g0, t0;
    int32_t n_rounds, k_ex;    // n_rounds x k_ex sweeps in this launch
    int32_t qcap;
    const uint32_t *planes_sched;  // annealing: [sweep][K/32][qmax][64] per-sweep planes, or null
    int32_t pt;                // fused PT (clusters of words_per_copy CTAs)
    uint32_t e0;
    int64_t *walker;
    int64_t *copy_best;
    int8_t *snap;
    const uint64_t *Tx;
    const int64_t *Tx_off;
    const int32_t *Tx_len;
    RoundKeys rk;
};

struct CsrI8Params {
    int8_t *s;                 // [n][R] internal vertex order, replica-minor
    const int32_t *rp;         // [n+1] internal
    const int32_t *col;        // internal ids
    const int32_t *ell_col;    // [n][4] padded neighbour table (pad -1) or null (CSR path)
    const int32_t *ell_w;      // [n][4] weights (int32 or float bits), pad 0
    int32_t ell_deg;           // used width of the ELL table (max degree, <= 4)
    const int32_t *wi;         // int weights or null
    const float *wf;           // float weights or null
    const uint32_t *orig;      // internal -> original id
    const uint64_t *T;         // [R][qmax+1] integer thresholds per LOCAL replica (q = dE/2)
    const float *betaf;        // [R] 2 * float(beta_k) per LOCAL replica, float weights
    int32_t R;                 // local replicas (multiple of 4)
    int32_t nq;                // R / 4
    int32_t nq_shift;          // log2(threads per vertex) if a power of two, else -1
    int32_t K;
    int64_t slot0;             // first global slot
    int32_t qmax;
    int32_t v_begin, v_end;    // vertex class range (internal)
    uint32_t t;
    RoundKeys rk;
};

// Fused PT run of a small int8 instance (k_i8_small): one CTA per local copy.
struct SmallI8Params {
    int8_t *s;                 // [n][R] internal order (the copy's K columns are contiguous)
    const int32_t *rp, *col, *wi;  // internal CSR, integer weights
    const uint32_t *orig;      // internal -> original id
    const int32_t *class_off;  // [ncol+1]
    const int32_t *ell_col, *ell_w;  // [n][4] padded neighbour table (pad -1, weight 0) or null
    int32_t max_class;         // largest colour class (vertices)
    const uint64_t *T;         // [R][qmax+1] per local replica
    int64_t *E_out, *walker, *copy_best;
    int8_t *snap;              // [C_local][n] original order
    const uint64_t *Tx;
    const int64_t *Tx_off;
    const int32_t *Tx_len;
    int32_t n, R, K, qmax, ncol;
    int64_t slot0;
    uint32_t t0, e0;
    int32_t n_rounds, k_ex;
    RoundKeys rk;
};
constexpr int32_t kI8SmallThreads = 1024;  // one 8-replica task per thread on C1 (512: -15%)
// largest n x K (bytes of one copy's spins) the fused int8 launch keeps in shared memory
constexpr int64_t kI8SmallMaxBytes = 96 * 1024;
// fused small int8 runs: spread each copy over a cluster of K/8 CTAs (K <= 64)
constexpr bool kI8Cluster = true;

// k_exchange: CTA size and the most CTAs (size of the handle's partial-best scratch)
constexpr int32_t kExThreads = 256, kExMaxBlocks = 64;

struct ExchangeParams {
    int64_t *xpart;            // [2 kExMaxBlocks] per-CTA best (E, slot) of the candidates
    uint32_t *xctr;            // CTA ticket (zero between launches)
    int64_t *E;                // [R_local] (int64 or double bits)
    int64_t *walker;           // [R_local]
    int64_t *cbest;            // [C_local][3] persistent per-copy best (E, slot, sweep)
    uint32_t *swapmask;        // [C_local][ceil(K/32)]
    BestDev *best;
    int8_t *best_spins;        // [n] original order
    const ising_record *recs;  // gathered records or null (local)
    int64_t n_recs;
    // configuration access for the snapshot
    int32_t layout;            // 0 bits, 1 i8
    const uint32_t *state;     // bits: [G][n] (grid: original order; csr: internal)
    const int8_t *s8;          // i8: [n][R] internal
    const uint32_t *perm_o2i;  // original -> internal id (null = identity)
    int32_t n;
    int32_t K, C_local, words_per_copy;
    int64_t slot0, R_local;
    int32_t is_float;
    uint32_t t, e;
    int32_t do_best, do_swap;
    const uint64_t *Tx;        // exchange thresholds flat
    const int64_t *Tx_off;     // [K-1] offset into Tx; entry for d<0 at Tx[off + (-d-1)]
    const int32_t *Tx_len;     // [K-1]
    RoundKeys rk;
};

struct IcmParams {
    uint32_t *state;           // [G][n] bit-packed (grid: original order, csr: internal order)
    int64_t *E;                // [R_local]
    int32_t n, kind;           // kind 0 grid, 1 csr
    int32_t Lx, Ly;
    const uint8_t *jbyte_orig; // grid: [n] original order, bit 0 J_right = -1, bit 1 J_down = -1
    const int32_t *rp;         // csr (internal)
    const uint32_t *nbr;
    const uint32_t *o2i;       // csr: original -> internal (null for grids)
    int32_t KW;
    uint32_t pair0;            // global pair index of local pair 0
    int32_t k_min;
    uint32_t f;                // cluster-move index
    int64_t m_edges;
    RoundKeys rk;
};

// Results of the device CSR checks (k_create.cu): the lowest failing vertex of each check
// (INT32_MAX = none) and the per-graph quantities the host path computed in its loops.
struct CsrCheck {
    int32_t bad_row;       // range, self-loop, duplicate, non-finite weight
    int32_t bad_sym;       // (i, j, w) without (j, i, w)
    int32_t bad_sum;       // integer weights: sum |w| at a vertex >= 2^30
    int32_t bad_colrange;  // caller colouring out of [0, 2^16)
    int32_t bad_proper;    // caller colouring not proper
    int32_t maxdeg;
    int32_t max_colour;
    uint32_t pm1;          // integer weights all +-1
    int64_t qmax;          // max per-vertex sum |w| (integer weights)
    int64_t sum_abs;       // sum over entries of |w| (each edge twice)
    int64_t W_int;         // sum of w over edges (each once)
    uint64_t hash;         // fingerprint of row_ptr / col / w (checkpoints)
};

// ----------------------------------------------------------------- launchers
cudaError_t launch_csr_check(int32_t n, const int64_t *rp, const int32_t *col, const int32_t *wi, const float *wf,
                             const int32_t *colour, CsrCheck *out, uint8_t *colour_used, cudaStream_t st);
cudaError_t colour_jp_device(int32_t n, const int64_t *rp, const int32_t *col, uint32_t *prio, int32_t *colour,
                             int32_t *counters, int32_t *ncol_out, cudaStream_t st);
cudaError_t build_order_device(int32_t n, int32_t ncol, const int32_t *colour, const int64_t *rp, uint32_t *orig,
                               uint32_t *o2i, int32_t *class_off, int32_t *rpi, cudaStream_t st);
cudaError_t launch_build_internal(int32_t n, const int64_t *rp, const int32_t *col, const uint32_t *w,
                                  const uint32_t *orig, const uint32_t *o2i, const int32_t *rpi, int32_t *ci,
                                  uint32_t *wo, int32_t *ell_col, uint32_t *ell_w, cudaStream_t st);
cudaError_t launch_hash_order(int32_t n, const uint32_t *orig, unsigned long long *hash, cudaStream_t st);
cudaError_t launch_extract_i8(const int8_t *s, int64_t R, int32_t n, int64_t rl, const uint32_t *o2i, int8_t *out,
                              cudaStream_t st);
cudaError_t launch_insert_i8(int8_t *s, int64_t R, int32_t n, int64_t rl, const uint32_t *o2i, const int8_t *in,
                             cudaStream_t st);
cudaError_t launch_icm_bits(const IcmParams &p, int32_t pairs, int32_t threads, cudaStream_t st);
cudaError_t launch_init_bits(uint32_t *state, int32_t G, int32_t n, const uint32_t *orig,
                             uint32_t g0, const RoundKeys &rk, cudaStream_t st);
cudaError_t launch_init_i8(int8_t *s, int32_t n, int32_t R, const uint32_t *orig, int64_t slot0,
                           const RoundKeys &rk, cudaStream_t st);
cudaError_t launch_grid_bits(const GridBitsParams &p, int32_t G, int32_t threads, size_t smem,
                             cudaStream_t st);
size_t grid_bits_smem(int32_t n);
// band-split torus kernel (k_grid_bands.cu): G word groups on 2 G CTAs
cudaError_t launch_grid_bands(const GridBitsParams &p, int32_t G, int32_t threads, size_t smem,
                              cudaStream_t st);
int32_t grid_bands_max_clusters(int32_t cluster, int32_t threads, size_t smem);
// persistent ticket-scheduled fused PT launch (k_grid_sched.cu): `ctas` resident CTAs
cudaError_t launch_grid_sched(const GridBitsParams &p, int32_t ctas, int32_t threads, size_t smem,
                              cudaStream_t st);
int32_t grid_sched_ctas(int32_t threads, size_t smem, bool spill);
int32_t grid_bits_qcap(int32_t n);
cudaError_t launch_csr_bits(const CsrBitsParams &p, int32_t G, int32_t threads, size_t smem,
                            cudaStream_t st);
size_t csr_bits_smem(int32_t n, int32_t qmax, int32_t words_per_copy);
int32_t csr_bits_qcap(int32_t n, int32_t qmax);
cudaError_t launch_csr_i8_phase(const CsrI8Params &p, int32_t threads, cudaStream_t st);
// packed-row sweeps: s[n][R] int8 <-> P[n][R/32] words (unpack = true: P -> s), and one colour
// phase on P (float weights, padded table, R % 256 == 0)
cudaError_t launch_pack_rows(const int8_t *s, uint32_t *P, int64_t n, int64_t R, bool unpack, cudaStream_t st);
cudaError_t launch_csr_packed_phase(const CsrI8Params &p, uint32_t *P, cudaStream_t st);
cudaError_t launch_energy_i8(const int8_t *s, const int32_t *rp, const int32_t *col,
                             const int32_t *wi, const float *wf, int32_t n, int32_t R,
                             int64_t *Ei, double *Ef, void *scratch, size_t scratch_bytes,
                             cudaStream_t st);
size_t energy_i8_scratch(int32_t n, int32_t R);
cudaError_t launch_exchange(const ExchangeParams &p, cudaStream_t st);
cudaError_t launch_i8_small(const SmallI8Params &p, int32_t C_local, cudaStream_t st);
cudaError_t launch_merge_copy_best(const int64_t *copy_best, const int8_t *snap, int32_t C_local,
                                   int32_t n, BestDev *best, int8_t *best_spins, int64_t *cbest,
                                   cudaStream_t st);
cudaError_t launch_swap_bits(uint32_t *state, const uint32_t *swapmask, int32_t n, int32_t C_local,
                             int32_t words_per_copy, cudaStream_t st);
cudaError_t launch_swap_i8(int8_t *s, const uint32_t *swapmask, int32_t n, int32_t R, int32_t K,
                           cudaStream_t st);
cudaError_t launch_records(const int64_t *E, ising_record *out, int64_t R, int64_t slot0,
                           cudaStream_t st);
cudaError_t launch_merge_best(const int64_t *recs, int64_t n, int32_t is_float, int64_t *out,
                              cudaStream_t st);
cudaError_t launch_extract_bits(const uint32_t *state, int32_t n, int32_t gl, int32_t bit,
                                const uint32_t *perm_o2i, int8_t *out, cudaStream_t st);
cudaError_t launch_insert_bits(uint32_t *state, int32_t n, int32_t gl, int32_t bit,
                               const uint32_t *perm_o2i, const int8_t *in, cudaStream_t st);
cudaError_t launch_debug_exp_bound(const float *beta2, int32_t n_beta, uint32_t *out, cudaStream_t st);
cudaError_t launch_debug_philox(const uint32_t *in, int32_t n, uint32_t *out_lib,
                                uint32_t *out_curand, cudaStream_t st);

}  // namespace ising

/*
 * ising.h -- C ABI of libising.so, the B200 (sm_100a) engine for the
 * data-parallel hot path behind arXiv 2311.09275 ("Improved Sparse Ising
 * Optimization", K. M. Zick): replica-parallel Metropolis single-spin-flip
 * sweeps over sparse Ising couplings with parallel-tempering (PT) exchange.
 *
 * Problem statement: binary variables with pairwise couplings on a sparse
 * graph -- sparse Ising / weighted MaxCut (Table I
 * P:25-35).  The method the paper benchmarks (Cosm) is undisclosed (P:17,
 * P:59); the calls below implement the north-star hot path of BASELINE.json:
 * Metropolis sweeps, PT exchange ("simulates replicas
 * of a system at different temperatures and exchanges replicas across
 * temperatures"), energies/cuts and best-so-far tracking
 * (S:261-264).  Every numerical convention (RNG counters, thresholds,
 * update order, tie-breaks) is the contract of DESIGN.md §3; the CPU oracle
 * under oracle/ implements the same contract independently.
 *
 * Conventions used by every call
 *   - Spins are +1/-1.  Packed words store bit 1 for -1.
 *   - Energy  E(s) = sum over undirected edges {i,j} of w_ij s_i s_j (each edge
 *     once).  Cut = (W - E)/2 with W = sum of w_ij (signed).
 *   - Replica slots: K temperatures x C copies, global slot r = c*K + k; slot r
 *     always runs at beta_k.  A PT exchange moves CONFIGURATIONS between the
 *     two slots of a pair (the walker id travels with the configuration).
 *   - A handle simulates the contiguous copy shard [copy_begin, copy_end) of a
 *     C-copy ensemble; every RNG counter uses GLOBAL ids, so the union of the
 *     shards equals one handle holding all copies, bit for bit.
 *   - Vertex ids in and out of the ABI are the caller's ORIGINAL ids.
 *
 * Errors: every int-returning call returns an ising_status (0 = OK, < 0 =
 * error), never aborts and never throws; ising_last_error() gives a
 * thread-local message naming the offending argument or index.
 *
 * Ownership: inputs are borrowed for the duration of the call and copied.
 * Outputs go to caller-allocated buffers.  The handle owns all device memory;
 * it is single-owner and not thread-safe.  Distinct handles may run
 * concurrently (one process per GPU is the intended deployment).
 *
 * Streams: all device work of a handle is enqueued on desc->stream (a
 * cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream; NULL = the
 * legacy default stream).  Calls documented "async" return before the work
 * completes; calls documented "syncs" synchronise that stream.
 */
#ifndef ISING_H
#define ISING_H

#include <stdint.h>

#if defined(__GNUC__)
#define ISING_API __attribute__((visibility("default")))
#else
#define ISING_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ising_handle ising_handle;

typedef enum {
    ISING_OK = 0,
    ISING_E_ARG = -1,         /* bad argument: NULL, n < 1, bad ladder, bad shard, ... */
    ISING_E_GRAPH = -2,       /* invalid couplings: self-loop, duplicate, asymmetric, range, colouring */
    ISING_E_UNSUPPORTED = -3, /* valid but not implemented (see each call) */
    ISING_E_CUDA = -4,        /* CUDA runtime failure (message has the CUDA error string) */
    ISING_E_OOM = -5,         /* device allocation failed */
    ISING_E_STATE = -6        /* call out of order / data not held by this handle */
} ising_status;

typedef enum { ISING_W_I32 = 0, ISING_W_F32 = 1 } ising_wtype;

/* Spin storage.  BITS: 32 replicas per uint32 word (multi-spin coding), requires
 * integer weights in {-1,+1} and the PLANE RNG contract.  I8: one int8 per
 * (vertex, replica), replica-minor, any int32 or float32 weights, WORD contract. */
typedef enum { ISING_SPINS_BITS = 0, ISING_SPINS_I8 = 1 } ising_layout;

/* RNG contract: PLANE = bit-sliced 64-bit uniforms shared by 32
 * replicas of a word, compared MSB-first; WORD = one 64-bit uniform per replica. */
typedef enum { ISING_RNG_PLANE = 0, ISING_RNG_WORD = 1 } ising_rng;

/* Colouring ising_create_csr computes when the caller passes none (SURVEY §8(c) #13,
 * DESIGN.md R12/R12c).  GREEDY: vertices in ascending id, smallest colour unused by coloured
 * neighbours (host, sequential).  JP: the same greedy rule in Jones-Plassmann priority order --
 * decreasing pr(i) = word 0 of Philox4x32-10(i, 0, 0, 6 << 24) under key (0, 0), ties to the
 * lower id -- computed on the GPU in parallel rounds (a vertex is coloured once all its
 * higher-priority neighbours are); at most max degree + 1 colours. */
typedef enum { ISING_COLOUR_GREEDY = 0, ISING_COLOUR_JP = 1 } ising_colouring;

typedef struct {
    uint64_t seed;         /* Philox key = (seed & 0xffffffff, seed >> 32) */
    int32_t n_temps;       /* K >= 1; BITS layout needs K % 32 == 0 */
    int32_t n_copies;      /* C >= 1 (global ensemble size) */
    int32_t copy_begin;    /* this handle's shard [copy_begin, copy_end), 0 <= b < e <= C */
    int32_t copy_end;
    const double *betas;   /* K inverse temperatures, > 0, strictly increasing */
    int32_t layout;        /* ising_layout */
    int32_t rng;           /* ising_rng; must be PLANE for BITS and WORD for I8 */
    int32_t device;        /* CUDA device ordinal */
    int32_t block_threads; /* 0 = default; else threads per CTA of the sweep kernels */
    void *stream;          /* cudaStream_t or NULL */
    int32_t colouring;     /* ising_colouring used by ising_create_csr when colour == NULL */
} ising_run_desc;

/* Per-slot record written by ising_exchange_begin (16 bytes): energy (int64, or
 * the bits of a double for float weights) and the GLOBAL slot id. */
typedef struct {
    int64_t energy;
    int64_t slot;
} ising_record;

/* Best record of one rank for ising_merge_best (24 bytes): energy (int64, or the bits of a
 * double for float weights), the sweep t at which it was reached, its GLOBAL slot (< 0: the
 * rank has no record yet). */
typedef struct {
    int64_t energy;
    int64_t sweep;
    int64_t slot;
} ising_best_record;

typedef struct {
    int32_t n;            /* vertices */
    int32_t n_colours;    /* colour classes swept per sweep */
    int64_t n_edges;      /* undirected edges m */
    int32_t n_temps, n_copies, copy_begin, copy_end;
    int64_t slot_begin;   /* first global slot of this handle = copy_begin*K */
    int64_t n_slots;      /* local slots R = (copy_end-copy_begin)*K */
    int32_t layout, rng, wtype, kernel; /* kernel: 0 grid-bits, 1 csr-bits, 2 csr-i8 */
    int64_t sweeps_done;  /* t */
    int64_t exchanges_done; /* e */
    int64_t W_int;        /* sum of weights (integer weights) */
    double W_f64;         /* sum of weights (float weights, float64 sum in edge order) */
    int32_t bands;        /* grid BITS: rows of a word group split over this many CTAs (1 or 2) */
    int32_t fused_pt;     /* 1 if ising_run runs all rounds in one launch; 2: one cooperative launch
                             whose copies span K/32 clusters (band split); 3: one persistent
                             ticket-scheduled launch (grid BITS with more word groups than
                             resident CTAs); 0: per-round launches */
} ising_info_t;

/* Create from a periodic Lx x Ly grid (torus).  Site i = x + Lx*y; J_right[i]
 * couples i with ((x+1)%Lx, y), J_down[i] with (x, (y+1)%Ly); values must be +-1
 * (Gset spin-glass tori).  Lx, Ly even and >= 4 (checkerboard colouring
 * (x+y)&1).  Uploads, initialises spins from the INIT stream
 * and computes initial energies.  Errors: ISING_E_ARG (NULL, odd/small dims,
 * bad desc), ISING_E_GRAPH (a J not in {-1,+1}), ISING_E_UNSUPPORTED (BITS with
 * a lattice too large for one CTA's shared memory), ISING_E_CUDA/OOM.
 * With layout I8 the torus runs on the generic CSR kernels (row order right,
 * left, down, up; checkerboard colouring). */
ISING_API int ising_create_grid(int32_t Lx, int32_t Ly, const int8_t *J_right, const int8_t *J_down,
                      const ising_run_desc *desc, ising_handle **out);

/* Create from a symmetric CSR: row_ptr[n+1] (int64, row_ptr[0]=0, non-decreasing),
 * col[row_ptr[n]] (int32 in [0,n)), w[row_ptr[n]] (int32 or float32 per wtype).
 * Invariants: no self-loops, no duplicate neighbours in a row, and
 * (i,j,w) present iff (j,i,w) present.  colour[n] (optional, NULL -> desc->colouring:
 * greedy in ascending id or in Jones-Plassmann priority order) must be a proper
 * colouring with ids 0..ncol-1.  Row order is kept as given (it fixes the
 * float32 field summation order).  With the I8 layout the checks, the colouring, the
 * colour-sorted internal order and the internal tables are computed on the GPU (one upload
 * of the CSR); errors are the same (lowest failing vertex first).  Errors: ISING_E_GRAPH
 * (message names the offending vertex/entry), ISING_E_UNSUPPORTED (BITS with weights not
 * +-1, float weights with BITS), ISING_E_ARG, ISING_E_CUDA/OOM. */
ISING_API int ising_create_csr(int32_t n, const int64_t *row_ptr, const int32_t *col, const void *w,
                     int32_t wtype, const int32_t *colour, const ising_run_desc *desc,
                     ising_handle **out);

/* n_sweeps Metropolis sweeps of every local replica (async).  Sweep t visits the
 * colour classes in order; each vertex of a class attempts one flip per replica:
 * dE = -2 s_i h_i, h_i = sum_j w_ij s_j; accept if dE <= 0, else iff
 * U64 < floor(exp(-beta_k dE) 2^64) (float weights: the float32 contract
 * exponential).  Advances t by n_sweeps and refreshes the per-slot energies
 * at the end.  n_sweeps >= 0.  I8 layout with float weights, maximum degree <= 4 and
 * n_slots % 256 == 0: a call of >= 4 sweeps packs the int8 spins into a bit-packed working
 * copy (n x n_slots/8 bytes, allocated on first use; without room for it the int8 kernels
 * run), sweeps that, and unpacks it at the end -- the same decisions, so the same result
 * (environment ISING_I8_PACKED=0 / 1 forces the int8 / packed kernels). */
ISING_API int ising_sweep(ising_handle *h, int32_t n_sweeps);

/* Per-local-slot energies (syncs).  out: int64[n_slots] for integer weights,
 * double[n_slots] for float weights. */
ISING_API int ising_energy(ising_handle *h, void *out);

/* Per-local-slot cuts (W - E)/2 (syncs); int64 or double like ising_energy. */
ISING_API int ising_cut(ising_handle *h, void *out);

/* n_rounds x (k_ex sweeps, then ising_exchange) in as few launches as possible (async).
 * Identical results to calling ising_sweep(h, k_ex); ising_exchange(h) n_rounds times.
 * Bit-packed layouts run the whole sequence in ONE launch: clusters of K/32 CTAs (one copy
 * each; K/32 x 2 for the band-split torus kernel) keep the copy on chip and exchange
 * energies and boundary bit planes through distributed shared memory -- unless those
 * clusters would not all be resident at once, in which case the rounds run as per-round
 * launches.  Small int8 instances with integer weights (n*K <= 96 KB per copy) also run in
 * ONE launch (one CTA per copy).  ising_info.fused_pt says which.  Errors:
 * ISING_E_UNSUPPORTED for float weights. */
ISING_API int ising_run(ising_handle *h, int32_t n_rounds, int32_t k_ex);

/* Local PT step (async, single process): best-so-far check over the local slots,
 * then exchange number e among adjacent temperatures k, k+1 with k = e%2, e%2+2,
 * ...: d = E(c,k+1) - E(c,k); swap the two configurations iff d >= 0 or
 * U64x(k,e,c) < floor(exp((beta_{k+1}-beta_k) d) 2^64).  Advances e.
 * Errors: ISING_E_UNSUPPORTED for float weights (exchange needs exact energies). */
ISING_API int ising_exchange(ising_handle *h);

/* Simulated annealing (async launch, syncs at the end, PAPER.md P:53
 * "SA-based CMOS annealers"): n_sweeps Metropolis sweeps in which sweep s
 * uses the inverse temperature sched[s*K + k] for the slots of temperature index k
 * (schedule: n_sweeps x K doubles > 0, any order; a row equal to the ladder reproduces
 * ising_sweep).  Same RNG contracts and threshold formula as ising_sweep; advances t; ends
 * with a best-so-far check.  No exchange. */
ISING_API int ising_anneal(ising_handle *h, int32_t n_sweeps, const double *sched);

/* Houdayer / isoenergetic cluster move number f (async, PAPER.md
 * P:53, refs [20][21]).  For every copy pair (2p, 2p+1) of the shard and every temperature
 * k >= k_min: X_i = [s_a(i) != s_b(i)] for the slots a = (2p, k), b = (2p+1, k); the seed is
 * the first of 64 candidates i_j = (w_j n) >> 32 (w_j = word j&3 of Philox(k, f, p,
 * ICM<<24 | j>>2)) with X = 1; the connected component of the seed in the {X = 1} subgraph
 * flips in both replicas (E_a + E_b is conserved).  Energies are refreshed.  Advances f.
 * Errors: ISING_E_UNSUPPORTED for the I8 layout or a shard that splits a pair. */
ISING_API int ising_icm(ising_handle *h, int32_t k_min);

/* Multi-process PT step, first half (async): write one ising_record per local
 * slot (n_slots * 16 bytes) into the DEVICE buffer dev_send, to be all-gathered. */
ISING_API int ising_exchange_begin(ising_handle *h, void *dev_send);

/* Second half (async): dev_recv holds n_records gathered ising_records (device
 * memory).  Best-so-far check over ALL records (global argmin, ties -> lowest
 * global slot; the owning handle snapshots the configuration), then the local
 * swaps exactly as ising_exchange.  Advances e. */
ISING_API int ising_exchange_end(ising_handle *h, const void *dev_recv, int64_t n_records);

/* Best-so-far check only (async): dev_recv/n_records as above, or NULL/0 for the
 * local slots.  Used at the end of a run whose length is not a multiple of the
 * exchange interval. */
ISING_API int ising_check_best(ising_handle *h, const void *dev_recv, int64_t n_records);

/* Global best over per-rank best records (syncs): multi-process runs whose ranks keep local
 * best-so-far records gather every rank's ising_best into DEVICE memory (e.g. one NCCL
 * all-gather of n ising_best_record) and merge them here: the lexicographic minimum of
 * (energy, sweep, slot) -- the lowest energy, first reached, then the lowest slot --
 * computed by one kernel on the handle's stream.  best_E: int64* or double* (per the handle's
 * weights); slot, sweep: the winner's.  Errors: ISING_E_ARG (NULL, n < 1), ISING_E_STATE (no
 * record has a slot). */
ISING_API int ising_merge_best(ising_handle *h, const void *dev_recs, int64_t n, void *best_E, int64_t *slot,
                               int64_t *sweep);

/* Best record (syncs).  best_E: int64* or double*; slot: global slot; sweep: the t
 * at which it was first reached (strict <).  spins_out (n int8, original ids,
 * may be NULL) is only available on the handle that owns the slot; otherwise
 * ISING_E_STATE.  Before any check: ISING_E_STATE. */
ISING_API int ising_best(ising_handle *h, void *best_E, int64_t *slot, int64_t *sweep, int8_t *spins_out);

/* Per-copy best-so-far (syncs): for each local copy c (copies are independent PT ladders,
 * i.e. independent trials in the sense of PAPER.md P:37-45), the lowest energy reached at
 * any best-so-far check (strict <, ties -> lowest slot), its global slot and sweep.
 * best_E: int64[C_local] or double[C_local]; slot, sweep: int64[C_local]; slot = -1 before
 * the first check. */
ISING_API int ising_copy_best(ising_handle *h, void *best_E, int64_t *slot, int64_t *sweep);

/* Configuration of one LOCAL slot given by its GLOBAL id (syncs): n int8 +-1. */
ISING_API int ising_get_spins(ising_handle *h, int64_t slot, int8_t *out);

/* Overwrite one slot's configuration (syncs); values must be +-1.  Energies are
 * refreshed. */
ISING_API int ising_set_spins(ising_handle *h, int64_t slot, const int8_t *in);

/* Walker id (the global slot a configuration started in) per local slot (syncs). */
ISING_API int ising_get_walkers(ising_handle *h, int64_t *out);

ISING_API int ising_info(const ising_handle *h, ising_info_t *out);

/* ---- checkpoint / resume (SURVEY.md §5 "Checkpoint / resume"; SPEC S:326 seeds) -----
 * Every random number is keyed by (seed, vertex, sweep t, group/slot, exchange e,
 * cluster-move f), so the complete dynamic state of a handle is: the
 * configurations, the energies, the walker ids, the counters t/e/f and the best-so-far
 * records.  A handle created from the SAME instance, colouring, ladder, seed and shard
 * (copy_begin/copy_end) that loads a checkpoint continues bit for bit as the saving
 * handle would have (test_checkpoint_resume_parity).
 *
 * ising_state_size: bytes of this handle's checkpoint blob (host-only, no sync).
 * ising_state_save: writes the blob into the caller's HOST buffer buf of `bytes` >=
 *   the size (syncs).  Layout (little-endian, opaque to callers): a 128-byte header
 *   (magic "ISNGCKP1", shape, counters, fingerprints of the instance/ladder/colouring),
 *   then the state buffer in the handle's internal layout, E, walkers, per-copy best,
 *   the best record and the best configuration.
 * ising_state_load: restores a blob written by a compatible handle (syncs).
 *   ISING_E_ARG: NULL buf or bytes too small; ISING_E_STATE: bad magic/version or a
 *   header that does not match this handle (different n, m, weights sum, shard,
 *   layout, RNG contract, seed, ladder or colouring) -- the handle is left unchanged. */
ISING_API int ising_state_size(const ising_handle *h, int64_t *bytes);
ISING_API int ising_state_save(ising_handle *h, void *buf, int64_t bytes);
ISING_API int ising_state_load(ising_handle *h, const void *buf, int64_t bytes);

/* Block until all work enqueued by the handle has finished. */
ISING_API int ising_sync(ising_handle *h);

/* Thread-local message of the last failing call on this thread ("" if none). */
ISING_API const char *ising_last_error(void);

/* Release all device memory (syncs first).  NULL-safe. */
ISING_API void ising_destroy(ising_handle *h);

/* ---- host-only utilities (no GPU needed) ---------------------------------- */

/* The library's greedy colouring (same rule as ising_create_csr with colour=NULL).
 * Returns the number of colours, or < 0 on error (validated like create_csr). */
ISING_API int ising_greedy_colour(int32_t n, const int64_t *row_ptr, const int32_t *col,
                        int32_t *colour_out);

/* Smallest-last greedy colouring (R12b; a "greedy colouring" in the sense of
 * BASELINE configs[2], with at most degeneracy + 1 colours -- 3 on the sparse random
 * graphs of C3): repeatedly remove a vertex of minimum remaining degree (ties: lowest id),
 * then colour vertices in reverse removal order, each with the smallest colour unused by
 * its already-coloured neighbours.  Pass the result as `colour` to ising_create_csr.
 * row_ptr: n+1 int64, col: row_ptr[n] int32 (symmetric, as for create_csr); colour_out: n
 * int32 (caller-owned).  Returns the number of colours, or ISING_E_ARG on NULL / n < 1. */
ISING_API int ising_greedy_colour_sl(int32_t n, const int64_t *row_ptr, const int32_t *col,
                        int32_t *colour_out);

/* The Jones-Plassmann-order greedy colouring (ISING_COLOUR_JP) as ising_create_csr computes
 * it, on GPU `device` (syncs): row_ptr n+1 int64, col row_ptr[n] int32 (symmetric, ids in
 * range); colour_out n int32 (caller-owned).  Returns the number of colours, or < 0 on error
 * (ISING_E_ARG, ISING_E_GRAPH for a bad row_ptr or column id, ISING_E_CUDA). */
ISING_API int ising_colour_jp(int32_t device, int32_t n, const int64_t *row_ptr, const int32_t *col,
                              int32_t *colour_out);

/* Metropolis threshold floor(exp(-(beta*dE)) * 2^64) saturated to 2^64-1, as the
 * library's host tables compute it (integer dE > 0). */
ISING_API uint64_t ising_threshold(double beta, int64_t dE);

/* Library version string. */
ISING_API const char *ising_version(void);

/* ---- diagnostics (GPU) ------------------------------------------------------ */

/* Evaluate the library's device Philox4x32-10 and cuRAND's curand_Philox4x32_10
 * on n (counter, key) tuples: in[6n] = {c0,c1,c2,c3,k0,k1}; out_lib[4n], out_curand[4n]
 * are host buffers.  Syncs. */
ISING_API int ising_debug_philox(int32_t device, const uint32_t *in, int32_t n, uint32_t *out_lib,
                       uint32_t *out_curand);

/* Exhaustive check of the fast float decision used by the I8 kernels:
 * for each of the n_beta values 2*beta (float, the kernels' per-replica slope) and EVERY
 * float sh in [-80/(2 beta), 0], e = ex2.approx(RN(RN(2 beta log2e) sh + 16)) against the
 * contract value c = cexp32(RN(2 beta sh)) 2^16 (§3.5).  worst_rel = max |e/c - 1| where
 * c >= 1/2; max_small = max e where c < 1/2.  The kernels' 2^-16 margin decides exactly
 * when worst_rel < 2^-17 and max_small < 1.  Syncs; ISING_E_ARG for NULL or bad betas. */
ISING_API int ising_debug_exp_bound(int32_t device, const float *beta2, int32_t n_beta, float *worst_rel,
                                    float *max_small);

#ifdef __cplusplus
}
#endif

#endif /* ISING_H */

/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the hot path of
 * arXiv 2311.09275 ("Improved Sparse Ising Optimization") as scoped by
 * replica-parallel Metropolis single-spin-flip sweeps over a
 * sparse coupling graph plus parallel-tempering (PT) replica exchange.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code.  It shares NO code, header,
 * table or constant generator with the CUDA library under
 * paper_2311_09275_b200/; both are transcribed independently from the
 * contract in DESIGN.md §3.
 *
 * Plain scalar C, no SIMD, no threads inside a call.  Spins are int8 +-1,
 * stored s[rl*n + i] (local slot rl, ORIGINAL vertex id i).
 *
 * Citations (PAPER.md = P:line, SPEC.md = S:line):
 *   problem: sparse Ising / weighted MaxCut            P:13, Table I
 *   energy  E = sum_{ij in E} J_ij s_i s_j              S:127 (SURVEY §8 Conv)
 *   field   h_i = sum_j J_ij s_j, dE_i = -2 s_i h_i
 *   Metropolis sweep: accept dE<=0, else w.p. e^-b dE
 *   "sweeps (iterations)" as the unit of work
 *   PT: replicas at different temperatures exchange    P:53 (ref [19] P:142)
 *   exchange acceptance min(1, exp(dbeta*dH))
 *   counter-based RNG keyed by seed/stream
 *
 * Functions whose pin is only "same contract" and not a property the paper or
 * mathematics fixes are marked "parity unpinned" below (none at present; see
 * DESIGN.md §4 for the pin of every function).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Philox */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3").  One round:
 *   (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0))
 * with the key bumped by (W0, W1) between rounds.
 * Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt)
 * and on the GPU box by curand_Philox4x32_10. */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* RNG streams: top byte of counter word 3. */
enum { ST_INIT = 0, ST_PLANE = 1, ST_WORD_HI = 2, ST_WORD_LO = 3, ST_EXCH = 4, ST_ICM = 5 };
enum { RNG_PLANE = 0, RNG_WORD = 1 };

static void philox_at(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                      uint32_t out[4])
{
    uint32_t ctr[4] = {a, b, c, d};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    or_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------ probabilities */
/* p64(x) = min(floor(exp(x) * 2^64), 2^64-1) for x <= 0: the probability
 * exp(x) as a 64-bit integer threshold; a uniform U in [0, 2^64) satisfies
 * P(U < p64(x)) = floor(exp(x)*2^64)/2^64. */
uint64_t or_p64(double x)
{
    double p = exp(x);
    double v = ldexp(p, 64);
    if (v >= 18446744073709551616.0)
        return UINT64_MAX;
    return (uint64_t)v;
}

/* Metropolis threshold for an integer energy increase dE > 0 at inverse
 * temperature beta: accept iff U < exp(-beta*dE) ("with probability").
 * The expression -(beta * (double)dE) is part of the contract. */
uint64_t or_threshold_int(double beta, int64_t dE)
{
    return or_p64(-(beta * (double)dE));
}

/* Exchange threshold: accept iff U < exp((beta_{k+1}-beta_k) * d), d < 0. */
uint64_t or_threshold_exch(double beta_lo, double beta_hi, int64_t d)
{
    return or_p64((beta_hi - beta_lo) * (double)d);
}

/* cexp32: the fully specified float32 exponential of the contract
 * for x <= 0.  Transcribed from the contract text only. */
float or_cexp32(float x)
{
    if (x < -64.0f)
        return 0.0f;
    float k = floorf(x * 0x1.715476p+0f);  /* floor(x * log2 e), one RN multiply */
    float r = fmaf(-k, 0x1.62e400p-1f, x); /* x - k ln2_hi */
    r = fmaf(-k, 0x1.7f7d1cp-20f, r);      /* ... - k ln2_lo (Cody-Waite) */
    float p = 0x1.71de3ap-19f;             /* Horner, e^r ~ sum_{i<=9} r^i / i! */
    p = fmaf(p, r, 0x1.a01a02p-16f);
    p = fmaf(p, r, 0x1.a01a02p-13f);
    p = fmaf(p, r, 0x1.6c16c2p-10f);
    p = fmaf(p, r, 0x1.111112p-7f);
    p = fmaf(p, r, 0x1.555556p-5f);
    p = fmaf(p, r, 0x1.555556p-3f);
    p = fmaf(p, r, 0x1p-1f);
    p = fmaf(p, r, 0x1p+0f);
    p = fmaf(p, r, 0x1p+0f);
    return ldexpf(p, (int)k);
}

/* Float-weight Metropolis threshold for dE > 0 (float32 contract). */
uint64_t or_threshold_f32(double beta, float dE)
{
    float x = -((float)beta * dE);
    float r = or_cexp32(x);
    float v = ldexpf(r, 64);
    if (v >= 0x1p64f)
        return UINT64_MAX;
    return (uint64_t)v;
}

/* -------------------------------------------------------------- instances */
/* Torus -> CSR with row order (right, left, down, up); colour (x+y)&1.
 * rp: n+1, col/w: 4n, colour: n. */
void or_grid_to_csr(int32_t Lx, int32_t Ly, const int8_t *J_right, const int8_t *J_down,
                    int64_t *rp, int32_t *col, int32_t *w, int32_t *colour)
{
    int32_t n = Lx * Ly;
    for (int32_t y = 0; y < Ly; ++y) {
        for (int32_t x = 0; x < Lx; ++x) {
            int32_t i = x + Lx * y;
            int32_t right = ((x + 1) % Lx) + Lx * y;
            int32_t left = ((x + Lx - 1) % Lx) + Lx * y;
            int32_t down = x + Lx * ((y + 1) % Ly);
            int32_t up = x + Lx * ((y + Ly - 1) % Ly);
            rp[i] = 4 * (int64_t)i;
            col[4 * i + 0] = right; w[4 * i + 0] = J_right[i];
            col[4 * i + 1] = left;  w[4 * i + 1] = J_right[left];
            col[4 * i + 2] = down;  w[4 * i + 2] = J_down[i];
            col[4 * i + 3] = up;    w[4 * i + 3] = J_down[up];
            colour[i] = (x + y) & 1;
        }
    }
    rp[n] = 4 * (int64_t)n;
}

/* Greedy colouring: vertices in ascending id, each takes the smallest colour
 * not used by an already-coloured neighbour (SURVEY §8(c) reading #13).
 * Returns the number of colours. */
int32_t or_greedy_colour(int32_t n, const int64_t *rp, const int32_t *col, int32_t *colour)
{
    int32_t ncol = 0;
    int32_t maxdeg = 0;
    for (int32_t i = 0; i < n; ++i)
        if (rp[i + 1] - rp[i] > maxdeg)
            maxdeg = (int32_t)(rp[i + 1] - rp[i]);
    char *used = (char *)calloc((size_t)maxdeg + 2, 1);
    for (int32_t i = 0; i < n; ++i)
        colour[i] = -1;
    for (int32_t i = 0; i < n; ++i) {
        memset(used, 0, (size_t)maxdeg + 2);
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
            int32_t c = colour[col[e]];
            if (c >= 0 && c <= maxdeg + 1)
                used[c] = 1;
        }
        int32_t c = 0;
        while (used[c])
            ++c;
        colour[i] = c;
        if (c + 1 > ncol)
            ncol = c + 1;
    }
    free(used);
    return ncol;
}

/* Smallest-last greedy colouring (R12b): repeatedly remove a vertex of
 * minimum remaining degree, ties by lowest id; then colour the vertices in reverse
 * removal order, each with the smallest colour not used by an already-coloured
 * neighbour.  The minimum is kept in a binary min-heap of keys (degree << 32 | id);
 * a degree change pushes a new key and stale keys are skipped when popped.
 * Returns the number of colours. */
static void heap_push(uint64_t *h, int64_t *len, uint64_t key)
{
    int64_t k = (*len)++;
    h[k] = key;
    while (k > 0 && h[(k - 1) / 2] > h[k]) {
        uint64_t t = h[k];
        h[k] = h[(k - 1) / 2];
        h[(k - 1) / 2] = t;
        k = (k - 1) / 2;
    }
}

static uint64_t heap_pop(uint64_t *h, int64_t *len)
{
    uint64_t top = h[0];
    h[0] = h[--(*len)];
    int64_t k = 0;
    for (;;) {
        int64_t l = 2 * k + 1, r = l + 1, m = k;
        if (l < *len && h[l] < h[m])
            m = l;
        if (r < *len && h[r] < h[m])
            m = r;
        if (m == k)
            break;
        uint64_t t = h[k];
        h[k] = h[m];
        h[m] = t;
        k = m;
    }
    return top;
}

int32_t or_greedy_colour_sl(int32_t n, const int64_t *rp, const int32_t *col, int32_t *colour)
{
    int32_t maxdeg = 0;
    for (int32_t i = 0; i < n; ++i)
        if (rp[i + 1] - rp[i] > maxdeg)
            maxdeg = (int32_t)(rp[i + 1] - rp[i]);
    size_t nn = (size_t)(uint32_t)n;
    int32_t *deg = (int32_t *)malloc(sizeof(int32_t) * nn);
    char *gone = (char *)calloc(nn, 1);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * nn);
    uint64_t *heap = (uint64_t *)malloc(sizeof(uint64_t) * (nn + (size_t)rp[n] + 1));
    int64_t len = 0, nord = 0;
    for (int32_t i = 0; i < n; ++i) {
        deg[i] = (int32_t)(rp[i + 1] - rp[i]);
        heap_push(heap, &len, ((uint64_t)(uint32_t)deg[i] << 32) | (uint32_t)i);
    }
    while (len > 0) {
        uint64_t key = heap_pop(heap, &len);
        int32_t i = (int32_t)(key & 0xFFFFFFFFu);
        if (gone[i] || (int32_t)(key >> 32) != deg[i])
            continue; /* stale */
        gone[i] = 1;
        order[nord++] = i;
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
            int32_t j = col[e];
            if (gone[j])
                continue;
            deg[j]--;
            heap_push(heap, &len, ((uint64_t)(uint32_t)deg[j] << 32) | (uint32_t)j);
        }
    }
    char *used = (char *)calloc((size_t)maxdeg + 2, 1);
    for (int32_t i = 0; i < n; ++i)
        colour[i] = -1;
    int32_t ncol = 0;
    for (int64_t q = nord - 1; q >= 0; --q) {
        int32_t i = order[q];
        memset(used, 0, (size_t)maxdeg + 2);
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
            int32_t c = colour[col[e]];
            if (c >= 0 && c <= maxdeg + 1)
                used[c] = 1;
        }
        int32_t c = 0;
        while (used[c])
            ++c;
        colour[i] = c;
        if (c + 1 > ncol)
            ncol = c + 1;
    }
    free(used);
    free(deg);
    free(gone);
    free(order);
    free(heap);
    return ncol;
}

/* Greedy colouring in Jones-Plassmann priority order (R12c): vertex i has the
 * priority pr(i) = word 0 of Philox4x32-10(ctr = (i, 0, 0, COLOUR << 24), key = (0, 0)),
 * COLOUR = 6; vertices are coloured in decreasing priority (ties: lower id first), each with
 * the smallest colour not used by an already-coloured neighbour.  This is the sequential
 * definition of the colouring the Jones-Plassmann rounds compute in parallel (a vertex is
 * coloured once every higher-priority neighbour is).  Returns the number of colours. */
static const uint32_t *jp_prio;

static int jp_cmp(const void *a, const void *b)
{
    const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    if (jp_prio[x] != jp_prio[y])
        return jp_prio[x] > jp_prio[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

int32_t or_greedy_colour_jp(int32_t n, const int64_t *rp, const int32_t *col, int32_t *colour,
                            uint32_t *prio_out)
{
    int32_t maxdeg = 0;
    for (int32_t i = 0; i < n; ++i)
        if (rp[i + 1] - rp[i] > maxdeg)
            maxdeg = (int32_t)(rp[i + 1] - rp[i]);
    size_t nn = (size_t)(uint32_t)n;
    uint32_t *prio = (uint32_t *)malloc(sizeof(uint32_t) * nn);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * nn);
    const uint32_t key[2] = {0u, 0u};
    for (int32_t i = 0; i < n; ++i) {
        const uint32_t ctr[4] = {(uint32_t)i, 0u, 0u, 6u << 24};
        uint32_t w[4];
        or_philox4x32_10(ctr, key, w);
        prio[i] = w[0];
        order[i] = i;
        colour[i] = -1;
    }
    jp_prio = prio;
    qsort(order, nn, sizeof(int32_t), jp_cmp);
    char *used = (char *)calloc((size_t)maxdeg + 2, 1);
    int32_t ncol = 0;
    for (size_t q = 0; q < nn; ++q) {
        const int32_t i = order[q];
        memset(used, 0, (size_t)maxdeg + 2);
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
            const int32_t c = colour[col[e]];
            if (c >= 0 && c <= maxdeg + 1)
                used[c] = 1;
        }
        int32_t c = 0;
        while (used[c])
            ++c;
        colour[i] = c;
        if (c + 1 > ncol)
            ncol = c + 1;
    }
    if (prio_out)
        memcpy(prio_out, prio, sizeof(uint32_t) * nn);
    free(used);
    free(order);
    free(prio);
    return ncol;
}

/* ------------------------------------------------------------------- run */
typedef struct {
    int32_t n;
    const int64_t *rp;
    const int32_t *col;
    const int32_t *wi; /* integer weights, or NULL */
    const float *wf;   /* float weights, or NULL  */
    const int32_t *colour;
    int32_t ncol;
    uint64_t seed;
    int32_t K;          /* temperatures per copy */
    int32_t copy_begin; /* first global copy of this call */
    int32_t copy_end;
    const double *beta; /* K, strictly increasing */
    int32_t rng;        /* RNG_PLANE or RNG_WORD */
    int64_t slot_lo;    /* if slot_hi > slot_lo: simulate only global slots [slot_lo, slot_hi) */
    int64_t slot_hi;    /*   (replicas are independent without exchange; no or_exchange then) */
} or_run;

static int64_t run_slot0(const or_run *R)
{
    return R->slot_hi > R->slot_lo ? R->slot_lo : (int64_t)R->copy_begin * R->K;
}

static int64_t run_nrep(const or_run *R)
{
    return R->slot_hi > R->slot_lo ? R->slot_hi - R->slot_lo
                                   : (int64_t)(R->copy_end - R->copy_begin) * R->K;
}

/* Initial configuration ("uniform independent spins"):
 * s(r,i) = -1 iff bit (r & 31) of word 0 of Philox(i, 0, r>>5, INIT<<24). */
void or_init(const or_run *R, int8_t *s)
{
    int32_t n = R->n;
    int64_t slot0 = run_slot0(R);
    int64_t nrep = run_nrep(R);
    for (int64_t rl = 0; rl < nrep; ++rl) {
        int64_t r = slot0 + rl;
        for (int32_t i = 0; i < n; ++i) {
            uint32_t w[4];
            philox_at(R->seed, (uint32_t)i, 0u, (uint32_t)(r >> 5), (uint32_t)ST_INIT << 24, w);
            s[rl * n + i] = ((w[0] >> (r & 31)) & 1u) ? (int8_t)-1 : (int8_t)1;
        }
    }
}

/* Energy from its definition E = sum over edges {i,j} (each once) of
 * w_ij s_i s_j.  Integer weights -> Ei (exact int64); float weights
 * -> Ef (float64, sequential in ascending i then row order). */
void or_energy(const or_run *R, const int8_t *s, int64_t *Ei, double *Ef)
{
    int32_t n = R->n;
    int64_t nrep = run_nrep(R);
    for (int64_t rl = 0; rl < nrep; ++rl) {
        const int8_t *sr = s + rl * n;
        int64_t ei = 0;
        double ef = 0.0;
        for (int32_t i = 0; i < n; ++i) {
            for (int64_t e = R->rp[i]; e < R->rp[i + 1]; ++e) {
                int32_t j = R->col[e];
                if (j <= i)
                    continue;
                if (R->wi)
                    ei += (int64_t)R->wi[e] * sr[i] * sr[j];
                else
                    ef += (double)R->wf[e] * (double)sr[i] * (double)sr[j];
            }
        }
        if (Ei)
            Ei[rl] = ei;
        if (Ef)
            Ef[rl] = ef;
    }
}

/* U64 of the PLANE contract: bit (63-j) of U is bit (r&31) of word (j&3) of
 * Philox(i, t, r>>5, PLANE<<24 | j>>2), j = 0..63.  `planes` caches the 64
 * words of one (i, t, g). */
static void plane_words(uint64_t seed, uint32_t i, uint32_t t, uint32_t g, uint32_t planes[64])
{
    for (uint32_t q = 0; q < 16; ++q) {
        uint32_t w[4];
        philox_at(seed, i, t, g, ((uint32_t)ST_PLANE << 24) | q, w);
        for (int a = 0; a < 4; ++a)
            planes[4 * q + a] = w[a];
    }
}

static uint64_t plane_u64(const uint32_t planes[64], int64_t r)
{
    uint64_t u = 0;
    for (int j = 0; j < 64; ++j)
        u |= (uint64_t)((planes[j] >> (r & 31)) & 1u) << (63 - j);
    return u;
}

/* U64 of the WORD contract: U = hi16 * 2^48 + lo48 with
 * hi16 = 16-bit half (r & 1) (half 0 = the low 16 bits) of word ((r >> 1) & 3) of
 * Philox(i, t, r >> 3, WORD_HI<<24), and lo48 = w0 * 2^16 + (w1 >> 16) of
 * Philox(i, t, r, WORD_LO<<24).  Written out in full (the library draws lo48 only when
 * hi16 == T >> 48, which cannot change U < T). */
static uint64_t word_u64(uint64_t seed, uint32_t i, uint32_t t, int64_t r)
{
    uint32_t hi[4], lo[4];
    philox_at(seed, i, t, (uint32_t)(r >> 3), (uint32_t)ST_WORD_HI << 24, hi);
    philox_at(seed, i, t, (uint32_t)r, (uint32_t)ST_WORD_LO << 24, lo);
    uint32_t w = hi[(r >> 1) & 3];
    uint64_t hi16 = (r & 1) ? (w >> 16) : (w & 0xFFFFu);
    uint64_t lo48 = ((uint64_t)lo[0] << 16) | (uint64_t)(lo[1] >> 16);
    return (hi16 << 48) | lo48;
}

/* Metropolis sweeps t0 .. t0+nsweeps-1.  One sweep visits the colour classes
 * in order 0..ncol-1; inside a class vertices in ascending original id (a
 * class is an independent set, so the order inside it does not matter); for
 * each vertex every local replica attempts one flip.  Ei (may be NULL) is
 * tracked incrementally.  Returns accepted flips. */
int64_t or_sweeps(const or_run *R, int8_t *s, int64_t *Ei, uint32_t t0, int32_t nsweeps)
{
    int32_t n = R->n;
    int64_t slot0 = run_slot0(R);
    int64_t nrep = run_nrep(R);
    uint32_t planes[64];
    int64_t accepted = 0;
    for (int32_t ts = 0; ts < nsweeps; ++ts) {
        uint32_t t = t0 + (uint32_t)ts;
        for (int32_t c = 0; c < R->ncol; ++c) {
            for (int32_t i = 0; i < n; ++i) {
                if (R->colour[i] != c)
                    continue;
                int64_t cached_g = -1;
                for (int64_t rl = 0; rl < nrep; ++rl) {
                    int64_t r = slot0 + rl;
                    int32_t k = (int32_t)(r % R->K);
                    int8_t *sr = s + rl * n;
                    int accept;
                    int64_t dEi = 0;
                    if (R->wi) {
                        int64_t h = 0; /* h_i = sum_j J_ij s_j */
                        for (int64_t e = R->rp[i]; e < R->rp[i + 1]; ++e)
                            h += (int64_t)R->wi[e] * sr[R->col[e]];
                        dEi = -2 * (int64_t)sr[i] * h; /* dE = -2 s_i h_i */
                        if (dEi <= 0) {
                            accept = 1;
                        } else {
                            uint64_t T = or_threshold_int(R->beta[k], dEi);
                            uint64_t U;
                            if (R->rng == RNG_PLANE) {
                                if (cached_g != (r >> 5)) {
                                    cached_g = r >> 5;
                                    plane_words(R->seed, (uint32_t)i, t, (uint32_t)cached_g, planes);
                                }
                                U = plane_u64(planes, r);
                            } else {
                                U = word_u64(R->seed, (uint32_t)i, t, r);
                            }
                            accept = U < T;
                        }
                    } else {
                        float h = 0.0f; /* left fold in row order, RN, no FMA */
                        for (int64_t e = R->rp[i]; e < R->rp[i + 1]; ++e) {
                            float term = sr[R->col[e]] > 0 ? R->wf[e] : -R->wf[e];
                            h = h + term;
                        }
                        float dE = sr[i] > 0 ? -2.0f * h : 2.0f * h;
                        if (dE <= 0.0f) {
                            accept = 1;
                        } else {
                            uint64_t T = or_threshold_f32(R->beta[k], dE);
                            uint64_t U = word_u64(R->seed, (uint32_t)i, t, r);
                            accept = U < T;
                        }
                    }
                    if (accept) {
                        sr[i] = (int8_t)-sr[i];
                        if (Ei)
                            Ei[rl] += dEi;
                        ++accepted;
                    }
                }
            }
        }
    }
    return accepted;
}

/* Replica exchange number e for the copies of this call (integer weights).
 * For each copy c and k = e%2, e%2+2, ... with k+1 < K: a = slot (c,k),
 * b = slot (c,k+1), d = E_b - E_a; accept iff d >= 0 or
 * U64x(k,e,c) < p64((beta_{k+1}-beta_k) d)  [min(1, exp(dbeta*dH)), S:288,
 * S:292]; on acceptance the two configurations, energies and walker ids swap
 * slots ("exchanges replicas across temperatures").
 * U64x = (w0<<32)|w1 of Philox(k, e, c, EXCH<<24).  Returns accepted swaps. */
int64_t or_exchange(const or_run *R, int8_t *s, int64_t *Ei, int64_t *walker, uint32_t e)
{
    int32_t n = R->n;
    int32_t K = R->K;
    int64_t acc = 0;
    if (R->slot_hi > R->slot_lo)
        return -1; /* slot subsets carry no complete PT ladder */
    int8_t *tmp = (int8_t *)malloc((size_t)n);
    for (int32_t c = R->copy_begin; c < R->copy_end; ++c) {
        for (int32_t k = (int32_t)(e % 2u); k + 1 < K; k += 2) {
            int64_t a = (int64_t)(c - R->copy_begin) * K + k;
            int64_t b = a + 1;
            int64_t d = Ei[b] - Ei[a];
            int accept;
            if (d >= 0) {
                accept = 1;
            } else {
                uint32_t w[4];
                philox_at(R->seed, (uint32_t)k, e, (uint32_t)c, (uint32_t)ST_EXCH << 24, w);
                uint64_t U = ((uint64_t)w[0] << 32) | (uint64_t)w[1];
                accept = U < or_threshold_exch(R->beta[k], R->beta[k + 1], d);
            }
            if (accept) {
                memcpy(tmp, s + a * n, (size_t)n);
                memcpy(s + a * n, s + b * n, (size_t)n);
                memcpy(s + b * n, tmp, (size_t)n);
                int64_t te = Ei[a]; Ei[a] = Ei[b]; Ei[b] = te;
                int64_t tw = walker[a]; walker[a] = walker[b]; walker[b] = tw;
                ++acc;
            }
        }
    }
    free(tmp);
    return acc;
}

/* Energy of one configuration (integer weights), each edge once. */
static int64_t energy_one_int(const or_run *R, const int8_t *sr)
{
    int64_t e = 0;
    for (int32_t i = 0; i < R->n; ++i)
        for (int64_t k = R->rp[i]; k < R->rp[i + 1]; ++k)
            if (R->col[k] > i)
                e += (int64_t)R->wi[k] * sr[i] * sr[R->col[k]];
    return e;
}

/* Houdayer / isoenergetic cluster move number f ("two
 * replicas at the same temperature are compared and a cluster of spins is identified,
 * after which the sign of the cluster is changed in each replica"; refs [20][21]).
 * For every copy pair (2p, 2p+1) of this call and every temperature k >= k_min:
 * X_i = [s_a(i) != s_b(i)] for a = slot (2p, k), b = slot (2p+1, k).  Seed: the first of
 * 64 candidates i_j = (w_j * n) >> 32, w_j = word (j&3) of Philox(k, f, p, ICM<<24 | j>>2),
 * with X = 1 (none: no move).  The cluster is the connected component of the seed in the
 * subgraph induced by {X = 1} (breadth-first search); its spins flip in both replicas, so
 * E_a + E_b is unchanged (zero field).  Energies are recomputed from scratch.
 * Returns the number of clusters flipped; -1 if the copy range is not pair-aligned. */
int64_t or_icm(const or_run *R, int8_t *s, int64_t *Ei, uint32_t f, int32_t k_min)
{
    int32_t n = R->n, K = R->K;
    if ((R->copy_begin & 1) || ((R->copy_end - R->copy_begin) & 1) || R->slot_hi > R->slot_lo)
        return -1;
    char *vis = (char *)malloc((size_t)n);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t moves = 0;
    for (int32_t c = R->copy_begin; c < R->copy_end; c += 2) {
        uint32_t pair = (uint32_t)(c / 2);
        for (int32_t k = k_min < 0 ? 0 : k_min; k < K; ++k) {
            int64_t ra = (int64_t)(c - R->copy_begin) * K + k, rb = ra + K;
            int8_t *sa = s + ra * n, *sb = s + rb * n;
            int32_t seed = -1;
            uint32_t w[4];
            for (int j = 0; j < 64 && seed < 0; ++j) {
                if ((j & 3) == 0)
                    philox_at(R->seed, (uint32_t)k, f, pair, ((uint32_t)ST_ICM << 24) | (uint32_t)(j >> 2), w);
                int32_t i = (int32_t)(((uint64_t)w[j & 3] * (uint64_t)n) >> 32);
                if (sa[i] != sb[i])
                    seed = i;
            }
            if (seed < 0)
                continue;
            memset(vis, 0, (size_t)n);
            int32_t head = 0, tail = 0;
            queue[tail++] = seed;
            vis[seed] = 1;
            while (head < tail) {
                int32_t i = queue[head++];
                for (int64_t e = R->rp[i]; e < R->rp[i + 1]; ++e) {
                    int32_t j = R->col[e];
                    if (!vis[j] && sa[j] != sb[j]) {
                        vis[j] = 1;
                        queue[tail++] = j;
                    }
                }
            }
            for (int32_t q = 0; q < tail; ++q) {
                sa[queue[q]] = (int8_t)-sa[queue[q]];
                sb[queue[q]] = (int8_t)-sb[queue[q]];
            }
            if (Ei && R->wi) {
                Ei[ra] = energy_one_int(R, sa);
                Ei[rb] = energy_one_int(R, sb);
            }
            ++moves;
        }
    }
    free(vis);
    free(queue);
    return moves;
}

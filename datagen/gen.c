/*
 * datagen/gen.c -- seeded synthetic inputs shared by the oracle and the CUDA path.
 *
 * This module holds NONE of the method's arithmetic (no sorting into CSR/CSC,
 * no degrees, no normalisation, no aggregation).  It only draws random graphs
 * (COO edge lists) and random feature matrices, deterministically from a seed,
 * with the shapes and structure of the paper's workloads (Table 2,
 * P:2125-2159; recipe in DESIGN.md "Input recipe").
 *
 * Generators
 *   - Chung-Lu power-law, symmetric, simple: expected degree of vertex i is
 *     proportional to (i+1)^-beta.  Both endpoints of a candidate pair are drawn
 *     i.i.d. from an alias table over the weights; self-pairs and repeated
 *     unordered pairs are rejected and redrawn until exactly `npairs` distinct
 *     unordered pairs exist; each pair is emitted in both directions (GNN
 *     datasets store every edge in both directions).
 *   - R-MAT (Graph500 quadrant probabilities), directed, simple, NOT
 *     symmetrised: ids >= V, self-loops and repeated directed pairs rejected.
 *   Both then relabel vertices by a seeded random permutation (no id locality)
 *   and shuffle the COO order (so the builder's sort is exercised).
 *
 * PRNG: xoshiro256** seeded through splitmix64 (sequential generators);
 * features use a counter-based hash of (seed,row,col) so any rank can
 * regenerate any element independently.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------- PRNG --- */
static inline uint64_t splitmix64_next(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s[4]; } xo256;
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static void xo_seed(xo256 *r, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; i++) r->s[i] = splitmix64_next(&sm);
}
static inline uint64_t xo_next(xo256 *r) {
    uint64_t *s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}
/* uniform double in [0,1) with 53 random bits */
static inline double xo_unif(xo256 *r) { return (double)(xo_next(r) >> 11) * 0x1.0p-53; }
/* unbiased integer in [0,n) (Lemire's method with rejection) */
static inline uint64_t xo_below(xo256 *r, uint64_t n) {
    __uint128_t m = (__uint128_t)xo_next(r) * n;
    uint64_t l = (uint64_t)m;
    if (l < n) {
        uint64_t t = (0 - n) % n;
        while (l < t) { m = (__uint128_t)xo_next(r) * n; l = (uint64_t)m; }
    }
    return (uint64_t)(m >> 64);
}

/* ------------------------------------------------------------ hash set --- */
typedef struct { uint64_t *slot; uint64_t mask; } hset;
static int hs_init(hset *h, int64_t n) {
    uint64_t cap = 1024;
    while (cap < (uint64_t)(2 * n + 16)) cap <<= 1;
    h->slot = (uint64_t *)calloc(cap, sizeof(uint64_t));
    h->mask = cap - 1;
    return h->slot ? 0 : -1;
}
/* returns 1 if inserted, 0 if already present (keys stored +1, 0 = empty) */
static inline int hs_insert(hset *h, uint64_t key) {
    uint64_t k1 = key + 1, i = mix64(key) & h->mask;
    for (;;) {
        uint64_t v = h->slot[i];
        if (v == 0) { h->slot[i] = k1; return 1; }
        if (v == k1) return 0;
        i = (i + 1) & h->mask;
    }
}

/* --------------------------------------------- relabel + shuffle (both) --- */
static int relabel_and_shuffle(xo256 *r, int64_t V, int64_t E, int64_t *src, int64_t *dst) {
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)(V > 0 ? V : 1));
    if (!perm) return -1;
    for (int64_t i = 0; i < V; i++) perm[i] = i;
    for (int64_t i = V - 1; i > 0; i--) {
        int64_t j = (int64_t)xo_below(r, (uint64_t)(i + 1));
        int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    for (int64_t e = 0; e < E; e++) { src[e] = perm[src[e]]; dst[e] = perm[dst[e]]; }
    free(perm);
    for (int64_t i = E - 1; i > 0; i--) {
        int64_t j = (int64_t)xo_below(r, (uint64_t)(i + 1));
        int64_t ts = src[i]; src[i] = src[j]; src[j] = ts;
        int64_t td = dst[i]; dst[i] = dst[j]; dst[j] = td;
    }
    return 0;
}

/* --------------------------------------------------------- Chung-Lu ------ */
/* Emits 2*npairs directed edges into src/dst (caller-allocated).
 * Returns 0 on success, -1 OOM, -2 target unreachable within the draw budget. */
int gen_chung_lu(int64_t V, int64_t npairs, double beta, uint64_t seed,
                 int64_t *src, int64_t *dst) {
    if (V < 2 || npairs < 0) return npairs == 0 ? 0 : -2;
    if ((double)npairs > 0.5 * (double)V * (double)(V - 1)) return -2;
    xo256 rng; xo_seed(&rng, seed);
    /* Vose alias table over w_i = (i+1)^-beta */
    double *prob = (double *)malloc(sizeof(double) * V);
    int64_t *alias = (int64_t *)malloc(sizeof(int64_t) * V);
    int64_t *small = (int64_t *)malloc(sizeof(int64_t) * V);
    int64_t *large = (int64_t *)malloc(sizeof(int64_t) * V);
    if (!prob || !alias || !small || !large) { free(prob); free(alias); free(small); free(large); return -1; }
    double W = 0.0;
    for (int64_t i = 0; i < V; i++) { prob[i] = pow((double)(i + 1), -beta); W += prob[i]; }
    int64_t ns = 0, nl = 0;
    for (int64_t i = 0; i < V; i++) {
        prob[i] = prob[i] * (double)V / W;
        if (prob[i] < 1.0) small[ns++] = i; else large[nl++] = i;
    }
    while (ns > 0 && nl > 0) {
        int64_t s = small[--ns], l = large[--nl];
        alias[s] = l;
        prob[l] = (prob[l] + prob[s]) - 1.0;
        if (prob[l] < 1.0) small[ns++] = l; else large[nl++] = l;
    }
    while (nl > 0) { int64_t l = large[--nl]; prob[l] = 1.0; alias[l] = l; }
    while (ns > 0) { int64_t s = small[--ns]; prob[s] = 1.0; alias[s] = s; }
    free(small); free(large);

    hset hs;
    if (hs_init(&hs, npairs) != 0) { free(prob); free(alias); return -1; }
    int64_t got = 0;
    uint64_t budget = (uint64_t)npairs * 64 + 1000000, tries = 0;
    while (got < npairs) {
        if (++tries > budget) { free(prob); free(alias); free(hs.slot); return -2; }
        int64_t c0 = (int64_t)xo_below(&rng, (uint64_t)V);
        int64_t u = (xo_unif(&rng) < prob[c0]) ? c0 : alias[c0];
        int64_t c1 = (int64_t)xo_below(&rng, (uint64_t)V);
        int64_t v = (xo_unif(&rng) < prob[c1]) ? c1 : alias[c1];
        if (u == v) continue;
        uint64_t lo = (uint64_t)(u < v ? u : v), hi = (uint64_t)(u < v ? v : u);
        if (!hs_insert(&hs, lo * (uint64_t)V + hi)) continue;
        src[2 * got] = u;     dst[2 * got] = v;
        src[2 * got + 1] = v; dst[2 * got + 1] = u;
        got++;
    }
    free(prob); free(alias); free(hs.slot);
    return relabel_and_shuffle(&rng, V, 2 * npairs, src, dst);
}

/* ------------------------------------------------------------ R-MAT ------ */
/* Emits exactly E distinct directed non-loop edges with ids < V. */
int gen_rmat(int scale, int64_t V, int64_t E, double a, double b, double c,
             uint64_t seed, int64_t *src, int64_t *dst) {
    if (E == 0) return 0;
    if (V < 2 || scale < 1 || scale > 40 || V > ((int64_t)1 << scale)) return -2;
    if ((double)E > (double)V * (double)(V - 1)) return -2;
    xo256 rng; xo_seed(&rng, seed);
    hset hs;
    if (hs_init(&hs, E) != 0) return -1;
    int64_t got = 0;
    uint64_t budget = (uint64_t)E * 256 + 1000000, tries = 0;
    const double ab = a + b, abc = a + b + c;
    while (got < E) {
        if (++tries > budget) { free(hs.slot); return -2; }
        int64_t u = 0, v = 0;
        for (int l = 0; l < scale; l++) {
            double r = xo_unif(&rng);
            int bu, bv;
            if (r < a) { bu = 0; bv = 0; }
            else if (r < ab) { bu = 0; bv = 1; }
            else if (r < abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u = (u << 1) | bu; v = (v << 1) | bv;
        }
        if (u >= V || v >= V || u == v) continue;
        if (!hs_insert(&hs, (uint64_t)u * (uint64_t)V + (uint64_t)v)) continue;
        src[got] = u; dst[got] = v; got++;
    }
    free(hs.slot);
    return relabel_and_shuffle(&rng, V, E, src, dst);
}

/* ----------------------------------------------------------- Kronecker --- */
/* Graph500-style Kronecker graph (the paper's Kron-25, PAPER Table 2:
 * 2^25 vertices, 2^30 edges): npairs R-MAT draws with quadrant probabilities
 * (a, b, c, 1-a-b-c), duplicates and self-loops KEPT (the edge count is exact),
 * each emitted in both directions, then a seeded vertex relabelling.  Every
 * draw k uses a counter-based stream (seed, k, level), so the result does not
 * depend on the number of threads. */
int gen_kron(int scale, int64_t npairs, double a, double b, double c, uint64_t seed, int64_t *src, int64_t *dst) {
    if (scale < 1 || scale > 40) return -2;
    const int64_t V = (int64_t)1 << scale;
    const double ab = a + b, abc = a + b + c;
    const uint64_t s0 = mix64(seed ^ 0xA0761D6478BD642FULL);
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < npairs; k++) {
        uint64_t st = mix64(s0 + (uint64_t)k * 0x9E3779B97F4A7C15ULL);
        int64_t u = 0, v = 0;
        for (int l = 0; l < scale; l++) {
            st = mix64(st + 0xD1B54A32D192ED03ULL);
            double r = (double)(st >> 11) * 0x1.0p-53;
            int bu, bv;
            if (r < a) { bu = 0; bv = 0; }
            else if (r < ab) { bu = 0; bv = 1; }
            else if (r < abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u = (u << 1) | bu; v = (v << 1) | bv;
        }
        src[2 * k] = u; dst[2 * k] = v;
        src[2 * k + 1] = v; dst[2 * k + 1] = u;
    }
    /* seeded relabelling (Fisher-Yates), applied in parallel */
    xo256 rng; xo_seed(&rng, seed);
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    if (!perm) return -1;
    for (int64_t i = 0; i < V; i++) perm[i] = i;
    for (int64_t i = V - 1; i > 0; i--) {
        int64_t j = (int64_t)xo_below(&rng, (uint64_t)(i + 1));
        int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < 2 * npairs; e++) { src[e] = perm[src[e]]; dst[e] = perm[dst[e]]; }
    free(perm);
    return 0;
}

/* ------------------------------------------------------- features -------- */
/* Counter-based U[lo,hi) fp32 with 24 random bits per element: element (r,c)
 * depends only on (seed,r,c).  Padding columns [cols,ld) are set to 0. */
void gen_uniform_f32(uint64_t seed, int64_t rows, int64_t cols, int64_t ld,
                     float lo, float hi, float *out) {
    const uint64_t s0 = mix64(seed ^ 0x5DEECE66DULL);
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; r++) {
        const uint64_t sr = mix64(s0 + (uint64_t)r * 0x9E3779B97F4A7C15ULL);
        float *row = out + r * ld;
        for (int64_t c = 0; c < cols; c++) {
            uint64_t h = mix64(sr ^ ((uint64_t)c * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
            float u = (float)(h >> 40) * 0x1.0p-24f; /* exact in fp32 */
            row[c] = lo + (hi - lo) * u;
        }
        for (int64_t c = cols; c < ld; c++) row[c] = 0.0f;
    }
}

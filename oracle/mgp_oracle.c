/*
 * mgp_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C CPU restatement of the reference resampling hot path
 * (arXiv 2109.13504 "Megopolis", reference package pkg/src/megores).
 * It is the parity checker for the CUDA library: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2109_13504_b200) never links or calls it.
 *
 * Parity of this restatement is PINNED against golden vectors produced by the
 * unmodified reference (tests/golden/make_golden.py -> golden.npz/json), see
 * tests/test_oracle_golden.py.
 *
 * Every function cites the reference file:line it restates
 * (M/ = pkg/src/megores/).
 *
 * Two random streams:
 *   rng = 0 ("megores"): the reference's keyed splitmix64 hash, bit-exact.
 *   rng = 1 ("philox") : Philox4x32-10 words with the reference's counter layout
 *                        (DESIGN.md "Philox stream"); u = word * 2^-32,
 *                        uint_below(n) = (word * n) >> 32.  The acceptance
 *                        arithmetic is identical (FP64, zero rule).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>
#include <unistd.h>

#define M_LANE 0x9E3779B97F4A7C15ULL /* M/rng.py:45 */
#define M_CTR 0xD1B54A32D192ED03ULL  /* M/rng.py:46 */
#define M_SALT 0x8CB92BA72F3D8DD7ULL /* M/rng.py:47 */
#define MIX1 0xBF58476D1CE4E5B9ULL   /* M/rng.py:48 */
#define MIX2 0x94D049BB133111EBULL   /* M/rng.py:49 */
#define WARP_LANE_BASE (1ULL << 61)  /* M/rng.py:42 */
#define GLOBAL_OFFSET_LANE (1ULL << 62) /* M/rng.py:43 */
#define INV_2_53 (1.0 / 9007199254740992.0) /* M/rng.py:55 */

/* ------------------------------------------------------------------------ */
/* megores stream                                                           */

/* splitmix64 finaliser, M/rng.py:85-89 */
uint64_t mgo_mix(uint64_t x) {
    x = (x ^ (x >> 30)) * MIX1;
    x = (x ^ (x >> 27)) * MIX2;
    return x ^ (x >> 31);
}

/* keyed hash, M/rng.py:92-102 (wrap-around uint64 arithmetic) */
uint64_t mgo_hash_u64(uint64_t seed, uint64_t lane, uint64_t counter, uint64_t salt) {
    uint64_t base = mgo_mix(seed + M_LANE);
    return mgo_mix(base + lane * M_LANE + counter * M_CTR + salt * M_SALT);
}

/* u01, M/rng.py:105-108: float(h >> 11) * 2^-53 */
double mgo_u01(uint64_t seed, uint64_t lane, uint64_t counter) {
    return (double)(mgo_hash_u64(seed, lane, counter, 0) >> 11) * INV_2_53;
}

/* uint_below, M/rng.py:111-121: int64(u01 * float(n)), clamped to n-1 */
int64_t mgo_uint_below(uint64_t seed, uint64_t lane, uint64_t counter, int64_t n) {
    int64_t v = (int64_t)(mgo_u01(seed, lane, counter) * (double)n);
    if (v >= n) v = n - 1;
    return v;
}

/* derive_seed, M/rng.py:180-191 */
uint64_t mgo_derive_seed(uint64_t seed, const uint64_t *parts, int nparts) {
    uint64_t h = mgo_mix(seed + M_LANE);
    for (int i = 0; i < nparts; ++i) h = mgo_mix(h ^ (parts[i] * M_CTR + M_SALT));
    return h;
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11; constants as Random123 / curand)     */

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void mgo_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PHILOX_W0; k1 += PHILOX_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* word t of the (seed, lane) philox stream: block t>>2, word t&3 */
uint32_t mgo_philox_word(uint64_t seed, uint64_t lane, uint64_t t) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint64_t blk = t >> 2;
    uint32_t ctr[4] = {(uint32_t)lane, (uint32_t)(lane >> 32), (uint32_t)blk, (uint32_t)(blk >> 32)};
    uint32_t out[4];
    mgo_philox4x32_10(ctr, key, out);
    return out[t & 3];
}

static double philox_u01(uint64_t seed, uint64_t lane, uint64_t t) {
    return (double)mgo_philox_word(seed, lane, t) * (1.0 / 4294967296.0);
}

static int64_t philox_uint_below(uint64_t seed, uint64_t lane, uint64_t t, int64_t n) {
    return (int64_t)(((uint64_t)mgo_philox_word(seed, lane, t) * (uint64_t)n) >> 32);
}

/* Stream dispatch with a per-thread draw context: the megores key base
 * mix(seed + M_LANE) is computed once (M/rng.py:95 recomputes it per call; the
 * value is identical), and the last Philox block is cached (one block serves four
 * consecutive draws).  Results are identical to the per-call functions above. */
typedef struct {
    int rng;
    uint64_t seed, base;
    uint64_t blk_lane, blk_idx;
    int blk_valid;
    uint32_t blk[4];
} draw_ctx;

static inline void ctx_init(draw_ctx *c, int rng, uint64_t seed) {
    c->rng = rng; c->seed = seed; c->base = mgo_mix(seed + M_LANE); c->blk_valid = 0;
}

static inline uint64_t ctx_hash(const draw_ctx *c, uint64_t lane, uint64_t ctr) {
    return mgo_mix(c->base + lane * M_LANE + ctr * M_CTR);
}

static inline uint32_t ctx_word(draw_ctx *c, uint64_t lane, uint64_t t) {
    uint64_t b = t >> 2;
    if (!c->blk_valid || c->blk_lane != lane || c->blk_idx != b) {
        uint32_t key[2] = {(uint32_t)c->seed, (uint32_t)(c->seed >> 32)};
        uint32_t ctr[4] = {(uint32_t)lane, (uint32_t)(lane >> 32), (uint32_t)b, (uint32_t)(b >> 32)};
        mgo_philox4x32_10(ctr, key, c->blk);
        c->blk_lane = lane; c->blk_idx = b; c->blk_valid = 1;
    }
    return c->blk[t & 3];
}

static inline double ctx_u(draw_ctx *c, uint64_t lane, uint64_t ctr) {
    if (c->rng == 0) return (double)(ctx_hash(c, lane, ctr) >> 11) * INV_2_53;
    return (double)ctx_word(c, lane, ctr) * (1.0 / 4294967296.0);
}

static inline int64_t ctx_below(draw_ctx *c, uint64_t lane, uint64_t ctr, int64_t n) {
    if (c->rng == 0) {
        int64_t v = (int64_t)((double)(ctx_hash(c, lane, ctr) >> 11) * INV_2_53 * (double)n);
        return v >= n ? n - 1 : v;
    }
    return (int64_t)(((uint64_t)ctx_word(c, lane, ctr) * (uint64_t)n) >> 32);
}

static inline double draw_u(int rng, uint64_t seed, uint64_t lane, uint64_t ctr) {
    return rng == 0 ? mgo_u01(seed, lane, ctr) : philox_u01(seed, lane, ctr);
}
static inline int64_t draw_below(int rng, uint64_t seed, uint64_t lane, uint64_t ctr, int64_t n) {
    return rng == 0 ? mgo_uint_below(seed, lane, ctr, n) : philox_uint_below(seed, lane, ctr, n);
}

/* ------------------------------------------------------------------------ */
/* Resamplers                                                               */

/* acceptance rule, M/resample.py:118-122 (FP64; float32 weights promoted) */
static inline int accepts(double u, double wk, double wj) {
    if (wj == 0.0 && wk == 0.0) return 0;
    return u * wk <= wj;
}

static inline double wload(const void *w, int dtype, int64_t i) {
    return dtype == 0 ? (double)((const float *)w)[i] : ((const double *)w)[i];
}

/* megopolis_offsets, M/resample.py:263-265 (uniform_int_at on GLOBAL_OFFSET_LANE) */
void mgo_offsets(int64_t n, int64_t b, uint64_t seed, int rng, int64_t *out) {
    for (int64_t t = 0; t < b; ++t) out[t] = draw_below(rng, seed, GLOBAL_OFFSET_LANE, (uint64_t)t, n);
}

enum { K_METROPOLIS = 0, K_C1 = 1, K_C2 = 2, K_MEGOPOLIS = 3 };

/*
 * kind 0: _metropolis_kernel M/resample.py:125-138
 * kind 1: _c1_kernel         M/resample.py:141-158
 * kind 2: _c2_kernel         M/resample.py:161-177
 * kind 3: _megopolis_kernel  M/resample.py:180-198 (offsets from mgo_offsets)
 *
 * Precondition checks (M/resample.py:96-108, 84-93) live in oracle.py, as in
 * the reference they live in the Python wrappers.  Ancestors for particles
 * [p0, p1) only (the rest of anc is untouched) so a bounded sample of a large
 * workload can be timed / checked.
 */
typedef struct {
    int kind, dtype, rng;
    const void *w;
    int64_t n, b, warp, n_w, n_part, p0, p1;
    uint64_t seed;
    const int64_t *off;
    int64_t *anc;
} job_t;

static void resample_slice(const job_t *J) {
    const int64_t n = J->n, b = J->b, warp = J->warp, n_w = J->n_w, n_part = J->n_part;
    const int dtype = J->dtype, kind = J->kind;
    const void *w = J->w;
    draw_ctx C, CW;  /* particle-lane and warp-lane draw contexts */
    ctx_init(&C, J->rng, J->seed);
    ctx_init(&CW, J->rng, J->seed);
    for (int64_t i = J->p0; i < J->p1; ++i) {
        uint64_t lane = (uint64_t)i;
        int64_t k = i;
        if (kind == K_METROPOLIS) {
            for (int64_t r = 0; r < b; ++r) {
                double u = ctx_u(&C, lane, (uint64_t)(2 * r));
                int64_t j = ctx_below(&C, lane, (uint64_t)(2 * r + 1), n);
                if (accepts(u, wload(w, dtype, k), wload(w, dtype, j))) k = j;
            }
        } else if (kind == K_C1) {
            uint64_t wl = WARP_LANE_BASE + (uint64_t)(i / warp);
            int64_t lo = ctx_below(&CW, wl, 0, n_part) * n_w;
            for (int64_t r = 0; r < b; ++r) {
                double u = ctx_u(&C, lane, (uint64_t)(2 * r));
                int64_t j = lo + ctx_below(&C, lane, (uint64_t)(2 * r + 1), n_w);
                if (accepts(u, wload(w, dtype, k), wload(w, dtype, j))) k = j;
            }
        } else if (kind == K_C2) {
            uint64_t wl = WARP_LANE_BASE + (uint64_t)(i / warp);
            for (int64_t r = 0; r < b; ++r) {
                double u = ctx_u(&C, lane, (uint64_t)(2 * r));
                int64_t p = ctx_below(&CW, wl, (uint64_t)r, n_part);
                int64_t j = p * n_w + ctx_below(&C, lane, (uint64_t)(2 * r + 1), n_w);
                if (accepts(u, wload(w, dtype, k), wload(w, dtype, j))) k = j;
            }
        } else {
            int64_t i_al = i - i % warp;
            for (int64_t r = 0; r < b; ++r) {
                int64_t ob = J->off[r];
                int64_t o_al = ob - ob % warp;
                int64_t o_un = (i + ob) % warp;
                int64_t j = (i_al + o_al + o_un) % n;
                double u = ctx_u(&C, lane, (uint64_t)r);
                if (accepts(u, wload(w, dtype, k), wload(w, dtype, j))) k = j;
            }
        }
        J->anc[i] = k;
    }
}

static void *slice_thread(void *arg) {
    resample_slice((const job_t *)arg);
    return NULL;
}

int mgo_num_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

int mgo_resample_range(int kind, const void *w, int dtype, int64_t n, int64_t b, uint64_t seed,
                       int64_t warp, int64_t n_w, int rng, int64_t p0, int64_t p1, int64_t *anc,
                       int nthreads) {
    int64_t *off = NULL;
    if (kind == K_MEGOPOLIS) {
        off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(b > 0 ? b : 1));
        if (!off) return -1;
        mgo_offsets(n, b, seed, rng, off);
    }
    if (nthreads <= 0) nthreads = mgo_num_threads();
    if (nthreads > 256) nthreads = 256;
    int64_t total = p1 - p0;
    if (total < (int64_t)nthreads * 64) nthreads = 1;
    job_t jobs[256];
    pthread_t th[256];
    int64_t per = (total + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        job_t *J = &jobs[t];
        J->kind = kind; J->dtype = dtype; J->rng = rng; J->w = w; J->n = n; J->b = b;
        J->warp = warp; J->n_w = n_w; J->n_part = n_w > 0 ? n / n_w : 0; J->seed = seed;
        J->off = off; J->anc = anc;
        J->p0 = p0 + per * t;
        J->p1 = J->p0 + per < p1 ? J->p0 + per : p1;
        if (J->p0 > p1) J->p0 = p1;
    }
    int launched = 0;
    for (int t = 1; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, slice_thread, &jobs[t]) == 0) launched = t; else { resample_slice(&jobs[t]); }
    resample_slice(&jobs[0]);
    for (int t = 1; t <= launched; ++t) pthread_join(th[t], NULL);
    free(off);
    return 0;
}

int mgo_resample(int kind, const void *w, int dtype, int64_t n, int64_t b, uint64_t seed,
                 int64_t warp, int64_t n_w, int rng, int64_t *anc, int nthreads) {
    return mgo_resample_range(kind, w, dtype, n, b, seed, warp, n_w, rng, 0, n, anc, nthreads);
}

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation (np.add.reduce on a contiguous float64 array),
 * which is what np.asarray(w, float64).mean() uses at M/bench.py:119 and
 * T/conftest.py:29.  Verified bit-for-bit against numpy 2.3 (golden "means"). */

static double pairwise(const void *a, int dtype, int64_t lo, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += wload(a, dtype, lo + i);
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; ++j) r[j] = wload(a, dtype, lo + j);
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += wload(a, dtype, lo + i + j);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += wload(a, dtype, lo + i);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, dtype, lo, n2) + pairwise(a, dtype, lo + n2, n - n2);
}

double mgo_pairwise_sum(const void *a, int dtype, int64_t n) { return pairwise(a, dtype, 0, n); }

/* ancestors_to_offspring, M/resample.py:361-368 (range check in oracle.py) */
void mgo_offspring(const int64_t *anc, int64_t n_anc, int64_t n, int64_t *counts) {
    memset(counts, 0, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n_anc; ++i) counts[anc[i]] += 1;
}

/* apply_ancestors, M/resample.py:371-377 (row gather of row_bytes each) */
void mgo_gather(const void *states, int64_t row_bytes, const int64_t *anc, int64_t n, void *out) {
    for (int64_t i = 0; i < n; ++i)
        memcpy((char *)out + i * row_bytes, (const char *)states + anc[i] * row_bytes, (size_t)row_bytes);
}


/* ------------------------------------------------------------------------ */
/* Prefix-sum resamplers (M/resample.py:288-354)                            */

/* np.cumsum(values) (M/resample.py:288-291): a sequential left-to-right scan in the
 * array's own dtype (float32 for "single").  Built with -ffp-contract=off and without
 * fast-math, so every add is one IEEE binary32/binary64 round-to-nearest-even. */
void mgo_cumsum(const void *w, int dtype, int64_t n, void *out) {
    if (n <= 0) return;
    if (dtype == 0) {
        const float *a = (const float *)w;
        float *o = (float *)out, s = a[0];
        o[0] = s;
        for (int64_t k = 1; k < n; ++k) { s = s + a[k]; o[k] = s; }
    } else {
        const double *a = (const double *)w;
        double *o = (double *)out, s = a[0];
        o[0] = s;
        for (int64_t k = 1; k < n; ++k) { s = s + a[k]; o[k] = s; }
    }
}

/* multinomial (M/resample.py:295-304): u_i = uniform01_at(seed, i, 0) * total cast to the
 * weight dtype, ancestor = searchsorted(inclusive, u_i, side="right") clamped to n-1.
 * `cum` is the inclusive prefix (mgo_cumsum). */
void mgo_multinomial(const void *cum, int dtype, int64_t n, uint64_t seed, int64_t *anc) {
    const uint64_t base = mgo_mix(seed + M_LANE);
    const double total = dtype == 0 ? (double)((const float *)cum)[n - 1] : ((const double *)cum)[n - 1];
    for (int64_t i = 0; i < n; ++i) {
        const double ud = (double)(mgo_mix(base + (uint64_t)i * M_LANE) >> 11) * INV_2_53 * total;
        int64_t lo = 0, hi = n; /* first index with cum > u */
        if (dtype == 0) {
            const float u = (float)ud, *c = (const float *)cum;
            while (lo < hi) { int64_t mid = lo + (hi - lo) / 2; if (c[mid] <= u) lo = mid + 1; else hi = mid; }
        } else {
            const double *c = (const double *)cum;
            while (lo < hi) { int64_t mid = lo + (hi - lo) / 2; if (c[mid] <= ud) lo = mid + 1; else hi = mid; }
        }
        anc[i] = lo < n - 1 ? lo : n - 1;
    }
}

/* systematic_improved (M/resample.py:307-336): one shared u0 = uniform01_at(seed,
 * GLOBAL_OFFSET_LANE, 0); target_i = (i + u0) / n * total in float64; the forward/backward
 * scans settle on the first index a with float64(cum[a]) >= target_i, or n-1. */
void mgo_systematic(const void *cum, int dtype, int64_t n, uint64_t seed, int64_t *anc) {
    const double u0 = mgo_u01(seed, GLOBAL_OFFSET_LANE, 0);
    const double total = dtype == 0 ? (double)((const float *)cum)[n - 1] : ((const double *)cum)[n - 1];
    for (int64_t i = 0; i < n; ++i) {
        const double target = ((double)i + u0) / (double)n * total;
        int64_t lo = 0, hi = n; /* first index with cum >= target */
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            const double c = dtype == 0 ? (double)((const float *)cum)[mid] : ((const double *)cum)[mid];
            if (c < target) lo = mid + 1; else hi = mid;
        }
        anc[i] = lo < n - 1 ? lo : n - 1;
    }
}

/*
 * oracle.c -- CPU restatement of the reference dynamic random-walk path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Not part of the product; the
 * product path (paper_2512_00705_b200/csrc) never links or loads this file.
 *
 * Build: gcc -O2 -ffp-contract=off (the reference is built with plain -O2 on
 * baseline x86-64, which has no FMA, so no multiply-add is ever contracted;
 * SURVEY.md Appendix A "FP contraction").  All citations are relative to
 * /root/reference/proj.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* errors                                                                    */
/* ------------------------------------------------------------------------ */

static __thread char tl_err[512];
static char g_err[512];
static pthread_mutex_t g_err_mu = PTHREAD_MUTEX_INITIALIZER;

const char* orc_last_error(void) { return tl_err[0] ? tl_err : g_err; }

static void set_err(const char* msg) {
    snprintf(tl_err, sizeof tl_err, "%s", msg);
}

/* ------------------------------------------------------------------------ */
/* RNG: SplitMix64 / derive_seed  (include/dynwalk/rng.hpp:10-25)            */
/* ------------------------------------------------------------------------ */

static uint64_t splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
    uint64_t st = seed ^ (stream * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL);
    splitmix_next(&st);
    return splitmix_next(&st);
}

/* std::mt19937_64 (C++ [rand.predef]): the engine behind CountingRng
 * (rng.hpp:31-57).  Parameters fixed by the standard. */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

static uint64_t mt64_next(mt64* r) {
    if (r->mti >= 312) {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
            r->mt[i] = r->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        }
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

void orc_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out) {
    mt64 r;
    mt64_seed(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = mt64_next(&r);
}

/* Philox4x32-10 (Salmon et al. 2011; same constants as cuRAND
 * curand_philox4x32_x.h:88-91).  Pinned by Random123 known-answer vectors in
 * tests/test_oracle.py. */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* Walker stream: key = seed, counter = (draw>>1, step,
 * qid lo, qid hi); draw 2k is words (1,0) of block k, draw 2k+1 words (3,2). */
uint64_t orc_walker_draw(uint64_t seed, uint64_t qid, uint32_t step, uint64_t idx) {
    const uint32_t ctr[4] = {(uint32_t)(idx >> 1), step, (uint32_t)qid, (uint32_t)(qid >> 32)};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return (idx & 1) ? (((uint64_t)o[3] << 32) | o[2]) : (((uint64_t)o[1] << 32) | o[0]);
}

/* Draw-counting RNG with the reference bit maps (rng.hpp:40-50).  Kind
 * MT19937 = CountingRng(derive_seed(seed, qid)) per query
 * (runtime.cpp:65); kind PHILOX = counter stream re-keyed every step. */
typedef struct {
    int kind;
    uint64_t draws;
    mt64 mt;
    uint64_t seed, qid;
    uint32_t step;
    uint64_t idx;
    uint64_t cache_block;
    uint32_t cache[4];
    int have_cache;
} wrng;

static uint64_t wrng_next(wrng* r) {
    ++r->draws;
    if (r->kind == ORC_RNG_MT19937) return mt64_next(&r->mt);
    const uint64_t idx = r->idx++;
    const uint64_t block = idx >> 1;
    if (!r->have_cache || r->cache_block != block) {
        const uint32_t ctr[4] = {(uint32_t)block, r->step, (uint32_t)r->qid,
                                 (uint32_t)(r->qid >> 32)};
        const uint32_t key[2] = {(uint32_t)r->seed, (uint32_t)(r->seed >> 32)};
        orc_philox4x32_10(ctr, key, r->cache);
        r->cache_block = block;
        r->have_cache = 1;
    }
    return (idx & 1) ? (((uint64_t)r->cache[3] << 32) | r->cache[2])
                     : (((uint64_t)r->cache[1] << 32) | r->cache[0]);
}

static double wrng_uniform01(wrng* r) { return (double)(wrng_next(r) >> 11) * 0x1.0p-53; }
static double wrng_open01(wrng* r) { return ((double)(wrng_next(r) >> 11) + 0.5) * 0x1.0p-53; }
static uint64_t wrng_bounded(wrng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)wrng_next(r) * n) >> 64);
}

/* plain CountingRng for generators (rng.hpp:31-57) */
typedef struct {
    mt64 mt;
} crng;
static void crng_init(crng* r, uint64_t seed) { mt64_seed(&r->mt, seed); }
static uint64_t crng_next(crng* r) { return mt64_next(&r->mt); }
static double crng_uniform01(crng* r) { return (double)(crng_next(r) >> 11) * 0x1.0p-53; }
static double crng_open01(crng* r) { return ((double)(crng_next(r) >> 11) + 0.5) * 0x1.0p-53; }
static uint64_t crng_bounded(crng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)crng_next(r) * n) >> 64);
}

/* ------------------------------------------------------------------------ */
/* Graph (src/graph.cpp)                                                     */
/* ------------------------------------------------------------------------ */

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) {
        fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
        abort();
    }
    return p;
}

void orc_graph_free(orc_graph* g) {
    if (!g) return;
    free(g->row);
    free(g->col);
    free(g->prop);
    free(g->label);
    free(g->nmax);
    free(g->nsum);
    free(g);
}

/* Graph::recompute_aggregates (graph.cpp:83-98): ascending edge order. */
void orc_recompute_aggregates(orc_graph* g) {
    for (uint32_t v = 0; v < g->nv; ++v) {
        double mx = 0.0, sum = 0.0;
        for (uint64_t e = g->row[v]; e != g->row[v + 1]; ++e) {
            const double p = g->prop[e];
            if (p > mx) mx = p;
            sum += p;
        }
        g->nmax[v] = mx;
        g->nsum[v] = sum;
    }
}

typedef struct {
    uint32_t col;
    uint64_t pos;
} colpos;

static int colpos_cmp(const void* a, const void* b) {
    const colpos* x = (const colpos*)a;
    const colpos* y = (const colpos*)b;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* Graph::build (graph.cpp:15-81): mirror twins appended after the originals,
 * counting sort by source, per-slice stable sort by target (std::stable_sort
 * == sort by (target, original position)), aggregates. */
orc_graph* orc_graph_build(const uint32_t* src, const uint32_t* dst, const float* prop,
                           const uint16_t* label, uint64_t n, int has_labels, int mirror,
                           uint64_t nv_hint) {
    uint64_t total = n;
    if (mirror)
        for (uint64_t i = 0; i < n; ++i) total += (src[i] != dst[i]);
    uint32_t* s = (uint32_t*)xmalloc(total * sizeof(uint32_t));
    uint32_t* t = (uint32_t*)xmalloc(total * sizeof(uint32_t));
    float* p = (float*)xmalloc(total * sizeof(float));
    uint16_t* l = (uint16_t*)xmalloc(total * sizeof(uint16_t));
    for (uint64_t i = 0; i < n; ++i) {
        s[i] = src[i];
        t[i] = dst[i];
        p[i] = prop ? prop[i] : 1.0f;
        l[i] = label ? label[i] : 0;
    }
    uint64_t at = n;
    if (mirror)
        for (uint64_t i = 0; i < n; ++i)
            if (src[i] != dst[i]) {
                s[at] = dst[i];
                t[at] = src[i];
                p[at] = p[i];
                l[at] = l[i];
                ++at;
            }
    uint64_t nv = nv_hint;
    for (uint64_t i = 0; i < total; ++i) {
        if ((uint64_t)s[i] + 1 > nv) nv = (uint64_t)s[i] + 1;
        if ((uint64_t)t[i] + 1 > nv) nv = (uint64_t)t[i] + 1;
    }
    if (nv >= ORC_INVALID) {
        set_err("vertex id overflow");
        free(s); free(t); free(p); free(l);
        return NULL;
    }
    orc_graph* g = (orc_graph*)xmalloc(sizeof(orc_graph));
    g->nv = (uint32_t)nv;
    g->ne = total;
    g->row = (uint64_t*)calloc(nv + 1, sizeof(uint64_t));
    g->col = (uint32_t*)xmalloc(total * sizeof(uint32_t));
    g->prop = (float*)xmalloc(total * sizeof(float));
    g->label = has_labels ? (uint16_t*)xmalloc(total * sizeof(uint16_t)) : NULL;
    g->nmax = (double*)xmalloc(nv * sizeof(double));
    g->nsum = (double*)xmalloc(nv * sizeof(double));
    for (uint64_t i = 0; i < total; ++i) ++g->row[s[i] + 1];
    for (uint64_t v = 0; v < nv; ++v) g->row[v + 1] += g->row[v];
    uint64_t* cursor = (uint64_t*)xmalloc((nv + 1) * sizeof(uint64_t));
    memcpy(cursor, g->row, nv * sizeof(uint64_t));
    for (uint64_t i = 0; i < total; ++i) {
        const uint64_t e = cursor[s[i]]++;
        g->col[e] = t[i];
        g->prop[e] = p[i];
        if (has_labels) g->label[e] = l[i];
    }
    free(cursor);
    colpos* buf = NULL;
    uint64_t cap = 0;
    float* pt = NULL;
    uint16_t* lt = NULL;
    for (uint64_t v = 0; v < nv; ++v) {
        const uint64_t lo = g->row[v], hi = g->row[v + 1], d = hi - lo;
        if (d < 2) continue;
        if (d > cap) {
            cap = d;
            buf = (colpos*)realloc(buf, cap * sizeof(colpos));
            pt = (float*)realloc(pt, cap * sizeof(float));
            lt = (uint16_t*)realloc(lt, cap * sizeof(uint16_t));
        }
        for (uint64_t i = 0; i < d; ++i) {
            buf[i].col = g->col[lo + i];
            buf[i].pos = i;
        }
        qsort(buf, d, sizeof(colpos), colpos_cmp);
        for (uint64_t i = 0; i < d; ++i) {
            pt[i] = g->prop[lo + buf[i].pos];
            if (has_labels) lt[i] = g->label[lo + buf[i].pos];
        }
        for (uint64_t i = 0; i < d; ++i) {
            g->col[lo + i] = buf[i].col;
            g->prop[lo + i] = pt[i];
            if (has_labels) g->label[lo + i] = lt[i];
        }
    }
    free(buf);
    free(pt);
    free(lt);
    free(s);
    free(t);
    free(p);
    free(l);
    orc_recompute_aggregates(g);
    return g;
}

orc_graph* orc_graph_from_csr(uint32_t nv, uint64_t ne, const uint64_t* row,
                              const uint32_t* col, const float* prop, const uint16_t* label) {
    orc_graph* g = (orc_graph*)xmalloc(sizeof(orc_graph));
    g->nv = nv;
    g->ne = ne;
    g->row = (uint64_t*)xmalloc((nv + 1) * sizeof(uint64_t));
    g->col = (uint32_t*)xmalloc(ne * sizeof(uint32_t));
    g->prop = (float*)xmalloc(ne * sizeof(float));
    g->label = label ? (uint16_t*)xmalloc(ne * sizeof(uint16_t)) : NULL;
    g->nmax = (double*)xmalloc(nv * sizeof(double));
    g->nsum = (double*)xmalloc(nv * sizeof(double));
    memcpy(g->row, row, (nv + 1) * sizeof(uint64_t));
    memcpy(g->col, col, ne * sizeof(uint32_t));
    memcpy(g->prop, prop, ne * sizeof(float));
    if (label) memcpy(g->label, label, ne * sizeof(uint16_t));
    orc_recompute_aggregates(g);
    return g;
}

/* Graph::has_edge (graph.cpp:114-118): std::binary_search over the slice. */
int orc_has_edge(const orc_graph* g, uint32_t v, uint32_t u) {
    uint64_t lo = g->row[v], hi = g->row[v + 1];
    while (lo < hi) { /* lower_bound */
        const uint64_t mid = lo + (hi - lo) / 2;
        if (g->col[mid] < u)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < g->row[v + 1] && g->col[lo] == u;
}

/* ---- topology generators (src/gen.cpp) ---- */

typedef struct {
    uint32_t *s, *t;
    uint64_t n, cap;
} edgevec;

static void ev_push(edgevec* ev, uint32_t s, uint32_t t) {
    if (ev->n == ev->cap) {
        ev->cap = ev->cap ? ev->cap * 2 : 1024;
        ev->s = (uint32_t*)realloc(ev->s, ev->cap * sizeof(uint32_t));
        ev->t = (uint32_t*)realloc(ev->t, ev->cap * sizeof(uint32_t));
    }
    ev->s[ev->n] = s;
    ev->t[ev->n] = t;
    ++ev->n;
}

/* generate_uniform (gen.cpp:13-27) */
orc_graph* orc_gen_uniform(uint32_t n, uint32_t deg, uint64_t seed, int mirror) {
    crng r;
    crng_init(&r, orc_derive_seed(seed, 0x746f706fULL));
    edgevec ev = {0};
    for (uint32_t v = 0; v < n; ++v)
        for (uint32_t k = 0; k < deg; ++k) {
            uint32_t u = (uint32_t)crng_bounded(&r, n);
            for (int tries = 0; u == v && tries < 16; ++tries) u = (uint32_t)crng_bounded(&r, n);
            if (u == v) continue;
            ev_push(&ev, v, u);
        }
    orc_graph* g = orc_graph_build(ev.s, ev.t, NULL, NULL, ev.n, 0, mirror, n);
    free(ev.s);
    free(ev.t);
    return g;
}

/* generate_preferential (gen.cpp:29-68) */
orc_graph* orc_gen_ba(uint32_t n, uint32_t deg, uint64_t seed, int mirror) {
    crng r;
    crng_init(&r, orc_derive_seed(seed, 0x6261746f706fULL));
    const uint32_t m = deg > 1 ? deg : 1;
    edgevec ev = {0};
    uint64_t pool_n = 0, pool_cap = (uint64_t)n * m * 2 + 16;
    uint32_t* pool = (uint32_t*)xmalloc(pool_cap * sizeof(uint32_t));
    uint32_t* picked = (uint32_t*)xmalloc((m + 1) * sizeof(uint32_t));
    const uint32_t seed_nodes = n < m + 1 ? n : m + 1;
    for (uint32_t v = 1; v < seed_nodes; ++v) {
        ev_push(&ev, v, v - 1);
        pool[pool_n++] = v;
        pool[pool_n++] = v - 1;
    }
    for (uint32_t v = seed_nodes; v < n; ++v) {
        uint32_t npicked = 0;
        for (uint32_t k = 0; k < m; ++k) {
            uint32_t u = ORC_INVALID;
            for (int tries = 0; tries < 32; ++tries) {
                const uint32_t cand = pool_n == 0 ? (uint32_t)crng_bounded(&r, v)
                                                  : pool[crng_bounded(&r, pool_n)];
                int dup = 0;
                for (uint32_t j = 0; j < npicked; ++j) dup |= picked[j] == cand;
                if (cand != v && !dup) {
                    u = cand;
                    break;
                }
            }
            if (u == ORC_INVALID) continue;
            picked[npicked++] = u;
            ev_push(&ev, v, u);
            pool[pool_n++] = v;
            pool[pool_n++] = u;
        }
    }
    orc_graph* g = orc_graph_build(ev.s, ev.t, NULL, NULL, ev.n, 0, mirror, n);
    free(ev.s);
    free(ev.t);
    free(pool);
    free(picked);
    return g;
}

/* synthesize_weights (graph.cpp:302-352) with the reference CountingRng. */
int orc_synth_weights(orc_graph* g, int kind, double low, double high, double alpha,
                      uint64_t seed) {
    crng r;
    crng_init(&r, orc_derive_seed(seed, 0x77656967687473ULL));
    const uint64_t ne = g->ne;
    switch (kind) {
    case 0: /* UniformReal */
        if (!(low < high) || !(low > 0.0)) {
            set_err("uniform weight spec requires 0 < low < high");
            return -1;
        }
        for (uint64_t e = 0; e < ne; ++e)
            g->prop[e] = (float)(low + crng_uniform01(&r) * (high - low));
        break;
    case 1: { /* UniformIntLabel */
        if (!(low <= high) || low < 0 || high > 65535) {
            set_err("label spec requires 0 <= low <= high <= 65535");
            return -1;
        }
        const uint64_t lo = (uint64_t)low, span = (uint64_t)high - lo + 1;
        if (!g->label) g->label = (uint16_t*)xmalloc(ne * sizeof(uint16_t) + 2);
        for (uint64_t e = 0; e < ne; ++e) g->label[e] = (uint16_t)(lo + crng_bounded(&r, span));
        return 0; /* labels do not touch the aggregates */
    }
    case 2: { /* Pareto */
        if (!(alpha > 0.0)) {
            set_err("pareto weight spec requires alpha > 0");
            return -1;
        }
        const double inv = 1.0 / alpha;
        for (uint64_t e = 0; e < ne; ++e) g->prop[e] = (float)pow(crng_open01(&r), -inv);
        break;
    }
    case 3: /* DegreeBased */
        for (uint64_t e = 0; e < ne; ++e) {
            const uint32_t t = g->col[e];
            const uint64_t d = g->row[t + 1] - g->row[t];
            g->prop[e] = (float)(d > 1 ? d : 1);
        }
        break;
    default:
        set_err("unknown weight kind");
        return -1;
    }
    orc_recompute_aggregates(g);
    return 0;
}

/* ---- new synthetic workload: R-MAT + Philox weights ---- */

/* Graph500 R-MAT quadrant thresholds (A,B,C,D)=(.57,.19,.19,.05) as exact
 * 32-bit fixed point: floor(p * 2^32) of the cumulative sums. */
#define RMAT_TA 2448131358u   /* 0.57 */
#define RMAT_TAB 3264175144u  /* 0.76 */
#define RMAT_TABC 4080218931u /* 0.95 */

static uint32_t rmat_perm(uint32_t x, uint32_t scale, uint64_t pk) {
    /* bijection on [0, 2^scale): odd multiply + add, xorshift, twice */
    if (scale == 0) return 0;
    const uint32_t mask = scale >= 32 ? 0xFFFFFFFFu : ((1u << scale) - 1u);
    const uint32_t sh = scale / 2 + 1;
    const uint32_t m1 = ((uint32_t)pk | 1u), a1 = (uint32_t)(pk >> 32);
    const uint32_t m2 = ((uint32_t)(pk >> 17) | 1u), a2 = (uint32_t)(pk >> 7);
    x = (x * m1 + a1) & mask;
    x ^= x >> sh;
    x = (x * m2 + a2) & mask;
    x ^= x >> sh;
    return x & mask;
}

void orc_rmat_samples(uint32_t scale, uint64_t nsamples, uint64_t seed, uint32_t* src,
                      uint32_t* dst) {
    const uint64_t ks = orc_derive_seed(seed, 0x726d6174ULL); /* "rmat" */
    const uint64_t pk = orc_derive_seed(seed, 0x7065726dULL); /* "perm" */
    const uint32_t key[2] = {(uint32_t)ks, (uint32_t)(ks >> 32)};
    for (uint64_t i = 0; i < nsamples; ++i) {
        uint32_t u = 0, v = 0, rnd[4];
        for (uint32_t lvl = 0; lvl < scale; ++lvl) {
            if ((lvl & 3) == 0) {
                const uint32_t ctr[4] = {lvl >> 2, (uint32_t)i, (uint32_t)(i >> 32), 0x524d4154u};
                orc_philox4x32_10(ctr, key, rnd);
            }
            const uint32_t r = rnd[lvl & 3];
            const uint32_t bu = r >= RMAT_TAB, bv = (r >= RMAT_TA && r < RMAT_TAB) || r >= RMAT_TABC;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        src[i] = rmat_perm(u, scale, pk);
        dst[i] = rmat_perm(v, scale, pk);
    }
}

orc_graph* orc_gen_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed) {
    const uint64_t nv = 1ull << scale;
    const uint64_t ns = (uint64_t)(edge_factor / 2) * nv;
    uint32_t* s = (uint32_t*)xmalloc(ns * sizeof(uint32_t));
    uint32_t* t = (uint32_t*)xmalloc(ns * sizeof(uint32_t));
    orc_rmat_samples(scale, ns, seed, s, t);
    orc_graph* g = orc_graph_build(s, t, NULL, NULL, ns, 0, 1, nv);
    free(s);
    free(t);
    return g;
}

/* Parallel form of orc_gen_rmat for large scales (bench.py --impl reference
 * input): the same samples, mirrored, as one sorted (src,dst) key array.  A
 * full key sort equals Graph::build's per-slice stable sort by target here
 * because duplicates are indistinguishable before weights are synthesized. */
typedef struct {
    uint32_t scale;
    uint64_t ns, lo, hi;
    uint64_t seed;
    uint64_t* keys;
    uint64_t loops;
} rmat_task;

static void* rmat_task_run(void* arg) {
    rmat_task* t = (rmat_task*)arg;
    const uint64_t chunk = 4096;
    uint32_t s[4096], d[4096];
    for (uint64_t b = t->lo; b < t->hi; b += chunk) {
        const uint64_t n = b + chunk <= t->hi ? chunk : t->hi - b;
        /* sample ids b..b+n: same draws as orc_rmat_samples */
        const uint64_t ks = orc_derive_seed(t->seed, 0x726d6174ULL);
        const uint64_t pk = orc_derive_seed(t->seed, 0x7065726dULL);
        const uint32_t key[2] = {(uint32_t)ks, (uint32_t)(ks >> 32)};
        for (uint64_t j = 0; j < n; ++j) {
            const uint64_t i = b + j;
            uint32_t u = 0, v = 0, rnd[4];
            for (uint32_t lvl = 0; lvl < t->scale; ++lvl) {
                if ((lvl & 3) == 0) {
                    const uint32_t ctr[4] = {lvl >> 2, (uint32_t)i, (uint32_t)(i >> 32), 0x524d4154u};
                    orc_philox4x32_10(ctr, key, rnd);
                }
                const uint32_t r = rnd[lvl & 3];
                const uint32_t bu = r >= RMAT_TAB, bv = (r >= RMAT_TA && r < RMAT_TAB) || r >= RMAT_TABC;
                u = (u << 1) | bu;
                v = (v << 1) | bv;
            }
            s[j] = rmat_perm(u, t->scale, pk);
            d[j] = rmat_perm(v, t->scale, pk);
        }
        for (uint64_t j = 0; j < n; ++j) {
            const uint64_t i = b + j;
            t->keys[i] = ((uint64_t)s[j] << 32) | d[j];
            if (s[j] != d[j]) {
                t->keys[t->ns + i] = ((uint64_t)d[j] << 32) | s[j];
            } else {
                t->keys[t->ns + i] = (uint64_t)(1ull << t->scale) << 32; /* sentinel, sorts last */
                ++t->loops;
            }
        }
    }
    return NULL;
}

typedef struct {
    const uint64_t* in;
    uint64_t* out;
    uint64_t lo, hi;
    int shift;
    uint64_t* hist; /* [2048] per task, then its offsets */
} radix_task;

static void* radix_count(void* arg) {
    radix_task* t = (radix_task*)arg;
    memset(t->hist, 0, 2048 * sizeof(uint64_t));
    for (uint64_t i = t->lo; i < t->hi; ++i) ++t->hist[(t->in[i] >> t->shift) & 2047];
    return NULL;
}

static void* radix_scatter(void* arg) {
    radix_task* t = (radix_task*)arg;
    for (uint64_t i = t->lo; i < t->hi; ++i) t->out[t->hist[(t->in[i] >> t->shift) & 2047]++] = t->in[i];
    return NULL;
}

static void par_run(void* (*fn)(void*), void* tasks, size_t sz, int n) {
    pthread_t th[256];
    for (int i = 0; i < n; ++i) pthread_create(&th[i], NULL, fn, (char*)tasks + sz * (size_t)i);
    for (int i = 0; i < n; ++i) pthread_join(th[i], NULL);
}

/* stable LSD radix sort, 11-bit digits, over the low `bits` bits */
static uint64_t* radix_sort64(uint64_t* a, uint64_t* tmp, uint64_t n, int bits, int nt) {
    radix_task* tk = (radix_task*)xmalloc(sizeof(radix_task) * (size_t)nt);
    uint64_t* hist = (uint64_t*)xmalloc(sizeof(uint64_t) * 2048 * (size_t)nt);
    for (int shift = 0; shift < bits; shift += 11) {
        for (int t = 0; t < nt; ++t) {
            tk[t].in = a;
            tk[t].out = tmp;
            tk[t].lo = n * (uint64_t)t / (uint64_t)nt;
            tk[t].hi = n * (uint64_t)(t + 1) / (uint64_t)nt;
            tk[t].shift = shift;
            tk[t].hist = hist + 2048 * (size_t)t;
        }
        par_run(radix_count, tk, sizeof(radix_task), nt);
        uint64_t run = 0;
        for (int dgt = 0; dgt < 2048; ++dgt)
            for (int t = 0; t < nt; ++t) {
                const uint64_t c = tk[t].hist[dgt];
                tk[t].hist[dgt] = run;
                run += c;
            }
        par_run(radix_scatter, tk, sizeof(radix_task), nt);
        uint64_t* sw = a;
        a = tmp;
        tmp = sw;
    }
    free(tk);
    free(hist);
    return a;
}

typedef struct {
    orc_graph* g;
    const uint64_t* keys;
    uint64_t lo, hi;
    int what; /* 0 col, 1 rows, 2 uniform props, 3 aggregates */
    double low, high;
    uint64_t seed;
} fill_task;

static uint64_t edge_draw(uint64_t seed, uint64_t e, uint32_t tag);

static void* fill_run(void* arg) {
    fill_task* t = (fill_task*)arg;
    orc_graph* g = t->g;
    if (t->what == 0) {
        for (uint64_t e = t->lo; e < t->hi; ++e) g->col[e] = (uint32_t)t->keys[e];
    } else if (t->what == 1) {
        for (uint64_t v = t->lo; v < t->hi; ++v) { /* first key >= v<<32 */
            uint64_t lo = 0, hi = g->ne;
            while (lo < hi) {
                const uint64_t mid = lo + (hi - lo) / 2;
                if (t->keys[mid] < (v << 32)) lo = mid + 1; else hi = mid;
            }
            g->row[v] = lo;
        }
    } else if (t->what == 2) {
        for (uint64_t e = t->lo; e < t->hi; ++e) {
            const double u = (double)(edge_draw(t->seed, e, 0x57474854u) >> 11) * 0x1.0p-53;
            g->prop[e] = (float)(t->low + u * (t->high - t->low));
        }
    } else {
        for (uint64_t v = t->lo; v < t->hi; ++v) {
            double mx = 0.0, sum = 0.0;
            for (uint64_t e = g->row[v]; e != g->row[v + 1]; ++e) {
                const double p = g->prop[e];
                if (p > mx) mx = p;
                sum += p;
            }
            g->nmax[v] = mx;
            g->nsum[v] = sum;
        }
    }
    return NULL;
}

static void par_fill(orc_graph* g, const uint64_t* keys, uint64_t n, int what, double low,
                     double high, uint64_t seed, int nt) {
    fill_task* tk = (fill_task*)xmalloc(sizeof(fill_task) * (size_t)nt);
    for (int t = 0; t < nt; ++t) {
        fill_task x = {g, keys, n * (uint64_t)t / (uint64_t)nt, n * (uint64_t)(t + 1) / (uint64_t)nt,
                       what, low, high, seed};
        tk[t] = x;
    }
    par_run(fill_run, tk, sizeof(fill_task), nt);
    free(tk);
}

/* R-MAT + uniform[low,high) Philox weights (== orc_gen_rmat + orc_synth_philox
 * kind 0), multi-threaded. */
orc_graph* orc_gen_rmat_par(uint32_t scale, uint32_t edge_factor, uint64_t seed, double low,
                            double high, uint64_t wseed, int nt) {
    if (nt < 1) nt = 1;
    if (nt > 256) nt = 256;
    const uint64_t nv = 1ull << scale;
    const uint64_t ns = (uint64_t)(edge_factor / 2) * nv;
    uint64_t* keys = (uint64_t*)xmalloc(2 * ns * sizeof(uint64_t));
    uint64_t* tmp = (uint64_t*)xmalloc(2 * ns * sizeof(uint64_t));
    rmat_task* rt = (rmat_task*)xmalloc(sizeof(rmat_task) * (size_t)nt);
    for (int t = 0; t < nt; ++t) {
        rmat_task x = {scale, ns, ns * (uint64_t)t / (uint64_t)nt, ns * (uint64_t)(t + 1) / (uint64_t)nt,
                       seed, keys, 0};
        rt[t] = x;
    }
    par_run(rmat_task_run, rt, sizeof(rmat_task), nt);
    uint64_t loops = 0;
    for (int t = 0; t < nt; ++t) loops += rt[t].loops;
    free(rt);
    uint64_t* sorted = radix_sort64(keys, tmp, 2 * ns, 32 + (int)scale + 1, nt);
    orc_graph* g = (orc_graph*)xmalloc(sizeof(orc_graph));
    g->nv = (uint32_t)nv;
    g->ne = 2 * ns - loops;
    g->row = (uint64_t*)xmalloc((nv + 1) * sizeof(uint64_t));
    g->col = (uint32_t*)xmalloc(g->ne * sizeof(uint32_t));
    g->prop = (float*)xmalloc(g->ne * sizeof(float));
    g->label = NULL;
    g->nmax = (double*)xmalloc(nv * sizeof(double));
    g->nsum = (double*)xmalloc(nv * sizeof(double));
    par_fill(g, sorted, g->ne, 0, 0, 0, 0, nt);
    par_fill(g, sorted, nv, 1, 0, 0, 0, nt);
    g->row[nv] = g->ne;
    free(keys);
    free(tmp);
    par_fill(g, NULL, g->ne, 2, low, high, wseed, nt);
    par_fill(g, NULL, nv, 3, 0, 0, 0, nt);
    return g;
}

static uint64_t edge_draw(uint64_t seed, uint64_t e, uint32_t tag) {
    const uint32_t ctr[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0, tag};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return ((uint64_t)o[1] << 32) | o[0];
}

/* Philox-keyed-by-edge analog of synthesize_weights (same maps as
 * graph.cpp:308-341); identical on the device builder. */
int orc_synth_philox(orc_graph* g, int kind, double low, double high, double alpha,
                     uint64_t seed) {
    const uint64_t ne = g->ne;
    switch (kind) {
    case 0:
        if (!(low < high) || !(low > 0.0)) {
            set_err("uniform weight spec requires 0 < low < high");
            return -1;
        }
        for (uint64_t e = 0; e < ne; ++e) {
            const double u = (double)(edge_draw(seed, e, 0x57474854u) >> 11) * 0x1.0p-53;
            g->prop[e] = (float)(low + u * (high - low));
        }
        break;
    case 1: {
        if (!(low <= high) || low < 0 || high > 65535) {
            set_err("label spec requires 0 <= low <= high <= 65535");
            return -1;
        }
        const uint64_t lo = (uint64_t)low, span = (uint64_t)high - lo + 1;
        if (!g->label) g->label = (uint16_t*)xmalloc(ne * sizeof(uint16_t) + 2);
        for (uint64_t e = 0; e < ne; ++e) {
            const uint64_t r = edge_draw(seed, e, 0x4c41424cu);
            g->label[e] = (uint16_t)(lo + (uint64_t)(((unsigned __int128)r * span) >> 64));
        }
        return 0;
    }
    case 2: {
        if (!(alpha > 0.0)) {
            set_err("pareto weight spec requires alpha > 0");
            return -1;
        }
        const double inv = 1.0 / alpha;
        for (uint64_t e = 0; e < ne; ++e) {
            const double u =
                ((double)(edge_draw(seed, e, 0x50415245u) >> 11) + 0.5) * 0x1.0p-53;
            /* alpha == 1: u^-1 as one correctly rounded division on both sides */
            g->prop[e] = alpha == 1.0 ? (float)(1.0 / u) : (float)pow(u, -inv);
        }
        break;
    }
    default:
        set_err("unknown weight kind");
        return -1;
    }
    orc_recompute_aggregates(g);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Walk models (include/dynwalk/models.hpp:33-164)                           */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t cur, prev, prev_degree, step;
} wstate; /* WalkerState (walk_state.hpp:13-40) minus the path */

typedef struct {
    const orc_graph* g;
    const orc_model* m;
    int err;
} ctx_t;

static inline uint32_t degree(const orc_graph* g, uint32_t v) {
    return (uint32_t)(g->row[v + 1] - g->row[v]);
}

static double fmax3(double a, double b, double c) {
    double m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

/* Model::weight */
static double model_weight(ctx_t* c, const wstate* st, uint64_t e) {
    const orc_graph* g = c->g;
    const orc_model* m = c->m;
    const double h = m->weighted ? (double)g->prop[e] : 1.0;
    switch (m->kind) {
    case ORC_STATIC: /* models.hpp:36-38 */
        return h;
    case ORC_NODE2VEC: { /* models.hpp:62-69 */
        if (st->prev == ORC_INVALID) return h;
        const uint32_t u = g->col[e];
        if (u == st->prev) return h / m->a;
        if (orc_has_edge(g, st->prev, u)) return h;
        return h / m->b;
    }
    case ORC_METAPATH: { /* models.hpp:99-104 */
        if (st->step >= m->schema_len) {
            set_err("metapath walk stepped beyond its schema");
            c->err = 1;
            return 0.0;
        }
        const uint16_t lab = g->label ? g->label[e] : 0;
        return lab == m->schema[st->step] ? h : 0.0;
    }
    case ORC_PR2: { /* models.hpp:128-138 */
        if (st->prev == ORC_INVALID) return h;
        const double dcur = (double)degree(g, st->cur);
        const double dprev = (double)st->prev_degree;
        const double maxd = dcur < dprev ? dprev : dcur;
        const uint32_t u = g->col[e];
        if (u != st->prev && orc_has_edge(g, st->prev, u))
            return h * ((1.0 - m->gamma) / dcur + m->gamma / dprev) * maxd;
        return h * ((1.0 - m->gamma) / dcur) * maxd;
    }
    }
    return 0.0;
}

/* Model::estimate_bound */
static double model_bound(const ctx_t* c, const wstate* st) {
    const orc_graph* g = c->g;
    const orc_model* m = c->m;
    switch (m->kind) {
    case ORC_STATIC: /* models.hpp:42-44 */
    case ORC_METAPATH: /* models.hpp:108-111 */
        return m->weighted ? g->nmax[st->cur] : 1.0;
    case ORC_NODE2VEC: { /* models.hpp:74-79 */
        const double hmax = m->weighted ? g->nmax[st->cur] : 1.0;
        return fmax3(hmax / m->a, hmax, hmax / m->b);
    }
    case ORC_PR2: { /* models.hpp:142-151 */
        const double hmax = m->weighted ? g->nmax[st->cur] : 1.0;
        const double dcur = (double)degree(g, st->cur);
        const double dprev = st->prev != ORC_INVALID ? (double)st->prev_degree : dcur;
        const double maxd = dcur < dprev ? dprev : dcur;
        const double boosted = hmax * ((1.0 - m->gamma) / dcur + m->gamma / dprev) * maxd;
        const double plain = hmax * ((1.0 - m->gamma) / dcur) * maxd;
        return fmax3(hmax, boosted, plain);
    }
    }
    return 0.0;
}

/* Model::estimate_weight_sum */
static double model_sum(const ctx_t* c, const wstate* st) {
    const orc_graph* g = c->g;
    const orc_model* m = c->m;
    const double d = (double)degree(g, st->cur);
    switch (m->kind) {
    case ORC_STATIC: /* models.hpp:45-48 */
        return m->weighted ? g->nsum[st->cur] : d;
    case ORC_NODE2VEC: /* models.hpp:80-87 */
        if (m->weighted) {
            const double s = g->nsum[st->cur];
            return (s / m->a + s + s / m->b) / 3.0;
        }
        return ((1.0 / m->a + 1.0 + 1.0 / m->b) / 3.0) * d;
    case ORC_METAPATH: /* models.hpp:112-115 */
        if (m->weighted) return (g->nsum[st->cur] + 0.0) / 2.0;
        return ((1.0 + 0.0) / 2.0) * d;
    case ORC_PR2: { /* models.hpp:152-161 */
        const double dcur = d;
        const double dprev = st->prev != ORC_INVALID ? (double)st->prev_degree : dcur;
        const double maxd = dcur < dprev ? dprev : dcur;
        const double s = m->weighted ? g->nsum[st->cur] : 1.0;
        const double boosted = s * ((1.0 - m->gamma) / dcur + m->gamma / dprev) * maxd;
        const double plain = s * ((1.0 - m->gamma) / dcur) * maxd;
        const double avg = (s + boosted + plain) / 3.0;
        return m->weighted ? avg : avg * dcur;
    }
    }
    return 0.0;
}

static uint32_t model_max_steps(const orc_model* m) {
    return m->kind == ORC_METAPATH ? m->schema_len : 0xFFFFFFFFu;
}

/* ------------------------------------------------------------------------ */
/* Samplers (include/dynwalk/samplers.hpp)                                   */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t next;
    uint64_t trials, weight_reads, rng_draws;
    int fell_back;
} outcome; /* SampleOutcome (samplers.hpp:20-28); trials defaults to 1 */

static int check_weight(ctx_t* c, double w) { /* samplers.hpp:50-53 */
    if (w < 0.0 || !isfinite(w)) {
        char buf[128];
        snprintf(buf, sizeof buf, "model returned a negative or non-finite weight: %f", w);
        set_err(buf);
        c->err = 1;
        return 0;
    }
    return 1;
}

/* sample_ervs (samplers.hpp:65-107): exp-key reservoir with jumps. */
static outcome sample_ervs(ctx_t* c, const wstate* st, wrng* r) {
    outcome out = {ORC_INVALID, 1, 0, 0, 0};
    const orc_graph* g = c->g;
    const uint32_t d = degree(g, st->cur);
    const uint64_t e0 = g->row[st->cur];
    const uint64_t draws0 = r->draws;
    double best_log_key = -INFINITY;
    uint32_t best = ORC_INVALID;
    double skip_remaining = 0.0;
    int have_threshold = 0;
    for (uint32_t i = 0; i < d; ++i) {
        const double w = model_weight(c, st, e0 + i);
        if (c->err || !check_weight(c, w)) return out;
        ++out.weight_reads;
        if (w == 0.0) continue;
        if (best == ORC_INVALID) {
            best_log_key = log(wrng_open01(r)) / w;
            best = g->col[e0 + i];
            continue;
        }
        if (!have_threshold) {
            skip_remaining = log(wrng_open01(r)) / best_log_key;
            have_threshold = 1;
        }
        skip_remaining -= w;
        if (skip_remaining <= 0.0) {
            const double floor_u = exp(w * best_log_key);
            const double u = floor_u + wrng_open01(r) * (1.0 - floor_u);
            const double log_key = log(u) / w;
            if (log_key > best_log_key) {
                best_log_key = log_key;
                best = g->col[e0 + i];
            }
            have_threshold = 0;
        }
    }
    out.next = best;
    out.rng_draws = r->draws - draws0;
    return out;
}

/* sample_ervs_nojump (samplers.hpp:112-137) */
static outcome sample_ervs_nojump(ctx_t* c, const wstate* st, wrng* r) {
    outcome out = {ORC_INVALID, 1, 0, 0, 0};
    const orc_graph* g = c->g;
    const uint32_t d = degree(g, st->cur);
    const uint64_t e0 = g->row[st->cur];
    const uint64_t draws0 = r->draws;
    double best_log_key = -INFINITY;
    uint32_t best = ORC_INVALID;
    for (uint32_t i = 0; i < d; ++i) {
        const double w = model_weight(c, st, e0 + i);
        if (c->err || !check_weight(c, w)) return out;
        ++out.weight_reads;
        const double u = wrng_open01(r);
        if (w == 0.0) continue;
        const double log_key = log(u) / w;
        if (best == ORC_INVALID || log_key > best_log_key) {
            best_log_key = log_key;
            best = g->col[e0 + i];
        }
    }
    out.next = best;
    out.rng_draws = r->draws - draws0;
    return out;
}

/* Trial cap of an eRJS step: cap_per_degree * d (samplers.hpp:157), tightened
 * by the tier-2 hand-off when erjs_handoff > 0 (not in the reference; the
 * device rule of dw_walk_kernel.cuh step_cap, include/dynwalk_b200.h):
 * max(32, ceil(erjs_handoff * d / ratio)) trials, i.e. trials worth
 * erjs_handoff reservoir passes over the row under the cost model
 * (cost_model.hpp:46-56): a ski-rental bound of the rejection loop. */
static uint64_t erjs_cap(const orc_opts* o, uint32_t d) {
    uint64_t cap = o->cap_per_degree * d;
    if (o->erjs_handoff > 0.0) {
        const double h = ceil(o->erjs_handoff * (double)d / o->edge_cost_ratio);
        const uint64_t hc = !(h >= 32.0) ? 32u : (h >= 4294967295.0 ? 0xFFFFFFFFu : (uint64_t)h);
        if (hc < cap) cap = hc;
    }
    return cap;
}

/* sample_erjs (samplers.hpp:145-178); cap = the step's trial cap */
static outcome sample_erjs(ctx_t* c, const wstate* st, wrng* r, double bound, uint64_t cap) {
    const orc_graph* g = c->g;
    const uint32_t d = degree(g, st->cur);
    outcome out = {ORC_INVALID, 0, 0, 0, 0};
    if (d == 0) return out;
    if (!(bound > 0.0) || !isfinite(bound)) {
        char buf[128];
        snprintf(buf, sizeof buf, "rejection bound must be positive and finite, got %f", bound);
        set_err(buf);
        c->err = 1;
        return out;
    }
    const uint64_t e0 = g->row[st->cur];
    const uint64_t draws0 = r->draws;
    while (out.trials < cap) {
        const uint64_t x = wrng_bounded(r, d);
        const double y = wrng_uniform01(r) * bound;
        const double w = model_weight(c, st, e0 + x);
        if (c->err || !check_weight(c, w)) return out;
        ++out.trials;
        ++out.weight_reads;
        if (y < w) {
            out.next = g->col[e0 + x];
            out.rng_draws = r->draws - draws0;
            return out;
        }
    }
    outcome fb = sample_ervs(c, st, r);
    fb.fell_back = 1;
    fb.trials = out.trials;
    fb.weight_reads += out.weight_reads;
    fb.rng_draws = r->draws - draws0;
    return fb;
}

/* ------------------------------------------------------------------------ */
/* Walk loop + scheduler (src/runtime.cpp:59-153, 192-247)                   */
/* ------------------------------------------------------------------------ */

static void bucket(orc_stats* s, uint32_t degree_, int erjs) { /* runtime.cpp:42-46 */
    uint32_t b = 0;
    while (b < 31 && (1u << (b + 1)) <= degree_) ++b;
    ++s->sel_by_deg[b][erjs ? 1 : 0];
}

/* walk_query (runtime.cpp:59-153); returns path length, -1 on error */
static int64_t walk_query(ctx_t* c, const orc_opts* o, uint32_t start, uint64_t qid,
                          uint32_t* path, orc_stats* ls, wrng* r) {
    const orc_graph* g = c->g;
    const orc_model* m = c->m;
    wstate st = {start, ORC_INVALID, 0, 0};
    path[0] = start;
    uint32_t len = 1;
    r->draws = 0;
    if (r->kind == ORC_RNG_MT19937) {
        mt64_seed(&r->mt, orc_derive_seed(o->seed, qid));
    } else {
        r->seed = o->seed;
        r->qid = qid;
    }
    const uint32_t ms = model_max_steps(m);
    const uint32_t target = o->walk_length < ms ? o->walk_length : ms;
    while (st.step < target) {
        const uint32_t d = degree(g, st.cur);
        if (d == 0) break;
        if (r->kind == ORC_RNG_PHILOX) { /* stream keyed by (walker, step) */
            r->step = st.step;
            r->idx = 0;
            r->have_cache = 0;
        }
        outcome out;
        switch (o->mode) {
        case ORC_ADAPTIVE: { /* decide_sampler, cost_model.hpp:46-56 */
            const double est_max = model_bound(c, &st);
            const double est_sum = model_sum(c, &st);
            const int erjs = o->edge_cost_ratio * est_max < est_sum;
            bucket(ls, d, erjs);
            if (erjs) {
                ++ls->select_erjs;
                out = sample_erjs(c, &st, r, est_max, erjs_cap(o, d));
            } else {
                ++ls->select_ervs;
                out = sample_ervs(c, &st, r);
            }
            break;
        }
        case ORC_FORCE_ERVS:
            ++ls->select_ervs;
            bucket(ls, d, 0);
            out = sample_ervs(c, &st, r);
            break;
        case ORC_ERVS_NOJUMP:
            ++ls->select_ervs;
            bucket(ls, d, 0);
            out = sample_ervs_nojump(c, &st, r);
            break;
        case ORC_FORCE_ERJS: {
            const double est = model_bound(c, &st);
            ++ls->select_erjs;
            bucket(ls, d, 1);
            out = sample_erjs(c, &st, r, est, erjs_cap(o, d));
            break;
        }
        default:
            set_err("unsupported sampler mode");
            c->err = 1;
            return -1;
        }
        if (c->err) return -1;
        ++ls->steps;
        ls->trials += out.trials;
        ls->weight_reads += out.weight_reads;
        ls->rng_draws += out.rng_draws;
        if (out.fell_back) ++ls->erjs_fallbacks;
        if (out.next == ORC_INVALID) {
            ++ls->dead_ends;
            break;
        }
        /* WalkerState::advance (walk_state.hpp:33-39) */
        st.prev = st.cur;
        st.prev_degree = degree(g, st.cur);
        st.cur = out.next;
        ++st.step;
        path[len++] = out.next;
    }
    return len;
}

typedef struct {
    const orc_graph* g;
    const orc_model* m;
    const orc_opts* o;
    const uint32_t* queries;
    uint64_t nq;
    uint32_t* paths;
    uint32_t* lengths;
    uint64_t stride;
    uint64_t next;
    orc_stats total;
    pthread_mutex_t mu;
    int failed;
} run_shared;

static void merge_stats(orc_stats* into, const orc_stats* from) { /* runtime.cpp:155-188 */
    into->queries += from->queries;
    into->query_errors += from->query_errors;
    into->dead_ends += from->dead_ends;
    into->steps += from->steps;
    into->select_ervs += from->select_ervs;
    into->select_erjs += from->select_erjs;
    into->trials += from->trials;
    into->weight_reads += from->weight_reads;
    into->rng_draws += from->rng_draws;
    into->erjs_fallbacks += from->erjs_fallbacks;
    for (int b = 0; b < 33; ++b) {
        into->sel_by_deg[b][0] += from->sel_by_deg[b][0];
        into->sel_by_deg[b][1] += from->sel_by_deg[b][1];
    }
}

static void* run_worker(void* arg) {
    run_shared* sh = (run_shared*)arg;
    orc_stats ls;
    memset(&ls, 0, sizeof ls);
    wrng* r = (wrng*)calloc(1, sizeof(wrng));
    r->kind = sh->o->rng;
    ctx_t c = {sh->g, sh->m, 0};
    uint32_t* scratch = (uint32_t*)xmalloc(sh->stride * sizeof(uint32_t));
    for (;;) {
        const uint64_t i = __atomic_fetch_add(&sh->next, 1, __ATOMIC_RELAXED);
        if (i >= sh->nq) break;
        const uint32_t start = sh->queries[i];
        ++ls.queries;
        uint32_t* path = sh->paths ? sh->paths + i * sh->stride : scratch;
        for (uint64_t k = 0; k < sh->stride; ++k) path[k] = ORC_INVALID;
        if (start >= sh->g->nv) {
            ++ls.query_errors;
            if (sh->lengths) sh->lengths[i] = 0;
            continue;
        }
        const int64_t len = walk_query(&c, sh->o, start, sh->o->qids ? sh->o->qids[i] : sh->o->qid_base + i, path, &ls, r);
        if (len < 0) {
            pthread_mutex_lock(&g_err_mu);
            if (!sh->failed) {
                sh->failed = 1;
                snprintf(g_err, sizeof g_err, "%s", tl_err);
            }
            pthread_mutex_unlock(&g_err_mu);
            break;
        }
        if (sh->lengths) sh->lengths[i] = (uint32_t)len;
    }
    pthread_mutex_lock(&sh->mu);
    merge_stats(&sh->total, &ls);
    pthread_mutex_unlock(&sh->mu);
    free(scratch);
    free(r);
    return NULL;
}

/* run_queries (runtime.cpp:192-247); paths are nq x (walk_length+1),
 * ORC_INVALID-padded (may be NULL to discard). */
int orc_run(const orc_graph* g, const orc_model* m, const orc_opts* o, const uint32_t* queries,
            uint64_t nq, uint32_t* paths, uint32_t* lengths, orc_stats* stats, int nthreads) {
    tl_err[0] = 0;
    g_err[0] = 0;
    if (nthreads < 1) {
        set_err("worker count must be >= 1");
        return -1;
    }
    run_shared sh;
    memset(&sh, 0, sizeof sh);
    sh.g = g;
    sh.m = m;
    sh.o = o;
    sh.queries = queries;
    sh.nq = nq;
    sh.paths = paths;
    sh.lengths = lengths;
    sh.stride = (uint64_t)o->walk_length + 1;
    pthread_mutex_init(&sh.mu, NULL);
    if (nthreads == 1) {
        run_worker(&sh);
    } else {
        pthread_t* th = (pthread_t*)xmalloc(sizeof(pthread_t) * (size_t)nthreads);
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, run_worker, &sh);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    pthread_mutex_destroy(&sh.mu);
    if (stats) *stats = sh.total;
    if (sh.failed) {
        snprintf(tl_err, sizeof tl_err, "%s", g_err);
        return -1;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* helpers for tests                                                         */
/* ------------------------------------------------------------------------ */

static wstate make_state(const orc_graph* g, uint32_t cur, uint32_t prev, uint32_t step) {
    wstate st = {cur, prev, prev != ORC_INVALID ? degree(g, prev) : 0, step};
    return st;
}

int64_t orc_transition_probs(const orc_graph* g, const orc_model* m, uint32_t cur,
                             uint32_t prev, uint32_t step, double* probs) {
    ctx_t c = {g, m, 0};
    const wstate st = make_state(g, cur, prev, step);
    const uint32_t d = degree(g, cur);
    const uint64_t e0 = g->row[cur];
    double total = 0.0;
    for (uint32_t i = 0; i < d; ++i) {
        const double w = model_weight(&c, &st, e0 + i);
        if (c.err || !check_weight(&c, w)) return -1;
        probs[i] = w;
        total += w;
    }
    if (total <= 0.0) return 0;
    for (uint32_t i = 0; i < d; ++i) probs[i] /= total;
    return d;
}

int orc_decide(const orc_graph* g, const orc_model* m, uint32_t cur, uint32_t prev,
               uint32_t step, double ratio, double* est_max, double* est_sum) {
    ctx_t c = {g, m, 0};
    const wstate st = make_state(g, cur, prev, step);
    *est_max = model_bound(&c, &st);
    *est_sum = model_sum(&c, &st);
    return ratio * *est_max < *est_sum;
}

double orc_weight(const orc_graph* g, const orc_model* m, uint32_t cur, uint32_t prev,
                  uint32_t step, uint64_t e) {
    ctx_t c = {g, m, 0};
    const wstate st = make_state(g, cur, prev, step);
    const double w = model_weight(&c, &st, e);
    return c.err ? NAN : w;
}

/* Host libm (the reference's std::log / std::exp, samplers.hpp:82-97) over an
 * array: the counterpart of dw_selftest_math for the libdevice agreement test. */
void orc_libm(int fn, const double* x, double* y, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) y[i] = fn == 0 ? log(x[i]) : exp(x[i]);
}

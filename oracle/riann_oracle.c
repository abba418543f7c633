/*
 * riann_oracle.c -- CPU restatement of the reference RIANN per-frame query.
 *
 * TEST INFRASTRUCTURE ONLY (see riann_oracle.h).  Compiled with
 * -ffp-contract=off so every float64 operation is individually rounded, the
 * way numpy evaluates the reference's expressions.
 */
#include "riann_oracle.h"

#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <sched.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>

/* ------------------------------------------------------------------------ */
/* numpy float64 pairwise summation (the reduction np.sum applies along a
 * contiguous axis).  Restated from numpy's published algorithm. */
double rno_pairwise_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += a[i];
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) s += a[i];
        return s;
    }
    int64_t h = n / 2;
    h -= h % 8;
    return rno_pairwise_sum(a, h) + rno_pairwise_sum(a + h, n - h);
}

/* rno_pairwise_sum over the squared differences (f64(r_i) - f64(q_i))^2,
 * each term formed on the fly: the same individually rounded operations in
 * the same order as squaring into a buffer first (numpy's d = r - q; d * d;
 * np.sum), without the buffer round trip. */
static double pw_sq(const float *q, const float *r, int64_t n)
{
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double d = (double)r[i] - (double)q[i];
            s += d * d;
        }
        return s;
    }
    if (n <= 128) {
        double acc[8];
        for (int j = 0; j < 8; j++) {
            double d = (double)r[j] - (double)q[j];
            acc[j] = d * d;
        }
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) {
                double d = (double)r[i + j] - (double)q[i + j];
                acc[j] += d * d;
            }
        double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        for (; i < n; i++) {
            double d = (double)r[i] - (double)q[i];
            s += d * d;
        }
        return s;
    }
    int64_t h = n / 2;
    h -= h % 8;
    return pw_sq(q, r, h) + pw_sq(q + h, r + h, n - h);
}

/* patches.py:151-159 */
static double sq_dist(const float *q, const float *r, int dim, double *tmp)
{
    (void)tmp;
    return sqrt(pw_sq(q, r, dim));
}

void rno_one_to_many(const float *q, const float *refs, const int64_t *rows,
                     int64_t k, int dim, double *out)
{
    double *tmp = (double *)malloc(sizeof(double) * (size_t)dim);
    for (int64_t i = 0; i < k; i++) {
        int64_t r = rows ? rows[i] : i;
        out[i] = sq_dist(q, refs + r * dim, dim, tmp);
    }
    free(tmp);
}

/* patches.py:100-115 */
#define RNO_ZERO_NORM_EPS 1e-12
static void normalize_one(const float *v, int dim, float *unit, double *norm,
                          double *tmp)
{
    for (int i = 0; i < dim; i++) {
        double x = (double)v[i];
        tmp[i] = x * x;
    }
    double nr = sqrt(rno_pairwise_sum(tmp, dim));
    if (nr >= RNO_ZERO_NORM_EPS) {
        for (int i = 0; i < dim; i++) unit[i] = (float)((double)v[i] / nr);
        if (norm) *norm = nr;
    } else {
        for (int i = 0; i < dim; i++) unit[i] = 0.0f;
        if (norm) *norm = 0.0;
    }
}

void rno_normalize_rows(const float *values, int64_t m, int dim, float *unit,
                        double *norms)
{
    double *tmp = (double *)malloc(sizeof(double) * (size_t)dim);
    for (int64_t r = 0; r < m; r++)
        normalize_one(values + r * dim, dim, unit + r * dim, norms ? norms + r : NULL, tmp);
    free(tmp);
}

/* patches.py:65-97 + :100-115, plane-major channels for C > 1 */
int rno_frame_units(const float *frame, int H, int W, int C, int pw, int ph,
                    int y0, int y1, float *unit, double *norms)
{
    if (pw < 1 || ph < 1 || C < 1 || W < pw || H < ph) return -1;
    int gw = W - pw + 1, gh = H - ph + 1;
    if (y0 < 0 || y1 > gh || y0 > y1) return -1;
    int dim = pw * ph * C;
    float *raw = (float *)malloc(sizeof(float) * (size_t)dim);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)dim);
    for (int y = y0; y < y1; y++) {
        for (int x = 0; x < gw; x++) {
            int e = 0;
            for (int c = 0; c < C; c++)
                for (int dy = 0; dy < ph; dy++)
                    for (int dx = 0; dx < pw; dx++)
                        raw[e++] = frame[((int64_t)(y + dy) * W + (x + dx)) * C + c];
            int64_t row = (int64_t)(y - y0) * gw + x;
            normalize_one(raw, dim, unit + row * dim, norms ? norms + row : NULL, tmp);
        }
    }
    free(raw);
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Minimal work-sharing pool over an index range. */
typedef struct {
    int64_t next;
    int64_t end;
    int64_t chunk;
    pthread_mutex_t mu;
    void (*fn)(void *ctx, int64_t lo, int64_t hi, void *scratch);
    void *ctx;
    void *(*make_scratch)(void *ctx);
    void (*free_scratch)(void *scratch);
} rno_pool;

static void *pool_worker(void *arg)
{
    rno_pool *p = (rno_pool *)arg;
    void *scratch = p->make_scratch ? p->make_scratch(p->ctx) : NULL;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t lo = p->next;
        int64_t hi = lo + p->chunk;
        if (hi > p->end) hi = p->end;
        p->next = hi;
        pthread_mutex_unlock(&p->mu);
        if (lo >= hi) break;
        p->fn(p->ctx, lo, hi, scratch);
    }
    if (p->free_scratch) p->free_scratch(scratch);
    return NULL;
}

static void pool_run(int nthreads, int64_t count, int64_t chunk,
                     void (*fn)(void *, int64_t, int64_t, void *), void *ctx,
                     void *(*mk)(void *), void (*fr)(void *))
{
    rno_pool p;
    p.next = 0;
    p.end = count;
    p.chunk = chunk < 1 ? 1 : chunk;
    p.fn = fn;
    p.ctx = ctx;
    p.make_scratch = mk;
    p.free_scratch = fr;
    pthread_mutex_init(&p.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads == 1) {
        pool_worker(&p);
    } else {
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
        for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, pool_worker, &p);
        for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&p.mu);
}

/* ------------------------------------------------------------------------ */
/* model.py:162-189 compute_sorted_lists */

typedef struct {
    const float *refs;
    int64_t n;
    int dim;
    int64_t row0;
    float *sdist;
    int32_t *sidx;
} sorted_ctx;

typedef struct {
    double *tmp;
    uint64_t *keys;
} sorted_scratch;

static void *sorted_mk(void *c)
{
    sorted_ctx *s = (sorted_ctx *)c;
    sorted_scratch *k = (sorted_scratch *)malloc(sizeof(*k));
    k->tmp = (double *)malloc(sizeof(double) * (size_t)s->dim);
    k->keys = (uint64_t *)malloc(sizeof(uint64_t) * 2 * (size_t)s->n);
    return k;
}

static void sorted_fr(void *p)
{
    sorted_scratch *k = (sorted_scratch *)p;
    free(k->tmp);
    free(k->keys);
    free(k);
}

/* one row of compute_sorted_lists (model.py:177-188) */
static void build_row(const float *refs, int64_t n, int dim, int64_t i, float *dr, int32_t *ir,
                      double *tmp, uint64_t *keys)
{
    const float *qi = refs + i * dim;
    for (int64_t j = 0; j < n; j++) {
        float v = (float)sq_dist(qi, refs + j * dim, dim, tmp);
        uint32_t bits;
        memcpy(&bits, &v, 4);
        /* non-negative floats order like their bit patterns; the index in
         * the low word makes the order the stable argsort's */
        keys[j] = ((uint64_t)bits << 32) | (uint64_t)j;
    }
    /* stable LSD radix sort on the float bits (keys start in index order, so
     * equal distances keep ascending indices: argsort(kind='stable')) */
    {
        uint64_t *src = keys, *dst = keys + n;
        for (int shift = 32; shift < 64; shift += 16) {
            int64_t *cnt = (int64_t *)calloc(65537, sizeof(int64_t));
            for (int64_t j = 0; j < n; j++) cnt[((src[j] >> shift) & 0xffff) + 1]++;
            for (int b = 0; b < 65536; b++) cnt[b + 1] += cnt[b];
            for (int64_t j = 0; j < n; j++) dst[cnt[(src[j] >> shift) & 0xffff]++] = src[j];
            free(cnt);
            uint64_t *t = src;
            src = dst;
            dst = t;
        }
        /* two passes: the sorted keys are back in keys[0..n) */
    }
    int64_t self = 0;
    while ((int64_t)(uint32_t)keys[self] != i) self++;
    if (self != 0) { /* duplicates of i sort ahead of it: self goes first */
        uint64_t sk = keys[self];
        memmove(keys + 1, keys, sizeof(uint64_t) * (size_t)self);
        keys[0] = sk;
    }
    for (int64_t j = 0; j < n; j++) {
        uint32_t bits = (uint32_t)(keys[j] >> 32);
        memcpy(&dr[j], &bits, 4);
        ir[j] = (int32_t)(uint32_t)keys[j];
    }
}

static void sorted_rows(void *c, int64_t lo, int64_t hi, void *scr)
{
    sorted_ctx *s = (sorted_ctx *)c;
    sorted_scratch *k = (sorted_scratch *)scr;
    for (int64_t r = lo; r < hi; r++)
        build_row(s->refs, s->n, s->dim, s->row0 + r, s->sdist + r * s->n, s->sidx + r * s->n, k->tmp, k->keys);
}

int rno_sorted_lists(const float *refs, int64_t n, int dim, int64_t row0,
                     int64_t rows, float *sdist, int32_t *sidx, int nthreads)
{
    if (n < 1 || row0 < 0 || row0 + rows > n) return -1;
    sorted_ctx c = {refs, n, dim, row0, sdist, sidx};
    pool_run(nthreads, rows, 4, sorted_rows, &c, sorted_mk, sorted_fr);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* numpy SeedSequence / PCG64 / Generator.integers (published algorithms). */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hash(uint32_t v, uint32_t *hc)
{
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y)
{
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    return r ^ (r >> 16);
}

typedef unsigned __int128 u128;
static const u128 PCG_MULT =
    ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;

static u128 pcg_state(const rno_pcg64 *g) { return ((u128)g->state_hi << 64) | g->state_lo; }
static u128 pcg_inc(const rno_pcg64 *g) { return ((u128)g->inc_hi << 64) | g->inc_lo; }
static void pcg_set_state(rno_pcg64 *g, u128 s)
{
    g->state_hi = (uint64_t)(s >> 64);
    g->state_lo = (uint64_t)s;
}

void rno_pcg64_seed(rno_pcg64 *g, const uint32_t *words, int nwords)
{
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hash(i < nwords ? words[i] : 0u, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hash(pool[s], &hc));
    for (int s = 4; s < nwords; s++)
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hash(words[s], &hc));
    uint32_t st[8];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    uint64_t w0 = st[0] | ((uint64_t)st[1] << 32), w1 = st[2] | ((uint64_t)st[3] << 32);
    uint64_t w2 = st[4] | ((uint64_t)st[5] << 32), w3 = st[6] | ((uint64_t)st[7] << 32);
    u128 initstate = ((u128)w0 << 64) | w1;
    u128 initseq = ((u128)w2 << 64) | w3;
    u128 inc = (initseq << 1) | 1u;
    g->inc_hi = (uint64_t)(inc >> 64);
    g->inc_lo = (uint64_t)inc;
    u128 s = 0;
    s = s * PCG_MULT + inc;
    s += initstate;
    s = s * PCG_MULT + inc;
    pcg_set_state(g, s);
    g->has_uint32 = 0;
    g->uinteger = 0;
}

uint64_t rno_pcg64_next64(rno_pcg64 *g)
{
    u128 s = pcg_state(g) * PCG_MULT + pcg_inc(g);
    pcg_set_state(g, s);
    uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

uint32_t rno_pcg64_next32(rno_pcg64 *g)
{
    if (g->has_uint32) {
        g->has_uint32 = 0;
        return g->uinteger;
    }
    uint64_t v = rno_pcg64_next64(g);
    g->has_uint32 = 1;
    g->uinteger = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

uint64_t rno_integers(rno_pcg64 *g, uint64_t k)
{
    uint64_t rng = k - 1;
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFull) return rno_pcg64_next32(g);
    uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)rno_pcg64_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
        while (left < thr) {
            m = (uint64_t)rno_pcg64_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return m >> 32;
}

int rno_init_field(int gw, int gh, int64_t n, const uint32_t *seed_words,
                   int nwords, int32_t *out)
{
    if (n < 1 || gw < 1 || gh < 1) return -1;
    rno_pcg64 g;
    rno_pcg64_seed(&g, seed_words, nwords);
    int64_t total = (int64_t)gw * gh;
    for (int64_t i = 0; i < total; i++) out[i] = (int32_t)rno_integers(&g, (uint64_t)n);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* search.py:63-80: lo = searchsorted(row, d-eps, 'left'),
 * hi = searchsorted(row, d+eps, 'right'); row values compared as float64. */
void rno_ring_window(const float *row, int64_t n, double d, double eps,
                     int64_t *lo, int64_t *hi)
{
    double lv = d - eps, hv = d + eps;
    int64_t a = 0, b = n;
    while (a < b) {
        int64_t m = a + (b - a) / 2;
        if ((double)row[m] < lv) a = m + 1; else b = m;
    }
    *lo = a;
    a = 0;
    b = n;
    while (a < b) {
        int64_t m = a + (b - a) / 2;
        if ((double)row[m] <= hv) a = m + 1; else b = m;
    }
    *hi = a;
}

typedef struct {
    int32_t *cand, *tmp, *avail, *used;
    unsigned char *mark;
    double *dtmp;
    double *dists;
    uint64_t *keys; /* lazy row builds */
} query_scratch;

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

static void *query_mk_n(int64_t n, int dim)
{
    query_scratch *s = (query_scratch *)malloc(sizeof(*s));
    s->cand = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    s->tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    s->avail = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    s->used = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    s->mark = (unsigned char *)calloc((size_t)n, 1);
    s->dtmp = (double *)malloc(sizeof(double) * (size_t)dim);
    s->dists = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    s->keys = (uint64_t *)malloc(sizeof(uint64_t) * 2 * (size_t)n);
    return s;
}

static void query_fr(void *p)
{
    query_scratch *s = (query_scratch *)p;
    free(s->cand);
    free(s->tmp);
    free(s->avail);
    free(s->used);
    free(s->mark);
    free(s->dtmp);
    free(s->dists);
    free(s->keys);
    free(s);
}

static void ensure_row(const rno_model *m, int64_t a, query_scratch *s)
{
    if (!m->row_state) return;
    unsigned char *st = m->row_state + a;
    if (__atomic_load_n(st, __ATOMIC_ACQUIRE) == 2) return;
    unsigned char expect = 0;
    if (__atomic_compare_exchange_n(st, &expect, 1, 0, __ATOMIC_ACQ_REL, __ATOMIC_ACQUIRE)) {
        build_row(m->refs, m->n, m->dim, a, (float *)m->sorted_dist + a * m->n,
                  (int32_t *)m->sorted_idx + a * m->n, s->dtmp, s->keys);
        __atomic_store_n(st, 2, __ATOMIC_RELEASE);
    } else {
        while (__atomic_load_n(st, __ATOMIC_ACQUIRE) != 2) sched_yield();
    }
}

int rno_lazy_tables_create(int64_t n, float **sdist, int32_t **sidx, unsigned char **state)
{
    size_t bytes = (size_t)n * (size_t)n * 4;
    void *a = mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (a == MAP_FAILED) return -1;
    void *b = mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (b == MAP_FAILED) {
        munmap(a, bytes);
        return -1;
    }
    *sdist = (float *)a;
    *sidx = (int32_t *)b;
    *state = (unsigned char *)calloc((size_t)n, 1);
    return 0;
}

void rno_lazy_tables_free(int64_t n, float *sdist, int32_t *sidx, unsigned char *state)
{
    size_t bytes = (size_t)n * (size_t)n * 4;
    if (sdist) munmap(sdist, bytes);
    if (sidx) munmap(sidx, bytes);
    free(state);
}

int64_t rno_lazy_rows_ready(const unsigned char *state, int64_t n)
{
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++) c += state[i] == 2;
    return c;
}

/* search.py:83-151 */
static int query_impl(const rno_model *m, const float *q, int32_t prev, int L,
                      double alpha, int max_rings, const uint32_t *key, int nkey,
                      rno_result *res, int32_t *scanned, int64_t *nscanned,
                      query_scratch *s)
{
    int64_t n = m->n;
    int dim = m->dim;
    if (prev < 0 || prev >= n) return -2;
    ensure_row(m, prev, s);
    double d = sq_dist(q, m->refs + (int64_t)prev * dim, dim, s->dtmp);
    int64_t evals = 1;
    int64_t lo, hi;
    rno_ring_window(m->sorted_dist + (int64_t)prev * n, n, d, alpha * d, &lo, &hi);
    int64_t nc = hi - lo;
    memcpy(s->cand, m->sorted_idx + (int64_t)prev * n + lo, sizeof(int32_t) * (size_t)nc);
    qsort(s->cand, (size_t)nc, sizeof(int32_t), cmp_i32);
    int rings = 1;
    res->first_ring = nc;

    /* used anchors carry bit 1 of mark[]; ring members bit 0 */
    int64_t nused = 0;
    s->used[nused++] = prev;
    s->mark[prev] |= 2;
    int have_rng = 0;
    rno_pcg64 g;
    while (nc >= L && rings < max_rings) {
        int64_t na = 0;
        for (int64_t i = 0; i < nc; i++)
            if (!(s->mark[s->cand[i]] & 2)) s->avail[na++] = s->cand[i];
        if (na == 0) break;
        if (!have_rng) {
            rno_pcg64_seed(&g, key, nkey);
            have_rng = 1;
        }
        int32_t a = s->avail[rno_integers(&g, (uint64_t)na)];
        s->used[nused++] = a;
        s->mark[a] |= 2;
        double da = sq_dist(q, m->refs + (int64_t)a * dim, dim, s->dtmp);
        evals++;
        ensure_row(m, a, s);
        rno_ring_window(m->sorted_dist + (int64_t)a * n, n, da, alpha * da, &lo, &hi);
        const int32_t *ring = m->sorted_idx + (int64_t)a * n;
        for (int64_t i = lo; i < hi; i++) s->mark[ring[i]] |= 1;
        int64_t nn = 0;
        for (int64_t i = 0; i < nc; i++)
            if (s->mark[s->cand[i]] & 1) s->tmp[nn++] = s->cand[i];
        for (int64_t i = lo; i < hi; i++) s->mark[ring[i]] &= (unsigned char)~1u;
        rings++;
        if (nn == 0) break; /* rollback: keep the pre-intersection set */
        int32_t *t = s->cand;
        s->cand = s->tmp;
        s->tmp = t;
        nc = nn;
    }
    for (int64_t u = 0; u < nused; u++) s->mark[s->used[u]] = 0;

    /* scanned = union1d(cand, [prev]) */
    int64_t ns = 0;
    int inserted = 0;
    for (int64_t i = 0; i < nc; i++) {
        if (!inserted && prev <= s->cand[i]) {
            if (prev < s->cand[i]) s->tmp[ns++] = prev;
            inserted = 1;
        }
        s->tmp[ns++] = s->cand[i];
    }
    if (!inserted) s->tmp[ns++] = prev;
    int32_t best = -1;
    double bd = 0.0;
    for (int64_t i = 0; i < ns; i++) {
        double di = sq_dist(q, m->refs + (int64_t)s->tmp[i] * dim, dim, s->dtmp);
        if (best < 0 || di < bd) { /* strict: first minimum wins */
            best = s->tmp[i];
            bd = di;
        }
    }
    evals += ns;
    res->match_index = best;
    res->match_distance = bd;
    res->rings = rings;
    res->evals = evals;
    res->cand_final = nc;
    if (scanned) memcpy(scanned, s->tmp, sizeof(int32_t) * (size_t)ns);
    if (nscanned) *nscanned = ns;
    return 0;
}

int rno_query(const rno_model *m, const float *q, int32_t prev, int L,
              double alpha, int max_rings, const uint32_t *key, int nkey,
              rno_result *res, int32_t *scanned, int64_t *nscanned)
{
    query_scratch *s = (query_scratch *)query_mk_n(m->n, m->dim);
    int rc = query_impl(m, q, prev, L, alpha, max_rings, key, nkey, res, scanned, nscanned, s);
    query_fr(s);
    return rc;
}

static int key_words(uint64_t seed, uint32_t x, uint32_t y, uint32_t t, uint32_t *w)
{
    int k = 0;
    w[k++] = (uint32_t)seed;
    if (seed >> 32) w[k++] = (uint32_t)(seed >> 32);
    w[k++] = x;
    w[k++] = y;
    w[k++] = t;
    return k;
}

typedef struct {
    const rno_model *m;
    const float *units;
    const int32_t *prev;
    const int64_t *pos;
    int gw;
    uint64_t seed;
    uint32_t t;
    int L, max_rings;
    double alpha;
    int32_t *oi;
    double *od;
    int32_t *orings;
    int64_t *oe, *oc, *of;
    int err;
} pos_ctx;

static void *pos_mk(void *c)
{
    pos_ctx *p = (pos_ctx *)c;
    return query_mk_n(p->m->n, p->m->dim);
}

static void pos_run(void *c, int64_t lo, int64_t hi, void *scr)
{
    pos_ctx *p = (pos_ctx *)c;
    for (int64_t i = lo; i < hi; i++) {
        int64_t g = p->pos[i];
        uint32_t w[5];
        int nw = key_words(p->seed, (uint32_t)(g % p->gw), (uint32_t)(g / p->gw), p->t, w);
        rno_result r;
        int rc = query_impl(p->m, p->units + i * p->m->dim, p->prev[i], p->L, p->alpha,
                            p->max_rings, w, nw, &r, NULL, NULL, (query_scratch *)scr);
        if (rc) { p->err = rc; continue; }
        if (p->oi) p->oi[i] = r.match_index;
        if (p->od) p->od[i] = r.match_distance;
        if (p->orings) p->orings[i] = r.rings;
        if (p->oe) p->oe[i] = r.evals;
        if (p->oc) p->oc[i] = r.cand_final;
        if (p->of) p->of[i] = r.first_ring;
    }
}

int rno_query_positions(const rno_model *m, const float *units,
                        const int32_t *prev, const int64_t *positions,
                        int64_t count, int gw, uint64_t seed, uint32_t t,
                        int L, double alpha, int max_rings, int nthreads,
                        int32_t *out_idx, double *out_dist, int32_t *out_rings,
                        int64_t *out_evals, int64_t *out_cand,
                        int64_t *out_first)
{
    pos_ctx c = {m, units, prev, positions, gw, seed, t, L, max_rings, alpha,
                 out_idx, out_dist, out_rings, out_evals, out_cand, out_first, 0};
    /* chunks of ceil(count / (4 * threads)) positions (at most 64): every
     * thread gets work even for a few hundred positions */
    {
        int64_t nt = nthreads < 1 ? 1 : nthreads, ch = (count + 4 * nt - 1) / (4 * nt);
        if (ch > 64) ch = 64;
        pool_run(nthreads, count, ch, pos_run, &c, pos_mk, query_fr);
    }
    return c.err;
}

/* engine.py:163-171 */
double rno_temporal_change(const float *unit, const float *prev_unit,
                           int64_t rows, int dim)
{
    double *tmp = (double *)malloc(sizeof(double) * (size_t)dim);
    double *per = (double *)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
    for (int64_t r = 0; r < rows; r++) {
        const float *a = unit + r * dim, *b = prev_unit + r * dim;
        for (int i = 0; i < dim; i++) {
            double d = (double)a[i] - (double)b[i];
            tmp[i] = d * d;
        }
        per[r] = sqrt(rno_pairwise_sum(tmp, dim));
    }
    double s = rno_pairwise_sum(per, rows);
    free(tmp);
    free(per);
    return s;
}

/* evaluation.py:24-33 */
void rno_exact_nn(const float *refs, int64_t n, int dim, const float *q,
                  int32_t *idx, double *dist)
{
    double *tmp = (double *)malloc(sizeof(double) * (size_t)dim);
    int32_t best = 0;
    double bd = 0.0;
    for (int64_t j = 0; j < n; j++) {
        double d = sq_dist(q, refs + j * dim, dim, tmp);
        if (j == 0 || d < bd) {
            best = (int32_t)j;
            bd = d;
        }
    }
    free(tmp);
    *idx = best;
    *dist = bd;
}

typedef struct {
    const float *refs, *qs;
    int64_t n;
    int dim;
    int32_t *idx;
    double *dist;
} enn_ctx;

static void enn_run(void *c, int64_t lo, int64_t hi, void *scr)
{
    (void)scr;
    enn_ctx *e = (enn_ctx *)c;
    for (int64_t i = lo; i < hi; i++)
        rno_exact_nn(e->refs, e->n, e->dim, e->qs + i * e->dim, e->idx + i, e->dist + i);
}

int rno_exact_nn_batch(const float *refs, int64_t n, int dim,
                       const float *queries, int64_t count, int nthreads,
                       int32_t *idx, double *dist)
{
    enn_ctx c = {refs, queries, n, dim, idx, dist};
    {
        int64_t nt = nthreads < 1 ? 1 : nthreads, ch = (count + 4 * nt - 1) / (4 * nt);
        if (ch > 8) ch = 8;
        pool_run(nthreads, count, ch, enn_run, &c, NULL, NULL);
    }
    return 0;
}

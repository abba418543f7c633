/*
 * riann_oracle.h -- CPU restatement of the reference RIANN per-frame query path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline and
 * --impl reference legs).  Nothing in paper_1508_07953_b200/ links or calls it.
 *
 * Every function names the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/riann/).  Third-party arithmetic the reference relies
 * on (numpy 2.3.5, not vendored) is restated from numpy's published
 * algorithms: float64 pairwise summation, SeedSequence, PCG64, and
 * Generator.integers' 32-bit Lemire rejection sampler.  The restatement is
 * pinned against golden vectors generated from the live reference
 * (tests/golden/make_golden.py).
 */
#ifndef RIANN_ORACLE_H
#define RIANN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* numpy float64 pairwise summation (8 accumulators, blocks of <=128, halving
 * split rounded down to a multiple of 8).  Used by np.sum along a contiguous
 * axis: patches.py:110 (normalize_rows), :159 (one_to_many), engine.py:169. */
double rno_pairwise_sum(const double *a, int64_t n);

/* patches.py:151-159  EuclideanMetric.one_to_many: sqrt(sum((f64 r - f64 q)^2)).
 * rows == NULL means rows 0..k-1 of refs; otherwise refs[rows[i]]. */
void rno_one_to_many(const float *q, const float *refs, const int64_t *rows,
                     int64_t k, int dim, double *out);

/* patches.py:100-115 normalize_rows: f32(f64 v / sqrt(pairwise sum v^2)),
 * rows with norm < 1e-12 become zero with norm 0.  norms may be NULL. */
void rno_normalize_rows(const float *values, int64_t m, int dim, float *unit,
                        double *norms);

/* patches.py:65-97 extract_patches (stride 1, row-major dy*pw+dx) followed by
 * normalize_rows, for grid rows [y0, y1).  Frames are (H, W, C) row-major; for
 * C > 1 each patch is the plane-major concatenation c*pw*ph + dy*pw + dx
 * (transforms.py:152-157 precedent; the reference query path is luminance
 * only).  unit: (y1-y0)*gw rows of dim = pw*ph*C. */
int rno_frame_units(const float *frame, int H, int W, int C, int pw, int ph,
                    int y0, int y1, float *unit, double *norms);

/* model.py:162-189 compute_sorted_lists for rows [row0, row0+rows):
 * f32(f64 distance), stable ascending argsort, self entry forced first.
 * sdist/sidx are (rows, n). */
int rno_sorted_lists(const float *refs, int64_t n, int dim, int64_t row0,
                     int64_t rows, float *sdist, int32_t *sidx, int nthreads);

/* numpy SeedSequence -> PCG64 -> Generator.integers(k). */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int has_uint32;
    uint32_t uinteger;
} rno_pcg64;

/* _coerce_to_uint32_array + SeedSequence(pool 4).generate_state(4, u64) +
 * PCG64 seeding (pcg64_set_seed / srandom). */
void rno_pcg64_seed(rno_pcg64 *g, const uint32_t *words, int nwords);
uint64_t rno_pcg64_next64(rno_pcg64 *g);
uint32_t rno_pcg64_next32(rno_pcg64 *g);
/* Generator.integers(k) for 1 <= k <= 2^32 (k == 1 consumes nothing). */
uint64_t rno_integers(rno_pcg64 *g, uint64_t k);

/* engine.py:72-82 init_field indices: default_rng(seed).integers(0, n,
 * (gh, gw), int32), row-major.  seed_words as for rno_pcg64_seed. */
int rno_init_field(int gw, int gh, int64_t n, const uint32_t *seed_words,
                   int nwords, int32_t *out);

/* search.py:63-80 ring_candidates window [lo, hi) on one sorted row. */
void rno_ring_window(const float *row, int64_t n, double d, double eps,
                     int64_t *lo, int64_t *hi);

typedef struct {
    const float *refs;        /* (n, dim) */
    const float *sorted_dist; /* (n, n), values exactly the reference's f64 */
    const int32_t *sorted_idx;/* (n, n) */
    int64_t n;
    int dim;
    /* NULL: tables complete.  Otherwise per-row state (0 absent, 1 building,
     * 2 ready): rows are built on first use (model.py:162-189 per row), so a
     * sampled query run touches only the rows it needs. */
    unsigned char *row_state;
} rno_model;

/* Lazily backed (n, n) tables for rno_model.row_state mode (anonymous
 * MAP_NORESERVE mappings: untouched rows cost no memory). */
int rno_lazy_tables_create(int64_t n, float **sdist, int32_t **sidx, unsigned char **state);
void rno_lazy_tables_free(int64_t n, float *sdist, int32_t *sidx, unsigned char *state);
int64_t rno_lazy_rows_ready(const unsigned char *state, int64_t n);

typedef struct {
    int32_t match_index;
    int32_t rings;
    double match_distance;
    int64_t evals;
    int64_t cand_final;
    int64_t first_ring;       /* |S_1|, for the roofline byte count */
} rno_result;

/* search.py:83-151 riann_query with rng_state = key words (the engine's
 * query_rng_key (seed, x, y, t), search.py:154-157, coerced to uint32 words).
 * scanned (optional, capacity n+1) receives S u {prev} ascending. */
int rno_query(const rno_model *m, const float *q, int32_t prev, int L,
              double alpha, int max_rings, const uint32_t *key, int nkey,
              rno_result *res, int32_t *scanned, int64_t *nscanned);

/* engine.py:134-148 for an explicit list of grid positions g (y = g / gw,
 * x = g % gw), run with nthreads pthreads.  units: (count, dim) rows aligned
 * with positions; prev: per position previous index. */
int rno_query_positions(const rno_model *m, const float *units,
                        const int32_t *prev, const int64_t *positions,
                        int64_t count, int gw, uint64_t seed, uint32_t t,
                        int L, double alpha, int max_rings, int nthreads,
                        int32_t *out_idx, double *out_dist, int32_t *out_rings,
                        int64_t *out_evals, int64_t *out_cand,
                        int64_t *out_first);

/* engine.py:163-171 temporal_change: pairwise sum over rows of the f64
 * distance between unit rows. */
double rno_temporal_change(const float *unit, const float *prev_unit,
                           int64_t rows, int dim);

/* evaluation.py:24-33 exact_nn: full FP64 scan, first minimum. */
void rno_exact_nn(const float *refs, int64_t n, int dim, const float *q,
                  int32_t *idx, double *dist);
int rno_exact_nn_batch(const float *refs, int64_t n, int dim,
                       const float *queries, int64_t count, int nthreads,
                       int32_t *idx, double *dist);

#ifdef __cplusplus
}
#endif
#endif

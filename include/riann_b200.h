/*
 * riann_b200.h -- C ABI of the B200-native RIANN per-frame ANN-field query.
 *
 * The reference (/root/reference/pkg/src/riann, pure Python) has no FFI for
 * this path: its boundary is the module-level Python API.  Each entry point
 * below names the reference function it replaces (file:line); the Python
 * package paper_1508_07953_b200 binds these with ctypes (INTEGRATION.md shows
 * the binding a maintainer of the reference would add).
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types cross the ABI.
 *  - Every int-returning call returns RIANN_OK or an error code; the message is
 *    riann_last_error() (thread-local).  Codes map to the reference's
 *    exception types (errors.py:4-17 plus ValueError/IndexError).
 *  - Host pointers unless a flag says RIANN_F_DEVICE_PTRS.  Calls on one
 *    context are serialised by the caller; one context per GPU.
 *  - Floating point: every distance is the reference's float64 expression
 *    (patches.py:151-159) evaluated with individually rounded IEEE ops in
 *    numpy's pairwise-summation order, so results are bit-identical.
 */
#ifndef RIANN_B200_H
#define RIANN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RIANN_ABI_VERSION 2

enum {
    RIANN_OK = 0,
    RIANN_E_VALUE = 1,       /* ValueError        (search.py:42-48, engine.py:75-78) */
    RIANN_E_DIMENSION = 2,   /* DimensionError    (engine.py:111-119, search.py:105-108) */
    RIANN_E_INDEX = 3,       /* IndexError        (search.py:73-74, :110-111) */
    RIANN_E_CAPACITY = 4,    /* ModelCapacityError (model.py:252-257): device memory */
    RIANN_E_UNSUPPORTED = 5, /* metric_id != 0, >2^32 key words, ... (no fallback) */
    RIANN_E_CUDA = 6,        /* CUDA runtime failure */
    RIANN_E_STATE = 7        /* call order (no model / no tables / no field) */
};

/* flags for riann_process_frame */
#define RIANN_F_TEMPORAL 1u     /* compute temporal_change vs the units kept from the previous frame */
#define RIANN_F_DEVICE_PTRS 2u  /* frame / prev / outputs are device pointers on the ctx device */
#define RIANN_F_ASYNC 4u        /* do not synchronise (device-pointer mode only); stats invalid until riann_sync */
#define RIANN_F_KEEP_UNITS 8u   /* keep this frame's units as the next frame's prev units */

typedef struct riann_ctx riann_ctx;

/* FrameStats (engine.py:56-69) as integers plus the float64 temporal change;
 * mean_candidates = sum_cand_final / queries (engine.py:183). */
typedef struct {
    uint64_t total_rings;
    uint64_t total_distance_evals;
    uint64_t sum_cand_final;
    uint64_t sum_first_ring;   /* sum |S_1|: roofline byte count */
    uint64_t queries;
    double temporal_change;
    uint64_t sum_ring_tests;   /* sum over rings of |S| membership lookups */
    uint64_t sum_exact_evals;  /* FP64 distances actually evaluated (screening survivors) */
    uint64_t queries_fallback; /* queries the anchor-grouped path handed to the per-query kernel */
} riann_frame_stats;

int riann_abi_version(void);
/* 1 when the library was built with device-side bounds checks (-DRIANN_BOUNDS) */
int riann_debug_checks(void);
const char *riann_last_error(void);

/* ---- context ---------------------------------------------------------- */
int riann_ctx_create(int device, riann_ctx **out);
int riann_ctx_destroy(riann_ctx *ctx);
/* the context's CUDA stream (cudaStream_t), for event timing by the caller */
void *riann_ctx_stream(riann_ctx *ctx);
int riann_sync(riann_ctx *ctx);
/* device bytes currently held by the context */
uint64_t riann_ctx_device_bytes(riann_ctx *ctx);
/* Path selection mask: 0 = auto (anchor-grouped frame phases when n <= 65,536
 * and dim is 64 or 192; tensor-core exact comparator for dim 64 / 192);
 * bit 1 = per-query frame kernel only; bit 2 = SIMT exact comparator.
 * All paths produce identical results; the switch exists for testing. */
int riann_ctx_set_path(riann_ctx *ctx, int path);

/* ---- stream slots ------------------------------------------------------ */
/* The device-resident stream state (previous field, previous frame's unit
 * rows, replay snapshot) lives in a slot; the context has one active slot
 * (0 at creation) and keeps the others parked.  The reference's
 * stream_fields (engine.py:205-227) is a generator with no shared state, so
 * every stream (a clip, a row band) selects its own slot before
 * riann_process_frame: interleaved streams on one GPU never read each
 * other's field or units.  Selecting an unknown slot creates it empty;
 * freeing the active slot empties it and selects slot 0.  A model upload
 * invalidates every slot's field and units. */
int riann_slot_select(riann_ctx *ctx, int slot);
int riann_slot_current(riann_ctx *ctx);
int riann_slot_free(riann_ctx *ctx, int slot);

/* ---- model (model.py:56-83 ReferenceModel) ----------------------------- */
/* refs: (n, dim) float32 unit rows; patch (pw, ph); channels; metric_id must
 * be 0 (Euclidean, patches.py:164-179).  dim must equal pw*ph*channels. */
int riann_model_set_refs(riann_ctx *ctx, const float *refs, int64_t n, int dim,
                         int pw, int ph, int channels, int metric_id);
/* Upload reference-built sorted tables (compute_sorted_lists output):
 * sorted_dist float32 (n, n) (the reference's float64 values are exactly
 * float32), sorted_idx int32 (n, n).  Replaces model.py:162-189's result. */
int riann_model_set_tables(riann_ctx *ctx, const float *sorted_dist,
                           const int32_t *sorted_idx);
/* K3: build the sorted tables on the GPU, bit-identical to
 * compute_sorted_lists (model.py:162-189). */
int riann_model_build_tables(riann_ctx *ctx);
/* ---- row-sharded tables (config 4: n = 262,144 needs 768 GiB of tables) ---
 * K3 for rows [row0, row0 + rows) only (a shard; compute_sorted_lists
 * model.py:177-188 restricted to those rows).  A context holding a partial
 * range serves as a shard owner; it cannot run frames itself. */
int riann_model_build_table_rows(riann_ctx *ctx, int64_t row0, int64_t rows);
/* Device pointers of this context's table rows (sorted distances f32,
 * sorted indices u16 if n <= 65,536 else i32, index-ordered distances f32)
 * and the row range they hold. */
int riann_model_table_ptrs(riann_ctx *ctx, void **sdist, void **sidx, void **dmat, int64_t *row0,
                           int64_t *rows);
/* Use nshards row shards as this context's tables: row a lives in shard
 * a / shard_rows at offset (a % shard_rows) * n.  Shards on other GPUs are
 * read with NVLink peer loads (peer access is enabled here).  The frame path
 * then runs the per-query kernel (the anchor-grouped path needs local rank
 * rows).  The owners must outlive this context's use of the shards. */
int riann_model_attach_shards(riann_ctx *ctx, int nshards, int64_t shard_rows, void *const *sdist,
                              void *const *sidx, void *const *dmat);
/* Forget attached shards (before their owners free them): the context has no
 * tables afterwards, so frame calls fail with RIANN_E_STATE. */
int riann_model_detach_shards(riann_ctx *ctx);
/* Download rows [row0, row0+rows) of the sorted tables. */
int riann_model_get_tables(riann_ctx *ctx, int64_t row0, int64_t rows,
                           float *sorted_dist, int32_t *sorted_idx);

/* ---- frame path (engine.py:93-187 process_frame) ----------------------- */
/* frame: (H, W, C) float32 rows [gy0, gy0 + gh + ph - 1) of the full frame,
 * i.e. a row band with a (ph-1)-row halo; the band's grid rows are
 * [gy0, gy0 + H - ph + 1) of a grid gw = W - pw + 1 wide.  RNG keys use the
 * global (x, y) = (g % gw, gy0 + g / gw) and t (engine.py:124, 136-142).
 * prev_idx: (gh_band, gw) previous indices, or NULL to use the field kept on
 * the device by the previous call.  out_idx / out_dist may be NULL (the field
 * stays device-resident).  seed < 2^64. */
int riann_process_frame(riann_ctx *ctx, const float *frame, int H, int W, int C,
                        int gy0, const int32_t *prev_idx, uint64_t seed,
                        uint32_t t, int L, double alpha, int max_rings,
                        unsigned flags, int32_t *out_idx, double *out_dist,
                        riann_frame_stats *stats);
/* Upload prev units (rows, dim) for the next RIANN_F_TEMPORAL frame
 * (process_frame's prev_unit argument, engine.py:163-171). */
int riann_set_prev_units(riann_ctx *ctx, const float *units, int64_t rows, int dim);
/* Per-kernel CUDA-event timing of riann_process_frame on the ctx stream:
 * enable (on=1) clears the accumulators; read synchronises and returns the
 * summed milliseconds of [K1 units, K2 query, pairwise reduction], the number
 * of frames and of kernel launches since enable. */
int riann_timing_enable(riann_ctx *ctx, int on);
int riann_timing_read(riann_ctx *ctx, double *ms3, uint64_t *frames, uint64_t *launches);
/* Per-phase split of the same frames (CUDA events between the phases'
 * launches on the ctx stream, summed ms): units, p0a, p0b, draw, group,
 * window, filter, final, tail, query (riann_phase_name(k)).  The same
 * phases are NVTX ranges ("riann:<phase>") for ncu --nvtx. */
#define RIANN_NPHASES 10
int riann_timing_phases(riann_ctx *ctx, double *ms, int nphases);
/* The same split for one timed frame (frame < 0 counts from the last). */
int riann_timing_phases_frame(riann_ctx *ctx, int64_t frame, double *ms, int nphases);
const char *riann_phase_name(int k);
/* Snapshot / restore of the device-resident stream state (previous field and
 * previous units), e.g. to replay the same frames; one snapshot per context. */
int riann_state_save(riann_ctx *ctx);
int riann_state_restore(riann_ctx *ctx);
/* Per-position temporal-change terms ||unit_t[g] - unit_{t-1}[g]|| (float64)
 * of the last RIANN_F_TEMPORAL frame on this context (engine.py:163-171
 * before its sum), so that row bands can be summed in numpy's pairwise order
 * over the whole frame.  Valid until the next riann_process_frame on the
 * context; flags may hold RIANN_F_DEVICE_PTRS (out on the ctx device, no
 * synchronisation). */
int riann_tc_get(riann_ctx *ctx, double *out, int64_t count, unsigned flags);
/* Read back the device-resident field of the last frame. */
int riann_field_get(riann_ctx *ctx, int32_t *idx, double *dist, int64_t count);

/* extract_patches + normalize_rows (patches.py:65-115) on the GPU:
 * unit (Q, dim) float32, norms (Q,) float64 (either may be NULL). */
int riann_frame_units(riann_ctx *ctx, const float *frame, int H, int W, int C,
                      float *unit, double *norms);
/* normalize_rows (patches.py:100-115) on arbitrary rows. */
int riann_normalize_rows(riann_ctx *ctx, const float *values, int64_t m, int dim,
                         float *unit, double *norms);
/* float64-input variant (the reference converts any input to float64). */
int riann_normalize_rows_f64(riann_ctx *ctx, const double *values, int64_t m,
                             int dim, float *unit, double *norms);
/* EuclideanMetric.one_to_many (patches.py:151-159): q (dim,), rows (k, dim). */
int riann_one_to_many(riann_ctx *ctx, const float *q, const float *rows,
                      int64_t k, int dim, double *out);
int riann_one_to_many_f64(riann_ctx *ctx, const double *q, const double *rows,
                          int64_t k, int dim, double *out);
/* extract_patches (patches.py:65-97): raw windows at `stride`, row-major
 * dy*pw+dx, plane-major channels; out (gh*gw, pw*ph*C). */
int riann_extract_patches(riann_ctx *ctx, const float *frame, int H, int W,
                          int C, int pw, int ph, int stride, float *out);

/* ---- single / batched queries (search.py:63-151) ----------------------- */
/* ring_candidates (search.py:63-80) on the model's table: window [lo, hi) of
 * row `anchor` and (if out != NULL, capacity n) its index slice. */
int riann_ring_candidates(riann_ctx *ctx, int64_t anchor, double d, double eps,
                          int64_t *lo, int64_t *hi, int32_t *out);
/* riann_query (search.py:83-151) for m queries with explicit RNG keys:
 * key words of query i are key_words[key_off[i] .. key_off[i+1]) (numpy
 * SeedSequence entropy words, <= 16 per key).  Optional outputs may be NULL.
 * scanned: capacity m * (n + 1); query i writes S u {prev} ascending at
 * scanned + i*(n+1), its length in scanned_len[i]. */
int riann_query_batch(riann_ctx *ctx, const float *queries, const int32_t *prev,
                      const uint32_t *key_words, const int64_t *key_off, int64_t m,
                      int L, double alpha, int max_rings, int32_t *out_idx,
                      double *out_dist, int32_t *out_rings, int64_t *out_evals,
                      int64_t *out_cand, int64_t *out_first, int32_t *scanned,
                      int64_t *scanned_len);

/* ---- exact comparator (evaluation.py:24-50) ----------------------------- */
/* Exact nearest reference per query: index of the first minimum of the
 * float64 distances (numpy argmin), bit-identical to exact_nn.  For dim 64
 * and 192 the distances are screened on the tensor cores (tcgen05 bf16x3
 * split GEMM with rigorous bounds) and the survivors re-evaluated in float64;
 * riann_ctx_set_path bit 2 selects the SIMT full scan instead. */
int riann_exact_nn_batch(riann_ctx *ctx, const float *queries, int64_t m,
                         int32_t *out_idx, double *out_dist);
/* Same on device buffers, asynchronous on the context stream.  stats (may be
 * NULL; synchronises): [0] float64 re-checks, [1] queries that took the full
 * exact scan (screen list overflow). */
int riann_exact_nn_device(riann_ctx *ctx, const float *queries, int64_t m,
                          int32_t *out_idx, double *out_dist, uint64_t *stats);
int riann_exact_field(riann_ctx *ctx, const float *frame, int H, int W, int C,
                      int32_t *out_idx, double *out_dist);

/* ---- output side of the query ----------------------------- */
/* One ANNF frame payload (engine.py:257-267) from the device-resident field:
 * count little-endian u32 indices, then count f32 distances (f64 rounded to
 * nearest), 8 * count bytes.  count must equal the field's position count. */
int riann_field_pack(riann_ctx *ctx, void *payload, int64_t count);
/* apply_effect / reconstruct_frame (transforms.py:192-253) on a single-plane
 * frame (H, W): kind 0 reconstruction (payloads NULL = the model's refs,
 * rescaled by each query patch's norm), 1 full-patch, 2 chroma-pair (payload
 * width 2*pw*ph).  idx: (gh, gw) host matches, or NULL for the device field.
 * out_planes (planes, H, W) f32 may be NULL; out_rgb (H, W, 3) u8 for kind 2.
 * Bit-identical to numpy (same f32 add order, division and rounding). */
int riann_apply_effect(riann_ctx *ctx, const float *frame, int H, int W,
                       const int32_t *idx, const float *payloads, int64_t n_payloads,
                       int payload_dim, int kind, float *out_planes, uint8_t *out_rgb);

/* coherency_stats support (evaluation.py:86-138): for m index pairs,
 * out_ab[k] = dist(refs[ia[k]], refs[ib[k]]) and, when u (m, dim) is given,
 * out_au[k] = dist(refs[ia[k]], u[k]) -- numpy-order float64 distances. */
int riann_pair_dist(riann_ctx *ctx, const int32_t *ia, const int32_t *ib,
                    const float *u, int64_t m, double *out_ab, double *out_au);

/* ---- host helpers ------------------------------------------------------ */
/* init_field indices (engine.py:72-82): numpy default_rng(seed).integers(0,
 * n, (gh, gw), int32), bit-identical; seed given as SeedSequence words. */
int riann_init_field(int gw, int gh, int64_t n, const uint32_t *seed_words,
                     int nwords, int32_t *out);
/* numpy pairwise float64 sum (for the host side of multi-band reductions) */
double riann_pairwise_sum(const double *a, int64_t n);

#ifdef __cplusplus
}
#endif
#endif

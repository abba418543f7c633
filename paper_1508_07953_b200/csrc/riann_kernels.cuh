// riann_kernels.cuh -- the sm_100a kernels of the RIANN per-frame query path.
//
//   K1 units_kernel        extract_patches + normalize_rows (+ temporal change
//                          per position)            patches.py:65-115, engine.py:163-171
//   K2 query_kernel        riann_query per grid position, one warp per query
//                                                    search.py:63-151, engine.py:134-148
//   K3 table_keys_kernel   compute_sorted_lists distance rows (sorted by CUB
//      + self_first_kernel segmented radix sort)     model.py:162-189
//   K4 exact_nn_kernel     exact_nn / field_exact_oracle   evaluation.py:24-50
//   pw_tree_kernel         numpy pairwise sum over Q per-position values
#pragma once

#include <cuda_fp16.h>

#include "riann_device.cuh"

namespace rb {


// ---------------------------------------------------------------------------
// K1: one thread per grid position.  Frame (H, W, C) row-major; patch element
// e = c*pw*ph + dy*pw + dx (row-major window, plane-major channels).
struct UnitsParams {
    const float *frame;
    int H, W, C, pw, ph, gw;
    int64_t Q;
    int dim;
    float *unit;              // (Q, dim)
    double *norms;            // (Q) or null
    const float *prev_unit;   // (Q, dim) or null
    double *tc;               // (Q) or null
};

template <int PW, int PH>
struct FrameGet {
    const float *f;
    int W, C, pw, ph;
    __device__ __forceinline__ float raw(int64_t e) const
    {
        const int pp = (PW > 0 ? PW * PH : pw * ph);
        int c = (int)(e / pp);
        int r = (int)(e - (int64_t)c * pp);
        int dy = PW > 0 ? r / PW : r / pw;
        int dx = PW > 0 ? r % PW : r % pw;
        return f[((int64_t)dy * W + dx) * C + c];
    }
    __device__ __forceinline__ double operator()(int64_t e) const
    {
        double v = (double)raw(e);
        return __dmul_rn(v, v);
    }
};

struct DiffGet {
    const float *a, *b;
    __device__ __forceinline__ double operator()(int64_t i) const { return sqdiff(a[i], b[i]); }
};

template <int PW, int PH>
__global__ void __launch_bounds__(128) units_kernel(UnitsParams P)
{
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.Q) return;
    int x = (int)(g % P.gw), y = (int)(g / P.gw);
    FrameGet<PW, PH> get{P.frame + ((int64_t)y * P.W + x) * P.C, P.W, P.C, P.pw, P.ph};
    double nr = __dsqrt_rn(pw_sum(get, 0, P.dim));
    bool ok = nr >= 1e-12;
    float *u = P.unit + g * P.dim;
    for (int e = 0; e < P.dim; e++)
        u[e] = ok ? __double2float_rn(__ddiv_rn((double)get.raw(e), nr)) : 0.0f;
    if (P.norms) P.norms[g] = ok ? nr : 0.0;
    if (P.tc) {
        DiffGet dg{u, P.prev_unit + g * P.dim};
        P.tc[g] = __dsqrt_rn(pw_sum(dg, 0, P.dim));
    }
}

// K1, warp-cooperative form for 8x8 patches with D = 64 * C in {64, 192}:
// lane (h, dx) of a Lay<D>::G-lane group owns numpy's pairwise accumulator dx
// of half h, so the squared norm and the temporal-change distance come out of
// the same xor tree as exact_dist; unit rows are written by the group with
// 32-byte runs per step.  One group per grid position.
template <int D>
__global__ void __launch_bounds__(256) units_warp_kernel(UnitsParams P)
{
    constexpr int G = Lay<D>::G, PER = Lay<D>::PER, NG = WARP / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int64_t grp_global = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NG + lane / G;
    const int64_t ngroups = (((int64_t)gridDim.x * blockDim.x) >> 5) * NG;
    const int base = Lay<D>::base(gl);
    for (int64_t g0 = grp_global - lane / G; g0 < P.Q; g0 += ngroups) {
        const int64_t g = g0 + lane / G;
        const bool valid = g < P.Q;
        const int64_t gg = valid ? g : 0;
        const int x = (int)(gg % P.gw), y = (int)(gg / P.gw);
        float v[PER];
#pragma unroll
        for (int i = 0; i < PER; i++) {
            const int e = base + 8 * i;
            const int c = e >> 6, dy = (e >> 3) & 7, dx = e & 7;
            v[i] = __ldg(P.frame + ((int64_t)(y + dy) * P.W + (x + dx)) * P.C + c);
        }
        double acc = __dmul_rn((double)v[0], (double)v[0]);
#pragma unroll
        for (int i = 1; i < PER; i++) acc = __dadd_rn(acc, __dmul_rn((double)v[i], (double)v[i]));
        acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 1));
        acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 2));
        acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 4));
        if (G == 16) acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 8));
        const double nr = __dsqrt_rn(acc);
        const bool ok = nr >= 1e-12;
        if (valid && P.norms && gl == 0) P.norms[g] = ok ? nr : 0.0;
        if (!P.unit) continue;  // norms only (apply_effect)
        float u[PER];
#pragma unroll
        for (int i = 0; i < PER; i++) u[i] = ok ? __double2float_rn(__ddiv_rn((double)v[i], nr)) : 0.0f;
        if (valid) {
            float *ur = P.unit + g * D + base;
#pragma unroll
            for (int i = 0; i < PER; i++) ur[8 * i] = u[i];
        }
        if (P.tc) {
            const float *pr = P.prev_unit + gg * D + base;
            double t = sqdiff(u[0], __ldg(pr));
#pragma unroll
            for (int i = 1; i < PER; i++) t = __dadd_rn(t, sqdiff(u[i], __ldg(pr + 8 * i)));
            t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 1));
            t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 2));
            t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 4));
            if (G == 16) t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 8));
            if (valid && gl == 0) P.tc[g] = __dsqrt_rn(t);
        }
    }
}

// K1 with the frame staged through shared memory: a CTA owns a tile of
// K1_TW x K1_TH grid positions; the (K1_TH + 7) x (K1_TW + 7) x C frame region
// it needs is loaded once, coalesced (float4 when the region is 16-byte
// aligned), then every group of Lay<D>::G lanes builds its position's row from
// shared memory with the same per-lane numpy accumulators as units_warp_kernel.
constexpr int K1_TW = 32, K1_TH = 4;
template <int D>
__global__ void __launch_bounds__(256) units_tile_kernel(UnitsParams P)
{
    constexpr int G = Lay<D>::G, PER = Lay<D>::PER, NGB = 256 / G;  // groups per CTA
    constexpr int C = D / 64;
    constexpr int RW = K1_TW + 7, RH = K1_TH + 7;
    constexpr int RF = RW * C;  // floats per region row
    __shared__ __align__(16) float reg[RH * RF + 4];
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int grp = threadIdx.x / G;
    const int base = Lay<D>::base(gl);
    const int gh = P.H - 7;
    const int tiles_x = (P.gw + K1_TW - 1) / K1_TW, tiles_y = (gh + K1_TH - 1) / K1_TH;
    const int64_t ntiles = (int64_t)tiles_x * tiles_y;
    const int64_t WC = (int64_t)P.W * C;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int x0 = (int)(tile % tiles_x) * K1_TW, y0 = (int)(tile / tiles_x) * K1_TH;
        __syncthreads();
        const int cols = min(RW, P.W - x0) * C, rows = min(RH, P.H - y0);
        const float *src = P.frame + (int64_t)y0 * WC + (int64_t)x0 * C;
        if (((uintptr_t)src & 15) == 0 && (WC & 3) == 0) {
            const int c4 = cols >> 2;
            for (int e = threadIdx.x; e < rows * c4; e += 256) {
                const int r = e / c4, k = e - r * c4;
                const float4 v = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)r * WC) + k);
                float *d = reg + r * RF + 4 * k;
                d[0] = v.x;
                d[1] = v.y;
                d[2] = v.z;
                d[3] = v.w;
            }
            for (int e = threadIdx.x; e < rows * (cols & 3); e += 256) {
                const int r = e / (cols & 3), k = (c4 << 2) + e % (cols & 3);
                reg[r * RF + k] = __ldg(src + (int64_t)r * WC + k);
            }
        } else {
            for (int e = threadIdx.x; e < rows * cols; e += 256) {
                const int r = e / cols, k = e - r * cols;
                reg[r * RF + k] = __ldg(src + (int64_t)r * WC + k);
            }
        }
        __syncthreads();
        for (int pi = grp; pi < K1_TW * K1_TH; pi += NGB) {
            const int tx = pi % K1_TW, ty = pi / K1_TW;
            const int x = x0 + tx, y = y0 + ty;
            const bool valid = x < P.gw && y < gh;
            const int64_t g = valid ? (int64_t)y * P.gw + x : 0;
            float v[PER];
#pragma unroll
            for (int i = 0; i < PER; i++) {
                const int e = base + 8 * i;
                const int c = e >> 6, dy = (e >> 3) & 7, dx = e & 7;
                v[i] = valid ? reg[(ty + dy) * RF + (tx + dx) * C + c] : 0.f;
            }
            double acc = __dmul_rn((double)v[0], (double)v[0]);
#pragma unroll
            for (int i = 1; i < PER; i++) acc = __dadd_rn(acc, __dmul_rn((double)v[i], (double)v[i]));
            acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 1));
            acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 2));
            acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 4));
            if (G == 16) acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 8));
            const double nr = __dsqrt_rn(acc);
            const bool ok = nr >= 1e-12;
            if (valid && P.norms && gl == 0) P.norms[g] = ok ? nr : 0.0;
            if (!P.unit) continue;
            float u[PER];
#pragma unroll
            for (int i = 0; i < PER; i++) u[i] = ok ? __double2float_rn(__ddiv_rn((double)v[i], nr)) : 0.0f;
            if (valid) {
                float *ur = P.unit + g * D + base;
#pragma unroll
                for (int i = 0; i < PER; i++) ur[8 * i] = u[i];
            }
            if (P.tc) {
                const float *pr = P.prev_unit + g * D + base;
                double t = sqdiff(u[0], __ldg(pr));
#pragma unroll
                for (int i = 1; i < PER; i++) t = __dadd_rn(t, sqdiff(u[i], __ldg(pr + 8 * i)));
                t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 1));
                t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 2));
                t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 4));
                if (G == 16) t = __dadd_rn(t, __shfl_xor_sync(FULL, t, 8));
                if (valid && gl == 0) P.tc[g] = __dsqrt_rn(t);
            }
        }
    }
}

// normalize_rows on explicit rows (patches.py:100-115); T = float or double
// input (the reference converts any input to float64 first).
template <class T>
struct RowSqGet {
    const T *r;
    __device__ __forceinline__ double operator()(int64_t i) const
    {
        double v = (double)r[i];
        return __dmul_rn(v, v);
    }
};

template <class T>
__global__ void normalize_rows_kernel(const T *vals, int64_t m, int dim, float *unit, double *norms)
{
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= m) return;
    const T *r = vals + g * dim;
    RowSqGet<T> get{r};
    double nr = __dsqrt_rn(pw_sum(get, 0, dim));
    bool ok = nr >= 1e-12;
    for (int e = 0; e < dim; e++) unit[g * dim + e] = ok ? __double2float_rn(__ddiv_rn((double)r[e], nr)) : 0.0f;
    if (norms) norms[g] = ok ? nr : 0.0;
}

template <class T>
struct SqDiffGetT {
    const T *r, *q;
    __device__ __forceinline__ double operator()(int64_t i) const
    {
        double d = __dsub_rn((double)r[i], (double)q[i]);
        return __dmul_rn(d, d);
    }
};

template <class T>
__global__ void one_to_many_kernel(const T *q, const T *rows, int64_t k, int dim, double *out)
{
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= k) return;
    SqDiffGetT<T> get{rows + g * dim, q};
    out[g] = __dsqrt_rn(pw_sum(get, 0, dim));
}

// extract_patches (patches.py:65-97): raw windows at stride s, plane-major.
__global__ void extract_kernel(const float *frame, int W, int C, int pw, int ph, int stride, int gw, int64_t Q,
                               float *out)
{
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Q) return;
    int x = (int)(g % gw) * stride, y = (int)(g / gw) * stride;
    const int dim = pw * ph * C;
    float *o = out + g * dim;
    int e = 0;
    for (int c = 0; c < C; c++)
        for (int dy = 0; dy < ph; dy++)
            for (int dx = 0; dx < pw; dx++) o[e++] = frame[((int64_t)(y + dy) * W + (x + dx)) * C + c];
}

// ---------------------------------------------------------------------------
// numpy pairwise sum over Q values: leaves (len <= 128) then internal nodes
// level by level (host-built tree, deepest level first).  One block.
struct PwTreeParams {
    const double *vals;
    int nleaves;
    const int64_t *leaf_start;
    const int32_t *leaf_len;
    const int32_t *leaf_node;
    int nlevels;
    const int32_t *level_off;   // nlevels+1 offsets into inner_nodes (deepest first)
    const int32_t *inner_node;  // node ids
    const int32_t *left, *right;
    double *node_val;
    double *out;
};

struct ArrGet {
    const double *a;
    __device__ __forceinline__ double operator()(int64_t i) const { return a[i]; }
};

__global__ void __launch_bounds__(1024) pw_tree_kernel(PwTreeParams P)
{
    for (int i = threadIdx.x; i < P.nleaves; i += blockDim.x) {
        ArrGet g{P.vals};
        P.node_val[P.leaf_node[i]] = pw_block(g, P.leaf_start[i], P.leaf_len[i]);
    }
    __syncthreads();
    for (int l = 0; l < P.nlevels; l++) {
        for (int i = P.level_off[l] + threadIdx.x; i < P.level_off[l + 1]; i += blockDim.x) {
            int nd = P.inner_node[i];
            P.node_val[nd] = __dadd_rn(P.node_val[P.left[nd]], P.node_val[P.right[nd]]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *P.out = P.node_val[0];
}

// ---------------------------------------------------------------------------
// K2: riann_query, one warp per query, persistent grid.
//
// Per query (search.py:83-151):
//   d_prev exact; first ring = window of the previous match's sorted row
//   (17-ary warp binary search, search.py:77-79) enumerated from the u16/i32
//   index table and radix-sorted ascending (np.sort, search.py:116) into the
//   warp's candidate list S;
//   rings: anchor = k-th element of S minus used anchors (numpy RNG), exact
//   d_a, and membership of every j in S by one lookup in the index-ordered
//   distance matrix dmat[a][j] (== the sorted table's value, so lv <= v <= hv
//   is exactly the searchsorted window test) -- |S| reads instead of
//   enumerating the anchor's window (~30% of n at config 3);
//   final scan of S u {prev}: fp16-reference screening with a rigorous error
//   bound, exact FP64 (numpy order) only for the candidates that can still be
//   the first minimum.
struct QueryParams {
    const float *refs;
    const __half *refs16;   // fp16 copy of refs (screening)
    const float *err16;     // per row: upper bound of ||r - fp16(r)||
    const float *sdist;     // sorted distance rows (n, n)
    const void *sidx;       // sorted index rows (n, n): uint16 or int32
    const float *dmat;      // index-ordered distance rows (n, n)
    int64_t n;
    int dim;
    const float *units;   // (Q, dim)
    const int32_t *prev;  // (Q)
    int64_t Q;
    // RNG key: frame mode when key_words == null -> words(seed) ++ [x, y, t]
    uint32_t seed_lo, seed_hi;
    int seed_nw;
    int gw, gy0;
    uint32_t t;
    const uint32_t *key_words;
    const int64_t *key_off;
    int L;
    double alpha;
    int max_rings;
    int32_t *out_idx;
    double *out_dist;
    int32_t *out_rings;   // optional per-query outputs (batch API)
    int64_t *out_evals;
    int64_t *out_cand;
    int64_t *out_first;
    int32_t *scanned;     // optional, stride n+1
    int64_t *scanned_len;
    unsigned long long *stats;  // [6]: rings, evals, cand_final, first_ring, ring_tests, exact_evals
    int *err;
    uint32_t *overflow;   // per warp: 2n entries (list spill)
    int passes;           // radix passes for indices < n
    const int32_t *qlist; // optional: process only these queries (count *n_qlist)
    const int32_t *n_qlist;
    int64_t qlist_cap;    // > 0: at most this many entries of qlist
    // row-sharded tables (config 4: n x n tables larger than one GPU): row a of
    // each table lives in shard s = a / shard_rows at sh_*[s] + (a - s * shard_rows) * n,
    // on this GPU or a peer (NVLink peer pointers); nshards == 0: sdist/sidx/dmat above
    const float *const *sh_sdist;
    const void *const *sh_sidx;
    const float *const *sh_dmat;
    int64_t shard_rows;
    int nshards;
    // n <= 65,536 without shards: rank rows pos[a][j] (u16) replace the
    // index-ordered distance rows; membership of j in a's ring is then
    // lo_a <= pos[a][j] < hi_a with [lo_a, hi_a) the window on a's sorted row
    const uint16_t *pos;
};

__device__ __forceinline__ int64_t shard_of(const QueryParams &P, int64_t a, int64_t &r)
{
    const int64_t s = a / P.shard_rows;
    r = a - s * P.shard_rows;
    return s;
}
__device__ __forceinline__ const float *sdist_row(const QueryParams &P, int64_t a)
{
    if (P.nshards == 0) return P.sdist + a * P.n;
    int64_t r;
    const int64_t s = shard_of(P, a, r);
    return P.sh_sdist[s] + r * P.n;
}
__device__ __forceinline__ const float *dmat_row(const QueryParams &P, int64_t a)
{
    if (P.nshards == 0) return P.dmat + a * P.n;
    int64_t r;
    const int64_t s = shard_of(P, a, r);
    return P.sh_dmat[s] + r * P.n;
}
// sorted index row a as (base, element offset) for idx_at<IdxT>
__device__ __forceinline__ const void *sidx_base(const QueryParams &P, int64_t a, int64_t &off)
{
    if (P.nshards == 0) {
        off = a * P.n;
        return P.sidx;
    }
    int64_t r;
    const int64_t s = shard_of(P, a, r);
    off = r * P.n;
    return P.sh_sidx[s];
}

enum { ERR_PREV_RANGE = 3, ERR_USED_OVERFLOW = 5, ERR_INTERNAL = 9 };

// Bounds-checked builds (-DRIANN_BOUNDS, tests/test_gpu_bounds.py): index and
// capacity invariants of the frame kernels checked on the device; the first
// failing site is reported by riann_process_frame / riann_sync.  Stands in for
// compute-sanitizer, which the GPU pool does not allow.
#ifdef RIANN_BOUNDS
__device__ unsigned rb_bounds_site;
#define RB_CHECK(cond, site)                                                  \
    do {                                                                      \
        if (!(cond)) atomicCAS(&rb::rb_bounds_site, 0u, (unsigned)(site));    \
    } while (0)
#else
#define RB_CHECK(cond, site) \
    do {                     \
    } while (0)
#endif
constexpr int LIST_BYTES = 4096;                      // per list, per warp, in shared memory
#ifndef RIANN_K2_UMAX
#define RIANN_K2_UMAX 128
#endif
constexpr int UMAX = RIANN_K2_UMAX;                             // used anchors tracked inside S (K2), in the scratch words
constexpr int K2_SMEM_BYTES = 2 * LIST_BYTES + 1024;  // two lists + 256-word scratch

// Candidate list: the first LIST_BYTES/sizeof(T) entries in shared memory,
// the rest spilled to a per-warp global region.
template <class T>
struct QList {
    static constexpr int CAP = LIST_BYTES / (int)sizeof(T);
    T *sm;
    T *gl;
    __device__ __forceinline__ uint32_t get(int i) const { return i < CAP ? (uint32_t)sm[i] : (uint32_t)gl[i - CAP]; }
    __device__ __forceinline__ void put(int i, uint32_t v) const
    {
        if (i < CAP) sm[i] = (T)v;
        else gl[i - CAP] = (T)v;
    }
};

// L2 eviction-priority policies (createpolicy): the sorted tables and the
// index-ordered distance matrix are streamed (evict_first, no L1 allocate);
// the reference rows (f32 48 MB, fp16 24 MB at n=65,536) should stay L2-resident.
__device__ __forceinline__ uint64_t pol_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float ld_stream(const float *a, uint64_t pol)
{
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_keep16(const uint4 *a, uint64_t pol)
{
    uint4 v;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(a), "l"(pol));
    return v;
}
// one 32-byte sector per lane (sm_100: 256-bit global loads)
__device__ __forceinline__ void ld_keep32(const void *a, uint64_t pol, uint4 &lo, uint4 &hi)
{
    asm("ld.global.nc.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
        : "l"(a), "l"(pol));
}
// streamed once (candidate lists): no L1 allocation, evict first from L2
__device__ __forceinline__ uint4 ld_once16(const uint4 *a, uint64_t pol)
{
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_keep(const float *a, uint64_t pol)
{
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}

// search.py:77-79: lo = first v >= d-eps, hi = first v > d+eps (f32 values
// compared as f64).  Lanes 0-15 search lo, lanes 16-31 search hi, 17-ary.
__device__ __forceinline__ void ring_window(const float *__restrict__ row, int64_t n, double lv, double hv,
                                            int lane, int64_t &lo, int64_t &hi)
{
    const int h = lane >> 4, hl = lane & 15;
    const double thr = h ? hv : lv;
    int64_t b = 0, e = n;
    for (;;) {
        int64_t s = e - b;
        if (!__any_sync(FULL, s > 16)) break;
        int64_t p = b + ((int64_t)(hl + 1) * s) / 17;
        bool pr = false;
        if (s > 16) {
            double v = (double)__ldg(row + p);
            pr = h ? (v <= thr) : (v < thr);
        }
        unsigned ball = __ballot_sync(FULL, pr);
        int c = __popc((ball >> (h * 16)) & 0xffffu);
        int src_lo = h * 16 + (c > 0 ? c - 1 : 0);
        int src_hi = h * 16 + (c < 16 ? c : 15);
        int64_t p_lo = __shfl_sync(FULL, p, src_lo);
        int64_t p_hi = __shfl_sync(FULL, p, src_hi);
        if (s > 16) {
            if (c > 0) b = p_lo + 1;
            if (c < 16) e = p_hi;
        }
    }
    int64_t p = b + hl;
    bool pr = false;
    if (p < e) {
        double v = (double)__ldg(row + p);
        pr = h ? (v <= thr) : (v < thr);
    }
    unsigned ball = __ballot_sync(FULL, pr);
    int64_t res = b + __popc((ball >> (h * 16)) & 0xffffu);
    lo = __shfl_sync(FULL, res, 0);
    hi = __shfl_sync(FULL, res, 16);
}

// Stable LSD radix sort (8-bit digits) of list a[0..cnt) using b as buffer;
// the sorted result ends in `a` (the lists are swapped per pass).
template <class T>
__device__ __forceinline__ void warp_radix_sort(QList<T> &a, QList<T> &b, int cnt, int passes, uint32_t *hist, int lane)
{
    for (int ps = 0; ps < passes; ps++) {
        const int sh = 8 * ps;
        for (int i = lane; i < 256; i += 32) hist[i] = 0u;
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) atomicAdd(&hist[(a.get(i) >> sh) & 255u], 1u);
        __syncwarp();
        uint32_t v[8], s = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = hist[lane * 8 + k];
            s += v[k];
        }
        uint32_t run = (uint32_t)warp_incl_scan((int)s, lane) - s;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            hist[lane * 8 + k] = run;
            run += v[k];
        }
        __syncwarp();
        for (int base = 0; base < cnt; base += 32) {
            const int i = base + lane;
            const bool valid = i < cnt;
            const uint32_t key = valid ? a.get(i) : 0u;
            const uint32_t dg = valid ? ((key >> sh) & 255u) : 256u;
            const unsigned m = __match_any_sync(FULL, dg);
            const int rank = __popc(m & lanemask_lt());
            const uint32_t bse = valid ? hist[dg] : 0u;
            __syncwarp();
            if (valid) b.put((int)bse + rank, key);
            if (valid && rank == 0) hist[dg] = bse + (uint32_t)__popc(m);
            __syncwarp();
        }
        QList<T> t = a;
        a = b;
        b = t;
        __threadfence_block();
        __syncwarp();
    }
}

// first position in ascending list a[0..cnt) with value >= x (one lane)
template <class T>
__device__ __forceinline__ int list_lower_bound(const QList<T> &a, int cnt, uint32_t x)
{
    int lo = 0, hi = cnt;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a.get(mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// fp16 screening layout (D in {64, 192}): 8 lanes per candidate, lane l8
// owns elements m*64 + l8*8 + e (m < D/64, e < 8): one 16-byte load per m.
template <int D>
struct Scr {
    static constexpr bool on = (D == 64 || D == 192);
    static constexpr int NV = D / 64;
    static constexpr int PER = D / 8;
};

template <int D>
__device__ __forceinline__ float approx_sq(const __half *__restrict__ row16, const float (&q)[Scr<D>::PER], int l8,
                                           uint64_t pol)
{
    const uint4 *p = reinterpret_cast<const uint4 *>(row16) + l8;
    float acc = 0.f;
#pragma unroll
    for (int m = 0; m < Scr<D>::NV; m++) {
        uint4 v = ld_keep16(p + m * 8, pol);
        const __half2 *h2 = reinterpret_cast<const __half2 *>(&v);
#pragma unroll
        for (int e = 0; e < 4; e++) {
            float2 f = __half22float2(h2[e]);
            float d0 = __fsub_rn(f.x, q[m * 8 + 2 * e]);
            float d1 = __fsub_rn(f.y, q[m * 8 + 2 * e + 1]);
            acc = __fmaf_rn(d0, d0, acc);
            acc = __fmaf_rn(d1, d1, acc);
        }
    }
    acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, 4));
    return acc;
}

// Exact distance: warp-cooperative for numpy-mappable dims, else per lane.
template <int D>
__device__ __forceinline__ double exact_dist(const float *__restrict__ refs, int r, const float *__restrict__ q,
                                             int dim, int gl)
{
    if constexpr (D > 0) {
        const float *row = refs + (int64_t)r * D;
        const int base = Lay<D>::base(gl);
        const float *pr = row + base;
        const float *pq = q + base;
        double acc = sqdiff(__ldg(pr), __ldg(pq));
#pragma unroll
        for (int i = 1; i < Lay<D>::PER; i++) acc = __dadd_rn(acc, sqdiff(__ldg(pr + 8 * i), __ldg(pq + 8 * i)));
        acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 1));
        acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 2));
        acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 4));
        if (Lay<D>::G == 16) acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, 8));
        return __dsqrt_rn(acc);
    } else {
        return dist_thread(refs + (int64_t)r * dim, q, dim);
    }
}

// One exact distance that every lane needs (prev / anchors).
template <int D>
__device__ __forceinline__ double exact_dist_all(const float *refs, int r, const float *q, int dim, int lane)
{
    if constexpr (D > 0) return exact_dist<D>(refs, r, q, dim, lane % Lay<D>::G);
    else {
        double v = 0.0;
        if (lane == 0) v = dist_thread(refs + (int64_t)r * dim, q, dim);
        return __shfl_sync(FULL, v, 0);
    }
}

template <class IdxT>
__device__ __forceinline__ uint32_t idx_at(const void *sidx, int64_t off)
{
    return (uint32_t)__ldg(reinterpret_cast<const IdxT *>(sidx) + off);
}

// D > 0: compile-time dim; D == 0: runtime dim (generic, exact only).
// IdxT: sorted index table element; LT: candidate-list element (u16 if n <= 65536).
template <int D, class IdxT, class LT>
__global__ void __launch_bounds__(256, 3) query_kernel(QueryParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool FAST = D > 0;
    constexpr bool SCREEN = Scr<D>::on;
    constexpr int GX = FAST ? Lay<(FAST ? D : 64)>::G : 1;  // lanes per exact distance
    constexpr int NGX = WARP / GX;
    constexpr int SP = Scr<(SCREEN ? D : 64)>::PER;
    constexpr int SURV_CAP = 128;  // survivor slots (index + lower bound) in the scratch area

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    unsigned char *ws = smem_raw + (size_t)wib * K2_SMEM_BYTES;
    uint32_t *hist = reinterpret_cast<uint32_t *>(ws + 2 * LIST_BYTES);
    const int64_t gwarp = (int64_t)blockIdx.x * wpb + wib;
    const int64_t nwarps = (int64_t)gridDim.x * wpb;
    const int64_t n = P.n;
    const int dim = FAST ? D : P.dim;
    LT *spill = reinterpret_cast<LT *>(P.overflow) + gwarp * 2 * n;
    const uint64_t pol_stream = pol_evict_first();
    const uint64_t pol_keep = pol_evict_last();

    unsigned long long acc_r = 0, acc_e = 0, acc_c = 0, acc_f = 0, acc_t = 0, acc_x = 0;
    int64_t qn = P.qlist ? (int64_t)*P.n_qlist : P.Q;
    if (P.qlist && P.qlist_cap > 0 && qn > P.qlist_cap) qn = P.qlist_cap;

    for (int64_t gi = gwarp; gi < qn; gi += nwarps) {
        const int64_t g = P.qlist ? (int64_t)P.qlist[gi] : gi;
        QList<LT> A{reinterpret_cast<LT *>(ws), spill};
        QList<LT> B{reinterpret_cast<LT *>(ws + LIST_BYTES), spill + n};
        const float *q = P.units + g * dim;
        const int p = P.prev[g];
        if (p < 0 || p >= n) {
            if (lane == 0) atomicExch(P.err, ERR_PREV_RANGE);
            continue;
        }
        // ---- first ring around the previous match (search.py:114-117)
        const double d = exact_dist_all<D>(P.refs, p, q, dim, lane);
        long long exact_cnt = 1;
        int64_t lo, hi;
        ring_window(sdist_row(P, p), n, __dsub_rn(d, __dmul_rn(P.alpha, d)),
                    __dadd_rn(d, __dmul_rn(P.alpha, d)), lane, lo, hi);
        int cS = (int)(hi - lo);
        RB_CHECK(lo >= 0 && lo <= hi && hi <= n, 60);
        const int first = cS;
        bool p_in = false;
        int64_t prow_off;
        const void *prow = sidx_base(P, p, prow_off);
        for (int64_t k = lo + lane; k < hi; k += 32) {
            const uint32_t j = idx_at<IdxT>(prow, prow_off + k);
            A.put((int)(k - lo), j);
            p_in |= (j == (uint32_t)p);
        }
        p_in = __any_sync(FULL, p_in);
        __threadfence_block();
        __syncwarp();
        int rings = 1;
        long long tests = 0;
        if (cS >= P.L && P.max_rings > 1) {
            warp_radix_sort(A, B, cS, P.passes, hist, lane);
            // used anchors still inside S (search.py:120-122) with their positions
            // in S: (uv[i], up[i]) for i < nu in the scratch words (free after the
            // sort), up to UMAX of them
            uint32_t *uv = hist, *up = hist + UMAX;
            int nu = 0;
            if (p_in) {
                nu = 1;
                if (lane == 0) {
                    uv[0] = (uint32_t)p;
                    up[0] = (uint32_t)list_lower_bound(A, cS, (uint32_t)p);
                }
            }
            __syncwarp();
            bool have_rng = false;
            Pcg64 rng;
            while (cS >= P.L && rings < P.max_rings) {
                const int na = cS - nu;
                if (na <= 0) break;
                if (!have_rng) {
                    if (P.key_words) {
                        const uint32_t *kw = P.key_words + P.key_off[g];
                        const int nk = (int)(P.key_off[g + 1] - P.key_off[g]);
                        struct KW {
                            const uint32_t *w;
                            __device__ uint32_t operator()(int i) const { return __ldg(w + i); }
                        } kf{kw};
                        pcg_seed(rng, kf, nk);
                    } else {
                        struct FW {
                            uint32_t s0, s1, x, y, t;
                            int snw;
                            __device__ uint32_t operator()(int i) const
                            {
                                if (i < snw) return i == 0 ? s0 : s1;
                                i -= snw;
                                return i == 0 ? x : (i == 1 ? y : t);
                            }
                        } fw{P.seed_lo, P.seed_hi, (uint32_t)(g % P.gw), (uint32_t)(P.gy0 + g / P.gw), P.t,
                             P.seed_nw};
                        pcg_seed(rng, fw, P.seed_nw + 3);
                    }
                    have_rng = true;
                }
                // search.py:129: anchor = avail[integers(|avail|)], avail = S \ used, ascending
                const int k = (int)pcg_integers(rng, (uint64_t)na);
                int pos = k;
                for (int it = 0; it <= nu; it++) {
                    int c = 0;
                    for (int b = 0; b < nu; b += 32)
                        c += __popc(__ballot_sync(FULL, b + lane < nu && (int)up[b + lane] <= pos));
                    if (k + c == pos) break;
                    pos = k + c;
                }
                RB_CHECK(pos >= 0 && pos < cS, 61);
                const int a = (int)A.get(pos);
                RB_CHECK(a >= 0 && a < n, 62);
                if (nu >= UMAX) {
                    if (lane == 0) atomicExch(P.err, ERR_USED_OVERFLOW);
                    break;
                }
                __syncwarp();
                if (lane == 0) {
                    uv[nu] = (uint32_t)a;
                    up[nu] = (uint32_t)pos;
                }
                __syncwarp();
                nu++;
                // search.py:131-135: ring around the anchor, intersect with S by
                // lookups in the anchor's index-ordered distance row
                const double da = exact_dist_all<D>(P.refs, a, q, dim, lane);
                exact_cnt++;
                const double lv = __dsub_rn(da, __dmul_rn(P.alpha, da));
                const double hv = __dadd_rn(da, __dmul_rn(P.alpha, da));
                // ring membership: rank in a's window (rank rows) or the value in
                // a's index-ordered distance row -- the same searchsorted test
                const bool use_pos = P.pos != nullptr;
                const float *drow = use_pos ? nullptr : dmat_row(P, a);
                const uint16_t *prank = use_pos ? P.pos + (int64_t)a * n : nullptr;
                uint32_t a_lo = 0, a_w = 0;
                if (use_pos) {
                    int64_t wlo, whi;
                    ring_window(sdist_row(P, a), n, lv, hv, lane, wlo, whi);
                    a_lo = (uint32_t)wlo;
                    a_w = (uint32_t)(whi - wlo);
                }
                auto member = [&](uint32_t jj, float dvf) {
                    if (use_pos) return (uint32_t)__ldg(prank + jj) - a_lo < a_w;
                    const double dv = (double)dvf;
                    return lv <= dv && dv <= hv;
                };
                int nh = 0;
                for (int base = 0; base < cS; base += 256) {
                    uint32_t j[8];
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int i = base + u * 32 + lane;
                        j[u] = i < cS ? A.get(i) : 0xffffffffu;
                    }
                    if (!use_pos) {
#pragma unroll
                        for (int u = 0; u < 8; u++) v[u] = j[u] != 0xffffffffu ? ld_stream(drow + j[u], pol_stream) : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const bool keep = j[u] != 0xffffffffu && member(j[u], v[u]);
                        const unsigned ball = __ballot_sync(FULL, keep);
                        if (keep) B.put(nh + __popc(ball & lanemask_lt()), j[u]);
                        nh += __popc(ball);
                    }
                }
                tests += cS;
                rings++;
                if (nh == 0) break;  // search.py:136-137 rollback: keep S
                __threadfence_block();
                __syncwarp();
                {
                    QList<LT> t = A;
                    A = B;
                    B = t;
                }
                cS = nh;
                // used anchors still in S (stable compaction), with their new positions
                int nkeep = 0;
                bool pin = false;
                for (int b = 0; b < nu; b += 32) {
                    const int i = b + lane;
                    const uint32_t vi = i < nu ? uv[i] : 0u;
                    bool keep = false;
                    if (i < nu) keep = member(vi, use_pos ? 0.f : ld_stream(drow + vi, pol_stream));
                    const unsigned kb = __ballot_sync(FULL, keep);
                    const int np = keep ? list_lower_bound(A, cS, vi) : 0;
                    __syncwarp();
                    if (keep) {
                        const int o = nkeep + __popc(kb & lanemask_lt());
                        uv[o] = vi;
                        up[o] = (uint32_t)np;
                        pin |= vi == (uint32_t)p;
                    }
                    nkeep += __popc(kb);
                    __syncwarp();
                }
                nu = nkeep;
                p_in = __any_sync(FULL, pin);
            }
        } else if (cS > 0 && P.scanned) {
            // no rings drawn: order is irrelevant to the argmin, but the scanned
            // output (batch API) is ascending
            warp_radix_sort(A, B, cS, P.passes, hist, lane);
        }

        // ---- final scan of S u {prev}, first minimum (search.py:140-143)
        double bd = d;
        int bi = p;
        if constexpr (SCREEN) {
            // fp16 screening with a running upper bound; candidates whose lower
            // bound can still reach the minimum go to the survivor slots and get
            // the exact FP64 distance.
            float qs[SP];
            const int grp8 = lane >> 3, l8 = lane & 7;
#pragma unroll
            for (int m = 0; m < Scr<D>::NV; m++)
#pragma unroll
                for (int e = 0; e < 8; e++) qs[m * 8 + e] = __ldg(q + m * 64 + l8 * 8 + e);
            uint32_t *sv_j = hist;                                       // survivor index
            float *sv_lb = reinterpret_cast<float *>(hist + SURV_CAP);   // survivor lower bound
            float ub_min = __double2float_ru(d);  // the previous match's exact distance
            int nsv = 0;
            auto flush = [&](bool all) {
                // exact re-check of the survivors that can still win
                __syncwarp();
                int m = 0;
                for (int b0 = 0; b0 < nsv; b0 += 32) {
                    const int i = b0 + lane;
                    const bool ok = i < nsv && sv_lb[i] <= ub_min;
                    const uint32_t jj = i < nsv ? sv_j[i] : 0u;
                    const unsigned ball = __ballot_sync(FULL, ok);
                    __syncwarp();
                    if (ok) sv_j[m + __popc(ball & lanemask_lt())] = jj;
                    m += __popc(ball);
                    __syncwarp();
                }
                for (int s0 = 0; s0 < m; s0 += NGX) {
                    const int si = s0 + lane / GX;
                    const bool ok = si < m;
                    const int jj = (int)sv_j[ok ? si : 0];
                    const double dj = exact_dist<D>(P.refs, jj, q, dim, lane % GX);
                    if (ok) argmin_merge(bd, bi, dj, jj);
                }
                exact_cnt += m;
                nsv = 0;
                __syncwarp();
                (void)all;
            };
            for (int e0 = 0; e0 < cS; e0 += 4) {
                const int e = e0 + grp8;
                const bool valid = e < cS;
                const uint32_t j = A.get(valid ? e : 0);
                const float s = approx_sq<D>(P.refs16 + (int64_t)j * D, qs, l8, pol_keep);
                // s: fp32 sum with relative error <= 29u; the fp16 row differs from
                // the reference row by at most err16[j] in L2 norm
                const float e16 = ld_keep(P.err16 + j, pol_keep);
                const float ub = __fadd_ru(__fsqrt_ru(__fmul_ru(s, 1.00001f)), __fadd_ru(e16, 1e-12f));
                const float lb = __fsub_rd(__fsqrt_rd(__fmul_rd(s, 0.99999f)), __fadd_ru(e16, 1e-12f));
                float m = valid ? ub : ub_min;
                m = fminf(m, __shfl_xor_sync(FULL, m, 8));
                m = fminf(m, __shfl_xor_sync(FULL, m, 16));
                ub_min = fminf(ub_min, m);
                const bool surv = valid && l8 == 0 && lb <= ub_min;
                const unsigned ball = __ballot_sync(FULL, surv);
                const int add = __popc(ball);
                if (nsv + add > SURV_CAP) flush(false);
                if (surv) {
                    const int slot = nsv + __popc(ball & lanemask_lt());
                    sv_j[slot] = j;
                    sv_lb[slot] = lb;
                }
                nsv += add;
            }
            flush(true);
        } else {
            for (int e0 = 0; e0 < cS; e0 += NGX) {
                const int e = e0 + lane / GX;
                const bool valid = e < cS;
                const int j = (int)A.get(valid ? e : 0);
                if constexpr (FAST) {
                    const double dj = exact_dist<D>(P.refs, j, q, dim, lane % GX);
                    if (valid) argmin_merge(bd, bi, dj, j);
                } else {
                    if (valid) argmin_merge(bd, bi, dist_thread(P.refs + (int64_t)j * dim, q, dim), j);
                }
            }
            exact_cnt += cS;
        }
        warp_argmin(bd, bi);
        const int nscan = cS + (p_in ? 0 : 1);
        const long long evals = rings + nscan;
        if (P.scanned) {
            int32_t *so = P.scanned + g * (n + 1);
            int below = 0;
            for (int base = 0; base < cS; base += 32) {
                const int e = base + lane;
                uint32_t j = e < cS ? A.get(e) : 0xffffffffu;
                below += __popc(__ballot_sync(FULL, e < cS && j < (uint32_t)p));
                if (e < cS) so[e + ((!p_in && j > (uint32_t)p) ? 1 : 0)] = (int32_t)j;
            }
            if (!p_in && lane == 0) so[below] = p;
        }
        if (lane == 0) {
            P.out_idx[g] = bi;
            P.out_dist[g] = bd;
            if (P.out_rings) P.out_rings[g] = rings;
            if (P.out_evals) P.out_evals[g] = evals;
            if (P.out_cand) P.out_cand[g] = cS;
            if (P.out_first) P.out_first[g] = first;
            if (P.scanned_len) P.scanned_len[g] = nscan;
        }
        acc_r += rings;
        acc_e += evals;
        acc_c += cS;
        acc_f += first;
        acc_t += tests;
        acc_x += exact_cnt;
        __syncwarp();
    }
    if (lane == 0 && P.stats) {
        atomicAdd(P.stats + 0, acc_r);
        atomicAdd(P.stats + 1, acc_e);
        atomicAdd(P.stats + 2, acc_c);
        atomicAdd(P.stats + 3, acc_f);
        atomicAdd(P.stats + 4, acc_t);
        atomicAdd(P.stats + 5, acc_x);
        if (P.qlist && gwarp == 0) atomicAdd(P.stats + 6, (unsigned long long)qn);
    }
}

// one-warp ring window (ring_candidates API)
__global__ void ring_window_kernel(const float *row, int64_t n, double lv, double hv, int64_t *out)
{
    int64_t lo, hi;
    ring_window(row, n, lv, hv, threadIdx.x & 31, lo, hi);
    if (threadIdx.x == 0) {
        out[0] = lo;
        out[1] = hi;
    }
}

// ---------------------------------------------------------------------------
// Model preparation: fp16 screening copy of the references with a rigorous
// per-row bound err16[j] >= ||r_j - fp16(r_j)|| (rounded up).
__global__ void refs16_kernel(const float *refs, int64_t n, int dim, __half *r16, float *err)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double acc = 0.0;
    for (int e = 0; e < dim; e++) {
        float v = refs[j * dim + e];
        __half h = __float2half_rn(v);
        r16[j * dim + e] = h;
        double dlt = (double)v - (double)__half2float(h);  // exact (both f32-representable, close)
        acc = __fma_ru(dlt, dlt, acc);
    }
    err[j] = __double2float_ru(__dsqrt_ru(acc) * (1.0 + 1e-12));
}

// dmat[a][sidx[a][k]] = sdist[a][k]: index-ordered copy of the sorted rows.
template <class IdxT>
__global__ void dmat_scatter_kernel(const float *sdist, const IdxT *sidx, int64_t n, int64_t rows, float *dmat)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * n) return;
    int64_t a = i / n;
    dmat[a * n + (int64_t)sidx[i]] = sdist[i];
}

__global__ void narrow_u16_kernel(const int32_t *src, uint16_t *dst, int64_t cnt)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) dst[i] = (uint16_t)src[i];
}

__global__ void widen_u16_kernel(const uint16_t *src, int32_t *dst, int64_t cnt)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) dst[i] = (int32_t)src[i];
}

// ---------------------------------------------------------------------------
// K3: exact f32(f64 distance) keys for rows [r0, r0+rows) x all n columns.
// One warp per row; fast dims use the group layout (NG pairs per step).
template <int D>
__global__ void __launch_bounds__(256) table_keys_kernel(const float *refs, int64_t n, int dim, int64_t r0,
                                                         int64_t rows, uint32_t *keys, int32_t *vals)
{
    constexpr bool FAST = D > 0;
    constexpr int DD = FAST ? D : 64;
    constexpr int G = FAST ? Lay<DD>::G : 1;
    constexpr int NG = WARP / G;
    constexpr int PER = FAST ? Lay<DD>::PER : 1;
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int gl = lane % G, grp = lane / G;
    for (int64_t r = wid; r < rows; r += nwarps) {
        const int64_t i = r0 + r;
        const float *qi = refs + i * dim;
        uint32_t *kr = keys + r * n;
        int32_t *vr = vals + r * n;
        if constexpr (FAST) {
            float qv[PER];
            const int base = Lay<DD>::base(gl);
#pragma unroll
            for (int k = 0; k < PER; k++) qv[k] = __ldg(qi + base + 8 * k);
            for (int64_t j0 = 0; j0 < n; j0 += NG) {
                const int64_t j = j0 + grp;
                const bool valid = j < n;
                const double dj = group_dist<DD>(refs + (valid ? j : 0) * D, qv, gl);
                if (valid && gl == 0) {
                    kr[j] = __float_as_uint(__double2float_rn(dj));
                    vr[j] = (int32_t)j;
                }
            }
        } else {
            for (int64_t j = lane; j < n; j += 32) {
                const double dj = dist_thread(refs + j * dim, qi, dim);
                kr[j] = __float_as_uint(__double2float_rn(dj));
                vr[j] = (int32_t)j;
            }
        }
    }
}

// model.py:181-186: exact duplicates of i sort ahead of it; rotate the
// self entry to position 0 (all entries before it have distance 0).
__global__ void self_first_kernel(const uint32_t *keys, int32_t *vals, int64_t n, int64_t r0, int64_t rows)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int32_t i = (int32_t)(r0 + r);
    int32_t *vr = vals + r * n;
    const uint32_t *kr = keys + r * n;
    if (vr[0] == i) return;
    int64_t pos = 1;
    while (pos < n && vr[pos] != i && kr[pos] == 0u) pos++;
    if (pos >= n || vr[pos] != i) return;  // cannot happen: self distance is exactly 0
    for (int64_t k = pos; k > 0; k--) vr[k] = vr[k - 1];
    vr[0] = i;
}

// ---------------------------------------------------------------------------
// K4 (round-1 form): exact nearest reference by full FP64 scan, warp per
// query, ties to the lowest index (evaluation.py:24-33).
template <int D>
__global__ void __launch_bounds__(256) exact_nn_kernel(const float *refs, int64_t n, int dim, const float *qs,
                                                       int64_t m, int32_t *out_idx, double *out_dist)
{
    constexpr bool FAST = D > 0;
    constexpr int DD = FAST ? D : 64;
    constexpr int G = FAST ? Lay<DD>::G : 1;
    constexpr int NG = WARP / G;
    constexpr int PER = FAST ? Lay<DD>::PER : 1;
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int gl = lane % G, grp = lane / G;
    for (int64_t g = wid; g < m; g += nwarps) {
        const float *q = qs + g * dim;
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bi = 0x7fffffff;
        if constexpr (FAST) {
            float qv[PER];
            const int base = Lay<DD>::base(gl);
#pragma unroll
            for (int k = 0; k < PER; k++) qv[k] = __ldg(q + base + 8 * k);
            for (int64_t j0 = 0; j0 < n; j0 += NG) {
                const int64_t j = j0 + grp;
                const bool valid = j < n;
                const double dj = group_dist<DD>(refs + (valid ? j : 0) * D, qv, gl);
                if (valid) argmin_merge(bd, bi, dj, (int)j);
            }
        } else {
            for (int64_t j = lane; j < n; j += 32) argmin_merge(bd, bi, dist_thread(refs + j * dim, q, dim), (int)j);
        }
        warp_argmin(bd, bi);
        if (lane == 0) {
            out_idx[g] = bi;
            out_dist[g] = bd;
        }
    }
}

}  // namespace rb

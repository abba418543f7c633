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

#include "riann_device.cuh"

namespace rb {

constexpr int HIT_CAP = 1024;  // per-warp shared hit list (u32 entries); overflow spills to global

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
struct QueryParams {
    const float *refs;
    const float *sdist;
    const int32_t *sidx;
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
    unsigned long long *stats;  // [4]: rings, evals, cand_final, first_ring
    int *err;
    int32_t *overflow;    // per warp: n entries
    int nw;               // bitmap words per warp (multiple of 32)
};

enum { ERR_PREV_RANGE = 3, ERR_USED_OVERFLOW = 5 };

struct WarpList {
    uint32_t *sm;
    int32_t *gl;
    __device__ __forceinline__ void put(int pos, int v) const
    {
        if (pos < HIT_CAP) sm[pos] = (uint32_t)v;
        else gl[pos - HIT_CAP] = v;
    }
    __device__ __forceinline__ int get(int pos) const
    {
        return pos < HIT_CAP ? (int)sm[pos] : gl[pos - HIT_CAP];
    }
};

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

// k-th (0-based) set bit of the warp's bitmap (ascending order).
__device__ __forceinline__ int rank_select(const uint32_t *bm, int nw, int k, int lane)
{
    const int CH = nw >> 5;
    const uint32_t *mine = bm + lane * CH;
    int c = 0;
    for (int w = 0; w < CH; w++) c += __popc(mine[w]);
    int inc = warp_incl_scan(c, lane);
    unsigned ball = __ballot_sync(FULL, k < inc);
    int L = __ffs(ball) - 1;
    int kk = k - __shfl_sync(FULL, inc - c, L);
    const uint32_t *ch = bm + L * CH;
    for (int base = 0; base < CH; base += 32) {
        uint32_t w = (base + lane < CH) ? ch[base + lane] : 0u;
        int pc = __popc(w);
        int inc2 = warp_incl_scan(pc, lane);
        int tot = __shfl_sync(FULL, inc2, 31);
        if (kk < tot) {
            unsigned b2 = __ballot_sync(FULL, kk < inc2);
            int L2 = __ffs(b2) - 1;
            int k2 = kk - __shfl_sync(FULL, inc2 - pc, L2);
            uint32_t word = __shfl_sync(FULL, w, L2);
            for (int i = 0; i < k2; i++) word &= word - 1;
            return (L * CH + base + L2) * 32 + (__ffs(word) - 1);
        }
        kk -= tot;
    }
    return -1;  // unreachable when k < popcount
}

__device__ __forceinline__ bool bit_test(const uint32_t *bm, int j)
{
    return (bm[j >> 5] >> (j & 31)) & 1u;
}

// D > 0: compile-time dim with the warp-cooperative exact distance;
// D == 0: runtime dim, one lane per distance.
template <int D>
__global__ void __launch_bounds__(256) query_kernel(QueryParams P)
{
    extern __shared__ uint32_t smem[];
    constexpr bool FAST = D > 0;
    constexpr int G = FAST ? Lay<(FAST ? D : 64)>::G : 1;
    constexpr int NG = WARP / G;
    constexpr int PER = FAST ? Lay<(FAST ? D : 64)>::PER : 1;
    constexpr int DD = FAST ? D : 64;

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    uint32_t *bm = smem + wib * (P.nw + HIT_CAP);
    const int64_t gwarp = (int64_t)blockIdx.x * wpb + wib;
    const int64_t nwarps = (int64_t)gridDim.x * wpb;
    WarpList list{bm + P.nw, P.overflow + gwarp * P.n};
    const int gl = lane % G, grp = lane / G;
    const int64_t n = P.n;
    const int dim = FAST ? D : P.dim;

    for (int w = lane; w < P.nw; w += 32) bm[w] = 0u;
    __syncwarp();

    unsigned long long acc_r = 0, acc_e = 0, acc_c = 0, acc_f = 0;

    for (int64_t g = gwarp; g < P.Q; g += nwarps) {
        const float *q = P.units + g * dim;
        float qv[PER];
        if (FAST) {
            const int base = Lay<DD>::base(gl);
#pragma unroll
            for (int i = 0; i < PER; i++) qv[i] = __ldg(q + base + 8 * i);
        }
        auto dist = [&](int r) -> double {
            if constexpr (FAST) return group_dist<DD>(P.refs + (int64_t)r * D, qv, gl);
            else return dist_thread(P.refs + (int64_t)r * dim, q, dim);
        };

        const int p = P.prev[g];
        if (p < 0 || p >= n) {
            if (lane == 0) atomicExch(P.err, ERR_PREV_RANGE);
            continue;
        }
        // search.py:114-117: first ring around the previous match
        double d = dist(p);
        int64_t lo, hi;
        ring_window(P.sdist + (int64_t)p * n, n, __dsub_rn(d, __dmul_rn(P.alpha, d)),
                    __dadd_rn(d, __dmul_rn(P.alpha, d)), lane, lo, hi);
        {
            const int32_t *ir = P.sidx + (int64_t)p * n;
            for (int64_t k = lo + lane; k < hi; k += 32) {
                int j = __ldg(ir + k);
                atomicOr(&bm[j >> 5], 1u << (j & 31));
            }
        }
        __syncwarp();
        int cS = (int)(hi - lo);
        const int first = cS;
        int rings = 1;
        long long evals = 1;

        // used anchors still inside S (search.py:120-122), lane-distributed
        int nu = 0, u_val = -1;
        if (bit_test(bm, p)) {
            nu = 1;
            if (lane == 0) u_val = p;
        }
        bool have_rng = false;
        Pcg64 rng;
        while (cS >= P.L && rings < P.max_rings) {
            int na = cS - nu;
            if (na <= 0) break;
            if (!have_rng) {
                if (P.key_words) {
                    const uint32_t *kw = P.key_words + P.key_off[g];
                    int nk = (int)(P.key_off[g + 1] - P.key_off[g]);
                    pcg_seed(rng, [&](int i) { return __ldg(kw + i); }, nk);
                } else {
                    const uint32_t x = (uint32_t)(g % P.gw), y = (uint32_t)(P.gy0 + g / P.gw);
                    const int snw = P.seed_nw;
                    const uint32_t s0 = P.seed_lo, s1 = P.seed_hi, tt = P.t;
                    pcg_seed(rng, [&](int i) -> uint32_t {
                        if (i < snw) return i == 0 ? s0 : s1;
                        i -= snw;
                        return i == 0 ? x : (i == 1 ? y : tt);
                    }, snw + 3);
                }
                have_rng = true;
            }
            // search.py:129: anchor = avail[integers(|avail|)], avail ascending
            const int k = (int)pcg_integers(rng, (uint64_t)na);
            if (lane < nu) atomicAnd(&bm[u_val >> 5], ~(1u << (u_val & 31)));
            __syncwarp();
            const int a = rank_select(bm, P.nw, k, lane);
            __syncwarp();
            if (lane < nu) atomicOr(&bm[u_val >> 5], 1u << (u_val & 31));
            __syncwarp();
            if (nu >= 32) {
                if (lane == 0) atomicExch(P.err, ERR_USED_OVERFLOW);
                break;
            }
            if (lane == nu) u_val = a;
            nu++;
            // search.py:131-135: ring around the anchor, intersect
            const double da = dist(a);
            evals++;
            ring_window(P.sdist + (int64_t)a * n, n, __dsub_rn(da, __dmul_rn(P.alpha, da)),
                        __dadd_rn(da, __dmul_rn(P.alpha, da)), lane, lo, hi);
            const int32_t *ir = P.sidx + (int64_t)a * n;
            int nh = 0;
            for (int64_t kb = lo; kb < hi; kb += 128) {
                int j0 = -1, j1 = -1, j2 = -1, j3 = -1;
                int64_t k0 = kb + lane;
                if (k0 < hi) j0 = __ldg(ir + k0);
                if (k0 + 32 < hi) j1 = __ldg(ir + k0 + 32);
                if (k0 + 64 < hi) j2 = __ldg(ir + k0 + 64);
                if (k0 + 96 < hi) j3 = __ldg(ir + k0 + 96);
                int js[4] = {j0, j1, j2, j3};
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int j = js[u];
                    const bool hit = j >= 0 && bit_test(bm, j);
                    const unsigned ball = __ballot_sync(FULL, hit);
                    if (hit) list.put(nh + __popc(ball & lanemask_lt()), j);
                    nh += __popc(ball);
                }
            }
            rings++;
            if (nh == 0) break;  // search.py:136-137 rollback: keep S
            __threadfence_block();
            __syncwarp();
            for (int w = lane; w < P.nw; w += 32) bm[w] = 0u;
            __syncwarp();
            for (int e = lane; e < nh; e += 32) {
                int j = list.get(e);
                atomicOr(&bm[j >> 5], 1u << (j & 31));
            }
            __syncwarp();
            cS = nh;
            // keep only used anchors still in S
            bool keep = lane < nu && bit_test(bm, u_val);
            int nnu = 0, nv = -1;
            for (int i = 0; i < nu; i++) {
                int ki = __shfl_sync(FULL, (int)keep, i);
                int vi = __shfl_sync(FULL, u_val, i);
                if (ki) {
                    if (lane == nnu) nv = vi;
                    nnu++;
                }
            }
            nu = nnu;
            u_val = nv;
        }

        // search.py:140-143: scan S u {prev}, first minimum (lowest index)
        const bool p_in = bit_test(bm, p);
        __syncwarp();
        if (lane == 0 && !p_in) atomicOr(&bm[p >> 5], 1u << (p & 31));
        __syncwarp();
        const int nscan = cS + (p_in ? 0 : 1);
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bi = 0x7fffffff;
        int written = 0;
        int32_t *sc_out = P.scanned ? P.scanned + g * (n + 1) : nullptr;
        for (int wb = 0; wb < P.nw; wb += 32) {
            uint32_t w = bm[wb + lane];
            if (!__any_sync(FULL, w != 0u)) continue;
            bm[wb + lane] = 0u;
            const int pc = __popc(w);
            const int inc = warp_incl_scan(pc, lane);
            const int tot = __shfl_sync(FULL, inc, 31);
            int pos = inc - pc;
            while (w) {
                int b = __ffs(w) - 1;
                w &= w - 1;
                int j = (wb + lane) * 32 + b;
                list.sm[pos] = (uint32_t)j;
                if (sc_out) sc_out[written + pos] = j;
                pos++;
            }
            __syncwarp();
            if constexpr (FAST) {
                for (int e0 = 0; e0 < tot; e0 += NG) {
                    const int e = e0 + grp;
                    const bool valid = e < tot;
                    const int j = (int)list.sm[valid ? e : 0];
                    const double dj = dist(j);
                    if (valid) argmin_merge(bd, bi, dj, j);
                }
            } else {
                for (int e = lane; e < tot; e += 32) {
                    const int j = (int)list.sm[e];
                    argmin_merge(bd, bi, dist(j), j);
                }
            }
            written += tot;
            __syncwarp();
        }
        warp_argmin(bd, bi);
        evals += nscan;
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
    }
    if (lane == 0 && P.stats) {
        atomicAdd(P.stats + 0, acc_r);
        atomicAdd(P.stats + 1, acc_e);
        atomicAdd(P.stats + 2, acc_c);
        atomicAdd(P.stats + 3, acc_f);
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

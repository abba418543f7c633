// riann_bulk.cuh -- anchor-grouped ("bulk") frame path for models with n <= 65,536.
//
// The per-query kernel (K2) pays one random DRAM fetch (~64 B) per ring
// membership test: ~4,000 tests per query at config 3.  Here the frame runs in
// phases instead:
//   P0   (warp per query): exact d_prev, first-ring window (coarse + fine
//        search), window copy + radix sort into the query's candidate slot,
//        first anchor draw (numpy RNG).
//   ring phase k (<= max_rings-1 times): active queries are bucketed by their
//        anchor (counting sort); one CTA loads an anchor's rank row
//        pos[a][*] (u16, 128 KB) into shared memory once and filters the
//        candidate lists of every query that drew that anchor (lo <= pos[a][j]
//        < hi is exactly the searchsorted window test), then draws each
//        query's next anchor.
//   F    (warp per query): fp16-screened final scan of S u {prev} with exact
//        FP64 re-check.
// A query that does not fit (first ring > LIGHT_MAX, > BULK_U used anchors
// still in S) is marked heavy and recomputed from scratch by K2, so results
// never depend on the path taken.
#pragma once

#include "riann_kernels.cuh"

namespace rb {

constexpr int LIGHT_MAX = 16384;  // largest first ring handled by the bulk path (u16 entries)
constexpr int BULK_U = 4;        // used anchors tracked per query
constexpr int COARSE = 64;       // coarse index stride of the sorted rows
constexpr int PH_WARPS = 16;     // warps per ring-phase CTA
constexpr int PH_CHUNK = 64;     // queries per ring-phase work item

enum { ST_DONE = 0, ST_ACTIVE = 1, ST_HEAVY = 2 };

struct __align__(16) QState {
    double d_prev;
    int64_t s_off;            // candidate slot offset in the pool
    uint64_t sh, sl, ih, il;  // PCG64 state and increment
    int32_t cS, first, rings, status;
    int32_t anchor, nu, rng_has, p_in;
    uint32_t rng_buf;
    int32_t tests, exact, pad;
    int32_t u[BULK_U];
};

struct BulkParams {
    const float *refs;
    const __half *refs16;
    const float *err16;
    const float *sdist;
    const uint16_t *sidx;
    const uint16_t *pos;     // rank rows: pos[a][sidx[a][k]] = k
    const float *coarse;     // coarse[a][b] = sdist[a][b*COARSE]
    int64_t n;
    int ncoarse;
    const float *units;
    const int32_t *prev;
    int64_t Q;
    uint32_t seed_lo, seed_hi;
    int seed_nw;
    int gw, gy0;
    uint32_t t;
    int L;
    double alpha;
    int max_rings;
    int passes;
    QState *st;
    uint16_t *pool;          // candidate slots (variable size, atomic allocation)
    unsigned long long *pool_top;
    int64_t pool_cap;
    uint16_t *p0_spill;      // per P0 warp: 2 * LIGHT_MAX entries
    int32_t *active_in;      // queries whose anchor is pending (this phase)
    const int32_t *n_active_in;
    int32_t *active_out;     // next phase
    int32_t *n_active_out;
    int32_t *heavy;          // queries for K2
    int32_t *n_heavy;
    int32_t *counts;         // per anchor row (n + 1)
    int32_t *starts;         // exclusive scan of counts
    int32_t *grouped;        // active queries grouped by anchor
    int32_t *item_next;      // work-item counter
    int32_t *seg_next;       // 16 segment counters (ring phase scheduling)
    int32_t *out_idx;
    double *out_dist;
    unsigned long long *stats;
    int *err;
};

__device__ __forceinline__ void seed_frame(Pcg64 &rng, const BulkParams &P, int64_t g)
{
    struct FW {
        uint32_t s0, s1, x, y, t;
        int snw;
        __device__ uint32_t operator()(int i) const
        {
            if (i < snw) return i == 0 ? s0 : s1;
            i -= snw;
            return i == 0 ? x : (i == 1 ? y : t);
        }
    } fw{P.seed_lo, P.seed_hi, (uint32_t)(g % P.gw), (uint32_t)(P.gy0 + g / P.gw), P.t, P.seed_nw};
    pcg_seed(rng, fw, P.seed_nw + 3);
}

__device__ __forceinline__ void rng_load(Pcg64 &r, const QState &s)
{
    r.sh = s.sh;
    r.sl = s.sl;
    r.ih = s.ih;
    r.il = s.il;
    r.has = s.rng_has;
    r.buf = s.rng_buf;
}

__device__ __forceinline__ void rng_store(QState &s, const Pcg64 &r)
{
    s.sh = r.sh;
    s.sl = r.sl;
    s.ih = r.ih;
    s.il = r.il;
    s.rng_has = r.has;
    s.rng_buf = r.buf;
}

// searchsorted pair on a sorted row through its coarse index: returns
// lo = first v >= lv and hi = first v > hv.  The coarse array (shared or global
// memory) is searched 17-ary by the two half-warps (as ring_window); the
// remaining <= 65 entries of the row are counted.
__device__ __forceinline__ void window_coarse(const float *__restrict__ row, const float *cs, int nb, int64_t n,
                                              double lv, double hv, int lane, int64_t &lo, int64_t &hi)
{
    const int h = lane >> 4, hl = lane & 15;
    const double thr = h ? hv : lv;
    int b0 = 0, b1 = nb;  // first coarse entry failing the predicate lies in [b0, b1]
    for (;;) {
        const int s = b1 - b0;
        if (!__any_sync(FULL, s > 16)) break;
        const int p = b0 + (int)(((int64_t)(hl + 1) * s) / 17);
        bool pr = false;
        if (s > 16) {
            const double v = (double)cs[p];
            pr = h ? (v <= thr) : (v < thr);
        }
        const unsigned ball = __ballot_sync(FULL, pr);
        const int c = __popc((ball >> (h * 16)) & 0xffffu);
        const int p_lo = __shfl_sync(FULL, p, h * 16 + (c > 0 ? c - 1 : 0));
        const int p_hi = __shfl_sync(FULL, p, h * 16 + (c < 16 ? c : 15));
        if (s > 16) {
            if (c > 0) b0 = p_lo + 1;
            if (c < 16) b1 = p_hi;
        }
    }
    {
        const int p = b0 + hl;
        bool pr = false;
        if (p < b1) {
            const double v = (double)cs[p];
            pr = h ? (v <= thr) : (v < thr);
        }
        const unsigned ball = __ballot_sync(FULL, pr);
        b0 += __popc((ball >> (h * 16)) & 0xffffu);
    }
    const int b = b0;  // coarse entries [0, b) satisfy the predicate
    const int64_t s0 = b > 0 ? (int64_t)(b - 1) * COARSE + 1 : 0;
    const int64_t s1 = (b < nb) ? (int64_t)b * COARSE : n;
    int cnt = 0;
    for (int64_t k = s0 + hl; k < s1; k += 16) {
        const double v = (double)__ldg(row + k);
        cnt += (h ? (v <= thr) : (v < thr)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
    const int64_t res = s0 + cnt;
    lo = __shfl_sync(FULL, res, 0);
    hi = __shfl_sync(FULL, res, 16);
}

// k-th (0-based) element of ascending list S minus the used anchors u[0..nu)
// (search.py:122, 129).  upos: positions of the used anchors in S.
__device__ __forceinline__ int avail_pos(int k, const int *upos, int nu)
{
    int pos = k;
    for (int it = 0; it <= nu; it++) {
        int c = 0;
        for (int i = 0; i < nu; i++) c += upos[i] <= pos ? 1 : 0;
        if (k + c == pos) break;
        pos = k + c;
    }
    return pos;
}

__device__ __forceinline__ int lower_bound_u16(const uint16_t *a, int cnt, uint32_t x)
{
    int lo = 0, hi = cnt;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((uint32_t)a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// P0: first ring, candidate slot, first anchor.  One warp per query.
// The first-ring window (unordered: distance order) becomes the ascending
// candidate list (np.sort, search.py:116) through a per-warp n-bit bitmap in
// shared memory, enumerated word-interleaved: at step t lane L takes word
// 32t + L, a warp prefix sum places its bits, so each step's stores fall in
// one short run of the slot.
__host__ __device__ constexpr int p0_words(int64_t n) { return (int)(((n + 4095) / 4096) * 128); }

template <int D>
__global__ void __launch_bounds__(256, 3) bulk_p0_kernel(BulkParams P)
{
    extern __shared__ __align__(16) uint32_t smem_w[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int64_t n = P.n;
    const int NW = p0_words(n);  // multiple of 128
    uint32_t *bm = smem_w + (size_t)wib * NW;
    const int64_t nwarps = (int64_t)gridDim.x * wpb;
    const int64_t gwarp = (int64_t)blockIdx.x * wpb + wib;
    for (int i = lane; i < NW; i += 32) bm[i] = 0u;
    __syncwarp();
    for (int64_t g = gwarp; g < P.Q; g += nwarps) {
        const float *q = P.units + g * D;
        const int p = P.prev[g];
        if (p < 0 || p >= n) {
            if (lane == 0) atomicExch(P.err, ERR_PREV_RANGE);
            if (lane == 0) P.st[g].status = ST_HEAVY + 100;  // skipped everywhere
            continue;
        }
        const double d = exact_dist_all<D>(P.refs, p, q, D, lane);
        int64_t lo, hi;
        window_coarse(P.sdist + (int64_t)p * n, P.coarse + (int64_t)p * P.ncoarse, P.ncoarse, n,
                      __dsub_rn(d, __dmul_rn(P.alpha, d)), __dadd_rn(d, __dmul_rn(P.alpha, d)), lane, lo, hi);
        const int cS = (int)(hi - lo);
        int64_t off = 0;
        if (lane == 0 && cS <= LIGHT_MAX) {
            off = (int64_t)atomicAdd(P.pool_top, (unsigned long long)((cS + 7) & ~7));
            if (off + cS > P.pool_cap) off = -1;
        }
        off = __shfl_sync(FULL, off, 0);
        if (cS > LIGHT_MAX || off < 0) {
            if (lane == 0) {
                P.st[g].status = ST_HEAVY;
                P.heavy[atomicAdd(P.n_heavy, 1)] = (int32_t)g;
            }
            continue;
        }
        // window of the u16 index row -> bitmap (16-byte vector loads on the aligned span)
        {
            const uint16_t *row = P.sidx + (int64_t)p * n;
            auto mark = [&](uint32_t j) { atomicOr(&bm[j >> 5], 1u << (j & 31)); };
            const int64_t a0 = (lo + 7) & ~(int64_t)7, a1 = hi & ~(int64_t)7;
            if (a0 < a1) {
                for (int64_t k = lo + lane; k < a0; k += 32) mark(__ldg(row + k));
                for (int64_t v0 = a0 + (int64_t)lane * 8; v0 < a1; v0 += 256) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(row + v0));
                    const uint16_t *e8 = reinterpret_cast<const uint16_t *>(&v);
#pragma unroll
                    for (int x = 0; x < 8; x++) mark(e8[x]);
                }
                for (int64_t k = a1 + lane; k < hi; k += 32) mark(__ldg(row + k));
            } else {
                for (int64_t k = lo + lane; k < hi; k += 32) mark(__ldg(row + k));
            }
        }
        __syncwarp();
        // enumerate ascending into the slot, clearing the bitmap; rank and presence of p.
        // Step t: lane L takes words 128t + 4L .. +3 (one LDS.128); one warp scan per step.
        uint16_t *slot = P.pool + off;
        const int wp = p >> 5;
        int run = 0, below = 0, p_in = 0;
        for (int t = 0; t < NW; t += 128) {
            const int w0 = t + 4 * lane;
            uint4 q4 = *reinterpret_cast<const uint4 *>(bm + w0);
            const uint32_t any4 = q4.x | q4.y | q4.z | q4.w;
            if (!__any_sync(FULL, any4 != 0u)) continue;
            if (any4) *reinterpret_cast<uint4 *>(bm + w0) = make_uint4(0u, 0u, 0u, 0u);
            const int c = __popc(q4.x) + __popc(q4.y) + __popc(q4.z) + __popc(q4.w);
            const int inc = warp_incl_scan(c, lane);
            int o = run + inc - c;
            if ((wp >> 2) == (w0 >> 2)) {  // this lane holds p's word
                const uint32_t wd[4] = {q4.x, q4.y, q4.z, q4.w};
                int bb = o;
                for (int k = 0; k < (wp & 3); k++) bb += __popc(wd[k]);
                below = bb + __popc(wd[wp & 3] & ((1u << (p & 31)) - 1u));
                p_in = (wd[wp & 3] >> (p & 31)) & 1u;
            }
            if (any4) {
                uint16_t *dst = slot + o;
                const uint32_t wd[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    uint32_t word = wd[k];
                    const uint32_t base = (uint32_t)(w0 + k) * 32u;
                    while (word) {
                        const int b = __ffs(word) - 1;
                        word &= word - 1;
                        *dst++ = (uint16_t)(base + b);
                    }
                }
            }
            run += __shfl_sync(FULL, inc, 31);
        }
        const int lp = (wp >> 2) & 31;
        below = __shfl_sync(FULL, below, lp);
        p_in = __shfl_sync(FULL, p_in, lp);
        __threadfence_block();
        __syncwarp();
        if (lane == 0) {
            QState s;
            const bool loop = cS >= P.L && P.max_rings > 1;
            s.d_prev = d;
            s.s_off = off;
            s.cS = cS;
            s.first = cS;
            s.rings = 1;
            s.tests = 0;
            s.exact = 1;
            s.p_in = p_in;
            s.nu = 0;
            s.rng_has = 0;
            s.rng_buf = 0;
            s.sh = s.sl = s.ih = s.il = 0;
            s.anchor = 0;
            int upos[BULK_U];
            if (p_in) {
                s.u[0] = p;
                upos[0] = below;
                s.nu = 1;
            }
            if (loop && cS - s.nu > 0) {
                Pcg64 rng;
                seed_frame(rng, P, g);
                const int k = (int)pcg_integers(rng, (uint64_t)(cS - s.nu));
                const int pos = avail_pos(k, upos, s.nu);
                s.anchor = (int)slot[pos];
                s.u[s.nu++] = s.anchor;
                rng_store(s, rng);
                s.status = ST_ACTIVE;
                P.active_out[atomicAdd(P.n_active_out, 1)] = (int32_t)g;
            } else {
                s.status = ST_DONE;
            }
            P.st[g] = s;
        }
        __syncwarp();
    }
}

// counting sort of the active queries by anchor row
__global__ void bulk_count_kernel(BulkParams P)
{
    const int m = *P.n_active_in;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        atomicAdd(P.counts + P.st[P.active_in[i]].anchor, 1);
}

__global__ void bulk_scatter_kernel(BulkParams P)
{
    const int m = *P.n_active_in;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const int g = P.active_in[i];
        const int a = P.st[g].anchor;
        P.grouped[P.starts[a] + atomicAdd(P.counts + a, 1)] = g;
    }
}

// ---------------------------------------------------------------------------
// Ring phase: CTA per work item (PH_CHUNK consecutive grouped queries).  For
// each run of queries sharing an anchor, one thread starts a TMA bulk copy of
// the anchor's rank row into shared memory; meanwhile every warp does its
// queries' row-independent work (state, exact d_a, window search on the sorted
// row); then the candidate lists are filtered against the shared row.
__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---------------------------------------------------------------------------
// Ring phase: one warp per (query, anchor), queries taken in anchor order so
// the ~200 anchor rank rows in flight at any time stay resident in L2 (a row
// is read from HBM about once per phase); membership tests are 8-deep
// independent lookups pos[a][j] per lane.
template <int D>
__global__ void __launch_bounds__(256, 4) bulk_ring_kernel(BulkParams P)
{
    const int lane = threadIdx.x & 31;
    const int64_t n = P.n;
    const int m = *P.n_active_in;
    // One entry per grab keeps the entries in flight GPU-wide -- and so the
    // anchor rank rows that must stay L2-resident -- at one per resident warp.
    // The anchor-ordered list is cut into NSEG segments with their own
    // counters (atomic traffic / NSEG); a warp whose segment is exhausted
    // steals from the next ones.
    constexpr int NSEG = 16;
    const int64_t gw0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int seg = (int)(gw0 % NSEG), tried = 0;
    for (;;) {
        int i = -1;
        if (lane == 0) {
            while (tried < NSEG) {
                const int s0 = (int)((int64_t)m * seg / NSEG), s1 = (int)((int64_t)m * (seg + 1) / NSEG);
                const int t = s0 + atomicAdd(P.seg_next + seg, 1);
                if (t < s1) {
                    i = t;
                    break;
                }
                seg = (seg + 1) % NSEG;
                tried++;
            }
        }
        i = __shfl_sync(FULL, i, 0);
        if (i < 0) break;
        const int64_t g = P.grouped[i];
        QState *sp = P.st + g;
        const int a = sp->anchor;
        const int cS = sp->cS;
        uint16_t *slot = P.pool + sp->s_off;
        const float *q = P.units + g * D;
        // search.py:131-133: exact d_a (numpy order), window on row a
        const double da = exact_dist<D>(P.refs, a, q, D, lane % Lay<D>::G);
        int64_t lo, hi;
        window_coarse(P.sdist + (int64_t)a * n, P.coarse + (int64_t)a * P.ncoarse, P.ncoarse, n,
                      __dsub_rn(da, __dmul_rn(P.alpha, da)), __dadd_rn(da, __dmul_rn(P.alpha, da)), lane, lo, hi);
        const uint16_t *prow = P.pos + (int64_t)a * n;
        // search.py:134: S' = S n ring, order kept, filtered in place; per block of
        // 1024 entries all list loads, then all rank lookups, are issued together
        int nh = 0;
        for (int base = 0; base < cS; base += 1024) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int i0 = base + k * 256 + lane * 8;
                v[k] = i0 < cS ? *reinterpret_cast<const uint4 *>(slot + i0) : make_uint4(0, 0, 0, 0);
            }
            uint32_t keep4 = 0;  // 8 bits per k
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int i0 = base + k * 256 + lane * 8;
                const uint16_t *e8 = reinterpret_cast<const uint16_t *>(&v[k]);
                uint16_t pk[8];
#pragma unroll
                for (int x = 0; x < 8; x++) pk[x] = (i0 + x < cS) ? __ldg(prow + e8[x]) : (uint16_t)0xffff;
#pragma unroll
                for (int x = 0; x < 8; x++)
                    if (i0 + x < cS && pk[x] >= lo && pk[x] < hi) keep4 |= 1u << (8 * k + x);
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (base + k * 256 >= cS) break;
                const unsigned keepm = (keep4 >> (8 * k)) & 0xffu;
                const int kc = __popc(keepm);
                const int inc = warp_incl_scan(kc, lane);
                const int tot = __shfl_sync(FULL, inc, 31);
                const uint16_t *e8 = reinterpret_cast<const uint16_t *>(&v[k]);
                int o = nh + inc - kc;
#pragma unroll
                for (int x = 0; x < 8; x++)
                    if ((keepm >> x) & 1u) slot[o++] = e8[x];
                nh += tot;
            }
            __syncwarp();
        }
        if (lane == 0) {
            sp->tests += cS;
            sp->exact += 1;
            const int rings = sp->rings + 1;
            sp->rings = rings;
            int status = ST_DONE;  // nh == 0: search.py:136-137 rollback
            if (nh > 0) {
                sp->cS = nh;
                int u[BULK_U];
                int nu = 0;
                const int nu0 = sp->nu;
                for (int k = 0; k < nu0; k++) {
                    const int uk = sp->u[k];
                    const int pk = __ldg(prow + uk);
                    if (pk >= lo && pk < hi) u[nu++] = uk;
                }
                bool pin = false;
                for (int k = 0; k < nu; k++) pin |= u[k] == P.prev[g];
                sp->p_in = pin;
                if (nh >= P.L && rings < P.max_rings && nh - nu > 0) {
                    int upos[BULK_U];
                    for (int k = 0; k < nu; k++) upos[k] = lower_bound_u16(slot, nh, (uint32_t)u[k]);
                    Pcg64 rng;
                    rng.sh = sp->sh;
                    rng.sl = sp->sl;
                    rng.ih = sp->ih;
                    rng.il = sp->il;
                    rng.has = sp->rng_has;
                    rng.buf = sp->rng_buf;
                    const int k = (int)pcg_integers(rng, (uint64_t)(nh - nu));
                    const int pos = avail_pos(k, upos, nu);
                    if (nu >= BULK_U) {
                        status = ST_HEAVY;
                        P.heavy[atomicAdd(P.n_heavy, 1)] = (int32_t)g;
                    } else {
                        const int an = (int)slot[pos];
                        sp->anchor = an;
                        u[nu++] = an;
                        sp->sh = rng.sh;
                        sp->sl = rng.sl;
                        sp->rng_has = rng.has;
                        sp->rng_buf = rng.buf;
                        status = ST_ACTIVE;
                        P.active_out[atomicAdd(P.n_active_out, 1)] = (int32_t)g;
                    }
                }
                for (int k = 0; k < nu; k++) sp->u[k] = u[k];
                sp->nu = nu;
            }
            sp->status = status;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// F: final scan of S u {prev} for every light query (status DONE).
//
// Screening in the references' PCA basis: q' = T^T q (cuBLAS SGEMM, pedantic
// fp32) and r' = fp16(T^T r) (per-row bound e16p[r]).  For T with
// ||T^T T - I|| <= eta, the true distance d = ||q - r|| satisfies
//   (||q' - r'|| - dq - e16p[r]) / (1 + eta) <= d <= (||q' - r'|| + dq + e16p[r]) / (1 - eta)
// (dq bounds the SGEMM rounding error).  Partial sums of squares over the
// leading 16-component chunks are lower bounds of the full sum, so a candidate
// is abandoned as soon as its partial lower bound exceeds the best upper bound
// (initially the previous match's exact distance).  Survivors of all chunks
// whose lower bound can still reach the minimum get the exact FP64 distance
// (numpy order), so the first minimum (lowest index on ties) is exact.
struct ScreenParams {
    const __half *refs_pca16;  // (n, D) fp16, PCA order
    const float *e16p;         // per-row bound
    const float *units_pca;    // (Q, D) fp32
    float slack;               // dq + max_r e16p[r] + 1e-12 (chunk rejection)
    float dq;                  // + 1e-12
    float one_plus_eta, one_minus_eta;
};

constexpr int FB = 512;  // candidates per screening block

template <int D>
__global__ void __launch_bounds__(256, 3) bulk_final_kernel(BulkParams P, ScreenParams SP)
{
    constexpr int GX = Lay<D>::G;
    constexpr int NGX = WARP / GX;
    constexpr int NCH = D / 16;
    constexpr int SURV_CAP = 128;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    // per warp: two (index, partial) lists of FB entries + survivor slots
    unsigned char *ws = smem_raw + (size_t)wib * (2 * FB * 8 + SURV_CAP * 8);
    uint32_t *Aj = reinterpret_cast<uint32_t *>(ws);
    float *As = reinterpret_cast<float *>(ws + FB * 4);
    uint32_t *Bj = reinterpret_cast<uint32_t *>(ws + FB * 8);
    float *Bs = reinterpret_cast<float *>(ws + FB * 12);
    uint32_t *sv_j = reinterpret_cast<uint32_t *>(ws + FB * 16);
    float *sv_lb = reinterpret_cast<float *>(ws + FB * 16 + SURV_CAP * 4);
    const int64_t nwarps = (int64_t)gridDim.x * wpb;
    const uint64_t pol_keep = pol_evict_last();
    unsigned long long acc_r = 0, acc_e = 0, acc_c = 0, acc_f = 0, acc_t = 0, acc_x = 0;
    for (int64_t g = (int64_t)blockIdx.x * wpb + wib; g < P.Q; g += nwarps) {
        const QState &sr = P.st[g];
        if (sr.status != ST_DONE) continue;
        const int cS = sr.cS;
        const int p = P.prev[g];
        const double d = sr.d_prev;
        const float *q = P.units + g * D;
        const float *qp = SP.units_pca + g * D;
        const uint16_t *slot = P.pool + sr.s_off;
        double bd = d;
        int bi = p;
        long long exact_cnt = sr.exact;
        float ub = __double2float_ru(d);
        int nsv = 0;
        auto flush = [&]() {
            __syncwarp();
            int mcount = 0;
            for (int b0 = 0; b0 < nsv; b0 += 32) {
                const int i = b0 + lane;
                const bool ok = i < nsv && sv_lb[i] <= ub;
                const uint32_t jj = i < nsv ? sv_j[i] : 0u;
                const unsigned ball = __ballot_sync(FULL, ok);
                __syncwarp();
                if (ok) sv_j[mcount + __popc(ball & lanemask_lt())] = jj;
                mcount += __popc(ball);
                __syncwarp();
            }
            for (int s0 = 0; s0 < mcount; s0 += NGX) {
                const int si = s0 + lane / GX;
                const bool ok = si < mcount;
                const int jj = (int)sv_j[ok ? si : 0];
                const double dj = exact_dist<D>(P.refs, jj, q, D, lane % GX);
                if (ok) argmin_merge(bd, bi, dj, jj);
            }
            exact_cnt += mcount;
            nsv = 0;
            __syncwarp();
        };
        // partial lower bound in distance space for a partial sum s
        auto lb_of = [&](float s, float sl) {
            return __fdiv_rd(__fsub_rd(__fsqrt_rd(__fmul_rd(s, 0.99997f)), sl), SP.one_plus_eta);
        };
        // chunk test without sqrt/div: (sqrt(0.99997 s) - slack) / (1 + eta) <= ub  <=>
        // s <= (ub (1 + eta) + slack)^2 / 0.99997; thr is that bound rounded up (a superset)
        auto thr_of = [&](float ubv) {
            const float r = __fadd_ru(__fmul_ru(ubv, SP.one_plus_eta), SP.slack);
            return __fdiv_ru(__fmul_ru(r, r), 0.99997f);
        };
        float thr = thr_of(ub);
        for (int blk = 0; blk < cS; blk += FB) {
            const int bn = min(FB, cS - blk);
            // chunk 0 over the block, one candidate per lane
            float qc[16];
            {
                const float4 *q4 = reinterpret_cast<const float4 *>(qp);
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const float4 v = __ldg(q4 + k);
                    qc[4 * k] = v.x;
                    qc[4 * k + 1] = v.y;
                    qc[4 * k + 2] = v.z;
                    qc[4 * k + 3] = v.w;
                }
            }
            int nA = 0;
            for (int e0 = 0; e0 < bn; e0 += 32) {
                const int e = e0 + lane;
                const bool valid = e < bn;
                const uint32_t j = slot[blk + (valid ? e : 0)];
                const uint4 *rp = reinterpret_cast<const uint4 *>(SP.refs_pca16 + (int64_t)j * D);
                const uint4 v0 = ld_keep16(rp, pol_keep), v1 = ld_keep16(rp + 1, pol_keep);
                float s = 0.f;
                const __half2 *h0 = reinterpret_cast<const __half2 *>(&v0);
                const __half2 *h1 = reinterpret_cast<const __half2 *>(&v1);
#pragma unroll
                for (int x = 0; x < 4; x++) {
                    float2 f = __half22float2(h0[x]);
                    float a0 = __fsub_rn(f.x, qc[2 * x]), a1 = __fsub_rn(f.y, qc[2 * x + 1]);
                    s = __fmaf_rn(a0, a0, s);
                    s = __fmaf_rn(a1, a1, s);
                    f = __half22float2(h1[x]);
                    a0 = __fsub_rn(f.x, qc[8 + 2 * x]);
                    a1 = __fsub_rn(f.y, qc[8 + 2 * x + 1]);
                    s = __fmaf_rn(a0, a0, s);
                    s = __fmaf_rn(a1, a1, s);
                }
                const bool keep = valid && s <= thr;
                const unsigned ball = __ballot_sync(FULL, keep);
                if (keep) {
                    const int o = nA + __popc(ball & lanemask_lt());
                    Aj[o] = j;
                    As[o] = s;
                }
                nA += __popc(ball);
            }
            __syncwarp();
            // further chunks for the candidates still alive
            for (int c = 1; c < NCH && nA > 0; c++) {
                {
                    const float4 *q4 = reinterpret_cast<const float4 *>(qp + 16 * c);
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const float4 v = __ldg(q4 + k);
                        qc[4 * k] = v.x;
                        qc[4 * k + 1] = v.y;
                        qc[4 * k + 2] = v.z;
                        qc[4 * k + 3] = v.w;
                    }
                }
                const bool last = c == NCH - 1;
                int nB = 0;
                for (int i0 = 0; i0 < nA; i0 += 32) {
                    const int i = i0 + lane;
                    const bool valid = i < nA;
                    const uint32_t j = valid ? Aj[i] : Aj[0];
                    float s = valid ? As[i] : 0.f;
                    const uint4 *rp = reinterpret_cast<const uint4 *>(SP.refs_pca16 + (int64_t)j * D) + 2 * c;
                    const uint4 v0 = ld_keep16(rp, pol_keep), v1 = ld_keep16(rp + 1, pol_keep);
                    const __half2 *h0 = reinterpret_cast<const __half2 *>(&v0);
                    const __half2 *h1 = reinterpret_cast<const __half2 *>(&v1);
#pragma unroll
                    for (int x = 0; x < 4; x++) {
                        float2 f = __half22float2(h0[x]);
                        float a0 = __fsub_rn(f.x, qc[2 * x]), a1 = __fsub_rn(f.y, qc[2 * x + 1]);
                        s = __fmaf_rn(a0, a0, s);
                        s = __fmaf_rn(a1, a1, s);
                        f = __half22float2(h1[x]);
                        a0 = __fsub_rn(f.x, qc[8 + 2 * x]);
                        a1 = __fsub_rn(f.y, qc[8 + 2 * x + 1]);
                        s = __fmaf_rn(a0, a0, s);
                        s = __fmaf_rn(a1, a1, s);
                    }
                    if (!last) {
                        const bool keep = valid && s <= thr;
                        const unsigned ball = __ballot_sync(FULL, keep);
                        if (keep) {
                            const int o = nB + __popc(ball & lanemask_lt());
                            Bj[o] = j;
                            Bs[o] = s;
                        }
                        nB += __popc(ball);
                    } else {
                        // complete sums: tighten the upper bound, collect survivors
                        float e16 = valid ? ld_keep(SP.e16p + j, pol_keep) : 0.f;
                        const float sl = __fadd_ru(SP.dq, e16);
                        const float u =
                            valid ? __fdiv_ru(__fadd_ru(__fsqrt_ru(__fmul_ru(s, 1.00003f)), sl), SP.one_minus_eta)
                                  : ub;
                        float mv = u;
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) mv = fminf(mv, __shfl_xor_sync(FULL, mv, o));
                        if (mv < ub) {
                            ub = mv;
                            thr = thr_of(ub);
                        }
                        const float lb = lb_of(s, sl);
                        const bool surv = valid && lb <= ub;
                        const unsigned ball = __ballot_sync(FULL, surv);
                        const int add = __popc(ball);
                        if (nsv + add > SURV_CAP) flush();
                        if (surv) {
                            const int o = nsv + __popc(ball & lanemask_lt());
                            sv_j[o] = j;
                            sv_lb[o] = lb;
                        }
                        nsv += add;
                    }
                }
                __syncwarp();
                if (!last) {
                    // swap lists
                    uint32_t *tj = Aj;
                    float *ts = As;
                    Aj = Bj;
                    As = Bs;
                    Bj = tj;
                    Bs = ts;
                    nA = nB;
                }
            }
        }
        flush();
        warp_argmin(bd, bi);
        const int nscan = cS + (sr.p_in ? 0 : 1);
        if (lane == 0) {
            P.out_idx[g] = bi;
            P.out_dist[g] = bd;
        }
        acc_r += sr.rings;
        acc_e += sr.rings + nscan;
        acc_c += cS;
        acc_f += sr.first;
        acc_t += sr.tests;
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
    }
}

// r' = fp16(T^T r) per reference row, e16p = rigorous bound of ||r' - T^T r||
// (T^T r evaluated in float64), and the maximum bound (as float bits).
__global__ void refs_pca_kernel(const float *refs, const float *T, int64_t n, int dim, __half *out, float *e16,
                                unsigned *e16max)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const float *r = refs + j * dim;
    double acc = 0.0;
    for (int i = 0; i < dim; i++) {
        double y = 0.0;
        for (int k = 0; k < dim; k++) y = fma((double)T[(int64_t)k * dim + i], (double)r[k], y);
        const __half h = __float2half_rn((float)y);
        out[j * dim + i] = h;
        const double dl = (double)__half2float(h) - y;
        acc = __fma_ru(dl, dl, acc);
    }
    // + dim * 1e-15 covers the float64 evaluation error of y
    const float b = __double2float_ru(__dsqrt_ru(acc) + 1e-13);
    e16[j] = b;
    atomicMax(e16max, __float_as_uint(b));
}

// rank rows and coarse rows of the sorted tables (built once per model)
__global__ void pos_scatter_kernel(const uint16_t *sidx, int64_t n, int64_t rows, uint16_t *pos)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * n) return;
    int64_t a = i / n;
    pos[a * n + sidx[i]] = (uint16_t)(i - a * n);
}

__global__ void coarse_kernel(const float *sdist, int64_t n, int nb, float *coarse)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * nb) return;
    int64_t a = i / nb, b = i - a * nb;
    coarse[i] = sdist[a * n + b * COARSE];
}

}  // namespace rb

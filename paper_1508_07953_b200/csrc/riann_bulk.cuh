// riann_bulk.cuh -- anchor-grouped ("bulk") frame path for models with n <= 65,536.
//
// The per-query kernel (K2) pays one random DRAM fetch (~64 B) per ring
// membership test: ~5,000 tests per query at config 3.  Here the frame runs in
// phases instead, all in query-independent bulk steps:
//   P0a  (eight lanes per query): exact d_prev, first-ring window (level-1 /
//        coarse / row search), list allocation (search.py:114-117).
//   P0b  (warp per query): the window as an ascending fixed list (np.sort,
//        search.py:116) split in two parts (j < n/2, j >= n/2, each padded to
//        8 entries) with an alive bitmap.
//   draw (eight lanes per query): |S'|, empty-intersection rollback
//        (search.py:136-137), next anchor avail[k] (search.py:122-130) selected
//        over the alive bits with the key's numpy generator; counts anchors.
//   ring phase k (<= max_rings-1 times):
//     group    queries counting-sorted by anchor, one 16-byte descriptor each.
//     window   (eight lanes per query, anchor order) exact d_a and the
//              anchor's window (search.py:131-133).
//     filter   (CTA per (anchor, half-row) item): one TMA bulk copy of half the
//              anchor's rank row pos[a][*] (n bytes) into shared memory; the
//              queries' list groups and alive bytes are loaded into registers;
//              lo <= pos[a][j] < hi is exactly the searchsorted window test of
//              search.py:77-79, 133-134.  Every anchor row is read from HBM
//              once per phase.
//     draw     as above.
//   F    (warp per query): fp16 PCA-basis screened final scan of S u {prev}
//        with exact FP64 re-check (search.py:140-150).
// A query that does not fit (first ring > LIGHT_MAX, > BULK_U used anchors) is
// marked heavy and recomputed from scratch by K2, so results never depend on
// the path taken.
#pragma once

#include "riann_kernels.cuh"

// occupancy knobs (development A/B builds override them with -D)
#ifndef RIANN_FINAL_FB
#define RIANN_FINAL_FB 512
#endif
#ifndef RIANN_FINAL_MINB
#define RIANN_FINAL_MINB 3
#endif
#ifndef RIANN_P0_WPB
#define RIANN_P0_WPB 8
#endif
#ifndef RIANN_P0A_MINB
#define RIANN_P0A_MINB 3
#endif
#ifndef RIANN_FILTER_MINB
#define RIANN_FILTER_MINB 3
#endif
#ifndef RIANN_FILTER_ROUNDS
#define RIANN_FILTER_ROUNDS 2
#endif
#ifndef RIANN_WIN_MINB
#define RIANN_WIN_MINB 4
#endif
#ifndef RIANN_DRAW_MINB
#define RIANN_DRAW_MINB 5
#endif

namespace rb {

constexpr int LIGHT_MAX = 65520;  // largest first ring handled by the bulk path (list positions < 65,536 fit u16)
constexpr int BULK_U = 8;        // used anchors tracked per query (prev + 7 draws at max_rings = 8)
constexpr int COARSE = 64;       // coarse index stride of the sorted rows
#ifndef RIANN_FCAP
#define RIANN_FCAP 248  // three filter CTAs (64 KB half row each) fit an SM
#endif
constexpr int FCAP = RIANN_FCAP;  // query descriptors per filter stage
#ifndef RIANN_FILTER_WARPS
#define RIANN_FILTER_WARPS 16
#endif
constexpr int FW2 = RIANN_FILTER_WARPS;  // warps per filter CTA
#ifndef RIANN_FDIRECT
#define RIANN_FDIRECT 64
#endif
// (anchor, half) items with at most fdirect list groups (8 entries each) look
// ranks up in global memory instead of staging the half row (n bytes): one
// 32-byte sector per entry against n / (8 * groups) bytes of row per entry.
// Enabled by the host when queries per anchor are few (row bands on many
// GPUs: measured -0.5 ms/frame at 1/8 of config 3, +0.3 ms on the whole frame).
constexpr int FDIRECT = RIANN_FDIRECT;
constexpr int FSEG = 256;        // list entries per final-scan fill round (8 per lane)

enum { ST_DONE = 0, ST_ACTIVE = 1, ST_HEAVY = 2, ST_FINISHED = 3 };

// Per-query state.  The candidate list is fixed after P0: S is the set of
// alive entries (bit set in bits[sel]) of the list at pool[s_off ..
// s_off + lenA8 + lenB8), ascending; entries of part A (j < n/2) come first.
struct __align__(16) QState {
    double d_prev;
    int64_t s_off;            // multiple of 128 entries
    uint64_t sh, sl, ih, il;  // PCG64 state and increment
    int32_t cS, first, rings, status;
    int32_t lenA8, lenB8, nu, rng_has;
    uint32_t rng_buf;
    int32_t tests, exact, pin_pos;  // pin_pos: list position of prev (-1: not in the first ring)
    int32_t sel, anchor, lo, hi;    // bits buffer holding S; drawn anchor and its window [lo, hi)
    uint16_t up[BULK_U];            // list positions of the used anchors (search.py:120, 130)
};

struct BulkParams {
    const float *refs;
    const __half *refs16;
    const float *err16;
    const float *sdist;
    const uint16_t *sidx;
    const uint16_t *pos;     // rank rows: pos[a][sidx[a][k]] = k
    const float *coarse;     // coarse[a][b] = sdist[a][b*COARSE]
    const float *coarse1;    // coarse1[a][k] = coarse[a][k*cs1] (k < 32; +inf past the row)
    int64_t n;
    int ncoarse, cs1;
    int vec_probe;           // window search with 16-byte probes (cs1 % 4 == 0, ncoarse % 4 == 0, n % 64 == 0)
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
    uint16_t *pool;          // fixed candidate lists (atomic allocation)
    unsigned long long *pool_top;
    int64_t pool_cap;
    uint8_t *bits0, *bits1;  // alive bits of the pool entries, double-buffered by phase
    int32_t *kept;           // per query: entries kept by the current filter phase
    int32_t *active_in;      // queries whose anchor is pending (this phase)
    const int32_t *n_active_in;
    int32_t *active_out;     // next phase
    int32_t *n_active_out;
    int32_t *heavy;          // queries for K2
    int32_t *n_heavy;
    int32_t *counts;         // per anchor row (n + 1)
    int32_t *starts;         // exclusive scan of counts
    int4 *gdesc;             // per active query in anchor order: (g, s_off/128, lo | lenA8/8 << 17, hi | lenB8/8 << 17)
    int32_t *item_next;      // filter work-item counter
    const int32_t *qin;      // P0a: process only these queries (n_qin of them) -- later passes
    int64_t n_qin;
    int fdirect;             // filter: direct rank lookups for items of <= fdirect list groups
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

__device__ __forceinline__ void rng_store(QState &s, const Pcg64 &r)
{
    s.sh = r.sh;
    s.sl = r.sl;
    s.ih = r.ih;
    s.il = r.il;
    s.rng_has = r.has;
    s.rng_buf = r.buf;
}

// position of the set bit of rank r (0-based, r < popc(w)): five popcount halvings
// (__fns is a software loop)
__device__ __forceinline__ int nth_bit(uint32_t w, int r)
{
    int pos = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const int c = __popc(w & ((1u << s) - 1u));
        const bool up = r >= c;
        r -= up ? c : 0;
        pos += up ? s : 0;
        w = up ? (w >> s) : w;
    }
    return pos;
}

__device__ __forceinline__ int bit_at(const uint8_t *bits, int64_t e) { return (bits[e >> 3] >> (e & 7)) & 1; }

// ---------------------------------------------------------------------------
// P0b: the first ring as a fixed ascending candidate list.  One warp per query.
// The first-ring window (unordered: distance order) becomes the ascending
// candidate list (np.sort, search.py:116) through a per-warp n-bit bitmap in
// shared memory, enumerated word-interleaved: at step t lane L takes words
// 128t + 4L .. +3, a warp prefix sum places its bits, so each step's stores
// fall in one short run of the slot.  Part B (j >= n/2) starts at the next
// multiple of 8 after part A.
__host__ __device__ constexpr int p0_words(int64_t n) { return (int)(((n + 4095) / 4096) * 128); }
// per-warp shared words: the n-bit bitmap, at least 8 KB (the radix path's buffers)
__host__ __device__ constexpr int p0_smem_words(int64_t n) { return p0_words(n) > 2048 ? p0_words(n) : 2048; }
#ifndef RIANN_P0_DENSE_STEP
#define RIANN_P0_DENSE_STEP 2048
#endif
constexpr int P0_DENSE_STEP = RIANN_P0_DENSE_STEP;  // entries per 4,096-bit step from which unstaged steps go word by word
#ifndef RIANN_P0_RADIX_CAP
#define RIANN_P0_RADIX_CAP 512
#endif
constexpr int P0_RADIX_CAP = RIANN_P0_RADIX_CAP;  // windows up to this many entries take the radix path

template <int D>
__global__ void __launch_bounds__(RIANN_P0_WPB * 32, 24 / RIANN_P0_WPB) bulk_p0_kernel(BulkParams P)
{
    extern __shared__ __align__(16) uint32_t smem_w[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int64_t n = P.n;
    const int jh = (int)(n >> 1);
    const int NW = p0_words(n);  // multiple of 128
    uint32_t *bm = smem_w + (size_t)wib * p0_smem_words(n);
    const int64_t nwarps = (int64_t)gridDim.x * wpb;
    const int64_t gwarp = (int64_t)blockIdx.x * wpb + wib;
    for (int i = lane; i < p0_smem_words(n); i += 32) bm[i] = 0u;
    __syncwarp();
    for (int64_t g = gwarp; g < P.Q; g += nwarps) {
        QState *sp = P.st + g;
        // the state in one round: lane l (< 8) holds bytes 16 l .. 16 l + 15
        uint4 sv = make_uint4(0u, 0u, 0u, 0u);
        if (lane < 8) sv = reinterpret_cast<const uint4 *>(sp)[lane];
        const int p = P.prev[g];
        auto word = [&](int wi) {
            const uint32_t c = (wi & 3) == 0 ? sv.x : (wi & 3) == 1 ? sv.y : (wi & 3) == 2 ? sv.z : sv.w;
            return __shfl_sync(FULL, c, wi >> 2);
        };
        if (word(15) != (uint32_t)ST_ACTIVE) continue;  // heavy (K2) or invalid prev
        const int64_t lo = (int)word(26), hi = (int)word(27);
        const int cS = (int)word(12);
        const int64_t off = (int64_t)((uint64_t)word(2) | ((uint64_t)word(3) << 32));
        const int alloc = (cS + 14 + 127) & ~127;
        int cA, lenA8, lenB8, gap, below = 0, p_in = 0;
#ifndef RIANN_P0_RADIX
#define RIANN_P0_RADIX 1
#endif
        if (RIANN_P0_RADIX && cS > 0 && cS <= P0_RADIX_CAP) {
            // small window: bucket the entries by their high bits (counting sort with
            // shared-memory cursors), insertion-sort each lane's 8 buckets, copy
            // out in order -- no n-bit bitmap to scan (the bitmap area is reused
            // and zeroed again afterwards)
            uint32_t *cnt = bm;                                             // 256 cursors
            uint16_t *bst = reinterpret_cast<uint16_t *>(bm + 256);         // 256 bucket starts
            uint16_t *keys = reinterpret_cast<uint16_t *>(bm + 384);        // P0_RADIX_CAP entries
            const int bsh = max(0, 24 - __clz((int)(n - 1)));                // bucket = j >> bsh < 256
            const uint16_t *row = P.sidx + (int64_t)p * n;
            for (int64_t k = lo + lane; k < hi; k += 32) atomicAdd(&cnt[(uint32_t)__ldg(row + k) >> bsh], 1u);
            __syncwarp();
            {
                uint32_t v[8], sm = 0;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    v[k] = cnt[lane * 8 + k];
                    sm += v[k];
                }
                uint32_t run = (uint32_t)warp_incl_scan((int)sm, lane) - sm;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    bst[lane * 8 + k] = (uint16_t)run;
                    cnt[lane * 8 + k] = run;
                    run += v[k];
                }
            }
            __syncwarp();
            for (int64_t k = lo + lane; k < hi; k += 32) {
                const uint32_t j = __ldg(row + k);
                keys[atomicAdd(&cnt[j >> bsh], 1u)] = (uint16_t)j;
            }
            __syncwarp();
            // each lane sorts its buckets (cnt[b] is now the end of bucket b)
            int ca_l = -1, bl_l = -1;
            const int jb = jh >> bsh, pb = p >> bsh;
#pragma unroll 1
            for (int b = lane * 8; b < lane * 8 + 8; b++) {
                const int s0 = bst[b], e0 = (int)cnt[b];
                for (int i = s0 + 1; i < e0; i++) {
                    const uint16_t key = keys[i];
                    int j2 = i - 1;
                    while (j2 >= s0 && keys[j2] > key) {
                        keys[j2 + 1] = keys[j2];
                        j2--;
                    }
                    keys[j2 + 1] = key;
                }
                if (b == jb) {  // entries < n/2 end inside (or at) this bucket
                    int c = s0;
                    while (c < e0 && (int)keys[c] < jh) c++;
                    ca_l = c;
                }
                if (b == pb) {
                    int c = s0;
                    while (c < e0 && (int)keys[c] < p) c++;
                    bl_l = c;
                }
            }
            cA = __shfl_sync(FULL, ca_l, jb >> 3);
            below = __shfl_sync(FULL, bl_l, pb >> 3);
            lenA8 = (cA + 7) & ~7;
            lenB8 = (cS - cA + 7) & ~7;
            gap = lenA8 - cA;
            p_in = (lo == 0) ? 1 : 0;  // p is rank 0 of its own row (self first, model.py:181-186)
            __syncwarp();
            uint16_t *slot = P.pool + off;
            for (int i = lane; i < cS; i += 32) slot[i < cA ? i : i + gap] = keys[i];
            __syncwarp();
            const int used_w = 384 + ((cS + 1) >> 1);
            for (int w = lane; w < used_w; w += 32) bm[w] = 0u;
            __syncwarp();
            RB_CHECK(cA <= cS && lenA8 + lenB8 <= alloc && below <= cS, 11);
        } else {
            // window of the u16 index row -> bitmap; the aligned span's 16-byte loads
            // are all issued before any marking (MB per lane per round)
            cA = 0;
            {
                const uint16_t *row = P.sidx + (int64_t)p * n;
                auto mark = [&](uint32_t j) {
                    atomicOr(&bm[j >> 5], 1u << (j & 31));
                    cA += (int)j < jh ? 1 : 0;
                };
                const int64_t a0 = (lo + 7) & ~(int64_t)7, a1 = hi & ~(int64_t)7;
                if (a0 < a1) {
                    constexpr int MB = 8;
                    uint16_t hd = 0xffff, tl = 0xffff;
                    if (lo + lane < a0) hd = __ldg(row + lo + lane);
                    if (a1 + lane < hi) tl = __ldg(row + a1 + lane);
                    for (int64_t base = a0; base < a1; base += 256 * MB) {
                        uint4 v[MB];
    #pragma unroll
                        for (int u = 0; u < MB; u++) {
                            const int64_t v0 = base + (int64_t)(u * 32 + lane) * 8;
                            v[u] = v0 < a1 ? __ldg(reinterpret_cast<const uint4 *>(row + v0)) : make_uint4(~0u, ~0u, ~0u, ~0u);
                        }
    #pragma unroll
                        for (int u = 0; u < MB; u++) {
                            const int64_t v0 = base + (int64_t)(u * 32 + lane) * 8;
                            if (v0 < a1) {
                                const uint16_t *e8 = reinterpret_cast<const uint16_t *>(&v[u]);
    #pragma unroll
                                for (int x = 0; x < 8; x++) mark(e8[x]);
                            }
                        }
                    }
                    if (lo + lane < a0) mark(hd);
                    if (a1 + lane < hi) mark(tl);
                } else {
                    for (int64_t k = lo + lane; k < hi; k += 32) mark(__ldg(row + k));
                }
            }
            cA = __reduce_add_sync(FULL, cA);
            lenA8 = (cA + 7) & ~7;
            lenB8 = (cS - cA + 7) & ~7;
            gap = lenA8 - cA;
            __syncwarp();
            // enumerate ascending; rank and presence of p.  Step t: lane L takes words
            // 128t + 4L .. +3 (one LDS.128); one warp scan per step.  The list is staged
            // in place, over the bitmap words the steps so far have consumed (a denser
            // window flushes and restarts the staging area; a step that still does not
            // fit goes straight to the slot), and copied out with 16-byte stores.
            uint16_t *slot = P.pool + off;
            // small n: the bitmap leaves at least half of the warp's 8 KB free; the list
            // is staged there (fixed capacity) instead of over the consumed words
            const bool tail_stage = NW <= 1024;
            const int tail_cap = 2 * (p0_smem_words(n) - NW);  // entries
            uint16_t *stg = reinterpret_cast<uint16_t *>(tail_stage ? bm + NW : bm);
            const int wp = p >> 5;
            int run = 0;
            // list positions [spos, fin) are staged at stg[pos - sbase] (sbase = spos & ~7)
            int spos = 0, fin = 0, sbase = 0;
            auto flush = [&]() {
                __syncwarp();
                const int a8 = min(fin, (spos + 7) & ~7);
                if (spos + lane < a8) slot[spos + lane] = stg[spos + lane - sbase];
                const int nv = (fin - a8) >> 3;
                for (int i = lane; i < nv; i += 32)
                    reinterpret_cast<uint4 *>(slot + a8)[i] = reinterpret_cast<const uint4 *>(stg + (a8 - sbase))[i];
                const int tp = a8 + 8 * nv;
                if (tp + lane < fin) slot[tp + lane] = stg[tp + lane - sbase];
                __syncwarp();
            };
            for (int t = 0; t < NW; t += 128) {
                const int w0 = t + 4 * lane;
                const uint4 q4 = *reinterpret_cast<const uint4 *>(bm + w0);
                const uint32_t any4 = q4.x | q4.y | q4.z | q4.w;
                if (!__any_sync(FULL, any4 != 0u)) continue;
                const int c = __popc(q4.x) + __popc(q4.y) + __popc(q4.z) + __popc(q4.w);
                const int inc = warp_incl_scan(c, lane);
                const int tot = __shfl_sync(FULL, inc, 31);
                int o = run + inc - c;
                if ((wp >> 2) == (w0 >> 2)) {  // this lane holds p's word
                    const uint32_t wd[4] = {q4.x, q4.y, q4.z, q4.w};
                    int bb = o;
                    for (int k = 0; k < (wp & 3); k++) bb += __popc(wd[k]);
                    below = bb + __popc(wd[wp & 3] & ((1u << (p & 31)) - 1u));
                    p_in = (wd[wp & 3] >> (p & 31)) & 1u;
                }
                // the step's entries end before position run + tot + 7; 2 (t + 128) entries
                // fit in the words consumed so far.  A denser window flushes what is
                // staged and restarts the staging area at this step's first position.
                const int posb = run < cA ? run : run + gap;
                const int cap_t = tail_stage ? tail_cap : 2 * (t + 128);
                bool stage_ok = run + tot + 7 - sbase <= cap_t;
                if (!stage_ok) {
                    if (fin > spos) flush();
                    spos = fin = posb;
                    sbase = spos & ~7;
                    stage_ok = run + tot + 7 - sbase <= cap_t;
                }
                __syncwarp();  // every lane holds its words: the staged list may grow over them
                auto emit = [&](uint16_t *out) {
                    bool crossed = w0 * 32 >= jh;
                    uint16_t *dst = out + o + (crossed ? gap : 0);
                    const uint32_t wd[4] = {q4.x, q4.y, q4.z, q4.w};
                    if ((jh & 31) == 0) {
                        // part boundary on a word boundary: one check per word
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            uint32_t word = wd[k];
                            const uint32_t base = (uint32_t)(w0 + k) * 32u;
                            if (!crossed && (int)base >= jh && word) {
                                crossed = true;
                                dst += gap;
                            }
                            while (word) {
                                *dst++ = (uint16_t)(base + (uint32_t)(__ffs(word) - 1));
                                word &= word - 1;
                            }
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            uint32_t word = wd[k];
                            const uint32_t base = (uint32_t)(w0 + k) * 32u;
                            while (word) {
                                const int b = __ffs(word) - 1;
                                word &= word - 1;
                                const uint32_t j = base + b;
                                if (!crossed && (int)j >= jh) {
                                    crossed = true;
                                    dst += gap;
                                }
                                *dst++ = (uint16_t)j;
                            }
                        }
                    }
                };
                if (stage_ok) {
                    if (any4) emit(stg - sbase);
                } else if (tot < P0_DENSE_STEP) {
                    if (any4) emit(slot);
                } else {
                    // a step too dense to stage (>= 1 entry per 16 bits so far): word by
                    // word, lane b takes bit b, so the set bits of a word go to consecutive
                    // list positions with one coalesced store
                    for (int ls = 0; ls < 32; ls++) {
                        const uint32_t wx = __shfl_sync(FULL, q4.x, ls), wy = __shfl_sync(FULL, q4.y, ls);
                        const uint32_t wz = __shfl_sync(FULL, q4.z, ls), ww = __shfl_sync(FULL, q4.w, ls);
                        int ob = __shfl_sync(FULL, o, ls);
                        if ((wx | wy | wz | ww) == 0u) continue;  // warp-uniform
                        const uint32_t wd[4] = {wx, wy, wz, ww};
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            const uint32_t word = wd[k];
                            const int j = (t + 4 * ls + k) * 32 + lane;
                            if ((word >> lane) & 1u)
                                slot[ob + __popc(word & lanemask_lt()) + (j >= jh ? gap : 0)] = (uint16_t)j;
                            ob += __popc(word);
                        }
                    }
                }
                run += tot;
                fin = run <= cA ? run : run + gap;
                if (!stage_ok) {  // written straight to the slot: nothing staged
                    spos = fin;
                    sbase = spos & ~7;
                }
            }
            if (fin > spos) flush();
            __syncwarp();
            // the bitmap and the radix path's cursors (words 0 .. 255) are zero between queries
            for (int w = lane * 4; w < max(NW, 256); w += 128) *reinterpret_cast<uint4 *>(bm + w) = make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
            const int lp = (wp >> 2) & 31;
            below = __shfl_sync(FULL, below, lp);
            p_in = __shfl_sync(FULL, p_in, lp);
            RB_CHECK(run == cS && cA <= cS && lenA8 + lenB8 <= alloc && below <= cS, 10);
        }
        // padding entries are valid indices of their part (the filter looks every
        // entry of a group up, alive or not)
        {
            uint16_t *slot = P.pool + off;
            if (lane < 8) {
                if (cA + lane < lenA8) slot[cA + lane] = 0;
            } else if (lane < 16) {
                const int i = lenA8 + (cS - cA) + (lane - 8);
                if (i < lenA8 + lenB8) slot[i] = (uint16_t)jh;
            }
        }
        // alive bits of the list (both buffers zero past the list end, whole words)
        {
            const int nb = (lenA8 + lenB8) >> 3, nbw = alloc >> 3;
            uint8_t *b0 = P.bits0 + (off >> 3), *b1 = P.bits1 + (off >> 3);
            for (int b = lane; b < nbw; b += 32) {
                uint8_t v = 0;
                if (b < nb) {
                    const int rem = b < (lenA8 >> 3) ? cA - 8 * b : (cS - cA) - 8 * (b - (lenA8 >> 3));
                    v = rem >= 8 ? 0xffu : (uint8_t)((1u << rem) - 1u);
                } else {
                    b1[b] = 0;
                }
                b0[b] = v;
            }
        }
        // the first anchor is drawn by the draw kernel (rings 0 -> 1, S in bits0)
        if (lane == 0) {
            const int pin = p_in ? below + (p >= jh ? gap : 0) : -1;
            sp->first = cS;
            sp->rings = 0;
            sp->tests = -cS;  // the draw adds |S|; the first ring is no membership test
            sp->exact = 1;
            sp->lenA8 = lenA8;
            sp->lenB8 = lenB8;
            sp->pin_pos = pin;
            sp->sel = 0;
            sp->nu = p_in ? 1 : 0;
            sp->rng_has = 0;
            sp->rng_buf = 0;
            uint4 u4 = make_uint4(p_in ? (uint32_t)pin : 0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4 *>(sp->up) = u4;
            P.kept[g] = cS;
        }
        __syncwarp();
    }
}

// descriptors of the active queries in anchor order
__global__ void bulk_scatter_kernel(BulkParams P)
{
    const int m = *P.n_active_in;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const int g = P.active_in[i];
        const QState &s = P.st[g];
        const int a = s.anchor;
        RB_CHECK(a >= 0 && a < P.n, 45);
        RB_CHECK(P.starts[a] + P.counts[a] < m + 1, 46);
        P.gdesc[P.starts[a] + atomicAdd(P.counts + a, 1)] =
            make_int4(g, (int)(s.s_off >> 7), s.lo | ((s.lenA8 >> 3) << 17), s.hi | ((s.lenB8 >> 3) << 17));
    }
}

// ---------------------------------------------------------------------------
// List compaction between ring phases (dense first rings: a stream's first
// frame, high-motion clips).  The fixed lists keep their dead entries, so every
// filter phase and the final scan pay for the first ring's size; once the dead
// entries of a query, times the filter phases left, outweigh one rewrite, the
// warp rewrites the list in place (ascending order kept, parts A / B
// compacted separately, padding as in P0b), sets the alive bits of the new
// layout and remaps the list positions the state holds (used anchors still in
// S, prev).  S itself does not change, so results are unaffected.
#ifndef RIANN_COMPACT_X2
#define RIANN_COMPACT_X2 3  // compact when 2 (W - |S|) phases_left >= RIANN_COMPACT_X2 W
#endif
#ifndef RIANN_COMPACT_CK
#define RIANN_COMPACT_CK 4  // chunks of 256 entries loaded per step
#endif
#ifndef RIANN_COMPACT_MINB
#define RIANN_COMPACT_MINB 4
#endif
__global__ void __launch_bounds__(256, RIANN_COMPACT_MINB) bulk_compact_kernel(BulkParams P, int phases_left)
{
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int m = *P.n_active_in;
    const int jh = (int)(P.n >> 1);
    constexpr int CK = RIANN_COMPACT_CK;
    __shared__ __align__(16) uint16_t stg_all[8][256 * CK + 16];
    uint16_t *stg = stg_all[threadIdx.x >> 5];
    for (int64_t ib = gwarp * 32; ib < m; ib += nwarps * 32) {
        // criterion, a lane per query
        int gq = -1;
        if (ib + lane < m) {
            const int g = P.active_in[ib + lane];
            const QState &s = P.st[g];
            const int W = s.lenA8 + s.lenB8;
            if (W >= 256 && 2ll * (W - s.cS) * phases_left >= (long long)RIANN_COMPACT_X2 * W) gq = g;
        }
        unsigned todo = __ballot_sync(FULL, gq >= 0);
        while (todo) {
            const int l = __ffs(todo) - 1;
            todo &= todo - 1;
            const int g = __shfl_sync(FULL, gq, l);
            QState *sp = P.st + g;
            const int64_t soff = sp->s_off;
            const int lenA8 = sp->lenA8, lenB8 = sp->lenB8, nu = sp->nu, pin = sp->pin_pos;
            uint16_t *slot = P.pool + soff;
            uint8_t *bs = (sp->sel ? P.bits1 : P.bits0) + (soff >> 3);  // the buffer holding S
            uint8_t *bo = (sp->sel ? P.bits0 : P.bits1) + (soff >> 3);  // the next filter's output
            // tracked list positions: lanes 0 .. nu - 1 the used anchors, lane nu prev
            int tpos = -1;
            if (lane < nu) tpos = sp->up[lane];
            else if (lane == nu) tpos = pin;
            int tval = -1;
            if (tpos >= 0 && ((bs[tpos >> 3] >> (tpos & 7)) & 1)) tval = slot[tpos];  // alive: its reference index
            __syncwarp();
            // compact one part: entries [r0, r0 + len8) -> from position w0; returns the
            // count.  CK chunks of 256 entries are loaded before any is written (the
            // output never passes the input), the survivors staged in shared memory
            // and copied out with 16-byte stores.
            auto part = [&](int r0, int len8, int w0) {
                int out = w0;
                for (int e0 = 0; e0 < len8; e0 += 256 * CK) {
                    uint4 v[CK];
                    uint32_t al[CK];
#pragma unroll
                    for (int u = 0; u < CK; u++) {
                        const int e = e0 + (u * 32 + lane) * 8;
                        v[u] = make_uint4(0u, 0u, 0u, 0u);
                        al[u] = 0;
                        if (e < len8) {
                            v[u] = *reinterpret_cast<const uint4 *>(slot + r0 + e);
                            al[u] = bs[(r0 + e) >> 3];
                        }
                    }
                    const int sbase = out & ~7;
                    int fin = out;
#pragma unroll
                    for (int u = 0; u < CK; u++) {
                        const int c = __popc(al[u]);
                        const int inc = warp_incl_scan(c, lane);
                        int o = fin + inc - c - sbase;
                        const uint16_t *e8 = reinterpret_cast<const uint16_t *>(&v[u]);
#pragma unroll
                        for (int x = 0; x < 8; x++)
                            if ((al[u] >> x) & 1u) stg[o++] = e8[x];
                        fin += __shfl_sync(FULL, inc, 31);
                    }
                    __syncwarp();
                    // list positions [out, fin) are staged at stg[pos - sbase]
                    const int a8 = min(fin, (out + 7) & ~7);
                    if (out + lane < a8) slot[out + lane] = stg[out + lane - sbase];
                    const int nv = (fin - a8) >> 3;
                    for (int i = lane; i < nv; i += 32)
                        reinterpret_cast<uint4 *>(slot + a8)[i] = reinterpret_cast<const uint4 *>(stg + (a8 - sbase))[i];
                    const int tp = a8 + 8 * nv;
                    if (tp + lane < fin) slot[tp + lane] = stg[tp + lane - sbase];
                    out = fin;
                    __syncwarp();
                }
                return out - w0;
            };
            const int cA = part(0, lenA8, 0);
            const int nA8 = (cA + 7) & ~7;
            if (cA + lane < nA8) slot[cA + lane] = 0;  // padding: valid indices of the part (P0b)
            __syncwarp();
            const int cB = part(lenA8, lenB8, nA8);
            const int nB8 = (cB + 7) & ~7;
            if (nA8 + cB + lane < nA8 + nB8) slot[nA8 + cB + lane] = (uint16_t)jh;
            // alive bits of the new layout in both buffers, zero up to the old end (whole
            // words: lists are allocated in multiples of 128 entries)
            {
                auto below = [](int x) { return x <= 0 ? 0u : x >= 32 ? 0xffffffffu : (1u << x) - 1u; };
                const int nwo = (lenA8 + lenB8 + 31) >> 5;
                uint32_t *ws = reinterpret_cast<uint32_t *>(bs), *wo = reinterpret_cast<uint32_t *>(bo);
                for (int w = lane; w < nwo; w += 32) {
                    const int i0 = 32 * w;
                    ws[w] = below(cA - i0) | (below(nA8 + cB - i0) & ~below(nA8 - i0));
                    wo[w] = 0u;
                }
            }
            __syncwarp();
            // new positions of the tracked entries: binary search of the index in its part
            int npos = -1;
            if (tval >= 0) {
                int lo = tval < jh ? 0 : nA8, hi = tval < jh ? cA : nA8 + cB;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if ((int)slot[mid] < tval) lo = mid + 1;
                    else hi = mid;
                }
                npos = lo;
                RB_CHECK(lo < nA8 + cB && (int)slot[lo] == tval, 60);
            }
            const unsigned keepm = __ballot_sync(FULL, lane < nu && npos >= 0);
            if (lane < nu && npos >= 0) sp->up[__popc(keepm & lanemask_lt())] = (uint16_t)npos;
            const int npin = __shfl_sync(FULL, npos, nu & 31);
            if (lane == 0) {
                sp->nu = __popc(keepm);
                sp->pin_pos = pin >= 0 ? npin : -1;
                sp->lenA8 = nA8;
                sp->lenB8 = nB8;
                RB_CHECK(cA + cB == sp->cS && nA8 <= lenA8 && nA8 + nB8 <= lenA8 + lenB8, 61);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
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

#ifdef RIANN_HANG_DEBUG
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    for (long long it = 0;; it++) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (it == (1ll << 24)) {
            printf("HANG block %d tid %d bar@%u parity %u\n", blockIdx.x, threadIdx.x, smem_addr(bar), parity);
            __trap();
        }
    }
}
#else
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
#endif

__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}


// ---------------------------------------------------------------------------
// Ring phase filter (search.py:133-134).  Work item (a, h): half h of anchor
// a's rank row (entries j in [h n/2, (h+1) n/2), n bytes) arrives in shared
// memory by one TMA bulk copy; meanwhile every thread loads its 8-entry groups
// of the queries' part-h lists and their alive bytes straight into registers
// (groups spread evenly over the CTA: coalesced 16-byte loads), then tests its
// alive entries: lo <= pos[a][j] < hi.  New alive bits go to the other bit
// buffer, kept counts to kept[g].  The next item's descriptors are fetched
// while the copy flies; two CTAs per SM overlap one CTA's copy with the
// other's filtering.  (Staging the lists by per-query TMA copies instead costs
// ~30 ns of TMA issue per copy: measured slower.)
__host__ __device__ constexpr size_t filter_smem(int64_t n)
{
    return (size_t)n + 2 * FCAP * 16 + (FCAP + 1) * 4 + FCAP + 4;
}

__global__ void __launch_bounds__(FW2 * 32, RIANN_FILTER_MINB) bulk_filter_kernel(BulkParams P, int cur)
{
    extern __shared__ __align__(128) unsigned char smem_f[];
    const int64_t n = P.n;
    const int jh = (int)(n >> 1);
    uint16_t *row = reinterpret_cast<uint16_t *>(smem_f);
    int4 *descb = reinterpret_cast<int4 *>(smem_f + n);
    int *qg0 = reinterpret_cast<int *>(descb + 2 * FCAP);  // group offsets of the chunk's queries with groups in part h
    uint8_t *qsel = reinterpret_cast<uint8_t *>(qg0 + FCAP + 1);  // ... and their descriptor slots
    __shared__ uint64_t dbar[2], rbar;
    __shared__ int s_it[2], s_cnt[2], s_start[2], s_ng, s_mc, s_direct;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint8_t *bcur = cur ? P.bits1 : P.bits0;
    uint8_t *bnxt = cur ? P.bits0 : P.bits1;
    auto fetch_desc = [&](int b, int start, int m) {  // one thread
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&dbar[b], (unsigned)m * 16u);
        tma_bulk_g2s(descb + b * FCAP, P.gdesc + start, (unsigned)m * 16u, &dbar[b]);
    };
    // work items: batches of FGRAB consecutive (anchor, half) items taken with
    // one atomic; warp 1 reads a batch's counts / starts in one load round into
    // a lane window, so only one item in FGRAB waits on memory (8: measured
    // best of 8 / 16 / 32)
#ifndef RIANN_FGRAB
#define RIANN_FGRAB 8
#endif
    constexpr int FGRAB = RIANN_FGRAB;
    const int nitems = (int)(2 * n);
    int win_it = -1, win_cnt = 0, win_start = 0;  // per lane of warp 1
    unsigned win_mask = 0;
    bool drained = false;
    auto next_item = [&](int &it, int &cnt, int &start) {  // all lanes of warp 1
        it = -1;
        cnt = start = 0;
        while (it < 0) {
            if (win_mask == 0) {
                if (drained) return;
                int base = 0;
                if (lane == 0) base = atomicAdd(P.item_next, FGRAB);
                base = __shfl_sync(FULL, base, 0);
                if (base >= nitems) {
                    drained = true;
                    return;
                }
                const int i = base + lane;
                win_it = (lane < FGRAB && i < nitems) ? i : -1;
                win_cnt = win_it >= 0 ? P.counts[i >> 1] : 0;
                win_start = win_cnt > 0 ? P.starts[i >> 1] : 0;
                win_mask = __ballot_sync(FULL, win_cnt > 0);
                continue;
            }
            const int l = __ffs(win_mask) - 1;
            win_mask &= win_mask - 1;
            it = __shfl_sync(FULL, win_it, l);
            cnt = __shfl_sync(FULL, win_cnt, l);
            start = __shfl_sync(FULL, win_start, l);
        }
    };
    if (tid == 0) {
        mbar_init(&dbar[0], 1);
        mbar_init(&dbar[1], 1);
        mbar_init(&rbar, 1);
    }
    __syncthreads();
    if (w == 1) {
        int it, cnt, start;
        next_item(it, cnt, start);
        if (lane == 0) {
            s_it[0] = it;
            s_cnt[0] = cnt;
            s_start[0] = start;
            if (it >= 0) fetch_desc(0, start, min(cnt, FCAP));
        }
    }
    __syncthreads();
    unsigned dpar0 = 0, dpar1 = 0, rpar = 0;
    int db = 0;
    for (;;) {
        const int it = s_it[db];
        if (it < 0) break;
        const int cnt = s_cnt[db], start = s_start[db];
        const int a = it >> 1, h = it & 1;
        int4 *desc = descb + db * FCAP;
        bool first_sub = true;
        for (int c0 = 0; c0 < cnt; c0 += FCAP) {
            const int m = min(FCAP, cnt - c0);
            if (c0 > 0 && tid == 0) fetch_desc(db, start + c0, m);
            if (db == 0) {
                mbar_wait(&dbar[0], dpar0);
                dpar0 ^= 1;
            } else {
                mbar_wait(&dbar[1], dpar1);
                dpar1 ^= 1;
            }
            // warp 0: group offsets of the chunk's queries that have groups in
            // part h (compacted: offsets strictly ascending) and the row copy
            if (w == 0) {
                int run = 0, mc = 0;
                for (int b = 0; b < m; b += 32) {
                    const int i = b + lane;
                    int ng = 0;
                    if (i < m) {
                        const int4 d = desc[i];
                        ng = h ? (d.w >> 17) : (d.z >> 17);
                    }
                    const int inc = warp_incl_scan(ng, lane);
                    const unsigned nz = __ballot_sync(FULL, ng > 0);
                    if (ng > 0) {
                        const int o = mc + __popc(nz & lanemask_lt());
                        qg0[o] = run + inc - ng;
                        qsel[o] = (uint8_t)i;
                    }
                    mc += __popc(nz);
                    run += __shfl_sync(FULL, inc, 31);
                }
                if (lane == 0) {
                    qg0[mc] = run;
                    s_ng = run;
                    s_mc = mc;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (first_sub) {
                        // few list groups for this (anchor, half): look the ranks up in
                        // global memory (L2) instead of staging the n-byte half row
                        s_direct = (cnt <= FCAP && run <= P.fdirect) ? 1 : 0;
                        if (!s_direct) {
                            mbar_expect_tx(&rbar, (unsigned)n);
                            tma_bulk_g2s(row, P.pos + (int64_t)a * n + (int64_t)h * jh, (unsigned)n, &rbar);
                        }
                    }
                }
                __syncwarp();
            }
            __syncthreads();
            const int NGt = s_ng;
            const bool direct = s_direct != 0;  // block-uniform, set with s_ng
            // the next item and its descriptors, while the copies fly
            if (first_sub && w == 1) {
                int nit, ncnt, nstart;
                next_item(nit, ncnt, nstart);
                if (lane == 0) {
                    s_it[db ^ 1] = nit;
                    s_cnt[db ^ 1] = ncnt;
                    s_start[db ^ 1] = nstart;
                    if (nit >= 0) fetch_desc(db ^ 1, nstart, min(ncnt, FCAP));
                }
            }
            // The chunk's NGt list groups are cut into FW2 contiguous spans of whole
            // 32-group rounds, one per warp; lane l of a round takes group Gr + l.
            // Its query: xc (the query holding Gr, warp-uniform) plus the number of
            // query boundaries in (Gr, Gr + l], a popcount over a 32-bit boundary
            // mask (the compacted offsets are strictly ascending, so at most 31
            // boundaries fall inside a round).  FR rounds are loaded before any is
            // tested.
            const int mc = s_mc;
            const int rpw = ((NGt + 31) / 32 + FW2 - 1) / FW2;  // rounds per warp
            const int gs = min(w * rpw * 32, NGt), ge = min(gs + rpw * 32, NGt);
            bool need_row = first_sub && !direct;  // block-uniform
            if (need_row) rpar ^= 1;
            const uint32_t hoff = (uint32_t)(h * jh), jmax = (uint32_t)(jh - 1);
            (void)jmax;
            const uint16_t *grow = P.pos + (int64_t)a * n;            // direct lookups: pos[a][e]
            const uint32_t rowb = smem_addr(row) - 2u * hoff;         // staged half row: byte address of entry e = rowb + 2 e
            if (gs < ge) {
                int xc;  // last compacted query with qg0[xc] <= gs
                {
                    const unsigned b1 = __ballot_sync(FULL, lane * 8 <= mc && qg0[min(lane * 8, mc)] <= gs);
                    const int blk = 31 - __clz((int)b1);
                    const int i1 = blk * 8 + (lane & 7);
                    const unsigned b2 = __ballot_sync(FULL, lane < 8 && i1 <= mc && qg0[min(i1, mc)] <= gs);
                    xc = blk * 8 + 31 - __clz((int)b2);
                }
                constexpr int FR = RIANN_FILTER_ROUNDS;
                const uint32_t le_mask = 0xffffffffu >> (31 - lane);  // bits 0 .. lane
                for (int Gb = gs; Gb < ge; Gb += 32 * FR) {
                    uint4 v[FR];
                    uint32_t al[FR];
                    uint32_t eg[FR];  // list group (8 entries) in the pool
                    int dsl[FR];  // descriptor slot, -1: no group
#pragma unroll
                    for (int r = 0; r < FR; r++) {
                        const int Gr = Gb + 32 * r;
                        dsl[r] = -1;
                        al[r] = 0;
                        eg[r] = 0;
                        v[r] = make_uint4(0u, 0u, 0u, 0u);
                        if (Gr < ge) {  // warp-uniform
                            const int bo = qg0[min(xc + 1 + lane, mc)] - Gr;  // >= 1, ascending over the lanes
                            const uint32_t bm = __reduce_or_sync(FULL, bo < 32 ? 1u << bo : 0u);
                            const int xl = xc + __popc(bm & le_mask);
                            xc += __popc(bm) + (__any_sync(FULL, bo == 32) ? 1 : 0);  // the query holding Gr + 32
                            const int Gl = Gr + lane;
                            if (Gl < ge) {
                                const int di = qsel[xl];
                                const int4 d = desc[di];
                                RB_CHECK(xl < mc && di < m && d.x >= 0 && d.x < P.Q && Gl >= qg0[xl] && Gl < qg0[xl + 1], 20);
                                dsl[r] = di;
                                eg[r] = ((uint32_t)d.y << 4) + (h ? (uint32_t)(d.z >> 17) : 0u) + (uint32_t)(Gl - qg0[xl]);
                                RB_CHECK((int64_t)eg[r] * 8 + 8 <= P.pool_cap, 21);
                                al[r] = bcur[eg[r]];
                                v[r] = reinterpret_cast<const uint4 *>(P.pool)[eg[r]];
                            }
                        }
                    }
                    if (need_row) {  // the first test of the item waits for the row copy
                        mbar_wait(&rbar, rpar ^ 1);
                        need_row = false;
                    }
#pragma unroll
                    for (int r = 0; r < FR; r++) {
                        if (Gb + 32 * r >= ge) break;  // warp-uniform
                        uint32_t keep = 0;
                        int gq = -1;
                        if (dsl[r] >= 0) {
                            const int4 d = desc[dsl[r]];
                            gq = d.x;
                            const uint32_t lo = (uint32_t)(d.z & 0x1ffff), wlen = (uint32_t)(d.w & 0x1ffff) - lo;
                            // all eight lookups issued unconditionally, the alive bits mask the
                            // result: dead and padding entries are indices of this half too (P0b)
                            const uint32_t w4[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
                            uint32_t rk[8];
                            if (direct) {
#pragma unroll
                                for (int k = 0; k < 8; k++) {
                                    const uint32_t e = (k & 1) ? (w4[k >> 1] >> 16) : (w4[k >> 1] & 0xffffu);
                                    RB_CHECK(e - hoff <= jmax, 22);
                                    rk[k] = __ldg(grow + e);
                                }
                            } else {
#pragma unroll
                                for (int k = 0; k < 8; k++) {
                                    const uint32_t e = (k & 1) ? (w4[k >> 1] >> 16) : (w4[k >> 1] & 0xffffu);
                                    RB_CHECK(e - hoff <= jmax, 22);
                                    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(rk[k]) : "r"(rowb + 2u * e));
                                }
                            }
#pragma unroll
                            for (int k = 0; k < 8; k++) keep |= (rk[k] - lo < wlen ? 1u : 0u) << k;  // lo <= r < hi
                            keep &= al[r];
                            bnxt[eg[r]] = (uint8_t)keep;
                        }
                        const int c = __popc(keep);
                        const int q_l0 = __shfl_sync(FULL, gq, 0);
                        if (__all_sync(FULL, gq == q_l0)) {
                            const int cw = __reduce_add_sync(FULL, c);
                            if (lane == 0 && cw > 0) atomicAdd(P.kept + gq, cw);
                        } else if (c > 0) {
                            atomicAdd(P.kept + gq, c);
                        }
                    }
                }
            }
            // a warp without work still observes the copy: no row copy is in flight
            // when the next one is issued
            if (need_row) mbar_wait(&rbar, rpar ^ 1);
            first_sub = false;
            // every warp is done with the descriptors, qg0 and the row before they are rewritten
            __syncthreads();
        }
        db ^= 1;
    }
}

// ---------------------------------------------------------------------------
// Ring phase draw (search.py:121-137): four queries per warp, eight lanes each.
// |S'| = kept, rollback on an empty intersection, next anchor avail[k] from the
// query's generator (select over the alive bits), its exact distance (numpy
// order: lane j holds accumulator j of each 96/64-element half) and its window
// on the sorted row in three rounds: 32-entry level-1 index, 32 coarse entries,
// <= 64 row values.
template <int D>
__device__ __forceinline__ double dist8(const float *__restrict__ r, const float (&qv)[D / 8], int gl)
{
    constexpr int H = D > 128 ? D / 2 : D;  // numpy pairwise halves
    constexpr int PER = H / 8;
    double h0 = sqdiff(__ldg(r + gl), qv[0]);
#pragma unroll
    for (int i = 1; i < PER; i++) h0 = __dadd_rn(h0, sqdiff(__ldg(r + gl + 8 * i), qv[i]));
    double h1 = 0.0;
    if constexpr (D > 128) {
        h1 = sqdiff(__ldg(r + H + gl), qv[PER]);
#pragma unroll
        for (int i = 1; i < PER; i++) h1 = __dadd_rn(h1, sqdiff(__ldg(r + H + gl + 8 * i), qv[PER + i]));
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        h0 = __dadd_rn(h0, __shfl_xor_sync(FULL, h0, o));
        if constexpr (D > 128) h1 = __dadd_rn(h1, __shfl_xor_sync(FULL, h1, o));
    }
    if constexpr (D > 128) h0 = __dadd_rn(h0, h1);
    return __dsqrt_rn(h0);
}

__device__ __forceinline__ int grp_sum(int v)
{
    v += __shfl_xor_sync(FULL, v, 1);
    v += __shfl_xor_sync(FULL, v, 2);
    v += __shfl_xor_sync(FULL, v, 4);
    return v;
}

// exact distance d of the query (qv) to reference a and the window [wlo, whi)
// of row a for [d - alpha d, d + alpha d] (search.py:77-79), eight lanes:
// level-1 index (32 entries) with the reference row, then 32 coarse entries,
// then <= 63 row values.  act == false: no row reads past the first round.
template <int D>
__device__ __forceinline__ double dist_window8(const BulkParams &P, int a, const float (&qv)[D / 8], bool act, int gl,
                                               int gb, int &wlo, int &whi)
{
    const int64_t n = P.n;
    const int nb = P.ncoarse, cs1 = P.cs1;
    float4 l1 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) l1 = __ldg(reinterpret_cast<const float4 *>(P.coarse1 + (int64_t)a * 32) + gl);
    const double da = dist8<D>(P.refs + (int64_t)a * D, qv, gl);
    const double lv = __dsub_rn(da, __dmul_rn(P.alpha, da)), hv = __dadd_rn(da, __dmul_rn(P.alpha, da));
    int b1lo, b1hi;
    {
        const float e[4] = {l1.x, l1.y, l1.z, l1.w};
        int cl = 0, ch = 0;
#pragma unroll
        for (int x = 0; x < 4; x++) {
            cl += (double)e[x] < lv ? 1 : 0;
            ch += (double)e[x] <= hv ? 1 : 0;
        }
        b1lo = grp_sum(cl);
        b1hi = grp_sum(ch);
    }
    // coarse round: lanes 0-3 of the group for lo, 4-7 for hi
    const bool sh = gl >= 4;
    const int sl = gl & 3;
    const double thr = sh ? hv : lv;
    int res;
    if (P.vec_probe) {
        // 16-byte probes of aligned blocks (cs1 % 4 == 0, nb % 4 == 0, n % 64 == 0).
        // The level-1 block's first coarse entry (coarse1[b1 - 1]) is known to
        // pass, the next block's first entry to fail, so counting the aligned 32
        // entries [cb, cb + 32) gives b directly; the same one level down.
        int b;
        {
            const int b1 = sh ? b1hi : b1lo;
            const int cb = (b1 - 1) * cs1;
            int cnt = 0;
            if (act && b1 > 0) {
                const int cend = min(b1 * cs1, nb);
                const float *cr = P.coarse + (int64_t)a * nb;
                float4 c4[2];
#pragma unroll
                for (int x = 0; x < 2; x++) {
                    const int ci = cb + sl * 8 + 4 * x;
                    c4[x] = ci < cend ? __ldg(reinterpret_cast<const float4 *>(cr + ci)) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int x = 0; x < 2; x++) {
                    const int ci = cb + sl * 8 + 4 * x;
                    const float e[4] = {c4[x].x, c4[x].y, c4[x].z, c4[x].w};
#pragma unroll
                    for (int y = 0; y < 4; y++) {
                        const double v = (double)e[y];
                        cnt += (ci + y < cend && (sh ? v <= thr : v < thr)) ? 1 : 0;
                    }
                }
            }
            cnt += __shfl_xor_sync(FULL, cnt, 1);
            cnt += __shfl_xor_sync(FULL, cnt, 2);
            b = b1 > 0 ? cb + cnt : 0;
        }
        {
            const int64_t blk = (int64_t)max(b - 1, 0) * COARSE;  // 64 row values [blk, blk + 64)
            int cnt = 0;
            if (act) {
                const float *rr = P.sdist + (int64_t)a * n + blk;
                float4 r4[4];
#pragma unroll
                for (int x = 0; x < 4; x++) r4[x] = __ldg(reinterpret_cast<const float4 *>(rr + sl * 16) + x);
#pragma unroll
                for (int x = 0; x < 4; x++) {
                    const float e[4] = {r4[x].x, r4[x].y, r4[x].z, r4[x].w};
#pragma unroll
                    for (int y = 0; y < 4; y++) {
                        const double v = (double)e[y];
                        cnt += (sh ? v <= thr : v < thr) ? 1 : 0;
                    }
                }
            }
            cnt += __shfl_xor_sync(FULL, cnt, 1);
            cnt += __shfl_xor_sync(FULL, cnt, 2);
            res = (int)(blk + cnt);
        }
    } else {
    int b;
    {
        const int b1 = sh ? b1hi : b1lo;
        int cnt = 0;
        const int cb = (b1 - 1) * cs1;
        if (act && b1 > 0) {
            const int cend = min(b1 * cs1, nb);
            const float *cr = P.coarse + (int64_t)a * nb;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                const int ci = cb + 1 + sl * 8 + x;
                if (ci < cend) {
                    const double v = (double)__ldg(cr + ci);
                    cnt += (sh ? v <= thr : v < thr) ? 1 : 0;
                }
            }
        }
        cnt += __shfl_xor_sync(FULL, cnt, 1);
        cnt += __shfl_xor_sync(FULL, cnt, 2);
        b = b1 > 0 ? cb + 1 + cnt : 0;
    }
    // fine round: <= 63 row values
    {
        const int64_t s0 = b > 0 ? (int64_t)(b - 1) * COARSE + 1 : 0;
        const int64_t s1 = b < nb ? (int64_t)b * COARSE : n;
        int cnt = 0;
        if (act) {
            const float *rr = P.sdist + (int64_t)a * n;
#pragma unroll
            for (int x = 0; x < 16; x++) {
                const int64_t k = s0 + sl * 16 + x;
                if (k < s1) {
                    const double v = (double)__ldg(rr + k);
                    cnt += (sh ? v <= thr : v < thr) ? 1 : 0;
                }
            }
        }
        cnt += __shfl_xor_sync(FULL, cnt, 1);
        cnt += __shfl_xor_sync(FULL, cnt, 2);
        res = (int)(s0 + cnt);
    }
    }
    wlo = __shfl_sync(FULL, res, gb);
    whi = __shfl_sync(FULL, res, gb | 4);
    return da;
}

template <int D>
__device__ __forceinline__ void load_qv8(const float *q, float (&qv)[D / 8], int gl)
{
    constexpr int HD = D > 128 ? D / 2 : D;
#pragma unroll
    for (int k = 0; k < HD / 8; k++) qv[k] = __ldg(q + gl + 8 * k);
    if constexpr (D > 128) {
#pragma unroll
        for (int k = 0; k < HD / 8; k++) qv[HD / 8 + k] = __ldg(q + HD + gl + 8 * k);
    }
}

// P0a (search.py:114-117): exact d_prev and the first-ring window on row prev,
// the list allocation; four queries per warp, in index order.  Queries whose
// first ring exceeds LIGHT_MAX (or the pool) go to K2.
template <int D>
__global__ void __launch_bounds__(256, RIANN_P0A_MINB) bulk_p0a_kernel(BulkParams P)
{
    const int lane = threadIdx.x & 31, gl = lane & 7, gb = lane & ~7;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nq = P.qin ? P.n_qin : P.Q;
    for (int64_t ib = gwarp * 4; ib < nq; ib += nwarps * 4) {
        const int64_t gi = ib + (lane >> 3);
        const int64_t g = gi < nq ? (P.qin ? (int64_t)P.qin[gi] : gi) : 0;
        const int p = P.prev[g];
        const bool ok = gi < nq && p >= 0 && p < P.n;
        if (gi < nq && !ok && gl == 0) {
            atomicExch(P.err, ERR_PREV_RANGE);
            P.st[g].status = ST_HEAVY + 100;  // skipped everywhere
        }
        if (!__any_sync(FULL, ok)) continue;
        float qv[D / 8];
        load_qv8<D>(P.units + g * D, qv, gl);
        int lo, hi;
        const double d = dist_window8<D>(P, ok ? p : 0, qv, ok, gl, gb, lo, hi);
        // list allocation: one atomic per warp for its (up to four) queries
        const int cS = hi - lo;
        const int alloc = (cS + 14 + 127) & ~127;  // >= lenA8 + lenB8; bits of a list 16-byte aligned
        int64_t off = -1;
        {
            const int want = (ok && gl == 0 && cS <= LIGHT_MAX) ? alloc : 0;
            int inc = want;  // inclusive sum over the group leaders (lanes 0, 8, 16, 24)
            inc += __shfl_up_sync(FULL, inc, 8) * (lane >= 8 ? 1 : 0);
            inc += __shfl_up_sync(FULL, inc, 16) * (lane >= 16 ? 1 : 0);
            const int tot = __shfl_sync(FULL, inc, 24);
            unsigned long long base = 0;
            if (lane == 0 && tot > 0) base = atomicAdd(P.pool_top, (unsigned long long)tot);
            base = __shfl_sync(FULL, base, 0);
            if (want > 0) {
                off = (int64_t)base + (inc - want);
                if (off + alloc > P.pool_cap) off = -1;
            }
        }
        if (ok && gl == 0) {
            QState *sp = P.st + g;
            RB_CHECK(lo >= 0 && lo <= hi && hi <= P.n, 1);
            RB_CHECK(off < 0 || off + alloc <= P.pool_cap, 2);
            sp->d_prev = d;
            sp->lo = lo;
            sp->hi = hi;
            sp->cS = cS;
            if (off < 0) {
                sp->status = ST_HEAVY;
                P.heavy[atomicAdd(P.n_heavy, 1)] = (int32_t)g;
            } else {
                sp->s_off = off;
                sp->status = ST_ACTIVE;
            }
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256, RIANN_DRAW_MINB) bulk_draw_kernel(BulkParams P, int cur)
{
    static_assert(D % 8 == 0 && D <= 256, "draw kernel dims");
    const int lane = threadIdx.x & 31, gl = lane & 7, gb = lane & ~7;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint8_t *bnxt = cur ? P.bits0 : P.bits1;
    // queries in index order (the state, unit rows, lists and bits then stream
    // sequentially); those filtered this phase have status ACTIVE
    for (int64_t ib = gwarp * 4; ib < P.Q; ib += nwarps * 4) {
        const int64_t gi = ib + (lane >> 3);
        const int64_t g = gi < P.Q ? gi : 0;
        QState *sp = P.st + g;
        // the whole state: lane gl holds bytes 16 gl .. 16 gl + 15
        uint4 sv = gi < P.Q ? reinterpret_cast<const uint4 *>(sp)[gl] : make_uint4(0u, 0u, 0u, 0u);
        const bool has = __shfl_sync(FULL, sv.w, gb | 3) == (uint32_t)ST_ACTIVE && gi < P.Q;  // word 15: status
        if (!has) sv = make_uint4(0u, 0u, 0u, 0u);
        if (!__any_sync(FULL, has)) continue;
        const int kept = has ? P.kept[g] : 0;
        auto word = [&](int wi) {  // 32-bit word wi of the state (compile-time wi)
            const uint32_t c = (wi & 3) == 0 ? sv.x : (wi & 3) == 1 ? sv.y : (wi & 3) == 2 ? sv.z : sv.w;
            return __shfl_sync(FULL, c, gb | (wi >> 2));
        };
        const int64_t soff = (int64_t)((uint64_t)word(2) | ((uint64_t)word(3) << 32));
        const int cS = (int)word(12);
        const int rings = (int)word(14) + 1;
        const int W = (int)word(16) + (int)word(17);
        const int nu = (int)word(18);
        uint16_t up[BULK_U];
        {
            const uint32_t u0 = word(28), u1 = word(29), u2 = word(30), u3 = word(31);
            up[0] = (uint16_t)u0; up[1] = (uint16_t)(u0 >> 16);
            up[2] = (uint16_t)u1; up[3] = (uint16_t)(u1 >> 16);
            up[4] = (uint16_t)u2; up[5] = (uint16_t)(u2 >> 16);
            up[6] = (uint16_t)u3; up[7] = (uint16_t)(u3 >> 16);
        }
        const uint8_t *bq = bnxt + (soff >> 3);
        int ub = 0;
        if (kept > 0 && gl < nu) ub = bit_at(bq, up[gl]);
        const int nua = grp_sum(ub);
        const bool want = kept > 0 && kept >= P.L && rings < P.max_rings && kept - nua > 0;
        const bool drew = want && nu < BULK_U;
        // numpy Generator.integers(|avail|) by the group's lane 0
        Pcg64 rng;
        rng.sh = (uint64_t)word(4) | ((uint64_t)word(5) << 32);
        rng.sl = (uint64_t)word(6) | ((uint64_t)word(7) << 32);
        rng.ih = (uint64_t)word(8) | ((uint64_t)word(9) << 32);
        rng.il = (uint64_t)word(10) | ((uint64_t)word(11) << 32);
        rng.has = (int)word(19);
        rng.buf = word(20);
        int kk = 0;
        if (drew && gl == 0) {
            if (rings == 1) seed_frame(rng, P, g);  // first draw (after P0): the key's generator (search.py:125-128)
            kk = (int)pcg_integers(rng, (uint64_t)(kept - nua));
        }
        kk = __shfl_sync(FULL, kk, gb);
        // avail[kk]: 32 bit words per round, 4 per lane
        int apos = -1;
        {
            const int nw = drew ? (W + 31) >> 5 : 0;
            int rounds = (nw + 31) >> 5;
            rounds = __reduce_max_sync(FULL, rounds);
            int run = 0;
            for (int r = 0; r < rounds; r++) {
                const int w0 = r * 32 + gl * 4;
                uint32_t wd[4] = {0u, 0u, 0u, 0u};
                if (w0 < nw) {
                    const uint4 b4 = *reinterpret_cast<const uint4 *>(bq + (int64_t)w0 * 4);
                    wd[0] = b4.x;
                    wd[1] = b4.y;
                    wd[2] = b4.z;
                    wd[3] = b4.w;
                }
#pragma unroll
                for (int u = 0; u < BULK_U; u++) {
                    const int wu = (int)(up[u] >> 5) - w0;
                    if (u < nu && wu >= 0 && wu < 4) {
#pragma unroll
                        for (int x = 0; x < 4; x++)
                            if (x == wu) wd[x] &= ~(1u << (up[u] & 31));
                    }
                }
                const int c = __popc(wd[0]) + __popc(wd[1]) + __popc(wd[2]) + __popc(wd[3]);
                int inc = c;
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    const int t = __shfl_up_sync(FULL, inc, o);
                    if (gl >= o) inc += t;
                }
                const int tot = __shfl_sync(FULL, inc, gb | 7);
                const int ex = run + inc - c;
                if (apos < 0 && kk >= ex && kk < ex + c) {
                    int kr = kk - ex, xs = 0, ks = 0;
                    uint32_t ws = 0;
#pragma unroll
                    for (int x = 0; x < 4; x++) {
                        const int cx = __popc(wd[x]);
                        if (kr >= 0 && kr < cx) {
                            ws = wd[x];
                            xs = x;
                            ks = kr;
                        }
                        kr -= cx;
                    }
#ifdef RIANN_DRAW_FNS
                    apos = (w0 + xs) * 32 + (int)__fns(ws, 0u, ks + 1);
#else
                    apos = (w0 + xs) * 32 + nth_bit(ws, ks);
#endif
                }
                run += tot;
            }
            // broadcast within the group
            const unsigned bal = __ballot_sync(FULL, apos >= 0) & (0xffu << gb);
            apos = __shfl_sync(FULL, apos, bal ? __ffs(bal) - 1 : gb);
            if (!drew) apos = -1;
        }
        int an = 0;
        if (drew && gl == 0) {
            RB_CHECK(apos >= 0 && apos < W && soff + W <= P.pool_cap, 30);
            an = (int)P.pool[soff + apos];
            RB_CHECK(an >= 0 && an < P.n && nu < BULK_U, 31);
        }
        an = __shfl_sync(FULL, an, gb);
        // active list slots: one atomic per warp for its (up to four) drawing queries
        const unsigned act_m = __ballot_sync(FULL, has && gl == 0 && drew);
        int act_base = 0;
        if (lane == 0 && act_m) act_base = atomicAdd(P.n_active_out, __popc(act_m));
        act_base = __shfl_sync(FULL, act_base, 0);
        if (has && gl == 0) {
            sp->tests += cS;
            sp->rings = rings;
            P.kept[g] = 0;
            int status = ST_DONE;
            if (kept > 0) {
                sp->cS = kept;
                sp->sel = cur ^ 1;
            }
            if (drew) {
                sp->exact += 1;
                sp->anchor = an;
                sp->up[nu] = (uint16_t)apos;
                sp->nu = nu + 1;
                rng_store(*sp, rng);
                status = ST_ACTIVE;
                P.active_out[act_base + __popc(act_m & lanemask_lt())] = (int32_t)g;
                atomicAdd(P.counts + an, 1);  // grouping by anchor for the next phase
            } else if (want) {
                status = ST_HEAVY;
                P.heavy[atomicAdd(P.n_heavy, 1)] = (int32_t)g;
            }
            sp->status = status;
        }
    }
}

// ---------------------------------------------------------------------------
// Ring phase window (search.py:131-133), after grouping: for the active
// queries in anchor order (four per warp, eight lanes each) the exact d_a and
// the window [lo, hi) on the anchor's sorted row, written into the queries'
// descriptors.  Consecutive queries share their anchor, so its reference row,
// level-1 and coarse entries are served by L1.
template <int D>
__global__ void __launch_bounds__(256, RIANN_WIN_MINB) bulk_window_kernel(BulkParams P)
{
    const int lane = threadIdx.x & 31, gl = lane & 7, gb = lane & ~7;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int m = *P.n_active_in;
    for (int64_t ib = gwarp * 4; ib < m; ib += nwarps * 4) {
        const int64_t i = ib + (lane >> 3);
        const bool has = i < m;
        int4 d = has ? P.gdesc[i] : make_int4(0, 0, 0, 0);
        const int64_t g = has ? d.x : 0;
        int a = 0;
        if (has && gl == 0) a = P.st[g].anchor;
        a = __shfl_sync(FULL, a, gb);
        float qv[D / 8];
        load_qv8<D>(P.units + g * D, qv, gl);
        int lo, hi;
        dist_window8<D>(P, a, qv, has, gl, gb, lo, hi);
        if (has && gl == 0) {
            RB_CHECK(a >= 0 && a < P.n && lo >= 0 && lo <= hi && hi <= P.n, 40);
            d.z = (d.z & ~0x1ffff) | lo;
            d.w = (d.w & ~0x1ffff) | hi;
            P.gdesc[i] = d;
        }
    }
}

// ---------------------------------------------------------------------------
// F: final scan of S u {prev} for every light query (status DONE).
//
// Screening in the references' PCA basis: q' = T^T q (proj_kernel, fp32 FMA
// fp32) and r' = fp16(T^T r) (per-row bound e16p[r]).  For T with
// ||T^T T - I|| <= eta, the true distance d = ||q - r|| satisfies
//   (||q' - r'|| - dq - e16p[r]) / (1 + eta) <= d <= (||q' - r'|| + dq + e16p[r]) / (1 - eta)
// (dq bounds the GEMM rounding error, any order).  Partial sums of squares over the
// leading 16-component chunks are lower bounds of the full sum, so a candidate
// is abandoned as soon as its partial lower bound exceeds the best upper bound
// (initially the previous match's exact distance).  Survivors of all chunks
// whose lower bound can still reach the minimum get the exact FP64 distance
// (numpy order), so the first minimum (lowest index on ties) is exact.
// refs_pca16 is chunk-major: the 16-component chunk c of reference j is the
// 32 bytes at (c * n + j) * 16 halves, so chunk 0 of all references (the
// chunk every candidate is screened with) is one dense n * 32-byte block
// that stays L2-resident.
#ifndef RIANN_PCA_CHUNKMAJOR
#define RIANN_PCA_CHUNKMAJOR 1
#endif
__host__ __device__ __forceinline__ int64_t pca_chunk_off(int64_t j, int c, int64_t n, int D)
{
#if RIANN_PCA_CHUNKMAJOR
    (void)D;
    return ((int64_t)c * n + j) * 16;
#else
    (void)n;
    return j * D + 16 * c;
#endif
}

struct ScreenParams {
    const __half *refs_pca16;  // (n, D) fp16, PCA order, chunk-major (pca_chunk_off)
    const float *e16p;         // per-row bound
    const float *units_pca;    // (Q, D) fp32
    float slack;               // dq + max_r e16p[r] + 1e-12 (chunk rejection)
    float dq;                  // + 1e-12
    float one_plus_eta, one_minus_eta;
};

constexpr int FB = RIANN_FINAL_FB;  // candidates per screening block
#ifndef RIANN_FINAL_U16
#define RIANN_FINAL_U16 1
#endif
using FIdx = std::conditional_t<RIANN_FINAL_U16 != 0, uint16_t, uint32_t>;  // candidate index in the final scan (n <= 65,536)
constexpr int FSURV = 128;
__host__ __device__ constexpr size_t final_warp_bytes() { return (size_t)FB * (8 + 2 * sizeof(FIdx)) + FSURV * 8; }

template <int D>
__global__ void __launch_bounds__(256, RIANN_FINAL_MINB) bulk_final_kernel(BulkParams P, ScreenParams SP)
{
    constexpr int GX = Lay<D>::G;
    constexpr int NGX = WARP / GX;
    constexpr int NCH = D / 16;
    constexpr int SURV_CAP = FSURV;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    // per warp: two (index, partial) lists of FB entries + survivor slots
    // per warp: partial sums As/Bs (f32), candidate lists Aj/Bj (FIdx), survivors
    unsigned char *ws = smem_raw + (size_t)wib * final_warp_bytes();
    float *As = reinterpret_cast<float *>(ws);
    float *Bs = reinterpret_cast<float *>(ws + FB * 4);
    FIdx *Aj = reinterpret_cast<FIdx *>(ws + FB * 8);
    FIdx *Bj = reinterpret_cast<FIdx *>(ws + FB * 8 + FB * sizeof(FIdx));
    uint32_t *sv_j = reinterpret_cast<uint32_t *>(ws + FB * (8 + 2 * sizeof(FIdx)));
    float *sv_lb = reinterpret_cast<float *>(ws + FB * (8 + 2 * sizeof(FIdx)) + SURV_CAP * 4);
    const int64_t nwarps = (int64_t)gridDim.x * wpb;
    const uint64_t pol_keep = pol_evict_last();
#ifndef RIANN_FINAL_LIST_ONCE
#define RIANN_FINAL_LIST_ONCE 1
#endif
#if RIANN_FINAL_LIST_ONCE
    const uint64_t pol_once = pol_evict_first();
#endif
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
        const uint8_t *bq = (sr.sel ? P.bits1 : P.bits0) + (sr.s_off >> 3);
        const int Wl = sr.lenA8 + sr.lenB8;
        const bool p_in = sr.pin_pos >= 0 && bit_at(bq, sr.pin_pos);
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
        for (int lp = 0; lp < Wl;) {
            // S = the alive list entries: up to FB of them into Bj's space
            FIdx *Cj = Bj;
            int bn = 0;
            while (lp < Wl && bn <= FB - FSEG) {
                const int e0 = lp + lane * 8;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                uint32_t al = 0;
                if (e0 < Wl) {
#if RIANN_FINAL_LIST_ONCE
                    v = ld_once16(reinterpret_cast<const uint4 *>(slot + e0), pol_once);
#else
                    v = *reinterpret_cast<const uint4 *>(slot + e0);
#endif
                    al = bq[e0 >> 3];
                }
                const int c = __popc(al);
                const int inc = warp_incl_scan(c, lane);
                int o = bn + inc - c;
                const uint16_t *e8 = reinterpret_cast<const uint16_t *>(&v);
#pragma unroll
                for (int x = 0; x < 8; x++)
                    if ((al >> x) & 1u) Cj[o++] = e8[x];
                bn += __shfl_sync(FULL, inc, 31);
                RB_CHECK(bn <= FB, 50);
                lp += FSEG;
            }
            __syncwarp();
            // chunk 0 over the block: a lane per candidate, one 32-byte load each
            // (one L1 wavefront per candidate); later chunks: a lane pair per
            // survivor, each lane one 16-byte half of the 32-byte chunk
            const int hh = lane & 1;
            const unsigned EVEN = 0x55555555u;
            auto part = [&](const uint4 &v, const float (&qc)[8]) {
                float s = 0.f;
                const __half2 *h2 = reinterpret_cast<const __half2 *>(&v);
#pragma unroll
                for (int x = 0; x < 4; x++) {
                    const float2 f = __half22float2(h2[x]);
                    const float a0 = __fsub_rn(f.x, qc[2 * x]), a1 = __fsub_rn(f.y, qc[2 * x + 1]);
                    s = __fmaf_rn(a0, a0, s);
                    s = __fmaf_rn(a1, a1, s);
                }
                return __fadd_rn(s, __shfl_xor_sync(FULL, s, 1));
            };
            int nA = 0;
            {
                float q0[16];
                {
                    const float4 *q4 = reinterpret_cast<const float4 *>(qp);
#pragma unroll
                    for (int x = 0; x < 4; x++) {
                        const float4 t = __ldg(q4 + x);
                        q0[4 * x] = t.x; q0[4 * x + 1] = t.y; q0[4 * x + 2] = t.z; q0[4 * x + 3] = t.w;
                    }
                }
                auto part16 = [&](const uint4 &va, const uint4 &vb) {
                    float s = 0.f;
                    const __half2 *ha = reinterpret_cast<const __half2 *>(&va);
                    const __half2 *hb = reinterpret_cast<const __half2 *>(&vb);
#pragma unroll
                    for (int x = 0; x < 4; x++) {
                        const float2 f = __half22float2(ha[x]);
                        const float a0 = __fsub_rn(f.x, q0[2 * x]), a1 = __fsub_rn(f.y, q0[2 * x + 1]);
                        s = __fmaf_rn(a0, a0, s);
                        s = __fmaf_rn(a1, a1, s);
                    }
#pragma unroll
                    for (int x = 0; x < 4; x++) {
                        const float2 f = __half22float2(hb[x]);
                        const float a0 = __fsub_rn(f.x, q0[8 + 2 * x]), a1 = __fsub_rn(f.y, q0[8 + 2 * x + 1]);
                        s = __fmaf_rn(a0, a0, s);
                        s = __fmaf_rn(a1, a1, s);
                    }
                    return s;
                };
                // FU rounds of 32 candidates per iteration, their loads issued together
#ifndef RIANN_FINAL_FU
#define RIANN_FINAL_FU 2
#endif
                constexpr int FU = RIANN_FINAL_FU;
                for (int e0 = 0; e0 < bn; e0 += 32 * FU) {
                    uint4 va[FU], vb[FU];
                    uint32_t jj[FU];
#pragma unroll
                    for (int u = 0; u < FU; u++) {
                        const int e = e0 + 32 * u + lane;
                        jj[u] = Cj[e < bn ? e : 0];
                        ld_keep32(SP.refs_pca16 + pca_chunk_off(jj[u], 0, P.n, D), pol_keep, va[u], vb[u]);
                    }
#pragma unroll
                    for (int u = 0; u < FU; u++) {
                        const int e = e0 + 32 * u + lane;
                        const float s = part16(va[u], vb[u]);
                        const bool keep = e < bn && s <= thr;
                        const unsigned ball = __ballot_sync(FULL, keep);
                        if (keep) {
                            const int o = nA + __popc(ball & lanemask_lt());
                            Aj[o] = jj[u];
                            As[o] = s;
                        }
                        nA += __popc(ball);
                    }
                }
            }
            __syncwarp();
            // further chunks for the candidates still alive, FCW chunks per step
            // (partial sums only grow: one test after the step's last chunk)
#ifndef RIANN_FINAL_CW
#define RIANN_FINAL_CW 2
#endif
            constexpr int FCW = RIANN_FINAL_CW;
            for (int c = 1; c < NCH && nA > 0; c += FCW) {
                const int cn = min(FCW, NCH - c);
                float qcs[FCW][8];
#pragma unroll
                for (int k = 0; k < FCW; k++) {
                    if (k < cn) {
                        const float4 *q4 = reinterpret_cast<const float4 *>(qp + 16 * (c + k)) + 2 * hh;
                        const float4 va = __ldg(q4), vb = __ldg(q4 + 1);
                        qcs[k][0] = va.x; qcs[k][1] = va.y; qcs[k][2] = va.z; qcs[k][3] = va.w;
                        qcs[k][4] = vb.x; qcs[k][5] = vb.y; qcs[k][6] = vb.z; qcs[k][7] = vb.w;
                    }
                }
                const bool last = c + cn == NCH;
                int nB = 0;
                for (int i0 = 0; i0 < nA; i0 += 16) {
                    const int i = i0 + (lane >> 1);
                    const bool valid = i < nA;
                    const uint32_t j = valid ? Aj[i] : Aj[0];
                    const float s0 = valid ? As[i] : 0.f;
                    uint4 v[FCW];
#pragma unroll
                    for (int k = 0; k < FCW; k++)
                        if (k < cn)
                            v[k] = ld_keep16(
                                reinterpret_cast<const uint4 *>(SP.refs_pca16 + pca_chunk_off(j, c + k, P.n, D)) + hh, pol_keep);
                    float s = s0;
#pragma unroll
                    for (int k = 0; k < FCW; k++)
                        if (k < cn) s = __fadd_rn(s, part(v[k], qcs[k]));
                    if (!last) {
                        const bool keep = valid && s <= thr;
                        const unsigned ball = __ballot_sync(FULL, keep) & EVEN;
                        if (keep && hh == 0) {
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
                        const unsigned ball = __ballot_sync(FULL, surv) & EVEN;
                        const int add = __popc(ball);
                        if (nsv + add > SURV_CAP) flush();
                        if (surv && hh == 0) {
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
                    FIdx *tj = Aj;
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
        RB_CHECK(bi >= 0 && bi < P.n && sr.s_off + Wl <= P.pool_cap && sr.pin_pos < Wl, 51);
        const int nscan = cS + (p_in ? 0 : 1);
        if (lane == 0) {
            P.out_idx[g] = bi;
            P.out_dist[g] = bd;
            P.st[g].status = ST_FINISHED;  // later passes (pool-sized query batches) skip it
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
        out[(dim % 16 == 0) ? pca_chunk_off(j, i >> 4, n, dim) + (i & 15) : j * dim + i] = h;
        const double dl = (double)__half2float(h) - y;
        acc = __fma_ru(dl, dl, acc);
    }
    // + dim * 1e-15 covers the float64 evaluation error of y
    const float b = __double2float_ru(__dsqrt_ru(acc) + 1e-13);
    e16[j] = b;
    atomicMax(e16max, __float_as_uint(b));
}

// ---------------------------------------------------------------------------
// Exclusive scan of the per-anchor counts (n + 1 ints) into starts, counts
// zeroed for the scatter's cursors: one CTA of 1024 threads, each owning a
// contiguous run (coalesced through shared memory), a warp-shuffle scan of
// the run totals.  Replaces a library scan + memset (two launches) per ring
// phase.
constexpr int SCAN_T = 1024;
constexpr int SCAN_E = 68;  // counts per thread of the one-pass scan: 1,024 x 68 >= 65,536 + 1
__global__ void __launch_bounds__(SCAN_T) anchor_scan_kernel(int32_t *counts, int32_t *starts, int m)
{
    __shared__ int32_t wsum[SCAN_T / 32];
    __shared__ int32_t carry_s;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) carry_s = 0;
    __syncthreads();
    // m <= SCAN_T * SCAN_E (every bulk-path n): a thread owns `per` contiguous counts
    // (a multiple of 4): one round of independent loads for the thread sums, one
    // block scan, a second round (cache hits) for the prefix and the stores
    if (m <= SCAN_T * SCAN_E) {
        const int per = (((m + SCAN_T - 1) / SCAN_T) + 3) & ~3;
        const int i0 = tid * per;
        auto ld4 = [&](int i) {
            int4 v = make_int4(0, 0, 0, 0);
            if (i + 3 < m) {
                v = *reinterpret_cast<const int4 *>(counts + i);
            } else if (i < m) {
                v.x = counts[i];
                if (i + 1 < m) v.y = counts[i + 1];
                if (i + 2 < m) v.z = counts[i + 2];
            }
            return v;
        };
        int tsum = 0;
#pragma unroll 17
        for (int k = 0; k < per; k += 4) {
            const int4 v = ld4(i0 + k);
            tsum += v.x + v.y + v.z + v.w;
        }
        int inc = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        if (w == 0) {
            const int x = wsum[lane];
            int xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            wsum[lane] = xi - x;  // exclusive warp offsets
        }
        __syncthreads();
        int run = wsum[w] + inc - tsum;
#pragma unroll 4
        for (int k = 0; k < per; k += 4) {
            const int i = i0 + k;
            if (i >= m) break;
            const int4 v = ld4(i);
            int4 o4;
            o4.x = run;
            o4.y = o4.x + v.x;
            o4.z = o4.y + v.y;
            o4.w = o4.z + v.z;
            run = o4.w + v.w;
            if (i + 3 < m) {
                *reinterpret_cast<int4 *>(starts + i) = o4;
                *reinterpret_cast<int4 *>(counts + i) = make_int4(0, 0, 0, 0);
            } else {
                starts[i] = o4.x;
                counts[i] = 0;
                if (i + 1 < m) { starts[i + 1] = o4.y; counts[i + 1] = 0; }
                if (i + 2 < m) { starts[i + 2] = o4.z; counts[i + 2] = 0; }
            }
        }
        return;
    }
    // tiles of SCAN_T * 4 elements, int4-coalesced per thread
    for (int base = 0; base < m; base += SCAN_T * 4) {
        int v[4];
        const int i0 = base + tid * 4;
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = (i0 + k < m) ? counts[i0 + k] : 0;
        const int tsum = v[0] + v[1] + v[2] + v[3];
        int inc = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        if (w == 0) {
            int x = wsum[lane];
            int xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            wsum[lane] = xi - x;  // exclusive warp offsets
        }
        __syncthreads();
        int run = carry_s + wsum[w] + inc - tsum;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (i0 + k < m) {
                starts[i0 + k] = run;
                counts[i0 + k] = 0;
            }
            run += v[k];
        }
        __syncthreads();
        if (tid == SCAN_T - 1) carry_s = run;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Final-scan projection q' = T^T q (T: D x D, T[k][i] = entry k of basis
// vector i) for every unit row: a register-tiled SIMT GEMM with fp32 FMAs.
// Each CTA owns PQ queries x all D outputs; K staged through shared memory in
// chunks of PK.  Any summation order keeps the screening bound dq
// (gamma_D * sqrt(D) * ||q||, build_pca) valid.
#ifndef RIANN_PROJ_PQ
#define RIANN_PROJ_PQ 64
#endif
#ifndef RIANN_PROJ_TM
#define RIANN_PROJ_TM 8
#endif
template <int D>
struct ProjCfg {
    static constexpr int PQ = RIANN_PROJ_PQ;    // queries per CTA
    static constexpr int TM = RIANN_PROJ_TM;    // queries per thread
    static constexpr int TN = D == 192 ? 12 : 4;  // outputs per thread
    static constexpr int THREADS = (PQ / TM) * (D / TN);
    static constexpr int PK = 32;               // k per stage
};

template <int D>
__global__ void __launch_bounds__(ProjCfg<D>::THREADS) proj_kernel(const float *__restrict__ units,
                                                                   const float *__restrict__ T, int64_t Q,
                                                                   float *__restrict__ out)
{
    using CF = ProjCfg<D>;
    constexpr int PQ = CF::PQ, TM = CF::TM, TN = CF::TN, PK = CF::PK, NT = CF::THREADS;
    constexpr int TX = D / TN;  // threads along the outputs
    __shared__ __align__(16) float us[PK][PQ + 4];  // us[k][q]
    __shared__ __align__(16) float ts[PK][D];       // ts[k][i]
    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    for (int64_t q0 = (int64_t)blockIdx.x * PQ; q0 < Q; q0 += (int64_t)gridDim.x * PQ) {
        float acc[TM][TN];
#pragma unroll
        for (int a = 0; a < TM; a++)
#pragma unroll
            for (int b = 0; b < TN; b++) acc[a][b] = 0.f;
        for (int k0 = 0; k0 < D; k0 += PK) {
            __syncthreads();
            // unit tile: PQ rows x PK columns (float4 along k), stored transposed
            for (int e = tid; e < PQ * PK / 4; e += NT) {
                const int qq = e / (PK / 4), kk = (e % (PK / 4)) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (q0 + qq < Q) v = *reinterpret_cast<const float4 *>(units + (q0 + qq) * D + k0 + kk);
                us[kk + 0][qq] = v.x;
                us[kk + 1][qq] = v.y;
                us[kk + 2][qq] = v.z;
                us[kk + 3][qq] = v.w;
            }
            for (int e = tid; e < PK * D / 4; e += NT) {
                const int kk = e / (D / 4), ii = (e % (D / 4)) * 4;
                *reinterpret_cast<float4 *>(&ts[kk][ii]) =
                    *reinterpret_cast<const float4 *>(T + (int64_t)(k0 + kk) * D + ii);
            }
            __syncthreads();
#pragma unroll 4
            for (int k = 0; k < PK; k++) {
                float a[TM], b[TN];
#pragma unroll
                for (int x = 0; x < TM; x += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(&us[k][ty * TM + x]);
                    a[x] = v.x;
                    a[x + 1] = v.y;
                    a[x + 2] = v.z;
                    a[x + 3] = v.w;
                }
#pragma unroll
                for (int x = 0; x < TN; x += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(&ts[k][tx * TN + x]);
                    b[x] = v.x;
                    b[x + 1] = v.y;
                    b[x + 2] = v.z;
                    b[x + 3] = v.w;
                }
#pragma unroll
                for (int i = 0; i < TM; i++)
#pragma unroll
                    for (int j = 0; j < TN; j++) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
            }
        }
#pragma unroll
        for (int i = 0; i < TM; i++) {
            const int64_t q = q0 + ty * TM + i;
            if (q < Q) {
#pragma unroll
                for (int x = 0; x < TN; x += 4)
                    *reinterpret_cast<float4 *>(out + q * D + tx * TN + x) =
                        make_float4(acc[i][x], acc[i][x + 1], acc[i][x + 2], acc[i][x + 3]);
            }
        }
    }
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

// level-1 index of the coarse rows: 32 entries per row, +inf past the row
__global__ void coarse1_kernel(const float *coarse, int64_t n, int nb, int cs1, float *c1)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 32) return;
    int64_t a = i >> 5;
    int k = (int)(i & 31);
    c1[i] = (int64_t)k * cs1 < nb ? coarse[a * nb + (int64_t)k * cs1] : __int_as_float(0x7f800000);
}

}  // namespace rb

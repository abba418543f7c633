// riann_device.cuh -- device building blocks shared by the RIANN kernels.
//
// Bit-exactness contract (SURVEY.md §7 "hard parts" 1-2): every float64
// operation below is an explicitly rounded IEEE op (__dadd_rn/__dsub_rn/
// __dmul_rn/__ddiv_rn/__dsqrt_rn), never contracted into FMA, and sums follow
// numpy's pairwise order, so results equal the reference's numpy results bit
// for bit.  The RNG reproduces numpy's SeedSequence -> PCG64 ->
// Generator.integers chain (search.py:125-129).
#pragma once

#include <cstdint>

namespace rb {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARP = 32;

// ---------------------------------------------------------------------------
// numpy float64 pairwise summation over get(i), i in [s, s+n).
// (numpy: n < 8 sequential from 0.0; n <= 128: 8 accumulators + tree +
//  sequential tail; else split at n/2 rounded down to a multiple of 8.)
template <class G>
__device__ __forceinline__ double pw_block(const G &get, int64_t s, int64_t n)
{
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r = __dadd_rn(r, get(s + i));
        return r;
    }
    double r0 = get(s + 0), r1 = get(s + 1), r2 = get(s + 2), r3 = get(s + 3);
    double r4 = get(s + 4), r5 = get(s + 5), r6 = get(s + 6), r7 = get(s + 7);
    int64_t i = 8;
    for (; i < n - (n & 7); i += 8) {
        r0 = __dadd_rn(r0, get(s + i + 0));
        r1 = __dadd_rn(r1, get(s + i + 1));
        r2 = __dadd_rn(r2, get(s + i + 2));
        r3 = __dadd_rn(r3, get(s + i + 3));
        r4 = __dadd_rn(r4, get(s + i + 4));
        r5 = __dadd_rn(r5, get(s + i + 5));
        r6 = __dadd_rn(r6, get(s + i + 6));
        r7 = __dadd_rn(r7, get(s + i + 7));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < n; i++) res = __dadd_rn(res, get(s + i));
    return res;
}

// General n: explicit-stack version of numpy's recursion (depth <= 24).
template <class G>
__device__ double pw_sum(const G &get, int64_t s, int64_t n)
{
    if (n <= 128) return pw_block(get, s, n);
    int64_t st_s[24], st_n[24];
    double st_left[24];
    int st_state[24];
    int sp = 0;
    st_s[0] = s;
    st_n[0] = n;
    st_state[0] = 0;
    double ret = 0.0;
    for (;;) {
        int64_t cs = st_s[sp], cn = st_n[sp];
        if (cn <= 128) {
            ret = pw_block(get, cs, cn);
            // pop and deliver
            for (;;) {
                if (sp == 0) return ret;
                sp--;
                if (st_state[sp] == 0) {  // left finished -> do right
                    st_left[sp] = ret;
                    st_state[sp] = 1;
                    int64_t h = st_n[sp] / 2;
                    h -= h % 8;
                    sp++;
                    st_s[sp] = st_s[sp - 1] + h;
                    st_n[sp] = st_n[sp - 1] - h;
                    st_state[sp] = 0;
                    break;
                } else {
                    ret = __dadd_rn(st_left[sp], ret);
                }
            }
        } else {
            int64_t h = cn / 2;
            h -= h % 8;
            sp++;
            st_s[sp] = cs;
            st_n[sp] = h;
            st_state[sp] = 0;
        }
    }
}

__device__ __forceinline__ double sqdiff(float r, float q)
{
    double d = __dsub_rn((double)r, (double)q);
    return __dmul_rn(d, d);
}

// Exact distance by one thread, generic dim (patches.py:151-159).
struct SqDiffGet {
    const float *r, *q;
    __device__ double operator()(int64_t i) const { return sqdiff(r[i], q[i]); }
};
__device__ __forceinline__ double dist_thread(const float *r, const float *q, int dim)
{
    SqDiffGet g{r, q};
    return __dsqrt_rn(pw_sum(g, 0, dim));
}

// ---------------------------------------------------------------------------
// Warp-cooperative exact distance for dims where numpy's pairwise tree maps
// onto lanes: D%8==0 && D<=128 -> 8-lane groups (lane j = accumulator j);
// 128<D<=256 && D%16==0 -> 16-lane groups (two 8-accumulator halves).
// Lane (gl) of a group sums elements h*D/2 + 8i + j sequentially, then the
// xor-shuffles reproduce ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and half0+half1.
template <int D>
struct Lay {
    static constexpr bool fast = (D % 8 == 0 && D >= 8 && D <= 128) || (D > 128 && D <= 256 && D % 16 == 0);
    static constexpr int G = D <= 128 ? 8 : 16;
    static constexpr int PER = D / G;
    static constexpr int NG = WARP / G;  // groups per warp
    __device__ static __forceinline__ int base(int gl)
    {
        return (G == 16 ? (gl >> 3) * (D / 2) : 0) + (gl & 7);
    }
};

template <int D>
__device__ __forceinline__ double group_dist(const float *__restrict__ row, const float (&qv)[Lay<D>::PER], int gl)
{
    const float *p = row + Lay<D>::base(gl);
    double r = sqdiff(__ldg(p), qv[0]);
#pragma unroll
    for (int i = 1; i < Lay<D>::PER; i++) r = __dadd_rn(r, sqdiff(__ldg(p + 8 * i), qv[i]));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
    if (Lay<D>::G == 16) r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 8));
    return __dsqrt_rn(r);
}

// ---------------------------------------------------------------------------
// numpy SeedSequence(pool 4) -> PCG64 -> Generator.integers (32-bit Lemire).
struct Pcg64 {
    uint64_t sh, sl, ih, il;
    uint32_t buf;
    int has;
};

constexpr uint64_t PCG_MH = 2549297995355413924ULL;
constexpr uint64_t PCG_ML = 4865540595714422341ULL;

__device__ __forceinline__ void pcg_step(Pcg64 &g)
{
    uint64_t lo = g.sl * PCG_ML;
    uint64_t hi = __umul64hi(g.sl, PCG_ML) + g.sh * PCG_ML + g.sl * PCG_MH;
    uint64_t lo2 = lo + g.il;
    hi += g.ih + (lo2 < lo ? 1ull : 0ull);
    g.sl = lo2;
    g.sh = hi;
}

__device__ __forceinline__ uint32_t ss_hash(uint32_t v, uint32_t &hc)
{
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
}

__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y)
{
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
}

// words(i) -> i-th entropy word, i < nw
template <class W>
__device__ void pcg_seed(Pcg64 &g, const W &words, int nw)
{
    uint32_t pool[4];
    uint32_t hc = 0x43b0d7e5u;
#pragma unroll
    for (int i = 0; i < 4; i++) pool[i] = ss_hash(i < nw ? words(i) : 0u, hc);
#pragma unroll
    for (int s = 0; s < 4; s++)
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hash(pool[s], hc));
    for (int s = 4; s < nw; s++) {
        uint32_t w = words(s);
#pragma unroll
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hash(w, hc));
    }
    uint32_t st[8];
    uint32_t hb = 0x8b51f9ddu;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= 0x58f38dedu;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    uint64_t w0 = st[0] | ((uint64_t)st[1] << 32), w1 = st[2] | ((uint64_t)st[3] << 32);
    uint64_t w2 = st[4] | ((uint64_t)st[5] << 32), w3 = st[6] | ((uint64_t)st[7] << 32);
    // inc = (initseq << 1) | 1, initseq = (w2:w3)
    g.ih = (w2 << 1) | (w3 >> 63);
    g.il = (w3 << 1) | 1ull;
    g.sh = 0;
    g.sl = 0;
    pcg_step(g);
    uint64_t lo = g.sl + w1;
    g.sh = g.sh + w0 + (lo < g.sl ? 1ull : 0ull);
    g.sl = lo;
    pcg_step(g);
    g.has = 0;
    g.buf = 0;
}

__device__ __forceinline__ uint64_t pcg_next64(Pcg64 &g)
{
    pcg_step(g);
    uint64_t x = g.sh ^ g.sl;
    unsigned rot = (unsigned)(g.sh >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint32_t pcg_next32(Pcg64 &g)
{
    if (g.has) {
        g.has = 0;
        return g.buf;
    }
    uint64_t v = pcg_next64(g);
    g.has = 1;
    g.buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

// Generator.integers(k), 1 <= k <= 2^32; k == 1 consumes nothing.
__device__ __forceinline__ uint64_t pcg_integers(Pcg64 &g, uint64_t k)
{
    uint64_t rng = k - 1;
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFull) return pcg_next32(g);
    uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (0xFFFFFFFFu - (uint32_t)rng) % excl;
        while (left < thr) {
            m = (uint64_t)pcg_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return m >> 32;
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// lexicographic (distance, index) minimum: ties resolve to the lowest index
// (np.argmin over an ascending scan, search.py:143 / evaluation.py:32).
__device__ __forceinline__ void argmin_merge(double &bd, int &bi, double od, int oi)
{
    if (od < bd || (od == bd && oi < bi)) {
        bd = od;
        bi = oi;
    }
}

__device__ __forceinline__ void warp_argmin(double &bd, int &bi)
{
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        double od = __shfl_xor_sync(FULL, bd, o);
        int oi = __shfl_xor_sync(FULL, bi, o);
        argmin_merge(bd, bi, od, oi);
    }
}

}  // namespace rb

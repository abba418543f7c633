// riann_exact_tc.cuh -- K4: exact nearest reference (evaluation.py:24-50) with
// the distance screen on the 5th-generation tensor cores.
//
//   ||q - r||^2 = ||q'||^2 + ||r'||^2 - 2 q'.r' on operands centred on the
//   reference mean (q' = q - c, r' = r - c), with q'.r' from one tcgen05 GEMM
//   over K = 3D bf16 columns: A = [q'_hi, q'_hi, q'_lo], B = [r'_hi, r'_lo,
//   r'_hi] (x_hi = bf16(x), x_lo = bf16(x - x_hi)), fp32 accumulation in TMEM.
//
// Warp roles per CTA (one 128-query M tile, all N tiles of 128 references):
//   warp 0  TMA producer (A and B K-blocks, 128B swizzle, 4-stage ring)
//   warp 1  MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M=128 N=128 K=16)
//   warp 2  TMEM allocator
//   warps 4-7 epilogue: tcgen05.ld of the accumulator (double-buffered in
//           TMEM), rigorous bounds, per-query running best upper bound and a
//           short list of candidates whose lower bound can still reach it.
// A second kernel re-evaluates the candidates with the exact float64 distance
// in numpy's order (first minimum, lowest index on ties); queries whose list
// overflowed take the exact full scan.  The screen only decides which
// candidates get the exact distance, so results are bit-identical.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "riann_kernels.cuh"

namespace rb {
namespace tc {

constexpr int BM = 128, BN = 128, BK = 64;  // BK bf16 = 128 bytes per row (one swizzle atom)
constexpr int STAGES = 4;
constexpr int A_BLOCK = BM * BK * 2;             // 16 KB: one K-block of the resident query tile
constexpr int STAGE_BYTES = BN * BK * 2;         // 16 KB: one K-block of a reference tile
constexpr int MAX_KB = 9;                        // 3D / BK for D = 192
__host__ __device__ constexpr int smem_bytes(int kb) { return kb * A_BLOCK + STAGES * STAGE_BYTES + 1024; }
constexpr int NCAND = 16;                      // candidates kept per query
constexpr int EPI_WARP0 = 4;

struct ExactParams {
    const float *nq;       // (m) ||q - c||^2 (float64 sum rounded to float)
    const float *nr;       // (n) ||r - c||^2
    int64_t m, n;
    int kblocks;           // 3D / BK
    float eps;             // |d2_est - d2| <= eps * (nq + nr)  (see exact_eps)
    int32_t *cand;         // (m, NCAND)
    float *cand_lb;        // (m, NCAND)
    int32_t *ncand;        // (m): count, or -1 on overflow
    float *best_ub;        // (m)
};

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t *b, unsigned c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c));
}
__device__ __forceinline__ void bar_expect(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            saddr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(saddr(bar))
        : "memory");
}

// K-major operand, 128B swizzle, rows of 128 bytes, 8-row groups 1024 bytes apart
__device__ __forceinline__ uint64_t smem_desc(const void *p)
{
    const uint64_t addr = saddr(p);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;        // start address
    d |= (uint64_t)1 << 16;               // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;     // stride byte offset: next 8-row group
    d |= (uint64_t)1 << 46;               // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;               // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, both K-major
__host__ __device__ constexpr uint32_t instr_desc(int M, int N)
{
    return (1u << 4)                      // D format F32
           | (1u << 7)                    // A format BF16
           | (1u << 10)                   // B format BF16
           | ((uint32_t)(N >> 3) << 17)   // N / 8
           | ((uint32_t)(M >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(256, 1) exact_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                                                           const __grid_constant__ CUtensorMap mapB, ExactParams P)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], acc_full[2], acc_empty[2], a_bar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int ntiles = (int)((P.n + BN - 1) / BN);
    const int kb = P.kblocks;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            bar_init(&full_bar[s], 1);
            bar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            bar_init(&acc_full[a], 1);
            bar_init(&acc_empty[a], 4);  // one arrive per epilogue warp
        }
        bar_init(&a_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                     "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;

    unsigned char *sA = smem;                    // kb resident K-blocks of the query tile
    unsigned char *sB = smem + kb * A_BLOCK;     // STAGES reference K-blocks
    if (warp == 0) {
        // ---- TMA producer
        if (lane == 0) {
            bar_expect(&a_bar, (unsigned)(kb * A_BLOCK));
            for (int k = 0; k < kb; k++) tma_load_2d(sA + k * A_BLOCK, &mapA, k * BK, (int)m0, &a_bar);
            int it = 0;
            for (int t = 0; t < ntiles; t++) {
                for (int k = 0; k < kb; k++, it++) {
                    const int s = it % STAGES;
                    if (it >= STAGES) bar_wait(&empty_bar[s], (unsigned)(((it / STAGES) - 1) & 1));
                    bar_expect(&full_bar[s], STAGE_BYTES);
                    tma_load_2d(sB + s * STAGE_BYTES, &mapB, k * BK, t * BN, &full_bar[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer
        const uint32_t idesc = instr_desc(BM, BN);
        bar_wait(&a_bar, 0);
        int it = 0;
        for (int t = 0; t < ntiles; t++) {
            const int acc = t & 1;
            if (t >= 2) bar_wait(&acc_empty[acc], (unsigned)(((t / 2) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tacc = tbase + (uint32_t)(acc * BN);
            for (int k = 0; k < kb; k++, it++) {
                const int s = it % STAGES;
                bar_wait(&full_bar[s], (unsigned)((it / STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint64_t da = smem_desc(sA + k * A_BLOCK), db = smem_desc(sB + s * STAGE_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++)  // 16 bf16 = 32 bytes per MMA step
                        mma_bf16(tacc, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc, (k | kk) ? 1u : 0u);
                    mma_commit(&empty_bar[s]);
                    if (k == kb - 1) mma_commit(&acc_full[acc]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ---- epilogue: thread owns query row r of the tile (TMEM lane r)
        const int q4 = warp - EPI_WARP0;  // TMEM lane quarter
        const int r = q4 * 32 + lane;
        const int64_t qi = m0 + r;
        const bool rowok = qi < P.m;
        const float nq = rowok ? P.nq[qi] : 0.f;
        // squared-distance space: u2 >= d^2 >= l2 for every reference
        float ub2 = __int_as_float(0x7f800000);
        int cnt = 0;
        int32_t cj[NCAND];
        float cl[NCAND];
        const float inf = __int_as_float(0x7f800000);
        // nr of the tile's 128 columns, 4 per lane (column c0 + x lives in lane x of nrv[c0 / 32])
        float nrv[BN / 32], nrn[BN / 32];
#pragma unroll
        for (int k = 0; k < BN / 32; k++) {
            const int64_t j = (int64_t)k * 32 + lane;
            nrv[k] = j < P.n ? __ldg(P.nr + j) : inf;
        }
        for (int t = 0; t < ntiles; t++) {
            const int acc = t & 1;
#pragma unroll
            for (int k = 0; k < BN / 32; k++) {  // prefetch the next tile's norms
                const int64_t j = (int64_t)(t + 1) * BN + k * 32 + lane;
                nrn[k] = j < P.n ? __ldg(P.nr + j) : inf;
            }
            bar_wait(&acc_full[acc], (unsigned)((t / 2) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int k = 0; k < BN / 32; k++) {
                uint32_t v[32];
                tmem_ld32(tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * BN + k * 32), v);
                float d2[32], e[32];
                float cmin = inf;
#pragma unroll
                for (int x = 0; x < 32; x++) {
                    const float s = __fadd_rn(nq, __shfl_sync(FULL, nrv[k], x));  // inf past n
                    d2[x] = __fmaf_rn(-2.f, __uint_as_float(v[x]), s);
                    e[x] = __fmul_ru(P.eps, s);
                    cmin = fminf(cmin, __fadd_ru(d2[x], e[x]));
                }
                ub2 = fminf(ub2, cmin);
                uint32_t mask = 0;
#pragma unroll
                for (int x = 0; x < 32; x++) mask |= (__fsub_rd(d2[x], e[x]) <= ub2 ? 1u : 0u) << x;
                if (!rowok) mask = 0;
                while (mask && cnt >= 0) {  // rare: candidates that can still win
                    const int x = __ffs(mask) - 1;
                    mask &= mask - 1;
                    float l2 = 0.f;
#pragma unroll
                    for (int y = 0; y < 32; y++)
                        if (y == x) l2 = __fsub_rd(d2[y], e[y]);
                    if (cnt == NCAND) {  // compact with the current bound
                        int w2 = 0;
#pragma unroll
                        for (int y = 0; y < NCAND; y++)
                            if (cl[y] <= ub2) {
                                cj[w2] = cj[y];
                                cl[w2] = cl[y];
                                w2++;
                            }
                        cnt = w2 == NCAND ? -1 : w2;  // -1: overflow, exact full scan
                    }
                    if (cnt >= 0) {
                        cj[cnt] = (int32_t)((int64_t)t * BN + k * 32 + x);
                        cl[cnt] = l2;
                        cnt++;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < BN / 32; k++) nrv[k] = nrn[k];
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive(&acc_empty[acc]);
        }
        if (rowok) {
            int w2 = 0;
            if (cnt >= 0) {
                for (int y = 0; y < cnt; y++)
                    if (cl[y] <= ub2) {
                        P.cand[qi * NCAND + w2] = cj[y];
                        P.cand_lb[qi * NCAND + w2] = cl[y];
                        w2++;
                    }
            }
            P.ncand[qi] = cnt >= 0 ? w2 : -1;
            P.best_ub[qi] = ub2;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(2 * BN));
}

// Operands are centred on the reference mean c before the split: distances
// are translation-invariant and the screen's error scales with |q-c| |r-c|
// (the patch spread) instead of |q| |r|.  v = fl(x - c) differs from x - c by
// at most 2^-24 |v| per component, which exact_eps covers.
// A rows: [v_hi, v_hi, v_lo], B rows: [v_hi, v_lo, v_hi];
// v_hi = bf16(v), v_lo = bf16(v - v_hi) (v - v_hi is exact in float).
__global__ void center_sum_kernel(const float *__restrict__ x, int64_t rows, int dim, double *__restrict__ acc)
{
    // block: dim threads (<= 256) over a chunk of 1024 rows
    const int e = threadIdx.x;
    if (e >= dim) return;
    const int64_t r0 = (int64_t)blockIdx.x * 1024, r1 = min(rows, r0 + 1024);
    double s = 0.0;
    for (int64_t r = r0; r < r1; r++) s += (double)x[r * dim + e];
    atomicAdd(acc + e, s);
}

__global__ void center_fin_kernel(const double *__restrict__ acc, int64_t rows, int dim, float *__restrict__ center)
{
    const int e = threadIdx.x;
    if (e < dim) center[e] = (float)(acc[e] / (double)rows);
}

__global__ void split_kernel(const float *__restrict__ x, const float *__restrict__ center, int64_t rows, int dim,
                             int a_side, __nv_bfloat16 *__restrict__ out)
{
    const int64_t total = rows * dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / dim;
        const int e = (int)(i - r * dim);
        const float v = __fsub_rn(x[i], center[e]);
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        const __nv_bfloat16 l = __float2bfloat16_rn(__fsub_rn(v, __bfloat162float(h)));
        __nv_bfloat16 *o = out + r * 3 * dim + e;
        o[0] = h;
        o[dim] = a_side ? h : l;
        o[2 * dim] = a_side ? l : h;
    }
}

// squared norms of the centred rows, float64 sum rounded to float (covered by
// eps); warp per row
__global__ void norm2_kernel(const float *__restrict__ x, const float *__restrict__ center, int64_t rows, int dim,
                             float *__restrict__ norm2)
{
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < rows; r += nw) {
        double s = 0.0;
        for (int e = lane; e < dim; e += 32) {
            const double v = (double)__fsub_rn(x[r * dim + e], center[e]);
            s = __fma_rn(v, v, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(FULL, s, o));
        if (lane == 0) norm2[r] = (float)s;
    }
}

// exact re-check of the screened candidates (numpy-order float64 distance)
template <int D>
__global__ void __launch_bounds__(256) exact_recheck_kernel(const float *refs, int64_t n, const float *qs, int64_t m,
                                                            const int32_t *cand, const float *cand_lb,
                                                            const int32_t *ncand, const float *best_ub,
                                                            int32_t *out_idx, double *out_dist, int32_t *fallback,
                                                            int32_t *nfallback, unsigned long long *nchecked)
{
    constexpr int GX = Lay<D>::G, NGX = WARP / GX;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = gw; g < m; g += nw) {
        const int c = ncand[g];
        if (c < 0) {
            if (lane == 0) fallback[atomicAdd(nfallback, 1)] = (int32_t)g;
            continue;
        }
        const float ub = best_ub[g];
        const float *q = qs + g * D;
        int checked = 0;
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bi = 0x7fffffff;
        for (int s0 = 0; s0 < c; s0 += NGX) {
            const int si = s0 + lane / GX;
            const bool ok = si < c && cand_lb[g * NCAND + si] <= ub;
            checked += __popc(__ballot_sync(FULL, ok)) / GX;
            const int j = cand[g * NCAND + (si < c ? si : 0)];
            const double dj = exact_dist<D>(refs, j, q, D, lane % GX);
            if (ok) argmin_merge(bd, bi, dj, j);
        }
        warp_argmin(bd, bi);
        if (lane == 0) {
            out_idx[g] = bi;
            out_dist[g] = bd;
            atomicAdd(nchecked, (unsigned long long)checked);
        }
    }
}

// full exact scan for the listed queries (overflowed candidate lists)
template <int D>
__global__ void __launch_bounds__(256) exact_list_kernel(const float *refs, int64_t n, const float *qs,
                                                         const int32_t *list, const int32_t *nlist, int32_t *out_idx,
                                                         double *out_dist)
{
    constexpr int GX = Lay<D>::G, NGX = WARP / GX;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int cnt = *nlist;
    for (int64_t i = gw; i < cnt; i += nw) {
        const int64_t g = list[i];
        const float *q = qs + g * D;
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bi = 0x7fffffff;
        for (int64_t j0 = 0; j0 < n; j0 += NGX) {
            const int64_t j = j0 + lane / GX;
            const bool ok = j < n;
            const double dj = exact_dist<D>(refs, (int)(ok ? j : 0), q, D, lane % GX);
            if (ok) argmin_merge(bd, bi, dj, (int)j);
        }
        warp_argmin(bd, bi);
        if (lane == 0) {
            out_idx[g] = bi;
            out_dist[g] = bd;
        }
    }
}

}  // namespace tc
}  // namespace rb

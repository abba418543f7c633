// riann_exact_tc.cuh -- K4: exact nearest reference (evaluation.py:24-50) with
// the distance screen on the 5th-generation tensor cores.
//
//   ||q - r||^2 = ||q'||^2 + ||r'||^2 - 2 q'.r' on operands centred on the
//   reference mean (q' = q - c, r' = r - c; distances are translation
//   invariant and the screen's error then scales with the patch spread), with
//   q'.r' from one tcgen05 GEMM (kind::f16, fp16 operands scaled by powers of
//   two into fp16's normal range, fp32 accumulation in TMEM), K = D.
//
//   Rigorous screen: |d2_est - d^2| <= E (||q'||^2 + ||r'||^2) + E_abs
//   (exact_eps, riann_b200.cu).  Each query keeps the smallest upper bound
//   u2 = d2_est + err and every reference whose lower bound l2 = d2_est - err
//   does not exceed it; the exact nearest reference always survives.
//
// Warp roles per CTA (one 128-query M tile resident in shared memory, all
// N tiles of 256 references streamed):
//   warp 0     TMA producer (query tile once; reference K-blocks through a
//              STAGES-deep ring, 128B swizzle)
//   warp 1     MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16)
//   warp 2     TMEM allocator (2 x 256 fp32 accumulator columns)
//   warps 4-11 epilogue: warp w reads TMEM lane quarter w%4 and column half
//              (w-4)/4 of the double-buffered accumulator (tcgen05.ld), two
//              FFMAs and a min per element, a short candidate list per
//              (query, half).
// exact_recheck_kernel re-evaluates the survivors with the exact float64
// distance in numpy's order (first minimum, lowest index on ties); queries
// whose list overflowed take the exact full scan (exact_list_kernel).  The
// screen only decides which references get the exact distance, so results
// are bit-identical to exact_nn.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "riann_kernels.cuh"

namespace rb {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;       // BK fp16 = 128 bytes per row (one swizzle atom)
constexpr int A_BLOCK = BM * BK * 2;             // 16 KB: one K-block of the resident query tile
constexpr int STAGE_BYTES = BN * BK * 2;         // 32 KB: one K-block of a reference tile
constexpr int NCAND = 16;                        // candidates kept per (query, column half)
constexpr int EPI_WARP0 = 4, EPI_WARPS = 8;
constexpr int THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int HALF = BN / 2;                     // columns per epilogue warp
constexpr int NRBUF = EPI_WARPS * 2 * HALF * 4;  // per-warp staged (1+E)nr, (1-E)nr
constexpr int SMEM_LIMIT = 227 * 1024;
__host__ __device__ constexpr int stages_for(int kb)
{
    return (SMEM_LIMIT - 1024 - NRBUF - kb * A_BLOCK) / STAGE_BYTES > 6
               ? 6
               : (SMEM_LIMIT - 1024 - NRBUF - kb * A_BLOCK) / STAGE_BYTES;
}
__host__ __device__ constexpr int smem_bytes(int kb) { return 1024 + kb * A_BLOCK + stages_for(kb) * STAGE_BYTES + NRBUF; }

// device-side scalars of one call (exact_scal_kernel)
struct Scal {
    float coef;   // -2 * 2^-(Sa + Sb): fp32 accumulator -> -2 q'.r'
    float eabs;   // absolute error term
    float E;      // relative error factor
    float hs;     // 2^(Sa + Sb - 1) = -1 / coef: squared distances in accumulator units
};

// w = nr' - acc with the -1 as an immediate (FFMA imm form: twice the 3-register issue rate)
__device__ __forceinline__ float sub_acc(float acc, float nr)
{
    float r;
    asm("fma.rn.f32 %0, %1, 0fBF800000, %2;" : "=f"(r) : "f"(acc), "f"(nr));
    return r;
}

struct ExactParams {
    const float *nq;       // (m) ||q'||^2 (float64 sum rounded to float)
    const float *nrU;      // (n) (1+E) ||r'||^2, rounded up
    const float *nrL;      // (n) (1-E) ||r'||^2, rounded down
    const float *dlt;      // (ceil(n/32)) per 32-column chunk: max (nrU - nrL) + 2^-21 max nrU, rounded up
    const Scal *scal;
    int64_t m, n;
    int kblocks;           // D / BK
    int stages;
    int32_t *cand;         // (m, 2, NCAND)
    float *cand_lb;        // (m, 2, NCAND) lower bounds (squared)
    int32_t *ncand;        // (m, 2): count, or -1 on overflow
    float *best_ub;        // (m, 2) smallest upper bound (squared)
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

// kind::f16 instruction descriptor: F16 x F16 -> F32 (A/B format 0 = F16), both K-major
__host__ __device__ constexpr uint32_t instr_desc(int M, int N)
{
    return (1u << 4)                      // D format F32
           | ((uint32_t)(N >> 3) << 17)   // N / 8
           | ((uint32_t)(M >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
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
}
// the registers of a tmem_ld32 are valid only after the next tmem_ld_wait
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__global__ void __launch_bounds__(THREADS, 1) exact_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                                                               const __grid_constant__ CUtensorMap mapB, ExactParams P)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle, by pointer arithmetic so accesses stay ld.shared
    unsigned char *smem = smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u);
    constexpr int MAXST = 8;
    __shared__ uint64_t full_bar[MAXST], empty_bar[MAXST], acc_full[2], acc_empty[2], a_bar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int ntiles = (int)((P.n + BN - 1) / BN);
    const int kb = P.kblocks, ST = P.stages;
    unsigned char *sA = smem;                         // kb resident K-blocks of the query tile
    unsigned char *sB = smem + kb * A_BLOCK;          // ST reference K-blocks
    float *sNr = reinterpret_cast<float *>(sB + ST * STAGE_BYTES);

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; s++) {
            bar_init(&full_bar[s], 1);
            bar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            bar_init(&acc_full[a], 1);
            bar_init(&acc_empty[a], EPI_WARPS);  // one arrive per epilogue warp
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

    if (warp == 0) {
        // ---- TMA producer
        if (lane == 0) {
            bar_expect(&a_bar, (unsigned)(kb * A_BLOCK));
            for (int k = 0; k < kb; k++) tma_load_2d(sA + k * A_BLOCK, &mapA, k * BK, (int)m0, &a_bar);
            int it = 0;
            for (int t = 0; t < ntiles; t++) {
                for (int k = 0; k < kb; k++, it++) {
                    const int s = it % ST;
                    if (it >= ST) bar_wait(&empty_bar[s], (unsigned)(((it / ST) - 1) & 1));
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
                const int s = it % ST;
                bar_wait(&full_bar[s], (unsigned)((it / ST) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint64_t da = smem_desc(sA + k * A_BLOCK), db = smem_desc(sB + s * STAGE_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++)  // 16 fp16 = 32 bytes per MMA step
#ifdef RIANN_K4_NOMMA  // timing probe: the epilogue alone (results are garbage)
                        if (P.n < 0)
#endif
                        mma_f16(tacc, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc, (k | kk) ? 1u : 0u);
                    mma_commit(&empty_bar[s]);
                    if (k == kb - 1) mma_commit(&acc_full[acc]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ---- epilogue: thread owns query row r (TMEM lane r), columns [h*HALF, (h+1)*HALF) of each tile
        const int ew = warp - EPI_WARP0;
        const int q4 = ew & 3, h = ew >> 2;
        const int r = q4 * 32 + lane;
        const int64_t qi = m0 + r;
        const bool rowok = qi < P.m;
        const Scal sc = *P.scal;
        const float nq = rowok ? P.nq[qi] : 0.f;
        // all bounds in accumulator units (x hs, an exact power of two):
        //   u2 = cu + (nrU - acc),  l2 = cl0 + (nrL - acc)
        const float hs = sc.hs;
        const float cu = __fmul_ru(__fadd_ru(__fmul_ru(__fadd_ru(1.f, sc.E), nq), sc.eabs), hs);
        const float cl0 = __fmul_rd(__fsub_rd(__fmul_rd(__fsub_rd(1.f, sc.E), nq), sc.eabs), hs);
        const float inf = __int_as_float(0x7f800000);
        float ub2 = inf;
        int cnt = rowok ? 0 : -2;
        int32_t cj[NCAND];
        float cl[NCAND];
        float *myU = sNr + ew * 2 * HALF, *myL = myU + HALF;
        const float sq = __fmul_ru(__fmul_ru(nq, 4.76837158203125e-7f), hs);  // 2^-21 nq: rounding slack of w, v
        // (1+E)nr / (1-E)nr of this warp's columns, 4 per lane, and the chunk slack dlt (lane k < 4 holds
        // chunk k), prefetched one tile ahead
        float pu[HALF / 32], pl[HALF / 32], pd;
        const int64_t nchunks = (P.n + 31) / 32;
#pragma unroll
        for (int k = 0; k < HALF / 32; k++) {
            const int64_t j = (int64_t)h * HALF + k * 32 + lane;
            pu[k] = j < P.n ? __ldg(P.nrU + j) : inf;
            pl[k] = j < P.n ? __ldg(P.nrL + j) : inf;
        }
        {
            const int64_t ch = (int64_t)h * (HALF / 32) + (lane & 3);
            pd = ch < nchunks ? __ldg(P.dlt + ch) : 0.f;
        }
        for (int t = 0; t < ntiles; t++) {
            const int acc = t & 1;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < HALF / 32; k++) {
                myU[k * 32 + lane] = pu[k] * hs;
                myL[k * 32 + lane] = pl[k] * hs;
            }
            __syncwarp();
            const float dcur = pd * hs;
#pragma unroll
            for (int k = 0; k < HALF / 32; k++) {
                const int64_t j = (int64_t)(t + 1) * BN + h * HALF + k * 32 + lane;
                pu[k] = j < P.n ? __ldg(P.nrU + j) : inf;
                pl[k] = j < P.n ? __ldg(P.nrL + j) : inf;
            }
            {
                const int64_t ch = ((int64_t)(t + 1) * BN + h * HALF) / 32 + (lane & 3);
                pd = ch < nchunks ? __ldg(P.dlt + ch) : 0.f;
            }
            bar_wait(&acc_full[acc], (unsigned)((t / 2) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // the TMEM load of column block k + 1 is in flight while block k is screened
            // (tcgen05.wait::ld covers every load issued before it, so the wait for
            // block k comes before block k + 1 is issued)
            const uint32_t tcol = tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * BN + h * HALF);
            uint32_t accA[32], accB[32];
            tmem_ld32(tcol, accA);
            auto screen = [&](const int k, const uint32_t (&acc32)[32]) {
                // fast path: w = (1+E)nr - acc; u2 = cu + w is an upper bound of d^2
                float wmin = inf;
#pragma unroll
                for (int x = 0; x < 32; x += 4) {
                    const float4 u4 = *reinterpret_cast<const float4 *>(myU + k * 32 + x);
                    wmin = fminf(wmin, fminf(fminf(sub_acc(__uint_as_float(acc32[x]), u4.x),
                                                   sub_acc(__uint_as_float(acc32[x + 1]), u4.y)),
                                             fminf(sub_acc(__uint_as_float(acc32[x + 2]), u4.z),
                                                   sub_acc(__uint_as_float(acc32[x + 3]), u4.w))));
                }
                ub2 = fminf(ub2, __fadd_ru(cu, wmin));
                const float thr = __fsub_ru(ub2, cl0);
                // v = (1-E)nr - acc >= w - dlt - sq, so no v <= thr unless wmin <= thr + dlt + sq
                const float dk = __shfl_sync(FULL, dcur, k);
                if (wmin <= __fadd_ru(__fadd_ru(thr, dk), sq) && cnt >= 0) {  // rare
                    uint32_t mask = 0;
                    float v[32];
#pragma unroll
                    for (int x = 0; x < 32; x += 4) {
                        const float4 l4 = *reinterpret_cast<const float4 *>(myL + k * 32 + x);
                        v[x] = sub_acc(__uint_as_float(acc32[x]), l4.x);
                        v[x + 1] = sub_acc(__uint_as_float(acc32[x + 1]), l4.y);
                        v[x + 2] = sub_acc(__uint_as_float(acc32[x + 2]), l4.z);
                        v[x + 3] = sub_acc(__uint_as_float(acc32[x + 3]), l4.w);
                    }
#pragma unroll
                    for (int x = 0; x < 32; x++) mask |= (v[x] <= thr ? 1u : 0u) << x;
                    while (mask && cnt >= 0) {
                        const int x = __ffs(mask) - 1;
                        mask &= mask - 1;
                        float vx = 0.f;
#pragma unroll
                        for (int y = 0; y < 32; y++) vx = y == x ? v[y] : vx;
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
                            if (cnt < 0) break;
                        }
                        cj[cnt] = (int32_t)((int64_t)t * BN + h * HALF + k * 32 + x);
                        cl[cnt] = __fadd_rd(cl0, vx);
                        cnt++;
                    }
                }
            };
#pragma unroll
            for (int k = 0; k < HALF / 32; k += 2) {
#ifdef RIANN_K4_NOEPI  // timing probe: the MMA pipeline alone (results are garbage)
                if (P.n > 0) break;
#endif
                tmem_ld_wait();
                tmem_ld32(tcol + (uint32_t)((k + 1) * 32), accB);
                screen(k, accA);
                tmem_ld_wait();
                if (k + 2 < HALF / 32) tmem_ld32(tcol + (uint32_t)((k + 2) * 32), accA);
                screen(k + 1, accB);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive(&acc_empty[acc]);
        }
        if (rowok) {
            const int64_t o = qi * 2 + h;
            int w2 = 0;
            if (cnt >= 0) {
                for (int y = 0; y < cnt; y++)
                    if (cl[y] <= ub2) {
                        P.cand[o * NCAND + w2] = cj[y];
                        P.cand_lb[o * NCAND + w2] = cl[y];
                        w2++;
                    }
            }
            P.ncand[o] = cnt >= 0 ? w2 : -1;
            P.best_ub[o] = ub2;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(2 * BN));
}

// ---- operand preparation ---------------------------------------------------
// centre c = mean of the references (float64 sums, rounded to float)
__global__ void center_sum_kernel(const float *__restrict__ x, int64_t rows, int dim, double *__restrict__ acc)
{
    const int e = threadIdx.x;  // block: dim threads (<= 256) over a chunk of 1024 rows
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

// max |fl(x - c)| (non-negative floats order like their bit patterns); warp per row
__global__ void absmax_kernel(const float *__restrict__ x, const float *__restrict__ center, int64_t rows, int dim,
                              unsigned *__restrict__ out)
{
    float mx = 0.f;
    const int64_t total = rows * dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmaxf(mx, fabsf(__fsub_rn(x[i], center[i % dim])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(mx));
}

// power-of-two exponent S with max * 2^S in [2^13, 2^14)
__device__ __forceinline__ int scale_exp(unsigned maxbits)
{
    const float mx = __uint_as_float(maxbits);
    if (!(mx > 0.f)) return 0;
    int ex;
    frexpf(mx, &ex);  // mx = f * 2^ex, f in [0.5, 1)
    return min(max(14 - ex, -60), 60);  // clamped: bounds stay finite in accumulator units
}

// fp16 operand rows: fl16(fl(x - c) * 2^S)
__global__ void split_kernel(const float *__restrict__ x, const float *__restrict__ center, int64_t rows, int dim,
                             const unsigned *__restrict__ maxbits, __half *__restrict__ out)
{
    const int S = scale_exp(*maxbits);
    const int64_t total = rows * dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __float2half_rn(ldexpf(__fsub_rn(x[i], center[i % dim]), S));
}

// ||fl(x - c)||^2 (float64 sum rounded to float, covered by E); with E given,
// also (1+E) n rounded up and (1-E) n rounded down.  Warp per row.
__global__ void norm2_kernel(const float *__restrict__ x, const float *__restrict__ center, int64_t rows, int dim,
                             float E, float *__restrict__ norm2, float *__restrict__ nU, float *__restrict__ nL)
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
        if (lane == 0) {
            const float n2 = (float)s;
            if (norm2) norm2[r] = n2;
            if (nU) nU[r] = __fmul_ru(__fadd_ru(1.f, E), __double2float_ru(s));
            if (nL) nL[r] = __fmul_rd(__fsub_rd(1.f, E), __double2float_rd(s));
        }
    }
}

// per 32-column chunk: max (nrU - nrL) + 2^-21 max nrU, rounded up (fast-path slack); warp per chunk
__global__ void chunk_slack_kernel(const float *__restrict__ nU, const float *__restrict__ nL, int64_t n,
                                   float *__restrict__ dlt)
{
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = w0; c < (n + 31) / 32; c += nw) {
        const int64_t j = c * 32 + lane;
        float d = 0.f, u = 0.f;
        if (j < n) {
            d = __fsub_ru(nU[j], nL[j]);
            u = nU[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            d = fmaxf(d, __shfl_xor_sync(FULL, d, o));
            u = fmaxf(u, __shfl_xor_sync(FULL, u, o));
        }
        if (lane == 0) dlt[c] = __fadd_ru(d, __fmul_ru(u, 4.76837158203125e-7f));
    }
}

// per-call scalars: coef = -2 * 2^-(Sa+Sb); eabs from the fp16 subnormal spacing
__global__ void exact_scal_kernel(const unsigned *__restrict__ maxq, const unsigned *__restrict__ maxr, int dim,
                                  float E, Scal *__restrict__ out)
{
    const int Sa = scale_exp(*maxq), Sb = scale_exp(*maxr);
    Scal s;
    s.coef = -2.f * ldexpf(1.f, -(Sa + Sb));
    // |fl16(v 2^S) - v 2^S| <= 2^-25 absolute below fp16's normal range, i.e. <= 2^-25-S in
    // original units (<= 2^-38 max|v|); dot error <= D (a_q maxr + a_r maxq) + D a_q a_r, doubled
    // for d^2, with a 4x margin
    const double mq = (double)__uint_as_float(*maxq), mr = (double)__uint_as_float(*maxr);
    const double aq = ldexp(1.0, -25 - Sa), ar = ldexp(1.0, -25 - Sb);
    s.eabs = (float)(8.0 * dim * (aq * mr + ar * mq + aq * ar) + 1e-30);
    s.E = E;
    s.hs = ldexpf(1.f, Sa + Sb - 1);
    *out = s;
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
        const int c0 = ncand[2 * g], c1 = ncand[2 * g + 1];
        if (c0 < 0 || c1 < 0) {
            if (lane == 0) fallback[atomicAdd(nfallback, 1)] = (int32_t)g;
            continue;
        }
        const float ub = fminf(best_ub[2 * g], best_ub[2 * g + 1]);
        const float *q = qs + g * D;
        const int c = c0 + c1;
        int checked = 0;
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        int bi = 0x7fffffff;
        for (int s0 = 0; s0 < c; s0 += NGX) {
            const int si = s0 + lane / GX;
            const int64_t slot = si < c0 ? 2 * g * NCAND + si : (2 * g + 1) * NCAND + (si - c0);
            const bool ok = si < c && cand_lb[si < c ? slot : 0] <= ub;
            checked += __popc(__ballot_sync(FULL, ok)) / GX;
            const int j = ok ? cand[slot] : 0;
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

// Stage latency/throughput: one 64 KB row copy plus NS small copies (SB bytes,
// random sources) on one mbarrier, 2 CTAs per SM, single-buffered (like the
// filter's item).  nvcc -O3 -arch=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_stage(const char *tab, int64_t tbytes, int NS, int SB, int iters, int *out, int use_ld)
{
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint64_t x = blockIdx.x * 0x9E3779B97F4A7C15ull + 1;
    int acc = 0;
    for (int it = 0; it < iters; it++) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const int64_t rowoff = (int64_t)(x % (uint64_t)(tbytes / 65536)) * 65536;
        if (threadIdx.x == 0) {
            const unsigned bytes = 65536 + (use_ld ? 0 : NS * SB);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm)), "l"(tab + rowoff), "r"(65536), "r"(sa(&bar)) : "memory");
        }
        __syncwarp();
        uint4 r = make_uint4(0, 0, 0, 0);
        if (threadIdx.x < 32) {
            for (int i = threadIdx.x; i < NS; i += 32) {
                uint64_t y = x * (i + 7) * 0x2545F4914F6CDD1Dull;
                const int64_t src = (int64_t)(y % (uint64_t)(tbytes / SB)) * SB;
                if (!use_ld)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + 65536 + i * SB)), "l"(tab + src), "r"(SB), "r"(sa(&bar)) : "memory");
            }
        }
        if (use_ld) {  // the same bytes as plain vector loads by all threads
            const int per = NS * SB / 16;
            for (int k = threadIdx.x; k < per; k += blockDim.x) {
                const int i = k / (SB / 16), o = k % (SB / 16);
                uint64_t y = x * (i + 7) * 0x2545F4914F6CDD1Dull;
                const int64_t src = (int64_t)(y % (uint64_t)(tbytes / SB)) * SB;
                const uint4 v = *reinterpret_cast<const uint4 *>(tab + src + o * 16);
                r.x ^= v.x; r.y ^= v.y;
            }
        }
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(&bar)), "r"(it & 1) : "memory");
        acc += sm[threadIdx.x * 64] + (int)r.x + (int)r.y;
        __syncthreads();
    }
    if (acc == 12345) out[0] = acc;
}
int main()
{
    size_t tb = (size_t)16 << 30;
    char *tab; cudaMalloc(&tab, tb); cudaMemset(tab, 1, tb);
    int *out; cudaMalloc(&out, 64);
    cudaFuncSetAttribute(k_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int cfg[][2] = {{0, 16}, {20, 1024}, {40, 512}, {20, 64}, {80, 256}};
    for (auto &c : cfg)
        for (int use_ld = 0; use_ld < 2; use_ld++) {
            int NS = c[0], SB = c[1];
            if (use_ld && NS == 0) continue;
            int iters = 300, grid = 148 * 2;
            size_t smem = 65536 + (size_t)NS * SB + 128;
            k_stage<<<grid, 512, smem>>>(tab, tb, NS, SB, 20, out, use_ld);
            cudaEventRecord(a);
            k_stage<<<grid, 512, smem>>>(tab, tb, NS, SB, iters, out, use_ld);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("NS=%2d SB=%5d %s: %.2f us per stage per CTA, %.0f GB/s\n", NS, SB, use_ld ? "ld " : "tma", ms * 1e3 / iters,
                   (double)grid * iters * (65536 + NS * SB) / ms / 1e6);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

// Per-SM TMA bulk-copy throughput: each CTA streams random rows (S bytes) of a
// large table into a ring of K shared-memory slots.  nvcc -O3 -arch=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_tma(const char *tab, int64_t rows, int S, int K, int iters, int *out)
{
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[8];
    if (threadIdx.x == 0)
        for (int i = 0; i < K; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint64_t x = blockIdx.x * 0x9E3779B97F4A7C15ull + 1;
    int acc = 0;
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters + K; it++) {
            const int sl = it % K;
            if (it >= K) {
                const unsigned par = ((it - K) / K) & 1;
                asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(&bar[sl])), "r"(par) : "memory");
                acc += sm[sl * S];
            }
            if (it < iters) {
                x ^= x << 13; x ^= x >> 7; x ^= x << 17;
                const char *src = tab + (int64_t)(x % rows) * S;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[sl])), "r"(S) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + sl * S)), "l"(src), "r"(S), "r"(sa(&bar[sl])) : "memory");
            }
        }
        out[blockIdx.x] = acc;
    }
}
int main()
{
    size_t tb = (size_t)16 << 30;
    char *tab; cudaMalloc(&tab, tb); cudaMemset(tab, 1, tb);
    int *out; cudaMalloc(&out, 4096 * 4);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int Ss[] = {16384, 65536};
    for (int S : Ss)
        for (int K = 1; K <= 3; K++) {
            for (int cps = 1; cps <= 2; cps++) {
                size_t smem = (size_t)S * K;
                if (smem * cps > 220 * 1024) continue;
                int iters = 200;
                int grid = 148 * cps;
                k_tma<<<grid, 32, smem>>>(tab, tb / S, S, K, 20, out);
                cudaEventRecord(a);
                k_tma<<<grid, 32, smem>>>(tab, tb / S, S, K, iters, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                printf("S=%6d K=%d ctas/SM=%d: %7.1f GB/s  (%.2f us per copy per CTA)\n", S, K, cps,
                       (double)grid * iters * S / ms / 1e6, ms * 1e3 / iters);
            }
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Random-read throughput vs footprint (TLB reach probe).  nvcc -O3 -arch=sm_100a tlb.cu -o tlb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rnd(const float *buf, uint64_t nflt, int iters, float *out, uint64_t stride_mask)
{
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 12345;
    float acc = 0.f;
    for (int i = 0; i < iters; i += 8) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            v[k] = __ldg(buf + ((x % nflt) & stride_mask));
        }
#pragma unroll
        for (int k = 0; k < 8; k++) acc += v[k];
    }
    if (acc == 1234.5f) out[0] = acc;
}
// dependent chain: latency
__global__ void chase(const uint64_t *buf, uint64_t n, int iters, uint64_t *out)
{
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 777;
    uint64_t p = x % n;
    for (int i = 0; i < iters; i++) {
        uint64_t v = __ldg(buf + p);
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        p = (x + v) % n;
    }
    if (p == 1) out[0] = p;
}
int main()
{
    size_t maxb = (size_t)40 << 30;
    float *buf;
    if (cudaMalloc(&buf, maxb) != cudaSuccess) { printf("alloc fail\n"); return 1; }
    cudaMemset(buf, 0, maxb);
    float *out; cudaMalloc(&out, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    size_t sizes[] = {(size_t)32 << 20, (size_t)128 << 20, (size_t)512 << 20, (size_t)2 << 30, (size_t)8 << 30, (size_t)16 << 30, (size_t)32 << 30};
    for (size_t s : sizes) {
        uint64_t nf = s / 4;
        int iters = 256;
        int blocks = 148 * 8, th = 256;
        rnd<<<blocks, th>>>(buf, nf, iters, out, ~0ull);
        cudaEventRecord(a);
        rnd<<<blocks, th>>>(buf, nf, iters, out, ~0ull);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double loads = (double)blocks * th * iters;
        chase<<<148 * 4, 32>>>((const uint64_t *)buf, s / 8, 64, (uint64_t *)out);
        cudaEventRecord(a);
        chase<<<148 * 4, 32>>>((const uint64_t *)buf, s / 8, 256, (uint64_t *)out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("footprint %6.2f GB: random 4B loads %7.2f G/s (%.0f GB/s of sectors); dependent latency %.0f ns\n",
               s / 1e9, loads / ms / 1e6, loads * 32 / ms / 1e6, ms2 * 1e6 / 256);
    }
    return 0;
}

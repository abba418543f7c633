// riann_effects.cuh -- the callers on the output side of the query:
//   * ANNF frame payload (engine.py:257-267): idx as u32, dist as f32, packed on
//     the device straight from the resident field (8 bytes per position leave
//     the GPU instead of 12);
//   * apply_effect / reconstruct_frame (transforms.py:175-253): gather each
//     position's payload row by its match, rescale by the query norm
//     (reconstruction kind), uniform average of the overlapping windows, and
//     for the chroma kind the integer YCoCg -> RGB finish.
// Every output is bit-identical to numpy: float32 adds in the reference's
// (dy, dx) loop order starting from 0, one correctly rounded f32 division,
// the f32/f64 rounding expressions of round_half_away.
#pragma once

#include "riann_kernels.cuh"

namespace rb {

enum { FX_RECONSTRUCTION = 0, FX_FULL = 1, FX_CHROMA = 2 };

// payload of one ANNF frame: Q little-endian u32 indices, then Q f32 distances
__global__ void pack_field_kernel(const int32_t *__restrict__ idx, const double *__restrict__ dist, int64_t Q,
                                  uint32_t *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    out[i] = (uint32_t)idx[i];                                      // astype("<u4"): same bits for 0 <= idx < 2^31
    out[Q + i] = __float_as_uint(__double2float_rn(dist[i]));       // astype("<f4"): round to nearest even
}

// norm of every query patch as normalize_rows computes it (patches.py:100-115):
// sqrt of numpy's pairwise f64 sum of squares, 0 below 1e-12 (any patch size;
// 8x8 patches use the warp-cooperative K1 kernel instead)
__global__ void effect_norms_kernel(const float *__restrict__ frame, int H, int W, int pw, int ph, int gw, int64_t Q,
                                    double *__restrict__ norms)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Q) return;
    const int x = (int)(g % gw), y = (int)(g / gw);
    FrameGet<0, 0> get{frame + (int64_t)y * W + x, W, 1, pw, ph};
    const double nr = __dsqrt_rn(pw_sum(get, 0, (int64_t)pw * ph));
    norms[g] = nr >= 1e-12 ? nr : 0.0;
}

// round_half_away on a float32 value (numpy evaluates it in float32 for f32 input)
__device__ __forceinline__ long long rha_f32(float x)
{
    const float a = floorf(__fadd_rn(fabsf(x), 0.5f));
    const float s = x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f);
    return (long long)__fmul_rn(s, a);
}

// round_half_away on a float64 value
__device__ __forceinline__ long long rha_f64(double x)
{
    const double a = floor(__dadd_rn(fabs(x), 0.5));
    const double s = x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0);
    return (long long)__dmul_rn(s, a);
}

struct BlendParams {
    const float *frame;       // (H, W) single plane
    int H, W, pw, ph, gw, gh;
    const int32_t *idx;       // (gh, gw) matches
    const float *payloads;    // (n, planes * pw * ph)
    int planes;               // 1 (reconstruction / full-patch) or 2 (chroma)
    int kind;
    const double *norms;      // (gh * gw) f64 query norms, reconstruction kind (rows scaled by f32(norm))
    float *out;               // (planes, H, W) f32, or null
    uint8_t *rgb;             // (H, W, 3) for the chroma kind, or null
};

// _blend_planes (transforms.py:175-189) + the kind-specific finish (:230-253):
// thread per output pixel; contributions summed in the reference's (dy, dx) order
__global__ void blend_kernel(BlendParams P)
{
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (int64_t)P.H * P.W) return;
    const int y = (int)(p / P.W), x = (int)(p - (int64_t)y * P.W);
    const int pp = P.pw * P.ph;
    float acc[2] = {0.f, 0.f};
    float cnt = 0.f;
    for (int dy = 0; dy < P.ph; dy++) {
        const int gy = y - dy;
        if (gy < 0 || gy >= P.gh) continue;
        for (int dx = 0; dx < P.pw; dx++) {
            const int gx = x - dx;
            if (gx < 0 || gx >= P.gw) continue;
            const int64_t g = (int64_t)gy * P.gw + gx;
            const float *row = P.payloads + (int64_t)P.idx[g] * P.planes * pp + dy * P.pw + dx;
            const float sc = P.kind == FX_RECONSTRUCTION ? __double2float_rn(P.norms[g]) : 1.f;
            for (int c = 0; c < P.planes; c++) {
                float v = __ldg(row + c * pp);
                if (P.kind == FX_RECONSTRUCTION) v = __fmul_rn(v, sc);
                acc[c] = __fadd_rn(acc[c], v);
            }
            cnt = __fadd_rn(cnt, 1.f);
        }
    }
    float pl[2];
    for (int c = 0; c < P.planes; c++) pl[c] = __fdiv_rn(acc[c], cnt);
    if (P.out)
        for (int c = 0; c < P.planes; c++) P.out[(int64_t)c * P.H * P.W + p] = pl[c];
    if (P.kind == FX_CHROMA && P.rgb) {
        // ycocg = (rha(frame * 255) f64, rha(co) f32, rha(cg) f32); ycocg_to_rgb; clip to u8
        const long long Y = rha_f64(__dmul_rn((double)P.frame[p], 255.0));
        const long long co = rha_f32(pl[0]), cg = rha_f32(pl[1]);
        const long long t = Y - (cg >> 1);
        const long long gg = cg + t;
        const long long b = t - (co >> 1);
        const long long r = b + co;
        const long long v3[3] = {r, gg, b};
        for (int c = 0; c < 3; c++) {
            const long long v = v3[c] < 0 ? 0 : (v3[c] > 255 ? 255 : v3[c]);
            P.rgb[p * 3 + c] = (uint8_t)v;
        }
    }
}

// Tiled form of blend_kernel for pw <= 16 (the same sums, same order): a CTA owns
// an output tile of BY x BX pixels; for each dy it stages, for every position that
// feeds the tile at that dy, the dy-th line of its payload row (pw values per plane,
// norm-scaled for the reconstruction kind) in shared memory; each pixel then adds
// the dx = 0..pw-1 contributions from shared memory.  dy outer, dx inner, as
// transforms.py:183-187 accumulates.
constexpr int BX = 64, BY = 8;

__global__ void __launch_bounds__(BX * BY) blend_tiled_kernel(BlendParams P)
{
    extern __shared__ float sline[];  // [planes][BY][pw][BX + pw - 1] (consecutive threads: consecutive words)
    const int pw = P.pw, ph = P.ph, pp = pw * ph;
    const int tx = threadIdx.x % BX, ty = threadIdx.x / BX;
    const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
    const int x = x0 + tx, y = y0 + ty;
    const int SX = BX + pw - 1;  // positions per staged row
    float acc[2] = {0.f, 0.f};
    float cnt = 0.f;
    for (int dy = 0; dy < ph; dy++) {
        // stage positions gy = y0 + r - dy (r < BY), gx = x0 - pw + 1 + s (s < SX)
        __syncthreads();
        for (int e = threadIdx.x; e < BY * SX; e += BX * BY) {
            const int r = e / SX, sx = e - r * SX;
            const int gy = y0 + r - dy, gx = x0 - pw + 1 + sx;
            const bool ok = gy >= 0 && gy < P.gh && gx >= 0 && gx < P.gw;
            const int64_t g = ok ? (int64_t)gy * P.gw + gx : 0;
            const float *row = P.payloads + (ok ? (int64_t)P.idx[g] * P.planes * pp : 0) + dy * pw;
            const float sc = (ok && P.kind == FX_RECONSTRUCTION) ? __double2float_rn(P.norms[g]) : 1.f;
            for (int c = 0; c < P.planes; c++) {
                float *dst = sline + ((size_t)c * BY + r) * pw * SX + sx;
                if ((pw & 3) == 0) {  // 16-byte vectors: row offsets are multiples of 4 floats
                    for (int d4 = 0; d4 < pw; d4 += 4) {
                        float4 v = ok ? __ldg(reinterpret_cast<const float4 *>(row + c * pp + d4))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                        if (P.kind == FX_RECONSTRUCTION) {
                            v.x = __fmul_rn(v.x, sc);
                            v.y = __fmul_rn(v.y, sc);
                            v.z = __fmul_rn(v.z, sc);
                            v.w = __fmul_rn(v.w, sc);
                        }
                        dst[(size_t)(d4 + 0) * SX] = v.x;
                        dst[(size_t)(d4 + 1) * SX] = v.y;
                        dst[(size_t)(d4 + 2) * SX] = v.z;
                        dst[(size_t)(d4 + 3) * SX] = v.w;
                    }
                } else {
                    for (int dx = 0; dx < pw; dx++) {
                        float v = ok ? __ldg(row + c * pp + dx) : 0.f;
                        if (P.kind == FX_RECONSTRUCTION) v = __fmul_rn(v, sc);
                        dst[(size_t)dx * SX] = v;
                    }
                }
            }
        }
        __syncthreads();
        const int gy = y - dy;
        if (y < P.H && x < P.W && gy >= 0 && gy < P.gh) {
            for (int dx = 0; dx < pw; dx++) {
                const int gx = x - dx;
                if (gx < 0 || gx >= P.gw) continue;
                const int sx = gx - (x0 - pw + 1);
                for (int c = 0; c < P.planes; c++)
                    acc[c] = __fadd_rn(acc[c], sline[(((size_t)c * BY + ty) * pw + dx) * SX + sx]);
                cnt = __fadd_rn(cnt, 1.f);
            }
        }
    }
    if (y >= P.H || x >= P.W) return;
    const int64_t p = (int64_t)y * P.W + x;
    float pl[2];
    for (int c = 0; c < P.planes; c++) pl[c] = __fdiv_rn(acc[c], cnt);
    if (P.out)
        for (int c = 0; c < P.planes; c++) P.out[(int64_t)c * P.H * P.W + p] = pl[c];
    if (P.kind == FX_CHROMA && P.rgb) {
        const long long Y = rha_f64(__dmul_rn((double)P.frame[p], 255.0));
        const long long co = rha_f32(pl[0]), cg = rha_f32(pl[1]);
        const long long t = Y - (cg >> 1);
        const long long gg = cg + t;
        const long long b = t - (co >> 1);
        const long long r = b + co;
        const long long v3[3] = {r, gg, b};
        for (int c = 0; c < 3; c++) {
            const long long v = v3[c] < 0 ? 0 : (v3[c] > 255 ? 255 : v3[c]);
            P.rgb[p * 3 + c] = (uint8_t)v;
        }
    }
}

// coherency_stats (evaluation.py:86-138): for index pairs (i, j) and query rows u,
// shift = dist(refs[i], refs[j]) and predictor = dist(refs[i], u), each the
// numpy-order f64 distance of EuclideanMetric.__call__ (patches.py:138-159).
// Warp-cooperative for numpy-mappable dims (groups of Lay<D>::G lanes).
template <int D>
__global__ void __launch_bounds__(256) pair_dist_kernel(const float *__restrict__ refs, const int32_t *__restrict__ ia,
                                                        const int32_t *__restrict__ ib, const float *__restrict__ u,
                                                        int64_t m, int dim, double *__restrict__ out_ab,
                                                        double *__restrict__ out_au)
{
    constexpr int GX = D > 0 ? Lay<D>::G : 1;
    constexpr int NG = WARP / GX;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k0 = w0 * NG; k0 < m; k0 += nw * NG) {
        const int64_t k = k0 + lane / GX;
        const bool ok = k < m;
        const int64_t kk = ok ? k : 0;
        const float *ri = refs + (int64_t)ia[kk] * dim;
        double dab, dau = 0.0;
        if constexpr (D > 0) {
            dab = exact_dist<D>(refs, ib[kk], ri, D, lane % GX);
            if (u) dau = exact_dist<D>(refs, ia[kk], u + kk * D, D, lane % GX);
        } else {
            dab = dist_thread(refs + (int64_t)ib[kk] * dim, ri, dim);
            if (u) dau = dist_thread(u + kk * dim, ri, dim);
        }
        if (ok && (lane % GX) == 0) {
            out_ab[k] = dab;
            if (u) out_au[k] = dau;
        }
    }
}

}  // namespace rb

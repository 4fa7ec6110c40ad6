// Sort-last 'over' compositor kernel (sm_100a).
//
// Replaces the reference's per-pixel cross-rank reduction -- the order-independent (t, globalId) min of
// pkg/src/dprt/bvh.py:246-248 applied by cycling rays through every rank (engine.py:282-310) -- with the
// order-dependent front-to-back 'over' of premultiplied RGBA fragments, fused with the final tone map
// (engine.py:500-502) for the row block a rank owns (engine.py:216-221).  HBM / NVLink bound: each
// pixel reads 16 B per fragment and writes 3 B (RGB8) and/or 16 B (RGBA); fragments may be peer
// pointers, so the same kernel is the fused direct-send + gather over NVLink.

#include "common.cuh"

namespace dprt {


__device__ __forceinline__ unsigned tone8(float x) {
    // floor(clip(x, 0, 1) * 255 + 0.5)   (engine.py:502)
    return (unsigned)floorf(fminf(fmaxf(x, 0.f), 1.f) * 255.f + 0.5f);
}

__device__ __forceinline__ float4 blend_pixel(const CompositeArgs& a, long long i) {
    float4 acc = __ldg(a.in[0] + i);
    for (int p = 1; p < a.P; ++p) {
        const float4 f = __ldg(a.in[p] + i);
        const float one = 1.f - acc.w;
        acc.x = fmaf(one, f.x, acc.x);
        acc.y = fmaf(one, f.y, acc.y);
        acc.z = fmaf(one, f.z, acc.z);
        acc.w = fmaf(one, f.w, acc.w);
    }
    return acc;
}

// Each thread composites 4 consecutive pixels so the RGB8 output is three aligned 32-bit stores.
__global__ void __launch_bounds__(256) composite_kernel(const CompositeArgs a) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long i0 = q * 4;
    if (i0 >= a.npix) return;
    const int cnt = (int)min(4LL, a.npix - i0);
    unsigned char px[12];
    for (int k = 0; k < cnt; ++k) {
        const float4 c = blend_pixel(a, i0 + k);
        if (a.flags & DPRT_COMPOSITE_RGBA) a.rgba[i0 + k] = c;
        if (a.flags & DPRT_COMPOSITE_TONEMAP) {
            const float one = 1.f - c.w;
            px[3 * k + 0] = (unsigned char)tone8(fmaf(one, a.bg[0], c.x));
            px[3 * k + 1] = (unsigned char)tone8(fmaf(one, a.bg[1], c.y));
            px[3 * k + 2] = (unsigned char)tone8(fmaf(one, a.bg[2], c.z));
        }
    }
    if (a.flags & DPRT_COMPOSITE_TONEMAP) {
        uint8_t* dst = a.rgb8 + 3 * i0;
        if (cnt == 4 && ((reinterpret_cast<uintptr_t>(dst) & 3) == 0)) {
            uint32_t w[3];
#pragma unroll
            for (int k = 0; k < 3; ++k)
                w[k] = (uint32_t)px[4 * k] | ((uint32_t)px[4 * k + 1] << 8) | ((uint32_t)px[4 * k + 2] << 16) |
                       ((uint32_t)px[4 * k + 3] << 24);
            uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
            d32[0] = w[0];
            d32[1] = w[1];
            d32[2] = w[2];
        } else {
            for (int k = 0; k < 3 * cnt; ++k) dst[k] = px[k];
        }
    }
}

cudaError_t launch_composite(const CompositeArgs& a, cudaStream_t stream) {
    const long long threads = (a.npix + 3) / 4;
    const int block = 256;
    const long long grid = (threads + block - 1) / block;
    if (grid == 0) return cudaSuccess;
    composite_kernel<<<(unsigned)grid, block, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace dprt

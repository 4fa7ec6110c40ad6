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

__device__ __forceinline__ void over(float4& acc, const float4 f) {
    const float one = 1.f - acc.w;
    acc.x = fmaf(one, f.x, acc.x);
    acc.y = fmaf(one, f.y, acc.y);
    acc.z = fmaf(one, f.z, acc.z);
    acc.w = fmaf(one, f.w, acc.w);
}

__device__ __forceinline__ uint32_t pack_rgb8(const float4 c, const float bg[3], int ch) {
    const float one = 1.f - c.w;
    const float v = ch == 0 ? fmaf(one, bg[0], c.x) : (ch == 1 ? fmaf(one, bg[1], c.y) : fmaf(one, bg[2], c.z));
    return tone8(v);
}

// fp16 RGBA fragment pixel (uint2 = two __half2) -> float4
__device__ __forceinline__ float4 h2f(const uint2 v) {
    const float2 rg = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
    const float2 ba = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
    return make_float4(rg.x, rg.y, ba.x, ba.y);
}

// one fragment pixel / four consecutive fragment pixels, f32 or fp16 storage
template <bool kHalf>
__device__ __forceinline__ float4 load1(const float4* frag, long long i) {
    if (kHalf) return h2f(__ldg(reinterpret_cast<const uint2*>(frag) + i));
    return __ldg(frag + i);
}
template <bool kHalf>
__device__ __forceinline__ void load4(const float4* frag, long long i, float4 f[4]) {
    if (kHalf) {
        const uint2* p = reinterpret_cast<const uint2*>(frag) + i;
        if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {  // two 16-byte loads carry the 4 pixels
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(p)), b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
            f[0] = h2f(make_uint2(a.x, a.y));
            f[1] = h2f(make_uint2(a.z, a.w));
            f[2] = h2f(make_uint2(b.x, b.y));
            f[3] = h2f(make_uint2(b.z, b.w));
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] = h2f(__ldg(p + k));
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) f[k] = __ldg(frag + i + k);
    }
}

// Each thread composites 4 consecutive pixels: per fragment it issues the four 16-byte loads together
// (and the next fragment's before blending, via unrolling), so P fragments keep 4-8 loads in flight;
// the 12 RGB8 bytes leave as three aligned 32-bit stores.  A fragment covers only the tile pixels
// [lo, hi) (a rank's footprint rows): outside them it is clear and is not read at all.
template <bool kHalf>
__device__ __forceinline__ void composite4_body(const CompositeArgs& a, long long q) {
    const long long i0 = q * 4;
    if (i0 >= a.npix) return;
    if (i0 + 4 <= a.npix) {
        float4 acc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
        for (int p = 0; p < a.P; ++p) {
            const long long lo = a.lo[p], hi = a.hi[p];
            const long long off = i0 - lo;
            float4 f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] = make_float4(0.f, 0.f, 0.f, 0.f);  // clear: over adds exact 0
            if (i0 >= lo && i0 + 4 <= hi) {
                load4<kHalf>(a.in[p], off, f);
            } else if (i0 + 4 > lo && i0 < hi) {  // a range edge inside this group (width not a multiple of 4)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (i0 + k >= lo && i0 + k < hi) f[k] = load1<kHalf>(a.in[p], off + k);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) over(acc[k], f[k]);
        }
        if (a.flags & DPRT_COMPOSITE_RGBA) {
#pragma unroll
            for (int k = 0; k < 4; ++k) a.rgba[i0 + k] = acc[k];
        }
        if (a.flags & DPRT_COMPOSITE_TONEMAP) {
            uint32_t b[12];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) b[3 * k + ch] = pack_rgb8(acc[k], a.bg, ch);
            uint8_t* dst = a.rgb8 + 3 * i0;
            if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
                uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
#pragma unroll
                for (int w = 0; w < 3; ++w)
                    d32[w] = b[4 * w] | (b[4 * w + 1] << 8) | (b[4 * w + 2] << 16) | (b[4 * w + 3] << 24);
            } else {
#pragma unroll
                for (int k = 0; k < 12; ++k) dst[k] = (uint8_t)b[k];
            }
        }
        return;
    }
    // tail: fewer than 4 pixels left
    for (long long i = i0; i < a.npix; ++i) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int p = 0; p < a.P; ++p)
            if (i >= a.lo[p] && i < a.hi[p]) over(acc, load1<kHalf>(a.in[p], i - a.lo[p]));
        if (a.flags & DPRT_COMPOSITE_RGBA) a.rgba[i] = acc;
        if (a.flags & DPRT_COMPOSITE_TONEMAP)
            for (int ch = 0; ch < 3; ++ch) a.rgb8[3 * i + ch] = (uint8_t)pack_rgb8(acc, a.bg, ch);
    }
}

// Grid-stride: one pass for the plain launch; a signalling launch (dprt_composite_signal) runs a capped grid
// so only a few CTAs per SM pay the system-scope fence of grid_signal.
template <bool kHalf, bool kSig>
__global__ void __launch_bounds__(256) composite_kernel(const CompositeArgs a) {
    const long long q0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (!kSig) {
        composite4_body<kHalf>(a, q0);
    } else {
        const long long n = (a.npix + 3) / 4, stride = (long long)gridDim.x * blockDim.x;
        for (long long q = q0; q < n; q += stride) composite4_body<kHalf>(a, q);
        grid_signal(a.sig_ctr, a.sig, a.n_sig, a.sig_epoch);  // e.g. rows written into rank 0's frame
    }
}

// Small tiles (a rank's row block after the exchange): one pixel per thread, so the grid still fills the
// 148 SMs, with up to 8 fragments' loads issued before the first is blended.
template <bool kHalf>
__device__ __forceinline__ void composite_px_body(const CompositeArgs& a, long long i) {
    if (i >= a.npix) return;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p0 = 0; p0 < a.P; p0 += 8) {
        float4 f[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int p = p0 + k;
            f[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p < a.P && i >= a.lo[p] && i < a.hi[p]) f[k] = load1<kHalf>(a.in[p], i - a.lo[p]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) over(acc, f[k]);
    }
    if (a.flags & DPRT_COMPOSITE_RGBA) a.rgba[i] = acc;
    if (a.flags & DPRT_COMPOSITE_TONEMAP)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) a.rgb8[3 * i + ch] = (uint8_t)pack_rgb8(acc, a.bg, ch);
}

template <bool kHalf, bool kSig>
__global__ void __launch_bounds__(256) composite_px_kernel(const CompositeArgs a) {
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (!kSig) {
        composite_px_body<kHalf>(a, i0);
    } else {
        const long long stride = (long long)gridDim.x * blockDim.x;
        for (long long i = i0; i < a.npix; i += stride) composite_px_body<kHalf>(a, i);
        grid_signal(a.sig_ctr, a.sig, a.n_sig, a.sig_epoch);
    }
}

// Stream-ordered wait for peers' epoch flags (dprt_wait_flags): one warp spins with system-scope acquire
// loads; a wait that outlives ~2^35 cycles (~17 s) traps instead of hanging the stream forever.
__global__ void wait_flags_kernel(const unsigned* __restrict__ flags, int n, unsigned epoch) {
    const long long t0 = clock64();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        while ((int)(ld_acquire_sys(flags + i) - epoch) < 0) {
            __nanosleep(128);
            if (clock64() - t0 > (1LL << 35)) __trap();
        }
    }
}

cudaError_t launch_wait_flags(const unsigned* flags, int n, unsigned epoch, cudaStream_t stream) {
    wait_flags_kernel<<<1, 32, 0, stream>>>(flags, n, epoch);
    return cudaGetLastError();
}

#ifndef DPRT_COMPOSITE_PX_BELOW
#define DPRT_COMPOSITE_PX_BELOW (1 << 22)  // tiles below this many pixels blending >= 3 fragments use one
#endif                                     // pixel per thread (graph-timed sweep, profiles/r01_composite_sweep.md)

cudaError_t launch_composite(const CompositeArgs& a, cudaStream_t stream) {
    const int block = 256;
    if (a.npix == 0) {
        if (a.n_sig) {  // nothing to blend: still signal (one CTA, no stores to fence but its own)
            CompositeArgs e = a;
            composite_px_kernel<false, true><<<1, 32, 0, stream>>>(e);
            return cudaGetLastError();
        }
        return cudaSuccess;
    }
    int cap = 0;  // signalling launches: at most 8 CTAs per SM
    if (a.n_sig) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cap = 8 * sms;
    }
    if (a.npix < DPRT_COMPOSITE_PX_BELOW && a.P >= 3) {
        long long grid = (a.npix + block - 1) / block;
        if (cap && grid > cap) grid = cap;
        const bool h = a.flags & DPRT_COMPOSITE_HALF_IN;
        if (a.n_sig)
            (h ? composite_px_kernel<true, true> : composite_px_kernel<false, true>)<<<(unsigned)grid, block, 0, stream>>>(a);
        else
            (h ? composite_px_kernel<true, false> : composite_px_kernel<false, false>)<<<(unsigned)grid, block, 0, stream>>>(a);
        return cudaGetLastError();
    }
    const long long threads = (a.npix + 3) / 4;
    long long grid = (threads + block - 1) / block;
    if (cap && grid > cap) grid = cap;
    const bool h = a.flags & DPRT_COMPOSITE_HALF_IN;
    if (a.n_sig)
        (h ? composite_kernel<true, true> : composite_kernel<false, true>)<<<(unsigned)grid, block, 0, stream>>>(a);
    else
        (h ? composite_kernel<true, false> : composite_kernel<false, false>)<<<(unsigned)grid, block, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace dprt

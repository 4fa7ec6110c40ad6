// Brick storage kernels: synthetic field generation and the macrocell min/max grid.
//
// The generator evaluates the blob mixture of DESIGN.md §2.2 in float64 with explicitly rounded ops in
// the same order as oracle/dvr_oracle.c (field_value), so GPU voxels are bit-identical to the CPU ones --
// the device-side counterpart of the reference's seeded, bit-reproducible scene generator
// (pkg/src/dprt/scene.py:250-289: "identical seeds give bit-identical scenes").

#include <cuda_fp16.h>

#include "common.cuh"

namespace dprt {

struct GenArgs {
    long long N[3];
    long long s_lo[3];
    long long sd[3];
    int kind;  // 0 blob mixture, 1 Marschner-Lobb (blobs[0..1] = f_M, alpha)
    int nb;
    double blobs[DPRT_MAX_BLOBS * 5];
};

// The oracle's reproducible cosine (oracle/dvr_oracle.c dvr_oracle_det_cos): 2pi reduction (hi + lo) and a
// 14-term even Taylor polynomial, each op one explicitly rounded f64 op in the oracle's order.
__constant__ double kMlCos[14] = {1.0, -0.5, 0.041666666666666664, -0.001388888888888889, 2.48015873015873e-05,
                                  -2.755731922398589e-07, 2.08767569878681e-09, -1.1470745597729725e-11,
                                  4.779477332387385e-14, -1.5619206968586225e-16, 4.110317623312165e-19,
                                  -8.896791392450574e-22, 1.6117375710961184e-24, -2.4795962632247976e-27};
constexpr double kTwoPi = 6.283185307179586, kTwoPiLo = 2.4492935982947064e-16;
constexpr double kInvTwoPi = 0.15915494309189535, kHalfPi = 1.5707963267948966;

__device__ double det_cos(double a) {
    const double k = floor(__dadd_rn(__dmul_rn(a, kInvTwoPi), 0.5));
    const double r = __dsub_rn(__dsub_rn(a, __dmul_rn(k, kTwoPi)), __dmul_rn(k, kTwoPiLo));
    const double r2 = __dmul_rn(r, r);
    double p = kMlCos[13];
#pragma unroll
    for (int i = 12; i >= 0; --i) p = __dadd_rn(__dmul_rn(p, r2), kMlCos[i]);
    return p;
}

// Marschner-Lobb, operation for operation as ml_value in oracle/dvr_oracle.c.
__device__ double ml_value(double ux, double uy, double uz, double fm, double alpha) {
    const double x = __dsub_rn(__dmul_rn(2.0, ux), 1.0);
    const double y = __dsub_rn(__dmul_rn(2.0, uy), 1.0);
    const double z = __dsub_rn(__dmul_rn(2.0, uz), 1.0);
    const double r = __dsqrt_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
    const double pr = det_cos(__dmul_rn(__dmul_rn(kTwoPi, fm), det_cos(__dmul_rn(kHalfPi, r))));
    const double sz = det_cos(__dsub_rn(__dmul_rn(kHalfPi, z), kHalfPi));
    double v = __ddiv_rn(__dadd_rn(__dsub_rn(1.0, sz), __dmul_rn(alpha, __dadd_rn(1.0, pr))),
                         __dmul_rn(2.0, __dadd_rn(1.0, alpha)));
    return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

__global__ void generate_kernel(const GenArgs g, float* __restrict__ out) {
    const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long y = blockIdx.y;
    const long long z = blockIdx.z;
    if (x >= g.sd[0]) return;
    const long long i = g.s_lo[0] + x, j = g.s_lo[1] + y, k = g.s_lo[2] + z;
    const double ux = g.N[0] > 1 ? __ddiv_rn((double)i, (double)(g.N[0] - 1)) : 0.0;
    const double uy = g.N[1] > 1 ? __ddiv_rn((double)j, (double)(g.N[1] - 1)) : 0.0;
    const double uz = g.N[2] > 1 ? __ddiv_rn((double)k, (double)(g.N[2] - 1)) : 0.0;
    if (g.kind == 1) {
        out[(z * g.sd[1] + y) * g.sd[0] + x] = __double2float_rn(ml_value(ux, uy, uz, g.blobs[0], g.blobs[1]));
        return;
    }
    double f = 0.0;
    for (int b = 0; b < g.nb; ++b) {
        const double* p = g.blobs + 5 * b;
        const double dx = __dsub_rn(ux, p[0]), dy = __dsub_rn(uy, p[1]), dz = __dsub_rn(uz, p[2]);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        const double q = __dsub_rn(1.0, __dmul_rn(r2, p[3]));
        if (q > 0.0) f = __dadd_rn(f, __dmul_rn(p[4], __dmul_rn(__dmul_rn(q, q), q)));
    }
    if (f > 1.0) f = 1.0;
    out[(z * g.sd[1] + y) * g.sd[0] + x] = __double2float_rn(f);
}

cudaError_t launch_generate(const DeviceBrick& b, const DprtFieldSpec& spec, cudaStream_t stream) {
    GenArgs g;
    for (int a = 0; a < 3; ++a) {
        g.N[a] = b.desc.dims[a];
        g.s_lo[a] = b.s_lo[a];
        g.sd[a] = b.sd[a];
    }
    g.kind = spec.kind;
    if (spec.kind == 1) {
        g.nb = 0;
        g.blobs[0] = spec.blobs[0];
        g.blobs[1] = spec.blobs[1];
    } else {
        g.nb = spec.n_blobs;
        for (int i = 0; i < 5 * spec.n_blobs; ++i) g.blobs[i] = spec.blobs[i];
    }
    dim3 block(256);
    dim3 grid((unsigned)((b.sd[0] + 255) / 256), (unsigned)b.sd[1], (unsigned)b.sd[2]);
    generate_kernel<<<grid, block, 0, stream>>>(g, b.vox);
    return cudaGetLastError();
}

// Macrocell m covers local cells [8m, 8m + 8) per axis, i.e. voxels [8m, 8m + 8]; its (min, max) is
// taken over the 1-voxel dilation [8m - 1, 8m + 9] so that samples whose f32 position rounds across a
// macrocell face are still bounded by it (skipping is exact, not approximate).
__global__ void macrocell_kernel(const float* __restrict__ vox, long long sd0, long long sd1, long long sd2,
                                 int mc0, int mc1, int mc2, int mshift, float2* __restrict__ macro) {
    const int mx = blockIdx.x * blockDim.x + threadIdx.x;
    const int my = blockIdx.y, mz = blockIdx.z;
    if (mx >= mc0) return;
    const long long m = 1LL << mshift;  // macrocell edge in cells
    const long long x0 = max(0LL, (long long)mx * m - 1), x1 = min(sd0 - 1, (long long)mx * m + m + 1);
    const long long y0 = max(0LL, (long long)my * m - 1), y1 = min(sd1 - 1, (long long)my * m + m + 1);
    const long long z0 = max(0LL, (long long)mz * m - 1), z1 = min(sd2 - 1, (long long)mz * m + m + 1);
    float lo = INFINITY, hi = -INFINITY;
    for (long long z = z0; z <= z1; ++z)
        for (long long y = y0; y <= y1; ++y) {
            const float* row = vox + (z * sd1 + y) * sd0;
            for (long long x = x0; x <= x1; ++x) {
                const float v = __ldg(row + x);
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
        }
    macro[((long long)mz * mc1 + my) * mc0 + mx] = make_float2(lo, hi);
}

// The eight 4^3-cell sub-blocks of every macrocell: (min, max) over the sub-block's voxels dilated by one
// voxel, like the macrocell's (the TF classifies them per version into the sub-block masks).
__global__ void subblock_kernel(const float* __restrict__ vox, long long sd0, long long sd1, long long sd2,
                                int mc0, int mc1, int mc2, int mshift, float2* __restrict__ sub) {
    const int sx = blockIdx.x * blockDim.x + threadIdx.x;  // sub-block grid: 2 per macrocell per axis
    const int sy = blockIdx.y, sz = blockIdx.z;
    if (sx >= 2 * mc0) return;
    const long long kS = 1LL << (mshift - 1);
    const long long x0 = max(0LL, (long long)sx * kS - 1), x1 = min(sd0 - 1, (long long)sx * kS + kS + 1);
    const long long y0 = max(0LL, (long long)sy * kS - 1), y1 = min(sd1 - 1, (long long)sy * kS + kS + 1);
    const long long z0 = max(0LL, (long long)sz * kS - 1), z1 = min(sd2 - 1, (long long)sz * kS + kS + 1);
    float lo = INFINITY, hi = -INFINITY;
    if (x0 <= x1 && y0 <= y1 && z0 <= z1) {
        for (long long z = z0; z <= z1; ++z)
            for (long long y = y0; y <= y1; ++y) {
                const float* row = vox + (z * sd1 + y) * sd0;
                for (long long x = x0; x <= x1; ++x) {
                    const float v = __ldg(row + x);
                    lo = fminf(lo, v);
                    hi = fmaxf(hi, v);
                }
            }
    }
    const long long mc = ((long long)(sz >> 1) * mc1 + (sy >> 1)) * mc0 + (sx >> 1);
    sub[mc * 8 + ((sx & 1) | ((sy & 1) << 1) | ((sz & 1) << 2))] = make_float2(lo, hi);
}

// Coefficient quads: the slot of voxel (x, y, z) holds the bilinear coefficients of the
// z-face of the cell it anchors, {a, b - a, c - a, d - c - b + a} for the corners a = v(x, y), b = v(x+1, y),
// c = v(x, y+1), d = v(x+1, y+1), so a face value is a + B fx + C fy + D fx fy (3 FFMA) and a trilinear
// sample is two 16-byte loads.  The grid carries one apron voxel on every side (index -1 and sd along each
// axis, coordinates clamped, hence zero slopes there): sample positions that float rounding puts a hair
// outside the stored box need no clamp in the marcher and reproduce the oracle's clamped cell exactly.
__global__ void quad_kernel(const float* __restrict__ vox, long long sd0, long long sd1, long long sd2,
                            float4* __restrict__ quad, int half, int* __restrict__ range_flag) {
    const long long qd0 = sd0 + 2, qd1 = sd1 + 2;
#if DPRT_QUAD_YFAST
    const long long qy = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (qy >= qd1) return;
    const long long qx = blockIdx.y, qz = blockIdx.z;
#else
    const long long qx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (qx >= qd0) return;
    const long long qy = blockIdx.y, qz = blockIdx.z;
#endif
    auto cl = [](long long v, long long n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); };
    const long long x0 = cl(qx - 1, sd0), x1 = cl(qx, sd0);
    const long long y0 = cl(qy - 1, sd1), y1 = cl(qy, sd1);
    const long long z = cl(qz - 1, sd2);
    const float* r0 = vox + (z * sd1 + y0) * sd0;
    const float* r1 = vox + (z * sd1 + y1) * sd0;
    const float a = r0[x0], b = r0[x1], c = r1[x0], d = r1[x1];
#if DPRT_QUAD_YFAST
    const long long qi = (qz * qd0 + qx) * qd1 + qy;
#else
    const long long qi = (qz * qd1 + qy) * qd0 + qx;
#endif
    if (half) {  // DPRT_BRICK_HALF_QUADS: the same coefficients, each rounded once to fp16
        // the stated fp16 bound is for values in [0, 1]; the rounding error grows with |value|
        // and the slopes overflow past 65504: flag any voxel outside [-kHalfQuadRange, kHalfQuadRange]
        if (!(fabsf(a) <= kHalfQuadRange)) *range_flag = 1;
        const __half2 ab = __floats2half2_rn(a, b - a), cd = __floats2half2_rn(c - a, (d - c) - (b - a));
        reinterpret_cast<uint2*>(quad)[qi] = make_uint2(*reinterpret_cast<const unsigned*>(&ab),
                                                        *reinterpret_cast<const unsigned*>(&cd));
    } else {
#if DPRT_QUAD_OCTET
        // the cell's far z-face too: the quad the next apron layer would hold
        const long long zf = cl(qz, sd2);
        const float* s0 = vox + (zf * sd1 + y0) * sd0;
        const float* s1 = vox + (zf * sd1 + y1) * sd0;
        const float e = s0[x0], f = s0[x1], g = s1[x0], h = s1[x1];
        quad[2 * qi] = make_float4(a, b - a, c - a, (d - c) - (b - a));
        quad[2 * qi + 1] = make_float4(e, f - e, g - e, (h - g) - (f - e));
#else
        quad[qi] = make_float4(a, b - a, c - a, (d - c) - (b - a));
#endif
    }
}

cudaError_t launch_macrocells(const DeviceBrick& b, cudaStream_t stream) {
    {
        dim3 qb(256);
#if DPRT_QUAD_YFAST
        dim3 qg((unsigned)((b.qd[1] + 255) / 256), (unsigned)b.qd[0], (unsigned)b.qd[2]);
#else
        dim3 qg((unsigned)((b.qd[0] + 255) / 256), (unsigned)b.qd[1], (unsigned)b.qd[2]);
#endif
        quad_kernel<<<qg, qb, 0, stream>>>(b.vox, b.sd[0], b.sd[1], b.sd[2], b.quad, b.half_quads,
                                           b.counters + 2 * DPRT_MARCH_COUNTER_SLOTS);
    }
    dim3 block(64);
    dim3 grid((unsigned)((b.mcd[0] + 63) / 64), (unsigned)b.mcd[1], (unsigned)b.mcd[2]);
    macrocell_kernel<<<grid, block, 0, stream>>>(b.vox, b.sd[0], b.sd[1], b.sd[2], (int)b.mcd[0], (int)b.mcd[1],
                                                 (int)b.mcd[2], b.mshift, b.macro);
    if (DPRT_SUBBLOCK) {
        dim3 sgrid((unsigned)((2 * b.mcd[0] + 63) / 64), (unsigned)(2 * b.mcd[1]), (unsigned)(2 * b.mcd[2]));
        subblock_kernel<<<sgrid, block, 0, stream>>>(b.vox, b.sd[0], b.sd[1], b.sd[2], (int)b.mcd[0],
                                                     (int)b.mcd[1], (int)b.mcd[2], b.mshift, b.sub);
    }
    return cudaGetLastError();
}

}  // namespace dprt

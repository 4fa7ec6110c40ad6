// Per-rank DVR ray marcher for one brick (sm_100a).
//
// Takes the slot of the reference's per-rank local work, trace_local_round -> trace_nearest_batch
// (pkg/src/dprt/engine.py:254-279, bvh.py:284-296): one thread per pixel of the full frame, outputs
// written in place.  Semantics: DESIGN.md §2; CPU statement: oracle/dvr_oracle.c.
//
// * Ray setup (primary ray geom.py:240-259, slab clip geom.py:171-209, lattice range) is float64 with
//   explicitly rounded intrinsics, so it is bit-identical to the oracle: ownership of every lattice
//   sample (and so the per-pixel sample count) is integer-exact and partition-invariant.
// * The sample loop is float32: incremental position (FMA), trilinear from the f32 brick through the
//   read-only path, transfer function from shared memory, front-to-back premultiplied blend, early ray
//   termination.  Exact empty-space skipping jumps over macrocells whose (1-voxel dilated) value range
//   maps to alpha == 0 everywhere in the TF: the skipped samples would add exact zeros.
// * Two kernels.  ray_setup: one thread per pixel (warps = 8x4 pixel tiles) does the exact f64 setup,
//   writes zeros / sample counts for pixels that miss the brick, and appends the rays that hit it to a
//   compact queue, one contiguous chunk per warp tile (spatially coherent).  march: a persistent grid
//   of warps drains the queue; each lane owns one ray, and when too many lanes of a warp have finished
//   the warp refills them from the queue in one batch, so lanes stay busy and no SM waits on a tail of
//   heavy tiles.

#include <math.h>

#include <mutex>

#include "common.cuh"

#ifndef DPRT_BOUNDS_CHECK
#define DPRT_BOUNDS_CHECK 0
#endif

namespace dprt {

#if DPRT_COUNTERS
__device__ unsigned long long g_counters[4];  // shaded samples, contributing samples, skip steps, rays
#define DPRT_COUNT(i, v) atomicAdd(&g_counters[i], (unsigned long long)(v))
#else
#define DPRT_COUNT(i, v) ((void)0)
#endif

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// geom.py:240-259 with every f64 op explicitly rounded (no FMA contraction), matching dvr_oracle.c.
__device__ __forceinline__ void primary_dir(const MarchArgs& a, int px, int py, double d[3]) {
    double sx = __dmul_rn(__dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn((double)px, 0.5), (double)a.W), 2.0), 1.0),
                          a.half_w);
    double sy = __dmul_rn(__dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn((double)py, 0.5), (double)a.H), 2.0)),
                          a.half_h);
    double dx = __dadd_rn(__dadd_rn(a.f[0], __dmul_rn(sx, a.r[0])), __dmul_rn(sy, a.u[0]));
    double dy = __dadd_rn(__dadd_rn(a.f[1], __dmul_rn(sx, a.r[1])), __dmul_rn(sy, a.u[1]));
    double dz = __dadd_rn(__dadd_rn(a.f[2], __dmul_rn(sx, a.r[2])), __dmul_rn(sy, a.u[2]));
    double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    d[0] = __ddiv_rn(dx, n);
    d[1] = __ddiv_rn(dy, n);
    d[2] = __ddiv_rn(dz, n);
}

// geom.py:171-200: slab interval of the ray against a box (empty box -> miss; a zero direction component
// is inside-or-miss for that slab), every f64 op explicitly rounded, matching dvr_oracle.c.
__device__ __forceinline__ bool slab_interval(const double o[3], const double d[3], const double lo[3],
                                              const double hi[3], double* pt0, double* pt1) {
    if (lo[0] > hi[0] || lo[1] > hi[1] || lo[2] > hi[2]) return false;
    double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double di = d[i], oi = o[i];
        if (di == 0.0) {
            if (oi < lo[i] || oi > hi[i]) return false;
            continue;
        }
        const double inv = __ddiv_rn(1.0, di);
        double ta = __dmul_rn(__dsub_rn(lo[i], oi), inv);
        double tb = __dmul_rn(__dsub_rn(hi[i], oi), inv);
        if (ta > tb) {
            const double s = ta;
            ta = tb;
            tb = s;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t1 < t0) return false;
    }
    *pt0 = t0;
    *pt1 = t1;
    return true;
}

// clip to [0, inf) (geom.py:203-209) + lattice range.
__device__ __forceinline__ int64_t lattice_range(const MarchArgs& a, const double d[3], int64_t* k0) {
    double t0, t1;
    if (!slab_interval(a.o, d, a.blo, a.bhi, &t0, &t1)) return 0;
    if (t0 < 0.0) t0 = 0.0;
    if (t1 < t0) return 0;
    // t / dt: for a power-of-two dt the product with the exact inverse is the identical IEEE result
    const int64_t ka = (int64_t)ceil(a.inv_dt_pow2 != 0.0 ? __dmul_rn(t0, a.inv_dt_pow2) : __ddiv_rn(t0, a.dt));
    const int64_t kb = (int64_t)ceil(a.inv_dt_pow2 != 0.0 ? __dmul_rn(t1, a.inv_dt_pow2) : __ddiv_rn(t1, a.dt));
    *k0 = ka;
    return kb > ka ? kb - ka : 0;
}

#if DPRT_SETUP_FAST
// Fast ray setup.  The same ray as primary_dir + lattice_range, in f64 with FMA, a Newton-refined approximate
// rsqrt for the normalisation and Newton-refined reciprocals for the slab divisions -- no correctly rounded
// division or square root (each a MUFU + 7 DFMA + a slow-path test).  Its values differ from the exact
// setup's by a few units in the last place, scaled up for a direction component d_i by S / |d_i| (the
// cancellation in f + sx r + sy u, S = 1 + half_w + half_h).  Each slab bound t carries that error bound e;
// the lattice range [ceil(max(t0, 0) / dt), ceil(t1 / dt)) is taken only when no lattice point lies within
// the widened interval of either end, so it equals the exact one; otherwise (a near-zero direction
// component, an end within ~1e-12 of a lattice point, an empty box) the caller runs the exact setup.
// Returns false for "not proven".  d[] (start position and step of the f32 march) is accurate to ~1e-15.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

// ceil(u) for every u in [lo, hi], or INT64_MIN if the interval holds a lattice point in its interior
__device__ __forceinline__ int64_t ceil_if_unique(double lo, double hi) {
    const double c = ceil(lo);
    return hi <= c ? (int64_t)c : INT64_MIN;
}

__device__ __forceinline__ bool fast_range(const MarchArgs& a, int px, int py, double d[3], int64_t* k0,
                                           int64_t* n) {
    const double sx = fma((double)px + 0.5, a.fs_iw2, -1.0) * a.half_w;
    const double sy = fma(-((double)py + 0.5), a.fs_ih2, 1.0) * a.half_h;
    double D[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) D[i] = fma(sy, a.u[i], fma(sx, a.r[i], a.f[i]));
    const double rn = rsqrt_nr(fma(D[0], D[0], fma(D[1], D[1], D[2] * D[2])));
    // |D| >= 1 (f is a unit vector orthogonal to r and u), so the absolute error of d_i is ~ 2^-50 S
    // per-axis relative bound of t against the exact setup's t: 2^-42 (S / |d_i| + 1) -- the analysis gives
    // 2^-46 S / |d_i| (D: a few roundings of terms <= S each way; |D| >= 1) + 2^-50 (rcp, products, t / dt)
    constexpr double kRel = 0x1p-42;
    double t0lo = -INFINITY, t0hi = -INFINITY, t1lo = INFINITY, t1hi = INFINITY;
    bool ok = a.fs_ok != 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        d[i] = D[i] * rn;
        const double ad = fabs(d[i]);
        ok = ok && ad > 1e-6;
        const double inv = rcp_nr(d[i]);
        const double ta = a.fs_L[i] * inv, tb = a.fs_H[i] * inv;
        const double tmn = fmin(ta, tb), tmx = fmax(ta, tb);
        const double rel = kRel * (a.fs_S / ad + 1.0);
        const double emn = fabs(tmn) * rel, emx = fabs(tmx) * rel;
        t0lo = fmax(t0lo, tmn - emn);
        t0hi = fmax(t0hi, tmn + emn);
        t1lo = fmin(t1lo, tmx - emx);
        t1hi = fmin(t1hi, tmx + emx);
    }
    if (!ok) return false;
    // the exact path's t / dt (one more rounding; or an exact power-of-two scaling) lies in the widened range
    const double idt = a.fs_idt;
    const double u0lo = fmax(t0lo, 0.0) * idt, u0hi = fmax(t0hi, 0.0) * idt;
    const double u1lo = t1lo * idt, u1hi = t1hi * idt;
    constexpr double kW = 0x1p-50;
    const int64_t ka = ceil_if_unique(u0lo - fabs(u0lo) * kW, u0hi + fabs(u0hi) * kW);
    const int64_t kb = ceil_if_unique(u1lo - fabs(u1lo) * kW, u1hi + fabs(u1hi) * kW);
    if (ka == INT64_MIN || kb == INT64_MIN) return false;
    *k0 = ka;
    *n = kb > ka ? kb - ka : 0;
    return true;
}
#endif

// Known-answer kernels: the marcher's own device functions applied to caller-supplied rays, so the
// reference's golden vectors (camera rays, slab intervals) are checked on the GPU code itself.
__global__ void kat_slab_kernel(const double* __restrict__ o, const double* __restrict__ d,
                                const double* __restrict__ lo, const double* __restrict__ hi, int n,
                                double* __restrict__ t01, int* __restrict__ hit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double t0 = 0.0, t1 = 0.0;
    const bool h = slab_interval(o + 3 * i, d + 3 * i, lo + 3 * i, hi + 3 * i, &t0, &t1);
    hit[i] = h ? 1 : 0;
    t01[2 * i] = h ? t0 : 0.0;
    t01[2 * i + 1] = h ? t1 : 0.0;
}

__global__ void kat_primary_kernel(const MarchArgs a, double* __restrict__ out) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y;
    if (px >= a.W) return;
    double d[3];
    primary_dir(a, px, py, d);
    double* o = out + 3 * ((long long)py * a.W + px);
    o[0] = d[0];
    o[1] = d[1];
    o[2] = d[2];
}

cudaError_t launch_kat_slab(const double* o, const double* d, const double* lo, const double* hi, int n, double* t01,
                            int* hit) {
    kat_slab_kernel<<<(n + 127) / 128, 128>>>(o, d, lo, hi, n, t01, hit);
    return cudaGetLastError();
}

cudaError_t launch_kat_primary(const MarchArgs& a, double* out) {
    kat_primary_kernel<<<dim3((a.W + 127) / 128, a.H), 128>>>(a, out);
    return cudaGetLastError();
}

#ifndef DPRT_REFILL_BELOW
#define DPRT_REFILL_BELOW 8
#endif
#ifndef DPRT_STEPS_PER_CHECK
#define DPRT_STEPS_PER_CHECK 16
#endif
constexpr int kRefillBelow = DPRT_REFILL_BELOW;  // refill a warp's idle lanes once fewer than this many march
constexpr int kStepsPerCheck = DPRT_STEPS_PER_CHECK;  // march steps between refill checks

// Pass 1: exact ray setup, zero-fill of pixels that miss the brick, compaction of the ones that hit.
__global__ void __launch_bounds__(kTileX * kTileY) ray_setup_kernel(const MarchArgs a) {
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int px = blockIdx.x * kTileX + (warp & 1) * 8 + (lane & 7);
    const int py = blockIdx.y * kTileY + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = px < a.W && py < a.H;
    const bool in_rect = inside && px >= a.rect[0] && py >= a.rect[1] && px < a.rect[2] && py < a.rect[3];
    int64_t k0 = 0, n = 0;
    double d[3];
    if (in_rect) {
        primary_dir(a, px, py, d);
        n = lattice_range(a, d, &k0);
    }
    const int64_t pix = (int64_t)py * a.W + px;
    if (inside) {
        if (a.samples) a.samples[pix] = (uint32_t)n;
        if (n == 0) a.out[pix] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool hit = n > 0;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (!m) return;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(a.counters, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (!hit) return;
    const int slot = base + __popc(m & ((1u << lane) - 1));
    // start position in local (stored) continuous index space and the per-sample step
    const double t0 = __dmul_rn((double)k0, a.dt);
    float p0[3], st[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double p = (a.o[i] + t0 * d[i] - a.origin[i]) * a.inv_spacing_d[i];
        p0[i] = (float)(p - a.stored_lo_d[i]);
        st[i] = (float)(a.dt * d[i]) * a.inv_spacing[i];
    }
    a.rays[2 * slot] = make_float4(p0[0], p0[1], p0[2], __int_as_float((int)pix));
    a.rays[2 * slot + 1] = make_float4(st[0], st[1], st[2], __int_as_float((int)n));
}

// One trilinear sample from the two coefficient quads of its cell (field.cu quad_kernel): each z-face is
// a + B fx + C fy + D fx fy, then a lerp along z (DESIGN.md §2.5 / §4.1).
__device__ __forceinline__ float trilerp(const float4 q0, const float4 q1, float fx, float fy, float fxy, float fz) {
    const float e0 = fmaf(q0.w, fxy, fmaf(q0.z, fy, fmaf(q0.y, fx, q0.x)));
    const float e1 = fmaf(q1.w, fxy, fmaf(q1.z, fy, fmaf(q1.y, fx, q1.x)));
    return fmaf(fz, e1 - e0, e0);
}

// fp16 quads (DPRT_BRICK_HALF_QUADS): the cell's two z-faces as 8-byte loads, widened to f32.
__device__ __forceinline__ void load_half_quads(const uint2* q, int qsz, float4& qa, float4& qb) {
    const uint2 ha = __ldg(q), hb = __ldg(q + qsz);
    const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&ha.x));
    const float2 a1 = __half22float2(*reinterpret_cast<const __half2*>(&ha.y));
    const float2 b0 = __half22float2(*reinterpret_cast<const __half2*>(&hb.x));
    const float2 b1 = __half22float2(*reinterpret_cast<const __half2*>(&hb.y));
    qa = make_float4(a0.x, a0.y, a1.x, a1.y);
    qb = make_float4(b0.x, b0.y, b1.x, b1.y);
}

// Quad offset of cell (ix, iy, iz) from the stored voxel (0, 0, 0) (memory order: DPRT_QUAD_YFAST); the unit
// stride is a plain add, so the index costs two IMADs in either order.
template <typename T>
__device__ __forceinline__ T quad_offset(T ix, T iy, T iz, T qsx, T qsy, T qsz) {
#if DPRT_QUAD_YFAST
    (void)qsy;
    return iz * qsz + ix * qsx + iy;
#else
    (void)qsx;
    return iz * qsz + iy * qsy + ix;
#endif
}

// f32 coefficient octet (DPRT_QUAD_OCTET): both z-faces of the cell in one 256-bit load.
__device__ __forceinline__ void load_octet(const float4* p, float4& qa, float4& qb) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(qa.x), "=f"(qa.y), "=f"(qa.z), "=f"(qa.w), "=f"(qb.x), "=f"(qb.y), "=f"(qb.z), "=f"(qb.w)
        : "l"(p));
}

// DPRT_BOUNDS_CHECK builds trap on a quad index (relative to qorg, both loads) outside the apron grid.
__device__ __forceinline__ void quad_bounds_check(const MarchArgs& a, long long qi) {
#if DPRT_BOUNDS_CHECK
    const long long org = (long long)a.qsz + a.qsy + a.qsx, total = (long long)a.qsz * (a.sd[2] + 2);
    if (qi + org < 0 || qi + org + a.qsz >= total) __trap();
#endif
}

// DPRT_BOUNDS_CHECK builds: every skip-distance load and every output store of the beam marcher traps
// outside its buffer (a debug build for the parity suite; compiled out otherwise)
__device__ __forceinline__ void skip_bounds_check(const MarchArgs& a, long long mci) {
#if DPRT_BOUNDS_CHECK
    if (mci < 0 || mci >= a.skip_n) __trap();
#else
    (void)a;
    (void)mci;
#endif
}

__device__ __forceinline__ void pix_bounds_check(const MarchArgs& a, long long pix) {
#if DPRT_BOUNDS_CHECK
    if (pix < 0 || pix >= (long long)a.W * a.H) __trap();
    if (!a.rgb8 && (pix - a.pix0 < 0 || pix - a.pix0 >= a.npix_buf) && (a.out || a.out16 || a.samples)) __trap();
#else
    (void)a;
    (void)pix;
#endif
}

// TF lookup and front-to-back premultiplied blend (§2.7) of one sample value.  Shared memory
// holds the entries (s_tf) and, in a second array, next - entry (s_dtf; 16-byte strides keep neighbouring
// lanes' LDS.128 on distinct banks); the last entry's difference is zero, so x = n - 1 needs no clamp.
__device__ __forceinline__ void tf_blend(const float4* s_tf, const float4* s_dtf, float v, float tns, float tno,
                                         float top, float& C0, float& C1, float& C2, float& A) {
    const float x = __saturatef(fmaf(v, tns, tno)) * top;
    const int ti = (int)x;
    const float tfr = x - (float)ti;
    const float4 e0 = s_tf[ti], de = s_dtf[ti];
    const float w = (1.f - A) * fmaf(tfr, de.w, e0.w);
    C0 = fmaf(w, fmaf(tfr, de.x, e0.x), C0);
    C1 = fmaf(w, fmaf(tfr, de.y, e0.y), C1);
    C2 = fmaf(w, fmaf(tfr, de.z, e0.z), C2);
    A += w;
}

// Pass 2: persistent warps march the queued rays.
#ifndef DPRT_MARCH_MINBLOCKS
#define DPRT_MARCH_MINBLOCKS 4
#endif
__global__ void __launch_bounds__(kTileX * kTileY, DPRT_MARCH_MINBLOCKS) march_kernel(const MarchArgs a) {
    // TF as entries + (next - entry) differences: the lerp e0 + (e1 - e0) * f becomes one FMA per channel
    // (the difference is formed once here instead of per sample).
    extern __shared__ float4 s_tf[];  // n_tf entries, then n_tf differences (dynamic)
    const int tid = threadIdx.x;
    for (int i = tid; i < a.n_tf; i += blockDim.x) {
        const float4 e0 = a.tf[i];
        const float4 e1 = i + 1 < a.n_tf ? a.tf[i + 1] : e0;
        s_tf[i] = e0;
        s_tf[a.n_tf + i] = make_float4(e1.x - e0.x, e1.y - e0.y, e1.z - e0.z, e1.w - e0.w);
    }
    __syncthreads();

    const int lane = tid & 31;
    const int total = a.counters[0];  // written by ray_setup_kernel, which completed before this launch
    const int chx = a.chi[0], chy = a.chi[1], chz = a.chi[2];
    const float4* __restrict__ qorg = a.qorg;
    const int qsx = a.qsx, qsy = a.qsy, qsz = a.qsz;
    const uint8_t* __restrict__ skipd = a.skipd;
    const int mcd0 = a.mcd[0], mcd1 = a.mcd[1], skip = a.skip;
    const int ms = a.mshift;  // macrocell shift of this brick
    const float tns = a.tf_ns, tno = a.tf_no, top = (float)(a.n_tf - 1), ert = a.ert;

    bool have = false, exhausted = false;
    int pix = 0, nn = 0, j = 0;
#if DPRT_COUNTERS
    unsigned long long c_shade = 0, c_contrib = 0, c_skip = 0, c_rays = 0;
#endif
    float p0[3] = {0.f, 0.f, 0.f}, st[3] = {0.f, 0.f, 0.f}, ist[3] = {0.f, 0.f, 0.f};
    float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
    while (true) {
        unsigned act = __ballot_sync(0xffffffffu, have);
        if (!exhausted && __popc(act) < kRefillBelow) {
            const unsigned need = ~act;
            const int k = __popc(need);
            int base = 0;
            if (lane == 0) base = atomicAdd(a.counters + 1, k);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base + k >= total) exhausted = true;
            if (!have) {
                const int idx = base + __popc(need & ((1u << lane) - 1));
                if (idx < total) {
                    const float4 r0 = __ldg(a.rays + 2 * idx), r1 = __ldg(a.rays + 2 * idx + 1);
                    p0[0] = r0.x; p0[1] = r0.y; p0[2] = r0.z;
                    st[0] = r1.x; st[1] = r1.y; st[2] = r1.z;
#pragma unroll
                    for (int i = 0; i < 3; ++i) ist[i] = st[i] != 0.f ? 1.f / st[i] : 0.f;
                    pix = __float_as_int(r0.w);
                    nn = __float_as_int(r1.w);
                    j = 0;
                    C0 = C1 = C2 = A = 0.f;
                    have = true;
#if DPRT_COUNTERS
                    ++c_rays;
#endif
                }
            }
            act = __ballot_sync(0xffffffffu, have);
        }
        if (act == 0) {
#if DPRT_COUNTERS
            DPRT_COUNT(0, c_shade);
            DPRT_COUNT(1, c_contrib);
            DPRT_COUNT(2, c_skip);
            DPRT_COUNT(3, c_rays);
#endif
            break;
        }
        for (int s = 0; have && s < kStepsPerCheck; ++s) {
            if (j >= nn) {
                a.out[pix] = make_float4(C0, C1, C2, A);
                have = false;
                break;
            }
            const float fs = (float)j;
            const float ux = fmaf(fs, st[0], p0[0]);
            const float uy = fmaf(fs, st[1], p0[1]);
            const float uz = fmaf(fs, st[2], p0[2]);
            const int ix = min(__float2int_rd(fmaxf(ux, 0.f)), chx);
            const int iy = min(__float2int_rd(fmaxf(uy, 0.f)), chy);
            const int iz = min(__float2int_rd(fmaxf(uz, 0.f)), chz);
            const int mx = ix >> ms, my = iy >> ms, mz = iz >> ms;
            // Skip distance of this sample's macrocell.  An empty macrocell's sample would add exact
            // zeros: drop it and jump over the empty cube around it.
            const int mc = (mz * mcd1 + my) * mcd0 + mx;
            const int dist = skip ? (int)__ldg(skipd + mc) : 0;
            if (dist > 0) {
                // jump to the exit of the empty cube of macrocells [m - dist + 1, m + dist]
                float je = 3.0e38f;
                if (st[0] != 0.f)
                    je = fminf(je, ((float)((st[0] > 0.f ? mx + dist : mx - dist + 1) << ms) - p0[0]) * ist[0]);
                if (st[1] != 0.f)
                    je = fminf(je, ((float)((st[1] > 0.f ? my + dist : my - dist + 1) << ms) - p0[1]) * ist[1]);
                if (st[2] != 0.f)
                    je = fminf(je, ((float)((st[2] > 0.f ? mz + dist : mz - dist + 1) << ms) - p0[2]) * ist[2]);
                const int jn = je < (float)nn ? (int)ceilf(je) : nn;
                j = jn > j ? jn : j + 1;
#if DPRT_COUNTERS
                ++c_skip;
#endif
                continue;
            }
            // trilinear + TF (§2.6) + front-to-back blend (§2.7) of one sample
            const int qi = quad_offset(ix, iy, iz, qsx, qsy, qsz);
            quad_bounds_check(a, qi);
            const float fx = __saturatef(ux - (float)ix), fy = __saturatef(uy - (float)iy);
#if DPRT_QUAD_OCTET
            float4 oa, ob;
            load_octet(qorg + 2 * (long long)qi, oa, ob);
            const float v = trilerp(oa, ob, fx, fy, fx * fy, __saturatef(uz - (float)iz));
#else
            const float4* q = qorg + qi;
            const float v = trilerp(__ldg(q), __ldg(q + qsz), fx, fy, fx * fy, __saturatef(uz - (float)iz));
#endif
            tf_blend(s_tf, s_tf + a.n_tf, v, tns, tno, top, C0, C1, C2, A);
            ++j;
            if (A >= ert) j = nn;  // early ray termination: the next step finishes the ray
        }
    }
}

// Pass 2 (beam variant): a warp marches one 8x4 pixel tile as a coherent beam, slab by slab along the
// beam's dominant axis (slab = one macrocell layer).  Per slab the warp bounds the beam's cells on the
// two other axes with warp reductions, reads those macrocells' skip distances cooperatively and either
// jumps every lane over the empty slabs at once or lets each lane shade its samples in the slab.  No
// per-sample skip test, lanes stay in step, and the 32 rays read the same L1 lines.
#ifndef DPRT_BEAM_UNROLL
#define DPRT_BEAM_UNROLL 4  // re-swept after every traversal change (4 -> 3 with the probe loop, 3 -> 4 with 4^3 macrocells)
#endif
constexpr int kBeamUnroll = DPRT_BEAM_UNROLL;

#ifndef DPRT_BEAM_W
#define DPRT_BEAM_W 4
#endif
constexpr int kBeamW = DPRT_BEAM_W;  // beam = kBeamW x (32 / kBeamW) pixels
#ifndef DPRT_BEAM_W_DEEP
#define DPRT_BEAM_W_DEEP DPRT_BEAM_W  // the large-brick configuration's beam width
#endif
#ifndef DPRT_MISS_TEST
#define DPRT_MISS_TEST 0  // 1: warps whose rays all miss skip the f64 setup (measured +0.4 % c2, +1 % config 3)
#endif
#ifndef DPRT_PROBE_LOOP
#define DPRT_PROBE_LOOP 1  // per-lane probe loops over consecutive empty cubes (0: one jump per warp iteration)
#endif
#if !DPRT_BEAM_PROBE
#undef DPRT_PROBE_PREFETCH
#define DPRT_PROBE_PREFETCH 0  // the prefetch feeds the per-lane probe
#endif
#ifndef DPRT_PROBE_PREFETCH
#define DPRT_PROBE_PREFETCH 1  // the next probe's skip distance loaded during the slab step (c2 -0.6 %, config 3 -1 %)
#endif
#ifndef DPRT_JUMP_BRANCHFREE
#define DPRT_JUMP_BRANCHFREE 1
#endif
#ifndef DPRT_SLAB_SHIFT
#if DPRT_BEAM_PROBE
#define DPRT_SLAB_SHIFT (DPRT_MACRO_SHIFT + 1)  // slab thickness (cells, log2): 16 since the probe loop (c2 -4 %)
#else
#define DPRT_SLAB_SHIFT DPRT_MACRO_SHIFT  // beam-wide skipping steps whole macrocell layers
#endif
#endif
constexpr int kSlabShift = DPRT_SLAB_SHIFT;
#ifndef DPRT_SLAB_SHIFT_DEEP
#define DPRT_SLAB_SHIFT_DEEP DPRT_MACRO_SHIFT  // large bricks: 8-cell slabs (all 8 config-3 ranks: critical path -2 %)
#endif

// Tile-queue order: 1 = rows of tiles centre-out (default), 2 = rows and the tiles within a
// row centre-out, 0 = row-major.  The queue then ends with the short rays at the footprint's top and bottom
// edges instead of whatever rows come last, which shortens the launch's tail (c2 0.243 -> 0.227 ms).
#ifndef DPRT_TILE_ORDER
#define DPRT_TILE_ORDER 1
#endif
#ifndef DPRT_BLEND_PREFIX
#define DPRT_BLEND_PREFIX 0
#endif
#ifndef DPRT_TILE_PREFETCH
#define DPRT_TILE_PREFETCH 0  // measured: c2 0.227 -> 0.313 ms (the live index register spills in the 80-register budget)
#endif
// k-th index of 0..n-1 in centre-out order: m, m-1, m+1, m-2, m+2, ... (m = n / 2)
__device__ __forceinline__ int center_out(int k, int n) {
    const int m = n >> 1, d = (k + 1) >> 1;
    return (k & 1) ? m - d : m + d;
}

__device__ __forceinline__ int fl2cell(float u, int hi) { return min(__float2int_rd(fmaxf(u, 0.f)), hi); }

// A pixel of the RGBA partial: the local buffer (out / out16 at pix - pix0) or, in the fused march +
// exchange (kPush, dprt_march_push), its row block's owner's inbox over NVLink.
// s_blk (kPush): the row -> row-block table in shared memory, built once per CTA in the kernel's prologue.
template <bool kPush>
__device__ __forceinline__ void store_partial(const MarchArgs& a, const uint8_t* s_blk, long long pix, int y, float C0,
                                              float C1, float C2, float A) {
    if constexpr (kPush) {
        const int b = s_blk[y];
        const long long e = pix - (long long)a.push_row[b] * a.W;
#if DPRT_BOUNDS_CHECK
        if (b < 0 || b >= a.push_P || e < 0 || e >= (long long)(a.push_row[b + 1] - a.push_row[b]) * a.W) __trap();
#endif
        if (a.half_out) {
            const __half2 rg = __floats2half2_rn(C0, C1), ba = __floats2half2_rn(C2, A);
            reinterpret_cast<uint2*>(a.push_dst[b])[e] = make_uint2(*reinterpret_cast<const unsigned*>(&rg),
                                                                    *reinterpret_cast<const unsigned*>(&ba));
        } else {
            reinterpret_cast<float4*>(a.push_dst[b])[e] = make_float4(C0, C1, C2, A);
        }
    } else {
        (void)y;
        (void)s_blk;
#if DPRT_BOUNDS_CHECK
        if (pix - a.pix0 < 0 || pix - a.pix0 >= a.npix_buf) __trap();
#endif
        if (a.half_out) {
            const __half2 rg = __floats2half2_rn(C0, C1), ba = __floats2half2_rn(C2, A);
            a.out16[pix - a.pix0] = make_uint2(*reinterpret_cast<const unsigned*>(&rg),
                                               *reinterpret_cast<const unsigned*>(&ba));
        } else {
            a.out[pix - a.pix0] = make_float4(C0, C1, C2, A);
        }
    }
}

// The pixels no beam covers -- rows [y0, y1) outside the footprint rectangle -- get their "nothing here"
// value inside the march kernel itself (no separate fill or memset pass): the tone-mapped background for
// the fused RGB8 frame, a clear fragment (0) for an RGBA partial.  Blocks take whole rows, threads 4-pixel
// groups; a group straddling the rectangle's edge writes only its outside pixels (the beams own the inside).
template <bool kPush>
__device__ void fill_outside_rect(const MarchArgs& a, const uint8_t* s_blk, int y0, int y1, int unit, int nunits, int t,
                                  int nt) {
    const uint32_t cr = (uint32_t)floorf(fminf(fmaxf(a.bg[0], 0.f), 1.f) * 255.f + 0.5f);
    const uint32_t cg = (uint32_t)floorf(fminf(fmaxf(a.bg[1], 0.f), 1.f) * 255.f + 0.5f);
    const uint32_t cb = (uint32_t)floorf(fminf(fmaxf(a.bg[2], 0.f), 1.f) * 255.f + 0.5f);
    const int W = a.W, qpr = (W + 3) / 4;  // 4-pixel groups per row (no index division: rows per block)
    for (int y = y0 + unit; y < y1; y += nunits) {
#if DPRT_BOUNDS_CHECK
        if (y < 0 || y >= a.H) __trap();
#endif
        const bool row_out = y < a.rect[1] || y >= a.rect[3];
        for (int q = t; q < qpr; q += nt) {
            const int x0 = 4 * q;
            if (!row_out && x0 >= a.rect[0] && x0 + 4 <= a.rect[2]) continue;  // inside: the beams' pixels
            const long long i0 = (long long)y * W + x0;
            if (a.rgb8) {
                uint8_t* dst = a.rgb8 + 3 * i0;
                const bool all = x0 + 4 <= W && (row_out || x0 + 4 <= a.rect[0] || x0 >= a.rect[2]);
                if (all && (reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
                    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
                    d32[0] = cr | (cg << 8) | (cb << 16) | (cr << 24);
                    d32[1] = cg | (cb << 8) | (cr << 16) | (cg << 24);
                    d32[2] = cb | (cr << 8) | (cg << 16) | (cb << 24);
                    continue;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int x = x0 + k;
                    if (x >= W || (!row_out && x >= a.rect[0] && x < a.rect[2])) continue;
                    dst[3 * k] = (uint8_t)cr;
                    dst[3 * k + 1] = (uint8_t)cg;
                    dst[3 * k + 2] = (uint8_t)cb;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int x = x0 + k;
                    if (x >= W || (!row_out && x >= a.rect[0] && x < a.rect[2])) continue;
                    store_partial<kPush>(a, s_blk, i0 + k, y, 0.f, 0.f, 0.f, 0.f);
                }
            }
        }
    }
}

// A pixel inside the footprint whose ray adds nothing (no owned sample, or a beam that misses the brick).
template <bool kPush>
__device__ __forceinline__ void write_clear(const MarchArgs& a, const uint8_t* s_blk, int pix, int py) {
    if (a.rgb8) {
        pix_bounds_check(a, pix);
        uint8_t* dst = a.rgb8 + 3 * (size_t)pix;
#pragma unroll
        for (int c = 0; c < 3; ++c) dst[c] = (uint8_t)floorf(fminf(fmaxf(a.bg[c], 0.f), 1.f) * 255.f + 0.5f);
    } else {
        store_partial<kPush>(a, s_blk, pix, py, 0.f, 0.f, 0.f, 0.f);
    }
}

#ifndef DPRT_DEEP_UNROLL
#define DPRT_DEEP_UNROLL 6
#endif
#ifndef DPRT_DEEP_MINBLOCKS
#define DPRT_DEEP_MINBLOCKS 2
#endif
constexpr int kDeepUnroll = DPRT_DEEP_UNROLL, kDeepBlocks = DPRT_DEEP_MINBLOCKS;
#ifndef DPRT_BEAM_MINBLOCKS
#define DPRT_BEAM_MINBLOCKS 3
#endif
#ifndef DPRT_BEAM_BLOCK
#define DPRT_BEAM_BLOCK 256
#endif
constexpr int kBeamBlock = DPRT_BEAM_BLOCK;  // threads per CTA (warps are independent beams)
// kWide: the brick holds >= 2^31 apron quads (a mass-balanced brick of a 2048^3 field can): quad offsets are
// unsigned 32-bit from the apron grid's first quad (+1 instruction per sample, ~2 %); other bricks keep the
// signed offsets from stored voxel (0, 0, 0).  (A 64-bit z-plane term measured 6-12 % slower.)
//
// kUnroll / kMinBlocks: samples per branch-free batch and CTAs per SM.  Small bricks (c2: ~0.3 GB of touched
// quads, L2 hit ~48 %) are issue / L1 bound and run 3 @ 3 CTAs (24 warps); large ones (c3: 2.5-4.4 GB of
// touched quads, L2 hit ~25 %) are memory-latency bound and run 6 @ 2 CTAs -- fewer warps, more loads in
// flight per warp (c3 slowest ranks -6 to -12 %, c2 +15 %).  Chosen per launch from the
// brick size (launch_march).
// kHalf: the brick's quads are 4 x fp16 (DPRT_BRICK_HALF_QUADS, opt-in): 8-byte loads, widened to f32 at once.
// kMark (diagnostic instantiation, dprt_march_stats): no image output; every real sample of a live ray sets
// its macrocell's byte in a.mark and the launch counts shaded / contributing samples into a.stats -- the
// macrocells the march must read (the roofline's needed bytes) and the shaded-sample rate.
// kPush: the fused march + exchange (dprt_march_push) -- partial pixels go to their row block owners' inboxes
// and the launch's last CTA raises the owners' epoch flags.
// kMS: the macrocell shift as a compile-time constant for the natural pairing (small-brick configuration
// with DPRT_MACRO_SHIFT_SMALL, large-brick configuration with DPRT_MACRO_SHIFT), 0 = read a.mshift at run
// time (the forced test configurations and the diagnostic instantiation; ~1 % slower).
template <bool kWide, int kUnroll, int kMinBlocks, bool kHalf, bool kMark = false, bool kPush = false, int kMS = 0>
__global__ void __launch_bounds__(kBeamBlock, kMinBlocks) march_beam_kernel(const MarchArgs a) {
    extern __shared__ float4 s_tf[];
    const int tid = threadIdx.x;
    for (int i = tid; i < a.n_tf; i += blockDim.x) {
        const float4 e0 = a.tf[i];
        const float4 e1 = i + 1 < a.n_tf ? a.tf[i + 1] : e0;
        s_tf[i] = e0;
        s_tf[a.n_tf + i] = make_float4(e1.x - e0.x, e1.y - e0.y, e1.z - e0.z, e1.w - e0.w);
    }
    uint8_t* s_blk = reinterpret_cast<uint8_t*>(s_tf + 2 * a.n_tf);  // kPush: row -> row block (H bytes)
    if constexpr (kPush) {
        for (int y = tid; y < a.H; y += blockDim.x) {
            int b = 0;
            while (b + 1 < a.push_P && y >= a.push_row[b + 1]) ++b;
            s_blk[y] = (uint8_t)b;
        }
    }
    __syncthreads();
    const unsigned FULL = 0xffffffffu;
    const int lane = tid & 31;
    const int rw = a.rect[2] - a.rect[0], rh = a.rect[3] - a.rect[1];
    constexpr bool kDeepBeam = kUnroll == kDeepUnroll && kMinBlocks == kDeepBlocks;
    constexpr int kBW = kDeepBeam ? DPRT_BEAM_W_DEEP : kBeamW, kBH = 32 / kBW;  // this configuration's beam
    const int tiles_x = (rw + kBW - 1) / kBW, tiles_y = (rh + kBH - 1) / kBH;
    const int ntiles = tiles_x * tiles_y;
    const int chx = a.chi[0], chy = a.chi[1], chz = a.chi[2];
    const float4* __restrict__ qorg = a.qorg;
    const float4* __restrict__ qorg1 = a.qorg + a.qsz;  // the cell's far z-face
    const unsigned qk = (unsigned)a.qsz + (unsigned)a.qsy + (unsigned)a.qsx;  // apron offset of stored voxel (0, 0, 0)
    const float4* __restrict__ qbase = a.qorg - (long long)(kHalf ? 1 : kQuadSlot) * qk;  // the apron grid's first slot (kWide)
    const float4* __restrict__ qbase1 = qbase + a.qsz;
    const uint2* __restrict__ hq_org = reinterpret_cast<const uint2*>(qbase) + qk;  // fp16 quads: 8-byte slots
    const int qsx = a.qsx, qsy = a.qsy, qsz = a.qsz;
    const uint8_t* __restrict__ skipd = a.skipd;
    const int mcd0 = a.mcd[0], mcd1 = a.mcd[1];
    const int ms = kMS ? kMS : a.mshift;  // macrocell shift of this brick (4^3 or 8^3 cells)
    constexpr bool kDeepCfg = kUnroll == kDeepUnroll && kMinBlocks == kDeepBlocks;
    constexpr int kSS = (DPRT_BEAM_PROBE && kDeepCfg) ? DPRT_SLAB_SHIFT_DEEP : kSlabShift;  // slab thickness
    const float tns = a.tf_ns, tno = a.tf_no, top = (float)(a.n_tf - 1), ert = a.ert;
    const float4* __restrict__ s_dtf = s_tf + a.n_tf;
#if DPRT_COUNTERS
    unsigned long long c_shade = 0, c_contrib = 0, c_skip = 0, c_rays = 0;
#endif
    unsigned long long m_shade = 0, m_contrib = 0;  // kMark only
#if DPRT_TILE_PREFETCH
    // the next tile's index is fetched while this tile marches: the queue atomic's round trip (hundreds of
    // cycles) no longer stalls the warp between tiles
    int next_tile = 0;
    if (lane == 0) next_tile = atomicAdd(a.counters + 1, 1);
#endif
    while (true) {
        int tile = 0;
#if DPRT_TILE_PREFETCH
        tile = __shfl_sync(FULL, next_tile, 0);
        if (tile >= ntiles) break;
        if (lane == 0) next_tile = atomicAdd(a.counters + 1, 1);
#else
        if (lane == 0) tile = atomicAdd(a.counters + 1, 1);
        tile = __shfl_sync(FULL, tile, 0);
        if (tile >= ntiles) break;
#endif
#if DPRT_TILE_ORDER
        // centre-out queue order: rows of tiles from the footprint's middle row outwards (and, with 2, the
        // tiles of a row from its middle outwards), so the queue ends with the short rays at the edges
        const int trow = center_out(tile / tiles_x, tiles_y);
        const int tcol = DPRT_TILE_ORDER >= 2 ? center_out(tile % tiles_x, tiles_x) : tile % tiles_x;
#else
        const int trow = tile / tiles_x, tcol = tile % tiles_x;
#endif
        const int px = a.rect[0] + tcol * kBW + (lane % kBW);
        const int py = a.rect[1] + trow * kBH + (lane / kBW);
        int nn = 0, pix = 0;
        float p0[3] = {0.f, 0.f, 0.f}, st[3] = {0.f, 0.f, 0.f};
        const bool inside = px < a.rect[2] && py < a.rect[3];
#if DPRT_MISS_TEST
        // conservative f32 pre-test against the owned box expanded by a margin: a warp all of whose rays miss
        // it needs no exact f64 setup (their exact sample counts are 0); any other warp runs the exact setup
        bool maybe = false;
        if (inside) {
            const float sxf = (((float)px + 0.5f) * a.mt_iw * 2.f - 1.f) * a.mt_hw;
            const float syf = (1.f - ((float)py + 0.5f) * a.mt_ih * 2.f) * a.mt_hh;
            float t0 = 0.f, t1 = 3.0e38f;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const float di = fmaf(syf, a.mt_u[i], fmaf(sxf, a.mt_r[i], a.mt_f[i]));
                const float inv = 1.f / di;  // IEEE: a zero component gives +-inf, an inside slab then no bound
                const float ta = a.mt_lo[i] * inv, tb = a.mt_hi[i] * inv;
                t0 = fmaxf(t0, fminf(ta, tb));
                t1 = fminf(t1, fmaxf(ta, tb));
            }
            maybe = !(t1 < t0);
        }
        if (!__any_sync(FULL, maybe)) {
            if (inside) {
                pix = py * a.W + px;
                if (!kMark && a.samples) a.samples[pix - a.pix0] = 0u;
            }
        } else
#endif
        if (inside) {
            // exact f64 ray setup for this lane's pixel, fused
            pix = py * a.W + px;
            double d[3];
            int64_t k0 = 0;
#if DPRT_SETUP_FAST
            int64_t n = 0;
            if (!fast_range(a, px, py, d, &k0, &n)) {
                primary_dir(a, px, py, d);
                n = lattice_range(a, d, &k0);
            }
#else
            primary_dir(a, px, py, d);
            const int64_t n = lattice_range(a, d, &k0);
#endif
            pix_bounds_check(a, pix);
            if (!kMark && a.samples) a.samples[pix - a.pix0] = (uint32_t)n;
            if (n > 0) {
                const double t0 = __dmul_rn((double)k0, a.dt);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const double pw = (a.o[i] + t0 * d[i] - a.origin[i]) * a.inv_spacing_d[i];
                    p0[i] = (float)(pw - a.stored_lo_d[i]);
                    st[i] = (float)(a.dt * d[i]) * a.inv_spacing[i];
                }
                nn = (int)n;
            }
        }
        const unsigned hitm = __ballot_sync(FULL, nn > 0);
        if (!hitm) {
            if (!kMark && inside && !a.accum) write_clear<kPush>(a, s_blk, pix, py);  // no ray of this beam meets the brick
            continue;
        }
#if DPRT_COUNTERS == 1
        c_rays += nn > 0;
#endif
        // dominant axis of the beam (from its first ray) and whether every ray agrees with it
        const int ref = __ffs(hitm) - 1;
        const float rx = __shfl_sync(FULL, st[0], ref), ry = __shfl_sync(FULL, st[1], ref), rz = __shfl_sync(FULL, st[2], ref);
        const float ax = fabsf(rx), ay = fabsf(ry), az = fabsf(rz);
        const int ka = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);
        // this ray's components permuted to (a, b, c) once, so the loops below index no arrays
        auto sel = [&](const float* v, int k3) { return k3 == 0 ? v[0] : (k3 == 1 ? v[1] : v[2]); };
        const float sa = sel(st, ka);
        const float pa = sel(p0, ka);
        const int cha = ka == 0 ? chx : (ka == 1 ? chy : chz);
        const bool pos = (ka == 0 ? rx : (ka == 1 ? ry : rz)) > 0.f;
#if !DPRT_BEAM_PROBE
        // beam-wide slab skipping (the measured alternative) bounds the beam's cells on the other two axes
        const int kb = ka == 0 ? 1 : 0, kc = ka == 2 ? 1 : 2;
        const float sb = sel(st, kb), sc = sel(st, kc);
        const float pb = sel(p0, kb), pc = sel(p0, kc);
        const int chb = kb == 0 ? chx : (kb == 1 ? chy : chz);
        const int chc = kc == 0 ? chx : (kc == 1 ? chy : chz);
        const bool ok = nn == 0 || ((sa > 0.f) == pos && sa != 0.f && fabsf(sb) <= fabsf(sa) && fabsf(sc) <= fabsf(sa));
        const bool dominant = __all_sync(FULL, ok);  // multi-slab jumps need |st_b|, |st_c| <= |st_a| on all rays
#endif
        const float isa = sa != 0.f ? 1.f / sa : 0.f;
#if DPRT_BEAM_PROBE
        float ist[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) ist[i] = st[i] != 0.f ? 1.f / st[i] : 0.f;
        // this ray's skip distances: the one-sided grid of its direction octant (a zero component may take
        // either side: the ray stays in its layer, which both boxes contain)
        const uint8_t* __restrict__ skipl =
            DPRT_SKIP_OCTANT ? skipd + (1 + (st[0] > 0.f ? 1 : 0) + (st[1] > 0.f ? 2 : 0) + (st[2] > 0.f ? 4 : 0)) * a.skip_n
                             : skipd;
#endif
        int j = 0;
        float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
        if (a.accum && nn > 0) {
            // ray cycling: continue this ray's front-to-back state from the bricks it has crossed
            const float4 s0 = a.out[pix - a.pix0];
            C0 = s0.x;
            C1 = s0.y;
            C2 = s0.z;
            A = s0.w;
            if (A >= ert) nn = 0;  // terminated in front of this brick: nothing to add, nothing to write
        }
        bool live = nn > 0;
#if DPRT_PROBE_PREFETCH
        int pf = -1;  // skip distance at sample j loaded ahead of the probe (-1: none)
#endif
        while (true) {
            const unsigned livem = __ballot_sync(FULL, live);
            if (!livem) break;
#if DPRT_COUNTERS == 2
            if (lane == 0) ++c_shade;  // [0]: warp slab iterations (probe + slab step)
#endif
#if DPRT_BEAM_PROBE
            // per-lane probe: a lane whose next sample sits in an empty macrocell jumps on its own to the exit
            // of the empty box its octant's skip distance guarantees ahead of it (exact: the skipped samples
            // add zeros); only lanes in non-empty macrocells go on to the slab step, which then needs no
            // beam-wide emptiness test
            bool samp = live;
#if DPRT_PROBE_LOOP
            // ... and keeps jumping until its next sample sits in a non-empty macrocell (then it shades in
            // this same iteration) or its ray is done: a jump costs the probe alone, not a whole warp
            // iteration (ballot, slab selection) per empty cube
            while (live && a.skip) {
#else
            if (live && a.skip) {
#endif
                const float fj = (float)j;
                const int cx = fl2cell(fmaf(fj, st[0], p0[0]), chx);
                const int cy = fl2cell(fmaf(fj, st[1], p0[1]), chy);
                const int cz = fl2cell(fmaf(fj, st[2], p0[2]), chz);
                const int mx = cx >> ms, my = cy >> ms, mz = cz >> ms;
                const int mci = (mz * mcd1 + my) * mcd0 + mx;
#if DPRT_PROBE_PREFETCH
                // the first probe of an iteration may have been loaded during the previous slab step
#if DPRT_SUBBLOCK == 2
                const unsigned smask = __ldg(a.subm + mci);  // issued with (not after) the distance load
#endif
                skip_bounds_check(a, mci);
                const int dist = pf >= 0 ? pf : (int)__ldg(skipl + mci);
                pf = -1;
#else
                const int dist = (int)__ldg(skipl + mci);
#endif
#if DPRT_PROBE_LOOP && DPRT_SUBBLOCK
                if (dist == 0) {
                    // a non-empty macrocell: is this sample's 4^3 sub-block empty too?  Then jump to its exit
                    // (the sub-block is the empty box; exact like the macrocell jump)
                    const int sbit = ((cx >> (ms - 1)) & 1) | (((cy >> (ms - 1)) & 1) << 1) |
                                     (((cz >> (ms - 1)) & 1) << 2);
#if DPRT_SUBBLOCK == 2
                    if ((smask >> sbit) & 1) break;
#else
                    if ((__ldg(a.subm + mci) >> sbit) & 1) break;
#endif
                    const int kSub = ms - 1;
                    const float sx = ((float)(((cx >> kSub) + (st[0] > 0.f ? 1 : 0)) << kSub) - p0[0]) * ist[0];
                    const float sy = ((float)(((cy >> kSub) + (st[1] > 0.f ? 1 : 0)) << kSub) - p0[1]) * ist[1];
                    const float sz = ((float)(((cz >> kSub) + (st[2] > 0.f ? 1 : 0)) << kSub) - p0[2]) * ist[2];
                    const float se = fminf(fminf(sx, sy), sz);
                    j = se < (float)nn ? max((int)ceilf(se), j + 1) : nn;
                    if (j >= nn) live = false;
                    samp = live;
                    continue;
                }
                {
#elif DPRT_PROBE_LOOP
                if (dist == 0) break;
                {
#else
                if (dist > 0) {
#endif
#if DPRT_JUMP_BRANCHFREE
                    // exit of the empty box along each axis, branch-free: an axis the ray does not move along
                    // has ist = 0 and so gives je = 0, which only shortens the jump to one sample (still exact;
                    // rays with an exactly zero direction component are rare)
                    const float jx = ((float)((st[0] > 0.f ? mx + dist : mx - dist + 1) << ms) - p0[0]) * ist[0];
                    const float jy = ((float)((st[1] > 0.f ? my + dist : my - dist + 1) << ms) - p0[1]) * ist[1];
                    const float jz = ((float)((st[2] > 0.f ? mz + dist : mz - dist + 1) << ms) - p0[2]) * ist[2];
                    const float je = fminf(fminf(jx, jy), jz);
#else
                    float je = 3.0e38f;
                    if (st[0] != 0.f)
                        je = fminf(je, ((float)((st[0] > 0.f ? mx + dist : mx - dist + 1) << ms) - p0[0]) * ist[0]);
                    if (st[1] != 0.f)
                        je = fminf(je, ((float)((st[1] > 0.f ? my + dist : my - dist + 1) << ms) - p0[1]) * ist[1]);
                    if (st[2] != 0.f)
                        je = fminf(je, ((float)((st[2] > 0.f ? mz + dist : mz - dist + 1) << ms) - p0[2]) * ist[2]);
#endif
                    j = je < (float)nn ? max((int)ceilf(je), j + 1) : nn;
                    if (j >= nn) live = false;
#if DPRT_PROBE_LOOP
                    samp = live;
#else
                    samp = false;
#endif
#if DPRT_COUNTERS == 1
                    ++c_skip;
#endif
                }
            }
            if (!__any_sync(FULL, samp)) continue;
#if DPRT_COUNTERS == 2
            if (lane == 0) ++c_contrib;  // [1]: warp iterations that shade
#endif
#else
            const bool samp = live;
#endif
            // current slab: the nearest (in the march direction) slab holding a sampling lane's next sample
            int ksl = 0;
            if (samp) ksl = fl2cell(fmaf((float)j, sa, pa), cha) >> kSS;
            const int key = samp ? (pos ? ksl : -ksl) : 0x7fffffff;
            const int kmin = __reduce_min_sync(FULL, key);
            const int K = pos ? kmin : -kmin;
            // this lane's samples in slab K: j .. jend-1 (first sample past the slab's far face)
            int jend = j;
            if (samp) {
                const float face = (float)((pos ? K + 1 : K) << kSS);
                const float je = (face - pa) * isa;
                jend = je < (float)nn ? max((int)ceilf(je), j + 1) : nn;  // >= 1 sample: progress
                if (ksl != K) jend = j;  // this ray is not in slab K yet
#if DPRT_PROBE_PREFETCH
                // next iteration's first probe: a lane waiting for its slab probes the same (non-empty)
                // macrocell again; a lane shading slab K probes sample jend -- load that skip distance now,
                // so its latency hides behind the batches
                if (ksl != K) {
                    pf = 0;
                } else if (a.skip && jend < nn) {
                    const float fe = (float)jend;
                    const int ex = fl2cell(fmaf(fe, st[0], p0[0]), chx) >> ms;
                    const int ey = fl2cell(fmaf(fe, st[1], p0[1]), chy) >> ms;
                    const int ez = fl2cell(fmaf(fe, st[2], p0[2]), chz) >> ms;
                    skip_bounds_check(a, (ez * mcd1 + ey) * mcd0 + ex);
                    pf = (int)__ldg(skipl + (ez * mcd1 + ey) * mcd0 + ex);
                }
#endif
            }
#if !DPRT_BEAM_PROBE
            // bound the beam's cells on the other two axes over all samples in the slab
            int b0 = 0x7fffffff, b1 = -1, c0 = 0x7fffffff, c1 = -1;
            if (jend > j) {
                const float f0 = (float)j, f1 = (float)(jend - 1);
                const int ub0 = fl2cell(fmaf(f0, sb, pb), chb), ub1 = fl2cell(fmaf(f1, sb, pb), chb);
                const int uc0 = fl2cell(fmaf(f0, sc, pc), chc), uc1 = fl2cell(fmaf(f1, sc, pc), chc);
                b0 = min(ub0, ub1) >> ms;
                b1 = max(ub0, ub1) >> ms;
                c0 = min(uc0, uc1) >> ms;
                c1 = max(uc0, uc1) >> ms;
            }
            const int B0 = __reduce_min_sync(FULL, b0), B1 = __reduce_max_sync(FULL, b1);
            const int Cc0 = __reduce_min_sync(FULL, c0), Cc1 = __reduce_max_sync(FULL, c1);
            int dmin = 0;
            if (a.skip && B1 >= B0) {
                const int nb = B1 - B0 + 1, nc = Cc1 - Cc0 + 1;
                // lanes enumerate the nb x nc macrocells on a power-of-two row pitch (no integer division)
                const int lg = nb > 1 ? 32 - __clz(nb - 1) : 0;
                if ((nc << lg) <= 32) {
                    int dl = 255;
                    if ((lane & ((1 << lg) - 1)) < nb && (lane >> lg) < nc) {
                        const int mb = B0 + (lane & ((1 << lg) - 1)), mc = Cc0 + (lane >> lg);
                        const int mx = ka == 0 ? K : (kb == 0 ? mb : mc);
                        const int my = ka == 1 ? K : (kb == 1 ? mb : mc);
                        const int mz = ka == 2 ? K : (kb == 2 ? mb : mc);
                        dl = (int)__ldg(skipd + (mz * mcd1 + my) * mcd0 + mx);
                    }
                    dmin = __reduce_min_sync(FULL, dl);
                }
            }
            if (dmin > 0) {
                // every macrocell the beam touches in slab K is empty; with all rays dominated by axis a
                // the next dmin - 1 slabs are inside their empty Chebyshev cubes too
                const int jump = dominant ? dmin : 1;
#if DPRT_COUNTERS
                c_skip += live;
#endif
                if (live && ksl == K) {
                    const float face = (float)((pos ? K + jump : K - jump + 1) << ms);
                    const float je = (face - pa) * isa;
                    j = je < (float)nn ? max((int)ceilf(je), j + 1) : nn;
                    if (j >= nn) live = false;
                }
                continue;
            }
#endif
            // Shade this lane's samples in the slab, kUnroll at a time: all their corner loads are
            // issued before the first is shaded, so each lane keeps several loads in flight.
            // branch-free batches: slots past the lane's last sample in the slab re-load that sample (same
            // address, an L1 hit) and contribute w = 0; ERT masks the rest of the batch the same way
            const float fend = (float)(jend - 1);
            while (j < jend) {
#if DPRT_COUNTERS == 2
                if (lane == __ffs(__activemask()) - 1) ++c_skip;  // [2]: warp batches
                ++c_rays;                                         // [3]: lane batches
#endif
                float4 qa[kUnroll], qb[kUnroll];
                float wx[kUnroll], wy[kUnroll], wz[kUnroll];
                const float fj = (float)j;  // exact: j < 2^24
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const float fs = fminf(fj + (float)u, fend);
                    const float ux = fmaf(fs, st[0], p0[0]);
                    const float uy = fmaf(fs, st[1], p0[1]);
                    const float uz = fmaf(fs, st[2], p0[2]);
                    const int ix = __float2int_rd(ux), iy = __float2int_rd(uy), iz = __float2int_rd(uz);
                    if constexpr (kWide) {
                        // >= 2^31 quads: offset from the apron grid's first quad as unsigned 32-bit (exact
                        // below 2^32 quads -- modular arithmetic, the true offset is non-negative); one IADD
                        // more than the signed form, no 64-bit registers
                        const unsigned qu = quad_offset((unsigned)ix, (unsigned)iy, (unsigned)iz, (unsigned)qsx, (unsigned)qsy, (unsigned)qsz) + qk;
                        quad_bounds_check(a, (long long)qu - qk);
                        if constexpr (kHalf) {
                            load_half_quads(reinterpret_cast<const uint2*>(qbase) + qu, qsz, qa[u], qb[u]);
                        } else {
#if DPRT_QUAD_OCTET
                            load_octet(qbase + 2 * (unsigned long long)qu, qa[u], qb[u]);
#else
                            qa[u] = __ldg(qbase + qu);
                            qb[u] = __ldg(qbase1 + qu);
#endif
                        }
                    } else {
                        const int qi = quad_offset(ix, iy, iz, qsx, qsy, qsz);
                        quad_bounds_check(a, qi);
                        if constexpr (kHalf) {
                            load_half_quads(hq_org + qi, qsz, qa[u], qb[u]);
                        } else {
#if DPRT_QUAD_OCTET
                            load_octet(qorg + 2 * (long long)qi, qa[u], qb[u]);
#elif DPRT_TIMING_PAIR == 1
                            // timing only (wrong image): the far face read from the adjacent slot
                            qa[u] = __ldg(qorg + qi);
                            qb[u] = __ldg(qorg + qi + 1);
#elif DPRT_TIMING_PAIR == 2
                            // timing only (wrong image): both faces from one aligned 32-byte slot
                            load_octet(qbase + ((qk + (unsigned)qi) & ~1u), qa[u], qb[u]);
#else
                            qa[u] = __ldg(qorg + qi);
                            qb[u] = __ldg(qorg1 + qi);
#endif
                        }
                    }
                    wx[u] = __saturatef(ux - (float)ix);
                    wy[u] = __saturatef(uy - (float)iy);
                    wz[u] = __saturatef(uz - (float)iz);
                }
                const int cnt = min(kUnroll, jend - j);
#if DPRT_BLEND_PREFIX
                // transmittance form with the per-slot dependency cut to one FMUL: w_u = T_u a_u and
                // T_{u+1} = T_u (1 - a_u); a slot contributes while the ray is live before it, (1 - T_u) < ert
                // (the same early-termination rule as A >= ert); A = 1 - T after the last live slot
                float T = 1.f - A, Tend = T;
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const float v = trilerp(qa[u], qb[u], wx[u], wy[u], wx[u] * wy[u], wz[u]);
                    const float x = __saturatef(fmaf(v, tns, tno)) * top;
                    const int ti = (int)x;
                    const float tfr = x - (float)ti;
                    const float4 e0 = s_tf[ti], de = s_dtf[ti];
                    const float al = u < cnt ? fmaf(tfr, de.w, e0.w) : 0.f;
                    const bool lv = (1.f - T) < ert;
                    const float w = lv ? T * al : 0.f;
                    C0 = fmaf(w, fmaf(tfr, de.x, e0.x), C0);
                    C1 = fmaf(w, fmaf(tfr, de.y, e0.y), C1);
                    C2 = fmaf(w, fmaf(tfr, de.z, e0.z), C2);
                    const float m = (lv && u < cnt) ? 1.f : 0.f;
#if DPRT_COUNTERS == 1
                    c_shade += m != 0.f;
                    c_contrib += w > 0.f;
#elif DPRT_COUNTERS == 3
                    // shaded samples by their macrocell: [0] all, [1] in an empty macrocell, [2] contributing,
                    // [3] non-contributing in a non-empty macrocell
                    if (m != 0.f) {
                        const float fs = fj + (float)u;
                        const int mx = fl2cell(fmaf(fs, st[0], p0[0]), chx) >> ms;
                        const int my = fl2cell(fmaf(fs, st[1], p0[1]), chy) >> ms;
                        const int mz = fl2cell(fmaf(fs, st[2], p0[2]), chz) >> ms;
                        const bool empty = __ldg(skipd + (mz * mcd1 + my) * mcd0 + mx) > 0;
                        ++c_shade;
                        c_contrib += empty;
                        c_skip += w > 0.f;
                        c_rays += !empty && !(w > 0.f);
                    }
#endif
                    if constexpr (kMark) {
                        if (m != 0.f) {
                            const float fs = fj + (float)u;
                            const int mx = fl2cell(fmaf(fs, st[0], p0[0]), chx) >> ms;
                            const int my = fl2cell(fmaf(fs, st[1], p0[1]), chy) >> ms;
                            const int mz = fl2cell(fmaf(fs, st[2], p0[2]), chz) >> ms;
                            a.mark[((long long)mz * mcd1 + my) * mcd0 + mx] = 1;
                            ++m_shade;
                            m_contrib += w > 0.f;
                        }
                    }
                    T *= 1.f - al;
                    Tend = lv ? T : Tend;
                }
                A = 1.f - Tend;
#else
                float m = 1.f;  // 1 while the slot is a real sample of a live ray, then 0
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    if (u >= cnt) m = 0.f;
                    const float v = trilerp(qa[u], qb[u], wx[u], wy[u], wx[u] * wy[u], wz[u]);
                    const float x = __saturatef(fmaf(v, tns, tno)) * top;
                    const int ti = (int)x;
                    const float tfr = x - (float)ti;
                    const float4 e0 = s_tf[ti], de = s_dtf[ti];
                    const float w = m * ((1.f - A) * fmaf(tfr, de.w, e0.w));
                    A += w;
                    C0 = fmaf(w, fmaf(tfr, de.x, e0.x), C0);
                    C1 = fmaf(w, fmaf(tfr, de.y, e0.y), C1);
                    C2 = fmaf(w, fmaf(tfr, de.z, e0.z), C2);
#if DPRT_COUNTERS == 1
                    c_shade += m != 0.f;
                    c_contrib += w > 0.f;
#elif DPRT_COUNTERS == 3
                    // shaded samples by their macrocell: [0] all, [1] in an empty macrocell, [2] contributing,
                    // [3] non-contributing in a non-empty macrocell
                    if (m != 0.f) {
                        const float fs = fj + (float)u;
                        const int mx = fl2cell(fmaf(fs, st[0], p0[0]), chx) >> ms;
                        const int my = fl2cell(fmaf(fs, st[1], p0[1]), chy) >> ms;
                        const int mz = fl2cell(fmaf(fs, st[2], p0[2]), chz) >> ms;
                        const bool empty = __ldg(skipd + (mz * mcd1 + my) * mcd0 + mx) > 0;
                        ++c_shade;
                        c_contrib += empty;
                        c_skip += w > 0.f;
                        c_rays += !empty && !(w > 0.f);
                    }
#endif
                    if constexpr (kMark) {
                        if (m != 0.f) {
                            const float fs = fj + (float)u;
                            const int mx = fl2cell(fmaf(fs, st[0], p0[0]), chx) >> ms;
                            const int my = fl2cell(fmaf(fs, st[1], p0[1]), chy) >> ms;
                            const int mz = fl2cell(fmaf(fs, st[2], p0[2]), chz) >> ms;
                            a.mark[((long long)mz * mcd1 + my) * mcd0 + mx] = 1;
                            ++m_shade;
                            m_contrib += w > 0.f;
                        }
                    }
                    if (A >= ert) m = 0.f;  // early ray termination: the rest of the batch adds nothing
                }
#endif
                j += cnt;
                if (A >= ert) {
                    live = false;
                    break;
                }
            }
            if (j >= nn) live = false;
        }
        if (!kMark && inside && (nn > 0 || !a.accum)) {  // accumulated state of a skipped ray stays as it was
            if (a.rgb8) {
                // single-rank frame: the over-background + tone map of the compositor, fused
                // (engine.py:500-502); a miss inside the footprint is the background itself
                const float one = 1.f - A;
                pix_bounds_check(a, pix);
                uint8_t* dst = a.rgb8 + 3 * (size_t)pix;
                dst[0] = (uint8_t)floorf(fminf(fmaxf(fmaf(one, a.bg[0], C0), 0.f), 1.f) * 255.f + 0.5f);
                dst[1] = (uint8_t)floorf(fminf(fmaxf(fmaf(one, a.bg[1], C1), 0.f), 1.f) * 255.f + 0.5f);
                dst[2] = (uint8_t)floorf(fminf(fmaxf(fmaf(one, a.bg[2], C2), 0.f), 1.f) * 255.f + 0.5f);
            } else {
                store_partial<kPush>(a, s_blk, pix, py, C0, C1, C2, A);
            }
        }
    }
    if constexpr (kMark) {
        atomicAdd(a.stats, m_shade);
        atomicAdd(a.stats + 1, m_contrib);
        return;
    }
    if (!a.accum) {
        // fused clear / background of the pixels no beam covers (no memset pass), done by each warp once
        // the tile queue is empty, so it overlaps the slowest beams instead of delaying the first ones
        const int y0 = a.band_clear ? a.rect[1] : (int)(a.pix0 / a.W);
        const int y1 = a.band_clear ? a.rect[3] : (int)((a.pix0 + a.npix_buf) / a.W);
        const int wpb = blockDim.x >> 5;
        fill_outside_rect<kPush>(a, s_blk, y0, y1, (int)blockIdx.x * wpb + (tid >> 5), (int)gridDim.x * wpb, lane, 32);
    }
    if constexpr (kPush) grid_signal(a.push_ctr, a.push_flag, a.push_P, a.push_epoch);  // fragments landed at owners
#if DPRT_COUNTERS
    DPRT_COUNT(0, c_shade);
    DPRT_COUNT(1, c_contrib);
    DPRT_COUNT(2, c_skip);
    DPRT_COUNT(3, c_rays);
#endif
}

// Skip distances.  classify: 0 for a macrocell whose dilated value range [min, max]
// can map to a non-zero alpha under the TF (conservatively one extra entry on each side), kSkipCap
// otherwise.  Then three separable passes turn it into the Chebyshev distance (in macrocells, capped)
// to the nearest non-empty macrocell: D(m) = min_c max(|m - c|_inf, E(c)).
__global__ void skip_classify_kernel(const float2* __restrict__ macro, long long nmc, const float4* __restrict__ tf,
                                     int n_tf, float vmin, float tf_scale, uint8_t* __restrict__ out) {
    __shared__ int s_next_nz[kMaxTf];
    const int tid = threadIdx.x;
    if (tid < 32) {
        int carry = n_tf;
        for (int base = ((n_tf - 1) / 32) * 32; base >= 0; base -= 32) {
            const int i = base + tid;
            const bool nz = i < n_tf && tf[i].w > 0.0f;
            const unsigned m = __ballot_sync(0xffffffffu, nz);
            const unsigned here = m & (0xffffffffu << tid);
            if (i < n_tf) s_next_nz[i] = here ? base + __ffs(here) - 1 : carry;
            const int lowest = m ? base + __ffs(m) - 1 : carry;
            carry = __shfl_sync(0xffffffffu, lowest, 0);
        }
    }
    __syncthreads();
    const float top = (float)(n_tf - 1);
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < nmc; i += (long long)gridDim.x * blockDim.x) {
        const float2 mm = macro[i];
        const float xl = fminf(fmaxf((mm.x - vmin) * tf_scale, 0.f), top);
        const float xh = fminf(fmaxf((mm.y - vmin) * tf_scale, 0.f), top);
        const int il = max((int)xl - 1, 0);
        const int ih = min((int)xh + 2, n_tf - 1);
        out[i] = s_next_nz[il] > ih ? (uint8_t)kSkipCap : (uint8_t)0;
    }
}

// Sub-block masks (DPRT_SUBBLOCK): bit b of a macrocell's byte = its 4^3 sub-block b may map to alpha > 0
// (the same conservative test as skip_classify_kernel, on the sub-block's dilated range).
__global__ void sub_classify_kernel(const float2* __restrict__ sub, long long nmc, const float4* __restrict__ tf,
                                    int n_tf, float vmin, float tf_scale, uint8_t* __restrict__ out) {
    __shared__ int s_next_nz[kMaxTf];
    const int tid = threadIdx.x;
    if (tid < 32) {
        int carry = n_tf;
        for (int base = ((n_tf - 1) / 32) * 32; base >= 0; base -= 32) {
            const int i = base + tid;
            const bool nz = i < n_tf && tf[i].w > 0.0f;
            const unsigned m = __ballot_sync(0xffffffffu, nz);
            const unsigned here = m & (0xffffffffu << tid);
            if (i < n_tf) s_next_nz[i] = here ? base + __ffs(here) - 1 : carry;
            const int lowest = m ? base + __ffs(m) - 1 : carry;
            carry = __shfl_sync(0xffffffffu, lowest, 0);
        }
    }
    __syncthreads();
    const float top = (float)(n_tf - 1);
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < nmc; i += (long long)gridDim.x * blockDim.x) {
        unsigned mask = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const float2 mm = sub[i * 8 + b];
            const float xl = fminf(fmaxf((mm.x - vmin) * tf_scale, 0.f), top);
            const float xh = fminf(fmaxf((mm.y - vmin) * tf_scale, 0.f), top);
            const int il = max((int)xl - 1, 0);
            const int ih = min((int)xh + 2, n_tf - 1);
            if (!(s_next_nz[il] > ih) && mm.x <= mm.y) mask |= 1u << b;
        }
        out[i] = (uint8_t)mask;
    }
}

// One separable pass of the distance transform for grid g = blockIdx.y: out = min over t of max(t, in) along
// `axis`, t steps towards both sides for the symmetric grid (g = 0) and only towards the octant's side for
// g = 1 + o (bit `axis` of o set: +).  The octant distance D(m) = min over non-empty c in the forward octant
// of max_i |c_i - m_i|: the box from m spanning D macrocells forward on every axis is empty, so a ray
// moving into that octant may jump to the box's exit (exact; the probe uses the same exit formula).
__global__ void skip_pass_kernel(const uint8_t* __restrict__ in, long long in_grid_stride, uint8_t* __restrict__ out,
                                 long long out_grid_stride, int n0, int n1, int n2, int axis) {
    const long long total = (long long)n0 * n1 * n2;
    const int g = blockIdx.y;
    const uint8_t* gin = in + g * in_grid_stride;
    uint8_t* gout = out + g * out_grid_stride;
    const bool both = g == 0;
    const int sgn = ((g - 1) >> axis) & 1 ? 1 : -1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % n0);
        const int y = (int)((i / n0) % n1);
        const int z = (int)(i / ((long long)n0 * n1));
        const int c = axis == 0 ? x : (axis == 1 ? y : z);
        const int n = axis == 0 ? n0 : (axis == 1 ? n1 : n2);
        const long long stride = axis == 0 ? 1 : (axis == 1 ? n0 : (long long)n0 * n1);
        int best = gin[i];
        for (int k = 1; k < best && k < kSkipCap; ++k) {
            if (both) {
                if (c - k >= 0) best = min(best, max(k, (int)gin[i - k * stride]));
                if (c + k < n) best = min(best, max(k, (int)gin[i + k * stride]));
            } else if (c + sgn * k >= 0 && c + sgn * k < n) {
                best = min(best, max(k, (int)gin[i + sgn * k * stride]));
            }
        }
        gout[i] = (uint8_t)best;
    }
}

cudaError_t launch_skip_build(const DeviceBrick& b, const MarchArgs& a, uint8_t* tmp, cudaStream_t stream) {
    const long long nmc = (long long)b.mcd[0] * b.mcd[1] * b.mcd[2];
    const int block = 256;
    const long long want = (nmc + block - 1) / block;
    const int grid = (int)(want < 148LL * 16 ? (want > 0 ? want : 1) : 148LL * 16);
    const int ng = DPRT_SKIP_OCTANT ? kSkipGrids : 1;
    uint8_t* t1 = tmp;
    uint8_t* t2 = tmp + nmc * kSkipGrids;
    const int m0 = (int)b.mcd[0], m1 = (int)b.mcd[1], m2 = (int)b.mcd[2];
    // emptiness (0 or the cap) into grid 0, then z, y, x passes for every grid at once; the z pass reads the
    // same emptiness for all grids (input grid stride 0) and the x pass writes the final grids
    skip_classify_kernel<<<grid, block, 0, stream>>>(b.macro, nmc, a.tf, a.n_tf, a.vmin, a.tf_scale, b.skipd);
    skip_pass_kernel<<<dim3(grid, ng), block, 0, stream>>>(b.skipd, 0, t1, nmc, m0, m1, m2, 2);
    skip_pass_kernel<<<dim3(grid, ng), block, 0, stream>>>(t1, nmc, t2, nmc, m0, m1, m2, 1);
    skip_pass_kernel<<<dim3(grid, ng), block, 0, stream>>>(t2, nmc, b.skipd, nmc, m0, m1, m2, 0);
    if (DPRT_SUBBLOCK) sub_classify_kernel<<<grid, block, 0, stream>>>(b.sub, nmc, a.tf, a.n_tf, a.vmin, a.tf_scale, b.subm);
    return cudaGetLastError();
}

cudaError_t read_counters(unsigned long long out[4], int reset) {
#if DPRT_COUNTERS
    cudaError_t e = cudaMemcpyFromSymbol(out, g_counters, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess && reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        e = cudaMemcpyToSymbol(g_counters, z, sizeof(z));
    }
    return e;
#else
    for (int i = 0; i < 4; ++i) out[i] = 0;
    (void)reset;
    return cudaSuccess;
#endif
}

// Host launchers (called from abi.cu).
//
// Per-launch host work is a cache lookup: the SM count per device and the occupancy per (kernel, shared
// memory, device) are queried once, not on every frame (a frame is ~0.2 ms of device time).
namespace {
struct OccKey {
    const void* kern;
    size_t smem;
    int dev;
    int per_sm;
};
std::mutex g_occ_mu;
OccKey g_occ[64];
int g_occ_n = 0;
int g_sms[64];

int grid_for(const void* kern, int block, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> lk(g_occ_mu);
    if (g_sms[dev] == 0) cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    for (int i = 0; i < g_occ_n; ++i)
        if (g_occ[i].kern == kern && g_occ[i].smem == smem && g_occ[i].dev == dev) return g_sms[dev] * g_occ[i].per_sm;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (per_sm < 1) per_sm = 1;
    if (g_occ_n < 64) g_occ[g_occ_n++] = OccKey{kern, smem, dev, per_sm};
    return g_sms[dev] * per_sm;
}
}  // namespace

cudaError_t launch_march(const MarchArgs& a, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(a.counters, 0, 2 * sizeof(int), stream);
    if (e != cudaSuccess) return e;
    dim3 block(kTileX * kTileY);
    dim3 grid((a.W + kTileX - 1) / kTileX, (a.H + kTileY - 1) / kTileY);
    if (!a.beam) {
        ray_setup_kernel<<<grid, block, 0, stream>>>(a);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const size_t smem = 2 * a.n_tf * sizeof(float4);
    if (a.beam) {
        // no clear pass: the beam kernel itself writes every pixel it is responsible for -- zero (RGBA
        // partial) or the tone-mapped background (RGB8 frame) outside the footprint and for misses
        // (fill_outside_rect, write_clear); accumulation leaves the rays' state alone
        if (a.samples) e = cudaMemsetAsync(a.samples, 0, (size_t)a.npix_buf * sizeof(uint32_t), stream);
        if (e != cudaSuccess) return e;
        using K = void (*)(const MarchArgs);
        constexpr int kSmallMS = DPRT_BEAM_PROBE ? DPRT_MACRO_SHIFT_SMALL : kMacroShift;
        // [push][natural macro shift][half][deep][wide]
#define DPRT_BEAM_K(H, D, W, P, N)                                                                           \
    march_beam_kernel<W, (D) ? kDeepUnroll : kBeamUnroll, (D) ? kDeepBlocks : DPRT_BEAM_MINBLOCKS, H, false, P, \
                      (N) ? ((D) ? kMacroShift : kSmallMS) : 0>
#define DPRT_BEAM_K4(H, P, N) {{DPRT_BEAM_K(H, 0, false, P, N), DPRT_BEAM_K(H, 0, true, P, N)}, \
                               {DPRT_BEAM_K(H, 1, false, P, N), DPRT_BEAM_K(H, 1, true, P, N)}}
        static const K kerns[2][2][2][2][2] = {
            {{DPRT_BEAM_K4(false, false, false), DPRT_BEAM_K4(true, false, false)},
             {DPRT_BEAM_K4(false, false, true), DPRT_BEAM_K4(true, false, true)}},
            {{DPRT_BEAM_K4(false, true, false), DPRT_BEAM_K4(true, true, false)},
             {DPRT_BEAM_K4(false, true, true), DPRT_BEAM_K4(true, true, true)}}};
#undef DPRT_BEAM_K4
#undef DPRT_BEAM_K
        const int hq = a.half_quads ? 1 : 0, dp = a.deep ? 1 : 0, wd = a.wide ? 1 : 0;
        const int natural = a.mshift == (a.deep ? kMacroShift : kSmallMS) ? 1 : 0;
        const K kern = kerns[a.push_P ? 1 : 0][natural][hq][dp][wd];
        const size_t sm = a.push_P ? smem + (size_t)((a.H + 15) & ~15) : smem;  // + the row -> block table
        kern<<<grid_for((const void*)kern, kBeamBlock, sm), kBeamBlock, sm, stream>>>(a);
        return cudaGetLastError();
    }
    march_kernel<<<grid_for((const void*)march_kernel, kTileX * kTileY, smem), block, smem, stream>>>(a);
    return cudaGetLastError();
}

// dprt_march_stats: the instrumented beam march (the production kernel's ray setup, skipping and batching
// decisions, no image output) marking the macrocells it shades samples in.
cudaError_t launch_march_mark(const MarchArgs& a, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(a.counters, 0, 2 * sizeof(int), stream);
    if (e != cudaSuccess) return e;
    const size_t smem = 2 * a.n_tf * sizeof(float4);
    using K = void (*)(const MarchArgs);
    const K kerns[2][2] = {{march_beam_kernel<false, kBeamUnroll, DPRT_BEAM_MINBLOCKS, false, true>,
                            march_beam_kernel<true, kBeamUnroll, DPRT_BEAM_MINBLOCKS, false, true>},
                           {march_beam_kernel<false, kBeamUnroll, DPRT_BEAM_MINBLOCKS, true, true>,
                            march_beam_kernel<true, kBeamUnroll, DPRT_BEAM_MINBLOCKS, true, true>}};
    const K kern = kerns[a.half_quads ? 1 : 0][a.wide ? 1 : 0];
    kern<<<grid_for((const void*)kern, kBeamBlock, smem), kBeamBlock, smem, stream>>>(a);
    return cudaGetLastError();
}

// Sum over the marked macrocells of their cell counts (the f32 voxels a perfect marcher reads once) and the
// number of marked macrocells.
__global__ void mark_reduce_kernel(const uint8_t* __restrict__ mark, int m0, int m1, int m2, int c0, int c1, int c2,
                                   int mshift, unsigned long long* __restrict__ out) {
    const long long kMacro = 1LL << mshift;
    unsigned long long cells = 0, n = 0;
    const long long total = (long long)m0 * m1 * m2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        if (!mark[i]) continue;
        const int x = (int)(i % m0), y = (int)((i / m0) % m1), z = (int)(i / ((long long)m0 * m1));
        const long long ex = min(kMacro, c0 - x * kMacro), ey = min(kMacro, c1 - y * kMacro),
                        ez = min(kMacro, c2 - z * kMacro);
        cells += (unsigned long long)(ex * ey * ez);
        ++n;
    }
    for (int o = 16; o > 0; o >>= 1) {
        cells += __shfl_down_sync(0xffffffffu, cells, o);
        n += __shfl_down_sync(0xffffffffu, n, o);
    }
    if ((threadIdx.x & 31) == 0 && n) {
        atomicAdd(out, cells);
        atomicAdd(out + 1, n);
    }
}

cudaError_t launch_mark_reduce(const uint8_t* mark, const int mcd[3], const int cells[3], int mshift,
                               unsigned long long* out, cudaStream_t stream) {
    mark_reduce_kernel<<<148 * 4, 256, 0, stream>>>(mark, mcd[0], mcd[1], mcd[2], cells[0], cells[1], cells[2], mshift,
                                                    out);
    return cudaGetLastError();
}

}  // namespace dprt

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

#include "common.cuh"

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

// geom.py:171-200 + clip to [0, inf) (geom.py:203-209) + lattice range.
__device__ __forceinline__ int64_t lattice_range(const MarchArgs& a, const double d[3], int64_t* k0) {
    double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double di = d[i], oi = a.o[i];
        if (di == 0.0) {
            if (oi < a.blo[i] || oi > a.bhi[i]) return 0;
            continue;
        }
        double inv = __ddiv_rn(1.0, di);
        double ta = __dmul_rn(__dsub_rn(a.blo[i], oi), inv);
        double tb = __dmul_rn(__dsub_rn(a.bhi[i], oi), inv);
        if (ta > tb) {
            double s = ta;
            ta = tb;
            tb = s;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t1 < t0) return 0;
    }
    if (t0 < 0.0) t0 = 0.0;
    if (t1 < t0) return 0;
    int64_t ka = (int64_t)ceil(__ddiv_rn(t0, a.dt));
    int64_t kb = (int64_t)ceil(__ddiv_rn(t1, a.dt));
    *k0 = ka;
    return kb > ka ? kb - ka : 0;
}

#ifndef DPRT_FAKE_MEM
#define DPRT_FAKE_MEM 0
#endif
#ifndef DPRT_CHUNKED
#define DPRT_CHUNKED 0
#endif
#ifndef DPRT_CHUNK
#define DPRT_CHUNK 32
#endif
constexpr int kChunk = DPRT_CHUNK;
#ifndef DPRT_REFILL_BELOW
#define DPRT_REFILL_BELOW 8
#endif
#ifndef DPRT_STEPS_PER_CHECK
#define DPRT_STEPS_PER_CHECK 16
#endif
constexpr int kRefillBelow = DPRT_REFILL_BELOW;  // refill a warp's idle lanes once fewer than this many march
constexpr int kStepsPerCheck = DPRT_STEPS_PER_CHECK;  // march steps between refill checks
#ifndef DPRT_ASYNC_DEPTH
#define DPRT_ASYNC_DEPTH 4
#endif
constexpr int kDepth = DPRT_ASYNC_DEPTH;  // cp.async samples in flight per lane (DPRT_ASYNC)
constexpr int kThreads = kTileX * kTileY;

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
        const double p = (a.o[i] + t0 * d[i] - a.origin[i]) / a.spacing[i];
        p0[i] = (float)(p - a.stored_lo_d[i]);
        st[i] = (float)(a.dt * d[i]) * a.inv_spacing[i];
    }
    a.rays[2 * slot] = make_float4(p0[0], p0[1], p0[2], __int_as_float((int)pix));
    a.rays[2 * slot + 1] = make_float4(st[0], st[1], st[2], __int_as_float((int)n));
}

// Pass 2: persistent warps march the queued rays.
#ifndef DPRT_MARCH_MINBLOCKS
#define DPRT_MARCH_MINBLOCKS 4
#endif
__global__ void __launch_bounds__(kTileX * kTileY, DPRT_MARCH_MINBLOCKS) march_kernel(const MarchArgs a) {
    // TF as (entry, next - entry) pairs: the lerp e0 + (e1 - e0) * f becomes one FMA per channel with the
    // identical rounding (the difference is formed once here instead of per sample).
    extern __shared__ float4 s_tf[];  // 2 * n_tf entries (dynamic)
    const int tid = threadIdx.x;
    for (int i = tid; i < a.n_tf; i += blockDim.x) {
        const float4 e0 = a.tf[i];
        const float4 e1 = i + 1 < a.n_tf ? a.tf[i + 1] : e0;
        s_tf[2 * i] = e0;
        s_tf[2 * i + 1] = make_float4(e1.x - e0.x, e1.y - e0.y, e1.z - e0.z, e1.w - e0.w);
    }
    __syncthreads();

    const int lane = tid & 31;
    const int total = a.counters[0];  // written by ray_setup_kernel, which completed before this launch
    const int chx = a.chi[0], chy = a.chi[1], chz = a.chi[2];
    const unsigned sy = (unsigned)a.sy, sz = (unsigned)a.sz;
    const float* __restrict__ vox = a.vox;
    const float4* __restrict__ quad = a.quad;
    const uint8_t* __restrict__ skipd = a.skipd;
    const int mcd0 = a.mcd[0], mcd1 = a.mcd[1], skip = a.skip;
    const float vmin = a.vmin, tscale = a.tf_scale, top = (float)(a.n_tf - 1), ert = a.ert;
    const int tmax = a.n_tf - 2;

    bool have = false, exhausted = false;
    int pix = 0, nn = 0, j = 0;
#if DPRT_ASYNC
    int jend = 0, jpf = 0;  // [j, jend): verified non-empty run; [j, jpf): samples whose copies are issued
    const unsigned ring = (unsigned)__cvta_generic_to_shared(s_tf + 2 * a.n_tf) + (unsigned)tid * 16u;
#endif
#if DPRT_COUNTERS
    unsigned long long c_shade = 0, c_contrib = 0, c_skip = 0, c_rays = 0;
#endif
    float p0[3] = {0.f, 0.f, 0.f}, st[3] = {0.f, 0.f, 0.f}, ist[3] = {0.f, 0.f, 0.f};
    float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
#if DPRT_CHUNKED
    // Warp-private window of the ray queue: [cbase, cbase + cleft) are reserved for this warp; the next
    // window is requested from the global counter as soon as the current one runs dry, so the atomic's
    // latency overlaps marching instead of stalling the refill.
    int cbase = 0, cleft = 0;
    if (lane == 0) cbase = atomicAdd(a.counters + 1, kChunk);
    cbase = __shfl_sync(0xffffffffu, cbase, 0);
    cleft = cbase < total ? min(kChunk, total - cbase) : 0;
    int nbase = -1;  // pending next window (warp-uniform), -1 = none requested
#endif
    while (true) {
        unsigned act = __ballot_sync(0xffffffffu, have);
#if DPRT_CHUNKED
        if (!exhausted && __popc(act) < kRefillBelow) {
            const unsigned need = ~act;
            int k = __popc(need);
            if (cleft == 0) {
                if (nbase < 0) {
                    if (lane == 0) nbase = atomicAdd(a.counters + 1, kChunk);
                    nbase = __shfl_sync(0xffffffffu, nbase, 0);
                }
                cbase = nbase;
                cleft = cbase < total ? min(kChunk, total - cbase) : 0;
                nbase = -1;
                if (cleft == 0) exhausted = true;
            }
            const int take = min(k, cleft);
            if (!have) {
                const int rank = __popc(need & ((1u << lane) - 1));
                if (rank < take) {
                    const int idx = cbase + rank;
                    const float4 r0 = __ldg(a.rays + 2 * idx), r1 = __ldg(a.rays + 2 * idx + 1);
                    p0[0] = r0.x; p0[1] = r0.y; p0[2] = r0.z;
                    st[0] = r1.x; st[1] = r1.y; st[2] = r1.z;
#pragma unroll
                    for (int i = 0; i < 3; ++i) ist[i] = st[i] != 0.f ? __frcp_rn(st[i]) : 0.f;
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
            cbase += take;
            cleft -= take;
            if (cleft == 0 && !exhausted && nbase < 0) {  // request the next window early
                if (lane == 0) nbase = atomicAdd(a.counters + 1, kChunk);
                nbase = __shfl_sync(0xffffffffu, nbase, 0);
            }
            act = __ballot_sync(0xffffffffu, have);
        }
#else
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
#if DPRT_ASYNC
                    jend = jpf = 0;
#endif
                    C0 = C1 = C2 = A = 0.f;
                    have = true;
#if DPRT_COUNTERS
                    ++c_rays;
#endif
                }
            }
            act = __ballot_sync(0xffffffffu, have);
        }
#endif
        if (act == 0) {
#if DPRT_COUNTERS
            DPRT_COUNT(0, c_shade);
            DPRT_COUNT(1, c_contrib);
            DPRT_COUNT(2, c_skip);
            DPRT_COUNT(3, c_rays);
#endif
            break;
        }
#if DPRT_ASYNC
        for (int s = 0; have && s < kStepsPerCheck; ++s) {
            if (j >= nn) {
                asm volatile("cp.async.wait_all;\n" ::: "memory");  // no copy may land in a reused slot
                a.out[pix] = make_float4(C0, C1, C2, A);
                have = false;
                break;
            }
            if (j >= jend) {
                // Start of a run: locate the macrocell of sample j; hop over empty cubes.
                const float fj = (float)j;
                const int mx = min(__float2int_rd(fmaxf(fmaf(fj, st[0], p0[0]), 0.f)), chx) >> kMacroShift;
                const int my = min(__float2int_rd(fmaxf(fmaf(fj, st[1], p0[1]), 0.f)), chy) >> kMacroShift;
                const int mz = min(__float2int_rd(fmaxf(fmaf(fj, st[2], p0[2]), 0.f)), chz) >> kMacroShift;
                const int dist = skip ? (int)__ldg(skipd + (mz * mcd1 + my) * mcd0 + mx) : 0;
                const int r = dist > 0 ? dist : 1;
                float je = 3.0e38f;
                if (st[0] != 0.f)
                    je = fminf(je, ((float)((st[0] > 0.f ? mx + r : mx - r + 1) << kMacroShift) - p0[0]) * ist[0]);
                if (st[1] != 0.f)
                    je = fminf(je, ((float)((st[1] > 0.f ? my + r : my - r + 1) << kMacroShift) - p0[1]) * ist[1]);
                if (st[2] != 0.f)
                    je = fminf(je, ((float)((st[2] > 0.f ? mz + r : mz - r + 1) << kMacroShift) - p0[2]) * ist[2]);
                int jn = je < (float)nn ? (int)ceilf(je) : nn;
                if (jn <= j) jn = j + 1;
#if DPRT_COUNTERS
                if (dist > 0) ++c_skip;
#endif
                if (dist > 0) {
                    j = jpf = jn;  // empty cube: its samples would add exact zeros
                    continue;
                }
                jend = jn;
                jpf = j;
            }
            // Keep up to kDepth samples of the run in flight: cp.async copies the two corner quads of each
            // into this lane's ring slot in shared memory -- no registers held while the loads are out.
            while (jpf < jend && jpf < j + kDepth) {
                const float fp = (float)jpf;
                const int px_ = min(__float2int_rd(fmaxf(fmaf(fp, st[0], p0[0]), 0.f)), chx);
                const int py_ = min(__float2int_rd(fmaxf(fmaf(fp, st[1], p0[1]), 0.f)), chy);
                const int pz_ = min(__float2int_rd(fmaxf(fmaf(fp, st[2], p0[2]), 0.f)), chz);
                const float4* q = quad + ((unsigned)pz_ * sz + (unsigned)py_ * sy + (unsigned)px_);
                const unsigned slot = (unsigned)(jpf % kDepth);
                const unsigned dst = ring + (slot * 2u * kThreads) * 16u;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(q) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst + kThreads * 16u), "l"(q + sz)
                             : "memory");
                asm volatile("cp.async.commit_group;\n" ::: "memory");
                ++jpf;
            }
            // wait for sample j's group: (jpf - j - 1) younger groups may still be in flight
            switch (jpf - j - 1) {
                case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
                case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
                case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
                case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
                case 4: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
                case 5: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
                case 6: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
                default: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
            }
            const unsigned slot = (unsigned)(j % kDepth);
            float4 qa, qb;
            {
                const unsigned src = ring + (slot * 2u * kThreads) * 16u;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                             : "=f"(qa.x), "=f"(qa.y), "=f"(qa.z), "=f"(qa.w) : "r"(src) : "memory");
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                             : "=f"(qb.x), "=f"(qb.y), "=f"(qb.z), "=f"(qb.w) : "r"(src + kThreads * 16u) : "memory");
            }
            const float fs = (float)j;
            const float ux = fmaf(fs, st[0], p0[0]);
            const float uy = fmaf(fs, st[1], p0[1]);
            const float uz = fmaf(fs, st[2], p0[2]);
            const float wx = __saturatef(ux - (float)min(__float2int_rd(fmaxf(ux, 0.f)), chx));
            const float wy = __saturatef(uy - (float)min(__float2int_rd(fmaxf(uy, 0.f)), chy));
            const float wz = __saturatef(uz - (float)min(__float2int_rd(fmaxf(uz, 0.f)), chz));
            // trilinear + TF (§2.6) + front-to-back blend (§2.7)
            const float c00 = fmaf(wx, qa.y - qa.x, qa.x);
            const float c10 = fmaf(wx, qa.w - qa.z, qa.z);
            const float c01 = fmaf(wx, qb.y - qb.x, qb.x);
            const float c11 = fmaf(wx, qb.w - qb.z, qb.z);
            const float c0 = fmaf(wy, c10 - c00, c00);
            const float c1 = fmaf(wy, c11 - c01, c01);
            const float v = fmaf(wz, c1 - c0, c0);
            const float x = fminf(fmaxf((v - vmin) * tscale, 0.f), top);
            const int ti = min((int)x, tmax);
            const float tfr = x - (float)ti;
            const float4 e0 = s_tf[2 * ti], de = s_tf[2 * ti + 1];
            const float w = (1.f - A) * fmaf(tfr, de.w, e0.w);
#if DPRT_COUNTERS
            ++c_shade;
            c_contrib += w > 0.f;
#endif
            C0 = fmaf(w, fmaf(tfr, de.x, e0.x), C0);
            C1 = fmaf(w, fmaf(tfr, de.y, e0.y), C1);
            C2 = fmaf(w, fmaf(tfr, de.z, e0.z), C2);
            A += w;
            ++j;
            if (A >= ert) j = jend = nn;  // early ray termination: the next step finishes the ray
        }
#else
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
            const int mx = ix >> kMacroShift, my = iy >> kMacroShift, mz = iz >> kMacroShift;
            // Skip distance of this sample's macrocell.  An empty macrocell's sample would add exact
            // zeros: drop it and jump over the empty cube around it.
            const int mc = (mz * mcd1 + my) * mcd0 + mx;
            const int dist = skip ? (int)__ldg(skipd + mc) : 0;
            if (dist > 0) {
                // jump to the exit of the empty cube of macrocells [m - dist + 1, m + dist]
                float je = 3.0e38f;
                if (st[0] != 0.f)
                    je = fminf(je, ((float)((st[0] > 0.f ? mx + dist : mx - dist + 1) << kMacroShift) - p0[0]) * ist[0]);
                if (st[1] != 0.f)
                    je = fminf(je, ((float)((st[1] > 0.f ? my + dist : my - dist + 1) << kMacroShift) - p0[1]) * ist[1]);
                if (st[2] != 0.f)
                    je = fminf(je, ((float)((st[2] > 0.f ? mz + dist : mz - dist + 1) << kMacroShift) - p0[2]) * ist[2]);
                const int jn = je < (float)nn ? (int)ceilf(je) : nn;
                j = jn > j ? jn : j + 1;
#if DPRT_COUNTERS
                ++c_skip;
#endif
                continue;
            }
            // trilinear + TF (§2.6) + front-to-back blend (§2.7) of one sample
            auto shade = [&](float4 qa, float4 qb, float wx, float wy, float wz) {
                const float c00 = fmaf(wx, qa.y - qa.x, qa.x);
                const float c10 = fmaf(wx, qa.w - qa.z, qa.z);
                const float c01 = fmaf(wx, qb.y - qb.x, qb.x);
                const float c11 = fmaf(wx, qb.w - qb.z, qb.z);
                const float c0 = fmaf(wy, c10 - c00, c00);
                const float c1 = fmaf(wy, c11 - c01, c01);
                const float v = fmaf(wz, c1 - c0, c0);
                const float x = fminf(fmaxf((v - vmin) * tscale, 0.f), top);
                const int ti = min((int)x, tmax);
                const float tfr = x - (float)ti;
                const float4 e0 = s_tf[2 * ti], de = s_tf[2 * ti + 1];
                const float w = (1.f - A) * fmaf(tfr, de.w, e0.w);
#if DPRT_COUNTERS
                ++c_shade;
                c_contrib += w > 0.f;
#endif
                C0 = fmaf(w, fmaf(tfr, de.x, e0.x), C0);
                C1 = fmaf(w, fmaf(tfr, de.y, e0.y), C1);
                C2 = fmaf(w, fmaf(tfr, de.z, e0.z), C2);
                A += w;
            };
#if DPRT_QUAD
            // quad layout: one 16-byte load brings the 4 corners of a z-face of the cell
#if DPRT_FAKE_MEM
            const float4* q = quad + (((unsigned)iz * sz + (unsigned)iy * sy + (unsigned)ix) & 4095u);  // timing experiment only
#else
            const float4* q = quad + ((unsigned)iz * sz + (unsigned)iy * sy + (unsigned)ix);
#endif
            const float4 qa = __ldg(q), qb = __ldg(q + sz);
#else
            const float* p = vox + ((unsigned)iz * sz + (unsigned)iy * sy + (unsigned)ix);
            const float4 qa = make_float4(__ldg(p), __ldg(p + 1), __ldg(p + sy), __ldg(p + sy + 1));
            const float4 qb = make_float4(__ldg(p + sz), __ldg(p + sz + 1), __ldg(p + sz + sy), __ldg(p + sz + sy + 1));
#endif
#if DPRT_PAIR && DPRT_QUAD
            // Second sample of the step (j + 1) when it is still in a non-empty macrocell: its corner
            // loads are issued before the first sample is shaded, doubling memory-level parallelism.
            const float fs1 = fs + 1.f;
            const float vx1 = fmaf(fs1, st[0], p0[0]);
            const float vy1 = fmaf(fs1, st[1], p0[1]);
            const float vz1 = fmaf(fs1, st[2], p0[2]);
            const int jx1 = min(__float2int_rd(fmaxf(vx1, 0.f)), chx);
            const int jy1 = min(__float2int_rd(fmaxf(vy1, 0.f)), chy);
            const int jz1 = min(__float2int_rd(fmaxf(vz1, 0.f)), chz);
            const int mc1 = ((jz1 >> kMacroShift) * mcd1 + (jy1 >> kMacroShift)) * mcd0 + (jx1 >> kMacroShift);
            bool two = j + 1 < nn;
            if (two && skip && mc1 != mc) two = __ldg(skipd + mc1) == 0;
            float4 qa1 = qa, qb1 = qb;
            if (two) {
                const float4* q1 = quad + ((unsigned)jz1 * sz + (unsigned)jy1 * sy + (unsigned)jx1);
                qa1 = __ldg(q1);
                qb1 = __ldg(q1 + sz);
            }
            shade(qa, qb, __saturatef(ux - (float)ix), __saturatef(uy - (float)iy), __saturatef(uz - (float)iz));
            ++j;
            if (A >= ert) {  // early ray termination: the next step finishes the ray
                j = nn;
                continue;
            }
            if (two) {
                shade(qa1, qb1, __saturatef(vx1 - (float)jx1), __saturatef(vy1 - (float)jy1),
                      __saturatef(vz1 - (float)jz1));
                ++j;
                if (A >= ert) j = nn;
            }
#else
            shade(qa, qb, __saturatef(ux - (float)ix), __saturatef(uy - (float)iy), __saturatef(uz - (float)iz));
            ++j;
            if (A >= ert) j = nn;  // early ray termination: the next step finishes the ray
#endif
        }
#endif
    }
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

__global__ void skip_pass_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int n0, int n1, int n2,
                                 int axis) {
    const long long total = (long long)n0 * n1 * n2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % n0);
        const int y = (int)((i / n0) % n1);
        const int z = (int)(i / ((long long)n0 * n1));
        const int c = axis == 0 ? x : (axis == 1 ? y : z);
        const int n = axis == 0 ? n0 : (axis == 1 ? n1 : n2);
        const long long stride = axis == 0 ? 1 : (axis == 1 ? n0 : (long long)n0 * n1);
        int best = in[i];
        for (int k = 1; k < best && k < kSkipCap; ++k) {
            if (c - k >= 0) best = min(best, max(k, (int)in[i - k * stride]));
            if (c + k < n) best = min(best, max(k, (int)in[i + k * stride]));
        }
        out[i] = (uint8_t)best;
    }
}

cudaError_t launch_skip_build(const DeviceBrick& b, const MarchArgs& a, uint8_t* tmp, cudaStream_t stream) {
    const long long nmc = (long long)b.mcd[0] * b.mcd[1] * b.mcd[2];
    const int block = 256;
    const long long want = (nmc + block - 1) / block;
    const int grid = (int)(want < 148LL * 16 ? (want > 0 ? want : 1) : 148LL * 16);
    skip_classify_kernel<<<grid, block, 0, stream>>>(b.macro, nmc, a.tf, a.n_tf, a.vmin, a.tf_scale, b.skipd);
    skip_pass_kernel<<<grid, block, 0, stream>>>(b.skipd, tmp, (int)b.mcd[0], (int)b.mcd[1], (int)b.mcd[2], 2);
    skip_pass_kernel<<<grid, block, 0, stream>>>(tmp, b.skipd, (int)b.mcd[0], (int)b.mcd[1], (int)b.mcd[2], 1);
    skip_pass_kernel<<<grid, block, 0, stream>>>(b.skipd, tmp, (int)b.mcd[0], (int)b.mcd[1], (int)b.mcd[2], 0);
    return cudaMemcpyAsync(b.skipd, tmp, (size_t)nmc, cudaMemcpyDeviceToDevice, stream);
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
cudaError_t launch_march(const MarchArgs& a, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(a.counters, 0, 2 * sizeof(int), stream);
    if (e != cudaSuccess) return e;
    dim3 block(kTileX * kTileY);
    dim3 grid((a.W + kTileX - 1) / kTileX, (a.H + kTileY - 1) / kTileY);
    ray_setup_kernel<<<grid, block, 0, stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t smem = 2 * a.n_tf * sizeof(float4);
#if DPRT_ASYNC
    smem += (size_t)kDepth * 2 * kThreads * sizeof(float4);  // per-lane ring of corner quads
    cudaFuncSetAttribute(march_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#endif
#ifdef DPRT_CARVEOUT
    cudaFuncSetAttribute(march_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, DPRT_CARVEOUT);
#endif
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_kernel, kTileX * kTileY, smem);
    if (per_sm < 1) per_sm = 1;
    march_kernel<<<sms * per_sm, block, smem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace dprt

// Triangle BVH traversal on the GPU: the reference's own per-rank compute slot, trace_nearest_batch /
// trace_any_batch (pkg/src/dprt/bvh.py:284-311, called by engine.trace_local_round, engine.py:254-279),
// restated as sm_100a kernels over the reference's flat Accel arrays (bvh.py:46-60) -- the triangle half of
// SURVEY §8(f) row 4 (ray-queue cycling on the GPU).  One thread per ray, an explicit traversal stack like
// the reference's (MAX_STACK = 64, bvh.py:23), and every float64 operation explicitly rounded in the
// reference's evaluation order (no FMA contraction), so each ray's (t, global id) -- and each shadow ray's
// occlusion bit -- is bit-identical to the numba reference (tests/test_gpu_trace.py, golden vectors
// generated from the reference, tests/golden/make_trace_golden.py).

#include <math.h>

#include "common.cuh"

namespace dprt {

constexpr int kTraceStack = 64;  // bvh.py:23 MAX_STACK

struct BvhArgs {
    const double* __restrict__ lo;
    const double* __restrict__ hi;
    const int64_t* __restrict__ left;
    const int64_t* __restrict__ right;
    const int64_t* __restrict__ first;
    const int64_t* __restrict__ count;
    int64_t root;
    const double* __restrict__ tv;   // (m, 9) v0 v1 v2
    const int64_t* __restrict__ tid;
};

// bvh.py:191-220 _node_interval: false on a definite miss (the reference's (1.0, -1.0)).
// ``inv[axis]`` = 1.0 / d[axis], the reference's per-node reciprocal -- the same correctly rounded value for
// every node, so it is formed once per ray (a float64 division is a long instruction sequence).
__device__ __forceinline__ bool node_interval(const BvhArgs& b, int64_t ni, const double o[3], const double d[3],
                                              const double inv[3], double* pt0, double* pt1) {
    double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
        const double lo = __ldg(b.lo + 3 * ni + axis), hi = __ldg(b.hi + 3 * ni + axis);
        if (d[axis] == 0.0) {
            if (o[axis] < lo || o[axis] > hi) return false;
            continue;
        }
        double ta = __dmul_rn(__dsub_rn(lo, o[axis]), inv[axis]);
        double tb = __dmul_rn(__dsub_rn(hi, o[axis]), inv[axis]);
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

// bvh.py:160-188 _tri_t: unbounded Moller-Trumbore t of triangle slot k, +inf on a miss.
__device__ __forceinline__ double tri_t(const double* __restrict__ tv, int64_t k, const double o[3], const double d[3]) {
    const double* v = tv + 9 * k;
    const double v0x = __ldg(v), v0y = __ldg(v + 1), v0z = __ldg(v + 2);
    const double e1x = __dsub_rn(__ldg(v + 3), v0x), e1y = __dsub_rn(__ldg(v + 4), v0y), e1z = __dsub_rn(__ldg(v + 5), v0z);
    const double e2x = __dsub_rn(__ldg(v + 6), v0x), e2y = __dsub_rn(__ldg(v + 7), v0y), e2z = __dsub_rn(__ldg(v + 8), v0z);
    const double px = __dsub_rn(__dmul_rn(d[1], e2z), __dmul_rn(d[2], e2y));
    const double py = __dsub_rn(__dmul_rn(d[2], e2x), __dmul_rn(d[0], e2z));
    const double pz = __dsub_rn(__dmul_rn(d[0], e2y), __dmul_rn(d[1], e2x));
    const double det = __dadd_rn(__dadd_rn(__dmul_rn(e1x, px), __dmul_rn(e1y, py)), __dmul_rn(e1z, pz));
    if (det == 0.0) return INFINITY;
    const double inv_det = __ddiv_rn(1.0, det);
    const double tx = __dsub_rn(o[0], v0x), ty = __dsub_rn(o[1], v0y), tz = __dsub_rn(o[2], v0z);
    const double u = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(tx, px), __dmul_rn(ty, py)), __dmul_rn(tz, pz)), inv_det);
    if (u < 0.0 || u > 1.0) return INFINITY;
    const double qx = __dsub_rn(__dmul_rn(ty, e1z), __dmul_rn(tz, e1y));
    const double qy = __dsub_rn(__dmul_rn(tz, e1x), __dmul_rn(tx, e1z));
    const double qz = __dsub_rn(__dmul_rn(tx, e1y), __dmul_rn(ty, e1x));
    const double vv = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], qx), __dmul_rn(d[1], qy)), __dmul_rn(d[2], qz)), inv_det);
    if (vv < 0.0 || __dadd_rn(u, vv) > 1.0) return INFINITY;
    return __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz)), inv_det);
}

// Push an inner node's children so that the one whose box centre lies nearer along the ray is popped first.
// The reference always descends left first (bvh.py:253-255); the order cannot change a result -- every hit is
// min-reduced with the (t, id) tie-break and a node is pruned only when its entry t exceeds the current best
// -- but nearer-first lets best_t shrink early and prune more.  The ordering key is float (a heuristic only).
#ifndef DPRT_TRACE_ORDERED
#define DPRT_TRACE_ORDERED 1
#endif
__device__ __forceinline__ void push_children(const BvhArgs& b, int ni, const float df[3], int* stack, int& sp) {
    const int l = (int)__ldg(b.left + ni), r = (int)__ldg(b.right + ni);
#if DPRT_TRACE_ORDERED
    float kl = 0.f, kr = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        kl = fmaf((float)(__ldg(b.lo + 3 * l + a) + __ldg(b.hi + 3 * l + a)), df[a], kl);
        kr = fmaf((float)(__ldg(b.lo + 3 * r + a) + __ldg(b.hi + 3 * r + a)), df[a], kr);
    }
    const bool left_first = kl <= kr;
    stack[sp] = left_first ? r : l;
    stack[sp + 1] = left_first ? l : r;
#else
    stack[sp] = r;
    stack[sp + 1] = l;
#endif
    sp += 2;
}

// bvh.py:223-256 _nearest_one, one thread per ray, (best_t, best_id) min-reduced in place.
__global__ void __launch_bounds__(128) trace_nearest_kernel(const BvhArgs b, long long n, const double* __restrict__ org,
                                                            const double* __restrict__ dirn,
                                                            const double* __restrict__ tmin_a,
                                                            const double* __restrict__ tmax_a, double* best_t_a,
                                                            int64_t* best_id_a) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double best_t = best_t_a[i];
        int64_t best_id = best_id_a[i];
        if (b.root >= 0) {
            const double o[3] = {org[3 * i], org[3 * i + 1], org[3 * i + 2]};
            const double d[3] = {dirn[3 * i], dirn[3 * i + 1], dirn[3 * i + 2]};
            const double tmin = tmin_a[i], tmax = tmax_a[i];
            double inv[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) inv[a] = d[a] != 0.0 ? __ddiv_rn(1.0, d[a]) : 0.0;
            const float df[3] = {(float)d[0], (float)d[1], (float)d[2]};
            int stack[kTraceStack];
            int sp = 0;
            stack[sp++] = (int)b.root;
            while (sp > 0) {
                const int ni = stack[--sp];
                double t0, t1;
                const bool hit = node_interval(b, ni, o, d, inv, &t0, &t1);
                const double limit = tmax < best_t ? tmax : best_t;
                if (!hit || t1 < tmin || t0 > limit) continue;
                const int64_t cnt = __ldg(b.count + ni);
                if (cnt > 0) {
                    const int64_t f = __ldg(b.first + ni);
                    for (int64_t k = f; k < f + cnt; ++k) {
                        const double t = tri_t(b.tv, k, o, d);
                        if (!(tmin <= t && t <= tmax && t < INFINITY)) continue;  // rejects NaN too
                        const int64_t id = __ldg(b.tid + k);
                        if (t < best_t || (t == best_t && id < best_id)) {
                            best_t = t;
                            best_id = id;
                        }
                    }
                } else {
                    push_children(b, ni, df, stack, sp);
                }
            }
        }
        best_t_a[i] = best_t;
        best_id_a[i] = best_id;
    }
}

// bvh.py:259-281 _any_one: occluded |= any triangle strictly inside (tmin, tmax); occluded rays are skipped.
__global__ void __launch_bounds__(128) trace_any_kernel(const BvhArgs b, long long n, const double* __restrict__ org,
                                                        const double* __restrict__ dirn,
                                                        const double* __restrict__ tmin_a,
                                                        const double* __restrict__ tmax_a, uint8_t* occluded) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (occluded[i] || b.root < 0) continue;
        const double o[3] = {org[3 * i], org[3 * i + 1], org[3 * i + 2]};
        const double d[3] = {dirn[3 * i], dirn[3 * i + 1], dirn[3 * i + 2]};
        const double tmin = tmin_a[i], tmax = tmax_a[i];
        double inv[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) inv[a] = d[a] != 0.0 ? __ddiv_rn(1.0, d[a]) : 0.0;
            const float df[3] = {(float)d[0], (float)d[1], (float)d[2]};
        int stack[kTraceStack];
        int sp = 0;
        stack[sp++] = (int)b.root;
        bool occ = false;
        while (sp > 0 && !occ) {
            const int ni = stack[--sp];
            double t0, t1;
            if (!node_interval(b, ni, o, d, inv, &t0, &t1) || t1 < tmin || t0 > tmax) continue;
            const int64_t cnt = __ldg(b.count + ni);
            if (cnt > 0) {
                const int64_t f = __ldg(b.first + ni);
                for (int64_t k = f; k < f + cnt; ++k) {
                    const double t = tri_t(b.tv, k, o, d);
                    if (tmin < t && t < tmax) {
                        occ = true;
                        break;
                    }
                }
            } else {
                push_children(b, ni, df, stack, sp);
            }
        }
        if (occ) occluded[i] = 1;
    }
}

cudaError_t launch_trace(const BvhArgs& b, long long n, const double* org, const double* dirn, const double* tmin,
                         const double* tmax, double* best_t, int64_t* best_id, uint8_t* occluded, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const long long want = (n + 127) / 128;
    const int grid = (int)(want < 148LL * 64 ? want : 148LL * 64);
    if (occluded)
        trace_any_kernel<<<grid, 128, 0, stream>>>(b, n, org, dirn, tmin, tmax, occluded);
    else
        trace_nearest_kernel<<<grid, 128, 0, stream>>>(b, n, org, dirn, tmin, tmax, best_t, best_id);
    return cudaGetLastError();
}

}  // namespace dprt

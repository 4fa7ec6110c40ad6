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
// * CTA = 16x16 pixel tile, each warp an 8x4 tile, so the 32 rays of a warp stay within a few voxels
//   of each other and their 8-corner gathers share L1 lines.

#include <math.h>

#include "common.cuh"

namespace dprt {

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

__global__ void __launch_bounds__(kTileX * kTileY) march_kernel(const MarchArgs a) {
    __shared__ float4 s_tf[kMaxTf];
    __shared__ int s_next_nz[kMaxTf];  // smallest entry index >= i whose alpha > 0 (n_tf if none)

    const int tid = threadIdx.x;
    for (int i = tid; i < a.n_tf; i += blockDim.x) s_tf[i] = a.tf[i];
    if (a.skip) {
        // suffix scan of "alpha > 0" by one warp (n_tf <= 1024)
        if (tid < 32) {
            int carry = a.n_tf;
            for (int base = ((a.n_tf - 1) / 32) * 32; base >= 0; base -= 32) {
                int i = base + tid;
                bool nz = i < a.n_tf && a.tf[i].w > 0.0f;
                unsigned m = __ballot_sync(0xffffffffu, nz);
                unsigned here = m & (0xffffffffu << tid);
                int nxt = here ? base + __ffs(here) - 1 : carry;
                if (i < a.n_tf) s_next_nz[i] = nxt;
                int lowest = m ? base + __ffs(m) - 1 : carry;
                carry = __shfl_sync(0xffffffffu, lowest, 0);
            }
        }
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;
    const int px = blockIdx.x * kTileX + (warp & 1) * 8 + (lane & 7);
    const int py = blockIdx.y * kTileY + (warp >> 1) * 4 + (lane >> 3);
    if (px >= a.W || py >= a.H) return;
    const int64_t pix = (int64_t)py * a.W + px;

    const bool in_rect = px >= a.rect[0] && py >= a.rect[1] && px < a.rect[2] && py < a.rect[3];
    int64_t k0 = 0, n = 0;
    double d[3];
    if (in_rect) {
        primary_dir(a, px, py, d);
        n = lattice_range(a, d, &k0);
    }
    float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
    if (n > 0) {
        // start position in local (stored) continuous index space, and per-sample step
        float p0[3], st[3];
        const double t0 = __dmul_rn((double)k0, a.dt);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double p = (a.o[i] + t0 * d[i] - a.origin[i]) / a.spacing[i];
            p0[i] = (float)(p - a.stored_lo_d[i]);
            st[i] = (float)(a.dt * d[i]) * a.inv_spacing[i];
        }
        const float top = (float)(a.n_tf - 1);
        int cur_mc = -1;
        int j = 0;
        const int nn = (int)n;
        while (j < nn) {
            const float fj = (float)j;
            const float ux = fmaf(fj, st[0], p0[0]);
            const float uy = fmaf(fj, st[1], p0[1]);
            const float uz = fmaf(fj, st[2], p0[2]);
            const int ix = clampi(__float2int_rd(ux), a.clo[0], a.chi[0]);
            const int iy = clampi(__float2int_rd(uy), a.clo[1], a.chi[1]);
            const int iz = clampi(__float2int_rd(uz), a.clo[2], a.chi[2]);
            if (a.skip) {
                const int mx = ix >> kMacroShift, my = iy >> kMacroShift, mz = iz >> kMacroShift;
                const int mc = (mz * a.mcd[1] + my) * a.mcd[0] + mx;
                if (mc != cur_mc) {
                    const float2 mm = __ldg(&a.macro[mc]);
                    const float xl = fminf(fmaxf((mm.x - a.vmin) * a.tf_scale, 0.f), top);
                    const float xh = fminf(fmaxf((mm.y - a.vmin) * a.tf_scale, 0.f), top);
                    const int il = (int)xl;
                    const int ih = min((int)xh + 2, a.n_tf - 1);
                    if (s_next_nz[il] > ih) {
                        // empty: jump to the first sample past this macrocell's far faces
                        float jx = INFINITY, jy = INFINITY, jz = INFINITY;
                        if (st[0] > 0.f) jx = ((float)((mx + 1) << kMacroShift) - p0[0]) / st[0];
                        else if (st[0] < 0.f) jx = ((float)(mx << kMacroShift) - p0[0]) / st[0];
                        if (st[1] > 0.f) jy = ((float)((my + 1) << kMacroShift) - p0[1]) / st[1];
                        else if (st[1] < 0.f) jy = ((float)(my << kMacroShift) - p0[1]) / st[1];
                        if (st[2] > 0.f) jz = ((float)((mz + 1) << kMacroShift) - p0[2]) / st[2];
                        else if (st[2] < 0.f) jz = ((float)(mz << kMacroShift) - p0[2]) / st[2];
                        const float je = fminf(jx, fminf(jy, jz));
                        int jn = je < (float)nn ? (int)ceilf(je) : nn;
                        j = jn > j ? jn : j + 1;
                        cur_mc = -1;
                        continue;
                    }
                    cur_mc = mc;
                }
            }
            const float wx = __saturatef(ux - (float)ix);
            const float wy = __saturatef(uy - (float)iy);
            const float wz = __saturatef(uz - (float)iz);
            const float* p = a.vox + (long long)iz * a.sz + (long long)iy * a.sy + ix;
            const float v000 = __ldg(p), v100 = __ldg(p + 1);
            const float v010 = __ldg(p + a.sy), v110 = __ldg(p + a.sy + 1);
            const float v001 = __ldg(p + a.sz), v101 = __ldg(p + a.sz + 1);
            const float v011 = __ldg(p + a.sz + a.sy), v111 = __ldg(p + a.sz + a.sy + 1);
            const float c00 = fmaf(wx, v100 - v000, v000);
            const float c10 = fmaf(wx, v110 - v010, v010);
            const float c01 = fmaf(wx, v101 - v001, v001);
            const float c11 = fmaf(wx, v111 - v011, v011);
            const float c0 = fmaf(wy, c10 - c00, c00);
            const float c1 = fmaf(wy, c11 - c01, c01);
            const float v = fmaf(wz, c1 - c0, c0);
            // transfer function
            const float x = fminf(fmaxf((v - a.vmin) * a.tf_scale, 0.f), top);
            const int ti = min((int)x, a.n_tf - 2);
            const float tfr = x - (float)ti;
            const float4 e0 = s_tf[ti], e1 = s_tf[ti + 1];
            const float ea = fmaf(tfr, e1.w - e0.w, e0.w);
            // front-to-back, premultiplied
            const float w = (1.f - A) * ea;
            C0 = fmaf(w, fmaf(tfr, e1.x - e0.x, e0.x), C0);
            C1 = fmaf(w, fmaf(tfr, e1.y - e0.y, e0.y), C1);
            C2 = fmaf(w, fmaf(tfr, e1.z - e0.z, e0.z), C2);
            A += w;
            if (A >= a.ert) break;
            ++j;
        }
    }
    a.out[pix] = make_float4(C0, C1, C2, A);
    if (a.samples) a.samples[pix] = (uint32_t)n;
}

// Host launcher (called from abi.cu).
cudaError_t launch_march(const MarchArgs& a, cudaStream_t stream) {
    dim3 block(kTileX * kTileY);
    dim3 grid((a.W + kTileX - 1) / kTileX, (a.H + kTileY - 1) / kTileY);
    march_kernel<<<grid, block, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace dprt

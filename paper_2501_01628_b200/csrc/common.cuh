// Shared definitions for the sm_100a kernels of libdprt_cuda.so (see include/dprt_cuda.h).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dprt_cuda.h"

#ifndef DPRT_BEAM_DEFAULT
#define DPRT_BEAM_DEFAULT 1
#endif
#ifndef DPRT_COUNTERS
#define DPRT_COUNTERS 0
#endif

// Quad memory order: 0 = x fastest (default), 1 = y fastest, then x, then z.  A warp beam is
// 4 x 8 pixels, tall in screen y, so with a y-up camera y-fastest quads put one batch's 32 loads into fewer
// 128-byte lines (c2 host replay: 13.6 -> 9.4 lines per load).  Measured (round 2): c2 0.2270 -> 0.2286 ms,
// config 3 even rank 5 0.774 -> 0.752, mass rank 7 0.543 -> 0.546 -- line count is not what bounds the
// loads (profiles/r02_variant_memory_side.json), so x-fastest stays.
// Coefficient octets (DPRT_QUAD_OCTET): the slot of a voxel holds both z-faces of its cell (32 bytes), one
// 256-bit load per sample instead of two 128-bit ones (f32 quads only; fp16 quads keep one face per slot).
#ifndef DPRT_QUAD_OCTET
#define DPRT_QUAD_OCTET 0
#endif

#ifndef DPRT_QUAD_YFAST
#define DPRT_QUAD_YFAST 0
#endif

namespace dprt {

#ifndef DPRT_MACRO_SHIFT
#define DPRT_MACRO_SHIFT 3
#endif
// Macrocell edge per brick (DeviceBrick::mshift): large bricks (>= 2^28 stored voxels, memory-latency bound)
// keep 8^3 macrocells; smaller ones (issue / L1 bound, where every skipped sample counts) use 4^3 -- c2 -4.7 %,
// config 3's mass-balanced slowest brick +1.5 % with 4^3 (profiles/r02_variant_memory_side.json).
#ifndef DPRT_BEAM_PROBE
#define DPRT_BEAM_PROBE 1  // per-lane skip probes (0: the measured beam-wide alternative, 8^3 macrocells only)
#endif
#ifndef DPRT_MACRO_SHIFT_SMALL
#define DPRT_MACRO_SHIFT_SMALL 2
#endif
constexpr int kMacroShift = DPRT_MACRO_SHIFT;  // the large-brick (and upper-bound) macrocell shift
constexpr int kQuadSlot = DPRT_QUAD_OCTET ? 2 : 1;  // float4s per f32 quad slot
constexpr int kMacro = 1 << kMacroShift;  // macrocell edge in cells (empty-space skipping granularity)
constexpr int kTileX = 16;         // marcher CTA screen tile: 16 x 16 pixels, warps are 8 x 4 pixel tiles
constexpr int kTileY = 16;
constexpr int kMaxTf = 1024;       // transfer-function entries held in shared memory
#ifndef DPRT_SKIP_CAP
#define DPRT_SKIP_CAP 31
#endif
constexpr int kSkipCap = DPRT_SKIP_CAP;  // Chebyshev skip distances are capped at this many macrocells
#ifndef DPRT_SKIP_OCTANT
#define DPRT_SKIP_OCTANT 1  // the beam marcher's per-lane probe jumps by one-sided (octant) distances
#endif
constexpr int kSkipGrids = 9;  // symmetric + 8 octants
#ifndef DPRT_SETUP_FAST
#define DPRT_SETUP_FAST 0  // beam marcher: f64 ray setup with Newton-refined rcp / rsqrt, the exact setup only for
#endif                     // lanes whose lattice range it cannot prove (march.cu fast_range)
#ifndef DPRT_SUBBLOCK
#define DPRT_SUBBLOCK 0  // 1 / 2: the probe also skips empty 4^3 sub-blocks of non-empty macrocells (measured:
#endif                   // 9 % fewer shaded samples on c2 but 0.7 % slower, config 3 2-4 % slower; not adopted)
constexpr float kHalfQuadRange = 8.0f;  // fp16 quads (DPRT_BRICK_HALF_QUADS) take field values within +-8

struct DeviceBrick {
    int device;
    DprtBrickDesc desc;
    int64_t s_lo[3];   // first stored voxel (global index)
    int64_t sd[3];     // stored voxel dims
    float* vox;        // sd[0]*sd[1]*sd[2] f32, x fastest
    float4* quad;      // coefficient quads over the apron grid qd (field.cu quad_kernel); with
                       // DPRT_BRICK_HALF_QUADS the same slots hold 4 x fp16 (uint2) instead
    int half_quads;
    int64_t qd[3];     // quad grid dims = sd + 2 (one apron voxel on every side)
    int64_t mcd[3];    // macrocell grid dims
    int mshift;        // macrocell edge = 1 << mshift cells (chosen by brick size at creation)
    float2* macro;     // per macrocell (min, max) over its dilated voxel range
    float2* sub;       // per macrocell, its eight 4^3-cell sub-blocks' dilated (min, max) (bit b: x, y, z halves)
    uint8_t* subm;     // per macrocell, bit b set = sub-block b is not empty under the current TF
    uint8_t* skipd;    // kSkipGrids grids of nmc bytes (TF-dependent): [0] per macrocell Chebyshev distance to
                       // the nearest non-empty macrocell; [1 + o] the same restricted to octant o of directions
                       // (bit i of o: + along axis i), which a ray moving into octant o may jump by
    uint8_t* skip_tmp; // scratch for the separable distance passes (2 x kSkipGrids x nmc)
    uint64_t skip_version;  // tf_version the skip distances were built for (0 = never)
    float4* rays;      // ray queue scratch (2 float4 per pixel of the largest frame marched so far)
    long long ray_cap; // pixels the queue can hold
    int* counters;     // queue counters (2 per slot), then the fp16-quad range flag
};

// Everything the marcher needs, by value (kernel parameter space).
struct MarchArgs {
    // camera (f64, host-evaluated basis)
    double o[3], f[3], r[3], u[3];
    double half_w, half_h;
    // owned box in world space, field origin and spacing (f64, exact ray setup)
    double blo[3], bhi[3];
    double origin[3], spacing[3];
    double dt;
    double inv_dt_pow2;       // 1 / dt when dt is a power of two (t / dt == t * inv exactly), else 0
    double inv_spacing_d[3];  // 1 / spacing (start positions only; not on the exact ownership path)
    // f32 march state
    float inv_spacing[3];
    double stored_lo_d[3];  // s_lo (local coordinate shift)
    int clo[3], chi[3];    // local clamp range of the cell index (macrocell lookups)
    int sd[3];
    long long sy, sz;      // voxel strides
    const float* __restrict__ vox;
    const float4* __restrict__ qorg;  // coefficient quad of stored voxel (0,0,0); apron at index -1 and sd
    int qsx, qsy, qsz;                // quad strides (apron grid; DPRT_QUAD_YFAST: y is the unit stride)
    int wide;                         // >= 2^31 apron quads: unsigned offsets from the apron base (kWide)
    int deep;                         // large brick: the memory-latency-bound configuration (kDeepUnroll)
    int half_quads;                   // quads stored as 4 x fp16 (DPRT_BRICK_HALF_QUADS)
    const uint8_t* __restrict__ skipd;  // the symmetric grid; octant o's at skipd + (1 + o) * skip_n
    long long skip_n;                   // macrocells per grid
    int mshift;                         // the brick's macrocell shift (DeviceBrick::mshift)
    // conservative f32 miss pre-test (DPRT_MISS_TEST): camera basis and the owned box relative to the eye,
    // expanded by a margin far above f32 rounding; a ray missing that box misses the exact one
    float mt_f[3], mt_r[3], mt_u[3], mt_lo[3], mt_hi[3];
    float mt_hw, mt_hh, mt_iw, mt_ih;
    const uint8_t* __restrict__ subm;   // per macrocell: non-empty 4^3 sub-blocks (DPRT_SUBBLOCK)
    // fast ray setup (DPRT_SETUP_FAST): 2/W, 2/H, the owned box relative to the eye (the exact path's own
    // f64 differences), 1/dt, the direction-component scale 1 + half_w + half_h; fs_ok = 0 -> exact only
    double fs_iw2, fs_ih2, fs_L[3], fs_H[3], fs_idt, fs_S;
    int fs_ok;
    int mcd[3];
    int skip;
    int band_clear;  // clear only the footprint's row band of the partial (DPRT_MARCH_BAND_CLEAR)
    int accum;       // continue from / write back each ray's accumulated state (DPRT_MARCH_ACCUM)
    int half_out;    // the partial is fp16 RGBA (DPRT_MARCH_HALF): out16 instead of out
    long long pix0;      // out[] and samples[] hold pixels from index pix0 = row0 * W on (row window)
    long long npix_buf;  // pixels out[] / samples[] hold (W * H, or the row window's)
    int beam;  // 1: march_beam_kernel (warp beams, per-pixel ray records); 0: ray queue + march_kernel
    // transfer function
    const float4* __restrict__ tf;
    int n_tf;
    float vmin, tf_scale, ert;
    float tf_ns, tf_no;  // normalised TF coordinate = sat(v * tf_ns + tf_no), tf_ns = 1 / (vmax - vmin)
    // output
    float4* __restrict__ out;
    uint2* __restrict__ out16;  // fp16 RGBA partial (4 halves per pixel)
    uint8_t* rgb8;  // non-null: write the tone-mapped frame over bg[] instead of the RGBA partial (R == 1)
    float bg[3];
    uint32_t* __restrict__ samples;
    float4* rays;   // compacted ray queue: 2 float4 per ray {p0, pixel}, {step, n}
    int* counters;  // [0] rays queued by ray_setup, [1] rays taken by march
    // fused march + exchange (dprt_march_push): row block b of the partial goes to push_dst[b] (its owner's
    // inbox, a peer pointer), pixel (x, y) at element (y - push_row[b]) * W + x; the launch's last CTA then
    // release-stores push_epoch into every push_flag[b]
    int push_P;                          // 0: the partial is out / out16 (local)
    int push_row[DPRT_MAX_PUSH + 1];
    char* push_dst[DPRT_MAX_PUSH];
    unsigned* push_flag[DPRT_MAX_PUSH];
    unsigned* push_ctr;
    unsigned push_epoch;
    uint8_t* mark;                    // dprt_march_stats: per-macrocell "a real sample was shaded here" bytes
    unsigned long long* stats;        // dprt_march_stats: {shaded samples, contributing samples}
    int W, H;
    int rect[4];
};

struct CompositeArgs {
    const float4* in[DPRT_MAX_PARTS];  // fragment i's element for tile pixel p is in[i][p - lo[i]]
                                       // (fp16 fragments with DPRT_COMPOSITE_HALF_IN: a uint2 per pixel)
    long long lo[DPRT_MAX_PARTS], hi[DPRT_MAX_PARTS];  // tile pixels [lo, hi) fragment i covers (else clear)
    int P;
    long long npix;
    float bg[3];
    int flags;
    uint8_t* rgb8;
    float4* rgba;
    // dprt_composite_signal: the launch's last CTA release-stores sig_epoch into sig[0 .. n_sig)
    int n_sig;
    unsigned sig_epoch;
    unsigned* sig_ctr;
    unsigned* sig[DPRT_MAX_PUSH];
};

// System-scope release / acquire on a flag word (local or peer memory over NVLink).
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Last-CTA completion signal.  The CTA's threads meet at a barrier and its thread 0 fences at system scope
// (cumulative: the fence orders every store the barrier ordered before it, the whole CTA's), then counts the
// CTA in one of up to 32 sub-counters (128-byte apart: a single counter serialised 4,000 CTAs of a 4K
// row-block blend for ~14 us); the CTA that completes a sub-counter fences and counts it in the top counter,
// and the one that completes the top counter fences and release-stores `epoch` into flags[0 .. n).
// atomicInc wraps every counter back to 0, ready for the next launch.  `ctr` points at
// DPRT_SIGNAL_COUNTER_WORDS zeroed words.  Every thread of every CTA must reach this call.
constexpr unsigned kSigSub = 32, kSigStride = 32;  // sub-counters, words between counters
#ifndef DPRT_SIGNAL_FENCE
#define DPRT_SIGNAL_FENCE 2  // per-CTA fence before counting: 2 = system scope, 1 = GPU scope, 0 = none (timing only)
#endif
__device__ __forceinline__ void grid_signal(unsigned* ctr, unsigned* const* flags, int n, unsigned epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
#if DPRT_SIGNAL_FENCE == 2
        __threadfence_system();
#elif DPRT_SIGNAL_FENCE == 1
        __threadfence();
#endif
        const unsigned total = gridDim.x * gridDim.y * gridDim.z;
        const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        const unsigned nsub = total < kSigSub ? total : kSigSub;
        const unsigned i = cta % nsub;
        const unsigned quota = total / nsub + (i < total % nsub ? 1u : 0u);
        if (atomicInc(ctr + kSigStride * (1 + i), quota - 1) == quota - 1) {
            __threadfence_system();
            if (atomicInc(ctr, nsub - 1) == nsub - 1) {
                __threadfence_system();  // one release fence for all n flags (st.release would fence per store)
                for (int f = 0; f < n; ++f) st_relaxed_sys(flags[f], epoch);
            }
        }
    }
}

}  // namespace dprt

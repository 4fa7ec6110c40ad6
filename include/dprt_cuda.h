/*
 * dprt_cuda.h -- C ABI of libdprt_cuda.so, the B200 (sm_100a) data path for per-rank direct volume
 * rendering of a brick and sort-last compositing of the RGBA partials.
 *
 * The reference (arxiv/paper_2501_01628, Python package `dprt`) has no native code; its per-rank compute
 * slot is a numba call with flat contiguous arrays, outputs mutated in place, no return value and the GIL
 * released (pkg/src/dprt/engine.py:254-279 -> bvh.py:284-311, `@njit(nogil=True)` bvh.py:160).  Each entry
 * point below takes that slot's place in the same style: plain pointers and sizes, no torch types,
 * results written in place into caller-owned buffers, stream ordered, and errors returned as status codes
 * (never thrown across the ABI).  The host wrapper (paper_2501_01628_b200/_lib.py) maps the codes onto the
 * reference's exception taxonomy (pkg/src/dprt/errors.py:4-29).
 *
 * Ownership: the caller (Python / torch) owns every image, transfer-function and frame buffer; the library
 * borrows device pointers until the stream work completes.  Opaque handles (DprtBrick) are owned by the
 * library and released by *_destroy, mirroring RefCounted.release (pkg/src/dprt/refcount.py:39-48).
 * Threading: every call binds `device` itself; calls on different devices may run concurrently from
 * different host threads (one thread per rank, as run_collective does, transport.py:545-548).
 */
#ifndef DPRT_CUDA_H
#define DPRT_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPRT_ABI_VERSION 11

/* status codes -> Python exceptions (errors.py:4-29) */
#define DPRT_OK 0
#define DPRT_E_USAGE -1     /* UsageError: bad argument, dead handle */
#define DPRT_E_CUDA -2      /* TransportError subclass DeviceError: CUDA runtime failure */
#define DPRT_E_NOMEM -3     /* DeviceError: allocation failed */
#define DPRT_E_TRANSPORT -4 /* TransportError: peer memory (IPC) failure */

#define DPRT_MAX_BLOBS 64
#define DPRT_MAX_PARTS 64

/* Brick descriptor: a vertex-centred f32 field of dims[0] x dims[1] x dims[2] voxels (x fastest);
 * voxel (i, j, k) sits at origin + (i, j, k) * spacing.  The brick OWNS cells [lo, hi) (0 <= lo < hi <=
 * dims - 1) and stores voxels [max(lo - ghost, 0), min(hi + ghost, dims - 1)].
 * Replaces the per-rank triangle set a Partition hands each rank (pkg/src/dprt/scene.py:52-58). */
typedef struct DprtBrickDesc {
    int64_t dims[3];
    int64_t lo[3];
    int64_t hi[3];
    int32_t ghost;
    int32_t flags; /* DPRT_BRICK_* (0 = defaults) */
    double origin[3];
    double spacing[3];
} DprtBrickDesc;

#define DPRT_BRICK_HALF_QUADS 1 /* opt-in: the coefficient quads in fp16 (8 B per voxel instead of 16) -- half
                                    the quad bytes for memory-bound bricks at a stated precision cost
                                    (DESIGN.md §5); beam marcher only.  The stated bound assumes field values
                                    in [0, 1] (the rounding error scales with |value|); upload / generate fail
                                    with DPRT_E_USAGE if any voxel lies outside [-8, 8] */

/* Pinhole camera, host-evaluated exactly as CameraSpec.basis() (geom.py:163-168) and
 * camera_primary_ray's half extents (geom.py:250-251). */
typedef struct DprtCamera {
    double pos[3];
    double fwd[3];
    double right[3];
    double up[3];
    double half_w;
    double half_h;
} DprtCamera;

/* Synthetic field: kind 0 = blob mixture, `blobs` = host array of n_blobs x {cx, cy, cz, inv_rho2, amp}
 * in unit-cube coordinates (parameters drawn as scene.py:258-262).
 * kind 1 = Marschner-Lobb over [-1, 1]^3, `blobs` = host array {f_M, alpha}, n_blobs = 1 (§2.2b).
 * Both are evaluated in f64 with explicitly rounded ops, bit-identical to oracle/dvr_oracle.c. */
typedef struct DprtFieldSpec {
    int32_t kind;
    int32_t n_blobs;
    const double* blobs;
} DprtFieldSpec;

/* March parameters.  tf_rgba: DEVICE pointer to n_tf x {r, g, b, a} f32.
 * tf_version: caller-maintained tag of the table contents; the brick caches its TF-dependent skip
 * distances per tag and rebuilds them when it changes (0 = rebuild every call). */
typedef struct DprtMarchParams {
    const float* tf_rgba;
    int32_t n_tf;
    int32_t flags; /* DPRT_MARCH_* */
    double vmin;
    double vmax;
    double dt;
    double ert;
    uint64_t tf_version;
    int32_t row0, row1; /* row1 > row0: march only pixel rows [row0, row1); partial_rgba and samples then
                           hold just those rows (pixel (x, y) at index (y - row0) * W + x).  0, 0: all rows */
    int32_t counter_slot; /* 0..DPRT_MARCH_COUNTER_SLOTS-1: the brick's tile-queue counter this launch uses.
                             Marches of one brick that may run concurrently (frames in flight on different
                             streams) must use different slots; 0 for stream-ordered use */
    int32_t reserved;
} DprtMarchParams;

#define DPRT_MARCH_COUNTER_SLOTS 4

#define DPRT_MARCH_NO_SKIP 1      /* disable exact empty-space skipping (macrocell skip distances) */
#define DPRT_MARCH_FULL_FRAME 2   /* march every pixel instead of the brick's screen footprint */
#define DPRT_MARCH_BEAM 4         /* force the warp-beam marcher (8x4 pixel beams, slab-wise skipping) */
#define DPRT_MARCH_QUEUE 8        /* force the ray-queue marcher (persistent warps, per-lane refill) */
#define DPRT_MARCH_BAND_CLEAR 16  /* beam marcher: clear only the footprint's row band of the partial; rows
                                     outside it are left as they were (for band-clipped compositing) */
#define DPRT_MARCH_ACCUM 32       /* ray cycling: partial_rgba holds each ray's accumulated front-to-back
                                     state; the march continues from it (ERT on the accumulated alpha, rays
                                     already at ERT are skipped) and writes it back; nothing is cleared */
#define DPRT_MARCH_HALF 64        /* beam marcher: partial_rgba is fp16 RGBA (8 B per pixel) -- half-size
                                     fragments for the exchange; not with DPRT_MARCH_ACCUM */
#define DPRT_MARCH_WIDE 128       /* beam marcher: the wide-brick addressing (unsigned 32-bit quad offsets from the
                                     apron grid's start) even for a brick of < 2^31 quads -- bricks of 2^31 to
                                     2^32 - 1 quads always use it; for testing that path */
#define DPRT_MARCH_DEEP 256       /* beam marcher: the large-brick configuration (6-sample batches, 2 CTAs/SM)
                                     even for a brick of < 2^28 stored voxels; for testing / tuning */

#define DPRT_COMPOSITE_TONEMAP 1  /* write rgb8 = tone_map(C + (1 - A) * bg) (engine.py:500-502) */
#define DPRT_COMPOSITE_RGBA 2     /* write the blended premultiplied RGBA (no background) */
#define DPRT_COMPOSITE_HALF_IN 4  /* fragments are fp16 RGBA (8 B per pixel, 8-byte aligned) */

typedef struct DprtBrick DprtBrick;

int dprt_cuda_version(void);
const char* dprt_last_error(void); /* thread-local message of the last failing call on this thread */
int dprt_device_count(int* n);

/* Brick lifecycle.  Replaces World._on_commit's accel build (pkg/src/dprt/api.py:146-171) and
 * build_bvh (bvh.py:105-157): the brick's device storage is the per-rank acceleration state (f32 voxels,
 * 16-byte coefficient quads over a one-voxel apron, macrocell min/max).  A brick holds < 2^32 apron quads
 * ((stored dims + 2) per axis, multiplied); DPRT_E_USAGE beyond that. */
int dprt_brick_create(int device, const DprtBrickDesc* desc, DprtBrick** out);
int dprt_brick_stored(const DprtBrick* b, int64_t stored_lo[3], int64_t stored_dims[3]);
/* The brick's macrocell edge (empty-space skipping granularity) as log2 cells: 2 (4^3) for bricks of < 2^28
 * stored voxels, 3 (8^3) for larger ones. */
int dprt_brick_macro_shift(const DprtBrick* b, int32_t* shift);
int dprt_brick_upload(DprtBrick* b, const float* src, int src_is_device, void* stream);
int dprt_brick_download(const DprtBrick* b, float* dst, int dst_is_device, void* stream);
int dprt_brick_generate(DprtBrick* b, const DprtFieldSpec* spec, void* stream);
/* Rebuild the macrocell min/max grid used for exact empty-space skipping (called by upload/generate). */
int dprt_brick_build_macrocells(DprtBrick* b, void* stream);
int dprt_brick_destroy(DprtBrick* b);

/* Screen footprint [x0, y0, x1, y1) of the owned box under `cam` (whole frame if the eye is too close). */
int dprt_brick_footprint(const DprtBrick* b, const DprtCamera* cam, int W, int H, int32_t rect[4]);
/* The same rectangle from a descriptor alone (host-only, no device): every rank computes every brick's
 * footprint locally, so the compositor can clip the exchange without communicating rectangles. */
int dprt_desc_footprint(const DprtBrickDesc* desc, const DprtCamera* cam, int W, int H, int32_t rect[4]);

/* Per-rank local work: replaces trace_local_round -> trace_nearest_batch (engine.py:254-279,
 * bvh.py:284-296).  Writes the full-frame premultiplied RGBA partial (W*H*4 f32, zero outside the
 * footprint) and, if `samples` is non-NULL, the owned lattice sample count per pixel (W*H u32). */
int dprt_march(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, float* partial_rgba,
               uint32_t* samples, int W, int H, void* stream);

/* Roofline instrumentation (diagnostic, synchronous): the same beam march as dprt_march -- ray setup, exact
 * skipping, slab and batch decisions -- with no image output, counting what it must read and shade:
 * out[0] = f32 voxels (cells) of the macrocells in which at least one real sample of a live ray is shaded
 * (x 4 B = the brick bytes a perfect marcher reads once; DESIGN.md §7 "needed bytes"), out[1] = shaded
 * samples, out[2] = contributing samples (weight > 0), out[3] = those macrocells.  Blocks until done. */
int dprt_march_stats(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, int W, int H, uint64_t out[4],
                     void* stream);

/* Single-rank frame (R == 1): the same march with the compositor's over-background and tone map fused
 * into the ray's last step -- writes the (W*H*3) RGB8 frame directly, no RGBA partial, no composite pass.
 * Equivalent to dprt_march + dprt_composite(P = 1, DPRT_COMPOSITE_TONEMAP). */
int dprt_march_rgb8(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, const float bg[3],
                    uint8_t* rgb8, uint32_t* samples, int W, int H, void* stream);

/* Sort-last 'over' of P contiguous fragments of npix pixels each, already in front-to-back order
 * (DESIGN.md §2.8).  Replaces the reference's order-independent (t, gid) min (bvh.py:246-248) plus
 * the final tone map (engine.py:500-502) for the pixels a rank owns (engine.py:216-221).  `inputs`
 * is a HOST array of P device pointers -- local buffers, received fragments or mapped peer pointers
 * (NVLink P2P), so the same kernel is the single-GPU, NCCL and fused-P2P compositor.  rgb8 (npix*3) and
 * rgba_out (npix*4) may also be peer pointers (fused gather into rank 0's frame). */
int dprt_composite(int device, const float* const* inputs, int P, int64_t npix, const float bg[3], int flags,
                   uint8_t* rgb8, float* rgba_out, void* stream);

/* The same with per-fragment pixel ranges (HOST array of P {lo, hi} pairs within [0, npix)): fragment i
 * covers tile pixels [lo_i, hi_i) only -- inputs[i] points at its element for pixel lo_i -- and is clear
 * elsewhere (never read).  Lets the exchange move only the rows of each rank's screen footprint
 * (DESIGN.md §6); ranges = NULL means every fragment covers the whole tile. */
int dprt_composite_ranged(int device, const float* const* inputs, const int64_t* ranges, int P, int64_t npix,
                          const float bg[3], int flags, uint8_t* rgb8, float* rgba_out, void* stream);

/* Fused march + exchange ("p2p_push"): the march of one rank writes each row block b of its
 * RGBA partial (assign_pixels rows [row_start[b], row_start[b+1]), engine.py:216-221) straight into block
 * b's owner -- a peer pointer over NVLink -- as its tiles finish, so the fragment exchange overlaps the
 * march tile by tile (the reference's cycle_batch / ring_exchange step, engine.py:282-310,
 * transport.py:457-462, and the pull of the fused P2P compositor both disappear).  When the launch's last
 * CTA retires, every CTA having fenced its stores at system scope, it release-stores `epoch` into flags[b]
 * for every b (the slot for THIS rank in block b's owner's flag array).  The owner blends once all P flags
 * of its block reach the frame's epoch (dprt_wait_flags, then dprt_composite_ranged on local memory).
 * All arrays are HOST arrays of P entries; pointers are device pointers (local or peer-mapped). */
#define DPRT_MAX_PUSH 16
#define DPRT_SIGNAL_COUNTER_WORDS 1056 /* 33 counters 128 bytes apart (a top counter + 32 sub-counters) */
typedef struct DprtPushTargets {
    int32_t P;                 /* row blocks (ranks), 2..DPRT_MAX_PUSH */
    int32_t reserved;
    const int32_t* row_start;  /* P + 1 row boundaries, row_start[0] = 0, row_start[P] = H */
    void* const* dst;          /* dst[b]: this rank's fragment of block b at its owner; pixel (x, y) of the
                                  block at element (y - row_start[b]) * W + x (16 B f32 / 8 B fp16 RGBA) */
    uint32_t* const* flags;    /* flags[b]: this rank's epoch word at block b's owner */
    uint32_t* counter;         /* DPRT_SIGNAL_COUNTER_WORDS device words, zero before the first launch
                                  (self-resetting CTA counts); one set per concurrently running launch */
    uint32_t epoch;            /* frame tag written to every flags[b]; nonzero, increasing per frame */
    uint32_t reserved2;
} DprtPushTargets;

/* dprt_march into peers' inboxes (DprtPushTargets).  Row windows and accumulation are not available here;
 * DPRT_MARCH_HALF selects fp16 fragments, DPRT_MARCH_BAND_CLEAR clears only the footprint's row band. */
int dprt_march_push(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, const DprtPushTargets* t,
                    uint32_t* samples, int W, int H, void* stream);

/* Stream-ordered wait: work issued on `stream` after this call runs once every flags[i] (i < n, device words,
 * e.g. written by peers' dprt_march_push or dprt_signal_flags) has reached `epoch` (wrap-safe compare).  One
 * 32-thread CTA spins with acquire loads at system scope.  Only for flags written by work that does not
 * itself wait on this stream -- other GPUs, or work already complete. */
int dprt_wait_flags(int device, const uint32_t* flags, int n, uint32_t epoch, void* stream);

/* dprt_composite_ranged that also signals: when its last CTA retires (every CTA having fenced its stores
 * -- e.g. RGB8 rows written into rank 0's frame over NVLink -- at system scope) it release-stores `epoch`
 * into flags[i] (i < n_flags; HOST array of device pointers, local or peer).  counter: DPRT_SIGNAL_COUNTER_WORDS
 * device words, zero before the first launch (self-resetting). */
int dprt_composite_signal(int device, const float* const* inputs, const int64_t* ranges, int P, int64_t npix,
                          const float bg[3], int flags, uint8_t* rgb8, float* rgba_out, uint32_t* counter,
                          uint32_t* const* signal, int n_signal, uint32_t epoch, void* stream);

/* Peer memory over NVLink for the fused direct-send compositor (one process per GPU).  Buffers that peers
 * map must come from dprt_device_alloc so the IPC handle covers exactly [ptr, ptr + bytes). */
int dprt_device_alloc(int device, uint64_t bytes, void** out_ptr);
int dprt_device_free(int device, void* ptr);
int dprt_ipc_handle(int device, const void* dev_ptr, uint8_t handle[64]);
int dprt_ipc_open(int device, const uint8_t handle[64], void** out_ptr);
int dprt_ipc_close(int device, void* ptr);
int dprt_enable_peer(int device, int peer);

/* Known-answer entry points: the marcher's own device functions (slab interval, primary ray) applied to
 * caller-supplied inputs, HOST arrays in and out.  Used to check the reference's golden vectors
 * (geom.py:171-200, geom.py:240-259 via engine.gen_primary_batch) on the GPU code itself. */
int dprt_kat_slab(int device, int n, const double* o, const double* d, const double* lo, const double* hi,
                  double* t01, int32_t* hit);
int dprt_kat_primary_dirs(int device, const DprtCamera* cam, int W, int H, double* out);

/* Instrumented builds (-DDPRT_COUNTERS=1) count {shaded samples, contributing samples, skip steps, rays}
 * in march_kernel; other builds report zeros. */
int dprt_march_counters(int device, uint64_t out[4], int reset);

/* Triangle BVH traversal (the triangle half): replaces the reference's numba compute slot
 * trace_nearest_batch / trace_any_batch (pkg/src/dprt/bvh.py:284-311) as called by engine.trace_local_round
 * (engine.py:254-279), over the same flat Accel arrays (bvh.py:46-60), all DEVICE pointers.  Traversal
 * stack depth 64 like the reference (bvh.py:23): the caller guarantees a tree depth below 63
 * (paper_2501_01628_b200/trace.py checks it when it uploads a BVH).  Results are bit-identical to the
 * reference: float64 throughout, explicitly rounded in its evaluation order. */
typedef struct DprtBvh {
    const double* node_lo;      /* (num_nodes, 3) */
    const double* node_hi;      /* (num_nodes, 3) */
    const int64_t* node_left;   /* (num_nodes,), -1 for leaves */
    const int64_t* node_right;  /* (num_nodes,), -1 for leaves */
    const int64_t* node_first;  /* (num_nodes,) leaf range start */
    const int64_t* node_count;  /* (num_nodes,) 0 for inner nodes */
    int64_t num_nodes;
    int64_t root;               /* -1: empty */
    const double* tri_v;        /* (num_prims, 9) v0 v1 v2, leaf order */
    const int64_t* tri_id;      /* (num_prims,) global ids */
    int64_t num_prims;
} DprtBvh;

/* In place: (best_t[i], best_id[i]) = min over hits with tmin <= t <= tmax of (t, global id), starting from
 * the values passed in (the reference's cross-rank (t, gid) reduction, bvh.py:246-248).  org / dirn (n, 3). */
int dprt_trace_nearest(int device, const DprtBvh* bvh, int64_t n, const double* org, const double* dirn,
                       const double* tmin, const double* tmax, double* best_t, int64_t* best_id, void* stream);
/* In place: occluded[i] |= any hit strictly inside (tmin, tmax); rays already occluded are skipped. */
int dprt_trace_any(int device, const DprtBvh* bvh, int64_t n, const double* org, const double* dirn,
                   const double* tmin, const double* tmax, uint8_t* occluded, void* stream);

/* Per-frame inputs (TF table, small parameter blocks) from PINNED host memory into device memory, copied
 * by the SMs through the mapped host pointer (one tiny kernel on `stream`), not by a copy engine: a
 * 4 KiB TF upload then never queues behind the previous frame's multi-MB read-back on the shared DMA
 * engine (measured: +40 us per frame with cudaMemcpyAsync).  src must be page-locked
 * (cudaHostAlloc / torch pin_memory); bytes <= 1 MiB. */
int dprt_stage_input(int device, void* dst_dev, const void* src_pinned, uint64_t bytes, void* stream);

/* Stream-ordered helpers for the host driver (no torch types): device sync; a pitched 2-D copy between
 * device and (pinned) host memory -- `rows` rows of `width_bytes`, row pitches in bytes -- used to read back
 * only the footprint rectangle of a frame whose outside pixels the host buffer already holds. */
int dprt_device_synchronize(int device);
int dprt_copy_2d(int device, void* dst, uint64_t dst_pitch, const void* src, uint64_t src_pitch, uint64_t width_bytes,
                 uint64_t rows, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DPRT_CUDA_H */

// extern "C" entry points of libdprt_cuda.so (declared in include/dprt_cuda.h).
//
// Host-side glue only: argument validation, device binding, allocation, kernel-argument packing.  No
// exception crosses the ABI; failures return a negative status and leave a thread-local message that
// the Python wrapper maps onto the reference's error taxonomy (pkg/src/dprt/errors.py:4-29).

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace dprt {
cudaError_t launch_march(const MarchArgs& a, cudaStream_t stream);
struct BvhArgs;
cudaError_t launch_trace(const BvhArgs& b, long long n, const double* org, const double* dirn, const double* tmin,
                         const double* tmax, double* best_t, int64_t* best_id, uint8_t* occluded, cudaStream_t stream);
cudaError_t launch_march_mark(const MarchArgs& a, cudaStream_t stream);
cudaError_t launch_mark_reduce(const uint8_t* mark, const int mcd[3], const int cells[3], int mshift, unsigned long long* out,
                               cudaStream_t stream);
cudaError_t launch_skip_build(const DeviceBrick& b, const MarchArgs& a, uint8_t* tmp, cudaStream_t stream);
cudaError_t launch_generate(const DeviceBrick& b, const DprtFieldSpec& spec, cudaStream_t stream);
cudaError_t launch_macrocells(const DeviceBrick& b, cudaStream_t stream);
cudaError_t launch_composite(const CompositeArgs& a, cudaStream_t stream);
cudaError_t launch_wait_flags(const unsigned* flags, int n, unsigned epoch, cudaStream_t stream);
cudaError_t read_counters(unsigned long long out[4], int reset);
cudaError_t launch_kat_slab(const double* o, const double* d, const double* lo, const double* hi, int n, double* t01,
                            int* hit);
cudaError_t launch_kat_primary(const MarchArgs& a, double* out);
}  // namespace dprt

struct DprtBrick : dprt::DeviceBrick {};

namespace {

thread_local std::string g_err;

// dprt_composite_signal's completion signal, handed to dprt_composite_ranged on the calling thread
struct PendingSignal {
    int n = 0;
    uint32_t epoch = 0;
    uint32_t* counter = nullptr;
    uint32_t* flags[DPRT_MAX_PUSH] = {};
};
thread_local PendingSignal g_sig;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    int code = (e == cudaErrorMemoryAllocation) ? DPRT_E_NOMEM : DPRT_E_CUDA;
    return fail(code, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(call, what)                                  \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

// Device binding on every call (a rank thread may have touched another device): the device count is
// queried once per process, and cudaSetDevice is skipped when the thread is already on `device`.
int bind(int device) {
    static std::once_flag once;
    static int n_dev = 0;
    static cudaError_t count_err = cudaSuccess;
    std::call_once(once, [] { count_err = cudaGetDeviceCount(&n_dev); });
    if (count_err != cudaSuccess) return cuda_fail(count_err, "cudaGetDeviceCount");
    if (device < 0 || device >= n_dev) return fail(DPRT_E_USAGE, "device %d outside [0, %d)", device, n_dev);
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur == device) return DPRT_OK;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    return DPRT_OK;
}

}  // namespace

extern "C" {

int dprt_cuda_version(void) { return DPRT_ABI_VERSION; }

const char* dprt_last_error(void) { return g_err.c_str(); }

int dprt_device_count(int* n) {
    if (!n) return fail(DPRT_E_USAGE, "null output");
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return DPRT_OK;
}

int dprt_device_synchronize(int device) {
    int rc = bind(device);
    if (rc) return rc;
    CK(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    return DPRT_OK;
}

int dprt_brick_create(int device, const DprtBrickDesc* desc, DprtBrick** out) {
    if (!desc || !out) return fail(DPRT_E_USAGE, "null brick descriptor or output");
    *out = nullptr;
    for (int a = 0; a < 3; ++a) {
        if (desc->dims[a] < 2) return fail(DPRT_E_USAGE, "dims[%d] = %lld: need >= 2 voxels", a, (long long)desc->dims[a]);
        if (!(0 <= desc->lo[a] && desc->lo[a] < desc->hi[a] && desc->hi[a] <= desc->dims[a] - 1))
            return fail(DPRT_E_USAGE, "owned cells [%lld, %lld) invalid on axis %d for %lld voxels",
                        (long long)desc->lo[a], (long long)desc->hi[a], a, (long long)desc->dims[a]);
        if (!(desc->spacing[a] > 0.0) || !isfinite(desc->spacing[a]) || !isfinite(desc->origin[a]))
            return fail(DPRT_E_USAGE, "spacing/origin on axis %d must be finite, spacing > 0", a);
    }
    if (desc->ghost < 0) return fail(DPRT_E_USAGE, "ghost must be >= 0");
    if (desc->flags & ~DPRT_BRICK_HALF_QUADS) return fail(DPRT_E_USAGE, "unknown brick flags 0x%x", desc->flags);
    {
        long long nv = 1, nq = 1;
        for (int a = 0; a < 3; ++a) {
            long long lo = desc->lo[a] - desc->ghost < 0 ? 0 : desc->lo[a] - desc->ghost;
            long long hi = desc->hi[a] + desc->ghost > desc->dims[a] - 1 ? desc->dims[a] - 1 : desc->hi[a] + desc->ghost;
            nv *= hi - lo + 1;
            nq *= hi - lo + 3;
        }
        // the beam marcher addresses quads with signed 32-bit offsets, or unsigned ones from the apron
        // grid's start once a brick holds >= 2^31 of them (march_beam_kernel<true>); the queue marcher
        // takes < 2^31 only
        if (nq >= (1LL << 32))
            return fail(DPRT_E_USAGE, "brick stores %lld voxels (%lld with the quad apron); the limit is 2^32 - 1",
                        nv, nq);
    }
    int rc = bind(device);
    if (rc) return rc;
    DprtBrick* b = new DprtBrick();
    b->device = device;
    b->desc = *desc;
    long long nvox = 1, nmc = 1, nq = 1;
    for (int a = 0; a < 3; ++a) {
        long long lo = desc->lo[a] - desc->ghost;
        long long hi = desc->hi[a] + desc->ghost;
        if (lo < 0) lo = 0;
        if (hi > desc->dims[a] - 1) hi = desc->dims[a] - 1;
        b->s_lo[a] = lo;
        b->sd[a] = hi - lo + 1;
        b->mcd[a] = 0;  // below, once the macrocell size is chosen
        b->qd[a] = b->sd[a] + 2;
        nvox *= b->sd[a];
        nq *= b->qd[a];
        nmc *= b->mcd[a];
    }
    b->mshift = (nvox >= (1LL << 28) || !DPRT_BEAM_PROBE) ? dprt::kMacroShift : DPRT_MACRO_SHIFT_SMALL;
    nmc = 1;
    for (int a = 0; a < 3; ++a) {
        const long long m = 1LL << b->mshift;
        b->mcd[a] = (b->sd[a] - 1 + m - 1) / m;
        nmc *= b->mcd[a];
    }
    b->vox = nullptr;
    b->macro = nullptr;
    b->sub = nullptr;
    b->subm = nullptr;
    b->skipd = nullptr;
    b->skip_tmp = nullptr;
    b->skip_version = 0;
    b->rays = nullptr;
    b->ray_cap = 0;
    b->counters = nullptr;
    b->quad = nullptr;
    b->half_quads = (desc->flags & DPRT_BRICK_HALF_QUADS) ? 1 : 0;
    cudaError_t e = cudaMalloc(&b->vox, (size_t)nvox * sizeof(float));
    if (e == cudaSuccess)  // 16 B per apron-grid voxel (8 B with fp16 quads)
        e = cudaMalloc(&b->quad, (size_t)nq * (b->half_quads ? sizeof(uint2) : dprt::kQuadSlot * sizeof(float4)));
    if (e == cudaSuccess) e = cudaMalloc(&b->counters, (2 * DPRT_MARCH_COUNTER_SLOTS + 1) * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&b->macro, (size_t)nmc * sizeof(float2));
    if (DPRT_SUBBLOCK && e == cudaSuccess) e = cudaMalloc(&b->sub, (size_t)nmc * 8 * sizeof(float2));
    if (DPRT_SUBBLOCK && e == cudaSuccess) e = cudaMalloc(&b->subm, (size_t)nmc);
    if (e == cudaSuccess) e = cudaMalloc(&b->skipd, (size_t)nmc * dprt::kSkipGrids);
    if (e == cudaSuccess) e = cudaMalloc(&b->skip_tmp, (size_t)nmc * 2 * dprt::kSkipGrids);
    if (e != cudaSuccess) {
        cudaFree(b->vox);
        cudaFree(b->macro);
        cudaFree(b->sub);
        cudaFree(b->subm);
        cudaFree(b->skipd);
        cudaFree(b->skip_tmp);
        cudaFree(b->counters);
        cudaFree(b->quad);
        delete b;
        return cuda_fail(e, "brick allocation");
    }
    *out = b;
    return DPRT_OK;
}

int dprt_brick_macro_shift(const DprtBrick* b, int32_t* shift) {
    if (!b || !shift) return fail(DPRT_E_USAGE, "null brick or output");
    *shift = b->mshift;
    return DPRT_OK;
}

int dprt_brick_stored(const DprtBrick* b, int64_t stored_lo[3], int64_t stored_dims[3]) {
    if (!b) return fail(DPRT_E_USAGE, "null brick");
    for (int a = 0; a < 3; ++a) {
        if (stored_lo) stored_lo[a] = b->s_lo[a];
        if (stored_dims) stored_dims[a] = b->sd[a];
    }
    return DPRT_OK;
}

static size_t brick_bytes(const DprtBrick* b) { return (size_t)b->sd[0] * b->sd[1] * b->sd[2] * sizeof(float); }

int dprt_brick_build_macrocells(DprtBrick* b, void* stream) {
    if (!b) return fail(DPRT_E_USAGE, "null brick");
    int rc = bind(b->device);
    if (rc) return rc;
    int* flag = b->counters + 2 * DPRT_MARCH_COUNTER_SLOTS;
    if (b->half_quads) CK(cudaMemsetAsync(flag, 0, sizeof(int), (cudaStream_t)stream), "range flag reset");
    CK(dprt::launch_macrocells(*b, (cudaStream_t)stream), "macrocell kernel launch");
    b->skip_version = 0;  // TF-dependent skip distances must be rebuilt from the new min/max grid
    if (b->half_quads) {  // commit-time check of the fp16 quads' value range (one 4-byte read-back)
        int h = 0;
        CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream), "range flag read");
        CK(cudaStreamSynchronize((cudaStream_t)stream), "range flag sync");
        if (h) return fail(DPRT_E_USAGE, "fp16 quads need field values within [-%g, %g] (the stated bound is for [0, 1]); "
                           "use f32 quads for this field", (double)dprt::kHalfQuadRange, (double)dprt::kHalfQuadRange);
    }
    return DPRT_OK;
}

int dprt_brick_upload(DprtBrick* b, const float* src, int src_is_device, void* stream) {
    if (!b || !src) return fail(DPRT_E_USAGE, "null brick or source");
    int rc = bind(b->device);
    if (rc) return rc;
    CK(cudaMemcpyAsync(b->vox, src, brick_bytes(b), src_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       (cudaStream_t)stream),
       "brick upload");
    return dprt_brick_build_macrocells(b, stream);
}

int dprt_brick_download(const DprtBrick* b, float* dst, int dst_is_device, void* stream) {
    if (!b || !dst) return fail(DPRT_E_USAGE, "null brick or destination");
    int rc = bind(b->device);
    if (rc) return rc;
    CK(cudaMemcpyAsync(dst, b->vox, brick_bytes(b), dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       (cudaStream_t)stream),
       "brick download");
    if (!dst_is_device) CK(cudaStreamSynchronize((cudaStream_t)stream), "brick download sync");
    return DPRT_OK;
}

int dprt_brick_generate(DprtBrick* b, const DprtFieldSpec* spec, void* stream) {
    if (!b || !spec) return fail(DPRT_E_USAGE, "null brick or field spec");
    if (spec->kind != 0 && spec->kind != 1) return fail(DPRT_E_USAGE, "unknown field kind %d", spec->kind);
    if (spec->kind == 1) {
        if (!spec->blobs || !(spec->blobs[0] > 0.0) || !(spec->blobs[1] >= 0.0))
            return fail(DPRT_E_USAGE, "Marschner-Lobb field needs {f_M > 0, alpha >= 0}");
    } else if (spec->n_blobs < 0 || spec->n_blobs > DPRT_MAX_BLOBS || (spec->n_blobs > 0 && !spec->blobs)) {
        return fail(DPRT_E_USAGE, "n_blobs %d outside [0, %d]", spec->n_blobs, DPRT_MAX_BLOBS);
    }
    int rc = bind(b->device);
    if (rc) return rc;
    CK(dprt::launch_generate(*b, *spec, (cudaStream_t)stream), "generate kernel launch");
    return dprt_brick_build_macrocells(b, stream);
}

int dprt_brick_destroy(DprtBrick* b) {
    if (!b) return DPRT_OK;
    int rc = bind(b->device);
    if (rc) return rc;
    cudaFree(b->vox);
    cudaFree(b->macro);
    cudaFree(b->sub);
    cudaFree(b->subm);
    cudaFree(b->skipd);
    cudaFree(b->skip_tmp);
    cudaFree(b->rays);
    cudaFree(b->counters);
    cudaFree(b->quad);
    delete b;
    return DPRT_OK;
}

static void owned_box_desc(const DprtBrickDesc* d, double lo[3], double hi[3]) {
    for (int a = 0; a < 3; ++a) {
        lo[a] = d->origin[a] + (double)d->lo[a] * d->spacing[a];
        hi[a] = d->origin[a] + (double)d->hi[a] * d->spacing[a];
    }
}

static void owned_box(const DprtBrick* b, double lo[3], double hi[3]) { owned_box_desc(&b->desc, lo, hi); }

static int box_footprint(const double lo[3], const double hi[3], const DprtCamera* cam, int W, int H, int32_t rect[4]);

int dprt_brick_footprint(const DprtBrick* b, const DprtCamera* cam, int W, int H, int32_t rect[4]) {
    if (!b || !cam || !rect || W <= 0 || H <= 0) return fail(DPRT_E_USAGE, "bad footprint arguments");
    double lo[3], hi[3];
    owned_box(b, lo, hi);
    return box_footprint(lo, hi, cam, W, H, rect);
}

int dprt_desc_footprint(const DprtBrickDesc* desc, const DprtCamera* cam, int W, int H, int32_t rect[4]) {
    if (!desc || !cam || !rect || W <= 0 || H <= 0) return fail(DPRT_E_USAGE, "bad footprint arguments");
    double lo[3], hi[3];
    owned_box_desc(desc, lo, hi);
    return box_footprint(lo, hi, cam, W, H, rect);
}

static int box_footprint(const double lo[3], const double hi[3], const DprtCamera* cam, int W, int H, int32_t rect[4]) {
    double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    bool full = false;
    for (int c = 0; c < 8 && !full; ++c) {
        double p[3] = {(c & 1) ? hi[0] : lo[0], (c & 2) ? hi[1] : lo[1], (c & 4) ? hi[2] : lo[2]};
        double v[3] = {p[0] - cam->pos[0], p[1] - cam->pos[1], p[2] - cam->pos[2]};
        double z = v[0] * cam->fwd[0] + v[1] * cam->fwd[1] + v[2] * cam->fwd[2];
        double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        if (!(z > 1e-6 * (len + 1.0))) {
            full = true;
            break;
        }
        double x = (v[0] * cam->right[0] + v[1] * cam->right[1] + v[2] * cam->right[2]) / z;
        double y = (v[0] * cam->up[0] + v[1] * cam->up[1] + v[2] * cam->up[2]) / z;
        // invert geom.py:252-253 for the pixel coordinate of the film point
        double px = (x / cam->half_w + 1.0) * 0.5 * W - 0.5;
        double py = (1.0 - y / cam->half_h) * 0.5 * H - 0.5;
        xmin = fmin(xmin, px);
        xmax = fmax(xmax, px);
        ymin = fmin(ymin, py);
        ymax = fmax(ymax, py);
    }
    if (full) {
        rect[0] = 0;
        rect[1] = 0;
        rect[2] = W;
        rect[3] = H;
        return DPRT_OK;
    }
    // one pixel of slack on every side keeps the rectangle conservative under rounding
    double x0 = floor(xmin) - 1.0, x1 = ceil(xmax) + 2.0, y0 = floor(ymin) - 1.0, y1 = ceil(ymax) + 2.0;
    rect[0] = (int32_t)fmax(0.0, fmin((double)W, x0));
    rect[1] = (int32_t)fmax(0.0, fmin((double)H, y0));
    rect[2] = (int32_t)fmax(0.0, fmin((double)W, x1));
    rect[3] = (int32_t)fmax(0.0, fmin((double)H, y1));
    return DPRT_OK;
}

static int march_impl(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, float* partial_rgba,
                      const float* bg, uint8_t* rgb8, uint32_t* samples, int W, int H, void* stream,
                      uint64_t* stats = nullptr, const DprtPushTargets* push = nullptr);

int dprt_march(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, float* partial_rgba,
               uint32_t* samples, int W, int H, void* stream) {
    if (!partial_rgba) return fail(DPRT_E_USAGE, "null partial buffer");
    return march_impl(b, cam, p, partial_rgba, nullptr, nullptr, samples, W, H, stream);
}

int dprt_march_rgb8(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, const float bg[3],
                    uint8_t* rgb8, uint32_t* samples, int W, int H, void* stream) {
    if (!rgb8 || !bg) return fail(DPRT_E_USAGE, "null rgb8 frame or background");
    return march_impl(b, cam, p, nullptr, bg, rgb8, samples, W, H, stream);
}

int dprt_march_stats(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, int W, int H, uint64_t out[4],
                     void* stream) {
    if (!out) return fail(DPRT_E_USAGE, "null stats output");
    return march_impl(b, cam, p, nullptr, nullptr, nullptr, nullptr, W, H, stream, out);
}

int dprt_march_push(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, const DprtPushTargets* t,
                    uint32_t* samples, int W, int H, void* stream) {
    if (!t) return fail(DPRT_E_USAGE, "null push targets");
    if (t->P < 2 || t->P > DPRT_MAX_PUSH) return fail(DPRT_E_USAGE, "push needs 2..%d row blocks (got %d)", DPRT_MAX_PUSH, t->P);
    if (!t->row_start || !t->dst || !t->flags || !t->counter) return fail(DPRT_E_USAGE, "null push target array");
    if (t->epoch == 0) return fail(DPRT_E_USAGE, "push epoch must be nonzero (flags start at 0)");
    if (t->row_start[0] != 0 || t->row_start[t->P] != H)
        return fail(DPRT_E_USAGE, "row blocks must cover rows [0, %d) (got [%d, %d))", H, t->row_start[0], t->row_start[t->P]);
    const int align = (p && (p->flags & DPRT_MARCH_HALF)) ? 8 : 16;
    for (int i = 0; i < t->P; ++i) {
        if (t->row_start[i + 1] < t->row_start[i]) return fail(DPRT_E_USAGE, "row block %d is negative", i);
        if (t->row_start[i + 1] > t->row_start[i] && !t->dst[i]) return fail(DPRT_E_USAGE, "push target %d is null", i);
        if (reinterpret_cast<uintptr_t>(t->dst[i]) % align) return fail(DPRT_E_USAGE, "push target %d not %d-byte aligned", i, align);
        if (!t->flags[i]) return fail(DPRT_E_USAGE, "push flag %d is null", i);
    }
    if (p && (p->flags & DPRT_MARCH_ACCUM)) return fail(DPRT_E_USAGE, "push marches do not accumulate");
    if (p && p->row1 > p->row0) return fail(DPRT_E_USAGE, "push marches cover whole row blocks, not a row window");
    return march_impl(b, cam, p, reinterpret_cast<float*>(t->dst[0]), nullptr, nullptr, samples, W, H, stream, nullptr, t);
}

static int march_impl(const DprtBrick* b, const DprtCamera* cam, const DprtMarchParams* p, float* partial_rgba,
                      const float* bg, uint8_t* rgb8, uint32_t* samples, int W, int H, void* stream,
                      uint64_t* stats, const DprtPushTargets* push) {
    if (!b || !cam || !p) return fail(DPRT_E_USAGE, "null march argument");
    if (W <= 0 || H <= 0) return fail(DPRT_E_USAGE, "frame size %dx%d must be positive", W, H);
    if (p->n_tf < 2 || p->n_tf > dprt::kMaxTf || !p->tf_rgba)
        return fail(DPRT_E_USAGE, "transfer function needs 2..%d entries (got %d)", dprt::kMaxTf, p->n_tf);
    if (!(p->vmax > p->vmin)) return fail(DPRT_E_USAGE, "transfer function range needs vmax > vmin");
    if (!(p->dt > 0.0) || !isfinite(p->dt)) return fail(DPRT_E_USAGE, "dt must be finite and > 0");
    if (!(cam->half_w > 0.0) || !(cam->half_h > 0.0)) return fail(DPRT_E_USAGE, "camera half extents must be > 0");
    {
        // the sample loop indexes a ray's samples in f32 (exact below 2^24) and 32-bit counts: bound the
        // samples any ray can own in this brick by the owned box's diagonal / dt
        double lo[3], hi[3], d2 = 0.0;
        owned_box(b, lo, hi);
        for (int a = 0; a < 3; ++a) d2 += (hi[a] - lo[a]) * (hi[a] - lo[a]);
        if (sqrt(d2) / p->dt + 2.0 >= 16777216.0)
            return fail(DPRT_E_USAGE, "dt %g gives up to %.0f samples per ray in this brick; the limit is 2^24",
                        p->dt, sqrt(d2) / p->dt + 2.0);
    }
    if (p->counter_slot < 0 || p->counter_slot >= DPRT_MARCH_COUNTER_SLOTS)
        return fail(DPRT_E_USAGE, "counter slot %d outside [0, %d)", p->counter_slot, DPRT_MARCH_COUNTER_SLOTS);
    int rc = bind(b->device);
    if (rc) return rc;
    dprt::MarchArgs a;
    memset(&a, 0, sizeof(a));
    for (int i = 0; i < 3; ++i) {
        a.o[i] = cam->pos[i];
        a.f[i] = cam->fwd[i];
        a.r[i] = cam->right[i];
        a.u[i] = cam->up[i];
        a.origin[i] = b->desc.origin[i];
        a.spacing[i] = b->desc.spacing[i];
        a.inv_spacing[i] = (float)(1.0 / b->desc.spacing[i]);
        a.inv_spacing_d[i] = 1.0 / b->desc.spacing[i];
        a.stored_lo_d[i] = (double)b->s_lo[i];
        a.clo[i] = 0;
        a.chi[i] = (int)(b->sd[i] - 2);
        a.sd[i] = (int)b->sd[i];
        a.mcd[i] = (int)b->mcd[i];
    }
    owned_box(b, a.blo, a.bhi);
    a.half_w = cam->half_w;
    a.half_h = cam->half_h;
    {
        double ext = 0.0, dist = 0.0;
        for (int i = 0; i < 3; ++i) {
            ext += (a.bhi[i] - a.blo[i]) * (a.bhi[i] - a.blo[i]);
            const double c = 0.5 * (a.blo[i] + a.bhi[i]) - cam->pos[i];
            dist += c * c;
        }
        const double margin = 1e-3 * (1.0 + sqrt(ext) + sqrt(dist));
        for (int i = 0; i < 3; ++i) {
            a.mt_f[i] = (float)cam->fwd[i];
            a.mt_r[i] = (float)cam->right[i];
            a.mt_u[i] = (float)cam->up[i];
            a.mt_lo[i] = (float)(a.blo[i] - cam->pos[i] - margin);
            a.mt_hi[i] = (float)(a.bhi[i] - cam->pos[i] + margin);
        }
        a.mt_hw = (float)cam->half_w;
        a.mt_hh = (float)cam->half_h;
        a.mt_iw = (float)(1.0 / W);
        a.mt_ih = (float)(1.0 / H);
    }
    a.dt = p->dt;
    {
        int ex;
        a.inv_dt_pow2 = (frexp(p->dt, &ex) == 0.5) ? 1.0 / p->dt : 0.0;  // exact inverse of a power of two
    }
    a.fs_iw2 = 2.0 / W;
    a.fs_ih2 = 2.0 / H;
    for (int i = 0; i < 3; ++i) {
        a.fs_L[i] = a.blo[i] - cam->pos[i];  // == __dsub_rn(lo, o) of the exact path
        a.fs_H[i] = a.bhi[i] - cam->pos[i];
    }
    a.fs_idt = 1.0 / p->dt;
    a.fs_S = 1.0 + fabs(cam->half_w) + fabs(cam->half_h);
    a.fs_ok = a.blo[0] <= a.bhi[0] && a.blo[1] <= a.bhi[1] && a.blo[2] <= a.bhi[2] && isfinite(a.fs_S);
    {  // the fast setup's error bound needs |f + sx r + sy u| >= 1: an orthonormal camera basis
        const double* v[3] = {cam->fwd, cam->right, cam->up};
        for (int i = 0; i < 3; ++i)
            for (int j = i; j < 3; ++j) {
                const double g = v[i][0] * v[j][0] + v[i][1] * v[j][1] + v[i][2] * v[j][2];
                if (!(fabs(g - (i == j ? 1.0 : 0.0)) <= 1e-9)) a.fs_ok = 0;
            }
    }
    a.sy = (long long)b->sd[0];
    a.sz = (long long)b->sd[0] * b->sd[1];
    a.vox = b->vox;
    a.qsx = DPRT_QUAD_YFAST ? (int)b->qd[1] : 1;
    a.qsy = DPRT_QUAD_YFAST ? 1 : (int)b->qd[0];
    a.qsz = (int)(b->qd[0] * b->qd[1]);
    // fp16 quads: reinterpreted as uint2 at the same element offsets; f32 octets: two float4 per slot
    a.qorg = b->quad + (long long)(b->half_quads ? 1 : dprt::kQuadSlot) * (a.qsz + a.qsy + a.qsx);
    a.half_quads = b->half_quads;
    a.wide = ((long long)b->qd[0] * b->qd[1] * b->qd[2] >= (1LL << 31) || (p->flags & DPRT_MARCH_WIDE)) ? 1 : 0;
    // bricks of >= 2^28 stored voxels (4.3 GB of quads; c3's 1026^3 bricks, not c2's 513^3) touch far more
    // quads than L2 holds per frame: run the deeper-batch, fewer-warp configuration
    a.deep = ((long long)b->sd[0] * b->sd[1] * b->sd[2] >= (1LL << 28) || (p->flags & DPRT_MARCH_DEEP)) ? 1 : 0;
    a.skipd = b->skipd;
    a.skip_n = (long long)b->mcd[0] * b->mcd[1] * b->mcd[2];
    a.mshift = b->mshift;
    a.subm = b->subm;
    a.skip = (p->flags & DPRT_MARCH_NO_SKIP) ? 0 : 1;
    a.band_clear = (p->flags & DPRT_MARCH_BAND_CLEAR) ? 1 : 0;
    a.accum = (p->flags & DPRT_MARCH_ACCUM) ? 1 : 0;
    a.half_out = (p->flags & DPRT_MARCH_HALF) ? 1 : 0;
    if (a.half_out && (a.accum || rgb8)) return fail(DPRT_E_USAGE, "fp16 partials exclude accumulation and RGB8 output");
    const bool window = p->row1 > p->row0;
    if (window && (p->row0 < 0 || p->row1 > H)) return fail(DPRT_E_USAGE, "row window [%d, %d) outside [0, %d)", p->row0, p->row1, H);
    if ((a.accum || window) && rgb8) return fail(DPRT_E_USAGE, "row windows and accumulation need an RGBA partial");
    a.pix0 = window ? (long long)p->row0 * W : 0;
    a.npix_buf = window ? (long long)(p->row1 - p->row0) * W : (long long)W * H;
    a.beam = (p->flags & DPRT_MARCH_BEAM) ? 1 : ((p->flags & DPRT_MARCH_QUEUE) ? 0 : DPRT_BEAM_DEFAULT);
    if (rgb8 || a.accum || window || a.half_out || stats || push) a.beam = 1;  // these exist in the beam marcher only
    if (push) {
        a.push_P = push->P;
        for (int i = 0; i <= push->P; ++i) a.push_row[i] = push->row_start[i];
        for (int i = 0; i < push->P; ++i) {
            a.push_dst[i] = static_cast<char*>(push->dst[i]);
            a.push_flag[i] = push->flags[i];
        }
        a.push_ctr = push->counter;
        a.push_epoch = push->epoch;
    }
    if (!a.beam && a.wide) return fail(DPRT_E_USAGE, "the queue marcher takes bricks of < 2^31 quads; use the beam marcher");
    if (!a.beam && a.half_quads) return fail(DPRT_E_USAGE, "fp16 quads need the beam marcher");
    a.tf = reinterpret_cast<const float4*>(p->tf_rgba);
    a.n_tf = p->n_tf;
    a.vmin = (float)p->vmin;
    a.tf_scale = (float)((double)(p->n_tf - 1) / (p->vmax - p->vmin));
    a.tf_ns = (float)(1.0 / (p->vmax - p->vmin));
    a.tf_no = (float)(-p->vmin / (p->vmax - p->vmin));
    a.ert = (float)p->ert;
    a.out = a.half_out ? nullptr : reinterpret_cast<float4*>(partial_rgba);
    a.out16 = a.half_out ? reinterpret_cast<uint2*>(partial_rgba) : nullptr;
    a.rgb8 = rgb8;
    if (bg) {
        a.bg[0] = bg[0];
        a.bg[1] = bg[1];
        a.bg[2] = bg[2];
    }
    a.samples = samples;
    a.W = W;
    a.H = H;
    if (p->flags & DPRT_MARCH_FULL_FRAME) {
        a.rect[0] = 0;
        a.rect[1] = 0;
        a.rect[2] = W;
        a.rect[3] = H;
    } else {
        rc = dprt_brick_footprint(b, cam, W, H, a.rect);
        if (rc) return rc;
    }
    if (window) {  // rays only in rows [row0, row1)
        if (a.rect[1] < p->row0) a.rect[1] = p->row0;
        if (a.rect[3] > p->row1) a.rect[3] = p->row1;
        if (a.rect[3] < a.rect[1]) a.rect[3] = a.rect[1];
    }
    DprtBrick* mb = const_cast<DprtBrick*>(b);  // ray queue + skip-distance cache are mutable scratch
    if (!a.beam && (long long)W * H > mb->ray_cap) {  // the queue marcher needs 32 B per pixel
        CK(cudaStreamSynchronize((cudaStream_t)stream), "ray queue resize sync");
        cudaFree(mb->rays);
        mb->rays = nullptr;
        mb->ray_cap = 0;
        CK(cudaMalloc(&mb->rays, (size_t)W * H * 2 * sizeof(float4)), "ray queue allocation");
        mb->ray_cap = (long long)W * H;
    }
    a.rays = mb->rays;
    a.counters = mb->counters + 2 * p->counter_slot;  // one tile queue per concurrently running frame
    if (a.skip && (p->tf_version == 0 || b->skip_version != p->tf_version)) {
        CK(dprt::launch_skip_build(*mb, a, mb->skip_tmp, (cudaStream_t)stream), "skip-distance build");
        mb->skip_version = p->tf_version;
    }
    if (!stats) {
        CK(dprt::launch_march(a, (cudaStream_t)stream), "march kernel launch");
        return DPRT_OK;
    }
    // dprt_march_stats: instrumented march into a per-macrocell mark grid, reduced to the needed voxels
    const long long nmc = (long long)b->mcd[0] * b->mcd[1] * b->mcd[2];
    uint8_t* mark = nullptr;
    unsigned long long* cnt = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMalloc(&mark, (size_t)nmc), "mark grid");
    cudaError_t e = cudaMalloc(&cnt, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(mark, 0, (size_t)nmc, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), st);
    a.mark = mark;
    a.stats = cnt;
    if (e == cudaSuccess) e = dprt::launch_march_mark(a, st);
    const int mcd[3] = {(int)b->mcd[0], (int)b->mcd[1], (int)b->mcd[2]};
    const int cells[3] = {(int)(b->sd[0] - 1), (int)(b->sd[1] - 1), (int)(b->sd[2] - 1)};
    if (e == cudaSuccess) e = dprt::launch_mark_reduce(mark, mcd, cells, b->mshift, cnt + 2, st);
    unsigned long long h[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(mark);
    cudaFree(cnt);
    if (e != cudaSuccess) return cuda_fail(e, "march stats");
    stats[0] = h[2];  // voxels (cells) of the marked macrocells
    stats[1] = h[0];  // shaded samples (real samples of live rays)
    stats[2] = h[1];  // contributing samples (w > 0)
    stats[3] = h[3];  // marked macrocells
    return DPRT_OK;
}

int dprt_composite_ranged(int device, const float* const* inputs, const int64_t* ranges, int P, int64_t npix,
                          const float bg[3], int flags, uint8_t* rgb8, float* rgba_out, void* stream) {
    if (!inputs || P < 1 || P > DPRT_MAX_PARTS) return fail(DPRT_E_USAGE, "need 1..%d fragments (got %d)", DPRT_MAX_PARTS, P);
    if (npix < 0) return fail(DPRT_E_USAGE, "negative pixel count");
    if ((flags & DPRT_COMPOSITE_TONEMAP) && (!rgb8 || !bg)) return fail(DPRT_E_USAGE, "tone map needs rgb8 and bg");
    if ((flags & DPRT_COMPOSITE_RGBA) && !rgba_out) return fail(DPRT_E_USAGE, "RGBA output requested but null");
    if (!(flags & (DPRT_COMPOSITE_TONEMAP | DPRT_COMPOSITE_RGBA))) return fail(DPRT_E_USAGE, "no composite output selected");
    int rc = bind(device);
    if (rc) return rc;
    dprt::CompositeArgs a;
    memset(&a, 0, sizeof(a));
    for (int i = 0; i < P; ++i) {
        const int64_t lo = ranges ? ranges[2 * i] : 0, hi = ranges ? ranges[2 * i + 1] : npix;
        if (lo < 0 || hi > npix || lo > hi) return fail(DPRT_E_USAGE, "fragment %d range [%lld, %lld) outside [0, %lld)",
                                                        i, (long long)lo, (long long)hi, (long long)npix);
        if (hi > lo && !inputs[i]) return fail(DPRT_E_USAGE, "fragment %d is null", i);
        if (reinterpret_cast<uintptr_t>(inputs[i]) & ((flags & DPRT_COMPOSITE_HALF_IN) ? 7 : 15))
            return fail(DPRT_E_USAGE, "fragment %d not %d-byte aligned", i, (flags & DPRT_COMPOSITE_HALF_IN) ? 8 : 16);
        a.in[i] = reinterpret_cast<const float4*>(inputs[i]);
        a.lo[i] = lo;
        a.hi[i] = hi;
    }
    a.P = P;
    a.npix = npix;
    if (bg) {
        a.bg[0] = bg[0];
        a.bg[1] = bg[1];
        a.bg[2] = bg[2];
    }
    a.flags = flags;
    a.rgb8 = rgb8;
    a.rgba = reinterpret_cast<float4*>(rgba_out);
    a.n_sig = g_sig.n;  // dprt_composite_signal (this thread's pending signal), else 0
    a.sig_epoch = g_sig.epoch;
    a.sig_ctr = g_sig.counter;
    for (int i = 0; i < g_sig.n; ++i) a.sig[i] = g_sig.flags[i];
    CK(dprt::launch_composite(a, (cudaStream_t)stream), "composite kernel launch");
    return DPRT_OK;
}

int dprt_composite(int device, const float* const* inputs, int P, int64_t npix, const float bg[3], int flags,
                   uint8_t* rgb8, float* rgba_out, void* stream) {
    return dprt_composite_ranged(device, inputs, nullptr, P, npix, bg, flags, rgb8, rgba_out, stream);
}

int dprt_composite_signal(int device, const float* const* inputs, const int64_t* ranges, int P, int64_t npix,
                          const float bg[3], int flags, uint8_t* rgb8, float* rgba_out, uint32_t* counter,
                          uint32_t* const* signal, int n_signal, uint32_t epoch, void* stream) {
    if (n_signal < 1 || n_signal > DPRT_MAX_PUSH || !signal || !counter)
        return fail(DPRT_E_USAGE, "need 1..%d signal flags and a counter", DPRT_MAX_PUSH);
    for (int i = 0; i < n_signal; ++i)
        if (!signal[i]) return fail(DPRT_E_USAGE, "signal flag %d is null", i);
    g_sig.n = n_signal;
    g_sig.epoch = epoch;
    g_sig.counter = counter;
    for (int i = 0; i < n_signal; ++i) g_sig.flags[i] = signal[i];
    const int rc = dprt_composite_ranged(device, inputs, ranges, P, npix, bg, flags, rgb8, rgba_out, stream);
    g_sig.n = 0;
    return rc;
}

int dprt_wait_flags(int device, const uint32_t* flags, int n, uint32_t epoch, void* stream) {
    if (n < 1 || !flags) return fail(DPRT_E_USAGE, "need at least one flag to wait on");
    int rc = bind(device);
    if (rc) return rc;
    CK(dprt::launch_wait_flags(flags, n, epoch, (cudaStream_t)stream), "wait-flags kernel launch");
    return DPRT_OK;
}

int dprt_march_counters(int device, uint64_t out[4], int reset) {
    if (!out) return fail(DPRT_E_USAGE, "null output");
    int rc = bind(device);
    if (rc) return rc;
    unsigned long long tmp[4];
    CK(dprt::read_counters(tmp, reset), "march counters");
    for (int i = 0; i < 4; ++i) out[i] = tmp[i];
    return DPRT_OK;
}

int dprt_kat_slab(int device, int n, const double* o, const double* d, const double* lo, const double* hi,
                  double* t01, int32_t* hit) {
    if (n < 0 || (n > 0 && (!o || !d || !lo || !hi || !t01 || !hit))) return fail(DPRT_E_USAGE, "bad KAT arguments");
    if (n == 0) return DPRT_OK;
    int rc = bind(device);
    if (rc) return rc;
    double* buf = nullptr;
    int* h = nullptr;
    const size_t vec = (size_t)n * 3 * sizeof(double);
    CK(cudaMalloc(&buf, 4 * vec + (size_t)n * 2 * sizeof(double)), "KAT buffers");
    cudaError_t e = cudaMalloc(&h, (size_t)n * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(buf, o, vec, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(buf + 3 * n, d, vec, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(buf + 6 * n, lo, vec, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(buf + 9 * n, hi, vec, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = dprt::launch_kat_slab(buf, buf + 3 * n, buf + 6 * n, buf + 9 * n, n, buf + 12 * n, h);
    if (e == cudaSuccess) e = cudaMemcpy(t01, buf + 12 * n, (size_t)n * 2 * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(hit, h, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    cudaFree(h);
    if (e != cudaSuccess) return cuda_fail(e, "slab KAT");
    return DPRT_OK;
}

int dprt_kat_primary_dirs(int device, const DprtCamera* cam, int W, int H, double* out) {
    if (!cam || !out || W <= 0 || H <= 0) return fail(DPRT_E_USAGE, "bad KAT arguments");
    int rc = bind(device);
    if (rc) return rc;
    dprt::MarchArgs a;
    memset(&a, 0, sizeof(a));
    for (int i = 0; i < 3; ++i) {
        a.f[i] = cam->fwd[i];
        a.r[i] = cam->right[i];
        a.u[i] = cam->up[i];
    }
    a.half_w = cam->half_w;
    a.half_h = cam->half_h;
    {
        double ext = 0.0, dist = 0.0;
        for (int i = 0; i < 3; ++i) {
            ext += (a.bhi[i] - a.blo[i]) * (a.bhi[i] - a.blo[i]);
            const double c = 0.5 * (a.blo[i] + a.bhi[i]) - cam->pos[i];
            dist += c * c;
        }
        const double margin = 1e-3 * (1.0 + sqrt(ext) + sqrt(dist));
        for (int i = 0; i < 3; ++i) {
            a.mt_f[i] = (float)cam->fwd[i];
            a.mt_r[i] = (float)cam->right[i];
            a.mt_u[i] = (float)cam->up[i];
            a.mt_lo[i] = (float)(a.blo[i] - cam->pos[i] - margin);
            a.mt_hi[i] = (float)(a.bhi[i] - cam->pos[i] + margin);
        }
        a.mt_hw = (float)cam->half_w;
        a.mt_hh = (float)cam->half_h;
        a.mt_iw = (float)(1.0 / W);
        a.mt_ih = (float)(1.0 / H);
    }
    a.W = W;
    a.H = H;
    double* buf = nullptr;
    const size_t bytes = (size_t)W * H * 3 * sizeof(double);
    CK(cudaMalloc(&buf, bytes), "KAT buffer");
    cudaError_t e = dprt::launch_kat_primary(a, buf);
    if (e == cudaSuccess) e = cudaMemcpy(out, buf, bytes, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e != cudaSuccess) return cuda_fail(e, "primary-ray KAT");
    return DPRT_OK;
}

namespace dprt {
struct BvhArgs {  // layout shared with trace.cu
    const double* lo;
    const double* hi;
    const int64_t* left;
    const int64_t* right;
    const int64_t* first;
    const int64_t* count;
    int64_t root;
    const double* tv;
    const int64_t* tid;
};
}  // namespace dprt

static int trace_impl(int device, const DprtBvh* bvh, int64_t n, const double* org, const double* dirn,
                      const double* tmin, const double* tmax, double* best_t, int64_t* best_id, uint8_t* occluded,
                      void* stream) {
    if (!bvh) return fail(DPRT_E_USAGE, "null BVH");
    if (n < 0) return fail(DPRT_E_USAGE, "negative ray count");
    if (n == 0) return DPRT_OK;
    if (!org || !dirn || !tmin || !tmax || (!occluded && (!best_t || !best_id)))
        return fail(DPRT_E_USAGE, "null ray array");
    if (bvh->root >= bvh->num_nodes || bvh->root < -1) return fail(DPRT_E_USAGE, "BVH root %lld outside [-1, %lld)",
                                                                  (long long)bvh->root, (long long)bvh->num_nodes);
    if (bvh->root >= 0 && (!bvh->node_lo || !bvh->node_hi || !bvh->node_left || !bvh->node_right || !bvh->node_first ||
                           !bvh->node_count || !bvh->tri_v || !bvh->tri_id))
        return fail(DPRT_E_USAGE, "null BVH array");
    if (bvh->num_nodes >= (1LL << 31)) return fail(DPRT_E_USAGE, "BVH has %lld nodes; the limit is 2^31 - 1",
                                                   (long long)bvh->num_nodes);
    int rc = bind(device);
    if (rc) return rc;
    const dprt::BvhArgs b{bvh->node_lo, bvh->node_hi, bvh->node_left, bvh->node_right, bvh->node_first,
                          bvh->node_count, bvh->root, bvh->tri_v, bvh->tri_id};
    CK(dprt::launch_trace(b, (long long)n, org, dirn, tmin, tmax, best_t, best_id, occluded, (cudaStream_t)stream),
       "trace kernel launch");
    return DPRT_OK;
}

int dprt_trace_nearest(int device, const DprtBvh* bvh, int64_t n, const double* org, const double* dirn,
                       const double* tmin, const double* tmax, double* best_t, int64_t* best_id, void* stream) {
    return trace_impl(device, bvh, n, org, dirn, tmin, tmax, best_t, best_id, nullptr, stream);
}

int dprt_trace_any(int device, const DprtBvh* bvh, int64_t n, const double* org, const double* dirn,
                   const double* tmin, const double* tmax, uint8_t* occluded, void* stream) {
    if (!occluded && n > 0) return fail(DPRT_E_USAGE, "null occlusion array");
    return trace_impl(device, bvh, n, org, dirn, tmin, tmax, nullptr, nullptr, occluded, stream);
}

namespace {
// SM-driven copy of a small input block from mapped pinned host memory (16-byte vectors + byte tail).
__global__ void stage_input_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, unsigned long long n) {
    const unsigned long long nv = n / 16;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (unsigned long long)gridDim.x * blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = __ldcv(reinterpret_cast<const uint4*>(src) + i);  // no stale cache lines
    if (blockIdx.x == 0 && threadIdx.x < n % 16) dst[nv * 16 + threadIdx.x] = src[nv * 16 + threadIdx.x];
}
}  // namespace

int dprt_stage_input(int device, void* dst_dev, const void* src_pinned, uint64_t bytes, void* stream) {
    if (!dst_dev || !src_pinned) return fail(DPRT_E_USAGE, "null staging pointer");
    if (bytes == 0) return DPRT_OK;
    if (bytes > (1ull << 20)) return fail(DPRT_E_USAGE, "dprt_stage_input is for small inputs (%llu bytes > 1 MiB)",
                                          (unsigned long long)bytes);
    if (((uintptr_t)dst_dev | (uintptr_t)src_pinned) & 15u) return fail(DPRT_E_USAGE, "staging pointers must be 16-byte aligned");
    int rc = bind(device);
    if (rc) return rc;
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, src_pinned) != cudaSuccess || pa.type != cudaMemoryTypeHost ||
        !pa.devicePointer) {
        cudaGetLastError();
        return fail(DPRT_E_USAGE, "dprt_stage_input source is not page-locked host memory");
    }
    const unsigned long long nv = (bytes + 15) / 16;
    const unsigned blocks = (unsigned)((nv + 255) / 256);
    stage_input_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<uint8_t*>(dst_dev),
                                                                 static_cast<const uint8_t*>(pa.devicePointer), bytes);
    CK(cudaGetLastError(), "stage_input kernel launch");
    return DPRT_OK;
}

int dprt_copy_2d(int device, void* dst, uint64_t dst_pitch, const void* src, uint64_t src_pitch, uint64_t width_bytes,
                 uint64_t rows, void* stream) {
    if (rows == 0 || width_bytes == 0) return DPRT_OK;
    if (!dst || !src) return fail(DPRT_E_USAGE, "null copy pointer");
    if (width_bytes > dst_pitch || width_bytes > src_pitch) return fail(DPRT_E_USAGE, "copy width exceeds a row pitch");
    int rc = bind(device);
    if (rc) return rc;
    CK(cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch, (size_t)width_bytes, (size_t)rows,
                         cudaMemcpyDefault, (cudaStream_t)stream),
       "dprt_copy_2d");
    return DPRT_OK;
}

int dprt_device_alloc(int device, uint64_t bytes, void** out_ptr) {
    if (!out_ptr || bytes == 0) return fail(DPRT_E_USAGE, "bad allocation request");
    *out_ptr = nullptr;
    int rc = bind(device);
    if (rc) return rc;
    CK(cudaMalloc(out_ptr, (size_t)bytes), "dprt_device_alloc");
    return DPRT_OK;
}

int dprt_device_free(int device, void* ptr) {
    if (!ptr) return DPRT_OK;
    int rc = bind(device);
    if (rc) return rc;
    CK(cudaFree(ptr), "dprt_device_free");
    return DPRT_OK;
}

int dprt_ipc_handle(int device, const void* dev_ptr, uint8_t handle[64]) {
    if (!dev_ptr || !handle) return fail(DPRT_E_USAGE, "null IPC argument");
    int rc = bind(device);
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaIpcGetMemHandle");
        return DPRT_E_TRANSPORT;
    }
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(handle, &h, 64);
    return DPRT_OK;
}

int dprt_ipc_open(int device, const uint8_t handle[64], void** out_ptr) {
    if (!handle || !out_ptr) return fail(DPRT_E_USAGE, "null IPC argument");
    int rc = bind(device);
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaIpcOpenMemHandle");
        return DPRT_E_TRANSPORT;
    }
    return DPRT_OK;
}

int dprt_ipc_close(int device, void* ptr) {
    int rc = bind(device);
    if (rc) return rc;
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaIpcCloseMemHandle");
        return DPRT_E_TRANSPORT;
    }
    return DPRT_OK;
}

int dprt_enable_peer(int device, int peer) {
    int rc = bind(device);
    if (rc) return rc;
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, device, peer), "cudaDeviceCanAccessPeer");
    if (!can) return fail(DPRT_E_TRANSPORT, "device %d cannot access peer %d", device, peer);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    cudaGetLastError();
    return DPRT_OK;
}

}  // extern "C"

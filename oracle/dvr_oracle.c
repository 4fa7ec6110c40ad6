/*
 * dvr_oracle.c -- CPU ORACLE (test infrastructure only; never shipped, never measured as the product).
 *
 * A scalar, float64 restatement of the DVR + sort-last path fixed in DESIGN.md §2.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this.
 *
 * The reference (arxiv/paper_2501_01628, package `dprt`) has no volume rendering, so the parts that
 * pin to reference code are the ones the reference does have, restated here operation for operation:
 *   - pinhole primary ray through the pixel centre  : pkg/src/dprt/geom.py:240-259 (camera_primary_ray)
 *                                                     and engine.py:224-251 (gen_primary_batch)
 *   - vector norm / normalize                        : geom.py:47-55
 *   - slab interval with zero-direction semantics    : geom.py:171-200 (ray_aabb_intersect),
 *                                                     clip to [tmin, tmax] as geom.py:203-209
 *   - scalar brute-force "truth" style               : pkg/tests/util.py:95-148 (scalar_reference_render)
 * DVR arithmetic (lattice, trilinear, TF, front-to-back, ERT) follows DESIGN.md §2 and is pinned by the
 * repo's own KATs (tests/test_oracle.py) and golden vectors (tests/golden/), not by a reference test:
 * "parity of DVR arithmetic unpinned by any reference test".
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off; no -ffast-math: every + - * / sqrt is a
 * single correctly rounded IEEE f64 op, in the written order, so results are bit-reproducible).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_ABI_VERSION 7

int dvr_oracle_version(void) { return ORACLE_ABI_VERSION; }

/* camera layout (14 doubles): pos[3] fwd[3] right[3] up[3] half_w half_h -- basis() of geom.py:163-168
 * and half_h = tan(radians(fov_y) * 0.5), half_w = half_h * aspect (geom.py:250-251) are evaluated by
 * the host in Python exactly as the reference does and passed in, so no libm call differs. */

/* geom.py:240-259: ray through the centre of pixel (px, py); image y grows downward. */
static void primary_dir(const double* cam, int px, int py, int W, int H, double d[3]) {
    const double* f = cam + 3;
    const double* r = cam + 6;
    const double* u = cam + 9;
    double half_w = cam[12], half_h = cam[13];
    double sx = (((double)px + 0.5) / (double)W * 2.0 - 1.0) * half_w;
    double sy = (1.0 - ((double)py + 0.5) / (double)H * 2.0) * half_h;
    double dx = f[0] + sx * r[0] + sy * u[0];
    double dy = f[1] + sx * r[1] + sy * u[1];
    double dz = f[2] + sx * r[2] + sy * u[2];
    double n = sqrt(dx * dx + dy * dy + dz * dz); /* geom.py:47-48 */
    d[0] = dx / n;                                /* geom.py:55: divide, not reciprocal-multiply */
    d[1] = dy / n;
    d[2] = dz / n;
}

void dvr_oracle_primary_dirs(const double* cam, int W, int H, double* out) {
    for (int py = 0; py < H; ++py)
        for (int px = 0; px < W; ++px) primary_dir(cam, px, py, W, H, out + 3 * ((int64_t)py * W + px));
}

/* geom.py:171-200.  Returns 1 and (t0, t1) on a hit of the unclipped slab interval, 0 on a miss. */
static int slab(const double o[3], const double d[3], const double lo[3], const double hi[3], double* pt0,
                double* pt1) {
    if (lo[0] > hi[0] || lo[1] > hi[1] || lo[2] > hi[2]) return 0; /* empty box, geom.py:82-83 */
    double t0 = -INFINITY, t1 = INFINITY;
    for (int i = 0; i < 3; ++i) {
        double di = d[i], oi = o[i];
        if (di == 0.0) {
            if (oi < lo[i] || oi > hi[i]) return 0;
            continue;
        }
        double inv = 1.0 / di;
        double ta = (lo[i] - oi) * inv;
        double tb = (hi[i] - oi) * inv;
        if (ta > tb) {
            double s = ta;
            ta = tb;
            tb = s;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t1 < t0) return 0;
    }
    *pt0 = t0;
    *pt1 = t1;
    return 1;
}

int dvr_oracle_slab(const double* o, const double* d, const double* lo, const double* hi, double* t01) {
    return slab(o, d, lo, hi, &t01[0], &t01[1]);
}

/* the brick owns lattice samples t_k = k*dt for k in [ceil(t0/dt), ceil(t1/dt)), where
 * (t0, t1) is the slab interval against the OWNED box clipped to the ray's [0, inf) (geom.py:203-209). */
static int64_t lattice_range(const double o[3], const double d[3], const double lo[3], const double hi[3],
                             double dt, int64_t* k0) {
    double t0, t1;
    if (!slab(o, d, lo, hi, &t0, &t1)) return 0;
    if (t0 < 0.0) t0 = 0.0;
    if (t1 < t0) return 0;
    int64_t a = (int64_t)ceil(t0 / dt);
    int64_t b = (int64_t)ceil(t1 / dt);
    *k0 = a;
    return b > a ? b - a : 0;
}

int64_t dvr_oracle_lattice(const double* o, const double* d, const double* lo, const double* hi, double dt,
                           int64_t* k0) {
    *k0 = 0;
    return lattice_range(o, d, lo, hi, dt, k0);
}

/* blob mixture, evaluated in f64 per voxel in blob order, clamped to 1, rounded to f32.
 * blob layout: cx cy cz inv_rho2 amp (5 doubles).  Coordinates are unit-cube u = i / (N - 1). */
static float field_value(const int64_t N[3], int64_t i, int64_t j, int64_t k, int nb, const double* blobs) {
    double ux = N[0] > 1 ? (double)i / (double)(N[0] - 1) : 0.0;
    double uy = N[1] > 1 ? (double)j / (double)(N[1] - 1) : 0.0;
    double uz = N[2] > 1 ? (double)k / (double)(N[2] - 1) : 0.0;
    double f = 0.0;
    for (int b = 0; b < nb; ++b) {
        const double* p = blobs + 5 * b;
        double dx = ux - p[0], dy = uy - p[1], dz = uz - p[2];
        double r2 = dx * dx + dy * dy + dz * dz;
        double q = 1.0 - r2 * p[3];
        if (q > 0.0) f = f + p[4] * (q * q * q);
    }
    if (f > 1.0) f = 1.0;
    return (float)f;
}

/* Fill out[sd2][sd1][sd0] (x fastest) with the field over global voxels s_lo .. s_lo + sd - 1. */
void dvr_oracle_generate(const int64_t* N, const int64_t* s_lo, const int64_t* sd, int nb, const double* blobs,
                         float* out, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < sd[2]; ++z)
        for (int64_t y = 0; y < sd[1]; ++y) {
            float* row = out + (z * sd[1] + y) * sd[0];
            for (int64_t x = 0; x < sd[0]; ++x)
                row[x] = field_value(N, s_lo[0] + x, s_lo[1] + y, s_lo[2] + z, nb, blobs);
        }
}

/* The same voxels as dvr_oracle_generate, faster: per voxel row (y, z) only the blobs whose support can
 * reach the row are evaluated (the y/z part of r^2 alone already gives q <= 0 for the others, with margin),
 * in blob order and with the identical per-voxel expression -- a skipped blob is one the scalar loop skips
 * too (q > 0 false), so every voxel is bit-identical (tests/test_oracle.py).  Used where whole 1024^3
 * bricks are generated on the host (bench.py's config-3 CPU baseline). */
void dvr_oracle_generate_fast(const int64_t* N, const int64_t* s_lo, const int64_t* sd, int nb, const double* blobs,
                              float* out, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < sd[2]; ++z)
        for (int64_t y = 0; y < sd[1]; ++y) {
            const int64_t j = s_lo[1] + y, k = s_lo[2] + z;
            const double uy = N[1] > 1 ? (double)j / (double)(N[1] - 1) : 0.0;
            const double uz = N[2] > 1 ? (double)k / (double)(N[2] - 1) : 0.0;
            int live[64];
            int nl = 0;
            for (int b = 0; b < nb && b < 64; ++b) {
                const double* p = blobs + 5 * b;
                const double dy = uy - p[1], dz = uz - p[2];
                if ((dy * dy + dz * dz) * p[3] < 1.0 + 1e-9) live[nl++] = b;
            }
            float* row = out + (z * sd[1] + y) * sd[0];
            for (int64_t x = 0; x < sd[0]; ++x) {
                const int64_t i = s_lo[0] + x;
                const double ux = N[0] > 1 ? (double)i / (double)(N[0] - 1) : 0.0;
                double f = 0.0;
                for (int l = 0; l < nl; ++l) {
                    const double* p = blobs + 5 * live[l];
                    double dx = ux - p[0], dy = uy - p[1], dz = uz - p[2];
                    double r2 = dx * dx + dy * dy + dz * dz;
                    double q = 1.0 - r2 * p[3];
                    if (q > 0.0) f = f + p[4] * (q * q * q);
                }
                if (f > 1.0) f = 1.0;
                row[x] = (float)f;
            }
        }
}

/* the Marschner-Lobb test signal (Marschner & Lobb, 1994) on [-1, 1]^3,
 *   rho(x, y, z) = (1 - sin(pi z / 2) + alpha (1 + cos(2 pi f_M cos(pi r / 2)))) / (2 (1 + alpha)),
 *   r = sqrt(x^2 + y^2),
 * the smooth high-frequency stress field of SURVEY.md §8(d).  libm's sin/cos are not reproducible between
 * the CPU and the GPU, so the cosine here is a fixed recipe -- reduction by 2pi (hi + lo), then a 14-term
 * even Taylor polynomial in Horner form -- and the GPU generator (field.cu) repeats it operation for
 * operation with explicitly rounded ops: voxels agree bit for bit.  |error| vs libm < 1e-13 on the
 * arguments used (|a| < 2 pi f_M + pi). */
static const double kMlCos[14] = {1.0, -0.5, 0.041666666666666664, -0.001388888888888889, 2.48015873015873e-05,
                                  -2.755731922398589e-07, 2.08767569878681e-09, -1.1470745597729725e-11,
                                  4.779477332387385e-14, -1.5619206968586225e-16, 4.110317623312165e-19,
                                  -8.896791392450574e-22, 1.6117375710961184e-24, -2.4795962632247976e-27};
#define ML_TWO_PI 6.283185307179586
#define ML_TWO_PI_LO 2.4492935982947064e-16
#define ML_INV_TWO_PI 0.15915494309189535
#define ML_HALF_PI 1.5707963267948966

double dvr_oracle_det_cos(double a) {
    const double k = floor(a * ML_INV_TWO_PI + 0.5);
    const double r = (a - k * ML_TWO_PI) - k * ML_TWO_PI_LO;
    const double r2 = r * r;
    double p = kMlCos[13];
    for (int i = 12; i >= 0; --i) p = p * r2 + kMlCos[i];
    return p;
}

static float ml_value(const int64_t N[3], int64_t i, int64_t j, int64_t k, double fm, double alpha) {
    const double x = 2.0 * (N[0] > 1 ? (double)i / (double)(N[0] - 1) : 0.0) - 1.0;
    const double y = 2.0 * (N[1] > 1 ? (double)j / (double)(N[1] - 1) : 0.0) - 1.0;
    const double z = 2.0 * (N[2] > 1 ? (double)k / (double)(N[2] - 1) : 0.0) - 1.0;
    const double r = sqrt(x * x + y * y);
    const double pr = dvr_oracle_det_cos((ML_TWO_PI * fm) * dvr_oracle_det_cos(ML_HALF_PI * r));
    const double sz = dvr_oracle_det_cos(ML_HALF_PI * z - ML_HALF_PI); /* sin(pi z / 2) */
    double v = ((1.0 - sz) + alpha * (1.0 + pr)) / (2.0 * (1.0 + alpha));
    if (v < 0.0) v = 0.0;
    if (v > 1.0) v = 1.0;
    return (float)v;
}

/* Marschner-Lobb voxels over the stored region (params = {f_M, alpha}), layout as dvr_oracle_generate. */
void dvr_oracle_generate_ml(const int64_t* N, const int64_t* s_lo, const int64_t* sd, const double* params,
                            float* out, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < sd[2]; ++z)
        for (int64_t y = 0; y < sd[1]; ++y) {
            float* row = out + (z * sd[1] + y) * sd[0];
            for (int64_t x = 0; x < sd[0]; ++x)
                row[x] = ml_value(N, s_lo[0] + x, s_lo[1] + y, s_lo[2] + z, params[0], params[1]);
        }
}

static inline double lerp(double a, double b, double f) { return a + (b - a) * f; }

typedef struct {
    const float* vox;
    int64_t s_lo[3], sd[3], N[3];
    int64_t clo[3], chi[3]; /* clamp range for the cell index (global) */
    double lo_w[3], hi_w[3], origin[3], spacing[3];
    const float* tf;
    int n_tf;
    double vmin, tf_scale, dt, ert;
} Brick;

/* trilinear on the global field through the stored voxels, x then y then z. */
static double trilinear(const Brick* b, const double u[3]) {
    int64_t c[3];
    double fr[3];
    for (int a = 0; a < 3; ++a) {
        double fl = floor(u[a]);
        int64_t ci = (int64_t)fl;
        if (ci < b->clo[a]) ci = b->clo[a];
        if (ci > b->chi[a]) ci = b->chi[a];
        double f = u[a] - (double)ci;
        if (f < 0.0) f = 0.0;
        if (f > 1.0) f = 1.0;
        c[a] = ci - b->s_lo[a];
        fr[a] = f;
    }
    const int64_t sx = 1, sy = b->sd[0], sz = b->sd[0] * b->sd[1];
    const float* p = b->vox + c[2] * sz + c[1] * sy + c[0];
    double v000 = p[0], v100 = p[sx], v010 = p[sy], v110 = p[sy + sx];
    double v001 = p[sz], v101 = p[sz + sx], v011 = p[sz + sy], v111 = p[sz + sy + sx];
    double c00 = lerp(v000, v100, fr[0]);
    double c10 = lerp(v010, v110, fr[0]);
    double c01 = lerp(v001, v101, fr[0]);
    double c11 = lerp(v011, v111, fr[0]);
    double c0 = lerp(c00, c10, fr[1]);
    double c1 = lerp(c01, c11, fr[1]);
    return lerp(c0, c1, fr[2]);
}

/* 1D RGBA table, linear between entries, clamped. */
static void tf_lookup(const Brick* b, double v, double out[4]) {
    double x = (v - b->vmin) * b->tf_scale;
    double top = (double)(b->n_tf - 1);
    if (x < 0.0) x = 0.0;
    if (x > top) x = top;
    int64_t i = (int64_t)floor(x);
    if (i > b->n_tf - 2) i = b->n_tf - 2;
    double f = x - (double)i;
    const float* e0 = b->tf + 4 * i;
    const float* e1 = e0 + 4;
    for (int c = 0; c < 4; ++c) out[c] = lerp((double)e0[c], (double)e1[c], f);
}

/* One pixel of one brick: returns the owned lattice sample count; rgba = premultiplied partial. */
/* accum = 0: the brick's own partial from a clear ray (sort-last).  accum = 1: continue the ray's
 * accumulated state in rgba (ray cycling): ERT on the accumulated alpha, a ray already at
 * ERT adds nothing. */
static int64_t march_pixel(const Brick* b, const double* cam, int px, int py, int W, int H, double rgba[4],
                           int accum) {
    double d[3];
    primary_dir(cam, px, py, W, H, d);
    const double* o = cam;
    int64_t k0 = 0;
    int64_t n = lattice_range(o, d, b->lo_w, b->hi_w, b->dt, &k0);
    double C0 = 0.0, C1 = 0.0, C2 = 0.0, A = 0.0;
    if (accum) {
        C0 = rgba[0];
        C1 = rgba[1];
        C2 = rgba[2];
        A = rgba[3];
        if (A >= b->ert) return n;
    }
    for (int64_t k = k0; k < k0 + n; ++k) {
        double t = (double)k * b->dt;
        double u[3];
        for (int a = 0; a < 3; ++a) {
            double p = o[a] + t * d[a];
            u[a] = (p - b->origin[a]) / b->spacing[a];
        }
        double v = trilinear(b, u);
        double e[4];
        tf_lookup(b, v, e);
        double w = (1.0 - A) * e[3]; /* front-to-back, premultiplied */
        C0 = C0 + w * e[0];
        C1 = C1 + w * e[1];
        C2 = C2 + w * e[2];
        A = A + w;
        if (A >= b->ert) break; /* early ray termination, per brick */
    }
    rgba[0] = C0;
    rgba[1] = C1;
    rgba[2] = C2;
    rgba[3] = A;
    return n;
}

/* Render rows row0, row0+row_step, ... < row1 of the full W x H frame for one brick.
 * geo: s_lo[3] sd[3] N[3] lo[3] hi[3] (int64); wgeo: origin[3] spacing[3] (double).
 * out_rgba: H*W*4 doubles (full-frame indexing); samples: H*W uint32 (may be NULL). */
static int brick_setup(Brick* b, const float* vox, const int64_t* geo, const double* wgeo, const float* tf, int n_tf,
                       double vmin, double tf_scale, double dt, double ert) {
    b->vox = vox;
    for (int a = 0; a < 3; ++a) {
        b->s_lo[a] = geo[a];
        b->sd[a] = geo[3 + a];
        b->N[a] = geo[6 + a];
        int64_t lo = geo[9 + a], hi = geo[12 + a];
        b->origin[a] = wgeo[a];
        b->spacing[a] = wgeo[3 + a];
        b->lo_w[a] = b->origin[a] + (double)lo * b->spacing[a];
        b->hi_w[a] = b->origin[a] + (double)hi * b->spacing[a];
        int64_t clo = b->s_lo[a] > 0 ? b->s_lo[a] : 0;
        int64_t chi = b->s_lo[a] + b->sd[a] - 2;
        if (chi > b->N[a] - 2) chi = b->N[a] - 2;
        if (chi < clo) return -2; /* every axis needs >= 2 stored voxels */
        b->clo[a] = clo;
        b->chi[a] = chi;
    }
    b->tf = tf;
    b->n_tf = n_tf;
    b->vmin = vmin;
    b->tf_scale = tf_scale;
    b->dt = dt;
    b->ert = ert;
    return 0;
}

int dvr_oracle_render_brick(const float* vox, const int64_t* geo, const double* wgeo, const double* cam,
                            const float* tf, int n_tf, double vmin, double tf_scale, double dt, double ert,
                            int W, int H, int row0, int row1, int row_step, double* out_rgba,
                            uint32_t* samples, int nthreads) {
    if (n_tf < 2 || !(dt > 0.0) || W <= 0 || H <= 0 || row_step <= 0) return -1;
    Brick b;
    int rc = brick_setup(&b, vox, geo, wgeo, tf, n_tf, vmin, tf_scale, dt, ert);
    if (rc) return rc;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    int nrows = row1 > row0 ? (row1 - row0 + row_step - 1) / row_step : 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int ri = 0; ri < nrows; ++ri) {
        int py = row0 + ri * row_step;
        for (int px = 0; px < W; ++px) {
            int64_t pix = (int64_t)py * W + px;
            double rgba[4];
            int64_t n = march_pixel(&b, cam, px, py, W, H, rgba, 0);
            double* dst = out_rgba + 4 * pix;
            dst[0] = rgba[0];
            dst[1] = rgba[1];
            dst[2] = rgba[2];
            dst[3] = rgba[3];
            if (samples) samples[pix] = (uint32_t)n;
        }
    }
    return 0;
}

/* Ray cycling: continue the accumulated front-to-back state of rows row0 <= y < row1
 * through this brick.  state: H*W*4 doubles (full-frame indexing), read and written in place. */
/* One brick's RGBA partial on a strided pixel lattice: pixels (x0 + i * xs, y0 + j * ys), i < nx, j < ny,
 * written compactly to out_rgba[(j * nx + i) * 4] (f64, premultiplied).  The same march_pixel as
 * dvr_oracle_render_brick, parallel over all sampled pixels (the config-3 CPU baseline's 1/64 subset). */
int dvr_oracle_render_lattice(const float* vox, const int64_t* geo, const double* wgeo, const double* cam,
                              const float* tf, int n_tf, double vmin, double tf_scale, double dt, double ert,
                              int W, int H, int x0, int xs, int nx, int y0, int ys, int ny, double* out_rgba,
                              int nthreads) {
    if (n_tf < 2 || !(dt > 0.0) || W <= 0 || H <= 0 || xs <= 0 || ys <= 0 || nx < 0 || ny < 0) return -1;
    Brick b;
    int rc = brick_setup(&b, vox, geo, wgeo, tf, n_tf, vmin, tf_scale, dt, ert);
    if (rc) return rc;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    const int64_t n = (int64_t)nx * ny;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t q = 0; q < n; ++q) {
        const int px = x0 + (int)(q % nx) * xs, py = y0 + (int)(q / nx) * ys;
        double rgba[4] = {0.0, 0.0, 0.0, 0.0};
        if (px < W && py < H) march_pixel(&b, cam, px, py, W, H, rgba, 0);
        memcpy(out_rgba + 4 * q, rgba, sizeof(rgba));
    }
    return 0;
}

int dvr_oracle_render_brick_accum(const float* vox, const int64_t* geo, const double* wgeo, const double* cam,
                                  const float* tf, int n_tf, double vmin, double tf_scale, double dt, double ert,
                                  int W, int H, int row0, int row1, double* state, int nthreads) {
    if (n_tf < 2 || !(dt > 0.0) || W <= 0 || H <= 0 || row0 < 0 || row1 > H) return -1;
    Brick b;
    int rc = brick_setup(&b, vox, geo, wgeo, tf, n_tf, vmin, tf_scale, dt, ert);
    if (rc) return rc;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int py = row0; py < row1; ++py)
        for (int px = 0; px < W; ++px) march_pixel(&b, cam, px, py, W, H, state + 4 * ((int64_t)py * W + px), 1);
    return 0;
}

/* Owned lattice sample counts only (no marching): per pixel of the full W x H frame for the owned box
 * [lo_w, hi_w] -- the integer-exact ownership check used at full BASELINE sizes. */
void dvr_oracle_sample_counts(const double* lo_w, const double* hi_w, const double* cam, double dt, int W, int H,
                              uint32_t* out, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
    for (int py = 0; py < H; ++py)
        for (int px = 0; px < W; ++px) {
            double d[3];
            primary_dir(cam, px, py, W, H, d);
            int64_t k0 = 0;
            out[(int64_t)py * W + px] = (uint32_t)lattice_range(cam, d, lo_w, hi_w, dt, &k0);
        }
}

int dvr_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

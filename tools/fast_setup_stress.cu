// Stress check of the beam marcher's fast ray setup (DPRT_SETUP_FAST, march.cu fast_range) against the exact
// f64 setup (primary_dir + lattice_range, bit-exact with the oracle): for random and adversarial cameras,
// boxes and sample spacings, every ray whose lattice range fast_range claims must equal the exact one
// (first lattice index and sample count); rays it declines fall back to the exact setup in the marcher.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fss tools/fast_setup_stress.cu && /tmp/fss [configs]
//
// Prints one JSON line: rays, hits, declined (fallback) and wrong (must be 0); exits 1 on any wrong ray.
#define DPRT_SETUP_FAST 1
#include "../paper_2501_01628_b200/csrc/march.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace dprt;

__global__ void stress_kernel(const MarchArgs a, unsigned long long* cnt) {
    const long long np = (long long)a.W * a.H;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np; p += (long long)gridDim.x * blockDim.x) {
        const int px = (int)(p % a.W), py = (int)(p / a.W);
        double d1[3], d2[3];
        int64_t k1 = 0, n1 = 0, k2 = 0;
        const bool ok = fast_range(a, px, py, d1, &k1, &n1);
        primary_dir(a, px, py, d2);
        const int64_t n2 = lattice_range(a, d2, &k2);
        atomicAdd(&cnt[0], 1ull);
        if (n2 > 0) atomicAdd(&cnt[1], 1ull);
        if (!ok) {
            atomicAdd(&cnt[2], 1ull);
            continue;
        }
        if (n1 != n2 || (n2 > 0 && k1 != k2)) atomicAdd(&cnt[3], 1ull);
        double e = 0.0;
        for (int i = 0; i < 3; ++i) e = fmax(e, fabs(d1[i] - d2[i]));
        atomicMax(&cnt[4], (unsigned long long)__double_as_longlong(e));  // e >= 0: bit order == value order
    }
}

static unsigned long long rng = 0x9E3779B97F4A7C15ull;
static double urand() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return (rng >> 11) * (1.0 / 9007199254740992.0);
}
static double urange(double lo, double hi) { return lo + (hi - lo) * urand(); }

static void normalize(double v[3]) {
    const double n = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int i = 0; i < 3; ++i) v[i] /= n;
}
static void cross(const double a[3], const double b[3], double c[3]) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

int main(int argc, char** argv) {
    const int configs = argc > 1 ? atoi(argv[1]) : 3000;
    unsigned long long* cnt;
    cudaMalloc(&cnt, 5 * sizeof(unsigned long long));
    cudaMemset(cnt, 0, 5 * sizeof(unsigned long long));
    const double dts[] = {1.0, 0.5, 0.25, 2.0, 0.7, 1.0 / 3.0, 0.1, 0.37};
    for (int c = 0; c < configs; ++c) {
        MarchArgs a;
        memset(&a, 0, sizeof(a));
        const int kind = c % 4;  // 0 random, 1 axis-aligned view, 2 lattice-aligned box + eye, 3 eye inside the box
        const double dt = (c % 3 == 0) ? urange(0.05, 3.0) : dts[c % 8];
        double lo[3], hi[3], pos[3], tgt[3], up[3] = {0.0, 1.0, 0.0};
        for (int i = 0; i < 3; ++i) {
            lo[i] = kind == 2 ? dt * floor(urange(-50, 50)) : urange(-300, 300);
            hi[i] = lo[i] + (kind == 2 ? dt * floor(urange(1, 200)) : urange(0.5, 600));
            tgt[i] = urange(lo[i], hi[i]);
        }
        for (int i = 0; i < 3; ++i) {
            if (kind == 3)
                pos[i] = urange(lo[i], hi[i]);
            else if (kind == 2)
                pos[i] = lo[i] - dt * floor(urange(1, 400)) * (urand() < 0.5 ? 1 : -1);
            else
                pos[i] = urange(-2000, 2000);
        }
        double f[3], r[3], u[3];
        if (kind == 1 || kind == 2) {  // view along an axis: exact zero direction components on centre rays
            const int ax = c % 3;
            const double s = urand() < 0.5 ? 1.0 : -1.0;
            for (int i = 0; i < 3; ++i) f[i] = i == ax ? s : 0.0;
            for (int i = 0; i < 3; ++i) up[i] = i == (ax + 1) % 3 ? 1.0 : 0.0;
        } else {
            for (int i = 0; i < 3; ++i) f[i] = tgt[i] - pos[i];
            normalize(f);
            for (int i = 0; i < 3; ++i) up[i] = urange(-1, 1);
        }
        cross(f, up, r);
        normalize(r);
        cross(r, f, u);
        const int W = 16 + (int)(urand() * 400), H = 16 + (int)(urand() * 300);
        const double fov = urange(5.0, 120.0) * M_PI / 180.0;
        for (int i = 0; i < 3; ++i) {
            a.o[i] = pos[i];
            a.f[i] = f[i];
            a.r[i] = r[i];
            a.u[i] = u[i];
            a.blo[i] = lo[i];
            a.bhi[i] = hi[i];
            a.fs_L[i] = lo[i] - pos[i];
            a.fs_H[i] = hi[i] - pos[i];
        }
        a.half_h = tan(0.5 * fov);
        a.half_w = a.half_h * W / H;
        a.W = W;
        a.H = H;
        a.dt = dt;
        int ex;
        a.inv_dt_pow2 = (frexp(dt, &ex) == 0.5) ? 1.0 / dt : 0.0;
        a.fs_iw2 = 2.0 / W;
        a.fs_ih2 = 2.0 / H;
        a.fs_idt = 1.0 / dt;
        a.fs_S = 1.0 + fabs(a.half_w) + fabs(a.half_h);
        a.fs_ok = 1;
        stress_kernel<<<296, 256>>>(a, cnt);
    }
    unsigned long long h[5];
    cudaError_t e = cudaMemcpy(h, cnt, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 2;
    }
    double maxd;
    memcpy(&maxd, &h[4], 8);
    printf("{\"configs\": %d, \"rays\": %llu, \"hits\": %llu, \"declined\": %llu, \"wrong\": %llu, "
           "\"declined_frac\": %.3g, \"max_abs_dir_diff\": %.3g}\n",
           configs, h[0], h[1], h[2], h[3], (double)h[2] / (double)h[0], maxd);
    return h[3] ? 1 : 0;
}

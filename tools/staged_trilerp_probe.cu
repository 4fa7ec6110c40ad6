// Instruction-count probe: the beam marcher's batch loop (unroll 4, TF lookup, blend) with the
// trilinear taken from an f32 slab box in shared memory -- what a TMA-staged marcher executes per sample.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cubin tools/staged_trilerp_probe.cu && cuobjdump -sass
__device__ __forceinline__ float lerp(float a, float b, float f) { return fmaf(f, b - a, a); }
extern "C" __global__ void __launch_bounds__(256, 2) staged(const float* __restrict__ g, const float4* __restrict__ tf, float4* out,
    float p00, float p01, float p02, float s0, float s1, float s2, int n, int py, int pz, float tns, float tno, float top, float ert) {
    extern __shared__ float sm[];
    float4* s_tf = reinterpret_cast<float4*>(sm);
    float4* s_dtf = s_tf + 256;
    float* box = sm + 2048 + (threadIdx.x >> 5) * 3072;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) { s_tf[i] = tf[i]; s_dtf[i] = tf[i + 256]; }
    for (int i = threadIdx.x; i < 3072 * 8; i += blockDim.x) sm[2048 + i] = g[i];
    __syncthreads();
    float C0 = 0, C1 = 0, C2 = 0, A = 0;
    const float p0[3] = {p00 + threadIdx.x * 0.01f, p01, p02};
    const float st[3] = {s0, s1, s2};
    int j = 0; const int jend = n;
    const float fend = (float)(jend - 1);
    while (j < jend) {
        float c[4][8], wx[4], wy[4], wz[4];
        const float fj = (float)j;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float fs = fminf(fj + (float)u, fend);
            const float ux = fmaf(fs, st[0], p0[0]), uy = fmaf(fs, st[1], p0[1]), uz = fmaf(fs, st[2], p0[2]);
            const int ix = __float2int_rd(ux), iy = __float2int_rd(uy), iz = __float2int_rd(uz);
            const float* b = box + iz * pz + iy * py + ix;
            c[u][0] = b[0]; c[u][1] = b[1]; c[u][2] = b[py]; c[u][3] = b[py + 1];
            c[u][4] = b[pz]; c[u][5] = b[pz + 1]; c[u][6] = b[pz + py]; c[u][7] = b[pz + py + 1];
            wx[u] = __saturatef(ux - (float)ix); wy[u] = __saturatef(uy - (float)iy); wz[u] = __saturatef(uz - (float)iz);
        }
        const int cnt = min(4, jend - j);
        float m = 1.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (u >= cnt) m = 0.f;
            const float e00 = lerp(c[u][0], c[u][1], wx[u]), e01 = lerp(c[u][2], c[u][3], wx[u]);
            const float e10 = lerp(c[u][4], c[u][5], wx[u]), e11 = lerp(c[u][6], c[u][7], wx[u]);
            const float v = lerp(lerp(e00, e01, wy[u]), lerp(e10, e11, wy[u]), wz[u]);
            const float x = __saturatef(fmaf(v, tns, tno)) * top;
            const int ti = (int)x;
            const float tfr = x - (float)ti;
            const float4 e0 = s_tf[ti], de = s_dtf[ti];
            const float w = m * ((1.f - A) * fmaf(tfr, de.w, e0.w));
            A += w;
            C0 = fmaf(w, fmaf(tfr, de.x, e0.x), C0);
            C1 = fmaf(w, fmaf(tfr, de.y, e0.y), C1);
            C2 = fmaf(w, fmaf(tfr, de.z, e0.z), C2);
            if (A >= ert) m = 0.f;
        }
        j += cnt;
        if (A >= ert) break;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = make_float4(C0, C1, C2, A);
}

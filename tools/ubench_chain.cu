// Microbenchmark: cycles per element of a dependent DSUB chain (one thread)
// when the chain is (a) alone, (b) interleaved with independent DMULs,
// (c) interleaved with shared-memory loads, (d) both — the pattern of the
// exact coarse solve's backward row chain.  usage: ubench_chain
#include <cstdio>
__global__ void k(int mode, int iters, double* out, long long* cyc) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-300 * (i + 1);
    __syncthreads();
    if (threadIdx.x != 0) return;
    double s = 1.0, p[8], q[8];
    for (int t = 0; t < 8; ++t) { p[t] = sm[t]; q[t] = sm[t + 8]; }
    long long t0 = clock64();
    int j = 0;
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
#pragma unroll
            for (int t = 0; t < 8; ++t) s = __dsub_rn(s, p[t]);
        } else if (mode == 1) {
#pragma unroll
            for (int t = 0; t < 8; ++t) { s = __dsub_rn(s, p[t]); q[t] = __dmul_rn(q[t], 1.0000001); }
        } else if (mode == 2) {
#pragma unroll
            for (int t = 0; t < 8; ++t) { s = __dsub_rn(s, p[t]); q[t] = sm[(j + t) & 1023]; }
            j += 8;
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) { s = __dsub_rn(s, p[t]); q[t] = __dmul_rn(sm[(j + t) & 1023], sm[(j + t + 64) & 1023]); }
            j += 8;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) { double x = p[t]; p[t] = q[t]; q[t] = x; }
    }
    long long t1 = clock64();
    double a = s;
    for (int t = 0; t < 8; ++t) a += p[t] + q[t];
    out[0] = a;
    cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    const char* names[4] = {"chain alone", "+ DMUL", "+ LDS", "+ LDS + DMUL"};
    for (int mode = 0; mode < 4; ++mode) {
        k<<<1, 32>>>(mode, 100, o, c);
        k<<<1, 32>>>(mode, 10000, o, c);
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-14s %.2f cycles per chain element\n", names[mode], (double)h / 80000.0);
    }
    return 0;
}

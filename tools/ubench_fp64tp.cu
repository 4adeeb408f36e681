// Microbenchmark: fp64 issue throughput of one SM (DFMA / DADD), 512 threads,
// 8 independent chains per thread.
#include <cstdio>
template <int OP>
__global__ void tp(double* out, int iters, double a, long long* cyc) {
    double s[8];
    for (int j = 0; j < 8; ++j) s[j] = a + threadIdx.x + j;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = OP == 0 ? __fma_rn(s[j], 0.999999, 1e-7) : __dadd_rn(s[j], 1e-300);
    __syncthreads();
    long long t1 = clock64();
    double r = 0;
    for (int j = 0; j < 8; ++j) r += s[j];
    out[threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
    long long h;
    for (int th : {128, 512, 1024}) {
        tp<0><<<1, th>>>(o, 100, 1.0, c); cudaDeviceSynchronize();
        tp<0><<<1, th>>>(o, 10000, 1.0, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d DFMA: %.2f thread-ops/clk/SM\n", th, 8.0 * 10000 * th / h);
        tp<1><<<1, th>>>(o, 10000, 1.0, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d DADD: %.2f thread-ops/clk/SM\n", th, 8.0 * 10000 * th / h);
    }
    return 0;
}

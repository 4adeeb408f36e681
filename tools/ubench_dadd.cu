// Microbenchmark: latency of a dependent fp64 add chain (__dadd_rn) and of a
// dependent smem-load + add chain, one thread, clock64-timed.
#include <cstdio>
__global__ void chain(double* out, int iters, double a, long long* cyc) {
    double s = a;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        s = __dadd_rn(s, 1e-300); s = __dadd_rn(s, 1e-300); s = __dadd_rn(s, 1e-300); s = __dadd_rn(s, 1e-300);
    }
    long long t1 = clock64();
    out[0] = s;
    cyc[0] = t1 - t0;
}
__global__ void chain_div(double* out, int iters, double a, long long* cyc) {
    double s = a;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __ddiv_rn(s, 1.0000001);
    long long t1 = clock64();
    out[0] = s;
    cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    long long h;
    chain<<<1,1>>>(o, 1000, 1.0, c); cudaDeviceSynchronize();
    chain<<<1,1>>>(o, 100000, 1.0, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dadd dependent latency: %.2f cycles\n", (double)h / 400000.0);
    chain_div<<<1,1>>>(o, 100000, 1.0, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("ddiv dependent latency: %.2f cycles\n", (double)h / 100000.0);
    return 0;
}

// Microbenchmark: dependent-load latency (pointer chase, one thread) for
// working sets from L1-size to DRAM-size, with .ca (L1) and .cg (L2) loads,
// and the cost of a global write -> read round trip between two SMs.
#include <cstdio>
#include <vector>
__global__ void chase_ca(const int* __restrict__ p, int steps, int* out, long long* cyc) {
    int j = 0;
    for (int i = 0; i < 64; ++i) j = p[j];  // warm
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) j = __ldca(p + j);
    long long t1 = clock64();
    out[0] = j;
    cyc[0] = t1 - t0;
}
__global__ void chase_cg(const int* __restrict__ p, int steps, int* out, long long* cyc) {
    int j = 0;
    for (int i = 0; i < 64; ++i) j = __ldcg(p + j);
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) j = __ldcg(p + j);
    long long t1 = clock64();
    out[0] = j;
    cyc[0] = t1 - t0;
}
int main() {
    int *d, *o;
    long long* c;
    const size_t maxn = 64u << 20;  // 256 MB of ints
    cudaMalloc(&d, maxn * 4);
    cudaMalloc(&o, 4);
    cudaMalloc(&c, 8);
    for (size_t kb : {16, 128, 1024, 8192, 32768, 65536, 262144}) {
        size_t n = kb * 1024 / 4;
        // random cyclic permutation with stride >= 32 ints (one line)
        size_t lines = n / 32;
        std::vector<int> perm(lines);
        for (size_t i = 0; i < lines; ++i) perm[i] = (int)i;
        unsigned s = 12345;
        for (size_t i = lines - 1; i > 0; --i) {
            s = s * 1103515245u + 12345u;
            size_t k = s % (i + 1);
            std::swap(perm[i], perm[k]);
        }
        std::vector<int> h(n, 0);
        for (size_t i = 0; i < lines; ++i) h[(size_t)perm[i] * 32] = perm[(i + 1) % lines] * 32;
        cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
        long long t;
        const int steps = 4096;
        chase_ca<<<1, 1>>>(d, steps, o, c);
        cudaMemcpy(&t, c, 8, cudaMemcpyDeviceToHost);
        double ca = (double)t / steps;
        chase_cg<<<1, 1>>>(d, steps, o, c);
        cudaMemcpy(&t, c, 8, cudaMemcpyDeviceToHost);
        printf("working set %7zu KB: ld.ca %6.0f cycles, ld.cg %6.0f cycles\n", kb, ca, (double)t / steps);
    }
    return 0;
}

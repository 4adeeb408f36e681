// Microbenchmark: latency of reading, right after a grid barrier, data that
// other SMs wrote just before it (pointer chase through lines written by
// other blocks), vs. reading long-resident data.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int* buf, int n, int* out, long long* cyc, int mode) {
    cg::grid_group g = cg::this_grid();
    // every block writes a chain segment: buf[b*64] -> next block's slot
    if (threadIdx.x == 0) buf[blockIdx.x * 64] = ((blockIdx.x + 37) % gridDim.x) * 64;
    g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int j = 0;
        long long t0 = clock64();
        for (int i = 0; i < 16; ++i) j = mode == 0 ? __ldcg(buf + j) : (mode == 1 ? __ldca(buf + j) : *(volatile int*)(buf + j));
        long long t1 = clock64();
        out[0] = j;
        cyc[0] = (t1 - t0) / 16;
        // second pass over the same (now cached) lines
        t0 = clock64();
        for (int i = 0; i < 16; ++i) j = __ldcg(buf + j);
        t1 = clock64();
        out[1] = j;
        cyc[1] = (t1 - t0) / 16;
    }
}
int main() {
    int *b, *o;
    long long* c;
    cudaMalloc(&b, 4 << 20);
    cudaMalloc(&o, 8);
    cudaMalloc(&c, 16);
    for (int mode = 0; mode < 3; ++mode)
        for (int grid : {148, 592}) {
            int n = 0;
            void* args[] = {&b, &n, &o, &c, &mode};
            for (int r = 0; r < 3; ++r) cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
            long long h[2];
            cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
            printf("mode %s grid %d: first read after barrier %lld cycles/load, re-read %lld cycles/load\n",
                   mode == 0 ? "ld.cg" : (mode == 1 ? "ld.ca" : "volatile"), grid, h[0], h[1]);
        }
    return 0;
}

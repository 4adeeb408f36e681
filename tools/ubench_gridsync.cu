// Microbenchmark: cost of cooperative-groups grid.sync() on this GPU.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
int main() {
    int* o;
    cudaMalloc(&o, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int bps : {1, 2, 4, 8}) {
        for (int th : {128, 256}) {
            int grid = 148 * bps, it0 = 0, it1 = 1000;
            void* args0[] = {&it0, &o};
            void* args1[] = {&it1, &o};
            cudaLaunchCooperativeKernel((void*)k, grid, th, args0, 0, 0);
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r) cudaLaunchCooperativeKernel((void*)k, grid, th, args0, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float t0;
            cudaEventElapsedTime(&t0, a, b);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k, grid, th, args1, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float t1;
            cudaEventElapsedTime(&t1, a, b);
            printf("grid %4d x %3d: empty launch %.2f us, grid.sync %.3f us (%s)\n", grid, th, 1e3 * t0 / 10,
                   1e3 * t1 / it1, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

// Microbenchmark: cost of small "row pass" phases separated by grid barriers
// inside one cooperative kernel (the V-cycle tail's structure): 151 rows x 7
// nnz, r = f - A u with u written by the previous phase on other SMs.
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void k(int n, const int* rp, const int* col, const double* val, double* u, double* r, int phases,
                  unsigned long long* tr, int mode) {
    cg::grid_group g = cg::this_grid();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int p = 0; p < phases; ++p) {
        if (tid < n) {
            double s = 0;
            for (int k = __ldg(rp + tid); k < __ldg(rp + tid + 1); ++k)
                s += __ldg(val + k) * (mode ? __ldcg(u + __ldg(col + k)) : u[__ldg(col + k)]);
            r[tid] = 1.0 - s;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) tr[2 * p] = gt();
        g.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) tr[2 * p + 1] = gt();
        if (tid < n) u[(tid * 37) % n] = __ldcg(r + tid) * 0.5;  // "restrict" writes u on other threads' rows
        g.sync();
    }
}
int main() {
    const int n = 151;
    std::vector<int> rp(n + 1), col;
    std::vector<double> val;
    for (int i = 0; i < n; ++i) {
        rp[i] = (int)col.size();
        for (int d : {-20, -5, -1, 0, 1, 5, 20})
            if (i + d >= 0 && i + d < n) {
                col.push_back(i + d);
                val.push_back(d == 0 ? 4.0 : -0.5);
            }
    }
    rp[n] = (int)col.size();
    int *drp, *dcol;
    double *dval, *du, *dr;
    unsigned long long* tr;
    cudaMalloc(&drp, 4 * (n + 1));
    cudaMalloc(&dcol, 4 * col.size());
    cudaMalloc(&dval, 8 * val.size());
    cudaMalloc(&du, 8 * n);
    cudaMalloc(&dr, 8 * n);
    cudaMalloc(&tr, 8 * 256);
    cudaMemcpy(drp, rp.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(dcol, col.data(), 4 * col.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dval, val.data(), 8 * val.size(), cudaMemcpyHostToDevice);
    cudaMemset(du, 0, 8 * n);
    int phases = 20;
    for (int mode = 0; mode < 2; ++mode)
        for (int grid : {1, 148, 592}) {
            for (int th : {256, 1024}) {
                if (grid == 592 && th == 1024) continue;
                void* args[] = {(void*)&n, &drp, &dcol, &dval, &du, &dr, &phases, &tr, &mode};
                for (int rep = 0; rep < 2; ++rep)
                    cudaLaunchCooperativeKernel((void*)k, grid, th, args, 0, 0);
                unsigned long long h[256];
                cudaMemcpy(h, tr, 8 * 2 * phases, cudaMemcpyDeviceToHost);
                double work = 0, all = 0;
                for (int p = 1; p < phases; ++p) {
                    work += (h[2 * p] - h[2 * p - 1]) / 1e3;
                    all += (h[2 * p + 1] - h[2 * p - 1]) / 1e3;
                }
                printf("mode %s grid %3d x %4d: row phase (block 0) %.2f us, row+restrict+2 syncs %.2f us  (%s)\n",
                       mode ? "ldcg" : "plain", grid, th, work / (phases - 1), all / (phases - 1),
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}

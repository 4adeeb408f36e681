// Micro-benchmark of the coarsest-level dense kernels (LU factor / inverse)
// on a 149 x 149 system like the C3 hierarchy's coarsest level (argument 2 "s":
// sparse, ~7 entries per row, diagonally dominant; default dense random).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 --expt-relaxed-constexpr
//      -I paper_2108_02054_b200/csrc -I include tools/ubench_dense.cu -o tools/ubench_dense
#include "../paper_2108_02054_b200/csrc/kernels_core.cu"

#include <cstdio>
#include <cstring>
namespace amgr {
void probe_begin(Ctx&, const char*, double) {}
void probe_end(Ctx&, const char*) {}
}  // namespace amgr
#include <random>
#include <vector>

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 149;
    std::vector<double> a(n * n);
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> u(-1, 1);
    const bool sparse = argc > 2 && argv[2][0] == 's';  // like the C3 coarsest level: ~7 entries per row
    if (sparse) {
        std::uniform_int_distribution<int> col(0, n - 1);
        for (int i = 0; i < n; ++i) {
            double d = 1.0;
            for (int t = 0; t < 6; ++t) {
                const int j = col(g);
                if (j == i) continue;
                const double v = -std::abs(u(g));
                a[i * n + j] += v;
                a[j * n + i] += v;
            }
        }
        for (int i = 0; i < n; ++i) {
            double r = 1.0;
            for (int j = 0; j < n; ++j)
                if (j != i) r += std::abs(a[i * n + j]);
            a[i * n + i] = r;
        }
    } else {
        for (auto& x : a) x = u(g);
        for (int i = 0; i < n; ++i) a[i * n + i] += 4.0;
    }
    double *da, *dm, *di;
    int64_t* piv;
    int* st;
    cudaMalloc(&da, 8 * n * n);
    cudaMalloc(&dm, 8 * n * n);
    cudaMalloc(&di, 8 * n * n);
    cudaMalloc(&piv, 8 * n);
    cudaMalloc(&st, 4);
    cudaMemcpy(da, a.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto fn) {
        for (int w = 0; w < 3; ++w) fn();
        cudaEventRecord(e0);
        const int R = 20;
        for (int r = 0; r < R; ++r) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-22s n=%d  %8.2f us/launch  (%s)\n", name, n, 1e3 * ms / R, cudaGetErrorString(cudaGetLastError()));
    };
    cudaFuncSetAttribute(amgr::k_dense_reg<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 160 * 160);
    timeit("dense_reg LU", [&] {
        cudaMemcpyAsync(dm, da, 8 * n * n, cudaMemcpyDeviceToDevice);
        amgr::k_dense_reg<false><<<1, amgr::DR_THREADS, 8 * n * n>>>(n, dm, dm, piv, st, nullptr);
    });
    timeit("dense_reg GJ inverse", [&] { amgr::k_dense_reg<true><<<1, amgr::DR_THREADS>>>(n, da, di, piv, st, nullptr); });
    cudaFuncSetAttribute(amgr::k_lu_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
    timeit("lu_factor (smem)", [&] {
        cudaMemcpyAsync(dm, da, 8 * n * n, cudaMemcpyDeviceToDevice);
        amgr::k_lu_factor<<<1, amgr::LU_THREADS, 8 * n * n>>>(n, dm, piv, st, 1);
    });
    timeit("memcpy only", [&] { cudaMemcpyAsync(dm, da, 8 * n * n, cudaMemcpyDeviceToDevice); });
    // check GJ inverse: || A * inv - I ||
    std::vector<double> inv(n * n);
    amgr::k_dense_reg<true><<<1, amgr::DR_THREADS>>>(n, da, di, piv, st, nullptr);
    cudaMemcpy(inv.data(), di, 8 * n * n, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += a[i * n + k] * inv[k * n + j];
            err = std::max(err, std::abs(s - (i == j)));
        }
    printf("GJ inverse max |A inv - I| = %.3e\n", err);
    // LU: register kernel vs the shared-memory kernel, bit for bit
    std::vector<double> l1(n * n), l2(n * n);
    std::vector<int64_t> p1(n), p2(n);
    cudaMemcpy(dm, da, 8 * n * n, cudaMemcpyDeviceToDevice);
    amgr::k_dense_reg<false><<<1, amgr::DR_THREADS, 8 * n * n>>>(n, dm, dm, piv, st, nullptr);
    cudaMemcpy(l1.data(), dm, 8 * n * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(p1.data(), piv, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(dm, da, 8 * n * n, cudaMemcpyDeviceToDevice);
    amgr::k_lu_factor<<<1, amgr::LU_THREADS, 8 * n * n>>>(n, dm, piv, st, 1);
    cudaMemcpy(l2.data(), dm, 8 * n * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(p2.data(), piv, 8 * n, cudaMemcpyDeviceToHost);
    printf("LU register vs smem kernel: %s\n",
           (memcmp(l1.data(), l2.data(), 8 * n * n) == 0 && p1 == p2) ? "bit-identical" : "DIFFERENT");
    return 0;
}

// Microbenchmark: where the multi-warp exact coarse solve spends its time.
// A copy of the library's k_lu_solve_mw structure (kernels_core.cu) with
// clock64 stamps: start, factor landed, forward done, backward done, plus the
// cycles the chain spent waiting for helper product rows and the cycles in
// its DSUB loops.  Random diagonally dominant LU of size n.
// usage: ubench_lusolve_mw [n]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>

constexpr int LW_Q = 5, LM_HELP = 3, LM_PAD = 24;
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ bool mk_range(double v) {
    const int e = (__double2hiint(v) >> 20) & 0x7ff;
    return e >= 600 && e <= 1446;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
#ifndef SYNC_MODE
#define SYNC_MODE 0
#endif
__device__ __forceinline__ void st_rel(int* p, int v) {
#if SYNC_MODE == 0
    asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(su32(p)), "r"(v) : "memory");
#elif SYNC_MODE == 1
    __threadfence_block();
    *reinterpret_cast<volatile int*>(p) = v;
#else
    *reinterpret_cast<volatile int*>(p) = v;
#endif
}
__device__ __forceinline__ int ld_acq(const int* p) {
#if SYNC_MODE == 0
    int v;
    asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(su32(p)) : "memory");
    return v;
#else
    return *reinterpret_cast<const volatile int*>(p);
#endif
}

__global__ void __launch_bounds__(128) k_mw(int n, const double* __restrict__ m, const double* b, double* x,
                                            long long* st) {
    extern __shared__ __align__(128) double sm[];
    __shared__ int s_prog, s_ready[3];
    __shared__ long long stamp[256];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nn2 = (n * n + 1) & ~1, W = n + LM_PAD;
    double* ms = sm;
    double* xs = sm + nn2;
    double* pb = xs + W;
    double* rd = pb + 3 * W;
    int* okd = reinterpret_cast<int*>(rd + n);
    long long t0 = clock64();
    for (int i = tid; i < nn2; i += blockDim.x) ms[i] = m[i];
    for (int i = tid; i < 4 * W; i += blockDim.x) xs[i] = 0.0;
    if (tid == 0) {
        s_prog = n;
        s_ready[0] = s_ready[1] = s_ready[2] = -1;
    }
    __syncthreads();
    long long t1 = clock64();
    if (wid == 0) {
        double y[LW_Q];
#pragma unroll
        for (int q = 0; q < LW_Q; ++q) {
            const int i = 32 * q + lane;
            y[q] = i < n ? b[i] : 0.0;
        }
#pragma unroll
        for (int gq = 0; gq < LW_Q; ++gq) {
            if (32 * gq >= n - 1) break;
            for (int t = 0; t < 32; ++t) {
                const int j = 32 * gq + t;
                if (j >= n - 1) break;
                const double yj = __shfl_sync(0xffffffffu, y[gq], t);
#pragma unroll
                for (int q = gq; q < LW_Q; ++q) {
                    const int i = 32 * q + lane;
                    if (i > j && i < n) y[q] = xsub(y[q], xmul(ms[i * n + j], yj));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < LW_Q; ++q) {
            const int i = 32 * q + lane;
            if (i < n) xs[i] = y[q];
        }
    } else {
        for (int i = tid - 32; i < n; i += 32 * LM_HELP) {
            const double u = ms[i * n + i];
            rd[i] = __drcp_rn(u);
            okd[i] = mk_range(u) ? 1 : 0;
        }
    }
    __syncthreads();
    long long t2 = clock64(), wait = 0, loop = 0;
    if (wid == 0) {
        if (lane == 0) {
            // row i's scalars, loaded one row ahead
            auto mk = [&](double s, double u, double yv, int ok) -> double {
                if (ok && mk_range(s)) {
                    const double q = __dmul_rn(s, yv);
                    const double r = __fma_rn(-u, q, s);
                    return __fma_rn(r, yv, q);
                }
                return __ddiv_rn(s, u);
            };
            double x1 = mk(xs[n - 1], ms[(n - 1) * n + n - 1], rd[n - 1], okd[n - 1]), x2 = 0.0;
            xs[n - 1] = x1;
            st_rel(&s_prog, n - 1);
            int i = n - 2;
            double cy = xs[i], cu1 = ms[i * n + i + 1], cu2 = i + 2 < n ? ms[i * n + i + 2] : 0.0;
            double cuu = ms[i * n + i], crd = rd[i];
            int cok = okd[i];
            for (; i >= 0; --i) {
                // prefetch row i - 1
                const int k = i > 0 ? i - 1 : 0;
                const double ny = xs[k], nu1 = ms[k * n + k + 1], nu2 = ms[k * n + k + 2], nuu = ms[k * n + k];
                const double nrd = rd[k];
                const int nok = okd[k];
                const double* P = pb + (i % 3) * W;
                double a[8];
                const bool chain = i + 3 < n;
                if (chain) {
#if SYNC_MODE != 3
                    while (ld_acq(&s_ready[i % 3]) != i) {
                    }
#endif
#pragma unroll
                    for (int t = 0; t < 8; ++t) a[t] = P[i + 3 + t];
                }
                const double p2 = xmul(cu2, x2);
                double s = xsub(cy, xmul(cu1, x1));
                if (i + 2 < n) s = xsub(s, p2);
                if (chain) {
                    for (int j = i + 3; j < n; j += 8) {
                        double c[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) c[t] = P[j + 8 + t];
#pragma unroll
                        for (int t = 0; t < 8; ++t) s = xsub(s, a[t]);
#pragma unroll
                        for (int t = 0; t < 8; ++t) a[t] = c[t];
                    }
                }
                const double xi = mk(s, cuu, crd, cok);
                xs[i] = xi;
                st_rel(&s_prog, i);
                stamp[i] = clock64();
                x2 = x1;
                x1 = xi;
                cy = ny;
                cu1 = nu1;
                cu2 = nu2;
                cuu = nuu;
                crd = nrd;
                cok = nok;
            }
        }
    } else {
        const int hid = tid - 32;
        for (int i = n - 4; i >= 0; --i) {
#if SYNC_MODE == 3
            break;  // timing only: the chain does not wait (results wrong)
#endif
            while (ld_acq(&s_prog) > i + 3) {
#if SYNC_MODE == 4
                __nanosleep(40);
#endif
            }
            double* P = pb + (i % 3) * W;
            const double* mi = ms + i * n;
            for (int j = i + 3 + hid; j < n; j += 32 * LM_HELP) P[j] = xmul(mi[j], xs[j]);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LM_HELP) : "memory");
            if (hid == 0) st_rel(&s_ready[i % 3], i);
        }
    }
    __syncthreads();
    long long t3 = clock64();
    for (int i = tid; i < n; i += blockDim.x) x[i] = xs[i];
    for (int i = tid; i < n - 1; i += blockDim.x) st[8 + i] = stamp[i];
    if (tid == 0) {
        st[5] = t2;
        st[0] = t1 - t0;
        st[1] = t2 - t1;
        st[2] = t3 - t2;
        st[3] = wait;
        st[4] = loop;
    }
}

// the reference's order (dense_lu.cpp:52-73 without pivots), one thread
__global__ void k_ref(int n, const double* m, const double* b, double* x) {
    for (int i = 0; i < n; ++i) x[i] = b[i];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) x[i] = xsub(x[i], xmul(m[i * n + j], x[j]));
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int j = i + 1; j < n; ++j) s = xsub(s, xmul(m[i * n + j], x[j]));
        x[i] = __ddiv_rn(s, m[i * n + i]);
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 149;
    std::vector<double> h(static_cast<size_t>(n) * n), hb(n);
    srand(1);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[i * n + j] = (i == j) ? 4.0 + rand() % 7 : (rand() % 1000) / 1000.0 - 0.5;
    for (int i = 0; i < n; ++i) hb[i] = (rand() % 1000) / 100.0;
    double *dm, *db, *dx;
    long long* ds;
    cudaMalloc(&dm, h.size() * 8);
    cudaMalloc(&db, n * 8);
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&ds, 8 * 512);
    cudaMemcpy(dm, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), n * 8, cudaMemcpyHostToDevice);
    const int W = n + LM_PAD;
    const size_t sm = sizeof(double) * (((n * n + 1) & ~1) + 4 * W + n) + sizeof(int) * n;
    cudaFuncSetAttribute(k_mw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int r = 0; r < 3; ++r) k_mw<<<1, 128, sm>>>(n, dm, db, dx, ds);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) k_mw<<<1, 128, sm>>>(n, dm, db, dx, ds);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms_ = 0;
    cudaEventElapsedTime(&ms_, e0, e1);
    double* dr;
    cudaMalloc(&dr, n * 8);
    k_ref<<<1, 1>>>(n, dm, db, dr);
    std::vector<double> h1(n), h2(n);
    cudaMemcpy(h1.data(), dx, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), dr, n * 8, cudaMemcpyDeviceToHost);
    int diff = 0;
    for (int i = 0; i < n; ++i) diff += memcmp(&h1[i], &h2[i], 8) != 0;
    printf("{\"bit_mismatches_vs_serial\": %d}\n", diff);
    long long hs[512];
    cudaMemcpy(hs, ds, 8 * 512, cudaMemcpyDeviceToHost);
    // row i's duration = stamp[i] - stamp[i+1] (row n-2 from the backward start)
    printf("{\"row_cycles\": [");
    for (int i = n - 2; i >= 0; --i) {
        const long long prev = i == n - 2 ? hs[5] : hs[8 + i + 1];
        printf("%s[%d, %lld]", i == n - 2 ? "" : ", ", n - 1 - i, hs[8 + i] - prev);
    }
    printf("]}\n");
    const long long nel = static_cast<long long>(n) * (n - 1) / 2;
    printf("{\"n\": %d, \"us_per_call\": %.2f, \"load_cycles\": %lld, \"forward_cycles\": %lld, \"backward_cycles\": %lld, "
           "\"chain_wait_cycles\": %lld, \"chain_loop_cycles\": %lld, \"loop_cycles_per_entry\": %.2f, \"%s\": 0}\n",
           n, ms_ * 1000 / 20, hs[0], hs[1], hs[2], hs[3], hs[4], (double)hs[4] / nel, cudaGetErrorString(cudaGetLastError()));
    return 0;
}

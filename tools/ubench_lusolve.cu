// Microbenchmark: where the single-warp exact coarse solve spends its time.
// A copy of the library's k_lu_solve_warp structure (kernels_core.cu) with
// clock64 stamps at the phase boundaries, on a random diagonally dominant
// LU of size n (values do not matter for timing).  usage: ubench_lusolve [n]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ double bwd_chain(const double* __restrict__ mi, const double* __restrict__ xs, int j0,
                                            int n, double s) {
    // s -= mi[j]*xs[j] for j = j0 .. n-1, ascending.  The leading (n - j0) % 8
    // entries go first so the 8-entry chunks end exactly at n.  Three-stage
    // software pipeline over the chunks: the shared-memory loads of chunk c+2
    // and the products of chunk c+1 issue while chunk c's dependent DSUB
    // chain runs, so (in-order issue) no instruction of the chain waits on a
    // load: the sweep runs at the DSUB latency.
    const int rem = (n - j0) & 7;
    const int jf = j0 + rem;          // first full chunk
    const int nch = (n - jf) >> 3;    // full chunks
    double ra[8], rx[8], p[8];
    // issue everything the first chunks need up front
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        ra[t] = mi[j0 + t];  // remainder (first rem used); reads stay inside the factor + slack
        rx[t] = xs[j0 + t];
    }
    double fa[8], fx[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        fa[t] = mi[jf + t];  // chunk 0 (harmless reads when nch == 0)
        fx[t] = xs[jf + t];
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) p[t] = xmul(ra[t], rx[t]);
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (t < rem) s = xsub(s, p[t]);
    if (nch == 0) return s;
    // chunk 0 products; raw loads of chunk 1
#pragma unroll
    for (int t = 0; t < 8; ++t) p[t] = xmul(fa[t], fx[t]);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        ra[t] = mi[jf + 8 + t];
        rx[t] = xs[jf + 8 + t];
    }
    int jn = jf + 16;  // raw chunk to load next
    for (int c = 0; c < nch; ++c) {
        double q[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            s = xsub(s, p[t]);
            q[t] = xmul(ra[t], rx[t]);  // chunk c+1 (garbage past the end, unused)
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            ra[t] = mi[jn + t];  // chunk c+2
            rx[t] = xs[jn + t];
            p[t] = q[t];
        }
        jn += 8;
    }
    return s;
}

template <int MODE>  // 0 full, 1 no division (multiply), 2 chain only (no per-row overhead measured separately)
__global__ void k(int n, const double* __restrict__ m, const double* b, double* x, long long* stamps) {
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x;
    const int nn2 = (n * n + 1) & ~1;
    double* ms = sm;
    double* xs = sm + nn2;
    long long t0 = clock64();
    for (int i = lane; i < nn2; i += 32) ms[i] = m[i];
    __syncwarp();
    long long t1 = clock64();
    double y[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = 32 * q + lane;
        y[q] = i < n ? b[i] : 0.0;
    }
#pragma unroll
    for (int gq = 0; gq < 5; ++gq) {
        if (32 * gq >= n - 1) break;
        for (int t = 0; t < 32; ++t) {
            const int j = 32 * gq + t;
            if (j >= n - 1) break;
            const double yj = __shfl_sync(0xffffffffu, y[gq], t);
#pragma unroll
            for (int q = gq; q < 5; ++q) {
                const int i = 32 * q + lane;
                if (i > j && i < n) y[q] = xsub(y[q], xmul(ms[i * n + j], yj));
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = 32 * q + lane;
        if (i < n) xs[i] = y[q];
    }
    if (lane < 16) xs[n + lane] = 0.0;
    __syncwarp();
    long long t2 = clock64();
    long long tdiv = 0, tchain = 0;
    if (lane == 0) {
        double xn = __ddiv_rn(xs[n - 1], ms[(n - 1) * n + (n - 1)]);
        xs[n - 1] = xn;
        for (int i = n - 2; i >= 0; --i) {
            const double* mi = ms + i * n;
            long long a = clock64();
            double s = xsub(xs[i], xmul(mi[i + 1], xn));
            if (i + 2 < n) s = bwd_chain(mi, xs, i + 2, n, s);
            long long bb = clock64();
            xn = MODE == 1 ? xmul(s, mi[i]) : __ddiv_rn(s, mi[i]);
            xs[i] = xn;
            long long c = clock64();
            tchain += bb - a;
            tdiv += c - bb;
        }
    }
    __syncwarp();
    long long t3 = clock64();
    for (int i = lane; i < n; i += 32) x[i] = xs[i];
    if (lane == 0) {
        stamps[0] = t1 - t0;
        stamps[1] = t2 - t1;
        stamps[2] = t3 - t2;
        stamps[3] = tchain;
        stamps[4] = tdiv;
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 143;
    std::vector<double> h(n * n + 2);
    for (int i = 0; i < n * n; ++i) h[i] = 0.001 * ((i * 7919) % 1000) / 1000.0;
    for (int i = 0; i < n; ++i) h[i * n + i] = 4.0 + i;
    double *m, *b, *x;
    long long* st;
    cudaMalloc(&m, sizeof(double) * (n * n + 2));
    cudaMalloc(&b, sizeof(double) * n);
    cudaMalloc(&x, sizeof(double) * n);
    cudaMalloc(&st, sizeof(long long) * 8);
    cudaMemcpy(m, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    std::vector<double> hb(n, 1.0);
    cudaMemcpy(b, hb.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(double) * (((n * n + 1) & ~1) + n + 16);
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<1, 32, smem>>>(n, m, b, x, st);
            else k<1><<<1, 32, smem>>>(n, m, b, x, st);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms_ = 0;
            cudaEventElapsedTime(&ms_, e0, e1);
            long long s[5];
            cudaMemcpy(s, st, sizeof(s), cudaMemcpyDeviceToHost);
            printf("mode %d n=%d: %.1f us; cycles load %lld fwd %lld bwd %lld (chain %lld, div %lld)\n", mode, n,
                   ms_ * 1e3, s[0], s[1], s[2], s[3], s[4]);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Exhaustive-ish check of the division used by k_lu_solve_mw's backward
// chain: with y = __drcp_rn(u) (correctly rounded 1/u), q = RN(s*y),
// r = fma(-u, q, s), x = fma(r, y, q) must equal RN(s/u) bit for bit when
// both s and u have biased exponents in [600, 1446] (kernels_core.cu
// mk_range).  Random (s, u) pairs over that whole range plus pairs built to
// sit near rounding boundaries (s = u * q' for q' a double, nudged by +-1..4
// ulp).  Prints the number of mismatches (expected 0).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/ubench_markstein.cu -o tools/ubench_markstein
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double mkd(uint64_t r, int elo, int ehi) {
    const uint64_t e = elo + (r >> 52) % (ehi - elo + 1);
    const uint64_t sign = (r >> 51) & 1;
    return __longlong_as_double(static_cast<long long>((sign << 63) | (e << 52) | (r & 0xfffffffffffffull)));
}
__global__ void k_check(uint64_t seed, int64_t n, unsigned long long* bad, int mode) {
    unsigned long long nb = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r1 = mix(seed ^ (2 * t)), r2 = mix(seed ^ (2 * t + 1));
        double u = mkd(r2, 600, 1446), s;
        if (mode == 0) {
            s = mkd(r1, 600, 1446);
        } else {
            // s near u * q' for a random double q' (products land near rounding boundaries)
            const double qq = mkd(r1, 1000, 1046);
            s = __dmul_rn(u, qq);
            const long long k = static_cast<long long>(r1 & 7) - 4;
            s = __longlong_as_double(__double_as_longlong(s) + k);
            const int e = (__double2hiint(s) >> 20) & 0x7ff;
            if (e < 600 || e > 1446) continue;
        }
        const double y = __drcp_rn(u);
        const double q = __dmul_rn(s, y);
        const double rr = __fma_rn(-u, q, s);
        const double x = __fma_rn(rr, y, q);
        if (__double_as_longlong(x) != __double_as_longlong(__ddiv_rn(s, u))) ++nb;
    }
    atomicAdd(bad, nb);
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(d, 0, 8);
        const int64_t n = int64_t{1} << 32;
        k_check<<<148 * 16, 256>>>(0x1234567ull + mode, n, d, mode);
        unsigned long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"mode\": \"%s\", \"pairs\": %lld, \"mismatches\": %llu}\n", mode ? "near-boundary" : "uniform", (long long)n, h);
    }
    return 0;
}

// Exact-order arithmetic helpers and the deterministic grid reduction shared
// by the row-pass and Krylov kernels.
#pragma once

#include "kernels.cuh"

namespace amgr {
namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Deterministic block -> grid reduction of NDOT partial sums.
template <int NDOT>
__device__ __forceinline__ void block_dots(double (&d)[NDOT], const DotSink& s) {
    __shared__ double ws[32][NDOT];
    __shared__ int last;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NDOT; ++k)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) d[k] = dadd(d[k], __shfl_down_sync(0xffffffffu, d[k], off));
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NDOT; ++k) ws[w][k] = d[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NDOT; ++k) {
            double t = 0.0;
            for (int i = 0; i < nw; ++i) t = dadd(t, ws[i][k]);
            s.partials[blockIdx.x * NDOT + k] = t;
        }
        __threadfence();
        const unsigned tk = atomicAdd(s.ticket, 1u);
        last = (tk == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (last && w == 0) {
        __threadfence();
#pragma unroll
        for (int k = 0; k < NDOT; ++k) {
            double t = 0.0;
            for (unsigned b = lane; b < gridDim.x; b += 32) t = dadd(t, __ldcg(&s.partials[b * NDOT + k]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) t = dadd(t, __shfl_down_sync(0xffffffffu, t, off));
            if (lane == 0) s.out[k] = t;
        }
        if (lane == 0) *s.ticket = 0u;
    }
}

}  // namespace
}  // namespace amgr

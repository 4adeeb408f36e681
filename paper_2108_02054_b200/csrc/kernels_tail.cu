// Persistent "tail" of the V-cycle: every level below a size threshold
// (C3: levels 4..13, 292K rows down to ~150) runs inside ONE cooperative
// kernel per leg, with grid-wide barriers between the phases instead of one
// launch per pass.  On those levels a pass moves a few hundred KB to a few
// tens of MB that sit in L2, so launch and tail-of-grid latency, not bytes,
// set the time (measured ~0.6 ms per V-cycle across levels 3..13 as separate
// launches, against ~20 us of L2 traffic).
//
// Arithmetic is the V-cycle's, bit for bit (same per-row sequential order):
//   down, level l:  r_i = f_i - sum_j a_ij u0_j                    (OpDown)
//                   fc_C = sum_{i in C, ascending} r_i;            (k_restrict)
//                   u0c_C = 0 + (om * wc_C) * fc_C
//   up, level l:    x_j = u0_j + (0 + e_{agg j})  on the fly       (k_prolong)
//                   out_i = x_i + (om * w_i) * (f_i - sum_j a_ij x_j) (OpSmooth)
// The up pass fuses prolongation into the smoothing sweep (x_j recomputed
// from u0, agg and the coarse iterate per gathered column), so it writes a
// separate output array.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "reduce.cuh"

namespace cg = cooperative_groups;

namespace amgr {

namespace {

constexpr int TL_BLOCK = 1024;  // one block per SM: a finished block's barrier spin (L1 invalidate per poll) cannot thrash a co-resident working block's L1
constexpr int TL_BATCH = 8;

__device__ __forceinline__ double dsub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul_(double a, double b) { return __dmul_rn(a, b); }

// sum_j a_ij x(j) in column order, TL_BATCH gathers in flight
template <class X>
__device__ __forceinline__ double row_sum(const TailLevel& L, int i, X x) {
    int k = __ldg(L.rp + i);
    const int ke = __ldg(L.rp + i + 1);
    double s = 0.0;
    while (k < ke) {
        const int cnt = min(TL_BATCH, ke - k);
        double xv[TL_BATCH], av[TL_BATCH];
#pragma unroll
        for (int t = 0; t < TL_BATCH; ++t) {
            xv[t] = t < cnt ? x(__ldg(L.col + k + t)) : 0.0;
            av[t] = t < cnt ? __ldg(L.val + k + t) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < TL_BATCH; ++t)
            if (t < cnt) s = dadd(s, dmul_(av[t], xv[t]));
        k += cnt;
    }
    return s;
}

// CL = false: cooperative grid (grid-wide barriers); CL = true: the grid is
// ONE thread-block cluster (hardware cluster barriers, all CTAs in one GPC)
template <bool CL>
struct TailSync {
    __device__ __forceinline__ void sync() {
        if constexpr (CL)
            cg::this_cluster().sync();
        else
            cg::this_grid().sync();
    }
};

// cluster variant: 16 CTAs of 512 threads (a 16-CTA cluster of 1024-thread
// CTAs does not fit a B200 GPC)
constexpr int TL_CBLOCK = 512;
template <bool CL>
__global__ void __launch_bounds__(CL ? TL_CBLOCK : TL_BLOCK) k_tail_down(TailDesc d, double om, Gate g) {
    if (CL) pdl_enter();
    if (gated_off(g)) return;
    TailSync<CL> grid;
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
    // unrolled: every descriptor access has a compile-time offset (a dynamic
    // index into the parameter bank costs a slow indexed constant load per
    // warp per level — 60% of this kernel's time when measured)
#pragma unroll
    for (int l = 0; l < TAIL_MAX; ++l) {
        if (l >= d.count) break;
        const TailLevel L = d.lv[l];
        const double* u0 = L.u0;
        for (int64_t i = tid; i < L.n; i += nt) {
            const double s = row_sum(L, static_cast<int>(i), [&](int j) { return __ldcg(u0 + j); });
            L.r[i] = dsub_(__ldcg(L.f + i), s);  // f of level > first was written by this kernel
        }
        grid.sync();
        for (int64_t I = tid; I < L.nc; I += nt) {
            int p = __ldg(L.mptr + I);
            const int p1 = __ldg(L.mptr + I + 1);
            double s = 0.0;
            while (p < p1) {
                const int cnt = min(4, p1 - p);
                double rv[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) rv[t] = t < cnt ? __ldcg(L.r + __ldg(L.midx + p + t)) : 0.0;
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (t < cnt) s = dadd(s, rv[t]);
                p += cnt;
            }
            L.fc[I] = s;
            if (L.u0c) L.u0c[I] = dadd(0.0, dmul_(dmul_(om, __ldg(L.wc + I)), s));
        }
        if (l + 1 < d.count) grid.sync();
    }
}

template <bool CL>
__global__ void __launch_bounds__(CL ? TL_CBLOCK : TL_BLOCK) k_tail_up(TailDesc d, double om, Gate g) {
    if (CL) pdl_enter();
    if (gated_off(g)) return;
    TailSync<CL> grid;
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
#pragma unroll
    for (int k = 0; k < TAIL_MAX; ++k) {
        const int l = TAIL_MAX - 1 - k;
        if (l >= d.count) continue;
        const TailLevel L = d.lv[l];
        const double* u0 = L.u0;
        const int* agg = L.agg;
        const double* ec = L.ec;
        auto x = [&](int j) { return dadd(__ldcg(u0 + j), dadd(0.0, __ldcg(ec + __ldg(agg + j)))); };
        for (int64_t i = tid; i < L.n; i += nt) {
            const int ii = static_cast<int>(i);
            const double s = row_sum(L, ii, x);
            const double xi = x(ii);
            L.uout[i] = dadd(xi, dmul_(dmul_(om, __ldg(L.w + i)), dsub_(__ldg(L.f + i), s)));
        }
        if (l > 0) grid.sync();
    }
}

// cluster size of the cluster-scoped tail (AMGR_TAIL_CLUSTER, 0: cooperative grid)
int tail_cluster() {
    const char* e = std::getenv("AMGR_TAIL_CLUSTER");
    return e ? std::atoi(e) : 0;
}

template <class K>
void launch_coop(Ctx& c, const char* fam, K kernel, const TailDesc& d, double om, Gate g) {
    // enough threads for the largest tail level, at most one full wave
    int64_t nmax = 0;
    for (int l = 0; l < d.count; ++l) nmax = d.lv[l].n > nmax ? d.lv[l].n : nmax;
    int64_t blocks = (nmax + TL_BLOCK - 1) / TL_BLOCK;
    int64_t cap = static_cast<int64_t>(c.num_sms);  // one block per SM (see TL_BLOCK)
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    TailDesc dd = d;
    double omv = om;
    Gate gg = g;
    void* args[] = {&dd, &omv, &gg};
    probe_begin(c, fam, 0.0);
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(static_cast<unsigned>(blocks)),
                                   dim3(TL_BLOCK), args, 0, c.stream));
    probe_end(c, fam);
    ++c.launches;
}

template <class K>
void launch_cluster(Ctx& c, const char* fam, K kernel, const TailDesc& d, double om, Gate g, int cs) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(cs));
    cfg.blockDim = dim3(TL_CBLOCK);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = c.pdl ? 2 : 1;
    probe_begin(c, fam, 0.0);
    CK(cudaLaunchKernelEx(&cfg, kernel, d, om, g));
    probe_end(c, fam);
    ++c.launches;
}

}  // namespace

void tail_down(Ctx& c, const TailDesc& d, double om, Gate g) {
    if (d.count == 0) return;
    if (const int cs = tail_cluster())
        launch_cluster(c, "vcycle_tail", k_tail_down<true>, d, om, g, cs);
    else
        launch_coop(c, "vcycle_tail", k_tail_down<false>, d, om, g);
}

void tail_up(Ctx& c, const TailDesc& d, double om, Gate g) {
    if (d.count == 0) return;
    if (const int cs = tail_cluster())
        launch_cluster(c, "vcycle_tail", k_tail_up<true>, d, om, g, cs);
    else
        launch_coop(c, "vcycle_tail", k_tail_up<false>, d, om, g);
}

}  // namespace amgr

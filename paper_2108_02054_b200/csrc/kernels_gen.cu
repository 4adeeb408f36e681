// On-device synthetic problem sequences:
// g^3 7-point operators -div(c grad u) (+ shift, + upwind convection) with
// harmonic face averaging and homogeneous Dirichlet walls, lifted from the
// reference's 2D generator (proj/src/diffusion.cpp:54-118) to 3D.  Every
// arithmetic step uses explicit round-to-nearest intrinsics in the order the
// host restatement (oracle/amg_oracle.c) uses, so the Poisson and dam-break
// values are bit-identical to the host generator.  (The blob uses exp(),
// whose last bit may differ between CUDA and glibc; parity runs upload the
// host matrix instead.)
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "hierarchy.cuh"

namespace amgr {

namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

struct GenParams {
    int kind;
    int g;
    double inv_h2;
    double shift;        // POISSON
    double cx, cy, cz;   // BLOB centre (grid units)
    double contrast, inv_sigma2;
    double a_k, b_k;     // DAMBREAK water column x < a_k, z < b_k
    double bx, by, bz;   // CONVDIFF velocity (already divided by h)
};

__device__ __forceinline__ double node_coef(const GenParams& p, int x, int y, int z) {
    switch (p.kind) {
        case AMGR_PROBLEM_BLOB:
        case AMGR_PROBLEM_CONVDIFF: {
            const double dx = static_cast<double>(x) - p.cx;
            const double dy = static_cast<double>(y) - p.cy;
            const double dz = static_cast<double>(z) - p.cz;
            const double r2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
            return dadd(1.0, dmul(p.contrast - 1.0, exp(-dmul(r2, p.inv_sigma2))));
        }
        case AMGR_PROBLEM_DAMBREAK: {
            const bool water = static_cast<double>(x) < p.a_k && static_cast<double>(z) < p.b_k;
            return water ? ddiv(1.0, 1000.0) : 1.0;
        }
        default:
            return 1.0;
    }
}

// harmonic mean 2ab/(a+b) evaluated as ((2a)b)/(a+b) (diffusion.cpp:73)
__device__ __forceinline__ double harm(double a, double b) { return ddiv(dmul(dmul(2.0, a), b), dadd(a, b)); }

__global__ void k_pattern_count(int g, int* cnt) {
    const int64_t n = static_cast<int64_t>(g) * g * g;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % g), y = static_cast<int>((i / g) % g), z = static_cast<int>(i / (static_cast<int64_t>(g) * g));
        cnt[i] = 1 + (z > 0) + (y > 0) + (x > 0) + (x < g - 1) + (y < g - 1) + (z < g - 1);
    }
}

__global__ void k_pattern_fill(int g, const int* rp, int* col) {
    const int64_t n = static_cast<int64_t>(g) * g * g;
    const int64_t g2 = static_cast<int64_t>(g) * g;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % g), y = static_cast<int>((i / g) % g), z = static_cast<int>(i / g2);
        int k = rp[i];
        if (z > 0) col[k++] = static_cast<int>(i - g2);
        if (y > 0) col[k++] = static_cast<int>(i - g);
        if (x > 0) col[k++] = static_cast<int>(i - 1);
        col[k++] = static_cast<int>(i);
        if (x < g - 1) col[k++] = static_cast<int>(i + 1);
        if (y < g - 1) col[k++] = static_cast<int>(i + g);
        if (z < g - 1) col[k++] = static_cast<int>(i + g2);
    }
}

__global__ void k_values(GenParams p, const int* rp, double* val) {
    const int g = p.g;
    const int64_t n = static_cast<int64_t>(g) * g * g;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % g), y = static_cast<int>((i / g) % g), z = static_cast<int>(i / (static_cast<int64_t>(g) * g));
        const double k0 = node_coef(p, x, y, z);
        const double zlo = z > 0 ? harm(k0, node_coef(p, x, y, z - 1)) : k0;
        const double ylo = y > 0 ? harm(k0, node_coef(p, x, y - 1, z)) : k0;
        const double xlo = x > 0 ? harm(k0, node_coef(p, x - 1, y, z)) : k0;
        const double xhi = x < g - 1 ? harm(k0, node_coef(p, x + 1, y, z)) : k0;
        const double yhi = y < g - 1 ? harm(k0, node_coef(p, x, y + 1, z)) : k0;
        const double zhi = z < g - 1 ? harm(k0, node_coef(p, x, y, z + 1)) : k0;
        double dg = dmul(dadd(dadd(dadd(dadd(dadd(zlo, ylo), xlo), xhi), yhi), zhi), p.inv_h2);
        double czlo = 0, cylo = 0, cxlo = 0, cxhi = 0, cyhi = 0, czhi = 0;
        if (p.kind == AMGR_PROBLEM_CONVDIFF) {
            // first-order upwind b . grad u: +|b_d|/h on the diagonal, -|b_d|/h on
            // the upstream neighbour of each direction d
            const double ax = fabs(p.bx), ay = fabs(p.by), az = fabs(p.bz);
            dg = dadd(dg, dadd(dadd(ax, ay), az));
            if (p.bx > 0) cxlo = ax; else cxhi = ax;
            if (p.by > 0) cylo = ay; else cyhi = ay;
            if (p.bz > 0) czlo = az; else czhi = az;
        }
        if (p.kind == AMGR_PROBLEM_POISSON) dg = dadd(dg, p.shift);
        int k = rp[i];
        if (z > 0) val[k++] = -dadd(dmul(zlo, p.inv_h2), czlo);
        if (y > 0) val[k++] = -dadd(dmul(ylo, p.inv_h2), cylo);
        if (x > 0) val[k++] = -dadd(dmul(xlo, p.inv_h2), cxlo);
        val[k++] = dg;
        if (x < g - 1) val[k++] = -dadd(dmul(xhi, p.inv_h2), cxhi);
        if (y < g - 1) val[k++] = -dadd(dmul(yhi, p.inv_h2), cyhi);
        if (z < g - 1) val[k++] = -dadd(dmul(zhi, p.inv_h2), czhi);
    }
}

}  // namespace

void exclusive_sum_i32(Ctx& c, const int* in, int* out, int64_t n) {
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c.stream));
    DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
    CK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, c.stream));
    ++c.launches;
}

int64_t problem_nnz(int64_t g) { return 7 * g * g * g - 6 * g * g; }

void problem_pattern(Ctx& c, int64_t g, int* rp, int* col) {
    const int64_t n = g * g * g;
    DevArray<int> cnt(n + 1, c.stream);
    CK(cudaMemsetAsync(cnt.get() + n, 0, sizeof(int), c.stream));
    LAUNCH(c, "gen", 0.0, k_pattern_count, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(g), cnt.get());
    exclusive_sum_i32(c, cnt.get(), rp, n + 1);
    LAUNCH(c, "gen", 0.0, k_pattern_fill, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(g), rp, col);
}

// Host-side parameter derivation shared with oracle/amg_oracle.c
// (gen_params); see DESIGN.md §5 for the formulas.
void problem_values(Ctx& c, int kind, int64_t g, int64_t k, int64_t nsteps, double* val) {
    GenParams p{};
    p.kind = kind;
    p.g = static_cast<int>(g);
    const double h = 1.0 / static_cast<double>(g + 1);
    p.inv_h2 = 1.0 / (h * h);
    const double den = static_cast<double>(nsteps > 1 ? nsteps - 1 : 1);
    const double gd = static_cast<double>(g);
    switch (kind) {
        case AMGR_PROBLEM_POISSON:
            p.shift = 0.01 * static_cast<double>(k + 1) * (6.0 * p.inv_h2);
            break;
        case AMGR_PROBLEM_BLOB:
        case AMGR_PROBLEM_CONVDIFF: {
            p.contrast = 10.0;
            const double sigma = 0.2 * gd;
            p.inv_sigma2 = 1.0 / (sigma * sigma);
            const double limit = gd - 1.0;
            const double travel = static_cast<double>(k) * 0.25 / std::sqrt(3.0);
            double pos = std::fmod(travel, 2.0 * limit);
            if (pos > limit) pos = 2.0 * limit - pos;
            p.cx = p.cy = p.cz = pos;
            if (kind == AMGR_PROBLEM_CONVDIFF) {
                // rotating velocity, cell Peclet ~ 10: |b| h / kappa_min = 10
                const double th = 2.0 * M_PI * static_cast<double>(k) / den;
                const double speed = 10.0 / h;
                p.bx = speed * std::cos(th) / h;
                p.by = speed * std::sin(th) / h;
                p.bz = 0.5 * speed / h;
            }
            break;
        }
        case AMGR_PROBLEM_DAMBREAK:
            p.a_k = gd * (0.25 + 0.5 * static_cast<double>(k) / den);
            p.b_k = gd * (0.5 - 0.25 * static_cast<double>(k) / den);
            break;
        default:
            invalid("amgr_problem_values: unknown problem kind");
    }
    DevArray<int> rp(g * g * g + 1, c.stream);
    DevArray<int> cnt(g * g * g + 1, c.stream);
    const int64_t n = g * g * g;
    CK(cudaMemsetAsync(cnt.get() + n, 0, sizeof(int), c.stream));
    LAUNCH(c, "gen", 0.0, k_pattern_count, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(g), cnt.get());
    exclusive_sum_i32(c, cnt.get(), rp.get(), n + 1);
    LAUNCH(c, "gen", 0.0, k_values, grid_for(n, 256, c.num_sms * 16), 256, 0, p, rp.get(), val);
}

}  // namespace amgr

// Krylov kernels (sm_100a): fused vector updates + deterministic dots, and the
// one-thread scalar kernels that replay bicgstab.cpp's control flow on device.
#include <cuda_runtime.h>

#include "krylov.cuh"
#include "reduce.cuh"

namespace amgr {

namespace {

constexpr int VB = 256;

__device__ __forceinline__ int& flags_of(KState* s) { return s->flags; }

__device__ __forceinline__ double rel(const KState* s, double sq) { return sqrt(sq) / s->normf; }

// ---- BiCGStab scalar kernels ------------------------------------------------
__global__ void k_bicg_begin(KState* s) {
    pdl_enter();
    int f = s->flags;
    if (f & KF_DONE) return;
    if (s->it >= s->max_iter) {
        s->flags = f | KF_DONE;
        return;
    }
    s->it += 1;
    f &= ~(KF_HALF | KF_CHECK);
    const double rho = s->d_rtr;  // rho = dot(rtilde, r)
    s->rho = rho;
    if (fabs(rho) < s->floor) {
        s->flags = f | KF_BREAKDOWN | KF_DONE;
        return;
    }
    if (s->it > 1) s->beta = __dmul_rn(__ddiv_rn(rho, s->rho_old), __ddiv_rn(s->alpha, s->omega));
    s->flags = f;
}

__global__ void k_bicg_alpha(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & KF_DONE) return;
    const double rtv = s->d_rtv;
    if (fabs(rtv) < s->floor) {
        s->flags = f | KF_BREAKDOWN | KF_DONE;
        return;
    }
    s->alpha = __ddiv_rn(s->rho, rtv);
}

__global__ void k_bicg_half_test(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & KF_DONE) return;
    if (rel(s, s->d_ss) <= s->tol) s->flags = f | KF_HALF;
}

__global__ void k_bicg_half_check(KState* s) {
    pdl_enter();
    int f = s->flags;
    if ((f & KF_DONE) || !(f & KF_HALF)) return;
    const double res = rel(s, s->d_true);
    if (res <= s->tol) {
        s->res = res;
        s->flags = f | KF_CONVERGED | KF_DONE;
        return;
    }
    s->rho_old = s->rho;
    if (s->it >= s->max_iter) f |= KF_DONE;
    s->flags = f;
}

__global__ void k_bicg_omega(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & (KF_DONE | KF_HALF)) return;
    const double tt = s->d_tt;
    if (tt == 0.0) {
        s->flags = f | KF_BREAKDOWN | KF_DONE;
        return;
    }
    s->omega = __ddiv_rn(s->d_ts, tt);
}

__global__ void k_bicg_end_test(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & (KF_DONE | KF_HALF)) return;
    s->rho_old = s->rho;
    if (rel(s, s->d_rr) <= s->tol) s->flags = f | KF_CHECK;
}

__global__ void k_bicg_end_check(KState* s) {
    pdl_enter();
    int f = s->flags;
    if (f & (KF_DONE | KF_HALF)) return;
    if (f & KF_CHECK) {
        const double res = rel(s, s->d_true);
        if (res <= s->tol) {
            s->res = res;
            s->flags = f | KF_CONVERGED | KF_DONE;
            return;
        }
    }
    if (fabs(s->omega) < 1e-30) f |= KF_BREAKDOWN | KF_DONE;
    if (s->it >= s->max_iter) f |= KF_DONE;
    s->flags = f;
}

// ---- BiCGStab vector kernels --------------------------------------------------
__global__ void k_bicg_p(const KState* s, int n, const double* __restrict__ r, double* __restrict__ p,
                         const double* __restrict__ v) {
    pdl_enter();
    if (s->flags & KF_DONE) return;
    const bool first = s->it == 1;
    const double beta = s->beta, om = s->omega;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        p[i] = first ? r[i] : dadd(r[i], dmul(beta, dsub(p[i], dmul(om, v[i]))));
}

__global__ void __launch_bounds__(VB) k_bicg_s(const KState* s, int n, const double* __restrict__ r,
                                               const double* __restrict__ v, double* __restrict__ sv,
                                               DotSink ds) {
    pdl_enter();
    if (s->flags & KF_DONE) return;
    const double alpha = s->alpha;
    double d[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double t = dsub(r[i], dmul(alpha, v[i]));
        sv[i] = t;
        d[0] = dadd(d[0], dmul(t, t));
    }
    block_dots<1>(d, ds);
}

__global__ void k_bicg_half_u(const KState* s, int n, double* __restrict__ u, const double* __restrict__ ph) {
    pdl_enter();
    const int f = s->flags;
    if ((f & KF_DONE) || !(f & KF_HALF)) return;
    const double alpha = s->alpha;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        u[i] = dadd(u[i], dmul(alpha, ph[i]));
}

// half-step continue (bicgstab.cpp:98-99): r = s, and the next iteration's
// rho = dot(rtilde, r) (bicgstab.cpp:68) from the new r
__global__ void __launch_bounds__(VB) k_bicg_half_r(const KState* s, int n, double* __restrict__ r,
                                                    const double* __restrict__ sv, const double* __restrict__ rt,
                                                    DotSink ds) {
    pdl_enter();
    const int f = s->flags;
    if ((f & KF_DONE) || !(f & KF_HALF)) return;
    double d[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double si = sv[i];
        r[i] = si;
        d[0] = dadd(d[0], dmul(rt[i], si));
    }
    block_dots<1>(d, ds);
}

__global__ void __launch_bounds__(VB) k_bicg_update(const KState* s, int n, double* __restrict__ u,
                                                    const double* __restrict__ ph,
                                                    const double* __restrict__ sh, double* __restrict__ r,
                                                    const double* __restrict__ sv,
                                                    const double* __restrict__ t,
                                                    const double* __restrict__ rt, DotSink ds) {
    pdl_enter();
    if (s->flags & (KF_DONE | KF_HALF)) return;
    const double alpha = s->alpha, om = s->omega;
    double d[2] = {0.0, 0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        u[i] = dadd(u[i], dadd(dmul(alpha, ph[i]), dmul(om, sh[i])));
        const double ri = dsub(sv[i], dmul(om, t[i]));
        r[i] = ri;
        d[0] = dadd(d[0], dmul(ri, ri));
        d[1] = dadd(d[1], dmul(rt[i], ri));
    }
    block_dots<2>(d, ds);
}

// ---- CG ------------------------------------------------------------------------
__global__ void k_cg_begin(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & KF_DONE) return;
    if (s->it >= s->max_iter) {
        s->flags = f | KF_DONE;
        return;
    }
    s->it += 1;
    s->flags = f & ~KF_CHECK;
}
__global__ void k_cg_alpha(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & KF_DONE) return;
    const double pq = s->d_pq;
    if (fabs(pq) < s->floor || fabs(s->rho) < s->floor) {
        s->flags = f | KF_BREAKDOWN | KF_DONE;
        return;
    }
    s->alpha = __ddiv_rn(s->rho, pq);
}
__global__ void __launch_bounds__(VB) k_cg_update(const KState* s, int n, double* __restrict__ u,
                                                  double* __restrict__ r, const double* __restrict__ p,
                                                  const double* __restrict__ q, DotSink ds) {
    pdl_enter();
    if (s->flags & KF_DONE) return;
    const double a = s->alpha;
    double d[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        u[i] = dadd(u[i], dmul(a, p[i]));
        const double ri = dsub(r[i], dmul(a, q[i]));
        r[i] = ri;
        d[0] = dadd(d[0], dmul(ri, ri));
    }
    block_dots<1>(d, ds);
}
__global__ void k_cg_test(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & KF_DONE) return;
    if (rel(s, s->d_rr) <= s->tol) s->flags = f | KF_CHECK;
}
__global__ void k_cg_check(KState* s) {
    pdl_enter();
    int f = s->flags;
    if (f & KF_DONE) return;
    if (f & KF_CHECK) {
        const double res = rel(s, s->d_true);
        if (res <= s->tol) {
            s->res = res;
            s->flags = f | KF_CONVERGED | KF_DONE;
            return;
        }
    }
    if (s->it >= s->max_iter) f |= KF_DONE;
    s->flags = f;
}
__global__ void k_cg_beta(KState* s) {
    pdl_enter();
    const int f = s->flags;
    if (f & KF_DONE) return;
    const double rz = s->d_rz;
    s->beta = __ddiv_rn(rz, s->rho);
    s->rho = rz;
}
__global__ void k_cg_p(const KState* s, int n, const double* __restrict__ z, double* __restrict__ p) {
    pdl_enter();
    if (s->flags & KF_DONE) return;
    const double b = s->beta;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        p[i] = dadd(z[i], dmul(b, p[i]));
}

__global__ void __launch_bounds__(VB) k_dot(int n, const double* __restrict__ a, const double* __restrict__ b,
                                            DotSink ds, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    double d[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        d[0] = dadd(d[0], dmul(a[i], b[i]));
    block_dots<1>(d, ds);
}

constexpr int SD_THREADS = 256, SD_CH = 2048;

__global__ void __launch_bounds__(SD_THREADS) k_seq_dot(int64_t n, const double* __restrict__ a,
                                                        const double* __restrict__ b, double* out, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    __shared__ __align__(16) double buf[2][SD_CH + 8];
    const int tid = threadIdx.x;
    const int64_t nch = (n + SD_CH - 1) / SD_CH;
    auto fill = [&](int64_t ch, double* dst, int t0, int nt) {
        const int64_t base = ch * SD_CH;
        const int len = static_cast<int>(n - base < SD_CH ? n - base : SD_CH);
        for (int i = t0; i < len; i += nt) dst[i] = dmul(__ldg(a + base + i), __ldg(b + base + i));
        for (int i = len + t0; i < SD_CH + 8; i += nt) dst[i] = 0.0;
    };
    if (nch > 0) fill(0, buf[0], tid, SD_THREADS);
    __syncthreads();
    double s = 0.0;
    for (int64_t ch = 0; ch < nch; ++ch) {
        if (tid >= 32) {
            if (ch + 1 < nch) fill(ch + 1, buf[(ch + 1) & 1], tid - 32, SD_THREADS - 32);
        } else if (tid == 0) {
            const int64_t base = ch * SD_CH;
            const int len = static_cast<int>(n - base < SD_CH ? n - base : SD_CH);
            const double* p = buf[ch & 1];
            // s += p[i] for i < len, in order; 8-entry chunks read one chunk ahead
            int i = 0;
            double q[8], r[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) q[t] = p[t];
            for (; i + 16 <= len; i += 16) {
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    r[t] = p[i + 8 + t];
                    s = dadd(s, q[t]);
                }
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    q[t] = p[i + 16 + t];
                    s = dadd(s, r[t]);
                }
            }
            for (; i < len; ++i) s = dadd(s, p[i]);
        }
        __syncthreads();
    }
    if (tid == 0) *out = s;
}

}  // namespace

void seq_dot(Ctx& c, int64_t n, const double* a, const double* b, double* out, Gate g) {
    LAUNCH_PDL(c, "seq_dot", 16.0 * n, k_seq_dot, 1, SD_THREADS, 0, n, a, b, out, g);
}

Gate gate_of(const KState* st, int skip, int need) { return Gate{&st->flags, skip, need}; }

#define SCALAR(c, k, st) LAUNCH_PDL(c, "krylov_scalar", 0.0, k, 1, 1, 0, st)

void bicg_begin(Ctx& c, KState* st) { SCALAR(c, k_bicg_begin, st); }
void bicg_alpha(Ctx& c, KState* st) { SCALAR(c, k_bicg_alpha, st); }
void bicg_half_test(Ctx& c, KState* st) { SCALAR(c, k_bicg_half_test, st); }
void bicg_half_check(Ctx& c, KState* st) { SCALAR(c, k_bicg_half_check, st); }
void bicg_omega(Ctx& c, KState* st) { SCALAR(c, k_bicg_omega, st); }
void bicg_end_test(Ctx& c, KState* st) { SCALAR(c, k_bicg_end_test, st); }
void bicg_end_check(Ctx& c, KState* st) { SCALAR(c, k_bicg_end_check, st); }

void bicg_p(Ctx& c, KState* st, int64_t n, const double* r, double* p, const double* v) {
    LAUNCH_PDL(c, "krylov_vec", 32.0 * n, k_bicg_p, grid_for(n, VB, c.num_sms * 8), VB, 0, st, static_cast<int>(n), r,
           p, v);
}
void bicg_s(Ctx& c, KState* st, int64_t n, const double* r, const double* v, double* s, DotSink ds) {
    LAUNCH_PDL(c, "krylov_vec", 24.0 * n, k_bicg_s, dot_grid(c), VB, 0, st, static_cast<int>(n), r, v, s, ds);
}
void bicg_half_u(Ctx& c, KState* st, int64_t n, double* u, const double* phat) {
    LAUNCH_PDL(c, "krylov_vec", 24.0 * n, k_bicg_half_u, grid_for(n, VB, c.num_sms * 8), VB, 0, st,
           static_cast<int>(n), u, phat);
}
void bicg_half_r(Ctx& c, KState* st, int64_t n, double* r, const double* s, const double* rt, DotSink ds) {
    LAUNCH_PDL(c, "krylov_vec", 24.0 * n, k_bicg_half_r, dot_grid(c), VB, 0, st, static_cast<int>(n), r, s, rt, ds);
}
void bicg_update(Ctx& c, KState* st, int64_t n, double* u, const double* phat, const double* shat, double* r,
                 const double* s, const double* t, const double* rt, DotSink ds) {
    LAUNCH_PDL(c, "krylov_vec", 64.0 * n, k_bicg_update, dot_grid(c), VB, 0, st, static_cast<int>(n), u, phat, shat,
           r, s, t, rt, ds);
}

void cg_begin(Ctx& c, KState* st) { SCALAR(c, k_cg_begin, st); }
void cg_alpha(Ctx& c, KState* st) { SCALAR(c, k_cg_alpha, st); }
void cg_test(Ctx& c, KState* st) { SCALAR(c, k_cg_test, st); }
void cg_check(Ctx& c, KState* st) { SCALAR(c, k_cg_check, st); }
void cg_beta(Ctx& c, KState* st) { SCALAR(c, k_cg_beta, st); }
void cg_update(Ctx& c, KState* st, int64_t n, double* u, double* r, const double* p, const double* q,
               DotSink ds) {
    LAUNCH_PDL(c, "krylov_vec", 48.0 * n, k_cg_update, dot_grid(c), VB, 0, st, static_cast<int>(n), u, r, p, q, ds);
}
void cg_p(Ctx& c, KState* st, int64_t n, const double* z, double* p) {
    LAUNCH_PDL(c, "krylov_vec", 24.0 * n, k_cg_p, grid_for(n, VB, c.num_sms * 8), VB, 0, st, static_cast<int>(n), z,
           p);
}

void dot(Ctx& c, int64_t n, const double* a, const double* b, DotSink ds, Gate g) {
    LAUNCH_PDL(c, "krylov_vec", 16.0 * n, k_dot, dot_grid(c), VB, 0, static_cast<int>(n), a, b, ds, g);
}

}  // namespace amgr

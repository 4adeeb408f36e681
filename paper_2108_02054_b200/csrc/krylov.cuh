// Device-resident Krylov state and the vector / scalar kernels of the
// right-preconditioned BiCGStab (proj/src/bicgstab.cpp:21-135) and the
// preconditioned CG extension.  Every decision the reference takes on the host
// (breakdown thresholds, half-step exit, true-residual confirmation) is taken by
// a one-thread scalar kernel that sets flags; all other kernels are gated on
// those flags, so whole iterations are enqueued without host round trips.
#pragma once

#include "kernels.cuh"

namespace amgr {

struct KState {
    // inputs
    double normf = 0, floor = 0, tol = 0;
    int64_t max_iter = 0;
    // scalars
    double rho = 0, rho_old = 1, alpha = 1, omega = 1, beta = 0, res = 0;
    int64_t it = 0;
    int flags = 0;
    int pad = 0;
    // dot outputs (written by fused kernels)
    double d_rr = 0, d_rtr = 0, d_rtv = 0, d_ss = 0, d_ts = 0, d_tt = 0, d_true = 0;
    double d_pq = 0, d_rz = 0;
};

// ---- BiCGStab phases (bicgstab.cpp line numbers) ----
void bicg_begin(Ctx& c, KState* st);                                   // :67-73
void bicg_p(Ctx& c, KState* st, int64_t n, const double* r, double* p, const double* v);  // :74-79
void bicg_alpha(Ctx& c, KState* st);                                   // :82-88
void bicg_s(Ctx& c, KState* st, int64_t n, const double* r, const double* v, double* s,
            DotSink ds);                                               // :89
void bicg_half_test(Ctx& c, KState* st);                               // :91
void bicg_half_u(Ctx& c, KState* st, int64_t n, double* u, const double* phat);  // :92
void bicg_half_check(Ctx& c, KState* st);                              // :93-100
// r = s and rho_next = dot(rtilde, r) into ds (bicgstab.cpp:98, :68)
void bicg_half_r(Ctx& c, KState* st, int64_t n, double* r, const double* s, const double* rt, DotSink ds);
void bicg_omega(Ctx& c, KState* st);                                   // :106-111
void bicg_update(Ctx& c, KState* st, int64_t n, double* u, const double* phat, const double* shat,
                 double* r, const double* s, const double* t, const double* rt,
                 DotSink ds);                                          // :112-115
void bicg_end_test(Ctx& c, KState* st);                                // :116-118
void bicg_end_check(Ctx& c, KState* st);                               // :119-129

// ---- preconditioned CG (extension) ----
void cg_begin(Ctx& c, KState* st);
void cg_alpha(Ctx& c, KState* st);
void cg_update(Ctx& c, KState* st, int64_t n, double* u, double* r, const double* p, const double* q,
               DotSink ds);
void cg_test(Ctx& c, KState* st);
void cg_check(Ctx& c, KState* st);
void cg_beta(Ctx& c, KState* st);
void cg_p(Ctx& c, KState* st, int64_t n, const double* z, double* p);

// plain deterministic dot (fixed grid): out[0] = a . b
void dot(Ctx& c, int64_t n, const double* a, const double* b, DotSink ds, Gate g = {});

Gate gate_of(const KState* st, int skip, int need = 0);

// *out = sum_i a[i]*b[i] accumulated strictly left to right from 0.0, each
// product rounded before the add: the reference's dot (bicgstab.cpp:11-15)
// bit for bit.  One CTA; the products of the next chunk are formed by the
// other warps while one thread runs the dependent add chain.
void seq_dot(Ctx& c, int64_t n, const double* a, const double* b, double* out, Gate g = {});

}  // namespace amgr

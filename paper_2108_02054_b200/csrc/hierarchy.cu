// Host orchestration of the device AMG hierarchy.  Each function cites the
// reference function whose semantics (order of phases, error texts, timing
// buckets) it reproduces.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <cstring>
#include <sstream>

#include "hierarchy.cuh"

namespace amgr {

AmgP to_amgp(const amgr_amg_params* p) {
    AmgP a;
    if (!p) return a;
    a.eps = p->eps;
    a.omega = p->omega;
    a.pre = p->pre_sweeps;
    a.post = p->post_sweeps;
    a.coarse_enough = p->coarse_enough;
    a.max_direct = p->max_direct_size;
    a.smoother = p->smoother;
    a.coarsening = p->coarsening;
    a.sa_omega = p->sa_omega;
    a.cheb_degree = p->cheb_degree;
    a.power_iters = p->power_iters;
    a.cheb_lower = p->cheb_lower;
    a.cheb_safety = p->cheb_safety;
    a.coarse_solve = p->coarse_solve;
    return a;
}

namespace {

// ---- phase timers (SetupPhaseTimings, hierarchy.cpp:17-29) -------------------
enum Phase { PH_TRANSFER = 0, PH_GALERKIN = 1, PH_SMOOTHER = 2, PH_COARSE = 3 };

struct PhaseClock {
    Ctx& c;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[4];
    size_t base;
    explicit PhaseClock(Ctx& cc) : c(cc), base(cc.clock_used) {}
    ~PhaseClock() { c.clock_used = base; }  // events return to the context's pool
    cudaEvent_t take() {
        if (c.clock_used == c.clock_pool.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            c.clock_pool.push_back(e);
        }
        return c.clock_pool[c.clock_used++];
    }
    void begin(Phase ph) {
        cudaEvent_t a = take(), b = take();
        CK(cudaEventRecord(a, c.stream));
        ev[ph].push_back({a, b});
    }
    void end(Phase ph) { CK(cudaEventRecord(ev[ph].back().second, c.stream)); }
    // requires the stream to have passed the last event
    amgr_phase_timings collect() {
        CK(cudaStreamSynchronize(c.stream));
        double t[4] = {0, 0, 0, 0};
        for (int k = 0; k < 4; ++k)
            for (auto& p : ev[k]) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, p.first, p.second));
                t[k] += ms * 1e-3;
            }
        return amgr_phase_timings{t[0], t[1], t[2], t[3]};
    }
};

std::string level_prefix(size_t l) {
    std::ostringstream os;
    os << "level " << l << ": ";
    return os.str();
}

// Upload / adopt an amgr_csr pattern into int32 device arrays.
std::shared_ptr<Pattern> make_pattern(Ctx& c, const amgr_csr& A) {
    auto P = std::make_shared<Pattern>();
    P->n = A.nrows;
    P->ncols = A.ncols;
    P->nnz = A.nnz;
    if (A.nnz > INT32_MAX - 1 || A.nrows > INT32_MAX - 1 || A.ncols > INT32_MAX - 1)
        invalid("matrix too large for int32 device indices (> 2^31 entries per GPU)");
    P->rp.alloc(A.nrows + 1, c.stream);
    P->col.alloc(A.nnz, c.stream);
    const bool dev = A.location == AMGR_DEVICE;
    auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (A.index_bits == 32) {
        CK(cudaMemcpyAsync(P->rp.get(), A.row_ptr, sizeof(int) * (A.nrows + 1), kind, c.stream));
        if (A.nnz) CK(cudaMemcpyAsync(P->col.get(), A.col_idx, sizeof(int) * A.nnz, kind, c.stream));
    } else if (A.index_bits == 64) {
        DevArray<int> ovf(1, c.stream);
        CK(cudaMemsetAsync(ovf.get(), 0, sizeof(int), c.stream));
        DevArray<int64_t> tmp(std::max<int64_t>(A.nrows + 1, A.nnz), c.stream);
        CK(cudaMemcpyAsync(tmp.get(), A.row_ptr, sizeof(int64_t) * (A.nrows + 1), kind, c.stream));
        i64_to_i32(c, tmp.get(), P->rp.get(), A.nrows + 1, ovf.get());
        if (A.nnz) {
            CK(cudaMemcpyAsync(tmp.get(), A.col_idx, sizeof(int64_t) * A.nnz, kind, c.stream));
            i64_to_i32(c, tmp.get(), P->col.get(), A.nnz, ovf.get());
        }
        if (d2h_scalar(ovf.get(), c.stream)) invalid("index out of int32 range");
    } else {
        invalid("amgr_csr.index_bits must be 32 or 64");
    }
    P->diag.alloc(A.nrows, c.stream);
    CsrView v;
    v.n = P->n;
    v.ncols = P->ncols;
    v.nnz = P->nnz;
    v.rp = P->rp.get();
    v.col = P->col.get();
    find_diag(c, v, P->diag.get());
    P->max_span = max_group_span(c, P->rp.get(), P->n);
    return P;
}

void upload_values(Ctx& c, DevArray<double>& dst, const double* src, int64_t nnz, int location) {
    if (dst.size() != nnz) dst.alloc(nnz, c.stream);
    if (nnz == 0) return;
    CK(cudaMemcpyAsync(dst.get(), src, sizeof(double) * nnz,
                       location == AMGR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
}

bool same_pattern(Ctx& c, const Pattern& a, const Pattern& b) {
    if (a.n != b.n || a.ncols != b.ncols || a.nnz != b.nnz) return false;
    DevArray<int> diff(1, c.stream);
    CK(cudaMemsetAsync(diff.get(), 0, sizeof(int), c.stream));
    compare_i32(c, a.rp.get(), b.rp.get(), a.n + 1, diff.get());
    compare_i32(c, a.col.get(), b.col.get(), a.nnz, diff.get());
    return d2h_scalar(diff.get(), c.stream) == 0;
}

// Smoother rebuild of level l (build_smoother, smoother.cpp:8-32; SPAI0 and
// Chebyshev extensions).  Chebyshev: Jacobi weights + power iteration for
// lambda_max(D^-1 A) from the all-ones vector + coefficient table
// (oracle/amg_oracle.c power_lambda / smooth_cheb).
void build_smoother(Ctx& c, Level& L, const AmgP& p, int* bad) {
    const int64_t n = L.pat->n;
    if (L.w.size() != n) L.w.alloc(n, c.stream);
    if (p.smoother == AMGR_SMOOTHER_SPAI0)
        spai0_rebuild(c, L.view(), L.pat->diag.get(), L.w.get(), bad);
    else
        jacobi_rebuild(c, n, L.view().val, L.pat->diag.get(), L.w.get(), bad);
    L.has_smoother = true;
    if (p.smoother == AMGR_SMOOTHER_CHEBYSHEV) {
        if (p.cheb_degree < 1 || p.cheb_degree > 32) invalid("chebyshev: degree must be in [1, 32]");
        const CsrView A = L.view();
        DevArray<double> x(n, c.stream), y(n, c.stream), partials(static_cast<int64_t>(dot_grid(c)) * 2 + 8, c.stream);
        DevArray<unsigned> ticket(1, c.stream);
        CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), c.stream));
        if (L.pst.size() != 3) L.pst.alloc(3, c.stream);
        if (L.cheb.size() != 2 * p.cheb_degree + 1) L.cheb.alloc(2 * p.cheb_degree + 1, c.stream);
        power_start(c, n, x.get());
        const double init[3] = {0.0, static_cast<double>(n), 0.0};
        h2d(L.pst.get(), init, 3, c.stream);
        for (int it = 0; it < p.power_iters; ++it) {
            power_step(c, A, L.w.get(), x.get(), y.get(), DotSink{partials.get(), ticket.get(), L.pst.get()});
            power_norm(c, n, y.get(), x.get(), L.pst.get(), DotSink{partials.get(), ticket.get(), L.pst.get() + 1});
        }
        cheb_coef(c, L.pst.get(), p.cheb_safety, p.cheb_lower, p.cheb_degree, L.cheb.get());
    }
}

void coarse_factorize(Hier& h, int* status) {
    Ctx& c = *h.ctx;
    const Level& L = h.lv.back();
    h.nL = L.pat->n;
    if (h.lu.size() != h.nL * h.nL) h.lu.alloc(h.nL * h.nL, c.stream);
    if (h.piv.size() != h.nL) h.piv.alloc(h.nL, c.stream);
    h.lu_formed = true;
    if (h.prm.coarse_solve == AMGR_COARSE_INVERSE) {
        lu_densify(c, L.view(), h.lu.get());
        if (h.inv.size() != h.nL * h.nL) h.inv.alloc(h.nL * h.nL, c.stream);
        // small systems: direct Gauss-Jordan inverse, no LU factor is formed
        if (dense_inverse_direct(c, h.nL, h.lu.get(), h.inv.get(), h.piv.get(), status)) {
            h.lu_formed = false;
            return;
        }
        lu_factor(c, h.nL, h.lu.get(), h.piv.get(), status);
        lu_inverse(c, h.nL, h.lu.get(), h.piv.get(), h.inv.get());
        return;
    }
    if (h.perm.size() != h.nL) h.perm.alloc(h.nL, c.stream);
    if (lu_factor_csr(c, L.view(), h.lu.get(), h.piv.get(), status, h.perm.get())) return;
    // (staging the CSR operator inside k_dense_reg instead of densifying
    // first measured 10-30 us slower per factorization: lu_factor's A argument)
    lu_densify(c, L.view(), h.lu.get());
    lu_factor(c, h.nL, h.lu.get(), h.piv.get(), status, h.perm.get());
}

static void coarse_solve(Hier& h, const double* b, double* x, Gate g) {
    if (h.prm.coarse_solve == AMGR_COARSE_INVERSE)
        inv_apply(*h.ctx, h.nL, h.inv.get(), b, x, g);
    else
        lu_solve(*h.ctx, h.nL, h.lu.get(), h.piv.get(), b, x, g, h.perm.get());
}

void throw_lu(int st) {
    std::ostringstream os;
    os << "coarse_factorize: singular matrix (zero pivot at step " << st << ")";
    fail(AMGR_E_RUNTIME, os.str());
}

// ---- symmetric-stencil form of level 0 (sym_dia) ------------------------------
// A level-0 pattern whose columns are i + {0, +-o_0, .., +-o_{K-1}} (K = 2, 3:
// the 5-/7-point grid stencils of C1-C5), sorted and structurally symmetric,
// whose values are BITWISE symmetric (a(i,j) == a(j,i), re-checked at every
// rebuild) is also kept as D | U_0..U_{K-1}: the row passes then read
// 8 (K+1) + 1 bytes per row instead of 9 nnz/n + 4 (k_dia), with the same
// entries summed in the same order.  AMGR_SYM_DIA=0 disables it.
static bool sym_dia_enabled() {
    const char* e = std::getenv("AMGR_SYM_DIA");
    return !(e && e[0] == '0');
}

// eligibility of a pattern (examined once; host sync)
static bool sym_dia_pattern(Ctx& c, Pattern& P) {
    if (P.dia_k >= 0) return P.dia_k > 0;
    P.dia_k = 0;
    if (P.cc.mode != 1 || P.cc.ndict < 5 || P.cc.ndict > 7 || P.n != P.ncols) return false;
    std::vector<int> d(static_cast<size_t>(P.cc.ndict));
    d2h(d.data(), P.cc.dict.get(), P.cc.ndict, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    std::vector<int> pos;
    bool zero = false;
    for (int x : d) {
        if (x == 0) zero = true;
        if (x > 0) pos.push_back(x);
    }
    std::sort(pos.begin(), pos.end());
    const int K = static_cast<int>(pos.size());
    if (!zero || K < 2 || K > 3 || 2 * K + 1 != P.cc.ndict) return false;
    for (int o : pos)
        if (std::find(d.begin(), d.end(), -o) == d.end()) return false;
    DevArray<uint8_t> m(P.n, c.stream);
    if (!dia_masks(c, csr_view(P, nullptr), K, pos.data(), m.get())) return false;
    P.dmask = std::move(m);
    for (int k = 0; k < K; ++k) P.doff[k] = pos[k];
    P.dia_k = K;
    return true;
}

// level-0 values -> D | U (enqueued on the current stream); the bit-symmetry
// verdict is read by sym_dia_commit after the rebuild's sync
static bool sym_dia_prepare(Hier& h) {
    Level& L0 = h.lv.front();
    L0.dia_on = false;
    return h.lv.size() > 1 && sym_dia_enabled() && sym_dia_pattern(*h.ctx, *L0.pat);
}
static void sym_dia_values(Hier& h) {
    Ctx& c = *h.ctx;
    Level& L0 = h.lv.front();
    const Pattern& P = *L0.pat;
    const int64_t need = (P.dia_k + 1) * P.n;
    if (L0.dia.size() != need) L0.dia.alloc(need, c.stream);
    if (L0.dia_flag.size() != 1) L0.dia_flag.alloc(1, c.stream);
    dia_values(c, csr_view(P, L0.view().val), P.dia_k, P.doff, P.dmask.get(), L0.dia.get(), L0.dia_flag.get());
}
static void sym_dia_commit(Hier& h) {
    Level& L0 = h.lv.front();
    if (L0.dia_flag.size() != 1 || L0.pat->dia_k <= 0 || !sym_dia_enabled()) return;
    L0.dia_on = d2h_scalar(L0.dia_flag.get(), h.ctx->stream) == 0;
}

// Read the per-level smoother bad-row slots and the LU status in one sync
// and throw the first error in the reference's order.
void check_rebuild_errors(Hier& h, const char* what) {
    Work& W = work(h);
    const size_t L = h.lv.size();
    std::vector<int> e(L + 1);
    d2h(e.data(), W.err.get(), static_cast<int64_t>(L + 1), h.ctx->stream);
    CK(cudaStreamSynchronize(h.ctx->stream));
    sym_dia_commit(h);
    for (size_t l = 0; l + 1 < L; ++l)
        if (e[l] != 0x7fffffff) {
            std::ostringstream os;
            os << level_prefix(l) << what << ": zero diagonal at row " << e[l];
            invalid(os.str());
        }
    if (e[L] >= 0) throw_lu(e[L]);
}

void reset_err(Hier& h) {
    Work& W = work(h);
    reset_error_slots(*h.ctx, W.err.get(), static_cast<int64_t>(h.lv.size()));
}

// ---- smoothed aggregation (extension; oracle/amg_oracle.c) -------------------
// P = P_tent - (w D^-1) A P_tent on the pattern of A P_tent, R = P^T.
static void build_sa_transfer(Ctx& c, Level& cur, Transfer& T, double w, size_t l) {
    const CsrView Av = cur.view();
    DevArray<int> trp, tcol;
    DevArray<double> tval;
    tentative_csr(c, Av.n, T.agg.get(), trp, tcol, tval);
    SpgPlan ap0;
    spgemm_symbolic(c, Av, trp.get(), tcol.get(), T.nc, ap0, "smoothed_prolongator");
    DevArray<double> pv(ap0.nnz, c.stream);
    spgemm_numeric(c, ap0, Av.val, tval.get(), pv.get());
    DevArray<int> bad(1, c.stream);
    const int big = 0x7fffffff;
    h2d(bad.get(), &big, 1, c.stream);
    sa_prolongator_values(c, Av.n, ap0.rp.get(), ap0.col.get(), pv.get(), T.agg.get(), cur.pat->diag.get(), Av.val,
                          w, bad.get());
    const int b = d2h_scalar(bad.get(), c.stream);
    if (b != big) {
        std::ostringstream os;
        os << level_prefix(l) << "smoothed_prolongator: zero diagonal at row " << b;
        invalid(os.str());
    }
    auto P = std::make_shared<Pattern>();
    P->n = Av.n;
    P->ncols = T.nc;
    P->nnz = ap0.nnz;
    P->rp = std::move(ap0.rp);
    P->col = std::move(ap0.col);
    P->max_span = max_group_span(c, P->rp.get(), P->n);
    DevArray<int> rrp, rcol;
    DevArray<double> rv;
    transpose_csr(c, Av.n, T.nc, P->nnz, P->rp.get(), P->col.get(), pv.get(), rrp, rcol, rv);
    auto R = std::make_shared<Pattern>();
    R->n = T.nc;
    R->ncols = Av.n;
    R->nnz = P->nnz;
    R->rp = std::move(rrp);
    R->col = std::move(rcol);
    R->max_span = max_group_span(c, R->rp.get(), R->n);
    T.P = P;
    T.Pv = std::move(pv);
    T.R = R;
    T.Rv = std::move(rv);
    T.smoothed = true;
}

// Galerkin plan of a smoothed level: A P (pattern + plan) then R (A P); the
// coarse pattern is the structural pattern of R A P (o_galerkin).
static std::shared_ptr<Pattern> sa_galerkin_plan(Ctx& c, const CsrView& Av, const Transfer& T, RapPlan& plan) {
    plan.ap = std::make_shared<SpgPlan>();
    spgemm_symbolic(c, Av, T.P->rp.get(), T.P->col.get(), T.nc, *plan.ap, "galerkin");
    plan.ap_val.alloc(plan.ap->nnz, c.stream);
    CsrView rv = csr_view(*T.R, T.Rv.get());
    plan.rap = std::make_shared<SpgPlan>();
    spgemm_symbolic(c, rv, plan.ap->rp.get(), plan.ap->col.get(), T.nc, *plan.rap, "galerkin");
    plan.nnz_f = Av.nnz;
    plan.nnz_c = plan.rap->nnz;
    auto P = std::make_shared<Pattern>();
    P->n = T.nc;
    P->ncols = T.nc;
    P->nnz = plan.rap->nnz;
    P->rp = std::move(plan.rap->rp);
    P->col = std::move(plan.rap->col);
    P->diag.alloc(P->n, c.stream);
    P->max_span = max_group_span(c, P->rp.get(), P->n);
    return P;
}

static void sa_galerkin_numeric(Ctx& c, const RapPlan& plan, const double* af, const Transfer& T, double* ac) {
    spgemm_numeric(c, *plan.ap, af, T.Pv.get(), const_cast<double*>(plan.ap_val.get()));
    spgemm_numeric(c, *plan.rap, T.Rv.get(), plan.ap_val.get(), ac);
}

static bool any_smoothed(const Hier& h) {
    for (const auto& l : h.lv)
        if (l.T && l.T->smoothed) return true;
    return false;
}

// restriction / prolongation of level i (tentative: member sums and k_prolong;
// smoothed: row passes over R and P)
static void restrict_level(Ctx& c, const Level& Li, const double* r, double* fc, const double* wc, double om,
                           double* u0c, Gate g) {
    if (Li.T->smoothed)
        vc_restrict_general(c, csr_view(*Li.T->R, Li.T->Rv.get()), r, fc, wc, om, u0c, g);
    else
        restrict_sum(c, Li.T->nc, Li.T->mptr.get(), Li.T->midx.get(), r, fc, wc, om, u0c, g);
}
static void prolong_level(Ctx& c, const Level& Li, const double* u, const double* e, double* out, Gate g) {
    if (Li.T->smoothed)
        vc_prolong_general(c, csr_view(*Li.T->P, Li.T->Pv.get()), u, e, out, g);
    else
        vc_prolong(c, Li.pat->n, u, Li.T->agg.get(), e, out, g);
}

// Smoothed aggregation + Jacobi (extension): per-level weight
// om_l = min(omega, (4/3) / g_l), g_l = max_i sum_j |a_ij| / |a_ii| — the
// Galerkin operators of a smoothed P have lambda_max(D^-1 A_l) up to 4-15,
// where the fixed weight diverges (oracle/amg_oracle.c sa_jacobi_omega).
static void sa_jacobi_weights(Hier& h) {
    if (h.prm.coarsening != AMGR_COARSENING_SMOOTHED || h.prm.smoother != AMGR_SMOOTHER_JACOBI) return;
    Ctx& c = *h.ctx;
    const size_t L = h.lv.size();
    if (L < 2) return;
    DevArray<unsigned long long> gb(static_cast<int64_t>(L), c.stream);
    CK(cudaMemsetAsync(gb.get(), 0, sizeof(unsigned long long) * L, c.stream));
    for (size_t l = 0; l + 1 < L; ++l) gershgorin_bound(c, h.lv[l].view(), h.lv[l].pat->diag.get(), gb.get() + l);
    std::vector<unsigned long long> hb(L);
    d2h(hb.data(), gb.get(), static_cast<int64_t>(L), c.stream);
    CK(cudaStreamSynchronize(c.stream));
    for (size_t l = 0; l + 1 < L; ++l) {
        double g;
        std::memcpy(&g, &hb[l], sizeof(double));
        const double cap = (4.0 / 3.0) / g;
        h.lv[l].om = cap < h.prm.omega ? cap : h.prm.omega;
    }
}

// Member-row plans (k_rap_rows) for every plain-aggregation level, built
// once per pattern (setup / pattern change).  Opt-in (AMGR_RAP_ROWS=1) until
// the kernel beats k_rap_tma + k_jacobi.
static bool rap_rows_enabled() {
    const char* e = std::getenv("AMGR_RAP_ROWS");
    return e && e[0] == '1';
}
static void build_row_plans(Hier& h) {
    Ctx& c = *h.ctx;
    if (!rap_rows_enabled()) return;
    for (size_t i = 0; i + 1 < h.lv.size(); ++i) {
        Level& A = h.lv[i];
        if (!A.rap || !A.T || A.T->smoothed || A.rap->rows_tried) continue;
        A.rap->rows_tried = true;
        const Pattern& C = *h.lv[i + 1].pat;
        rap_rows_plan(c, A.view(), A.T->agg.get(), A.T->midx.get(), A.T->nc, C.rp.get(), C.col.get(), A.rap->rows);
    }
}

// Warp-group plans (k_rap_grp) for every plain-aggregation level, built
// lazily once per Galerkin plan.  Default; AMGR_RAP_GROUPS=0 keeps k_rap_tma
// + k_jacobi.
static bool rap_grp_enabled() {
    const char* e = std::getenv("AMGR_RAP_GROUPS");
    return !(e && e[0] == '0');
}
static void build_grp_plans(Hier& h, size_t start) {
    Ctx& c = *h.ctx;
    if (!rap_grp_enabled()) return;
    for (size_t i = start; i + 1 < h.lv.size(); ++i) {
        Level& A = h.lv[i];
        if (!A.rap || !A.T || A.T->smoothed || A.rap->grp_tried) continue;
        A.rap->grp_tried = true;
        const Pattern& C = *h.lv[i + 1].pat;
        rap_grp_plan(c, A.view(), A.T->mptr.get(), A.T->midx.get(), A.pat->diag.get(), A.T->nc, C.rp.get(),
                     A.rap->nnz_c, A.rap->cptr.get(), A.rap->contrib.get(), A.rap->grp);
    }
}

// Numeric pass of partial_update (hierarchy.cpp:121-147) on existing plans:
// the Galerkin chain, then the per-level smoother rebuilds (main stream)
// concurrently with the coarsest factorization (side stream).
void numeric_pass(Hier& h, PhaseClock& clk, size_t start = 0) {
    Ctx& c = *h.ctx;
    Work& W = work(h);
    const size_t L = h.lv.size();
    // Galerkin chain first.  Levels with a member-row plan run k_rap_rows,
    // which also rebuilds the damped-Jacobi weights of the coarse level (and
    // of the fine level at the head of the chain), so those levels need no
    // separate smoother kernel.  The coarsest dense factorization (one CTA)
    // runs on the side stream concurrently with the remaining smoother
    // rebuilds, which do not depend on it.  Errors are still reported in the
    // reference's order (check_rebuild_errors reads every slot).
    const bool fuse = h.prm.smoother == AMGR_SMOOTHER_JACOBI && rap_rows_enabled();
    if (fuse) build_row_plans(h);  // lazily, once per plan
    // Jacobi fused into k_rap_tma (default; AMGR_FUSE_JACOBI=0 runs k_jacobi per level)
    // AMGR_FUSE_JACOBI=1 (opt-in): the coarse level's weights come from the
    // RAP thread that sums each coarse diagonal (levels >= 1); level 0's
    // k_jacobi runs after the chain.  Measured slower at 256^3 (2.54 vs
    // 2.38 ms per rebuild: the fused k_rap_tma variant loses more than the
    // removed k_jacobi launches save, and the coarsest factorization is no
    // longer hidden behind the smoother kernels), so by default every level
    // runs k_jacobi after the chain, concurrently with the factorization.
    const char* fe = std::getenv("AMGR_FUSE_JACOBI");
    const bool jac = h.prm.smoother == AMGR_SMOOTHER_JACOBI && fe && fe[0] == '1';
    std::vector<char> wdone(L, 0);
    // level 0's symmetric-stencil copy: forked onto the side stream once the
    // wide Galerkin levels are done (AMGR_DIA_FORK, default after level 1),
    // so it overlaps the latency-bound small levels of the chain (next to the
    // level-0 product it would compete for bandwidth; next to the one-CTA
    // coarse factorization it cannot run: that CTA needs a whole SM)
    const bool dia = start == 0 && sym_dia_prepare(h);
    bool dia_done = false;
    const char* dfe = std::getenv("AMGR_DIA_FORK");
    const size_t dia_fork = dfe ? static_cast<size_t>(std::atoi(dfe)) : 1;
    build_grp_plans(h, start);
    for (size_t i = start; i + 1 < L; ++i) {
        c.cur_level = static_cast<int>(i);
        Level& A = h.lv[i];
        clk.begin(PH_GALERKIN);
        Level& B = h.lv[i + 1];
        if (B.val.size() != B.pat->nnz) B.val.alloc(B.pat->nnz, c.stream);
        if (A.T->smoothed) {
            sa_galerkin_numeric(c, *A.rap, A.view().val, *A.T, B.val.get());
        } else if (A.rap->grp.ok && rap_grp_enabled() && !(fuse && A.rap->rows.ok)) {
            // warp-group RAP; the fine level's damped-Jacobi weights come
            // from the member rows it stages (its values are final here)
            const GrpPlan& gp = A.rap->grp;
            GrpArgs ga;
            ga.ngroups = gp.ngroups;
            ga.desc = gp.desc.get();
            ga.mstart = gp.mstart.get();
            ga.mdoff = gp.mdoff.get();
            ga.midx = A.T->midx.get();
            ga.code = gp.code.get();
            ga.lanes = gp.lanes.get();
            ga.af = A.view().val;
            ga.ac = B.val.get();
            if (h.prm.smoother == AMGR_SMOOTHER_JACOBI && !wdone[i]) {
                if (A.w.size() != A.pat->n) A.w.alloc(A.pat->n, c.stream);
                ga.wf = A.w.get();
                ga.bad_f = W.err.get() + i;
                wdone[i] = 1;
                A.has_smoother = true;
            }
            rap_grp(c, ga, A.pat->n, B.pat->n, A.pat->nnz, B.pat->nnz);
        } else if (fuse && A.rap->rows.ok) {
            const RowPlan& rp = A.rap->rows;
            RapRowsArgs a;
            a.nc = static_cast<int>(B.pat->n);
            a.dmax = rp.dmax;
            a.mptr = A.T->mptr.get();
            a.midx = A.T->midx.get();
            a.mrp = rp.mrp.get();
            a.mlen = rp.mlen.get();
            a.code = rp.code.get();
            a.af = A.view().val;
            a.crp = B.pat->rp.get();
            a.cdiag = B.pat->diag.get();
            a.ac = B.val.get();
            if (!wdone[i]) {
                if (A.w.size() != A.pat->n) A.w.alloc(A.pat->n, c.stream);
                a.wf = A.w.get();
                a.bad_f = W.err.get() + i;
                wdone[i] = 1;
                A.has_smoother = true;
            }
            if (i + 2 < L) {
                if (B.w.size() != B.pat->n) B.w.alloc(B.pat->n, c.stream);
                a.wc = B.w.get();
                a.bad_c = W.err.get() + i + 1;
                wdone[i + 1] = 1;
                B.has_smoother = true;
            }
            rap_rows(c, a, rp.maxlen, A.pat->n, A.pat->nnz, B.pat->nnz);
        } else if (jac) {
            // k_rap_tma with the Jacobi rebuild of the coarse level (and of the
            // fine level at the head of the chain) in its epilogue
            RapPlan& rp = *A.rap;
            RapJacobi fj;
            if (i + 2 < L) {
                if (B.w.size() != B.pat->n) B.w.alloc(B.pat->n, c.stream);
                fj.ccol = B.pat->col.get();
                fj.wc = B.w.get();
                fj.bad_c = W.err.get() + i + 1;
            }
            if (rap_numeric(c, A.pat->n, B.pat->n, rp.nnz_c, rp.cptr.get(), rp.contrib.get(), A.view().val,
                            B.val.get(), A.pat->nnz, rp.max_chunk, fj.wc ? &fj : nullptr)) {
                wdone[i + 1] = 1;
                B.has_smoother = true;
            }
        } else {
            rap_numeric(c, A.pat->n, B.pat->n, A.rap->nnz_c, A.rap->cptr.get(), A.rap->contrib.get(), A.view().val,
                        B.val.get(), A.pat->nnz, A.rap->max_chunk);
        }
        clk.end(PH_GALERKIN);
        if (dia && !dia_done && i >= dia_fork) {
            on_side(c, [&] { sym_dia_values(h); });
            dia_done = true;
        }
    }
    c.cur_level = static_cast<int>(L - 1);
    on_side(c, [&] {
        clk.begin(PH_COARSE);
        coarse_factorize(h, W.err.get() + L);
        clk.end(PH_COARSE);
    });
    for (size_t i = start; i + 1 < L; ++i) {
        if (wdone[i]) continue;
        c.cur_level = static_cast<int>(i);
        clk.begin(PH_SMOOTHER);
        build_smoother(c, h.lv[i], h.prm, W.err.get() + i);
        clk.end(PH_SMOOTHER);
    }
    if (dia && !dia_done) sym_dia_values(h);
    join_side(c);
    c.cur_level = -1;
    sa_jacobi_weights(h);
}

// Symbolic pass with frozen transfers (pattern change under partial reuse).
void symbolic_pass(Hier& h) {
    Ctx& c = *h.ctx;
    for (size_t i = 0; i + 1 < h.lv.size(); ++i) {
        Level& A = h.lv[i];
        if (A.T->smoothed) {
            auto plan = std::make_shared<RapPlan>();
            auto P = sa_galerkin_plan(c, A.view(), *A.T, *plan);
            A.rap = plan;
            Level& B = h.lv[i + 1];
            B.pat = P;
            CsrView v = B.view();
            find_diag(c, v, P->diag.get());
            continue;
        }
        RapSymbolic s;
        rap_symbolic(c, A.view(), A.T->agg.get(), A.T->nc, s);
        auto plan = std::make_shared<RapPlan>();
        plan->nnz_f = A.pat->nnz;
        plan->nnz_c = s.nnz_c;
        plan->cptr = std::move(s.cptr);
        plan->contrib = std::move(s.contrib);
        plan->max_chunk = rap_chunk_max(c, plan->nnz_c, plan->cptr.get());
        A.rap = plan;
        auto P = std::make_shared<Pattern>();
        P->n = A.T->nc;
        P->ncols = A.T->nc;
        P->nnz = s.nnz_c;
        P->rp = std::move(s.rp);
        P->col = std::move(s.col);
        P->diag.alloc(P->n, c.stream);
        Level& B = h.lv[i + 1];
        B.pat = P;
        CsrView v = B.view();
        find_diag(c, v, P->diag.get());
        P->max_span = max_group_span(c, P->rp.get(), P->n);
    }
}

}  // namespace

Work& work(Hier& h) {
    Ctx& c = *h.ctx;
    std::vector<int64_t> shape;
    for (auto& l : h.lv) shape.push_back(l.pat->n);
    if (!h.ws || h.ws->shape != shape) {
        auto W = std::make_shared<Work>();
        W->shape = shape;
        const size_t L = h.lv.size();
        W->u.resize(L);
        W->t.resize(L);
        W->d0.resize(L);
        W->d1.resize(L);
        W->f.resize(L);
        W->r.resize(L);
        for (size_t i = 0; i < L; ++i) {
            const int64_t n = h.lv[i].pat->n;
            W->u[i].alloc(n, c.stream);
            W->t[i].alloc(n, c.stream);
            if (i > 0) W->f[i].alloc(n, c.stream);
            W->r[i].alloc(n, c.stream);
        }
        W->st.alloc(1, c.stream);
        W->partials.alloc(static_cast<int64_t>(dot_grid(c)) * 4 + 64, c.stream);
        W->ticket.alloc(1, c.stream);
        CK(cudaMemsetAsync(W->ticket.get(), 0, sizeof(unsigned), c.stream));
        W->err.alloc(static_cast<int64_t>(L + 1), c.stream);
        h.ws = W;
    }
    return *h.ws;
}

// Setup allocates and frees many large temporaries of varying sizes (sort
// buffers, plans).  When no free block of the stream-ordered pool fits, the
// pool maps new physical memory, which measured 0.1-0.5 s per GB-sized
// request and made setup times swing 0.3 -> 1.4 s at 256^3.  One large
// allocation up front (freed immediately; the context keeps the pool's
// memory, release threshold = max) leaves a single mapped region that the
// setup's temporaries are carved from.
static void reserve_pool(Ctx& c, int64_t nnz) {
    const char* e = std::getenv("AMGR_POOL_RESERVE_BYTES_PER_NNZ");
    // setup peak measured 82 B/nnz at 256^3 (AMGR_TRACE_SETUP), the hierarchy
    // itself 57 B/nnz; 256 B/nnz leaves room for a no-reuse step's new setup
    // while the previous hierarchy is alive (with 96 B/nnz the bench's
    // no-reuse steps still hit 0.2-2 s pool-growth stalls)
    const double per = e ? std::atof(e) : 256.0;
    size_t want = static_cast<size_t>(per * static_cast<double>(nnz));
    if (want == 0) return;
    cudaMemPool_t pool;
    CK(cudaDeviceGetMemPool(&pool, c.device));
    // the pool's idle part (reserved - used) must hold the setup's temporaries;
    // a live hierarchy (e.g. the previous step's under no-reuse) is "used"
    uint64_t reserved = 0, used = 0;
    CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
    if (reserved - used >= want) return;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    if (want > free_b / 2) want = free_b / 2;  // never take more than half of what is free
    if (reserved - used >= want) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, want, c.stream) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    CK(cudaFreeAsync(p, c.stream));
}

// ---- setup (hierarchy.cpp:45-105) ------------------------------------------------
std::unique_ptr<Hier> setup(Ctx& c, const amgr_csr& A, const AmgP& p) {
    if (A.nrows != A.ncols) invalid("setup: matrix is not square");
    if (A.nrows == 0) invalid("setup: empty matrix");
    auto h = std::make_unique<Hier>();
    h->ctx = &c;
    h->prm = p;
    PhaseClock clk(c);
    const auto t_setup = std::chrono::steady_clock::now();
    const bool trace = std::getenv("AMGR_TRACE_SETUP") != nullptr;

    reserve_pool(c, A.nnz);
    uint64_t used0 = 0;
    if (trace) {
        cudaMemPool_t pool;
        CK(cudaDeviceGetMemPool(&pool, c.device));
        CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used0));
        uint64_t zero = 0;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero));
    }
    Level L0;
    L0.pat = make_pattern(c, A);
    upload_values(c, L0.val, A.values, A.nnz, A.location);
    h->lv.push_back(std::move(L0));
    DevArray<int> bad(1, c.stream);
    DevArray<int> lu_status(1, c.stream);

    while (h->lv.back().pat->n > p.coarse_enough) {
        const size_t l = h->lv.size() - 1;
        Level& cur = h->lv.back();
        const CsrView Av = cur.view();
        auto T = std::make_shared<Transfer>();
        int64_t nc = 0;
        clk.begin(PH_TRANSFER);
        {
            // strength_graph (coarsening.cpp:11-34) error order: eps, then diagonal
            if (p.eps < 0.0 || p.eps >= 1.0) invalid(level_prefix(l) + "strength_graph: eps must be in [0, 1)");
            const int64_t badrow = first_bad_diag(c, Av, cur.pat->diag.get());
            if (badrow >= 0) {
                std::ostringstream os;
                os << level_prefix(l) << "strength_graph: zero diagonal at row " << badrow;
                invalid(os.str());
            }
            GraphDev g;
            strength_graph(c, Av, cur.pat->diag.get(), p.eps * p.eps, g);
            if (trace) {
                CK(cudaStreamSynchronize(c.stream));
                std::fprintf(stderr, "[amgr setup] level %zu: strength graph (%lld edges) t=%.1f ms\n", l,
                             static_cast<long long>(g.m),
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup)
                                 .count());
            }
            int64_t rounds = 0;
            nc = aggregate(c, g, T->agg, &rounds);
            h->agg_rounds += rounds;
            T->nf = Av.n;
            T->nc = nc;
            if (nc < Av.n) members(c, Av.n, nc, T->agg.get(), T->mptr, T->midx);
        }
        clk.end(PH_TRANSFER);
        if (trace)
            std::fprintf(stderr, "[amgr setup] level %zu: n=%lld nnz=%lld -> nc=%lld (agg rounds %lld) t=%.1f ms\n", l,
                         static_cast<long long>(Av.n), static_cast<long long>(Av.nnz), static_cast<long long>(nc),
                         static_cast<long long>(h->agg_rounds),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup).count());
        if (nc == Av.n) {
            // coarsening stalled (hierarchy.cpp:70-77)
            if (Av.n <= p.max_direct) break;
            std::ostringstream os;
            os << "setup: coarsening stalled at level " << l << " with " << Av.n
               << " unknowns (> max_direct_size " << p.max_direct << ")";
            fail(AMGR_E_RUNTIME, os.str());
        }
        if (p.coarsening == AMGR_COARSENING_SMOOTHED) {
            clk.begin(PH_TRANSFER);
            build_sa_transfer(c, cur, *T, p.sa_omega, l);
            clk.end(PH_TRANSFER);
        }
        // smoother (hierarchy.cpp:79-87)
        {
            const int big = 0x7fffffff;
            h2d(bad.get(), &big, 1, c.stream);
            clk.begin(PH_SMOOTHER);
            build_smoother(c, cur, p, bad.get());
            clk.end(PH_SMOOTHER);
            const int b = d2h_scalar(bad.get(), c.stream);
            if (b != big) {
                std::ostringstream os;
                os << level_prefix(l) << "build_smoother: zero diagonal at row " << b;
                invalid(os.str());
            }
        }
        // Galerkin product (hierarchy.cpp:89-93): symbolic plan + numeric values
        Level next;
        clk.begin(PH_GALERKIN);
        if (T->smoothed) {
            auto plan = std::make_shared<RapPlan>();
            auto P = sa_galerkin_plan(c, Av, *T, *plan);
            next.pat = P;
            next.val.alloc(P->nnz, c.stream);
            CsrView nv = next.view();
            find_diag(c, nv, P->diag.get());
            sa_galerkin_numeric(c, *plan, Av.val, *T, next.val.get());
            cur.rap = plan;
        } else {
            RapSymbolic s;
            rap_symbolic(c, Av, T->agg.get(), nc, s);
            auto plan = std::make_shared<RapPlan>();
            plan->nnz_f = Av.nnz;
            plan->nnz_c = s.nnz_c;
            plan->cptr = std::move(s.cptr);
            plan->contrib = std::move(s.contrib);
            plan->max_chunk = rap_chunk_max(c, plan->nnz_c, plan->cptr.get());
            auto P = std::make_shared<Pattern>();
            P->n = nc;
            P->ncols = nc;
            P->nnz = s.nnz_c;
            P->rp = std::move(s.rp);
            P->col = std::move(s.col);
            P->diag.alloc(nc, c.stream);
            next.pat = P;
            next.val.alloc(s.nnz_c, c.stream);
            CsrView nv = next.view();
            find_diag(c, nv, P->diag.get());
            rap_numeric(c, Av.n, nc, s.nnz_c, plan->cptr.get(), plan->contrib.get(), Av.val, next.val.get(), Av.nnz,
                        plan->max_chunk);
            P->max_span = max_group_span(c, P->rp.get(), P->n);
            cur.rap = plan;
        }
        clk.end(PH_GALERKIN);
        if (trace) {
            CK(cudaStreamSynchronize(c.stream));
            std::fprintf(stderr, "[amgr setup] level %zu: smoother + Galerkin done t=%.1f ms\n", l,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup).count());
        }
        cur.T = T;
        h->lv.push_back(std::move(next));
    }
    // coded column streams for the row passes (all levels but the coarsest,
    // which is solved densely)
    clk.begin(PH_GALERKIN);
    for (size_t l = 0; l + 1 < h->lv.size(); ++l) {
        Pattern& P = *h->lv[l].pat;
        encode_columns(c, P.n, P.nnz, P.rp.get(), P.col.get(), P.cc);
    }
    build_row_plans(*h);
    clk.end(PH_GALERKIN);
    sa_jacobi_weights(*h);
    clk.begin(PH_COARSE);
    coarse_factorize(*h, lu_status.get());
    clk.end(PH_COARSE);
    if (sym_dia_prepare(*h)) sym_dia_values(*h);
    const int st = d2h_scalar(lu_status.get(), c.stream);
    if (st >= 0) throw_lu(st);
    sym_dia_commit(*h);
    h->tm = clk.collect();
    work(*h);
    if (trace) {
        cudaMemPool_t pool;
        CK(cudaDeviceGetMemPool(&pool, c.device));
        uint64_t high = 0, now = 0;
        CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high));
        CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &now));
        std::fprintf(stderr, "[amgr setup] pool: peak +%.2f GB during setup (%.1f B/nnz), hierarchy +%.2f GB\n",
                     (high - used0) / 1e9, static_cast<double>(high - used0) / static_cast<double>(A.nnz),
                     (now - used0) / 1e9);
    }
    return h;
}

// ---- partial_update (hierarchy.cpp:107-150) -----------------------------------------
static void check_dims(const Hier& h, const amgr_csr& A) {
    const Pattern& P0 = *h.lv.front().pat;
    if (A.nrows != P0.n || A.ncols != P0.ncols) {
        std::ostringstream os;
        os << "partial update impossible, full rebuild required: new matrix is " << A.nrows << "x" << A.ncols
           << ", hierarchy was built for " << P0.n << "x" << P0.ncols;
        fail(AMGR_E_DIMENSION, os.str());
    }
}

static void rebuild_into(Hier& h, const amgr_csr& A) {
    Ctx& c = *h.ctx;
    // pattern: reuse the cached symbolic plan unless the structure changed
    std::shared_ptr<Pattern> np = make_pattern(c, A);
    const bool same = same_pattern(c, *np, *h.lv.front().pat);
    h.lv.front().ext_val = nullptr;
    upload_values(c, h.lv.front().val, A.values, A.nnz, A.location);
    if (!same) {
        h.lv.front().pat = np;
        symbolic_pass(h);
        // the new patterns need their coded column streams and member-row
        // plans too (as setup)
        for (size_t l = 0; l + 1 < h.lv.size(); ++l) {
            Pattern& P = *h.lv[l].pat;
            encode_columns(c, P.n, P.nnz, P.rp.get(), P.col.get(), P.cc);
        }
        build_row_plans(h);
        h.ws.reset();
    }
    work(h);
    reset_err(h);
    PhaseClock clk(c);
    numeric_pass(h, clk);
    check_rebuild_errors(h, "build_smoother");
    h.tm = clk.collect();
}

std::unique_ptr<Hier> partial_update(const Hier& h, const amgr_csr& A, const AmgP& p) {
    if (h.lv.empty()) invalid("partial_update: empty hierarchy");
    check_dims(h, A);
    Ctx& c = *h.ctx;
    auto out = std::make_unique<Hier>();
    out->ctx = &c;
    out->prm = p;
    out->ws = h.ws;
    out->agg_rounds = 0;
    for (const Level& L : h.lv) {
        Level n;
        n.pat = L.pat;  // shared structure
        n.T = L.T;      // shared frozen transfer operators
        n.rap = L.rap;  // shared cached Galerkin plan
        out->lv.push_back(std::move(n));
    }
    for (size_t i = 0; i < out->lv.size(); ++i) out->lv[i].val.alloc(out->lv[i].pat->nnz, c.stream);
    rebuild_into(*out, A);
    return out;
}

// Rebuild of levels start.. only (their A_start values already in place):
// the distributed rebuild's replicated tail (dist.cu).  Same kernels, order
// and error reporting as rebuild_into.
void rebuild_levels_from(Hier& h, size_t start) {
    work(h);
    reset_err(h);
    PhaseClock clk(*h.ctx);
    numeric_pass(h, clk, start);
    check_rebuild_errors(h, "build_smoother");
    h.tm = clk.collect();
}

void rebuild(Hier& h, const amgr_csr& A) {
    check_dims(h, A);
    rebuild_into(h, A);
}

Hier::~Hier() {
    if (staged_ev) cudaEventDestroy(staged_ev);
    if (main_ev) cudaEventDestroy(main_ev);
    if (rhs_ev) cudaEventDestroy(rhs_ev);
}

static void ensure_copy_stream(Hier& h) {
    Ctx& c = *h.ctx;
    if (!c.copy) CK(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    if (!h.staged_ev) {
        CK(cudaEventCreateWithFlags(&h.staged_ev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h.main_ev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h.rhs_ev, cudaEventDisableTiming));
    }
}

void stage_rhs(Hier& h, const double* f, int location) {
    Ctx& c = *h.ctx;
    if (location != AMGR_HOST && location != AMGR_DEVICE) invalid("stage_rhs: location must be HOST or DEVICE");
    if (!f) invalid("stage_rhs: f is null");
    ensure_copy_stream(h);
    const int64_t n = h.lv.front().pat->n;
    if (h.staged_rhs.size() != n) h.staged_rhs.alloc(n, c.stream);
    // the staging buffer may still be read by work queued on the main stream
    CK(cudaEventRecord(h.main_ev, c.stream));
    CK(cudaStreamWaitEvent(c.copy, h.main_ev, 0));
    CK(cudaMemcpyAsync(h.staged_rhs.get(), f, sizeof(double) * n,
                       location == AMGR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.copy));
    CK(cudaEventRecord(h.rhs_ev, c.copy));
    h.rhs_staged = true;
}

void commit_rhs(Hier& h) {
    Ctx& c = *h.ctx;
    CK(cudaStreamWaitEvent(c.stream, h.rhs_ev, 0));
    h.rhs.swap(h.staged_rhs);  // the previous RHS becomes the next staging buffer
    h.rhs_staged = false;
    h.rhs_ready = true;
}

const double* committed_rhs(Hier& h) {
    if (!h.rhs_ready)
        invalid("staged solve: no staged right-hand side (amgr_stage_rhs, then a STAGED rebuild commits it)");
    return h.rhs.get();
}

void stage_values(Hier& h, const double* values, int location) {
    Ctx& c = *h.ctx;
    if (location != AMGR_HOST && location != AMGR_DEVICE) invalid("stage_values: location must be HOST or DEVICE");
    ensure_copy_stream(h);
    const int64_t nnz = h.lv.front().pat->nnz;
    if (h.staged.size() != nnz) h.staged.alloc(nnz, c.stream);
    // the staging buffer may still be read by work queued on the main stream
    CK(cudaEventRecord(h.main_ev, c.stream));
    CK(cudaStreamWaitEvent(c.copy, h.main_ev, 0));
    if (nnz > 0)
        CK(cudaMemcpyAsync(h.staged.get(), values, sizeof(double) * nnz,
                           location == AMGR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.copy));
    CK(cudaEventRecord(h.staged_ev, c.copy));
    h.staged_ready = true;
}

void rebuild_values(Hier& h, const double* values, int location) {
    Ctx& c = *h.ctx;
    if (location == AMGR_STAGED) {
        if (!h.staged_ready) invalid("rebuild_values: no staged values (call amgr_stage_values first)");
        CK(cudaStreamWaitEvent(c.stream, h.staged_ev, 0));
        Level& L0 = h.lv.front();
        L0.ext_val = nullptr;
        if (L0.val.size() != L0.pat->nnz) L0.val.alloc(L0.pat->nnz, c.stream);
        L0.val.swap(h.staged);  // the previous values become the next staging buffer
        h.staged_ready = false;
        if (h.rhs_staged) commit_rhs(h);  // the step's RHS, staged with its values
    } else if (location == AMGR_DEVICE_ADOPT) {
        if (reinterpret_cast<uintptr_t>(values) % 16 != 0) invalid("rebuild_values: adopted buffer must be 16-byte aligned");
        h.lv.front().ext_val = values;
    } else {
        h.lv.front().ext_val = nullptr;
        upload_values(c, h.lv.front().val, values, h.lv.front().pat->nnz, location);
    }
    work(h);
    reset_err(h);
    PhaseClock clk(c);
    numeric_pass(h, clk);
    check_rebuild_errors(h, "build_smoother");
    h.tm = clk.collect();
}

// ---- V-cycle (hierarchy.cpp:152-186, smoothing as specified) --------
// Down leg per level: [premul on level 0] -> vc_down (r = f - A u0) ->
// restriction (also writing the next level's u0).  Up leg per level:
// prolongation x = u + P u_c (coalesced pass) -> post-smoothing sweeps.
// One Chebyshev sweep (oracle smooth_cheb) on level i from x (zero when
// from_zero) into *out; returns the buffer holding the result.
// Chebyshev direction vectors of every smoothed level (allocated lazily by
// the first sweep otherwise)
static void ensure_cheb_work(Hier& h) {
    if (h.prm.smoother != AMGR_SMOOTHER_CHEBYSHEV) return;
    Ctx& c = *h.ctx;
    Work& W = work(h);
    const size_t L = h.lv.size();
    if (W.d0.size() != L) {
        W.d0.resize(L);
        W.d1.resize(L);
    }
    for (size_t i = 0; i + 1 < L; ++i) {
        const int64_t n = h.lv[i].pat->n;
        if (W.d0[i].size() != n) W.d0[i].alloc(n, c.stream);
        if (W.d1[i].size() != n) W.d1[i].alloc(n, c.stream);
    }
}

static double* cheb_sweep(Hier& h, size_t i, const double* f, double* x, double* other, bool from_zero, Gate g) {
    Ctx& c = *h.ctx;
    Work& W = work(h);
    const Level& Li = h.lv[i];
    const CsrView A = Li.view();
    const int64_t n = A.n;
    if (W.d0[i].size() != n) W.d0[i].alloc(n, c.stream);
    if (W.d1[i].size() != n) W.d1[i].alloc(n, c.stream);
    double* d = W.d0[i].get();
    double* dn = W.d1[i].get();
    if (from_zero) {
        fill(c, x, n, 0.0, g);
        cheb_zero(c, n, f, Li.w.get(), Li.cheb.get(), d, g);
    } else {
        cheb_start(c, A, f, Li.w.get(), x, Li.cheb.get(), d, g);
    }
    double* xs = x;
    double* xo = other;
    for (int k = 1; k < h.prm.cheb_degree; ++k) {
        cheb_step(c, A, f, Li.w.get(), xs, d, Li.cheb.get(), k, xo, dn, g);
        std::swap(xs, xo);
        std::swap(d, dn);
    }
    axpy1(c, n, xs, d, g);
    return xs;
}

// V-cycle with the Chebyshev smoother (extension): generic sweeps, residual,
// restriction, prolongation (hierarchy.cpp:152-186 structure).
static void vcycle_cheb(Hier& h, const double* f, double* u, Gate g) {
    Ctx& c = *h.ctx;
    Work& W = work(h);
    const size_t L = h.lv.size();
    if (W.d0.size() != L) {
        W.d0.resize(L);
        W.d1.resize(L);
    }
    std::vector<const double*> fin(L), ufinal(L);
    fin[0] = f;
    for (size_t i = 1; i < L; ++i) fin[i] = W.f[i].get();
    std::vector<double*> cur(L);
    for (size_t i = 0; i + 1 < L; ++i) {
        c.cur_level = static_cast<int>(i);
        const Level& Li = h.lv[i];
        const CsrView A = Li.view();
        double* a = W.u[i].get();
        double* b = W.t[i].get();
        double* x = a;
        if (h.prm.pre <= 0) {
            fill(c, a, A.n, 0.0, g);
        } else {
            for (int s = 0; s < h.prm.pre; ++s) {
                double* other = (x == a) ? b : a;
                x = cheb_sweep(h, i, fin[i], x, other, s == 0, g);
            }
        }
        cur[i] = x;
        residual(c, A, fin[i], x, W.r[i].get(), g);
        restrict_level(c, Li, W.r[i].get(), W.f[i + 1].get(), nullptr, 0.0, nullptr, g);
    }
    c.cur_level = static_cast<int>(L - 1);
    coarse_solve(h, W.f[L - 1].get(), W.u[L - 1].get(), g);
    ufinal[L - 1] = W.u[L - 1].get();
    for (size_t i = L - 1; i-- > 0;) {
        c.cur_level = static_cast<int>(i);
        const Level& Li = h.lv[i];
        const CsrView A = Li.view();
        double* a = cur[i];
        double* b = (a == W.u[i].get()) ? W.t[i].get() : W.u[i].get();
        prolong_level(c, Li, a, ufinal[i + 1], b, g);
        double* x = b;
        for (int s = 0; s < h.prm.post; ++s) {
            double* other = (x == a) ? b : a;
            x = cheb_sweep(h, i, fin[i], x, other, false, g);
        }
        if (i == 0) {
            copy(c, u, x, A.n, g);
            ufinal[i] = u;
        } else {
            ufinal[i] = x;
        }
    }
    c.cur_level = -1;
}

// V-cycle over levels s..L-1 (s = 0: the whole hierarchy); f and u live on
// level s.  The partitioned multi-GPU solve runs the replicated coarse levels
// through this with s = T+1.
// Fold the first pre-smoothing iterate into the top level's down pass and
// prolongation (default on; AMGR_FOLD_PREMUL=0 materialises it with k_premul).
static bool fold_premul() {
    const char* e = std::getenv("AMGR_FOLD_PREMUL");
    return !(e && std::string(e) == "0");
}

// First level of the persistent V-cycle tail (kernels_tail.cu): the first
// level at or below s from which every operator has at most AMGR_TAIL_NNZ
// nonzeros; -1 = no tail.  Off by default: measured on B200 the grid-barrier
// version is slower than the per-level launches (each phase still pays ~3
// dependent L2 round trips plus a ~1.5 us grid barrier), see DESIGN.md.
static int tail_start(const Hier& h, size_t s) {
    const char* e = std::getenv("AMGR_TAIL_NNZ");
    const long thr = e ? std::atol(e) : 0L;
    const size_t L = h.lv.size();
    if (thr <= 0 || h.prm.pre != 1 || h.prm.post != 1 || h.prm.smoother == AMGR_SMOOTHER_CHEBYSHEV ||
        any_smoothed(h))
        return -1;
    for (size_t i = s; i + 1 < L; ++i) {
        bool small = true;
        for (size_t k = i; k + 1 < L; ++k) small = small && h.lv[k].pat->nnz <= thr;
        if (small) return (L - 1 - i) <= static_cast<size_t>(TAIL_MAX) ? static_cast<int>(i) : -1;
    }
    return -1;
}

static int lag_groups(Ctx& c, Pattern& P) {
    if (P.lag_groups >= 0) return P.lag_groups;
    P.lag_groups = 0;
    if (P.cc.mode == 1 && P.cc.ndict > 0) {
        std::vector<int> d(static_cast<size_t>(P.cc.ndict));
        d2h(d.data(), P.cc.dict.get(), P.cc.ndict, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        int m = 0;
        for (int x : d) m = std::max(m, x < 0 ? -x : x);
        P.lag_groups = (m + 31) / 32 + 2;
    }
    return P.lag_groups;
}

// opt-in (AMGR_LAG_FUSE=1): bit-identical, and it does save the DRAM sweep
// (ncu at 256^3: 1.98 GB moved vs 3.1 GB for the two kernels), but the fused
// kernel is issue-bound (IPC 2.2/SM, 64 registers x 32 warps) and takes
// 678 us against 266 + 255 us separately
static bool lag_enabled() {
    const char* e = std::getenv("AMGR_LAG_FUSE");
    return e && e[0] == '1';
}

// host syncs / allocations of the fused level-0 pass, done outside any capture
static void lag_prepare(Hier& h) {
    Ctx& c = *h.ctx;
    Work& W = work(h);
    Pattern& P0 = *h.lv.front().pat;
    if (lag_groups(c, P0) <= 0) return;
    const int64_t rounds = (P0.n + 31) / 32 / (static_cast<int64_t>(c.num_sms) * 32) + 2;  // >= rounds of the grid
    if (W.lagdone.size() < 64 * rounds) W.lagdone.alloc(64 * rounds, c.stream);
}

void vcycle_from(Hier& h, size_t s, const double* f, double* u, Gate g, NextSpmv* nx) {
    Ctx& c = *h.ctx;
    Work& W = work(h);
    const size_t L = h.lv.size();
    const double om = h.om_eff();
    if (s + 1 == L) {
        coarse_solve(h, f, u, g);
        return;
    }
    if (h.prm.smoother == AMGR_SMOOTHER_CHEBYSHEV) {
        if (s != 0) invalid("vcycle_from: Chebyshev smoother supports s = 0 only");
        vcycle_cheb(h, f, u, g);
        return;
    }
    std::vector<const double*> fin(L), ufinal(L);
    fin[s] = f;
    for (size_t i = s + 1; i < L; ++i) fin[i] = W.f[i].get();
    std::vector<double*> cur(L);
    const int pre = h.prm.pre, post = h.prm.post;
    const int ts = tail_start(h, s);
    const size_t top = ts >= 0 ? static_cast<size_t>(ts) : L - 1;  // levels >= top: tail kernels
    // one pre-sweep from zero: its iterate u0 = (om w) f is folded into the
    // top level's down pass and prolongation instead of being materialised
    const bool fold = pre == 1 && top > s && fold_premul() && !h.lv[s].T->smoothed;
    auto oml = [&](size_t l) { return h.om_level(l); };
    if (pre >= 1 && !fold) vc_premul(c, h.lv[s].pat->n, f, h.lv[s].w.get(), oml(s), W.u[s].get(), g);
    // down leg
    for (size_t i = s; i < top; ++i) {
        c.cur_level = static_cast<int>(i);
        const Level& Li = h.lv[i];
        const CsrView A = Li.view();
        double* a = W.u[i].get();  // holds u0 (premul / previous restriction) when pre >= 1
        double* b = W.t[i].get();
        double* r = W.r[i].get();
        if (pre <= 0) {
            fill(c, a, A.n, 0.0, g);
            copy(c, r, fin[i], A.n, g);
            cur[i] = a;
        } else {
            double* src = a;
            if (pre == 1) {
                if (fold && i == s)
                    vc_down_premul(c, A, fin[i], Li.w.get(), oml(i), r, g);
                else
                    vc_down(c, A, fin[i], a, r, g);
            } else {
                double* dst = b;
                for (int s = 1; s < pre; ++s) {
                    vc_smooth(c, A, fin[i], Li.w.get(), oml(i), src, dst, g);
                    std::swap(src, dst);
                }
                residual(c, A, fin[i], src, r, g);
            }
            cur[i] = src;
        }
        const bool next_smoothed = pre >= 1 && i + 2 < L;
        restrict_level(c, Li, r, W.f[i + 1].get(), next_smoothed ? h.lv[i + 1].w.get() : nullptr, oml(i + 1),
                       next_smoothed ? W.u[i + 1].get() : nullptr, g);
    }
    TailDesc td;
    if (ts >= 0) {
        for (size_t l = top; l + 1 < L; ++l) {
            const Level& Li = h.lv[l];
            const CsrView A = Li.view();
            TailLevel& t = td.lv[td.count++];
            t.n = static_cast<int>(A.n);
            t.nc = static_cast<int>(Li.T->nc);
            t.rp = A.rp;
            t.col = A.col;
            t.val = A.val;
            t.w = Li.w.get();
            t.agg = Li.T->agg.get();
            t.mptr = Li.T->mptr.get();
            t.midx = Li.T->midx.get();
            t.f = fin[l];
            t.u0 = W.u[l].get();
            t.r = W.r[l].get();
            t.fc = W.f[l + 1].get();
            t.u0c = l + 2 < L ? W.u[l + 1].get() : nullptr;
            t.wc = l + 2 < L ? h.lv[l + 1].w.get() : nullptr;
            t.uout = l == s ? u : W.t[l].get();
            t.ec = l + 2 < L ? W.t[l + 1].get() : W.u[L - 1].get();
            ufinal[l] = t.uout;
        }
        c.cur_level = static_cast<int>(top);
        tail_down(c, td, om, g);
    }
    // coarsest: direct solve (hierarchy.cpp:175)
    c.cur_level = static_cast<int>(L - 1);
    coarse_solve(h, W.f[L - 1].get(), W.u[L - 1].get(), g);
    ufinal[L - 1] = W.u[L - 1].get();
    if (ts >= 0) {
        c.cur_level = static_cast<int>(top);
        tail_up(c, td, om, g);
    }
    // up leg
    for (size_t i = top; i-- > s;) {
        c.cur_level = static_cast<int>(i);
        const Level& Li = h.lv[i];
        const CsrView A = Li.view();
        double* a = cur[i];
        double* b = (a == W.u[i].get()) ? W.t[i].get() : W.u[i].get();
        auto prolong = [&](double* dst) {
            if (fold && i == s)
                vc_prolong_premul(c, A.n, fin[i], Li.w.get(), oml(i), Li.T->agg.get(), ufinal[i + 1], dst, g);
            else
                prolong_level(c, Li, a, ufinal[i + 1], dst, g);
        };
        if (post <= 0) {
            double* t = (i == s) ? u : b;
            prolong(t);
            ufinal[i] = t;
            continue;
        }
        // x = u + P u_c into b, then the post-smoothing sweeps
        prolong(b);
        double* src = b;
        for (int k = 1; k <= post; ++k) {
            double* dst = (i == s && k == post) ? u : (src == b ? a : b);
            if (i == 0 && s == 0 && k == post && nx && !nx->done && lag_enabled() && W.lagdone.size() > 0) {
                // the last sweep + the caller's next SpMV in one pass over A_0
                // (lag_prepare ran before any graph capture)
                const int dg = h.lv[0].pat->lag_groups;
                if (smooth_then_spmv(c, A, fin[i], Li.w.get(), oml(i), src, dst, nx->kind, nx->y, nx->ab, nx->sink,
                                     W.lagdone.get(), dg, g)) {
                    nx->done = true;
                    src = dst;
                    continue;
                }
            }
            vc_smooth(c, A, fin[i], Li.w.get(), oml(i), src, dst, g);
            src = dst;
        }
        ufinal[i] = src;
    }
    c.cur_level = -1;
}

void vcycle(Hier& h, const double* f, double* u, Gate g, NextSpmv* nx) { vcycle_from(h, 0, f, u, g, nx); }

// ---- BiCGStab (bicgstab.cpp:21-135) ------------------------------------------------
namespace {

struct KrylovBufs {
    double *r, *rt, *p, *v, *s, *t, *ph, *sh;
    double* q;  // sequential-dot mode only (else null)
};

KrylovBufs krylov_bufs(Hier& h) {
    Work& W = work(h);
    Ctx& c = *h.ctx;
    const int64_t n = h.lv.front().pat->n;
    if (W.kr.size() != n) {
        W.kr.alloc(n, c.stream);
        W.krt.alloc(n, c.stream);
        W.kp.alloc(n, c.stream);
        W.kv.alloc(n, c.stream);
        W.ks.alloc(n, c.stream);
        W.kt.alloc(n, c.stream);
        W.kph.alloc(n, c.stream);
        W.ksh.alloc(n, c.stream);
    }
    if (c.seq_dots && W.kq.size() != n) W.kq.alloc(n, c.stream);
    return {W.kr.get(), W.krt.get(), W.kp.get(), W.kv.get(), W.ks.get(), W.kt.get(), W.kph.get(), W.ksh.get(),
            c.seq_dots ? W.kq.get() : nullptr};
}

DotSink sink(Hier& h, double* out) {
    Work& W = work(h);
    return DotSink{W.partials.get(), W.ticket.get(), out};
}

KState read_state(Hier& h) {
    KState s;
    d2h(&s, work(h).st.get(), 1, h.ctx->stream);
    CK(cudaStreamSynchronize(h.ctx->stream));
    return s;
}

void write_state(Hier& h, const KState& s) {
    h2d(work(h).st.get(), &s, 1, h.ctx->stream);
}

#define ST_FIELD(st, f) (&(st)->f)

// Sequential-dot mode (Ctx::seq_dots, amgr_ctx_set_dot_order): after each
// kernel that produced a fused blocked dot, the same dot is recomputed strictly
// left to right (seq_dot) into the same state field, gated like the producer.
struct SeqDots {
    Ctx& c;
    int64_t n;
    bool on;
    void operator()(const double* a, const double* b, double* out, Gate g = {}) const {
        if (on) seq_dot(c, n, a, b, out, g);
    }
};

// ||f - A u||^2 into *out (the reference's true_residual sum, bicgstab.cpp:45-53;
// also norm2(r)^2 of the initial residual when r is given)
void resid_sq(Hier& h, const CsrView& A, const double* f, const double* u, double* r, double* r2,
              const KrylovBufs& B, double* out, Gate g = {}) {
    Ctx& c = *h.ctx;
    if (!c.seq_dots) {
        resid_norm(c, A, f, u, r, r2, DotSink{work(h).partials.get(), work(h).ticket.get(), out}, g);
        return;
    }
    double* d = r ? r : B.q;
    resid_norm(c, A, f, u, d, r2, DotSink{work(h).partials.get(), work(h).ticket.get(), out}, g);
    seq_dot(c, A.n, d, d, out, g);
}

}  // namespace

// Run gated Krylov iterations: the per-iteration kernel sequence is captured
// once into a CUDA graph (every kernel is gated on the device-side solver
// flags, so the sequence is static), then replayed with one iteration in
// flight ahead of the host's convergence check (flags copied to pinned memory
// and signalled by an event).  Falls back to direct launches while a kernel
// probe is active (probe events must bracket individual launches).
void run_iterations(Hier& h, const std::function<void()>& enqueue_iter, KState& out, bool allow_graph) {
    Ctx& c = *h.ctx;
    KState* st = work(h).st.get();
    static thread_local KState* pinned = nullptr;
    if (!pinned) CK(cudaMallocHost(reinterpret_cast<void**>(&pinned), 2 * sizeof(KState)));
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    cudaGraphExec_t exec = nullptr;
    int64_t per_iter = 0;
    const bool use_graph = allow_graph && c.probe.family.empty() && !getenv("AMGR_NO_GRAPH");
    if (use_graph) {
        // no stream-ordered allocation may happen inside the capture (it would
        // become a graph-owned allocation that blocks relaunching the graph)
        ensure_cheb_work(h);
        cudaGraph_t graph;
        const int64_t l0 = c.launches;
        const auto t0 = std::chrono::steady_clock::now();
        CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
        enqueue_iter();
        CK(cudaStreamEndCapture(c.stream, &graph));
        per_iter = c.launches - l0;
        c.launches = l0;
        CK(cudaGraphInstantiate(&exec, graph, 0));
        CK(cudaGraphDestroy(graph));
        if (std::getenv("AMGR_TRACE_SOLVE"))
            std::fprintf(stderr, "[amgr solve] capture + instantiate of one iteration (%lld kernels): %.2f ms\n",
                         static_cast<long long>(per_iter),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    auto launch = [&](int slot) {
        if (use_graph) {
            CK(cudaGraphLaunch(exec, c.stream));
            c.launches += per_iter;
        } else {
            enqueue_iter();
        }
        CK(cudaMemcpyAsync(&pinned[slot], st, sizeof(KState), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaEventRecord(ev[slot], c.stream));
    };
    int64_t k = 0;
    launch(0);
    for (;;) {
        ++k;
        launch(static_cast<int>(k & 1));  // one iteration ahead (gated off if already done)
        CK(cudaEventSynchronize(ev[(k - 1) & 1]));
        if (pinned[(k - 1) & 1].flags & KF_DONE) break;
    }
    CK(cudaStreamSynchronize(c.stream));
    if (exec) CK(cudaGraphExecDestroy(exec));
    CK(cudaEventDestroy(ev[0]));
    CK(cudaEventDestroy(ev[1]));
    out = read_state(h);
}

void bicgstab(Hier& h, const double* f, const double* u0, double* u, const amgr_solve_params& sp,
              amgr_solve_stats& out) {
    if (sp.tol <= 0.0) invalid("bicgstab: tol must be positive");
    if (sp.max_iter < 1) invalid("bicgstab: max_iter must be >= 1");
    Ctx& c = *h.ctx;
    const CsrView A = h.lv.front().view();
    const int64_t n = A.n;
    KrylovBufs B = krylov_bufs(h);
    KState* st = work(h).st.get();
    out = amgr_solve_stats{0, 0.0, 0, 0};

    const SeqDots SD{c, n, c.seq_dots};
    KState s0;
    write_state(h, s0);
    dot(c, n, f, f, sink(h, ST_FIELD(st, d_true)));
    SD(f, f, ST_FIELD(st, d_true));
    KState s = read_state(h);
    const double normf = std::sqrt(s.d_true);
    if (normf == 0.0) {
        fill(c, u, n, 0.0);
        out.converged = 1;
        return;
    }
    if (u != u0) copy(c, u, u0, n);
    // r = f - A u ; rtilde = r   (bicgstab.cpp:41-43)
    resid_sq(h, A, f, u, B.r, B.rt, B, ST_FIELD(st, d_rr));
    dot(c, n, B.rt, B.r, sink(h, ST_FIELD(st, d_rtr)));
    SD(B.rt, B.r, ST_FIELD(st, d_rtr));
    s = read_state(h);
    out.relative_residual = std::sqrt(s.d_rr) / normf;
    if (out.relative_residual <= sp.tol) {
        resid_sq(h, A, f, u, nullptr, nullptr, B, ST_FIELD(st, d_true));
        s = read_state(h);
        out.relative_residual = std::sqrt(s.d_true) / normf;
        if (out.relative_residual <= sp.tol) {
            out.converged = 1;
            return;
        }
    }
    s.normf = normf;
    s.floor = 1e-30 * normf * normf;
    s.tol = sp.tol;
    s.max_iter = sp.max_iter;
    s.rho_old = 1.0;
    s.alpha = 1.0;
    s.omega = 1.0;
    s.it = 0;
    s.flags = 0;
    write_state(h, s);

    if (lag_enabled() && h.lv.size() > 1) lag_prepare(h);
    const Gate G = gate_of(st, KF_DONE);
    const Gate GH = gate_of(st, KF_DONE, KF_HALF);
    const Gate GF = gate_of(st, KF_DONE | KF_HALF);
    const Gate GC = gate_of(st, KF_DONE | KF_HALF, KF_CHECK);
    auto iter = [&]() {
        bicg_begin(c, st);
        bicg_p(c, st, n, B.r, B.p, B.v);
        NextSpmv n1{1, B.v, B.rt, sink(h, ST_FIELD(st, d_rtv))};
        vcycle(h, B.p, B.ph, G, &n1);
        if (!n1.done) spmv_dot(c, A, B.ph, B.v, B.rt, sink(h, ST_FIELD(st, d_rtv)), G);
        SD(B.rt, B.v, ST_FIELD(st, d_rtv), G);
        bicg_alpha(c, st);
        bicg_s(c, st, n, B.r, B.v, B.s, sink(h, ST_FIELD(st, d_ss)));
        SD(B.s, B.s, ST_FIELD(st, d_ss), G);
        bicg_half_test(c, st);
        bicg_half_u(c, st, n, u, B.ph);
        resid_sq(h, A, f, u, nullptr, nullptr, B, ST_FIELD(st, d_true), GH);
        bicg_half_check(c, st);
        bicg_half_r(c, st, n, B.r, B.s, B.rt, sink(h, ST_FIELD(st, d_rtr)));
        SD(B.rt, B.r, ST_FIELD(st, d_rtr), GH);
        NextSpmv n2{2, B.t, B.s, sink(h, ST_FIELD(st, d_ts))};
        vcycle(h, B.s, B.sh, GF, &n2);
        if (!n2.done) spmv_dot2(c, A, B.sh, B.t, B.s, sink(h, ST_FIELD(st, d_ts)), GF);
        SD(B.t, B.s, ST_FIELD(st, d_ts), GF);
        SD(B.t, B.t, ST_FIELD(st, d_tt), GF);
        bicg_omega(c, st);
        bicg_update(c, st, n, u, B.ph, B.sh, B.r, B.s, B.t, B.rt, sink(h, ST_FIELD(st, d_rr)));
        SD(B.r, B.r, ST_FIELD(st, d_rr), GF);
        SD(B.rt, B.r, ST_FIELD(st, d_rtr), GF);
        bicg_end_test(c, st);
        resid_sq(h, A, f, u, nullptr, nullptr, B, ST_FIELD(st, d_true), GC);
        bicg_end_check(c, st);
    };
    run_iterations(h, iter, s);
    out.iterations = s.it;
    if (s.flags & KF_CONVERGED) {
        out.converged = 1;
        out.relative_residual = s.res;
        return;
    }
    out.breakdown = (s.flags & KF_BREAKDOWN) ? 1 : 0;
    resid_sq(h, A, f, u, nullptr, nullptr, B, ST_FIELD(st, d_true));
    s = read_state(h);
    out.relative_residual = std::sqrt(s.d_true) / normf;
    out.converged = (out.relative_residual <= sp.tol && !out.breakdown) ? 1 : 0;
}

// ---- preconditioned CG (extension; restated oracle in oracle/amg_oracle.c) ------------
void cg(Hier& h, const double* f, const double* u0, double* u, const amgr_solve_params& sp,
        amgr_solve_stats& out) {
    if (sp.tol <= 0.0) invalid("cg: tol must be positive");
    if (sp.max_iter < 1) invalid("cg: max_iter must be >= 1");
    Ctx& c = *h.ctx;
    const CsrView A = h.lv.front().view();
    const int64_t n = A.n;
    KrylovBufs B = krylov_bufs(h);
    KState* st = work(h).st.get();
    out = amgr_solve_stats{0, 0.0, 0, 0};
    const SeqDots SD{c, n, c.seq_dots};
    KState s0;
    write_state(h, s0);
    dot(c, n, f, f, sink(h, ST_FIELD(st, d_true)));
    SD(f, f, ST_FIELD(st, d_true));
    KState s = read_state(h);
    const double normf = std::sqrt(s.d_true);
    if (normf == 0.0) {
        fill(c, u, n, 0.0);
        out.converged = 1;
        return;
    }
    if (u != u0) copy(c, u, u0, n);
    resid_sq(h, A, f, u, B.r, nullptr, B, ST_FIELD(st, d_rr));
    s = read_state(h);
    out.relative_residual = std::sqrt(s.d_rr) / normf;
    if (out.relative_residual <= sp.tol) {
        out.converged = 1;
        return;
    }
    // z = M r ; p = z ; rho = r.z
    vcycle(h, B.r, B.s, {});
    copy(c, B.p, B.s, n);
    dot(c, n, B.r, B.s, sink(h, ST_FIELD(st, d_rz)));
    SD(B.r, B.s, ST_FIELD(st, d_rz));
    s = read_state(h);
    s.normf = normf;
    s.floor = 1e-30 * normf * normf;
    s.tol = sp.tol;
    s.max_iter = sp.max_iter;
    s.rho = s.d_rz;
    s.it = 0;
    s.flags = 0;
    write_state(h, s);
    const Gate G = gate_of(st, KF_DONE);
    const Gate GC = gate_of(st, KF_DONE, KF_CHECK);
    auto iter = [&]() {
        cg_begin(c, st);
        spmv_dot(c, A, B.p, B.v, B.p, sink(h, ST_FIELD(st, d_pq)), G);
        SD(B.p, B.v, ST_FIELD(st, d_pq), G);
        cg_alpha(c, st);
        cg_update(c, st, n, u, B.r, B.p, B.v, sink(h, ST_FIELD(st, d_rr)));
        SD(B.r, B.r, ST_FIELD(st, d_rr), G);
        cg_test(c, st);
        resid_sq(h, A, f, u, nullptr, nullptr, B, ST_FIELD(st, d_true), GC);
        cg_check(c, st);
        vcycle(h, B.r, B.s, G);
        dot(c, n, B.r, B.s, sink(h, ST_FIELD(st, d_rz)), G);
        SD(B.r, B.s, ST_FIELD(st, d_rz), G);
        cg_beta(c, st);
        cg_p(c, st, n, B.s, B.p);
    };
    run_iterations(h, iter, s);
    out.iterations = s.it;
    if (s.flags & KF_CONVERGED) {
        out.converged = 1;
        out.relative_residual = s.res;
        return;
    }
    out.breakdown = (s.flags & KF_BREAKDOWN) ? 1 : 0;
    resid_sq(h, A, f, u, nullptr, nullptr, B, ST_FIELD(st, d_true));
    s = read_state(h);
    out.relative_residual = std::sqrt(s.d_true) / normf;
    out.converged = (out.relative_residual <= sp.tol && !out.breakdown) ? 1 : 0;
}

}  // namespace amgr

// ---- single-operator entry points (the reference's free functions) ------------------
// spmv (csr.cpp:76-85), build_smoother / smooth (smoother.cpp:8-48),
// coarse_factorize / coarse_solve (dense_lu.cpp:10-73) on one matrix, for the
// source-compatible C++ facade (include/amgreuse_gpu.hpp).  Same kernels and
// arithmetic order as inside the hierarchy.
namespace amgr {

namespace {
struct OneMatrix {
    std::shared_ptr<Pattern> pat;
    DevArray<double> val;
    CsrView view() const { return csr_view(*pat, val.get()); }
};
OneMatrix one_matrix(Ctx& c, const amgr_csr& A) {
    OneMatrix m;
    m.pat = make_pattern(c, A);
    upload_values(c, m.val, A.values, A.nnz, A.location);
    return m;
}
}  // namespace

void op_spmv(Ctx& c, const amgr_csr& A, const double* x, double* y) {
    OneMatrix M = one_matrix(c, A);
    spmv(c, M.view(), x, y);
}

void op_build_smoother(Ctx& c, const amgr_csr& A, double* w) {
    if (A.nrows != A.ncols) invalid("build_smoother: matrix is not square");
    OneMatrix M = one_matrix(c, A);
    DevArray<int> bad(1, c.stream);
    const int big = 0x7fffffff;
    h2d(bad.get(), &big, 1, c.stream);
    jacobi_rebuild(c, A.nrows, M.val.get(), M.pat->diag.get(), w, bad.get());
    const int b = d2h_scalar(bad.get(), c.stream);
    if (b != big) {
        std::ostringstream os;
        os << "build_smoother: zero diagonal at row " << b;
        invalid(os.str());
    }
}

void op_smooth(Ctx& c, const amgr_csr& A, const double* w, double omega, const double* f, double* u, int sweeps) {
    if (A.nrows != A.ncols) invalid("smooth: matrix is not square");
    if (sweeps <= 0) return;
    OneMatrix M = one_matrix(c, A);
    DevArray<double> t(A.nrows, c.stream);
    double* cur = u;
    double* nxt = t.get();
    for (int s = 0; s < sweeps; ++s) {
        vc_smooth(c, M.view(), f, w, omega, cur, nxt);
        std::swap(cur, nxt);
    }
    if (cur != u) d2d(u, cur, A.nrows, c.stream);
    CK(cudaStreamSynchronize(c.stream));
}

void op_coarse_factorize(Ctx& c, const amgr_csr& A, double* lu_host, int64_t* piv_host) {
    if (A.nrows != A.ncols) invalid("coarse_factorize: matrix is not square");
    const int64_t n = A.nrows;
    OneMatrix M = one_matrix(c, A);
    DevArray<double> lu(n * n, c.stream);
    DevArray<int64_t> piv(n, c.stream);
    DevArray<int> perm(n, c.stream), st(1, c.stream);
    const int ok = -1;
    h2d(st.get(), &ok, 1, c.stream);
    if (!lu_factor_csr(c, M.view(), lu.get(), piv.get(), st.get(), perm.get())) {
        lu_densify(c, M.view(), lu.get());
        lu_factor(c, n, lu.get(), piv.get(), st.get(), perm.get());
    }
    const int s = d2h_scalar(st.get(), c.stream);
    if (s >= 0) throw_lu(s);
    d2h(lu_host, lu.get(), n * n, c.stream);
    d2h(piv_host, piv.get(), n, c.stream);
    CK(cudaStreamSynchronize(c.stream));
}

void op_coarse_solve(Ctx& c, int64_t n, const double* lu_host, const int64_t* piv_host, const double* rhs,
                     double* x) {
    if (n == 0) return;
    DevArray<double> lu(n * n, c.stream), b(n, c.stream);
    DevArray<int64_t> piv(n, c.stream);
    h2d(lu.get(), lu_host, n * n, c.stream);
    h2d(piv.get(), piv_host, n, c.stream);
    h2d(b.get(), rhs, n, c.stream);
    lu_solve(c, n, lu.get(), piv.get(), b.get(), b.get());
    d2h(x, b.get(), n, c.stream);
    CK(cudaStreamSynchronize(c.stream));
}

}  // namespace amgr

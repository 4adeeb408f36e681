// Host-side orchestration of the device hierarchy (C++).  Mirrors the
// reference's Hierarchy / setup / partial_update / vcycle / bicgstab
// (proj/include/amgreuse/hierarchy.hpp, bicgstab.hpp) with device storage.
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "krylov.cuh"
#include "setup.cuh"

namespace amgr {

struct AmgP {
    double eps = 0.08, omega = 0.72;
    int pre = 1, post = 1;
    int64_t coarse_enough = 100, max_direct = 2000;
    int smoother = AMGR_SMOOTHER_JACOBI;
    int coarsening = AMGR_COARSENING_PLAIN;
    double sa_omega = 2.0 / 3.0;
    int cheb_degree = 3, power_iters = 10;
    double cheb_lower = 0.3, cheb_safety = 1.1;
    int coarse_solve = AMGR_COARSE_EXACT;
};
AmgP to_amgp(const amgr_amg_params* p);

// Structure of one level's operator (immutable, shared between hierarchies).
struct Pattern {
    int64_t n = 0, ncols = 0, nnz = 0;
    int max_span = 0;
    DevArray<int> rp, col, diag;
    ColCode cc;  // coded column stream for the row passes (mode 0: none)
    int lag_groups = -1;  // max |j - i| / 32 + 2 of a coded pattern (k_rowpass_lag), lazily
    // symmetric-stencil form (level 0): -1 not examined, 0 not a symmetric
    // stencil, else the number K of offset pairs (doff ascending) + row masks
    int dia_k = -1;
    int doff[3] = {0, 0, 0};
    DevArray<uint8_t> dmask;
};
inline void set_code(CsrView& v, const ColCode& cc) {
    v.cmode = cc.mode;
    v.ndict = cc.ndict;
    v.code = cc.mode == 1 ? static_cast<const void*>(cc.c8.get())
                          : cc.mode == 2 ? static_cast<const void*>(cc.c16.get()) : nullptr;
    v.dict = cc.mode ? cc.dict.get() : nullptr;
}
// Frozen transfer operators of one level: P (agg) and R = P^T (mptr/midx).
// Smoothed aggregation (extension) additionally keeps the general P and R.
struct Transfer {
    int64_t nf = 0, nc = 0;
    DevArray<int> agg, mptr, midx;
    bool smoothed = false;
    std::shared_ptr<struct Pattern> P, R;  // P: nf x nc, R = P^T: nc x nf
    DevArray<double> Pv, Rv;
};
// Cached Galerkin plan A_i -> A_{i+1}.
struct RapPlan {
    int64_t nnz_f = 0, nnz_c = 0;
    // smoothed aggregation: A_{i+1} = R (A P) as two plan-based numeric SpGEMMs
    std::shared_ptr<SpgPlan> ap, rap;
    DevArray<double> ap_val;
    int max_chunk = -1;  // largest contrib count of a k_rap_tma chunk (-1: not computed)
    DevArray<int> cptr, contrib;
    RowPlan rows;        // member-row plan (k_rap_rows) when the level fits
    bool rows_tried = false;
    GrpPlan grp;         // warp-group plan (k_rap_grp, default) when the level fits
    bool grp_tried = false;
};

inline CsrView csr_view(const Pattern& p, const double* val) {
    CsrView v;
    v.n = p.n;
    v.ncols = p.ncols;
    v.nnz = p.nnz;
    v.rp = p.rp.get();
    v.col = p.col.get();
    v.val = val;
    v.max_span = p.max_span;
    set_code(v, p.cc);
    return v;
}

struct Level {
    std::shared_ptr<Pattern> pat;
    DevArray<double> val;  // A_i values
    const double* ext_val = nullptr;  // adopted (zero-copy) A_0 values, see AMGR_DEVICE_ADOPT
    DevArray<double> w;    // smoother diagonal (inv_diag for Jacobi)
    DevArray<double> cheb; // Chebyshev coefficients (extension): theta, c1/c2 per step, hi
    DevArray<double> pst;  // power-iteration state {yy, xx, lam}
    bool has_smoother = false;
    double om = -1.0;  // per-level Jacobi weight of an SA hierarchy (sa_jacobi_weights); < 0: prm's
    std::shared_ptr<Transfer> T;   // null on the coarsest level
    std::shared_ptr<RapPlan> rap;  // null on the coarsest level
    // symmetric-stencil copy of this level's values (level 0; D | U_0..U_{K-1})
    // and its bit-symmetry flag; dia_on when the last rebuild found them equal
    DevArray<double> dia;
    DevArray<int> dia_flag;
    bool dia_on = false;
    CsrView view() const {
        CsrView v;
        v.n = pat->n;
        v.ncols = pat->ncols;
        v.nnz = pat->nnz;
        v.rp = pat->rp.get();
        v.col = pat->col.get();
        v.val = ext_val ? ext_val : val.get();
        v.max_span = pat->max_span;
        set_code(v, pat->cc);
        if (dia_on) {
            v.dia = dia.get();
            v.dmask = pat->dmask.get();
            v.dk = pat->dia_k;
            for (int k = 0; k < 3; ++k) v.doff[k] = pat->doff[k];
        }
        return v;
    }
};

// Per-shape work vectors, shared by hierarchies of the same shape (one
// context is single-threaded by contract).
struct Work {
    std::vector<DevArray<double>> u, t, f, r;
    std::vector<DevArray<double>> d0, d1;  // Chebyshev direction vectors (lazily allocated)
    DevArray<double> kr, krt, kp, kv, ks, kt, kph, ksh;
    DevArray<double> kq;  // sequential-dot mode: f - A u scratch
    DevArray<int> lagdone;  // k_rowpass_lag round counters
    DevArray<KState> st;
    DevArray<double> partials;
    DevArray<unsigned> ticket;
    DevArray<int> err;  // per level bad row (+1 slot for LU status)
    std::vector<int64_t> shape;
};

struct Timer {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[4];
};

struct Hier {
    Ctx* ctx = nullptr;
    AmgP prm;
    std::vector<Level> lv;
    DevArray<double> lu;
    bool lu_formed = false;   // false in the inverse mode when the direct Gauss-Jordan kernel ran
    DevArray<int64_t> piv;
    DevArray<int> perm;    // composed pivot swaps (lu_solve fast path)
    DevArray<double> inv;  // AMGR_COARSE_INVERSE
    DevArray<double> staged;  // next step's A_0 values (amgr_stage_values)
    cudaEvent_t staged_ev = nullptr, main_ev = nullptr;
    bool staged_ready = false;
    // staged right-hand side (amgr_stage_rhs): committed into rhs by the next
    // STAGED rebuild (or STAGED solve), read by amgr_bicgstab/amgr_cg(AMGR_STAGED)
    DevArray<double> staged_rhs, rhs;
    cudaEvent_t rhs_ev = nullptr;
    bool rhs_staged = false, rhs_ready = false;
    ~Hier();
    int64_t nL = 0;
    amgr_phase_timings tm{};
    std::shared_ptr<Work> ws;
    int64_t agg_rounds = 0;

    double om_eff() const { return prm.smoother == AMGR_SMOOTHER_SPAI0 ? 1.0 : prm.omega; }
    double om_level(size_t l) const { return l < lv.size() && lv[l].om > 0.0 ? lv[l].om : om_eff(); }
};

std::unique_ptr<Hier> setup(Ctx& c, const amgr_csr& A, const AmgP& p);
std::unique_ptr<Hier> partial_update(const Hier& h, const amgr_csr& A, const AmgP& p);
void rebuild(Hier& h, const amgr_csr& A);
// numeric rebuild of levels start.. from the values already in level `start`
void rebuild_levels_from(Hier& h, size_t start);
// single-operator entry points (device vectors; lu/piv/rhs/x of the LU pair on the host)
void op_spmv(Ctx& c, const amgr_csr& A, const double* x, double* y);
void op_build_smoother(Ctx& c, const amgr_csr& A, double* w);
void op_smooth(Ctx& c, const amgr_csr& A, const double* w, double omega, const double* f, double* u, int sweeps);
void op_coarse_factorize(Ctx& c, const amgr_csr& A, double* lu_host, int64_t* piv_host);
void op_coarse_solve(Ctx& c, int64_t n, const double* lu_host, const int64_t* piv_host, const double* rhs, double* x);
void rebuild_values(Hier& h, const double* values, int location);
void stage_values(Hier& h, const double* values, int location);
void stage_rhs(Hier& h, const double* f, int location);
// the RHS committed by the last STAGED rebuild (amgr_stage_rhs staged it)
const double* committed_rhs(Hier& h);
void commit_rhs(Hier& h);
// The SpMV a Krylov solver applies to the V-cycle's output next (v = A u with
// its dots): vcycle() fuses it into the last level-0 smoothing sweep
// (smooth_then_spmv) when it can and sets done; else the caller runs it.
struct NextSpmv {
    int kind = 1;            // 1: spmv_dot (out[0] = ab . y), 2: spmv_dot2 (y . ab, y . y)
    double* y = nullptr;
    const double* ab = nullptr;
    DotSink sink;
    bool done = false;
};
void vcycle(Hier& h, const double* f, double* u, Gate g = {}, NextSpmv* nx = nullptr);
void vcycle_from(Hier& h, size_t s, const double* f, double* u, Gate g = {}, NextSpmv* nx = nullptr);
void bicgstab(Hier& h, const double* f, const double* u0, double* u, const amgr_solve_params& sp,
              amgr_solve_stats& st);
void cg(Hier& h, const double* f, const double* u0, double* u, const amgr_solve_params& sp,
        amgr_solve_stats& st);
Work& work(Hier& h);
// Enqueue Krylov iterations with one iteration of look-ahead (gated kernels
// no-op once KF_DONE is set), as one CUDA graph when allowed; returns the
// final device state.
void run_iterations(Hier& h, const std::function<void()>& enqueue_iter, KState& out, bool allow_graph = true);

// device generators (kernels_gen.cu)
int64_t problem_nnz(int64_t g);
void problem_pattern(Ctx& c, int64_t g, int* rp, int* col);
void problem_values(Ctx& c, int kind, int64_t g, int64_t k, int64_t nsteps, double* val);
void exclusive_sum_i32(Ctx& c, const int* in, int* out, int64_t n);

}  // namespace amgr

// Opaque C-ABI hierarchy handle (include/amgr.h).
struct amgr_hier {
    std::unique_ptr<amgr::Hier> h;
};

// Kernel launchers of libamgr_b200.so (sm_100a).  All arithmetic that the
// reference performs in a fixed order is replayed in the same order with
// explicit round-to-nearest intrinsics (the library is also compiled with
// --fmad=false), so level values, smoother state, the coarse LU and the
// V-cycle are bit-identical to the reference built with -ffp-contract=off
// (DESIGN.md §3).
#pragma once

#include "common.cuh"

namespace amgr {

// Device view of one level's matrix (CSR, int32 indices, fp64 values).
struct CsrView {
    int64_t n = 0;     // rows
    int64_t ncols = 0;
    int64_t nnz = 0;
    const int* rp = nullptr;
    const int* col = nullptr;
    const double* val = nullptr;
    int max_span = 0;  // widest 16-byte-aligned nnz span of a 32-row group (row-pass chunk sizing)
    // coded column stream (encode_columns): col_k = row + dict[code_k]
    // cmode 0 = raw int32 columns, 1 = uint8 codes, 2 = uint16 codes
    int cmode = 0;
    int ndict = 0;
    const void* code = nullptr;
    const int* dict = nullptr;
    // symmetric-stencil form of level 0 (sym_dia, hierarchy.cu): when dia is
    // set, the row passes read D | U_0 .. U_{dk-1} (n values each; U_k[i] =
    // a(i, i + doff[k]), and a(i, i - doff[k]) = U_k[i - doff[k]]) and a
    // presence mask per row instead of the CSR arrays
    const double* dia = nullptr;
    const uint8_t* dmask = nullptr;
    int dk = 0;
    int doff[3] = {0, 0, 0};
};

// Deterministic multi-block dot products: per-block partials + last-block
// fixed-order final sum (no atomics on the values).
struct DotSink {
    double* partials = nullptr;   // [grid * ndot]
    unsigned* ticket = nullptr;   // zero-initialised counter
    double* out = nullptr;        // [ndot]
};

// Fixed grid for dot-producing kernels so the reduction order never changes.
int dot_grid(const Ctx& c);

// ---- symmetric-stencil form (level 0) -----------------------------------------
// presence masks of a pattern whose columns are i + {-off[K-1]..-off[0], 0,
// off[0]..off[K-1]} in ascending order and structurally symmetric; false (and
// no mask) otherwise.  Host sync.
bool dia_masks(Ctx& c, const CsrView& A, int K, const int* off, uint8_t* mask);
// D | U_0..U_{K-1} from the CSR values; *flag |= 1 when a(i, j) and a(j, i)
// differ in any bit (the form is then unusable for these values)
void dia_values(Ctx& c, const CsrView& A, int K, const int* off, const uint8_t* mask, double* dia, int* flag);

// ---- row-pass (CSR SpMV family) --------------------------------------------
void spmv(Ctx& c, const CsrView& A, const double* x, double* y, Gate g = {});
// r = f - A x
void residual(Ctx& c, const CsrView& A, const double* f, const double* x, double* r, Gate g = {});
// V-cycle down leg (hierarchy.cpp:165-172).  The first pre-smoothing sweep
// from a zero guess is u0 = 0 + (om*w) f: written by vc_premul on level 0 and
// by restrict_sum for coarser levels; vc_down then forms r = f - A u0.
void vc_premul(Ctx& c, int64_t n, const double* f, const double* w, double om, double* u0, Gate g = {});
void vc_down(Ctx& c, const CsrView& A, const double* f, const double* u0, double* r, Gate g = {});
// one smoothing sweep: out = u + (om*w)(f - A u)     (smoother.cpp:42-47)
// the same passes over a list of rows (bit-identical per row)
void vc_down_rows(Ctx& c, const CsrView& A, const int* rows, int64_t nrows, const double* f, const double* u0,
                  double* r, Gate g = {});
void vc_smooth_rows(Ctx& c, const CsrView& A, const int* rows, int64_t nrows, const double* f, const double* w,
                    double om, const double* u, double* out, Gate g = {});
void vc_smooth(Ctx& c, const CsrView& A, const double* f, const double* w, double om,
               const double* u, double* out, Gate g = {});
// prolongation (hierarchy.cpp:179-182): out = u + (0 + uc[agg])
// smoothed aggregation (extension): restriction / prolongation with general
// R and P (row passes over their CSR)
void vc_restrict_general(Ctx& c, const CsrView& R, const double* r, double* fc, const double* wc, double om,
                         double* u0c, Gate g);
void vc_prolong_general(Ctx& c, const CsrView& P, const double* u, const double* e, double* out, Gate g);
// premul folded into the top level's down leg and prolongation (pre == 1)
void vc_down_premul(Ctx& c, const CsrView& A, const double* f, const double* w, double om, double* r, Gate g);
void vc_prolong_premul(Ctx& c, int64_t n, const double* f, const double* w, double om, const int* agg,
                       const double* uc, double* out, Gate g);
void vc_prolong(Ctx& c, int64_t n, const double* u, const int* agg, const double* uc, double* out,
                Gate g = {});
// restriction fc[I] = sum over members ascending of r[m] (R spmv, csr.cpp:79-84);
// if u0c != nullptr also u0c = 0 + (om*wc) fc for the coarse level's pre-smoothing
void restrict_sum(Ctx& c, int64_t nc, const int* mptr, const int* midx, const double* r, double* fc,
                  const double* wc, double om, double* u0c, Gate g = {});

// Krylov-fused SpMVs (dots land in sink.out):
// y = A x ; out[0] = a . y
void spmv_dot(Ctx& c, const CsrView& A, const double* x, double* y, const double* a, DotSink s,
              Gate g = {});
// y = A x ; out[0] = y . b ; out[1] = y . y
void spmv_dot2(Ctx& c, const CsrView& A, const double* x, double* y, const double* b, DotSink s,
               Gate g = {});
// Fused (k_rowpass_lag): one smoothing sweep out = u + (om*w)(f - A u) and
// then y = A out with the Krylov dots of spmv_dot (kind 1: out[0] = ab . y)
// or spmv_dot2 (kind 2: out[0] = y . ab, out[1] = y . y), in one persistent
// kernel that re-reads A from L2 for the second pass.  Bit-identical to
// vc_smooth + spmv_dot/spmv_dot2.  false: not applicable (only the coded
// 1-byte level-0 layout), nothing launched.  done: >= 64 * rounds ints of
// scratch; dgroups: max |j - i| / 32 + 2 over the matrix.
bool smooth_then_spmv(Ctx& c, const CsrView& A, const double* f, const double* w, double om, const double* u,
                      double* out, int kind, double* y, const double* ab, DotSink s, int* done, int dgroups,
                      Gate g = {});
// out[0] = || f - A x ||^2 ; optionally r = f - A x and r2 = r
void resid_norm(Ctx& c, const CsrView& A, const double* f, const double* x, double* r, double* r2,
                DotSink s, Gate g = {});

// ---- rebuild ---------------------------------------------------------------
// Numeric Galerkin product on the cached plan (two-level bracket of
// spmm(R, spmm(A, P)), csr.cpp:145-194).  crp/cdiag/wc/bad are reserved for
// a fused coarse-level smoother rebuild (currently a separate kernel).
// ---- V-cycle tail (kernels_tail.cu) ----
struct TailLevel {
    int n = 0, nc = 0;
    const int* rp = nullptr;
    const int* col = nullptr;
    const double* val = nullptr;
    const double* w = nullptr;     // smoother weights of level l
    const int* agg = nullptr;      // level l -> l+1
    const int* mptr = nullptr;     // members of the level-(l+1) rows
    const int* midx = nullptr;
    const double* f = nullptr;     // rhs of level l
    double* u0 = nullptr;          // first iterate (premul / restriction)
    double* r = nullptr;           // residual scratch
    double* fc = nullptr;          // rhs of level l+1
    double* u0c = nullptr;         // first iterate of level l+1 (null: l+1 is the coarsest)
    const double* wc = nullptr;    // smoother weights of level l+1
    double* uout = nullptr;        // up-leg result of level l
    const double* ec = nullptr;    // final iterate of level l+1
};
constexpr int TAIL_MAX = 16;
struct TailDesc {
    int count = 0;                 // levels first .. first+count-1 (all above the coarsest)
    TailLevel lv[TAIL_MAX];
};
void tail_down(Ctx& c, const TailDesc& d, double om, Gate g);
void tail_up(Ctx& c, const TailDesc& d, double om, Gate g);

// largest contrib count of any RT_CH-entry chunk of a plan (TMA stage size; host sync)
int rap_chunk_max(Ctx& c, int64_t nnz_c, const int* cptr);
// Fused damped-Jacobi rebuild of the COARSE level inside the numeric RAP:
// the thread that sums a coarse diagonal entry (flagged in cptr bit 30 by
// rap_symbolic) writes wc[I] = 1/(A_{i+1})_II; first zero -> bad_c.
struct RapJacobi {
    const int* ccol = nullptr;  // coarse columns (I of a flagged diagonal entry)
    double* wc = nullptr;
    int* bad_c = nullptr;
};
// returns true when the coarse Jacobi rebuild was fused (TMA path taken)
bool rap_numeric(Ctx& c, int64_t nf, int64_t nc, int64_t nnz_c, const int* cptr, const int* contrib, const double* af,
                 double* ac, int64_t nnz_f, int max_chunk = -1, const RapJacobi* fj = nullptr);
// Member-row numeric Galerkin product (RowPlan, setup.cuh) with the damped
// Jacobi rebuild fused in: wf (fine level, only the first RAP of the chain)
// and wc (coarse level, unless it is the coarsest) get 1.0 / a_ii, first bad
// rows into bad_f / bad_c (smoother.cpp:8-32).  Bit-identical to rap_numeric.
struct RapRowsArgs {
    int nc = 0, dmax = 0;
    const int* mptr = nullptr;       // R: members of coarse row I
    const int* midx = nullptr;       // R: fine row of member j (only read for wf)
    const int* mrp = nullptr;        // start of member row j's entries
    const uint8_t* mlen = nullptr;   // its length
    const uint16_t* code = nullptr;  // accumulation codes (RowPlan)
    const double* af = nullptr;
    const int* crp = nullptr;        // coarse row pointers
    const int* cdiag = nullptr;      // coarse diagonal positions (for wc)
    double* ac = nullptr;
    double* wf = nullptr;
    double* wc = nullptr;
    int* bad_f = nullptr;
    int* bad_c = nullptr;
};
void rap_rows(Ctx& c, const RapRowsArgs& a, int maxlen, int64_t nf, int64_t nnz_f, int64_t nnz_c);
// Warp-group numeric Galerkin product (GrpPlan, setup.cuh), default for
// plain-aggregation levels whose plan fits; with wf set it also rebuilds the
// fine level's damped-Jacobi weights (first bad row into bad_f).
// Bit-identical to rap_numeric + jacobi_rebuild.
struct GrpArgs {
    int64_t ngroups = 0;
    const int4* desc = nullptr;
    const int* mstart = nullptr;
    const uint8_t* mdoff = nullptr;
    const int* midx = nullptr;
    const uint16_t* code = nullptr;
    const uint16_t* lanes = nullptr;
    const double* af = nullptr;
    double* ac = nullptr;
    double* wf = nullptr;
    int* bad_f = nullptr;
};
void rap_grp(Ctx& c, const GrpArgs& a, int64_t nf, int64_t nc, int64_t nnz_f, int64_t nnz_c);
// the per-level first-bad-row slots (0x7fffffff) and the LU status slot (-1)
void reset_error_slots(Ctx& c, int* err, int64_t nlevels);
// Jacobi: w[i] = 1.0 / a_ii (smoother.cpp:8-32); records the first bad row.
void jacobi_rebuild(Ctx& c, int64_t n, const double* val, const int* diag_pos, double* w,
                    int* bad_row);
// SPAI0 (extension): w[i] = a_ii / sum_j a_ij^2
void spai0_rebuild(Ctx& c, const CsrView& A, const int* diag_pos, double* w, int* bad_row);

// ---- coarse direct solver (dense_lu.cpp) ------------------------------------
void lu_densify(Ctx& c, const CsrView& A, double* dense);
// in-place LU with partial pivoting; piv[k]; *status = -1 ok, else the zero-pivot step
// perm (optional, n ints): the composed row swaps for lu_solve's fast path
// A: the operator as CSR (the dense copy is staged in shared memory for
// n <= 160, else densified into m first); null: m holds it dense
void lu_factor(Ctx& c, int64_t n, double* m, int64_t* piv, int* status, int* perm = nullptr,
               const CsrView* A = nullptr);
// x = LU \ b in the reference's order; x may alias b.  With perm (from
// lu_factor) and n <= 160: the single-warp kernel (k_lu_solve_warp)
void lu_solve(Ctx& c, int64_t n, const double* m, const int64_t* piv, const double* b, double* x,
              Gate g = {}, const int* perm = nullptr);

// densify + factor + composed permutation in one single-CTA kernel (n <= 160,
// perm required; AMGR_LU_COLS=0 disables); false: use lu_densify + lu_factor
bool lu_factor_csr(Ctx& c, const CsrView& A, double* lu, int64_t* piv, int* status, int* perm);
// FAST mode (extension): explicit inverse from the LU factors, applied as a matvec
void lu_inverse(Ctx& c, int64_t n, const double* m, const int64_t* piv, double* inv);
// Gauss-Jordan inverse of the dense matrix a (n <= 160) straight into inv;
// false when n is outside the register-resident kernel's range.
bool dense_inverse_direct(Ctx& c, int64_t n, const double* a, double* inv, int64_t* piv, int* status);
void inv_apply(Ctx& c, int64_t n, const double* inv, const double* b, double* x, Gate g = {});

// ---- Chebyshev smoother (extension; oracle/amg_oracle.c smooth_cheb / power_lambda) ----
// power iteration step y = D^-1 A x with y.y -> s.out[0]; normalisation x = y/|y|,
// st = {yy, xx, lam} (lam = |y|/|x_prev|), x.x -> s.out (= st[1])
void power_step(Ctx& c, const CsrView& A, const double* w, const double* x, double* y, DotSink s);
void power_start(Ctx& c, int64_t n, double* x);
// atomicMax of max_i sum_j |a_ij| / |a_ii| into *out (double bits; zero it first)
void gershgorin_bound(Ctx& c, const CsrView& A, const int* dpos, unsigned long long* out);
void power_norm(Ctx& c, int64_t n, const double* y, double* x, double* st, DotSink s);
// coef[0] = theta, coef[2k-1], coef[2k] = c1, c2 of step k, coef[2*degree] = hi
void cheb_coef(Ctx& c, const double* st, double safety, double lower, int degree, double* coef);
void cheb_start(Ctx& c, const CsrView& A, const double* f, const double* w, const double* x, const double* coef,
                double* d, Gate g = {});
void cheb_zero(Ctx& c, int64_t n, const double* f, const double* w, const double* coef, double* d, Gate g = {});
void cheb_step(Ctx& c, const CsrView& A, const double* f, const double* w, const double* x, const double* d,
               const double* coef, int k, double* xout, double* dout, Gate g = {});
void axpy1(Ctx& c, int64_t n, double* x, const double* d, Gate g = {});

// ---- misc vector kernels ------------------------------------------------------
void fill(Ctx& c, double* x, int64_t n, double v, Gate g = {});
void copy(Ctx& c, double* dst, const double* src, int64_t n, Gate g = {});
void find_diag(Ctx& c, const CsrView& A, int* diag_pos);
void i32_to_i64(Ctx& c, const int* src, int64_t* dst, int64_t n);
void i64_to_i32(Ctx& c, const int64_t* src, int* dst, int64_t n, int* overflow);
// compare two int32 arrays; *diff set to 1 if any element differs
// widest aligned nnz span over 32-row groups
int max_group_span(Ctx& c, const int* rp, int64_t n);
void compare_i32(Ctx& c, const int* a, const int* b, int64_t n, int* diff);

}  // namespace amgr

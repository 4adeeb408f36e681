/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * partial-reuse AMG path (/root/reference/proj), the checker for the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load liboracle.so.  Never linked into the product.
 *
 * Pinning: restated functions are checked bit-for-bit against the reference
 * itself (oracle/_ref/libamgref.so, built from the reference sources) and
 * against the known answers of the reference's unit tests
 * (proj/tests/unit/test_*.cpp) in tests/test_oracle.py.  Extensions the reference
 * does not implement (SPAI0, Chebyshev + power iteration, smoothed
 * aggregation, CG, the 3D generators) are "parity unpinned": they are pinned
 * only by definitional known-answer tests.
 */
#ifndef AMG_ORACLE_H
#define AMG_ORACLE_H

#include <stdint.h>

typedef int64_t idx_t;

typedef struct {
    idx_t nrows, ncols;
    idx_t* rp; /* nrows+1 */
    idx_t* ci; /* nnz */
    double* v; /* nnz */
} ocsr;

typedef struct {
    double eps, omega;
    int32_t pre_sweeps, post_sweeps;
    idx_t coarse_enough, max_direct_size;
    int32_t smoother;   /* 0 jacobi, 1 spai0, 2 chebyshev (extensions 1,2) */
    int32_t coarsening; /* 0 plain, 1 smoothed aggregation (extension)     */
    double sa_omega;
    int32_t cheb_degree, power_iters;
    double cheb_lower, cheb_safety;
} oparams;

typedef struct ohier ohier;

/* errors: return 0 ok, 1 invalid_argument, 2 runtime_error; message in err */
idx_t o_nnz(const ocsr* A);
void o_free_csr(ocsr* A);

/* sparse core (proj/src/csr.cpp) */
void o_spmv(const ocsr* A, const double* x, double* y);
int o_transpose(const ocsr* A, ocsr* T);
int o_spmm(const ocsr* A, const ocsr* B, ocsr* C, char* err, int errlen);
int o_galerkin(const ocsr* R, const ocsr* A, const ocsr* P, ocsr* C, char* err, int errlen);

/* coarsening (proj/src/coarsening.cpp) */
int o_strength(const ocsr* A, double eps, idx_t** adj_ptr, idx_t** adj, char* err, int errlen);
idx_t o_aggregate(idx_t n, const idx_t* adj_ptr, const idx_t* adj, idx_t* assignment);

/* dense LU (proj/src/dense_lu.cpp) */
int o_factorize(const ocsr* A, double* lu, idx_t* piv, char* err, int errlen);
void o_coarse_solve(idx_t n, const double* lu, const idx_t* piv, const double* rhs, double* x);

/* hierarchy (proj/src/hierarchy.cpp) */
int o_setup(const ocsr* A, const oparams* p, ohier** out, char* err, int errlen);
int o_partial_update(const ohier* h, const ocsr* A, const oparams* p, ohier** out, char* err, int errlen);
void o_vcycle(const ohier* h, const double* f, double* u);
void o_free_hier(ohier* h);
int o_num_levels(const ohier* h);
/* dims: nrows, nnz, has_P, n_coarse, has_smoother, nnzP */
void o_level_dims(const ohier* h, int l, idx_t* dims);
void o_level_A(const ohier* h, int l, idx_t* rp, idx_t* ci, double* v);
void o_level_P(const ohier* h, int l, idx_t* rp, idx_t* ci, double* v);
void o_level_R(const ohier* h, int l, idx_t* rp, idx_t* ci, double* v);
void o_level_smoother(const ohier* h, int l, double* w, double* extra);
idx_t o_coarse_n(const ohier* h);
void o_coarse(const ohier* h, double* lu, idx_t* piv);

/* Krylov (proj/src/bicgstab.cpp) + CG extension.
 * stats: [iterations, converged, breakdown] */
int o_bicgstab(const ohier* h, const double* f, const double* u0, double* u, double tol, idx_t max_iter,
               idx_t* stats, double* relres);
int o_cg(const ohier* h, const double* f, const double* u0, double* u, double tol, idx_t max_iter,
         idx_t* stats, double* relres);

/* generators: 0 poisson+shift, 1 blob, 2 dam-break, 3 conv-diff */
int o_grid3d(int kind, idx_t g, idx_t k, idx_t nsteps, idx_t* rp, idx_t* ci, double* v);

#endif

// amgreuse_gpu.hpp — source-compatible C++ facade of the reference library
// `amgreuse` (proj/include/amgreuse/*.hpp) over the C-ABI of libamgr_b200.so
// (include/amgr.h).  Code written against the reference's headers compiles
// unchanged against these declarations (include/amgreuse/<name>.hpp forward
// here) and runs every algorithm on the B200:
//
//   reference entry point                       here (device path)
//   csr_from_triplets   csr.cpp:24-75           amgr_csr_from_triplets
//   spmv                csr.cpp:76-91           amgr_csr_spmv
//   build_smoother      smoother.cpp:8-32       amgr_build_smoother
//   smooth              smoother.cpp:34-54      amgr_smooth
//   coarse_factorize    dense_lu.cpp:10-50      amgr_coarse_factorize
//   coarse_solve        dense_lu.cpp:52-73      amgr_coarse_solve
//   setup               hierarchy.cpp:45-105    amgr_setup (+ downloads)
//   partial_update      hierarchy.cpp:107-150   amgr_partial_update
//   vcycle              hierarchy.cpp:152-186   amgr_vcycle
//   bicgstab(h, ...)    bicgstab.cpp:21-135     amgr_bicgstab
//
// Host containers (CsrMatrix, Hierarchy::levels, ...) are value copies of the
// device data with the reference's layout (int64 indices), so tests can
// inspect them; a Hierarchy also owns its device handle.  Exceptions and
// their texts are the reference's (std::invalid_argument /
// std::runtime_error).
//
// Deliberate difference: `smooth(s, A, f, u, sweeps)` with a
// non-const std::vector lvalue `u` smooths IN PLACE, as SPEC.md documents and
// the reference's own unit tests expect; the reference's overload set binds
// that call to the copy-returning overload and drops the result.  The copy
// overloads remain for const lvalues and temporaries.
#pragma once

#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

struct amgr_ctx;
struct amgr_hier;

namespace amgreuse {

using index_t = std::int64_t;

// ---- sparse storage -------------------------------------------------------------------
struct Triplet {
    index_t row;
    index_t col;
    double value;
};

struct CsrMatrix {
    index_t nrows = 0;
    index_t ncols = 0;
    std::vector<index_t> row_ptr{0};
    std::vector<index_t> col_idx;
    std::vector<double> values;

    index_t nnz() const { return static_cast<index_t>(col_idx.size()); }
    std::span<const index_t> row_cols(index_t i) const {
        return {col_idx.data() + row_ptr[i], static_cast<std::size_t>(row_ptr[i + 1] - row_ptr[i])};
    }
    std::span<const double> row_vals(index_t i) const {
        return {values.data() + row_ptr[i], static_cast<std::size_t>(row_ptr[i + 1] - row_ptr[i])};
    }
    bool operator==(const CsrMatrix&) const = default;
};

CsrMatrix csr_from_triplets(index_t nrows, index_t ncols, std::span<const Triplet> entries);
void spmv(const CsrMatrix& A, std::span<const double> x, std::span<double> y);
std::vector<double> spmv(const CsrMatrix& A, std::span<const double> x);
// R = P^T with rows ascending (host; the device keeps R as member lists)
CsrMatrix transpose(const CsrMatrix& A);

// ---- smoother ---------------------------------------------------------------------------
struct JacobiSmoother {
    std::vector<double> inv_diag;
    double omega = 0.72;
    bool operator==(const JacobiSmoother&) const = default;
};
JacobiSmoother build_smoother(const CsrMatrix& A, double omega);
void smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f, std::span<double> u, int sweeps);
void smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f, std::vector<double>& u,
            int sweeps);
std::vector<double> smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f,
                           const std::vector<double>& u, int sweeps);
std::vector<double> smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f,
                           std::vector<double>&& u, int sweeps);

// ---- coarsest-level direct solver ---------------------------------------------------
struct DenseFactorization {
    index_t n = 0;
    std::vector<double> lu;    // row-major, unit-lower L and U in place
    std::vector<index_t> piv;  // row swapped with k at step k
    bool operator==(const DenseFactorization&) const = default;
};
DenseFactorization coarse_factorize(const CsrMatrix& A);
std::vector<double> coarse_solve(const DenseFactorization& f, std::span<const double> rhs);

// ---- hierarchy ----------------------------------------------------------------------
struct AmgParams {
    double eps = 0.08;
    double omega = 0.72;
    int pre_sweeps = 1;
    int post_sweeps = 1;
    index_t coarse_enough = 100;
    index_t max_direct_size = 2000;
};

struct SetupPhaseTimings {
    double transfer_ops = 0.0;
    double galerkin = 0.0;
    double smoother = 0.0;
    double coarse_solver = 0.0;
    double total() const { return transfer_ops + galerkin + smoother + coarse_solver; }
};

struct Level {
    CsrMatrix A;
    std::shared_ptr<const CsrMatrix> P;
    std::shared_ptr<const CsrMatrix> R;
    std::optional<JacobiSmoother> smoother;
};

struct Hierarchy {
    std::vector<Level> levels;
    DenseFactorization coarse_solver;
    SetupPhaseTimings setup_timings;
    // the device hierarchy these host copies mirror (shared by copies)
    std::shared_ptr<amgr_hier> device;
    AmgParams params;

    std::size_t num_levels() const { return levels.size(); }
    index_t finest_size() const { return levels.empty() ? 0 : levels.front().A.nrows; }
    double operator_complexity() const;
};

Hierarchy setup(const CsrMatrix& A, const AmgParams& prm = {});
Hierarchy partial_update(const Hierarchy& h, CsrMatrix A_new, const AmgParams& prm = {});
std::vector<double> vcycle(const Hierarchy& h, std::span<const double> f, const AmgParams& prm = {});

// ---- Krylov -------------------------------------------------------------------------
struct SolveParams {
    double tol = 1e-8;
    index_t max_iter = 100;
};
struct SolveStats {
    index_t iterations = 0;
    double relative_residual = 0.0;
    bool converged = false;
    bool breakdown = false;
};
// bicgstab(make_operator(h.levels.front().A), make_preconditioner(h, prm), f, u0, solve),
// the whole iteration on the device
std::pair<std::vector<double>, SolveStats> bicgstab(const Hierarchy& h, std::span<const double> f,
                                                    std::span<const double> u0, const SolveParams& prm = {});

// the context every facade call uses (device 0, its own stream)
amgr_ctx* facade_context();

}  // namespace amgreuse

// Source-compatible C++ facade (include/amgreuse_gpu.hpp) over the C-ABI of
// libamgr_b200.so.  Every algorithm runs on the device through amgr.h; this
// file only converts between the reference's host containers (int64 CSR,
// std::vector) and the C-ABI, and turns status codes back into the
// reference's exception types with their messages.
#include "amgreuse_gpu.hpp"

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "amgr.h"

namespace amgreuse {

namespace {

[[noreturn]] void raise(amgr_status st, const char* fallback) {
    const char* m = amgr_last_error(facade_context());
    const std::string msg = (m && *m) ? m : fallback;
    if (st == AMGR_E_INVALID_ARGUMENT || st == AMGR_E_DIMENSION) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void check(amgr_status st, const char* what) {
    if (st != AMGR_OK) raise(st, what);
}

amgr_csr view(const CsrMatrix& A) {
    amgr_csr c{};
    c.nrows = A.nrows;
    c.ncols = A.ncols;
    c.nnz = A.nnz();
    c.row_ptr = A.row_ptr.data();
    c.col_idx = A.col_idx.data();
    c.values = A.values.data();
    c.index_bits = 64;
    c.location = AMGR_HOST;
    return c;
}

amgr_amg_params params_of(const AmgParams& p) {
    amgr_amg_params c;
    amgr_amg_params_default(&c);
    c.eps = p.eps;
    c.omega = p.omega;
    c.pre_sweeps = p.pre_sweeps;
    c.post_sweeps = p.post_sweeps;
    c.coarse_enough = p.coarse_enough;
    c.max_direct_size = p.max_direct_size;
    c.coarse_solve = AMGR_COARSE_EXACT;
    return c;
}

bool same_smoothing(const AmgParams& a, const AmgParams& b) {
    return a.omega == b.omega && a.pre_sweeps == b.pre_sweeps && a.post_sweeps == b.post_sweeps;
}

std::shared_ptr<amgr_hier> own(amgr_hier* h) { return std::shared_ptr<amgr_hier>(h, amgr_hier_destroy); }

// Host mirror of a device hierarchy.  P/R of every level come from `shared`
// when given (partial_update shares the frozen transfer operators, as the
// reference's shared_ptr does, hierarchy.cpp:140).
Hierarchy mirror(std::shared_ptr<amgr_hier> dh, const AmgParams& prm, const Hierarchy* shared) {
    Hierarchy out;
    out.device = std::move(dh);
    out.params = prm;
    amgr_hier* h = out.device.get();
    const int L = amgr_hier_num_levels(h);
    for (int l = 0; l < L; ++l) {
        int64_t d[8] = {0};
        check(amgr_hier_level_dims(h, l, d), "level_dims");
        Level lv;
        lv.A.nrows = lv.A.ncols = d[0];
        lv.A.row_ptr.assign(static_cast<size_t>(d[0]) + 1, 0);
        lv.A.col_idx.resize(static_cast<size_t>(d[1]));
        lv.A.values.resize(static_cast<size_t>(d[1]));
        check(amgr_hier_level_A(h, l, lv.A.row_ptr.data(), lv.A.col_idx.data(), lv.A.values.data()), "level_A");
        if (d[2] > 0) {
            if (shared && l < static_cast<int>(shared->levels.size()) && shared->levels[l].P) {
                lv.P = shared->levels[l].P;
                lv.R = shared->levels[l].R;
            } else {
                // tentative prolongation (coarsening.cpp:122-132) and R = P^T
                auto P = std::make_shared<CsrMatrix>();
                P->nrows = d[0];
                P->ncols = d[2];
                P->row_ptr.resize(static_cast<size_t>(d[0]) + 1);
                for (int64_t i = 0; i <= d[0]; ++i) P->row_ptr[static_cast<size_t>(i)] = i;
                P->col_idx.resize(static_cast<size_t>(d[0]));
                P->values.assign(static_cast<size_t>(d[0]), 1.0);
                check(amgr_hier_level_P(h, l, P->col_idx.data()), "level_P");
                auto R = std::make_shared<CsrMatrix>();
                R->nrows = d[2];
                R->ncols = d[0];
                R->row_ptr.resize(static_cast<size_t>(d[2]) + 1);
                R->col_idx.resize(static_cast<size_t>(d[0]));
                R->values.assign(static_cast<size_t>(d[0]), 1.0);
                check(amgr_hier_level_R(h, l, R->row_ptr.data(), R->col_idx.data()), "level_R");
                lv.P = std::move(P);
                lv.R = std::move(R);
            }
        }
        if (d[3]) {
            JacobiSmoother s;
            s.omega = prm.omega;
            s.inv_diag.resize(static_cast<size_t>(d[0]));
            check(amgr_hier_level_smoother(h, l, s.inv_diag.data()), "level_smoother");
            lv.smoother = std::move(s);
        }
        out.levels.push_back(std::move(lv));
    }
    const int64_t nc = amgr_hier_coarse_n(h);
    out.coarse_solver.n = nc;
    out.coarse_solver.lu.resize(static_cast<size_t>(nc * nc));
    out.coarse_solver.piv.resize(static_cast<size_t>(nc));
    check(amgr_hier_coarse_lu(h, out.coarse_solver.lu.data(), out.coarse_solver.piv.data()), "coarse_lu");
    amgr_phase_timings t{};
    check(amgr_hier_timings(h, &t), "timings");
    out.setup_timings = {t.transfer_ops, t.galerkin, t.smoother, t.coarse_solver};
    return out;
}

}  // namespace

amgr_ctx* facade_context() {
    static std::once_flag once;
    static amgr_ctx* ctx = nullptr;
    std::call_once(once, [] {
        if (amgr_ctx_create(0, nullptr, &ctx) != AMGR_OK) {
            const char* m = amgr_last_error(nullptr);
            throw std::runtime_error(std::string("amgreuse_gpu: no usable B200: ") + (m ? m : ""));
        }
    });
    return ctx;
}

// ---- sparse ---------------------------------------------------------------------------
CsrMatrix csr_from_triplets(index_t nrows, index_t ncols, std::span<const Triplet> entries) {
    std::vector<int64_t> r(entries.size()), c(entries.size());
    std::vector<double> v(entries.size());
    for (size_t k = 0; k < entries.size(); ++k) {
        r[k] = entries[k].row;
        c[k] = entries[k].col;
        v[k] = entries[k].value;
    }
    amgr_ctx* ctx = facade_context();
    amgr_matrix* m = nullptr;
    check(amgr_csr_from_triplets(ctx, nrows, ncols, static_cast<int64_t>(entries.size()), r.data(), c.data(),
                                 v.data(), &m),
          "csr_from_triplets");
    amgr_csr d{};
    const amgr_status st = amgr_matrix_csr(m, &d);
    if (st != AMGR_OK) {
        amgr_matrix_free(m);
        raise(st, "csr_from_triplets");
    }
    CsrMatrix A;
    A.nrows = nrows;
    A.ncols = ncols;
    std::vector<int32_t> rp(static_cast<size_t>(nrows) + 1), ci(static_cast<size_t>(d.nnz));
    A.values.resize(static_cast<size_t>(d.nnz));
    amgr_copy_to_host(ctx, rp.data(), d.row_ptr, sizeof(int32_t) * rp.size());
    if (d.nnz) {
        amgr_copy_to_host(ctx, ci.data(), d.col_idx, sizeof(int32_t) * ci.size());
        amgr_copy_to_host(ctx, A.values.data(), d.values, sizeof(double) * A.values.size());
    }
    amgr_matrix_free(m);
    A.row_ptr.assign(rp.begin(), rp.end());
    A.col_idx.assign(ci.begin(), ci.end());
    return A;
}

void spmv(const CsrMatrix& A, std::span<const double> x, std::span<double> y) {
    if (static_cast<index_t>(x.size()) != A.ncols || static_cast<index_t>(y.size()) != A.nrows)
        throw std::invalid_argument("spmv: dimension mismatch");
    const amgr_csr c = view(A);
    check(amgr_csr_spmv(facade_context(), &c, x.data(), y.data(), AMGR_HOST), "spmv");
}

std::vector<double> spmv(const CsrMatrix& A, std::span<const double> x) {
    std::vector<double> y(static_cast<size_t>(A.nrows));
    spmv(A, x, y);
    return y;
}

CsrMatrix transpose(const CsrMatrix& A) {
    // counting sort by column, rows ascending inside each column (the
    // structure the device keeps as member lists, hierarchy R = P^T)
    CsrMatrix T;
    T.nrows = A.ncols;
    T.ncols = A.nrows;
    T.row_ptr.assign(static_cast<size_t>(A.ncols) + 1, 0);
    for (index_t c : A.col_idx) ++T.row_ptr[static_cast<size_t>(c) + 1];
    for (size_t j = 0; j < static_cast<size_t>(A.ncols); ++j) T.row_ptr[j + 1] += T.row_ptr[j];
    T.col_idx.resize(A.col_idx.size());
    T.values.resize(A.values.size());
    std::vector<index_t> pos(T.row_ptr.begin(), T.row_ptr.end() - 1);
    for (index_t i = 0; i < A.nrows; ++i)
        for (index_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
            const index_t p = pos[static_cast<size_t>(A.col_idx[k])]++;
            T.col_idx[static_cast<size_t>(p)] = i;
            T.values[static_cast<size_t>(p)] = A.values[static_cast<size_t>(k)];
        }
    return T;
}

// ---- smoother ---------------------------------------------------------------------------
JacobiSmoother build_smoother(const CsrMatrix& A, double omega) {
    JacobiSmoother s;
    s.omega = omega;
    s.inv_diag.resize(static_cast<size_t>(A.nrows));
    const amgr_csr c = view(A);
    check(amgr_build_smoother(facade_context(), &c, s.inv_diag.data(), AMGR_HOST), "build_smoother");
    return s;
}

void smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f, std::span<double> u,
            int sweeps) {
    if (A.nrows != A.ncols) throw std::invalid_argument("smooth: matrix is not square");
    if (static_cast<index_t>(f.size()) != A.nrows || static_cast<index_t>(u.size()) != A.nrows ||
        static_cast<index_t>(s.inv_diag.size()) != A.nrows)
        throw std::invalid_argument("smooth: dimension mismatch");
    const amgr_csr c = view(A);
    check(amgr_smooth(facade_context(), &c, s.inv_diag.data(), s.omega, f.data(), u.data(), sweeps, AMGR_HOST),
          "smooth");
}

void smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f, std::vector<double>& u,
            int sweeps) {
    smooth(s, A, f, std::span<double>(u), sweeps);
}

std::vector<double> smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f,
                           const std::vector<double>& u, int sweeps) {
    std::vector<double> v(u);
    smooth(s, A, f, std::span<double>(v), sweeps);
    return v;
}

std::vector<double> smooth(const JacobiSmoother& s, const CsrMatrix& A, std::span<const double> f,
                           std::vector<double>&& u, int sweeps) {
    std::vector<double> v(std::move(u));
    smooth(s, A, f, std::span<double>(v), sweeps);
    return v;
}

// ---- coarse solver ----------------------------------------------------------------------
DenseFactorization coarse_factorize(const CsrMatrix& A) {
    if (A.nrows != A.ncols) throw std::invalid_argument("coarse_factorize: matrix is not square");
    DenseFactorization f;
    f.n = A.nrows;
    f.lu.resize(static_cast<size_t>(f.n * f.n));
    f.piv.resize(static_cast<size_t>(f.n));
    const amgr_csr c = view(A);
    check(amgr_coarse_factorize(facade_context(), &c, f.lu.data(), f.piv.data()), "coarse_factorize");
    return f;
}

std::vector<double> coarse_solve(const DenseFactorization& f, std::span<const double> rhs) {
    if (static_cast<index_t>(rhs.size()) != f.n) throw std::invalid_argument("coarse_solve: dimension mismatch");
    std::vector<double> x(static_cast<size_t>(f.n));
    check(amgr_coarse_solve(facade_context(), f.n, f.lu.data(), f.piv.data(), rhs.data(), x.data()), "coarse_solve");
    return x;
}

// ---- hierarchy ----------------------------------------------------------------------
double Hierarchy::operator_complexity() const {
    double total = 0.0;
    for (const Level& l : levels) total += static_cast<double>(l.A.nnz());
    return total / static_cast<double>(levels.front().A.nnz());
}

Hierarchy setup(const CsrMatrix& A, const AmgParams& prm) {
    if (A.nrows != A.ncols) throw std::invalid_argument("setup: matrix is not square");
    if (A.nrows == 0) throw std::invalid_argument("setup: empty matrix");
    const amgr_csr c = view(A);
    const amgr_amg_params p = params_of(prm);
    amgr_hier* h = nullptr;
    check(amgr_setup(facade_context(), &c, &p, &h), "setup");
    return mirror(own(h), prm, nullptr);
}

Hierarchy partial_update(const Hierarchy& h, CsrMatrix A_new, const AmgParams& prm) {
    if (h.levels.empty() || !h.device) throw std::invalid_argument("partial_update: empty hierarchy");
    const amgr_csr c = view(A_new);
    const amgr_amg_params p = params_of(prm);
    amgr_hier* out = nullptr;
    check(amgr_partial_update(h.device.get(), &c, &p, &out), "partial_update");
    return mirror(own(out), prm, &h);
}

std::vector<double> vcycle(const Hierarchy& h, std::span<const double> f, const AmgParams& prm) {
    if (h.levels.empty() || !h.device) throw std::invalid_argument("vcycle: empty hierarchy");
    if (static_cast<index_t>(f.size()) != h.finest_size()) throw std::invalid_argument("vcycle: dimension mismatch");
    std::shared_ptr<amgr_hier> dev = h.device;
    if (!same_smoothing(prm, h.params)) {
        // the device hierarchy binds its smoothing parameters at build time:
        // re-derive one with these (frozen transfers, same values)
        const amgr_csr c = view(h.levels.front().A);
        const amgr_amg_params p = params_of(prm);
        amgr_hier* out = nullptr;
        check(amgr_partial_update(h.device.get(), &c, &p, &out), "vcycle");
        dev = own(out);
    }
    std::vector<double> u(f.size());
    check(amgr_vcycle(dev.get(), f.data(), u.data(), AMGR_HOST), "vcycle");
    return u;
}

std::pair<std::vector<double>, SolveStats> bicgstab(const Hierarchy& h, std::span<const double> f,
                                                    std::span<const double> u0, const SolveParams& prm) {
    if (f.size() != u0.size()) throw std::invalid_argument("bicgstab: dimension mismatch");
    if (!h.device) throw std::invalid_argument("bicgstab: empty hierarchy");
    amgr_solve_params sp{prm.tol, prm.max_iter};
    amgr_solve_stats st{};
    std::vector<double> u(f.size());
    check(amgr_bicgstab(h.device.get(), f.data(), u0.data(), u.data(), &sp, &st, AMGR_HOST), "bicgstab");
    return {std::move(u), SolveStats{st.iterations, st.relative_residual, st.converged != 0, st.breakdown != 0}};
}

}  // namespace amgreuse

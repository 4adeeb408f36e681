// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product.
//
// extern "C" shim over the UNMODIFIED reference library (`amgreuse`, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Only
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm
// load it, as the checker or as the timed CPU baseline.
//
// Two V-cycle variants are exposed:
//   * shipped: the reference's own `vcycle` (proj/src/hierarchy.cpp:152-186).
//     Its `smooth(..., us[i], ...)` calls bind to the value-returning overload
//     (proj/include/amgreuse/smoother.hpp:27-28) and discard the result, so the
//     shipped cycle performs no smoothing.
//   * fixed: the same algorithm re-composed from the reference's public
//     primitives with explicit spans — smooth(span) (smoother.hpp:23-24),
//     spmv (csr.hpp:77), coarse_solve (dense_lu.hpp:24) — which is what the
//     reference's docs/spec describe (SPEC.md "vcycle").  Solve parity is taken
//     against this one.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "amgreuse/bicgstab.hpp"
#include "amgreuse/coarsening.hpp"
#include "amgreuse/csr.hpp"
#include "amgreuse/dense_lu.hpp"
#include "amgreuse/hierarchy.hpp"
#include "amgreuse/matrix_market.hpp"
#include "amgreuse/smoother.hpp"
#include "bench_app.hpp"

#include <sstream>

using namespace amgreuse;

namespace {

using clk = std::chrono::steady_clock;

struct Params {
    double eps, omega;
    int32_t pre_sweeps, post_sweeps;
    int64_t coarse_enough, max_direct_size;
};

AmgParams to_amg(const Params* p) {
    AmgParams a;
    if (p) {
        a.eps = p->eps;
        a.omega = p->omega;
        a.pre_sweeps = p->pre_sweeps;
        a.post_sweeps = p->post_sweeps;
        a.coarse_enough = p->coarse_enough;
        a.max_direct_size = p->max_direct_size;
    }
    return a;
}

CsrMatrix make_csr(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                   const double* v) {
    CsrMatrix A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.row_ptr.assign(rp, rp + nrows + 1);
    const int64_t nnz = rp[nrows];
    A.col_idx.assign(ci, ci + nnz);
    A.values.assign(v, v + nnz);
    return A;
}

// error kind: 0 ok, 1 invalid_argument, 2 runtime_error, 3 other
int report(const std::exception& e, int kind, char* err, int errlen) {
    if (err && errlen > 0) {
        std::strncpy(err, e.what(), static_cast<size_t>(errlen - 1));
        err[errlen - 1] = '\0';
    }
    return kind;
}

double secs(clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); }

// Fixed V-cycle: hierarchy.cpp:152-186 with span-binding smooth calls.
void vcycle_fixed(const Hierarchy& h, std::span<const double> f, std::span<double> out,
                  const AmgParams& prm) {
    const std::size_t L = h.levels.size();
    std::vector<std::vector<double>> us(L), fs(L);
    fs[0].assign(f.begin(), f.end());
    std::vector<double> r;
    for (std::size_t i = 0; i + 1 < L; ++i) {
        const Level& lvl = h.levels[i];
        const std::size_t n = static_cast<std::size_t>(lvl.A.nrows);
        us[i].assign(n, 0.0);
        smooth(*lvl.smoother, lvl.A, fs[i], std::span<double>(us[i]), prm.pre_sweeps);
        r.resize(n);
        spmv(lvl.A, us[i], r);
        for (std::size_t k = 0; k < n; ++k) r[k] = fs[i][k] - r[k];
        fs[i + 1].resize(static_cast<std::size_t>(lvl.R->nrows));
        spmv(*lvl.R, r, fs[i + 1]);
    }
    us[L - 1] = coarse_solve(h.coarse_solver, fs[L - 1]);
    for (std::size_t i = L - 1; i-- > 0;) {
        const Level& lvl = h.levels[i];
        const std::size_t n = static_cast<std::size_t>(lvl.A.nrows);
        r.resize(n);
        spmv(*lvl.P, us[i + 1], r);
        for (std::size_t k = 0; k < n; ++k) us[i][k] += r[k];
        smooth(*lvl.smoother, lvl.A, fs[i], std::span<double>(us[i]), prm.post_sweeps);
    }
    std::copy(us[0].begin(), us[0].end(), out.begin());
}

} // namespace

extern "C" {

int ref_setup(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
              const Params* p, void** out, double* seconds, char* err, int errlen) {
    try {
        CsrMatrix A = make_csr(n, n, rp, ci, v);
        auto t0 = clk::now();
        auto* h = new Hierarchy(setup(A, to_amg(p)));
        if (seconds) *seconds = secs(t0);
        *out = h;
        return 0;
    } catch (const std::invalid_argument& e) {
        return report(e, 1, err, errlen);
    } catch (const std::runtime_error& e) {
        return report(e, 2, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 3, err, errlen);
    }
}

// Same as ref_setup but for a (possibly rectangular / non-square) input, to
// reproduce the reference's "not square" error path.
int ref_setup_rect(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                   const double* v, const Params* p, void** out, char* err, int errlen) {
    try {
        CsrMatrix A = make_csr(nrows, ncols, rp, ci, v);
        *out = new Hierarchy(setup(A, to_amg(p)));
        return 0;
    } catch (const std::invalid_argument& e) {
        return report(e, 1, err, errlen);
    } catch (const std::runtime_error& e) {
        return report(e, 2, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 3, err, errlen);
    }
}

int ref_partial_update(void* hp, int64_t nrows, int64_t ncols, const int64_t* rp,
                       const int64_t* ci, const double* v, const Params* p, void** out,
                       double* seconds, char* err, int errlen) {
    try {
        const Hierarchy& h = *static_cast<Hierarchy*>(hp);
        CsrMatrix A = make_csr(nrows, ncols, rp, ci, v);
        auto t0 = clk::now();
        auto* nh = new Hierarchy(partial_update(h, std::move(A), to_amg(p)));
        if (seconds) *seconds = secs(t0);
        *out = nh;
        return 0;
    } catch (const std::invalid_argument& e) {
        return report(e, 1, err, errlen);
    } catch (const std::runtime_error& e) {
        return report(e, 2, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 3, err, errlen);
    }
}

void ref_free(void* hp) { delete static_cast<Hierarchy*>(hp); }

int64_t ref_num_levels(void* hp) {
    return static_cast<int64_t>(static_cast<Hierarchy*>(hp)->levels.size());
}

// out: [nrows, nnz, has_P, n_coarse, has_smoother]
void ref_level_dims(void* hp, int64_t lvl, int64_t* out) {
    const Level& L = static_cast<Hierarchy*>(hp)->levels[static_cast<size_t>(lvl)];
    out[0] = L.A.nrows;
    out[1] = L.A.nnz();
    out[2] = L.P ? 1 : 0;
    out[3] = L.P ? L.P->ncols : 0;
    out[4] = L.smoother ? 1 : 0;
}

void ref_level_A(void* hp, int64_t lvl, int64_t* rp, int64_t* ci, double* v) {
    const Level& L = static_cast<Hierarchy*>(hp)->levels[static_cast<size_t>(lvl)];
    std::memcpy(rp, L.A.row_ptr.data(), sizeof(int64_t) * L.A.row_ptr.size());
    std::memcpy(ci, L.A.col_idx.data(), sizeof(int64_t) * L.A.col_idx.size());
    std::memcpy(v, L.A.values.data(), sizeof(double) * L.A.values.size());
}

// P is n_fine x n_coarse with one unit entry per row: export its col_idx and
// values (the aggregate assignment).
void ref_level_P(void* hp, int64_t lvl, int64_t* rp, int64_t* ci, double* v) {
    const Level& L = static_cast<Hierarchy*>(hp)->levels[static_cast<size_t>(lvl)];
    const CsrMatrix& P = *L.P;
    std::memcpy(rp, P.row_ptr.data(), sizeof(int64_t) * P.row_ptr.size());
    std::memcpy(ci, P.col_idx.data(), sizeof(int64_t) * P.col_idx.size());
    std::memcpy(v, P.values.data(), sizeof(double) * P.values.size());
}

void ref_level_R(void* hp, int64_t lvl, int64_t* rp, int64_t* ci, double* v) {
    const Level& L = static_cast<Hierarchy*>(hp)->levels[static_cast<size_t>(lvl)];
    const CsrMatrix& R = *L.R;
    std::memcpy(rp, R.row_ptr.data(), sizeof(int64_t) * R.row_ptr.size());
    std::memcpy(ci, R.col_idx.data(), sizeof(int64_t) * R.col_idx.size());
    std::memcpy(v, R.values.data(), sizeof(double) * R.values.size());
}

void ref_level_invdiag(void* hp, int64_t lvl, double* out, double* omega) {
    const Level& L = static_cast<Hierarchy*>(hp)->levels[static_cast<size_t>(lvl)];
    std::memcpy(out, L.smoother->inv_diag.data(), sizeof(double) * L.smoother->inv_diag.size());
    *omega = L.smoother->omega;
}

int64_t ref_coarse_n(void* hp) { return static_cast<Hierarchy*>(hp)->coarse_solver.n; }

void ref_coarse(void* hp, double* lu, int64_t* piv) {
    const DenseFactorization& f = static_cast<Hierarchy*>(hp)->coarse_solver;
    std::memcpy(lu, f.lu.data(), sizeof(double) * f.lu.size());
    std::memcpy(piv, f.piv.data(), sizeof(int64_t) * f.piv.size());
}

void ref_timings(void* hp, double* out) {
    const SetupPhaseTimings& t = static_cast<Hierarchy*>(hp)->setup_timings;
    out[0] = t.transfer_ops;
    out[1] = t.galerkin;
    out[2] = t.smoother;
    out[3] = t.coarse_solver;
}

double ref_operator_complexity(void* hp) {
    return static_cast<Hierarchy*>(hp)->operator_complexity();
}

int ref_vcycle(void* hp, const double* f, double* u, int fixed, const Params* p,
               double* seconds, char* err, int errlen) {
    try {
        const Hierarchy& h = *static_cast<Hierarchy*>(hp);
        const auto n = static_cast<size_t>(h.finest_size());
        const AmgParams prm = to_amg(p);
        auto t0 = clk::now();
        if (fixed) {
            vcycle_fixed(h, std::span<const double>(f, n), std::span<double>(u, n), prm);
        } else {
            auto z = vcycle(h, std::span<const double>(f, n), prm);
            std::copy(z.begin(), z.end(), u);
        }
        if (seconds) *seconds = secs(t0);
        return 0;
    } catch (const std::invalid_argument& e) {
        return report(e, 1, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 3, err, errlen);
    }
}

// Right-preconditioned BiCGStab (proj/src/bicgstab.cpp:21-135) with A = the
// hierarchy's finest matrix and M = one V-cycle (shipped or fixed).
// stats: [iterations, converged, breakdown]; relres out.
int ref_bicgstab(void* hp, const double* f, const double* u0, double* u, double tol,
                 int64_t max_iter, int fixed, const Params* p, int64_t* stats, double* relres,
                 double* seconds, char* err, int errlen) {
    try {
        const Hierarchy& h = *static_cast<Hierarchy*>(hp);
        const auto n = static_cast<size_t>(h.finest_size());
        const AmgParams prm = to_amg(p);
        LinearOperator A = make_operator(h.levels.front().A);
        LinearOperator M;
        if (fixed) {
            M = [&h, prm](std::span<const double> x, std::span<double> y) {
                vcycle_fixed(h, x, y, prm);
            };
        } else {
            M = make_preconditioner(h, prm);
        }
        SolveParams sp;
        sp.tol = tol;
        sp.max_iter = max_iter;
        auto t0 = clk::now();
        auto [x, st] = bicgstab(A, M, std::span<const double>(f, n),
                                std::span<const double>(u0, n), sp);
        if (seconds) *seconds = secs(t0);
        std::copy(x.begin(), x.end(), u);
        stats[0] = st.iterations;
        stats[1] = st.converged ? 1 : 0;
        stats[2] = st.breakdown ? 1 : 0;
        *relres = st.relative_residual;
        return 0;
    } catch (const std::invalid_argument& e) {
        return report(e, 1, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 3, err, errlen);
    }
}

// Unit-level hooks (strength graph / aggregation / spmv / galerkin) used to
// pin the restated oracle against the reference on random inputs.
int64_t ref_strength(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     double eps, int64_t* adj_ptr, int64_t* adj, int64_t cap, char* err,
                     int errlen) {
    try {
        CsrMatrix A = make_csr(n, n, rp, ci, v);
        StrengthGraph g = strength_graph(A, eps);
        if (adj_ptr) std::memcpy(adj_ptr, g.adj_ptr.data(), sizeof(int64_t) * (n + 1));
        if (adj && cap >= g.num_edges())
            std::memcpy(adj, g.adj.data(), sizeof(int64_t) * g.adj.size());
        return g.num_edges();
    } catch (const std::exception& e) {
        report(e, 1, err, errlen);
        return -1;
    }
}

int64_t ref_aggregate(int64_t n, const int64_t* adj_ptr, const int64_t* adj, int64_t* assignment) {
    StrengthGraph g;
    g.n = n;
    g.adj_ptr.assign(adj_ptr, adj_ptr + n + 1);
    g.adj.assign(adj, adj + adj_ptr[n]);
    Aggregates a = aggregate(g);
    std::memcpy(assignment, a.assignment.data(), sizeof(int64_t) * static_cast<size_t>(n));
    return a.n_coarse;
}

void ref_spmv(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
              const double* v, const double* x, double* y) {
    CsrMatrix A = make_csr(nrows, ncols, rp, ci, v);
    spmv(A, std::span<const double>(x, static_cast<size_t>(ncols)),
         std::span<double>(y, static_cast<size_t>(nrows)));
}

// C = R * A * P via the reference's galerkin_product; two calls: first with
// out arrays null to get nnz, then to fill.
int64_t ref_galerkin(int64_t nf, int64_t nc, const int64_t* arp, const int64_t* aci,
                     const double* av, const int64_t* agg, int64_t* crp, int64_t* cci,
                     double* cv) {
    CsrMatrix A = make_csr(nf, nf, arp, aci, av);
    Aggregates a;
    a.n_fine = nf;
    a.n_coarse = nc;
    a.assignment.assign(agg, agg + nf);
    CsrMatrix P = tentative_prolongation(a);
    CsrMatrix R = transpose(P);
    CsrMatrix C = galerkin_product(R, A, P);
    if (crp) {
        std::memcpy(crp, C.row_ptr.data(), sizeof(int64_t) * C.row_ptr.size());
        std::memcpy(cci, C.col_idx.data(), sizeof(int64_t) * C.col_idx.size());
        std::memcpy(cv, C.values.data(), sizeof(double) * C.values.size());
    }
    return C.nnz();
}

int ref_coarse_factorize(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                         double* lu, int64_t* piv, char* err, int errlen) {
    try {
        CsrMatrix A = make_csr(n, n, rp, ci, v);
        DenseFactorization f = coarse_factorize(A);
        std::memcpy(lu, f.lu.data(), sizeof(double) * f.lu.size());
        std::memcpy(piv, f.piv.data(), sizeof(int64_t) * f.piv.size());
        return 0;
    } catch (const std::runtime_error& e) {
        return report(e, 2, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 1, err, errlen);
    }
}

// mm_read (matrix_market.cpp:104-140): first call with rp == nullptr returns
// the dimensions; the second fills the CSR.  Re-reads the file each call.
int ref_mm_read(const char* path, int64_t* dims, int64_t* rp, int64_t* ci, double* v, char* err, int errlen) {
    try {
        CsrMatrix A = mm_read(path);
        dims[0] = A.nrows;
        dims[1] = A.ncols;
        dims[2] = A.nnz();
        if (rp) {
            std::memcpy(rp, A.row_ptr.data(), sizeof(int64_t) * A.row_ptr.size());
            std::memcpy(ci, A.col_idx.data(), sizeof(int64_t) * A.col_idx.size());
            std::memcpy(v, A.values.data(), sizeof(double) * A.values.size());
        }
        return 0;
    } catch (const std::runtime_error& e) {
        return report(e, 2, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 1, err, errlen);
    }
}

// mm_read_vector (matrix_market.cpp:176-203)
int ref_mm_read_vector(const char* path, int64_t* n, double* v, char* err, int errlen) {
    try {
        std::vector<double> x = mm_read_vector(path);
        *n = static_cast<int64_t>(x.size());
        if (v) std::memcpy(v, x.data(), sizeof(double) * x.size());
        return 0;
    } catch (const std::runtime_error& e) {
        return report(e, 2, err, errlen);
    } catch (const std::exception& e) {
        return report(e, 1, err, errlen);
    }
}

// Report renderers of the reference's bench tool (tools/bench_app.cpp:129-266)
// over caller-supplied run data: one run per strategy (repeat = 1), steps
// given as flat arrays.  which: 0 = render_report, 1 = write_per_step_csv.
int ref_render(int which, int format, const char* seqdir, double eps, double omega, int pre, int post,
               int64_t coarse_enough, double tol, int64_t max_iter, int64_t reuse_iter_limit, int64_t rebuild_every,
               int nstrat, const int* kinds, int64_t nsteps, const int* actions, const double* setup,
               const double* solve, const int64_t* iters, const int* conv, const double* phases, char* out,
               int outlen) {
    try {
        bench::BenchConfig cfg;
        cfg.sequence_dir = seqdir;
        cfg.amg.eps = eps;
        cfg.amg.omega = omega;
        cfg.amg.pre_sweeps = pre;
        cfg.amg.post_sweeps = post;
        cfg.amg.coarse_enough = coarse_enough;
        cfg.solve.tol = tol;
        cfg.solve.max_iter = max_iter;
        cfg.reuse_iter_limit = reuse_iter_limit;
        if (rebuild_every > 0) cfg.rebuild_every = rebuild_every;
        cfg.format = format == 0 ? bench::OutputFormat::markdown : bench::OutputFormat::csv;
        std::vector<bench::StrategyOutcome> outcomes;
        for (int s = 0; s < nstrat; ++s) {
            RunReport r;
            r.strategy.kind = static_cast<StrategyKind>(kinds[s]);
            double ts = 0.0, tv = 0.0, it = 0.0;
            for (int64_t k = 0; k < nsteps; ++k) {
                const int64_t x = s * nsteps + k;
                StepMetrics m;
                m.step = k;
                m.setup_time = setup[x];
                m.solve_time = solve[x];
                m.iterations = iters[x];
                m.converged = conv[x] != 0;
                m.action = static_cast<StepAction>(actions[x]);
                m.phase_timings.transfer_ops = phases[4 * x + 0];
                m.phase_timings.galerkin = phases[4 * x + 1];
                m.phase_timings.smoother = phases[4 * x + 2];
                m.phase_timings.coarse_solver = phases[4 * x + 3];
                if (m.action == StepAction::full_build) ++r.full_rebuilds;
                ts += m.setup_time;
                tv += m.solve_time;
                it += static_cast<double>(m.iterations);
                r.steps.push_back(m);
            }
            r.total_setup = ts;
            r.total_solve = tv;
            r.avg_iterations = it / static_cast<double>(nsteps);
            bench::StrategyOutcome o;
            o.kind = r.strategy.kind;
            o.runs.push_back(r);
            o.median = r;
            outcomes.push_back(o);
        }
        std::ostringstream os;
        if (which == 0)
            bench::render_report(os, cfg, outcomes);
        else
            bench::write_per_step_csv(os, outcomes);
        const std::string t = os.str();
        if (static_cast<int>(t.size()) >= outlen) return -static_cast<int>(t.size()) - 1;
        std::memcpy(out, t.data(), t.size());
        out[t.size()] = '\0';
        return 0;
    } catch (const std::exception& e) {
        return report(e, 1, out, outlen);
    }
}

} // extern "C"

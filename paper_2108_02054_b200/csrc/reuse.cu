// Reuse driver: the reference's run_sequence (proj/src/reuse.cpp:46-136) over
// the device hierarchy.  Per step: action choice (none / full / partial with
// the periodic and dimension-change rules), setup or in-place partial update
// timed, BiCGStab from the previous step's solution timed, full-reuse rebuild
// flag from the solve's convergence and iteration count.
#include <chrono>
#include <cmath>
#include <limits>
#include <sstream>

#include "hierarchy.cuh"

namespace amgr {

namespace {

using clk = std::chrono::steady_clock;

double since(clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); }

}  // namespace

void run_sequence(Ctx& c, int64_t nsteps, amgr_step_fn step, void* user, const amgr_strategy& st,
                  const AmgP& amg, const amgr_solve_params& sp, amgr_step_metrics* metrics, amgr_solution_fn sink,
                  void* sink_user) {
    if (nsteps <= 0) invalid("run_sequence: empty sequence");
    const int64_t iter_limit = st.reuse_iter_limit > 0 ? st.reuse_iter_limit : sp.max_iter;
    if (iter_limit > sp.max_iter) invalid("run_sequence: reuse_iter_limit exceeds max_iter");
    if (st.kind < AMGR_REUSE_NONE || st.kind > AMGR_REUSE_PARTIAL) invalid("run_sequence: unknown strategy kind");
    std::unique_ptr<Hier> h;
    bool rebuild_flag = false;
    DevArray<double> prev, u, f;
    for (int64_t k = 0; k < nsteps; ++k) {
        amgr_csr A{};
        const double* rhs = nullptr;
        int32_t rhs_loc = AMGR_HOST;
        if (step(user, k, &A, &rhs, &rhs_loc) != 0) invalid("run_sequence: step callback failed");
        amgr_step_metrics m{};
        m.step = k;
        const bool have = static_cast<bool>(h);
        const bool dims_changed = have && A.nrows != h->lv.front().pat->n;
        switch (st.kind) {
            case AMGR_REUSE_NONE:
                m.action = AMGR_ACTION_FULL_BUILD;
                break;
            case AMGR_REUSE_FULL:
                m.action = (!have || dims_changed || rebuild_flag) ? AMGR_ACTION_FULL_BUILD
                                                                  : AMGR_ACTION_REUSED_UNCHANGED;
                break;
            default: {
                const bool periodic = st.rebuild_every > 0 && k > 0 && k % st.rebuild_every == 0;
                const bool escalate = (st.flags & AMGR_STRATEGY_ESCALATE) && rebuild_flag;
                m.action = (!have || dims_changed || periodic || escalate) ? AMGR_ACTION_FULL_BUILD
                                                                           : AMGR_ACTION_PARTIAL_UPDATE;
            }
        }
        CK(cudaStreamSynchronize(c.stream));
        auto t0 = clk::now();
        if (m.action == AMGR_ACTION_FULL_BUILD) {
            h = setup(c, A, amg);
            CK(cudaStreamSynchronize(c.stream));
            m.setup_time = since(t0);
            m.phase_timings = h->tm;
        } else if (m.action == AMGR_ACTION_PARTIAL_UPDATE) {
            rebuild(*h, A);
            CK(cudaStreamSynchronize(c.stream));
            m.setup_time = since(t0);
            m.phase_timings = h->tm;
        }
        const int64_t n = h->lv.front().pat->n;
        if (f.size() != n) f.alloc(n, c.stream);
        CK(cudaMemcpyAsync(f.get(), rhs, sizeof(double) * n,
                           rhs_loc == AMGR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
        if (u.size() != n) u.alloc(n, c.stream);
        // initial guess: previous solution when sizes match (reuse.cpp:108-109)
        if (prev.size() == n)
            copy(c, u.get(), prev.get(), n);
        else
            fill(c, u.get(), n, 0.0);
        CK(cudaStreamSynchronize(c.stream));
        auto t1 = clk::now();
        amgr_solve_stats ss{};
        bicgstab(*h, f.get(), u.get(), u.get(), sp, ss);
        CK(cudaStreamSynchronize(c.stream));
        m.solve_time = since(t1);
        m.iterations = ss.iterations;
        m.converged = ss.converged;
        if (st.kind == AMGR_REUSE_FULL || (st.kind == AMGR_REUSE_PARTIAL && (st.flags & AMGR_STRATEGY_ESCALATE)))
            rebuild_flag = !ss.converged || ss.iterations >= iter_limit;
        if (prev.size() != n) prev.alloc(n, c.stream);
        copy(c, prev.get(), u.get(), n);
        if (sink) {
            CK(cudaStreamSynchronize(c.stream));
            sink(sink_user, k, u.get(), n);
        }
        metrics[k] = m;
    }
}

}  // namespace amgr

extern "C" {

amgr_status amgr_run_sequence(amgr_ctx* ctx, int64_t nsteps, amgr_step_fn step, void* user,
                              const amgr_strategy* strategy, const amgr_amg_params* amg,
                              const amgr_solve_params* solve, amgr_step_metrics* metrics, amgr_solution_fn sink,
                              void* sink_user) {
    if (!ctx || !step || !strategy || !metrics) return AMGR_E_INVALID_ARGUMENT;
    try {
        CK(cudaSetDevice(ctx->c.device));
        amgr_solve_params sp{1e-8, 100};
        if (solve) sp = *solve;
        amgr::run_sequence(ctx->c, nsteps, step, user, *strategy, amgr::to_amgp(amg), sp, metrics, sink, sink_user);
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        ctx->c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        ctx->c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

double amgr_speedup_percent(double t_base, double t_other) {
    if (t_other == 0.0) return std::numeric_limits<double>::infinity();
    return (t_base / t_other - 1.0) * 100.0;
}

}  // extern "C"

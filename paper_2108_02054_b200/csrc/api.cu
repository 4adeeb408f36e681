// extern "C" boundary of libamgr_b200.so (include/amgr.h).  Thin: validates
// arguments, converts exceptions into amgr_status + last-error text, and
// forwards to the C++ orchestration in hierarchy.cu.
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <string>

#include "hierarchy.cuh"


namespace amgr {

static bool probe_match(const Ctx& c, const char* family) {
    if (c.probe.family.empty() || c.probe.family != family) return false;
    return c.probe.level < 0 || c.probe.level == c.cur_level;
}
void probe_begin(Ctx& c, const char* family, double bytes) {
    if (!probe_match(c, family)) return;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c.stream));
    c.probe.events.push_back({a, b});
    c.probe.bytes.push_back(bytes);
}
void probe_end(Ctx& c, const char* family) {
    if (!probe_match(c, family)) return;
    CK(cudaEventRecord(c.probe.events.back().second, c.stream));
}

}  // namespace amgr

namespace {

thread_local std::string g_err;  // errors before a context exists

amgr_status guard_c(amgr::Ctx* ctx, const std::function<void()>& fn) {
    try {
        if (ctx) CK(cudaSetDevice(ctx->device));
        fn();
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        (ctx ? ctx->last_error : g_err) = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        (ctx ? ctx->last_error : g_err) = "out of host memory";
        return AMGR_E_RUNTIME;
    } catch (const std::exception& e) {
        (ctx ? ctx->last_error : g_err) = e.what();
        return AMGR_E_RUNTIME;
    }
}

amgr_status guard(amgr_ctx* ctx, const std::function<void()>& fn) { return guard_c(ctx ? &ctx->c : nullptr, fn); }

amgr::Ctx* ctx_of(const amgr_hier* h) { return h && h->h ? h->h->ctx : nullptr; }

}  // namespace


extern "C" {

const char* amgr_version(void) { return "amgr_b200 1.0 (sm_100a)"; }

void amgr_amg_params_default(amgr_amg_params* p) {
    if (!p) return;
    p->eps = 0.08;
    p->omega = 0.72;
    p->pre_sweeps = 1;
    p->post_sweeps = 1;
    p->coarse_enough = 100;
    p->max_direct_size = 2000;
    p->smoother = AMGR_SMOOTHER_JACOBI;
    p->coarsening = AMGR_COARSENING_PLAIN;
    p->sa_omega = 2.0 / 3.0;
    p->cheb_degree = 3;
    p->power_iters = 10;
    p->cheb_lower = 0.3;  // interval [0.3, 1] x lambda_max: robust on the nonsymmetric C5 operators
    p->cheb_safety = 1.1;
    p->coarse_solve = AMGR_COARSE_EXACT;
    p->reserved = 0;
}

void amgr_solve_params_default(amgr_solve_params* p) {
    if (!p) return;
    p->tol = 1e-8;
    p->max_iter = 100;
}

amgr_status amgr_ctx_create(int device, void* stream, amgr_ctx** out) {
    if (!out) return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    auto* ctx = new amgr_ctx();
    amgr_status st = guard(nullptr, [&] {
        CK(cudaSetDevice(device));
        ctx->c.device = device;
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        ctx->c.num_sms = sms;
        int major = 0, minor = 0;
        CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
        if (major != 10 || minor != 0)
            amgr::fail(AMGR_E_CUDA, "libamgr_b200 is built for sm_100a (B200); device reports sm_" +
                                        std::to_string(major) + std::to_string(minor));
        {
            const char* e = std::getenv("AMGR_PDL");
            ctx->c.pdl = !(e && std::string(e) == "0");
            const char* sd = std::getenv("AMGR_SEQ_DOTS");
            ctx->c.seq_dots = sd && std::string(sd) == "1";
        }
        if (stream) {
            ctx->c.stream = static_cast<cudaStream_t>(stream);
        } else {
            CK(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
            ctx->c.own_stream = true;
        }
        // keep freed stream-ordered memory in the pool between steps
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    });
    if (st != AMGR_OK) {
        delete ctx;
        return st;
    }
    *out = ctx;
    return AMGR_OK;
}

void amgr_ctx_destroy(amgr_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    for (auto& e : ctx->c.probe.events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    if (ctx->c.copy) {
        cudaStreamSynchronize(ctx->c.copy);
        cudaStreamDestroy(ctx->c.copy);
    }
    if (ctx->c.d2h) {
        cudaStreamSynchronize(ctx->c.d2h);
        if (ctx->c.snap) cudaFree(ctx->c.snap);
        cudaStreamDestroy(ctx->c.d2h);
        cudaEventDestroy(ctx->c.snap_ev);
        cudaEventDestroy(ctx->c.d2h_done_ev);
    }
    if (ctx->c.side) {
        cudaStreamSynchronize(ctx->c.side);
        cudaStreamDestroy(ctx->c.side);
        cudaEventDestroy(ctx->c.fork_ev);
        cudaEventDestroy(ctx->c.join_ev);
    }
    for (cudaEvent_t e : ctx->c.clock_pool) cudaEventDestroy(e);
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
}

const char* amgr_last_error(const amgr_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : g_err.c_str(); }
void* amgr_ctx_stream(const amgr_ctx* ctx) { return ctx ? ctx->c.stream : nullptr; }

amgr_status amgr_ctx_synchronize(amgr_ctx* ctx) {
    return guard(ctx, [&] {
        CK(cudaStreamSynchronize(ctx->c.stream));
        if (ctx->c.copy) CK(cudaStreamSynchronize(ctx->c.copy));
        if (ctx->c.d2h) CK(cudaStreamSynchronize(ctx->c.d2h));
    });
}

amgr_status amgr_ctx_set_dot_order(amgr_ctx* ctx, int order) {
    if (!ctx) return AMGR_E_INVALID_ARGUMENT;
    if (order != AMGR_DOTS_BLOCKED && order != AMGR_DOTS_SEQUENTIAL) {
        ctx->c.last_error = "amgr_ctx_set_dot_order: order must be AMGR_DOTS_BLOCKED or AMGR_DOTS_SEQUENTIAL";
        return AMGR_E_INVALID_ARGUMENT;
    }
    ctx->c.seq_dots = order == AMGR_DOTS_SEQUENTIAL;
    return AMGR_OK;
}

int amgr_ctx_dot_order(const amgr_ctx* ctx) {
    return ctx && ctx->c.seq_dots ? AMGR_DOTS_SEQUENTIAL : AMGR_DOTS_BLOCKED;
}

amgr_status amgr_download_async(amgr_ctx* ctx, const double* device_src, double* host_dst, int64_t n) {
    if (!ctx || n < 0 || (n > 0 && (!device_src || !host_dst))) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        amgr::Ctx& c = ctx->c;
        if (n == 0) return;
        if (!c.d2h) {
            CK(cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c.snap_ev, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c.d2h_done_ev, cudaEventDisableTiming));
            CK(cudaEventRecord(c.d2h_done_ev, c.d2h));
        }
        // the snapshot buffer is reused: the previous download must have drained it
        CK(cudaStreamWaitEvent(c.stream, c.d2h_done_ev, 0));
        if (c.snap_n < n) {
            if (c.snap) CK(cudaFreeAsync(c.snap, c.stream));
            CK(cudaMallocAsync(reinterpret_cast<void**>(&c.snap), sizeof(double) * static_cast<size_t>(n), c.stream));
            c.snap_n = n;
        }
        amgr::d2d(c.snap, device_src, n, c.stream);
        CK(cudaEventRecord(c.snap_ev, c.stream));
        CK(cudaStreamWaitEvent(c.d2h, c.snap_ev, 0));
        amgr::d2h(host_dst, c.snap, n, c.d2h);
        CK(cudaEventRecord(c.d2h_done_ev, c.d2h));
    });
}

amgr_status amgr_setup(amgr_ctx* ctx, const amgr_csr* A, const amgr_amg_params* prm, amgr_hier** out) {
    if (!ctx || !A || !out) return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = amgr::setup(ctx->c, *A, amgr::to_amgp(prm));
        auto* hh = new amgr_hier();
        hh->h = std::move(h);
        *out = hh;
    });
}

amgr_status amgr_partial_update(const amgr_hier* h, const amgr_csr* A, const amgr_amg_params* prm,
                                amgr_hier** out) {
    if (!h || !A || !out) return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    return guard_c(ctx_of(h), [&] {
        auto nh = amgr::partial_update(*h->h, *A, prm ? amgr::to_amgp(prm) : h->h->prm);
        auto* hh = new amgr_hier();
        hh->h = std::move(nh);
        *out = hh;
    });
}

amgr_status amgr_rebuild(amgr_hier* h, const amgr_csr* A) {
    if (!h || !A) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] { amgr::rebuild(*h->h, *A); });
}

amgr_status amgr_stage_values(amgr_hier* h, const double* values, int location) {
    if (!h || !values) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] { amgr::stage_values(*h->h, values, location); });
}

amgr_status amgr_stage_rhs(amgr_hier* h, const double* f, int location) {
    if (!h || !f) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] { amgr::stage_rhs(*h->h, f, location); });
}

amgr_status amgr_rebuild_values(amgr_hier* h, const double* values, int location) {
    if (!h || (!values && location != AMGR_STAGED)) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] { amgr::rebuild_values(*h->h, values, location); });
}

void amgr_hier_destroy(amgr_hier* h) {
    if (!h) return;
    if (h->h && h->h->ctx) cudaSetDevice(h->h->ctx->device);
    delete h;
}

namespace {
// Stage host vectors through device scratch.
struct VecIO {
    amgr::Ctx& c;
    int location;
    std::vector<amgr::DevArray<double>> tmp;
    VecIO(amgr::Ctx& cc, int loc) : c(cc), location(loc) {}
    const double* in(const double* p, int64_t n) {
        if (location == AMGR_DEVICE) return p;
        tmp.emplace_back(n, c.stream);
        amgr::h2d(tmp.back().get(), p, n, c.stream);
        return tmp.back().get();
    }
    double* out(double* p, int64_t n) {
        if (location == AMGR_DEVICE) return p;
        tmp.emplace_back(n, c.stream);
        return tmp.back().get();
    }
    void back(double* host, const double* dev, int64_t n) {
        if (location == AMGR_DEVICE) return;
        amgr::d2h(host, dev, n, c.stream);
        CK(cudaStreamSynchronize(c.stream));
    }
};
}  // namespace

amgr_status amgr_vcycle(amgr_hier* h, const double* f, double* u, int location) {
    if (!h || !f || !u) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        const int64_t n = H.lv.front().pat->n;
        VecIO io(*H.ctx, location);
        const double* fd = io.in(f, n);
        double* ud = io.out(u, n);
        if (fd == ud) amgr::invalid("vcycle: f and u must not alias");
        amgr::vcycle(H, fd, ud);
        io.back(u, ud, n);
    });
}

static amgr_status solve(amgr_hier* h, const double* f, const double* u0, double* u, const amgr_solve_params* prm,
                         amgr_solve_stats* stats, int location, bool use_cg) {
    if (!h || (!f && location != AMGR_STAGED) || !u0 || !u || !stats) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        const int64_t n = H.lv.front().pat->n;
        amgr_solve_params sp;
        amgr_solve_params_default(&sp);
        if (prm) sp = *prm;
        // AMGR_STAGED: f is the RHS staged by amgr_stage_rhs (committed by the
        // STAGED rebuild, or here), u0 / u are device pointers
        const bool staged = location == AMGR_STAGED;
        VecIO io(*H.ctx, staged ? AMGR_DEVICE : location);
        const double* fd = staged ? amgr::committed_rhs(H) : io.in(f, n);
        const bool dev = staged || location == AMGR_DEVICE;
        const double* u0d = (u0 == u && dev) ? u0 : io.in(u0, n);
        double* ud = dev ? u : io.out(u, n);
        if (use_cg)
            amgr::cg(H, fd, u0d, ud, sp, *stats);
        else
            amgr::bicgstab(H, fd, u0d, ud, sp, *stats);
        io.back(u, ud, n);
    });
}

amgr_status amgr_bicgstab(amgr_hier* h, const double* f, const double* u0, double* u,
                          const amgr_solve_params* prm, amgr_solve_stats* stats, int location) {
    return solve(h, f, u0, u, prm, stats, location, false);
}

amgr_status amgr_cg(amgr_hier* h, const double* f, const double* u0, double* u, const amgr_solve_params* prm,
                    amgr_solve_stats* stats, int location) {
    return solve(h, f, u0, u, prm, stats, location, true);
}

amgr_status amgr_spmv(amgr_hier* h, int level, const double* x, double* y, int location) {
    if (!h || !x || !y) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        if (level < 0 || level >= static_cast<int>(H.lv.size())) amgr::invalid("spmv: level out of range");
        const amgr::CsrView A = H.lv[level].view();
        VecIO io(*H.ctx, location);
        const double* xd = io.in(x, A.ncols);
        double* yd = io.out(y, A.n);
        amgr::spmv(*H.ctx, A, xd, yd);
        io.back(y, yd, A.n);
    });
}

// ---- single-operator entry points -------------------------------------------------
amgr_status amgr_csr_spmv(amgr_ctx* ctx, const amgr_csr* A, const double* x, double* y, int location) {
    if (!ctx || !A || (A->ncols > 0 && !x) || (A->nrows > 0 && !y)) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        amgr::Ctx& c = ctx->c;
        VecIO io(c, location);
        const double* xd = io.in(x, A->ncols);
        double* yd = io.out(y, A->nrows);
        amgr::op_spmv(c, *A, xd, yd);
        io.back(y, yd, A->nrows);
    });
}

amgr_status amgr_build_smoother(amgr_ctx* ctx, const amgr_csr* A, double* inv_diag, int location) {
    if (!ctx || !A || (A->nrows > 0 && !inv_diag)) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        amgr::Ctx& c = ctx->c;
        VecIO io(c, location);
        double* wd = io.out(inv_diag, A->nrows);
        amgr::op_build_smoother(c, *A, wd);
        io.back(inv_diag, wd, A->nrows);
    });
}

amgr_status amgr_smooth(amgr_ctx* ctx, const amgr_csr* A, const double* inv_diag, double omega, const double* f,
                        double* u, int sweeps, int location) {
    if (!ctx || !A || (A->nrows > 0 && (!inv_diag || !f || !u))) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        amgr::Ctx& c = ctx->c;
        VecIO io(c, location);
        const double* wd = io.in(inv_diag, A->nrows);
        const double* fd = io.in(f, A->nrows);
        double* ud = location == AMGR_DEVICE ? u : const_cast<double*>(io.in(u, A->nrows));
        amgr::op_smooth(c, *A, wd, omega, fd, ud, sweeps);
        io.back(u, ud, A->nrows);
    });
}

amgr_status amgr_coarse_factorize(amgr_ctx* ctx, const amgr_csr* A, double* lu, int64_t* piv) {
    if (!ctx || !A || (A->nrows > 0 && (!lu || !piv))) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] { amgr::op_coarse_factorize(ctx->c, *A, lu, piv); });
}

amgr_status amgr_coarse_solve(amgr_ctx* ctx, int64_t n, const double* lu, const int64_t* piv, const double* rhs,
                              double* x) {
    if (!ctx || n < 0 || (n > 0 && (!lu || !piv || !rhs || !x))) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] { amgr::op_coarse_solve(ctx->c, n, lu, piv, rhs, x); });
}

int amgr_hier_num_levels(const amgr_hier* h) { return h && h->h ? static_cast<int>(h->h->lv.size()) : 0; }

amgr_status amgr_hier_level_dims(const amgr_hier* h, int level, int64_t* dims) {
    if (!h || !dims) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        const amgr::Hier& H = *h->h;
        if (level < 0 || level >= static_cast<int>(H.lv.size())) amgr::invalid("level out of range");
        const amgr::Level& L = H.lv[level];
        dims[0] = L.pat->n;
        dims[1] = L.pat->nnz;
        dims[2] = L.T ? L.T->nc : 0;
        dims[3] = L.has_smoother ? 1 : 0;
    });
}

amgr_status amgr_hier_level_layout(const amgr_hier* h, int level, int32_t* col_bytes, int32_t* ndict) {
    if (!h) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        const amgr::Hier& H = *h->h;
        if (level < 0 || level >= static_cast<int>(H.lv.size())) amgr::invalid("level out of range");
        const amgr::ColCode& cc = H.lv[level].pat->cc;
        if (col_bytes) *col_bytes = cc.mode == 1 ? 1 : cc.mode == 2 ? 2 : 4;
        if (ndict) *ndict = cc.ndict;
    });
}

amgr_status amgr_hier_level_stencil(const amgr_hier* h, int level, int32_t* pairs, int32_t* off) {
    if (!h || !pairs) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        const amgr::Hier& H = *h->h;
        if (level < 0 || level >= static_cast<int>(H.lv.size())) amgr::invalid("level out of range");
        const amgr::Level& L = H.lv[level];
        *pairs = L.dia_on ? L.pat->dia_k : 0;
        if (off && L.dia_on)
            for (int k = 0; k < L.pat->dia_k; ++k) off[k] = L.pat->doff[k];
    });
}

amgr_status amgr_hier_level_A(const amgr_hier* h, int level, int64_t* row_ptr, int64_t* col, double* values) {
    if (!h) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        amgr::Ctx& c = *H.ctx;
        if (level < 0 || level >= static_cast<int>(H.lv.size())) amgr::invalid("level out of range");
        const amgr::Level& L = H.lv[level];
        amgr::DevArray<int64_t> t(std::max<int64_t>(L.pat->n + 1, L.pat->nnz), c.stream);
        if (row_ptr) {
            amgr::i32_to_i64(c, L.pat->rp.get(), t.get(), L.pat->n + 1);
            amgr::d2h(row_ptr, t.get(), L.pat->n + 1, c.stream);
            CK(cudaStreamSynchronize(c.stream));
        }
        if (col) {
            amgr::i32_to_i64(c, L.pat->col.get(), t.get(), L.pat->nnz);
            amgr::d2h(col, t.get(), L.pat->nnz, c.stream);
            CK(cudaStreamSynchronize(c.stream));
        }
        if (values) amgr::d2h(values, L.view().val, L.pat->nnz, c.stream);
        CK(cudaStreamSynchronize(c.stream));
    });
}

amgr_status amgr_hier_level_P(const amgr_hier* h, int level, int64_t* agg) {
    if (!h || !agg) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        amgr::Ctx& c = *H.ctx;
        if (level < 0 || level >= static_cast<int>(H.lv.size()) || !H.lv[level].T)
            amgr::invalid("level has no transfer operator");
        const amgr::Transfer& T = *H.lv[level].T;
        amgr::DevArray<int64_t> t(T.nf, c.stream);
        amgr::i32_to_i64(c, T.agg.get(), t.get(), T.nf);
        amgr::d2h(agg, t.get(), T.nf, c.stream);
        CK(cudaStreamSynchronize(c.stream));
    });
}

amgr_status amgr_hier_level_R(const amgr_hier* h, int level, int64_t* row_ptr, int64_t* col) {
    if (!h || !row_ptr || !col) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        amgr::Ctx& c = *H.ctx;
        if (level < 0 || level >= static_cast<int>(H.lv.size()) || !H.lv[level].T)
            amgr::invalid("level has no transfer operator");
        const amgr::Transfer& T = *H.lv[level].T;
        if (T.smoothed) amgr::invalid("smoothed aggregation level: use amgr_hier_level_transfer");
        amgr::DevArray<int64_t> t(std::max(T.nf, T.nc + 1), c.stream);
        amgr::i32_to_i64(c, T.mptr.get(), t.get(), T.nc + 1);
        amgr::d2h(row_ptr, t.get(), T.nc + 1, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        amgr::i32_to_i64(c, T.midx.get(), t.get(), T.nf);
        amgr::d2h(col, t.get(), T.nf, c.stream);
        CK(cudaStreamSynchronize(c.stream));
    });
}

amgr_status amgr_hier_level_transfer(const amgr_hier* h, int level, int which, int64_t* nnz, int64_t* row_ptr,
                                     int64_t* col, double* values) {
    if (!h || !nnz || (which != 0 && which != 1)) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        amgr::Ctx& c = *H.ctx;
        if (level < 0 || level >= static_cast<int>(H.lv.size()) || !H.lv[level].T)
            amgr::invalid("level has no transfer operator");
        const amgr::Transfer& T = *H.lv[level].T;
        const int64_t rows = which == 0 ? T.nf : T.nc;
        if (T.smoothed) {
            const amgr::Pattern& M = which == 0 ? *T.P : *T.R;
            *nnz = M.nnz;
            if (!row_ptr) return;
            if (!col || !values) amgr::invalid("amgr_hier_level_transfer: null output buffer");
            amgr::DevArray<int64_t> t(std::max(M.nnz, rows + 1), c.stream);
            amgr::i32_to_i64(c, M.rp.get(), t.get(), rows + 1);
            amgr::d2h(row_ptr, t.get(), rows + 1, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            amgr::i32_to_i64(c, M.col.get(), t.get(), M.nnz);
            amgr::d2h(col, t.get(), M.nnz, c.stream);
            amgr::d2h(values, (which == 0 ? T.Pv : T.Rv).get(), M.nnz, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            return;
        }
        // tentative: P row i = (agg_i, 1.0); R = member lists with 1.0
        *nnz = T.nf;
        if (!row_ptr) return;
        if (!col || !values) amgr::invalid("amgr_hier_level_transfer: null output buffer");
        amgr::DevArray<int64_t> t(T.nf + 1, c.stream);
        if (which == 0) {
            std::vector<int64_t> rp(static_cast<size_t>(T.nf + 1));
            for (int64_t i = 0; i <= T.nf; ++i) rp[i] = i;
            std::copy(rp.begin(), rp.end(), row_ptr);
            amgr::i32_to_i64(c, T.agg.get(), t.get(), T.nf);
        } else {
            amgr::i32_to_i64(c, T.mptr.get(), t.get(), T.nc + 1);
            amgr::d2h(row_ptr, t.get(), T.nc + 1, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            amgr::i32_to_i64(c, T.midx.get(), t.get(), T.nf);
        }
        amgr::d2h(col, t.get(), T.nf, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        for (int64_t k = 0; k < T.nf; ++k) values[k] = 1.0;
    });
}

amgr_status amgr_hier_level_smoother(const amgr_hier* h, int level, double* w) {
    if (!h || !w) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        if (level < 0 || level >= static_cast<int>(H.lv.size()) || !H.lv[level].has_smoother)
            amgr::invalid("level has no smoother");
        amgr::d2h(w, H.lv[level].w.get(), H.lv[level].pat->n, H.ctx->stream);
        CK(cudaStreamSynchronize(H.ctx->stream));
    });
}

amgr_status amgr_hier_level_lambda(const amgr_hier* h, int level, double* lam) {
    if (!h || !lam) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        if (level < 0 || level >= static_cast<int>(H.lv.size()) || H.lv[level].pst.size() != 3)
            amgr::invalid("level has no Chebyshev smoother");
        double st[3];
        amgr::d2h(st, H.lv[level].pst.get(), 3, H.ctx->stream);
        CK(cudaStreamSynchronize(H.ctx->stream));
        *lam = st[2];
    });
}

int64_t amgr_hier_coarse_n(const amgr_hier* h) { return h && h->h ? h->h->nL : 0; }

amgr_status amgr_hier_coarse_lu(const amgr_hier* h, double* lu, int64_t* piv) {
    if (!h || !lu || !piv) return AMGR_E_INVALID_ARGUMENT;
    return guard_c(ctx_of(h), [&] {
        amgr::Hier& H = *h->h;
        if (!H.lu_formed)
            amgr::invalid("amgr_hier_coarse_lu: no LU factor is formed in the inverse coarse-solve mode");
        amgr::d2h(lu, H.lu.get(), H.nL * H.nL, H.ctx->stream);
        amgr::d2h(piv, H.piv.get(), H.nL, H.ctx->stream);
        CK(cudaStreamSynchronize(H.ctx->stream));
    });
}

double amgr_hier_operator_complexity(const amgr_hier* h) {
    if (!h || !h->h) return 0.0;
    double t = 0;
    for (auto& L : h->h->lv) t += static_cast<double>(L.pat->nnz);
    return t / static_cast<double>(h->h->lv.front().pat->nnz);
}

amgr_status amgr_hier_timings(const amgr_hier* h, amgr_phase_timings* t) {
    if (!h || !t) return AMGR_E_INVALID_ARGUMENT;
    *t = h->h->tm;
    return AMGR_OK;
}

int amgr_hier_shares_transfer(const amgr_hier* a, const amgr_hier* b, int level) {
    if (!a || !b || !a->h || !b->h) return 0;
    if (level < 0 || level >= static_cast<int>(a->h->lv.size()) || level >= static_cast<int>(b->h->lv.size()))
        return 0;
    return a->h->lv[level].T && a->h->lv[level].T.get() == b->h->lv[level].T.get() ? 1 : 0;
}

int64_t amgr_problem_nnz(int64_t g) { return amgr::problem_nnz(g); }

amgr_status amgr_problem_pattern(amgr_ctx* ctx, int64_t g, int32_t* row_ptr, int32_t* col) {
    if (!ctx || !row_ptr || !col || g < 1) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] { amgr::problem_pattern(ctx->c, g, row_ptr, col); });
}

amgr_status amgr_problem_values(amgr_ctx* ctx, int kind, int64_t g, int64_t k, int64_t nsteps, double* values) {
    if (!ctx || !values || g < 1) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] { amgr::problem_values(ctx->c, kind, g, k, nsteps, values); });
}

amgr_status amgr_problem_rhs(amgr_ctx* ctx, int64_t n, uint64_t seed, double* out, int location) {
    if (!out || n < 0) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        // diffusion.cpp:38-41: std::mt19937_64(seed), uniform_real_distribution(0.1, 1.0)
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> dist(0.1, 1.0);
        std::vector<double> v(static_cast<size_t>(n));
        for (double& x : v) x = dist(rng);
        if (location == AMGR_DEVICE) {
            if (!ctx) amgr::invalid("device output needs a context");
            amgr::h2d(out, v.data(), n, ctx->c.stream);
            CK(cudaStreamSynchronize(ctx->c.stream));
        } else {
            std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(n));
        }
    });
}

amgr_status amgr_probe_enable(amgr_ctx* ctx, const char* family) {
    if (!ctx) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        CK(cudaStreamSynchronize(ctx->c.stream));
        for (auto& e : ctx->c.probe.events) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        ctx->c.probe.events.clear();
        ctx->c.probe.bytes.clear();
        std::string f = family ? family : "";
        int level = -1;
        const auto at = f.find('@');
        if (at != std::string::npos) {
            level = std::stoi(f.substr(at + 1));
            f = f.substr(0, at);
        }
        ctx->c.probe.family = f;
        ctx->c.probe.level = level;
    });
}

amgr_status amgr_probe_read(amgr_ctx* ctx, int64_t* launches, double* ms, double* bytes) {
    if (!ctx) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        CK(cudaStreamSynchronize(ctx->c.stream));
        double t = 0, b = 0;
        for (size_t i = 0; i < ctx->c.probe.events.size(); ++i) {
            float m = 0.f;
            CK(cudaEventElapsedTime(&m, ctx->c.probe.events[i].first, ctx->c.probe.events[i].second));
            t += m;
            b += ctx->c.probe.bytes[i];
        }
        if (launches) *launches = static_cast<int64_t>(ctx->c.probe.events.size());
        if (ms) *ms = t;
        if (bytes) *bytes = b;
    });
}

amgr_status amgr_copy_to_host(amgr_ctx* ctx, void* host, const void* device, size_t bytes) {
    if (!ctx || (!host && bytes)) return AMGR_E_INVALID_ARGUMENT;
    return guard(ctx, [&] {
        if (bytes) CK(cudaMemcpyAsync(host, device, bytes, cudaMemcpyDeviceToHost, ctx->c.stream));
        CK(cudaStreamSynchronize(ctx->c.stream));
    });
}

int64_t amgr_launch_count(const amgr_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

}  // extern "C"

/*
 * amgr.h — C-ABI of the B200-native partial-reuse AMG path (libamgr_b200.so).
 *
 * This is the drop-in boundary for the reference's C++ solver API
 * (/root/reference/proj, library `amgreuse`).  Every entry point names the
 * reference interface it replaces.  The reference's own FFI for this path is
 * the pybind11 module `_core` declared at proj/CMakeLists.txt:40-82 (its source
 * python/bindings.cpp is absent from the reference), so the binding a
 * maintainer adds is a ctypes / pybind / plain C++ stub over these symbols —
 * see INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types in signatures
 *    (streams are passed as void*, i.e. a cudaStream_t).
 *  - Index arrays may be int32 or int64 (amgr_csr.index_bits); values are fp64
 *    (the reference is fp64 throughout, SPEC.md "Real values are 64-bit").
 *  - Buffers may live on the host or on the device (amgr_csr.location /
 *    the `location` arguments); device buffers must belong to the context's
 *    device.  Host buffers are copied in/out inside the call.
 *  - Errors: every call returns amgr_status.  The message (same text as the
 *    reference's exception, e.g. "partial update impossible, full rebuild
 *    required: ...", "level 0: strength_graph: zero diagonal at row 3",
 *    "setup: coarsening stalled at level ...", "coarse_factorize: singular
 *    matrix (zero pivot at step k)") is available from amgr_last_error().
 *    AMGR_E_INVALID_ARGUMENT <-> std::invalid_argument,
 *    AMGR_E_RUNTIME <-> std::runtime_error.
 *  - Solver non-convergence / breakdown are NOT errors; they are reported in
 *    amgr_solve_stats exactly like the reference's SolveStats
 *    (proj/include/amgreuse/bicgstab.hpp:22-27).
 *  - Threading: a context (and every hierarchy created from it) is bound to
 *    one device and one stream; calls on one context must be serialised by
 *    the caller.  Hierarchies are immutable except through amgr_rebuild
 *    (the in-place variant of partial_update).
 */
#ifndef AMGR_H
#define AMGR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum amgr_status {
    AMGR_OK = 0,
    AMGR_E_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference     */
    AMGR_E_RUNTIME = 2,          /* std::runtime_error in the reference        */
    AMGR_E_CUDA = 3,             /* CUDA runtime / launch failure               */
    AMGR_E_NCCL = 4,             /* NCCL failure (multi-GPU path)               */
    AMGR_E_DIMENSION = 5         /* partial_update dimension change: the caller
                                    must do a full setup (reuse.cpp:69-70,84);
                                    message text identical to the reference's   */
} amgr_status;

enum { AMGR_HOST = 0, AMGR_DEVICE = 1,
       /* amgr_rebuild_values only: the hierarchy adopts the device buffer
        * (zero copy) until the next rebuild; it must stay valid and
        * unmodified, be 16-byte aligned and have >= 32 bytes of slack past
        * the last value (read by 16-byte TMA bulk copies). */
       AMGR_DEVICE_ADOPT = 2,
       /* amgr_rebuild_values (values = NULL): use the values staged by the
        * last amgr_stage_values (swapped in, no copy); a pending
        * amgr_stage_rhs is committed with them.  amgr_bicgstab / amgr_cg
        * (f = NULL): f = the RHS committed by the last STAGED rebuild
        * (staging the next step's RHS meanwhile does not change it), u0 and
        * u are device pointers. */
       AMGR_STAGED = 3 };

/* Smoother kinds.  JACOBI is the reference's (smoother.hpp:11-16); SPAI0 and
 * CHEBYSHEV are north-star extensions with restated oracles (parity unpinned
 * by the reference). */
enum { AMGR_SMOOTHER_JACOBI = 0, AMGR_SMOOTHER_SPAI0 = 1, AMGR_SMOOTHER_CHEBYSHEV = 2 };
/* Coarsening: plain (tentative, piecewise-constant P; the reference's only
 * kind, coarsening.hpp:48-50) or smoothed aggregation (extension). */
enum { AMGR_COARSENING_PLAIN = 0, AMGR_COARSENING_SMOOTHED = 1 };
/* Coarse direct solve: EXACT replays the reference's LU solve order
 * (dense_lu.cpp:52-73) bit for bit; INVERSE (extension) applies the explicit
 * inverse formed from the same LU factors at rebuild time (a parallel matvec,
 * rounding differs at the 1e-16 level). */
enum { AMGR_COARSE_EXACT = 0, AMGR_COARSE_INVERSE = 1 };

/* CSR input.  Invariants as CsrMatrix (proj/include/amgreuse/csr.hpp:20-27):
 * row_ptr non-decreasing, row_ptr[0]=0, row_ptr[nrows]=nnz, columns strictly
 * increasing within a row. */
typedef struct amgr_csr {
    int64_t nrows;
    int64_t ncols;
    int64_t nnz;
    const void* row_ptr; /* nrows+1 entries of int32 or int64              */
    const void* col_idx; /* nnz entries of int32 or int64                  */
    const double* values;
    int32_t index_bits;  /* 32 or 64                                       */
    int32_t location;    /* AMGR_HOST or AMGR_DEVICE                       */
} amgr_csr;

/* AmgParams (proj/include/amgreuse/hierarchy.hpp:14-21) + extensions. */
typedef struct amgr_amg_params {
    double eps;              /* 0.08  strength threshold                    */
    double omega;            /* 0.72  Jacobi damping                        */
    int32_t pre_sweeps;      /* 1                                           */
    int32_t post_sweeps;     /* 1                                           */
    int64_t coarse_enough;   /* 100                                         */
    int64_t max_direct_size; /* 2000                                        */
    int32_t smoother;        /* AMGR_SMOOTHER_*        (extension)          */
    int32_t coarsening;      /* AMGR_COARSENING_*      (extension)          */
    double sa_omega;         /* smoothed-aggregation damping (extension)    */
    int32_t cheb_degree;     /* Chebyshev degree (extension)                */
    int32_t power_iters;     /* power iterations for lambda_max (extension) */
    double cheb_lower;       /* lambda_min = cheb_lower * lambda_max (0.3)  */
    double cheb_safety;      /* lambda_max safety factor                    */
    int32_t coarse_solve;    /* AMGR_COARSE_*          (extension)          */
    int32_t reserved;
} amgr_amg_params;

/* SolveParams (bicgstab.hpp:17-20). */
typedef struct amgr_solve_params {
    double tol;       /* 1e-8 */
    int64_t max_iter; /* 100  */
} amgr_solve_params;

/* SolveStats (bicgstab.hpp:22-27). */
typedef struct amgr_solve_stats {
    int64_t iterations;
    double relative_residual;
    int32_t converged;
    int32_t breakdown;
} amgr_solve_stats;

/* SetupPhaseTimings (hierarchy.hpp:24-38), seconds, measured with CUDA events
 * on the context stream. */
typedef struct amgr_phase_timings {
    double transfer_ops;
    double galerkin;
    double smoother;
    double coarse_solver;
} amgr_phase_timings;

typedef struct amgr_ctx amgr_ctx;
typedef struct amgr_hier amgr_hier;

/* ---- context ------------------------------------------------------------ */
/* Binds a device and a stream (NULL stream => the library creates its own). */
amgr_status amgr_ctx_create(int device, void* stream, amgr_ctx** out);
void amgr_ctx_destroy(amgr_ctx* ctx);
const char* amgr_last_error(const amgr_ctx* ctx);
void* amgr_ctx_stream(const amgr_ctx* ctx);
/* Dot-product order of amgr_bicgstab / amgr_cg (parity mode, extension).
 * AMGR_DOTS_BLOCKED (default): deterministic per-block partials fused into the
 * producing kernels, fixed-order grid reduction.  AMGR_DOTS_SEQUENTIAL: every
 * dot and norm summed strictly left to right from 0.0 with rounded products,
 * exactly the reference's dot/norm2 (proj/src/bicgstab.cpp:11-17), so with
 * the exact coarse solve the iterates are bit-identical to the reference's
 * bicgstab (bicgstab.cpp:21-135) over the fixed V-cycle.  One CTA runs each
 * sum: ~8 ms per dot at 2.1M rows.  The environment variable AMGR_SEQ_DOTS=1
 * sets it at context creation. */
#define AMGR_DOTS_BLOCKED 0
#define AMGR_DOTS_SEQUENTIAL 1
amgr_status amgr_ctx_set_dot_order(amgr_ctx* ctx, int order);
int amgr_ctx_dot_order(const amgr_ctx* ctx);
/* Waits for the context stream and the copy / download streams. */
amgr_status amgr_ctx_synchronize(amgr_ctx* ctx);
/* Pipelining (extension): snapshot n doubles of device memory on the context
 * stream (after the work queued so far) and copy them to host_dst on a
 * download stream, so the transfer overlaps the next calls' device work.
 * host_dst is complete after amgr_ctx_synchronize (pinned memory for overlap). */
amgr_status amgr_download_async(amgr_ctx* ctx, const double* device_src, double* host_dst, int64_t n);
/* Library version string and the compiled architecture ("sm_100a"). */
const char* amgr_version(void);

/* Defaults of AmgParams / SolveParams (hierarchy.hpp:14-21, bicgstab.hpp:17-20). */
void amgr_amg_params_default(amgr_amg_params* p);
void amgr_solve_params_default(amgr_solve_params* p);

/* ---- hierarchy: setup / partial_update / vcycle -------------------------- */
/* Replaces `Hierarchy setup(const CsrMatrix&, const AmgParams&)`
 * (hierarchy.hpp:65, hierarchy.cpp:45-105): full AMG setup on the device —
 * strength graph, exact replay of the sequential greedy aggregation,
 * P/R, symbolic + numeric Galerkin product, smoothers, coarse LU. */
amgr_status amgr_setup(amgr_ctx* ctx, const amgr_csr* A, const amgr_amg_params* prm,
                       amgr_hier** out);

/* Replaces `Hierarchy partial_update(const Hierarchy&, CsrMatrix, const AmgParams&)`
 * (hierarchy.hpp:71, hierarchy.cpp:107-150): returns a NEW hierarchy that
 * shares the frozen transfer operators (and the cached Galerkin pattern) of
 * `h`; level matrices, smoothers and the coarse LU are recomputed from A_new.
 * A pattern change (same dimensions) re-runs the symbolic product.
 * Dimension change => AMGR_E_DIMENSION with the reference's message. */
amgr_status amgr_partial_update(const amgr_hier* h, const amgr_csr* A_new,
                                const amgr_amg_params* prm, amgr_hier** out);

/* In-place partial update ("rebuild(A)"): same semantics as
 * amgr_partial_update but overwrites `h` (no allocation on the values-only
 * path).  This is the per-time-step hot path. */
amgr_status amgr_rebuild(amgr_hier* h, const amgr_csr* A_new);

/* Values-only rebuild: `values` are the new A_0 entries in the CSR order of
 * the hierarchy's finest pattern (nnz of level 0 entries).  The caller
 * asserts the pattern is unchanged. */
/* Pipelining (extension): copy the NEXT step's A_0 values (host or device)
 * into a per-hierarchy staging buffer on the context's copy stream, ordered
 * after the work already queued on the context stream, so the transfer runs
 * on the copy engines while the current step's solve computes.  Consume with
 * amgr_rebuild_values(h, NULL, AMGR_STAGED). */
amgr_status amgr_stage_values(amgr_hier* h, const double* values, int location);
/* Pipelining (extension): the same for the next step's right-hand side
 * (finest_size entries); committed by the next STAGED rebuild, then read by
 * the STAGED solves until the following one. */
amgr_status amgr_stage_rhs(amgr_hier* h, const double* f, int location);
amgr_status amgr_rebuild_values(amgr_hier* h, const double* values, int location);

/* Replaces `std::vector<double> vcycle(const Hierarchy&, span f, const AmgParams&)`
 * (hierarchy.hpp:75-76, hierarchy.cpp:152-186) with the smoothing the
 * reference's documentation specifies.  f/u have
 * finest_size entries on `location`. */
amgr_status amgr_vcycle(amgr_hier* h, const double* f, double* u, int location);

void amgr_hier_destroy(amgr_hier* h);

/* ---- Krylov ------------------------------------------------------------- */
/* Replaces `bicgstab(make_operator(A), make_preconditioner(h), f, u0, prm)`
 * (bicgstab.hpp:34-44, bicgstab.cpp:21-135): right-preconditioned BiCGStab,
 * A = the hierarchy's finest matrix, M = one V-cycle.  u0 may equal u. */
amgr_status amgr_bicgstab(amgr_hier* h, const double* f, const double* u0, double* u,
                          const amgr_solve_params* prm, amgr_solve_stats* stats, int location);

/* Preconditioned CG (extension; SPEC.md lists CG as a non-goal of the
 * reference — restated oracle, parity unpinned). */
amgr_status amgr_cg(amgr_hier* h, const double* f, const double* u0, double* u,
                    const amgr_solve_params* prm, amgr_solve_stats* stats, int location);

/* y = A_level x (spmv, csr.hpp:77 / csr.cpp:76-85) on one level. */
amgr_status amgr_spmv(amgr_hier* h, int level, const double* x, double* y, int location);

/* ---- reuse driver (proj/include/amgreuse/reuse.hpp:13-81, src/reuse.cpp) -- */
/* StrategyKind (reuse.hpp:13) */
enum { AMGR_REUSE_NONE = 0, AMGR_REUSE_FULL = 1, AMGR_REUSE_PARTIAL = 2 };
/* StepAction (reuse.hpp:31) */
enum { AMGR_ACTION_FULL_BUILD = 0, AMGR_ACTION_PARTIAL_UPDATE = 1, AMGR_ACTION_REUSED_UNCHANGED = 2 };

/* StrategyConfig (reuse.hpp:20-28).  rebuild_every <= 0 means "absent".
 * flags (extension, SPEC.md:444-447 leaves it unspecified):
 * AMGR_STRATEGY_ESCALATE makes partial reuse convergence-triggered — after a
 * solve that did not converge or used >= reuse_iter_limit iterations (max_iter
 * when 0) the next step is a full build, the rule the reference applies to
 * full reuse (reuse.cpp:116-117). */
enum { AMGR_STRATEGY_ESCALATE = 1 };
typedef struct amgr_strategy {
    int32_t kind;
    int32_t flags;
    int64_t reuse_iter_limit;
    int64_t rebuild_every;
} amgr_strategy;

/* StepMetrics (reuse.hpp:33-41); times in seconds (CUDA events on the stream). */
typedef struct amgr_step_metrics {
    int64_t step;
    double setup_time;
    double solve_time;
    int64_t iterations;
    int32_t converged;
    int32_t action;
    amgr_phase_timings phase_timings;
} amgr_step_metrics;

/* ProblemSequence::step(k) (sequence.hpp:11-23): fill *A and *rhs for step k
 * (host or device buffers, valid until the next call).  Return 0 on success. */
typedef int (*amgr_step_fn)(void* user, int64_t k, amgr_csr* A, const double** rhs, int32_t* rhs_location);
/* Optional per-step solution sink: u has n entries on the device. */
typedef void (*amgr_solution_fn)(void* user, int64_t k, const double* u_device, int64_t n);

/* Replaces `RunResult run_sequence(const ProblemSequence&, const StrategyConfig&,
 * const AmgParams&, const SolveParams&)` (reuse.hpp:70-71, reuse.cpp:46-136):
 * same actions, chaining of the previous solution as the initial guess, the
 * full-reuse rebuild flag, the dimension-change fallback.  metrics: nsteps
 * entries.  Solver non-convergence is recorded, not raised. */
amgr_status amgr_run_sequence(amgr_ctx* ctx, int64_t nsteps, amgr_step_fn step, void* user,
                              const amgr_strategy* strategy, const amgr_amg_params* amg,
                              const amgr_solve_params* solve, amgr_step_metrics* metrics,
                              amgr_solution_fn sink, void* sink_user);

/* speedup_percent (reuse.cpp:138-147): (t_base / t_other - 1) * 100, +inf
 * when t_other == 0. */
double amgr_speedup_percent(double t_base, double t_other);

/* ---- row-partitioned multi-GPU solve ---------------------- */
/* One rank per GPU.  Every rank builds the same global hierarchy with
 * amgr_setup; levels 0..top are then row-partitioned (aggregate-consistent
 * ownership computed host-side by paper_2108_02054_b200/partition.py), levels
 * top+1.. are replicated.  Halo exchange: ncclSend/ncclRecv; dots: allgather
 * of per-rank partials summed in rank order (identical on every rank). */
typedef struct amgr_dist amgr_dist;
typedef struct amgr_dist_level {
    int64_t n_own, n_halo, nnz, n_coarse_owned;
    const int64_t* row_ptr;  /* n_own+1, local CSR rows = owned rows ascending   */
    const int64_t* col;      /* nnz, local column ids: owned [0,n_own) | halo      */
    const int64_t* nnz_map;  /* nnz, local entry -> global entry of level A_i      */
    const int64_t* owned;    /* n_own, global row ids                              */
    const int64_t* agg;      /* n_own, local coarse id (global id at level top)    */
    const int64_t* mptr;     /* n_coarse_owned+1, members of owned coarse rows     */
    const int64_t* midx;     /* local fine ids, ascending                          */
    int32_t n_send_peers, n_recv_peers;
    const int32_t* send_peer;
    const int64_t* send_cnt;
    const int64_t* send_idx; /* concatenated per send peer: local owned ids        */
    const int32_t* recv_peer;
    const int64_t* recv_off; /* offset of the peer's block inside the halo         */
    const int64_t* recv_cnt;
} amgr_dist_level;

amgr_status amgr_nccl_unique_id(void* out128);
/* t_counts[r]: level-(top+1) rows restricted by rank r (contiguous, rank order). */
amgr_status amgr_dist_create(amgr_hier* global, const void* nccl_id128, int rank, int world, int top,
                             const amgr_dist_level* levels, int64_t t_count_total, const int64_t* t_counts,
                             amgr_dist** out);
/* amgr_dist_rebuild_values: global rebuild on every rank + gather of the
 * local values (needs the global A_k on every rank).
 * amgr_dist_rebuild_local: partial rebuild from RANK-LOCAL values — this
 * rank's owned rows of A_k in the local CSR order (owned rows ascending, each
 * row's entries in the global column order, i.e. global_values[nnz_map]).
 * Each rank rebuilds the Jacobi weights of its rows and the numeric Galerkin
 * product of its own coarse rows (communication-free: the partition is
 * aggregate-consistent, so every member row is local; local plans built on the
 * device at amgr_dist_create), one allgather replicates A_{top+1}, and the
 * replicated levels are rebuilt on every rank.  Bit-identical to the global
 * partial_update; errors name the global row and are raised on every rank. */
amgr_status amgr_dist_rebuild_local(amgr_dist* d, const double* local_values, int location);
/* Partition built ON THE DEVICE from the hierarchy's own patterns and
 * aggregates (dist_plan.cu; the rules of partition.py, identical arrays):
 * levels with >= replicate_below rows (never the coarsest) are partitioned.
 * No host plan, no pattern download. */
amgr_status amgr_dist_create_auto(amgr_hier* global, const void* nccl_id128, int rank, int world,
                                  int64_t replicate_below, amgr_dist** out);
/* dims: {n_own, n_halo, nnz, n_coarse_owned, top} of partitioned level `level`. */
amgr_status amgr_dist_level_dims(const amgr_dist* d, int level, int64_t* dims);
/* owned: n_own global row ids; nnz_map: nnz global entry ids (either may be NULL). */
amgr_status amgr_dist_level_maps(amgr_dist* d, int level, int64_t* owned, int64_t* nnz_map);
/* bytes per entry of partitioned level `level`'s column stream in the row
 * passes: 1 / 2 (coded, col = row + dict[code]) or 4 (int32 columns). */
amgr_status amgr_dist_level_code(const amgr_dist* d, int level, int* col_bytes);
/* Test transport: W ranks of ONE process (one host thread and one context
 * each, same device) exchange through stream-ordered device copies and host
 * barriers instead of NCCL, so the multi-rank device path can be checked on
 * a single GPU.  Same plan arguments as amgr_dist_create. */
typedef struct amgr_loopback amgr_loopback;
amgr_status amgr_dist_loopback_create(int world, amgr_loopback** out);
void amgr_dist_loopback_destroy(amgr_loopback* lb);
amgr_status amgr_dist_create_auto_loopback(amgr_hier* global, amgr_loopback* lb, int rank, int world,
                                           int64_t replicate_below, amgr_dist** out);
amgr_status amgr_dist_create_loopback(amgr_hier* global, amgr_loopback* lb, int rank, int world, int top,
                                      const amgr_dist_level* levels, int64_t t_count_total, const int64_t* t_counts,
                                      amgr_dist** out);
amgr_status amgr_dist_rebuild_values(amgr_dist* d, const double* global_values, int location);
/* f/u: device vectors over the owned level-0 rows. */
amgr_status amgr_dist_vcycle(amgr_dist* d, const double* f_local, double* u_local);
amgr_status amgr_dist_bicgstab(amgr_dist* d, const double* f_local, double* u_local,
                               const amgr_solve_params* prm, amgr_solve_stats* stats);
void amgr_dist_destroy(amgr_dist* d);

/* ---- single-operator entry points ------------------------------------------
 * The reference's free functions on ONE matrix, for the source-compatible
 * C++ facade (include/amgreuse_gpu.hpp) and callers that need them outside a
 * hierarchy.  Vectors are host or device (location); the LU pair is host.
 * Errors carry the reference's texts. */
/* spmv(const CsrMatrix&, span x, span y)                      csr.cpp:76-85 */
amgr_status amgr_csr_spmv(amgr_ctx* ctx, const amgr_csr* A, const double* x, double* y, int location);
/* build_smoother(const CsrMatrix&, double) -> inv_diag          smoother.cpp:8-32
 * ("build_smoother: zero diagonal at row i", invalid argument) */
amgr_status amgr_build_smoother(amgr_ctx* ctx, const amgr_csr* A, double* inv_diag, int location);
/* smooth(s, A, f, span u, sweeps): u <- u + omega*inv_diag*(f - A u)  smoother.cpp:34-48 */
amgr_status amgr_smooth(amgr_ctx* ctx, const amgr_csr* A, const double* inv_diag, double omega, const double* f,
                        double* u, int sweeps, int location);
/* coarse_factorize(const CsrMatrix&): lu (n*n row-major) + piv   dense_lu.cpp:10-50
 * ("coarse_factorize: singular matrix (zero pivot at step k)", runtime error) */
amgr_status amgr_coarse_factorize(amgr_ctx* ctx, const amgr_csr* A, double* lu, int64_t* piv);
/* coarse_solve(const DenseFactorization&, span rhs)              dense_lu.cpp:52-73 */
amgr_status amgr_coarse_solve(amgr_ctx* ctx, int64_t n, const double* lu, const int64_t* piv, const double* rhs,
                              double* x);

/* ---- Matrix Market ingestion (matrix_market.hpp:12-27) -------------------- */
/* A device CSR owned by the library (int32 indices, fp64 values). */
typedef struct amgr_matrix amgr_matrix;
/* mm_read (matrix_market.cpp:104-140): coordinate real/integer, general or
 * symmetric (expanded); parsed on the host (multi-threaded), assembled on the
 * device exactly as csr_from_triplets (csr.cpp:24-75).  Errors: AMGR_E_RUNTIME
 * with the reference's "path:line: message" text. */
amgr_status amgr_mm_read(amgr_ctx* ctx, const char* path, amgr_matrix** out);
/* csr_from_triplets (csr.cpp:24-75) assembled on the device: rows sorted,
 * duplicates summed in input order; the reference's error texts. */
amgr_status amgr_csr_from_triplets(amgr_ctx* ctx, int64_t nrows, int64_t ncols, int64_t count, const int64_t* rows,
                                   const int64_t* cols, const double* values, amgr_matrix** out);
/* Device view for amgr_setup / amgr_rebuild (location AMGR_DEVICE). */
amgr_status amgr_matrix_csr(const amgr_matrix* m, amgr_csr* view);
void amgr_matrix_free(amgr_matrix* m);
/* mm_read_vector (matrix_market.cpp:176-203) into a host buffer: *n in =
 * capacity (values may be NULL to query), out = length. */
amgr_status amgr_mm_read_vector(amgr_ctx* ctx, const char* path, int64_t* n, double* values);

/* ---- introspection / download (parity dumps) ----------------------------- */
/* Number of levels, finest first (Hierarchy::num_levels, hierarchy.hpp:54). */
int amgr_hier_num_levels(const amgr_hier* h);
/* dims[0]=nrows, dims[1]=nnz, dims[2]=n_coarse (0 on the coarsest level),
 * dims[3]=has_smoother. */
amgr_status amgr_hier_level_dims(const amgr_hier* h, int level, int64_t* dims);
/* Row-pass layout of A_level (no reference counterpart):
 * *col_bytes = bytes per stored column in the row passes (4 = int32 columns,
 * 1 / 2 = coded column stream col = row + dict[code]), *ndict = dictionary
 * size (0 when uncoded).  Either pointer may be NULL. */
amgr_status amgr_hier_level_layout(const amgr_hier* h, int level, int32_t* col_bytes, int32_t* ndict);
/* Symmetric-stencil form of A_level (no reference counterpart):
 * *pairs = K > 0 when the row passes currently read A_level as its diagonal
 * plus K upper diagonals (columns i + {0, +-off[k]}, values bitwise symmetric,
 * checked at every rebuild), 0 when they read the CSR arrays; off (K ints,
 * may be NULL) receives the offsets. */
amgr_status amgr_hier_level_stencil(const amgr_hier* h, int level, int32_t* pairs, int32_t* off);
/* A_level as int64 CSR (row_ptr nrows+1, col nnz, values nnz) into host buffers. */
amgr_status amgr_hier_level_A(const amgr_hier* h, int level, int64_t* row_ptr, int64_t* col,
                              double* values);
/* Aggregate id of every fine row (= col_idx of the tentative P,
 * coarsening.cpp:122-132) and R = P^T as CSR (row_ptr n_coarse+1, col n). */
amgr_status amgr_hier_level_P(const amgr_hier* h, int level, int64_t* agg);
amgr_status amgr_hier_level_R(const amgr_hier* h, int level, int64_t* row_ptr, int64_t* col);
/* P (which = 0, nrows x n_coarse) or R = P^T (which = 1) of a level as a
 * general CSR with values: the tentative P (one 1.0 per row) or the smoothed
 * prolongator of the smoothed-aggregation extension.  Call with
 * row_ptr == NULL to query *nnz, then with buffers of nrows+1 / nnz / nnz. */
amgr_status amgr_hier_level_transfer(const amgr_hier* h, int level, int which, int64_t* nnz, int64_t* row_ptr,
                                     int64_t* col, double* values);
/* Smoother state: inv_diag (JacobiSmoother::inv_diag, smoother.hpp:11-16). */
amgr_status amgr_hier_level_smoother(const amgr_hier* h, int level, double* inv_diag);
/* Chebyshev extension: power-iteration estimate of lambda_max(D^-1 A) of a
 * level (before the safety factor). */
amgr_status amgr_hier_level_lambda(const amgr_hier* h, int level, double* lambda_max);
/* Coarse LU (DenseFactorization, dense_lu.hpp:12-18): lu n*n row-major, piv n. */
int64_t amgr_hier_coarse_n(const amgr_hier* h);
amgr_status amgr_hier_coarse_lu(const amgr_hier* h, double* lu, int64_t* piv);
/* Hierarchy::operator_complexity (hierarchy.cpp:39-43). */
double amgr_hier_operator_complexity(const amgr_hier* h);
/* setup_timings of the last setup / partial update / rebuild. */
amgr_status amgr_hier_timings(const amgr_hier* h, amgr_phase_timings* t);
/* Shared-transfer identity check (test_hierarchy.cpp:111-121 analogue):
 * returns 1 when both hierarchies share the same frozen P/R objects. */
int amgr_hier_shares_transfer(const amgr_hier* a, const amgr_hier* b, int level);

/* ---- synthetic problem sequences on the device ---------- */
enum {
    AMGR_PROBLEM_POISSON = 0,   /* 7-point Laplacian + shift s_k (config C1)     */
    AMGR_PROBLEM_BLOB = 1,      /* moving high-contrast blob kappa (config C2)  */
    AMGR_PROBLEM_DAMBREAK = 2,  /* 1000:1 collapsing water column (C3/C4)       */
    AMGR_PROBLEM_CONVDIFF = 3   /* upwind convection-diffusion (C5)             */
};
/* Pattern of the g^3 7-point operator: int32 CSR written to device buffers
 * (row_ptr n+1, col nnz).  nnz = 7g^3 - 6g^2. */
int64_t amgr_problem_nnz(int64_t g);
amgr_status amgr_problem_pattern(amgr_ctx* ctx, int64_t g, int32_t* row_ptr, int32_t* col);
/* Values of step k of `kind` (same CSR order) into a device buffer. */
amgr_status amgr_problem_values(amgr_ctx* ctx, int kind, int64_t g, int64_t k, int64_t nsteps,
                                double* values);
/* RHS f_i ~ U(0.1, 1.0) from std::mt19937_64(seed) (diffusion.cpp:38-41),
 * generated on the host and written to `location`. */
amgr_status amgr_problem_rhs(amgr_ctx* ctx, int64_t n, uint64_t seed, double* out, int location);

/* ---- measurement hooks ----------------------------------------------------- */
/* Kernel probe: when enabled, every launch of the named kernel family
 * ("rap", "vcycle_down", "vcycle_up", "spmv", ...) is bracketed by CUDA events
 * on the launching stream; amgr_probe_read returns launches, total device ms
 * and the algorithmic bytes those launches moved. */
amgr_status amgr_probe_enable(amgr_ctx* ctx, const char* family);
amgr_status amgr_probe_read(amgr_ctx* ctx, int64_t* launches, double* ms, double* bytes);
/* Stream-ordered device -> host copy on the context stream (synchronous). */
amgr_status amgr_copy_to_host(amgr_ctx* ctx, void* host, const void* device, size_t bytes);

/* Number of kernel launches the library issued on this context so far. */
int64_t amgr_launch_count(const amgr_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* AMGR_H */

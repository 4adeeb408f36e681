// Device-side full AMG setup (hierarchy.cpp:45-105): strength graph, exact
// parallel replay of the sequential greedy aggregation, P/R, and the symbolic
// Galerkin plan that partial rebuilds reuse.
#pragma once

#include "kernels.cuh"

namespace amgr {

struct GraphDev {
    int64_t n = 0, m = 0;
    DevArray<int> ptr, adj;
};

// Coded column stream of a pattern (row-pass layout): when the
// pattern's column offsets j - i take few distinct values (a stencil: 7 on the
// 7-point level 0, ~2K on its first aggregation level), the row passes read a
// 1- or 2-byte code per entry instead of the int32 column, col = i + dict[code].
// Columns, their order and the arithmetic are unchanged.
struct ColCode {
    int mode = 0;  // 0 raw, 1 uint8, 2 uint16
    int ndict = 0;
    DevArray<uint8_t> c8;
    DevArray<uint16_t> c16;
    DevArray<int> dict;
};
void encode_columns(Ctx& c, int64_t n, int64_t nnz, const int* rp, const int* col, ColCode& out,
                    bool narrow16 = false);

// First row (ascending) whose diagonal is missing or zero, or -1.
// (strength_graph, coarsening.cpp:19-32; build_smoother, smoother.cpp:12-28)
int64_t first_bad_diag(Ctx& c, const CsrView& A, const int* dpos);

// Symmetrised strong-coupling graph, adjacency sorted and unique
// (coarsening.cpp:11-75).  eps2 = eps*eps as the reference computes it.
void strength_graph(Ctx& c, const CsrView& A, const int* dpos, double eps2, GraphDev& g);

// Two-pass greedy aggregation (coarsening.cpp:77-120) replayed exactly in
// parallel rounds.  Returns n_coarse; agg has g.n entries.
int64_t aggregate(Ctx& c, const GraphDev& g, DevArray<int>& agg, int64_t* rounds);

// R = P^T: member lists per aggregate, ascending fine index (csr.cpp:93-113).
void members(Ctx& c, int64_t nf, int64_t nc, const int* agg, DevArray<int>& mptr, DevArray<int>& midx);

// Symbolic RAP + numeric plan.  Coarse pattern (sorted columns, structural,
// csr.cpp:115-143) and for every coarse entry its contributing fine entries in
// the reference's summation order with row-break flags.
struct RapSymbolic {
    int64_t nnz_c = 0;
    DevArray<int> rp, col;       // coarse pattern
    DevArray<int> cptr, contrib; // plan
};
void rap_symbolic(Ctx& c, const CsrView& A, const int* agg, int64_t nc, RapSymbolic& out);

// Member-row Galerkin plan (k_rap_rows): thread per coarse
// row I streams its member fine rows (R order, ascending) contiguously and
// scatters each entry into the local slot of its coarse column.  Per fine
// entry (CSR position of the row, i.e. aligned with the values) a 16-bit code
// lists the row's entries in accumulation order — grouped by slot, ascending
// k inside a group (the inner bracket of spmm(A, P), csr.cpp:145-184):
//   bits 0-4  offset of the entry inside its fine row (rows <= 32 entries)
//   bit  5    last entry of its slot group: commit the group's partial sum
//   bit  6    the entry is the row's diagonal (fused Jacobi, smoother.cpp:8-32)
//   bits 7-15 slot = position of the coarse column in coarse row I (<= 511)
struct RowPlan {
    bool ok = false;
    int dmax = 0;   // widest coarse row
    int maxlen = 0; // longest fine row
    DevArray<int> mrp;        // [nf] R order: start of member row midx[j]
    DevArray<uint8_t> mlen;   // [nf] R order: its length
    DevArray<uint16_t> code;  // [nnz_f]
};
// Builds the plan when the level fits (rows <= 32 entries, coarse rows <= 511);
// plan.ok tells.  crp/ccol: the coarse pattern from rap_symbolic.
void rap_rows_plan(Ctx& c, const CsrView& A, const int* agg, const int* midx, int64_t nc, const int* crp,
                   const int* ccol, RowPlan& plan);

// Warp-group Galerkin plan (k_rap_grp).  Coarse rows are
// cut into groups of consecutive rows with <= 255 contributions (= entries
// of their member rows) and <= 64 member rows; a warp gathers a group's
// contributions into shared memory in the plan's order (cptr/contrib, the
// reference's bracket, csr.cpp:145-194) and each lane sums one of 32
// contiguous runs of coarse entries, balanced by contribution count.  Per contribution the plan keeps 2 bytes
// (offset inside its member row, the member's number in the group, a bit
// for the first contribution of a coarse entry, the bracket bit), per member
// row its CSR start and diagonal offset (fused damped-Jacobi rebuild,
// smoother.cpp:8-32).
struct GrpPlan {
    bool ok = false;
    int64_t ngroups = 0;
    DevArray<int4> desc;      // [ngroups + 1] {first coarse row, first member (R order), first coarse entry, first contribution}
    DevArray<int> mstart;     // [nf] R order: first CSR position of member row midx[j]
    DevArray<uint8_t> mdoff;  // [nf] diagonal offset inside it (255: no diagonal)
    DevArray<uint16_t> code;  // [nnz_f + 8] row offset | member << 8 | entry start << 14 | bracket end << 15
    DevArray<uint16_t> lanes; // [ngroups * 32] per lane: first contribution | first entry << 8 (balanced split)
};
// Builds the plan when the level fits (plan.ok tells).  mptr/midx: R;
// dpos: diagonal CSR position per fine row (-1: none); crp: coarse row
// pointers; cptr/contrib: the level's RapPlan (global, or a rank's local
// plan: dist.cu).
void rap_grp_plan(Ctx& c, const CsrView& A, const int* mptr, const int* midx, const int* dpos, int64_t nc,
                  const int* crp, int64_t nnz_c, const int* cptr, const int* contrib, GrpPlan& plan);

// ---- smoothed aggregation (extension) ----
// Device SpGEMM C = A B: structural pattern of C (sorted columns) and the
// numeric plan (per output entry, its (a index, b index) products in the
// reference spmm's accumulation order).
struct SpgPlan {
    int64_t nnz = 0, products = 0;
    DevArray<int> rp, col;          // pattern of C (rows = A's rows)
    DevArray<int> optr, pa, pb;     // plan
};
void spgemm_symbolic(Ctx& c, const CsrView& A, const int* brp, const int* bcol, int64_t bcols, SpgPlan& out,
                     const char* what);
void spgemm_numeric(Ctx& c, const SpgPlan& p, const double* a, const double* b, double* out);
// P_tent as CSR (row i: column agg_i, value 1.0; coarsening.cpp:122-132)
void tentative_csr(Ctx& c, int64_t n, const int* agg, DevArray<int>& rp, DevArray<int>& col, DevArray<double>& val);
// in place on the values of A P_tent: v = (J == agg_i) - (w * (1/a_ii)) * v; first bad row -> *bad
void sa_prolongator_values(Ctx& c, int64_t n, const int* rp, const int* col, double* v, const int* agg,
                           const int* dpos, const double* aval, double w, int* bad);
// T = M^T (sorted columns, values carried)
void transpose_csr(Ctx& c, int64_t nrows, int64_t ncols, int64_t nnz, const int* rp, const int* col,
                   const double* val, DevArray<int>& trp, DevArray<int>& tcol, DevArray<double>& tval);

}  // namespace amgr

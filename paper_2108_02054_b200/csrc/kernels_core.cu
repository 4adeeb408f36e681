// Hot-path kernels of libamgr_b200.so, hand-written for sm_100a.
//
//  * k_rowpass<Op>: thread-per-row CSR pass with warp-cooperative staging of
//    the warp's contiguous nnz range through shared memory (coalesced 8-byte
//    loads, any row-length distribution, no padding), followed by a strictly
//    sequential per-row accumulation in column order — the reference's spmv
//    order (proj/src/csr.cpp:79-84) — so results are bit-identical.  The
//    Op supplies the on-the-fly operand x_j and the row epilogue, which is how
//    the V-cycle legs fuse smoothing, residual and prolongation into a single
//    pass over A_i, and how the Krylov SpMVs fuse their dot products.
//  * rap_numeric: numeric Galerkin product on the cached contribution plan.
//  * jacobi/spai0 rebuild, restriction, dense LU factor/solve.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kernels.cuh"
#include "reduce.cuh"

namespace amgr {

namespace {

constexpr int RP_WARPS = 4;                 // warps per block
constexpr int RP_BLOCK = RP_WARPS * 32;
constexpr int RP_CH = 256;                  // entries per TMA chunk (multiple of 16)
constexpr int RP_CH_W12 = 384;              // chunk of the 8..12-entries-per-row variant
constexpr int RP_BATCH = 8;                 // operand gathers in flight per thread
constexpr int RP_BLOCKS_PER_SM = 8;         // persistent grid: 32 warps per SM

// operand gathers per stored entry of a row-pass Op (default 1)
template <class Op, class = void>
struct gathers_of {
    static constexpr int v = 1;
};
template <class Op>
struct gathers_of<Op, std::void_t<decltype(Op::GATHERS)>> {
    static constexpr int v = Op::GATHERS;
};

// x_j of a batch of columns.  Ops with several operands per entry (GATHERS
// > 1) split x into gather + combine so every load of the batch is issued
// before the first arithmetic use: left fused, ptxas interleaved them and
// kept only ~2 entries' loads in flight (coded level-0 OpDownP 346 -> 275 us).
template <int NB, class Op>
__device__ __forceinline__ void gather_batch(const Op& op, const int (&cj)[NB], double (&xv)[NB]) {
    if constexpr (gathers_of<Op>::v > 1) {
        typename Op::G gv[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t) gv[t] = op.gather(cj[t]);
#pragma unroll
        for (int t = 0; t < NB; ++t) xv[t] = op.combine(gv[t]);
    } else {
#pragma unroll
        for (int t = 0; t < NB; ++t) xv[t] = op.x(cj[t]);
    }
}

// ---- TMA 1-D bulk copy + mbarrier helpers (sm_90+/sm_100a PTX) ----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Interleaved TMA chunk stream.  Warp w of W processes the 32-row groups
// w, w+W, w+2W, ... so all warps sweep the matrix as one narrow band (the
// +-g^2 z-neighbour gathers stay L2-resident).  A group's 16-byte-aligned nnz
// range (values + int32 columns) is cut into CH-entry chunks; the chunk
// sequence of the warp is double-buffered in shared memory by TMA 1-D bulk
// copies completing on per-stage mbarriers, always one chunk ahead of the
// consumer (the next chunk of the same group, or the first chunk of the next
// group).  Row pointers and epilogue operands of the next group are prefetched
// into registers.  Threads own rows and accumulate strictly in column order
// (csr.cpp:79-84), gathering up to RP_BATCH operands at a time.
// GATHER: 0 = RP_BATCH predicated gathers (level 0's 7-entry rows);
//         8 / 12 = that many unpredicated gathers (coarser levels: 8 for
//         > 12 nnz/row, 12 for 8..12 nnz/row; measured per level)
// CT: column stream element.  int = raw columns; uint8_t / uint16_t = coded
// columns (encode_columns), col = row + dict[code], the uint8 dictionary
// staged in shared memory.  Chunk ranges are aligned to 16 bytes of CT.
template <class Op, int CH, int GATHER, class CT>
__global__ void __launch_bounds__(RP_BLOCK) k_rowpass(CsrView A, Op op, Gate g, DotSink sink) {
    pdl_enter();
    if (gated_off(g)) return;
    constexpr int ND = Op::NDOT > 0 ? Op::NDOT : 1;
    constexpr bool CODED = sizeof(CT) < 4;
    constexpr int ALN = 16 / static_cast<int>(sizeof(CT));  // entries per 16 bytes of column stream
    extern __shared__ __align__(128) unsigned char rp_smem[];
    auto s_val = reinterpret_cast<double(*)[2][CH]>(rp_smem);
    auto s_col = reinterpret_cast<CT(*)[2][CH]>(rp_smem + sizeof(double) * RP_WARPS * 2 * CH);
    auto s_bar = reinterpret_cast<uint64_t(*)[2]>(rp_smem + sizeof(double) * RP_WARPS * 2 * CH +
                                                  sizeof(CT) * RP_WARPS * 2 * CH);
    int* s_dict = reinterpret_cast<int*>(rp_smem + sizeof(double) * RP_WARPS * 2 * CH +
                                         sizeof(CT) * RP_WARPS * 2 * CH + sizeof(uint64_t) * RP_WARPS * 2);
    const CT* colstream = CODED ? static_cast<const CT*>(A.code) : reinterpret_cast<const CT*>(A.col);
    if constexpr (sizeof(CT) == 1) {
        for (int t = threadIdx.x; t < A.ndict; t += blockDim.x) s_dict[t] = __ldg(A.dict + t);
        __syncthreads();
    }
    // value ranges are clamped to the 4-aligned end of the value array (a
    // caller's adopted buffer has no more slack than that)
    const int nnz4 = static_cast<int>((A.nnz + 3) & ~int64_t{3});
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = static_cast<int>(A.n);
    const int ngroups = (n + 31) >> 5;
    const int W = gridDim.x * RP_WARPS;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;

    int G = blockIdx.x * RP_WARPS + w;
    if (G < ngroups) {
        uint64_t* bar = s_bar[w];
        if (lane == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            mbar_fence_init();
        }
        __syncwarp();
        auto issue = [&](int base, int end, int st) {  // [base, min(base+CH, end)), base/end ALN-aligned
            const int cnt = min(CH, end - base);
            if (lane == 0) {
                fence_proxy_async();
                const int vcnt = CODED ? min(cnt, nnz4 - base) : cnt;
                const uint32_t bv = static_cast<uint32_t>(vcnt) * 8u,
                               bc = static_cast<uint32_t>(cnt) * static_cast<uint32_t>(sizeof(CT));
                mbar_expect_tx(&bar[st], bv + bc);
                tma_load_1d(&s_val[w][st][0], A.val + base, bv, &bar[st]);
                tma_load_1d(&s_col[w][st][0], colstream + base, bc, &bar[st]);
            }
        };
        auto colof = [&](int row, CT code) -> int {
            if constexpr (sizeof(CT) == 1) return row + s_dict[code];
            else if constexpr (sizeof(CT) == 2) return row + __ldg(A.dict + code);
            else return code;
        };
        auto rows_of = [&](int grp, int& rs, int& re) {
            const int row = grp * 32 + lane;
            const int last = min(grp * 32 + 32, n);
            rs = row < n ? __ldg(A.rp + row) : __ldg(A.rp + last);
            re = row < n ? __ldg(A.rp + row + 1) : rs;
        };
        int rs, re, nrs = 0, nre = 0;
        rows_of(G, rs, re);
        typename Op::Row rw, nrw;
        if (G * 32 + lane < n) rw = op.load(G * 32 + lane);
        int NG = G + W;
        if (NG < ngroups) {
            rows_of(NG, nrs, nre);
            if (NG * 32 + lane < n) nrw = op.load(NG * 32 + lane);
        }
        // group range (aligned) of the current group
        int gs = __shfl_sync(0xffffffffu, rs, 0), ge = __shfl_sync(0xffffffffu, re, 31);
        int ab = gs & ~(ALN - 1), ae = (ge + ALN - 1) & ~(ALN - 1);
        int st = 0;
        uint32_t phase = 0;
        int cb = ab;                     // base of the chunk to consume next
        bool ready = false;              // chunk cb is in flight in stage st
        if (ae > ab) {
            issue(cb, ae, st);
            ready = true;
        }
        double sum = 0.0;
        while (G < ngroups) {
            const int row = G * 32 + lane;
            // ---- consume chunk cb (if the group has entries) ----
            bool group_done;
            if (ae > ab) {
                if (!ready) issue(cb, ae, st);
                // prefetch the following chunk into the other stage
                int pb = -1, pe = 0;
                if (cb + CH < ae) {
                    pb = cb + CH;
                    pe = ae;
                } else if (NG < ngroups) {
                    const int ngs = __shfl_sync(0xffffffffu, nrs, 0), nge = __shfl_sync(0xffffffffu, nre, 31);
                    if (nge > ngs) {
                        pb = ngs & ~(ALN - 1);
                        pe = (nge + ALN - 1) & ~(ALN - 1);
                    }
                }
                if (pb >= 0) issue(pb, pe, st ^ 1);
                mbar_wait(&bar[st], (phase >> st) & 1u);
                phase ^= (1u << st);
                // row-parallel: lane l gathers the k-th operand of 32 consecutive rows
                // (contiguous for stencil-like matrices), RP_BATCH at a time, then
                // accumulates them strictly in column order
                {
                    int a = max(rs, cb);
                    const int b = min(re, cb + CH);
                    constexpr bool SPEC = GATHER > 0;
                    constexpr int NB = SPEC ? GATHER : RP_BATCH;
                    while (a < b) {
                        const int cnt = min(NB, b - a);
                        const int k = a - cb;
                        double xv[NB];
                        if constexpr (SPEC) {
                            // unpredicated gathers (lanes past the row end re-read the
                            // first entry's operand, a cache hit): with predicated loads
                            // the scheduler interleaves them with the DMULs and only ~2
                            // are outstanding (measured on levels >= 1)
                            int cj[NB];
#pragma unroll
                            for (int t = 0; t < NB; ++t) cj[t] = colof(row, s_col[w][st][k + (t < cnt ? t : 0)]);
                            gather_batch<NB>(op, cj, xv);
                        } else if constexpr (CODED) {
                            // decode the batch first (unpredicated shared-memory reads),
                            // then the gathers (all issued before the first use)
                            int cj[NB];
#pragma unroll
                            for (int t = 0; t < NB; ++t) cj[t] = colof(row, s_col[w][st][k + (t < cnt ? t : 0)]);
                            gather_batch<NB>(op, cj, xv);
                        } else {
#pragma unroll
                            for (int t = 0; t < NB; ++t) xv[t] = t < cnt ? op.x(s_col[w][st][k + t]) : 0.0;
                        }
#pragma unroll
                        for (int t = 0; t < NB; ++t)
                            if (t < cnt) sum = dadd(sum, dmul(s_val[w][st][k + t], xv[t]));
                        a += cnt;
                    }
                }
                __syncwarp();
                group_done = cb + CH >= ae;
                st ^= 1;
                ready = pb >= 0;
                cb = pb;
            } else {
                group_done = true;
            }
            if (!group_done) continue;
            // ---- epilogue of group G and rotation to G+W ----
            if (row < n) op.finish(row, sum, rw, dots);
            sum = 0.0;
            G = NG;
            rs = nrs;
            re = nre;
            rw = nrw;
            if (G >= ngroups) break;
            gs = __shfl_sync(0xffffffffu, rs, 0);
            ge = __shfl_sync(0xffffffffu, re, 31);
            ab = gs & ~(ALN - 1);
            ae = (ge + ALN - 1) & ~(ALN - 1);
            if (!ready || cb != ab) {  // first chunk of the new group not prefetched
                cb = ab;
                ready = false;
            }
            NG = G + W;
            if (NG < ngroups) {
                rows_of(NG, nrs, nre);
                if (NG * 32 + lane < n) nrw = op.load(NG * 32 + lane);
            }
        }
    }
    if constexpr (Op::NDOT > 0) block_dots<Op::NDOT>(dots, sink);
}

// ---- k_rowpass_lag: two dependent row passes over the same matrix in ONE sweep
// Op1 (a smoothing sweep producing x) and Op2 (an SpMV over that x) run in the
// same persistent kernel: warp w processes, round by round, Op1 on its group
// of round k and Op2 on its group of round k - LAG.  Op2 of a group gathers
// x_j of rows up to `dgroups` groups away, so before it starts, lane 0 waits
// (acquire) until every warp has published (release) Op1 of all rounds that
// cover them.  The matrix rows of a group are thus streamed from DRAM once for
// Op1 and re-read from L2 by Op2 LAG rounds later (one round = W groups =
// ~9.5 MB of level-0 entries), saving one DRAM sweep of A per fused pair.
// Rows, the group -> warp map, the grid and the per-thread dot order are those
// of the separate passes, so results (and the blocked dots) are bit-identical.
// All blocks must be co-resident (persistent grid at the kernel's occupancy).
constexpr int LAG_SLOTS = 64;

// Round counters: relaxed polling (an acquire would invalidate the SM's L1 on
// every poll and cost the gathers of all warps their L1 hits) against
// release increments.  When a reader sees round r complete, the rows of
// every round <= r were performed in L2 before the counters moved; the
// completed region is a prefix of whole 32-row groups (256-byte aligned), so
// no L1 line holding a row of it can have been filled before the row was
// final (rows are only gathered inside completed prefixes) — the Op2 gathers
// may go through L1.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <class Op1, class Op2, class CT>
__global__ void __launch_bounds__(RP_BLOCK, RP_BLOCKS_PER_SM) k_rowpass_lag(CsrView A, Op1 op1, Op2 op2, Gate g, DotSink sink,
                                                          int* __restrict__ done, int dgroups, int LAG_ROUNDS) {
    pdl_enter();
    if (gated_off(g)) return;
    constexpr int CH = RP_CH;
    constexpr int ND = Op2::NDOT > 0 ? Op2::NDOT : 1;
    constexpr bool CODED = sizeof(CT) < 4;
    constexpr int ALN = 16 / static_cast<int>(sizeof(CT));
    extern __shared__ __align__(128) unsigned char rp_smem[];
    auto s_val = reinterpret_cast<double(*)[2][CH]>(rp_smem);
    auto s_col = reinterpret_cast<CT(*)[2][CH]>(rp_smem + sizeof(double) * RP_WARPS * 2 * CH);
    auto s_bar = reinterpret_cast<uint64_t(*)[2]>(rp_smem + sizeof(double) * RP_WARPS * 2 * CH +
                                                  sizeof(CT) * RP_WARPS * 2 * CH);
    int* s_dict = reinterpret_cast<int*>(rp_smem + sizeof(double) * RP_WARPS * 2 * CH +
                                         sizeof(CT) * RP_WARPS * 2 * CH + sizeof(uint64_t) * RP_WARPS * 2);
    const CT* colstream = CODED ? static_cast<const CT*>(A.code) : reinterpret_cast<const CT*>(A.col);
    if constexpr (sizeof(CT) == 1) {
        for (int t = threadIdx.x; t < A.ndict; t += blockDim.x) s_dict[t] = __ldg(A.dict + t);
        __syncthreads();
    }
    const int nnz4 = static_cast<int>((A.nnz + 3) & ~int64_t{3});
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = static_cast<int>(A.n);
    const int ngroups = (n + 31) >> 5;
    const int W = gridDim.x * RP_WARPS;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;
    const int G0 = blockIdx.x * RP_WARPS + w;
    if (G0 < ngroups) {
        uint64_t* bar = s_bar[w];
        if (lane == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            mbar_fence_init();
        }
        __syncwarp();
        auto issue = [&](int base, int end, int st) {
            const int cnt = min(CH, end - base);
            if (lane == 0) {
                fence_proxy_async();
                const int vcnt = CODED ? min(cnt, nnz4 - base) : cnt;
                const uint32_t bv = static_cast<uint32_t>(vcnt) * 8u,
                               bc = static_cast<uint32_t>(cnt) * static_cast<uint32_t>(sizeof(CT));
                mbar_expect_tx(&bar[st], bv + bc);
                tma_load_1d(&s_val[w][st][0], A.val + base, bv, &bar[st]);
                tma_load_1d(&s_col[w][st][0], colstream + base, bc, &bar[st]);
            }
        };
        auto colof = [&](int row, CT code) -> int {
            if constexpr (sizeof(CT) == 1) return row + s_dict[code];
            else if constexpr (sizeof(CT) == 2) return row + __ldg(A.dict + code);
            else return code;
        };
        // aligned nnz range of a group (warp-uniform)
        auto range_of = [&](int grp, int& ab, int& ae) {
            const int row = grp * 32 + lane;
            const int last = min(grp * 32 + 32, n);
            const int rs = row < n ? __ldg(A.rp + row) : __ldg(A.rp + last);
            const int re = row < n ? __ldg(A.rp + row + 1) : rs;
            const int gs = __shfl_sync(0xffffffffu, rs, 0), ge = __shfl_sync(0xffffffffu, re, 31);
            ab = gs & ~(ALN - 1);
            ae = (ge + ALN - 1) & ~(ALN - 1);
        };
        const int nround = (ngroups - G0 + W - 1) / W;
        const int nitem = 2 * (nround + LAG_ROUNDS);
        // item t: round k = t / 2; t even: Op1 on round k, t odd: Op2 on round k - LAG
        auto valid = [&](int t) {
            const int k = t >> 1;
            return (t & 1) == 0 ? k < nround : (k >= LAG_ROUNDS && k - LAG_ROUNDS < nround);
        };
        auto group_of = [&](int t) { return G0 + ((t & 1) == 0 ? (t >> 1) : (t >> 1) - LAG_ROUNDS) * W; };
        auto next_valid = [&](int t) {
            for (++t; t < nitem; ++t)
                if (valid(t)) return t;
            return -1;
        };
        int t = 0;  // item 0 (Op1, round 0) is always valid
        int ab, ae;
        range_of(G0, ab, ae);
        int st = 0;
        uint32_t phase = 0;
        bool ready = false;
        if (ae > ab) {
            issue(ab, ae, st);
            ready = true;
        }
        int ok_round = -1;  // rounds whose Op1 is known complete on every warp
        while (t >= 0) {
            const int G = group_of(t);
            const bool second = (t & 1) != 0;
            const int row = G * 32 + lane;
            const int rs = row < n ? __ldg(A.rp + row) : 0, re = row < n ? __ldg(A.rp + row + 1) : 0;
            typename Op1::Row rw1;
            typename Op2::Row rw2;
            if (row < n) {
                if (second) rw2 = op2.load(row);
                else rw1 = op1.load(row);
            }
            const int tn = next_valid(t);
            int nab = 0, nae = 0;
            if (tn >= 0) range_of(group_of(tn), nab, nae);
            if (second) {
                // every group Op2 of G gathers from must have finished Op1
                // (round counters are split over LAG_SLOTS addresses so the
                // release atomics of a round do not serialise on one line)
                const int need = min(G + dgroups, ngroups - 1) / W;
                while (ok_round < need) {
                    const int r = ok_round + 1;
                    const int act = min(W, ngroups - r * W);  // warps with a group in round r
                    const int s0 = lane, s1 = lane + 32;
                    const int e0 = act > s0 ? (act - 1 - s0) / LAG_SLOTS + 1 : 0;
                    const int e1 = act > s1 ? (act - 1 - s1) / LAG_SLOTS + 1 : 0;
                    const int* d = done + static_cast<int64_t>(r) * LAG_SLOTS;
                    while (!__all_sync(0xffffffffu, ld_relaxed(d + s0) >= e0 && ld_relaxed(d + s1) >= e1))
                        __nanosleep(32);
                    ok_round = r;
                }
            }
            int cb = ab;
            // the chunk stream of this item, specialised per operator (one
            // clean loop per Op instead of a per-batch branch)
            auto run = [&](const auto& op, const auto& rw) {
                double sum = 0.0;
                while (ae > ab) {
                    if (!ready) issue(cb, ae, st);
                    int pb = -1, pe = 0;
                    if (cb + CH < ae) {
                        pb = cb + CH;
                        pe = ae;
                    } else if (tn >= 0 && nae > nab) {
                        pb = nab;
                        pe = nae;
                    }
                    if (pb >= 0) issue(pb, pe, st ^ 1);
                    mbar_wait(&bar[st], (phase >> st) & 1u);
                    phase ^= (1u << st);
                    {
                        int a = max(rs, cb);
                        const int b = min(re, cb + CH);
                        while (a < b) {
                            const int cnt = min(RP_BATCH, b - a);
                            const int k = a - cb;
                            double xv[RP_BATCH];
                            int cj[RP_BATCH];
#pragma unroll
                            for (int q = 0; q < RP_BATCH; ++q) cj[q] = colof(row, s_col[w][st][k + (q < cnt ? q : 0)]);
                            gather_batch<RP_BATCH>(op, cj, xv);
#pragma unroll
                            for (int q = 0; q < RP_BATCH; ++q)
                                if (q < cnt) sum = dadd(sum, dmul(s_val[w][st][k + q], xv[q]));
                            a += cnt;
                        }
                    }
                    __syncwarp();
                    st ^= 1;
                    const bool last = cb + CH >= ae;
                    ready = pb >= 0;
                    cb = pb;
                    if (last) break;
                }
                if (row < n) op.finish(row, sum, rw, dots);
            };
            if (second)
                run(op2, rw2);
            else
                run(op1, rw1);
            if (!second) {
                __syncwarp();  // the warp's rows of x, then one release increment
                if (lane == 0) red_release_add(done + static_cast<int64_t>(t >> 1) * LAG_SLOTS + (G0 & (LAG_SLOTS - 1)), 1);
            }
            // rotate to the next item; its first chunk was prefetched if the
            // current item had entries (else it is issued at the loop top)
            if (tn < 0) break;
            if (!ready || cb != nab) {
                ready = false;
            }
            ab = nab;
            ae = nae;
            t = tn;
        }
    }
    if constexpr (Op2::NDOT > 0) block_dots<Op2::NDOT>(dots, sink);
}

// ---- row-pass operators ----------------------------------------------------
struct NoRow {};
struct Row1 {
    double a;
};
struct Row3 {
    double f, w, x;
};

struct OpSpmv {
    static constexpr int NDOT = 0;
    using Row = NoRow;
    const double* xv;
    double* y;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int) const { return {}; }
    __device__ void finish(int i, double s, const Row&, double*) const { y[i] = s; }
};

struct OpResidual {
    static constexpr int NDOT = 0;
    using Row = Row1;
    const double* f;
    const double* xv;
    double* r;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(f + i)}; }
    __device__ void finish(int i, double s, const Row& q, double*) const { r[i] = dsub(q.a, s); }
};

// V-cycle down leg (hierarchy.cpp:165-170): the first pre-smoothing sweep from
// u = 0 gives u = 0 + (om*w)*(f - A*0) = u0, which the producer of f (the
// restriction, or premul on level 0) has already written; this pass forms the
// residual r = f - A u0.
struct OpDown {
    static constexpr int NDOT = 0;
    using Row = Row1;
    const double* f;
    const double* u0;
    double* r;
    __device__ double x(int j) const { return __ldg(u0 + j); }
    __device__ Row load(int i) const { return {__ldg(f + i)}; }
    __device__ void finish(int i, double s, const Row& q, double*) const { r[i] = dsub(q.a, s); }
};

// down leg at the V-cycle's top level with the first pre-smoothing iterate
// folded in: u0_j = 0 + (om*w_j)*f_j is formed per gathered column (the same
// operations as k_premul), so the premul pass disappears; the DRAM bytes are
// OpDown's (w replaces u0 as the gathered vector).
struct OpDownP {
    static constexpr int NDOT = 0;
    static constexpr int GATHERS = 2;  // w_j and f_j per entry
    using Row = Row1;
    const double* f;
    const double* w;
    double om;
    double* r;
    struct G {
        double w, f;
    };
    __device__ G gather(int j) const { return {__ldg(w + j), __ldg(f + j)}; }
    __device__ double combine(const G& g) const { return dadd(0.0, dmul(dmul(om, g.w), g.f)); }
    __device__ double x(int j) const { return combine(gather(j)); }
    __device__ Row load(int i) const { return {__ldg(f + i)}; }
    __device__ void finish(int i, double s, const Row& q, double*) const { r[i] = dsub(q.a, s); }
};

// one damped sweep (smoother.cpp:42-47): out_i = x_i + (om*w_i)*(f_i - (A x)_i)
struct OpSmooth {
    static constexpr int NDOT = 0;
    using Row = Row3;
    const double* f;
    const double* w;
    double om;
    const double* u;
    double* out;
    __device__ double x(int j) const { return __ldg(u + j); }
    __device__ Row load(int i) const { return {__ldg(f + i), __ldg(w + i), __ldg(u + i)}; }
    __device__ void finish(int i, double s, const Row& q, double*) const {
        out[i] = dadd(q.x, dmul(dmul(om, q.w), dsub(q.f, s)));
    }
};

// smoothed aggregation (extension): restriction f_c = R r as a row pass over
// R (o_vcycle: spmv(R, r)), with the coarse level's first iterate
// u0_c = 0 + (om*w_c)*f_c in the epilogue as k_restrict does
struct OpRestrictG {
    static constexpr int NDOT = 0;
    using Row = NoRow;
    const double* r;
    double* fc;
    const double* wc;
    double om;
    double* u0c;
    __device__ double x(int j) const { return __ldg(r + j); }
    __device__ Row load(int) const { return {}; }
    __device__ void finish(int i, double s, const Row&, double*) const {
        fc[i] = s;
        if (u0c) u0c[i] = dadd(0.0, dmul(dmul(om, wc[i]), s));
    }
};
// ... and prolongation out = u + P e (o_vcycle: r = spmv(P, e); u += r)
struct OpProlongG {
    static constexpr int NDOT = 0;
    using Row = Row1;
    const double* e;
    const double* u;
    double* out;
    __device__ double x(int j) const { return __ldg(e + j); }
    __device__ Row load(int i) const { return {__ldg(u + i)}; }
    __device__ void finish(int i, double s, const Row& q, double*) const { out[i] = dadd(q.a, s); }
};

struct OpSpmvDot {
    static constexpr int NDOT = 1;
    using Row = Row1;
    const double* xv;
    double* y;
    const double* a;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(a + i)}; }
    __device__ void finish(int i, double s, const Row& q, double* d) const {
        y[i] = s;
        d[0] = dadd(d[0], dmul(q.a, s));
    }
};

struct OpSpmvDot2 {
    static constexpr int NDOT = 2;
    using Row = Row1;
    const double* xv;
    double* y;
    const double* b;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(b + i)}; }
    __device__ void finish(int i, double s, const Row& q, double* d) const {
        y[i] = s;
        d[0] = dadd(d[0], dmul(s, q.a));
        d[1] = dadd(d[1], dmul(s, s));
    }
};

// Op2 of k_rowpass_lag: x was written by other SMs inside the same kernel;
// gathered only from completed 256-byte-aligned prefixes (see ld_relaxed)
struct OpSpmvDotL2 {
    static constexpr int NDOT = 1;
    using Row = Row1;
    const double* xv;
    double* y;
    const double* a;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(a + i)}; }
    __device__ void finish(int i, double s, const Row& q, double* d) const {
        y[i] = s;
        d[0] = dadd(d[0], dmul(q.a, s));
    }
};
struct OpSpmvDot2L2 {
    static constexpr int NDOT = 2;
    using Row = Row1;
    const double* xv;
    double* y;
    const double* b;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(b + i)}; }
    __device__ void finish(int i, double s, const Row& q, double* d) const {
        y[i] = s;
        d[0] = dadd(d[0], dmul(s, q.a));
        d[1] = dadd(d[1], dmul(s, s));
    }
};

struct OpResidNorm {
    static constexpr int NDOT = 1;
    using Row = Row1;
    const double* f;
    const double* xv;
    double* r;
    double* r2;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(f + i)}; }
    __device__ void finish(int i, double s, const Row& q, double* d) const {
        const double t = dsub(q.a, s);
        if (r) r[i] = t;
        if (r2) r2[i] = t;
        d[0] = dadd(d[0], dmul(t, t));
    }
};

// ---- Chebyshev smoother + power iteration (extension, oracle/amg_oracle.c) --
// power step: y = D^-1 A x (w = 1/a_ii), out[0] = y . y
struct OpPower {
    static constexpr int NDOT = 1;
    using Row = Row1;
    const double* xv;
    const double* w;
    double* y;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(w + i)}; }
    __device__ void finish(int i, double s, const Row& q, double* d) const {
        const double t = dmul(q.a, s);
        y[i] = t;
        d[0] = dadd(d[0], dmul(t, t));
    }
};

struct Row4 {
    double f, w, x, d;
};

// first Chebyshev step: r = w*(f - A x); d = r / theta
struct OpChebStart {
    static constexpr int NDOT = 0;
    using Row = Row3;
    const double* f;
    const double* w;
    const double* xv;
    const double* coef;  // coef[0] = theta
    double* dout;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ Row load(int i) const { return {__ldg(f + i), __ldg(w + i), 0.0}; }
    __device__ void finish(int i, double s, const Row& q, double*) const {
        const double r = dmul(q.w, dsub(q.f, s));
        dout[i] = __ddiv_rn(r, coef[0]);
    }
};

// Chebyshev step k (>= 1): x' = x + d; r = w*(f - A x'); d' = c1*d + c2*r
struct OpChebStep {
    static constexpr int NDOT = 0;
    static constexpr int GATHERS = 2;  // x_j and d_j per entry
    using Row = Row4;
    const double* f;
    const double* w;
    const double* xv;
    const double* dv;
    const double* coef;  // c1 = coef[2k-1], c2 = coef[2k]
    int k;
    double* xout;
    double* dout;
    struct G {
        double x, d;
    };
    __device__ G gather(int j) const { return {__ldg(xv + j), __ldg(dv + j)}; }
    __device__ double combine(const G& g) const { return dadd(g.x, g.d); }
    __device__ double x(int j) const { return combine(gather(j)); }
    __device__ Row load(int i) const { return {__ldg(f + i), __ldg(w + i), __ldg(xv + i), __ldg(dv + i)}; }
    __device__ void finish(int i, double s, const Row& q, double*) const {
        const double xn = dadd(q.x, q.d);
        const double r = dmul(q.w, dsub(q.f, s));
        xout[i] = xn;
        dout[i] = dadd(dmul(coef[2 * k - 1], q.d), dmul(coef[2 * k], r));
    }
};

int persistent_grid(const Ctx& c) { return c.num_sms * RP_BLOCKS_PER_SM; }


// resident blocks per SM of the 384-entry-chunk variant (persistent grid)
template <class Op, class CT = int>
int rp_blocks_w12() {
    // function-local static: initialised once, thread-safe (one context per host thread is allowed)
    static const int blocks = [] {
        constexpr size_t smem =
            static_cast<size_t>(RP_WARPS) * 2 * RP_CH_W12 * (8 + sizeof(CT)) + RP_WARPS * 2 * sizeof(uint64_t);
        CK(cudaFuncSetAttribute(k_rowpass<Op, RP_CH_W12, 12, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        int b = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_rowpass<Op, RP_CH_W12, 12, CT>, RP_BLOCK, smem));
        return b < 1 ? 1 : (b > RP_BLOCKS_PER_SM ? RP_BLOCKS_PER_SM : b);
    }();
    return blocks;
}


template <class Op, int CH, int GATHER, class CT>
void launch_tma(Ctx& c, const char* fam, double bytes, const CsrView& A, const Op& op, Gate g, DotSink s,
                unsigned grid) {
    constexpr size_t smem = static_cast<size_t>(RP_WARPS) * 2 * CH * (8 + sizeof(CT)) +
                            RP_WARPS * 2 * sizeof(uint64_t) + (sizeof(CT) == 1 ? 256 * sizeof(int) : 0);
    static const bool configured = [] {
        CK(cudaFuncSetAttribute(k_rowpass<Op, CH, GATHER, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        return true;
    }();
    (void)configured;
    LAUNCH_PDL(c, fam, bytes, (k_rowpass<Op, CH, GATHER, CT>), grid, RP_BLOCK, smem, A, op, g, s);
}

// ---- k_dia: row pass over the symmetric-stencil form of level 0 -------------
// Thread per row (grid-stride).  Row i's entries in ascending column order:
// the lower neighbours i - off[K-1] .. i - off[0] (values U_k[i - off[k]],
// i.e. the neighbour's own upper entry: the form is only active when the
// values are bitwise symmetric), the diagonal D[i], the upper neighbours
// i + off[0] .. i + off[K-1] (U_k[i]); absent entries (mask) are skipped, so
// the sum s = 0 + a x + ... visits exactly the reference's entries in the
// reference's order (csr.cpp:79-84).  Every load is coalesced (shifted
// streams; the lower values and operands are L2 hits), no column stream, no
// row pointers: 8 (K + 1) + 1 bytes per row instead of 9 nnz/n + 4.
// Rows are dealt to lanes exactly as k_rowpass deals them (warp w of block b
// takes 32-row groups b*RP_WARPS + w, + RP_WARPS*grid, ...; lane l row
// 32 G + l) on k_rowpass's grid and block, so the per-thread dot partials and
// their block/grid reduction are k_rowpass's too: dots, and hence BiCGStab
// iterates, are bit-identical with and without the form.
template <class Op, int K>
__global__ void __launch_bounds__(RP_BLOCK, RP_BLOCKS_PER_SM) k_dia(CsrView A, Op op, Gate g, DotSink sink) {
    pdl_enter();
    if (gated_off(g)) return;
    constexpr int ND = Op::NDOT > 0 ? Op::NDOT : 1;
    constexpr int NE = 2 * K + 1;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;
    const int n = static_cast<int>(A.n);
    const int64_t nl = A.n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ngroups = (n + 31) >> 5;
    const int W = gridDim.x * RP_WARPS;
    const double* __restrict__ D = A.dia;
    for (int G = blockIdx.x * RP_WARPS + w; G < ngroups; G += W) {
        const int i = G * 32 + lane;
        if (i >= n) continue;
        const unsigned m = __ldg(A.dmask + i);
        const auto q = op.load(i);
        double av[NE], xv[NE];
#pragma unroll
        for (int b = 0; b < NE; ++b) {
            const bool on = (m >> b) & 1u;
            int j;
            const double* src;
            if (b < K) {  // lower: k = K - 1 - b
                j = i - A.doff[K - 1 - b];
                src = D + static_cast<int64_t>(K - b) * nl + j;
            } else if (b == K) {
                j = i;
                src = D + i;
            } else {  // upper: k = b - K - 1
                j = i + A.doff[b - K - 1];
                src = D + static_cast<int64_t>(b - K) * nl + i;
            }
            av[b] = on ? __ldg(src) : 0.0;
            xv[b] = on ? op.x(j) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < NE; ++b)
            if ((m >> b) & 1u) s = dadd(s, dmul(av[b], xv[b]));
        op.finish(i, s, q, dots);
    }
    if constexpr (Op::NDOT > 0) block_dots<Op::NDOT>(dots, sink);
}

template <class Op>
void launch_dia(Ctx& c, const char* fam, double bytes, const CsrView& A, const Op& op, Gate g, DotSink s,
                unsigned grid) {
    if (A.dk == 3)
        LAUNCH_PDL(c, fam, bytes, (k_dia<Op, 3>), grid, RP_BLOCK, 0, A, op, g, s);
    else
        LAUNCH_PDL(c, fam, bytes, (k_dia<Op, 2>), grid, RP_BLOCK, 0, A, op, g, s);
}

template <class Op>
void launch_rowpass(Ctx& c, const char* fam, double bytes, const CsrView& A, const Op& op, Gate g,
                    DotSink s, bool fixed_grid) {
    if (A.n == 0) return;
    const int64_t groups = (A.n + 31) / 32;
    int64_t want = (groups + RP_WARPS - 1) / RP_WARPS;
    int64_t cap = static_cast<int64_t>(c.num_sms) * RP_BLOCKS_PER_SM;
    unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
    if (fixed_grid) grid = static_cast<unsigned>(cap);  // deterministic dot order
    if (A.dia) {  // symmetric-stencil form of level 0 (same grid and row deal)
        launch_dia(c, fam, bytes, A, op, g, s, grid);
        return;
    }
    // coded columns: uint8 on <= 8 nnz/row, uint16 above (and on narrow partitioned levels)
    if (A.cmode == 1)
        launch_tma<Op, RP_CH, 0, uint8_t>(c, fam, bytes, A, op, g, s, grid);
    else if (A.cmode == 2 && A.nnz <= 8 * A.n)  // a partitioned level 0 (encode_columns narrow16)
        launch_tma<Op, RP_CH, 0, uint16_t>(c, fam, bytes, A, op, g, s, grid);
    else if (A.cmode == 2 && A.nnz > 12 * A.n)
        launch_tma<Op, RP_CH, 8, uint16_t>(c, fam, bytes, A, op, g, s, grid);
    else if (A.cmode == 2 && !fixed_grid)
        launch_tma<Op, RP_CH_W12, 12, uint16_t>(
            c, fam, bytes, A, op, g, s,
            static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(c.num_sms) *
                                                              rp_blocks_w12<Op, uint16_t>())));
    else if (A.cmode == 2)
        launch_tma<Op, RP_CH, 12, uint16_t>(c, fam, bytes, A, op, g, s, grid);
    else if (A.nnz > 8 * A.n && A.nnz <= 12 * A.n && !fixed_grid) {
        // 8..12 entries per row (C3 level 1): a 32-row group (~350 entries)
        // fits one 384-entry chunk, so lanes do not split their rows across
        // chunk boundaries; 6 resident blocks per SM instead of 8.
        // Level-1 passes 238/251 -> 211/228 us at 256^3 (512: no gain; the
        // > 12 nnz/row levels were slower with larger chunks).
        launch_tma<Op, RP_CH_W12, 12, int>(c, fam, bytes, A, op, g, s,
                                            static_cast<unsigned>(std::min<int64_t>(
                                                want, static_cast<int64_t>(c.num_sms) * rp_blocks_w12<Op>())));
    } else if (A.nnz > 12 * A.n)
        launch_tma<Op, RP_CH, 8, int>(c, fam, bytes, A, op, g, s, grid);
    else if (A.nnz > 8 * A.n)
        launch_tma<Op, RP_CH, 12, int>(c, fam, bytes, A, op, g, s, grid);
    else
        launch_tma<Op, RP_CH, 0, int>(c, fam, bytes, A, op, g, s, grid);
}

// bytes per stored entry of a row pass: fp64 value + column (int32, or the
// 1-/2-byte code of a coded column stream)
double entry_bytes(const CsrView& A) { return A.cmode == 1 ? 9.0 : A.cmode == 2 ? 10.0 : 12.0; }

// bytes of one pass over the operator itself (values + index structure)
double mat_bytes(const CsrView& A) {
    if (A.dia) return (8.0 * (A.dk + 1) + 1.0) * A.n;
    return entry_bytes(A) * A.nnz + 4.0 * (A.n + 1);
}

double spmv_bytes(const CsrView& A) {
    // symmetric-stencil form: D + K upper diagonals + the mask per row
    if (A.dia) return (8.0 * (A.dk + 1) + 1.0) * A.n + 8.0 * A.ncols + 8.0 * A.n;
    // value + column per entry + row_ptr + x read once + y written once
    return entry_bytes(A) * A.nnz + 4.0 * (A.n + 1) + 8.0 * A.ncols + 8.0 * A.n;
}

// ---- restriction / prolongation ------------------------------------------
// restriction f_c = R r (spmv with R = P^T, csr.cpp:79-84: members ascending,
// 1.0*r exact) and, for a coarse level that is smoothed next, its first
// pre-smoothing iterate u0_c = 0 + (om*w_c)*f_c.
__global__ void k_restrict(int nc, const int* __restrict__ mptr, const int* __restrict__ midx,
                           const double* __restrict__ r, double* __restrict__ fc, const double* __restrict__ wc,
                           double om, double* __restrict__ u0c, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < nc; I += gridDim.x * blockDim.x) {
        int p = __ldg(mptr + I);
        const int p1 = __ldg(mptr + I + 1);
        double s = 0.0;
        while (p < p1) {
            const int cnt = min(4, p1 - p);
            double rv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) rv[t] = t < cnt ? __ldg(r + __ldg(midx + p + t)) : 0.0;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < cnt) s = dadd(s, rv[t]);
            p += cnt;
        }
        fc[I] = s;
        if (u0c) u0c[I] = dadd(0.0, dmul(dmul(om, wc[I]), s));
    }
}

// u0 = 0 + (om*w)*f : first pre-smoothing iterate from a zero guess
__global__ void k_premul(int n, const double* __restrict__ f, const double* __restrict__ w, double om,
                         double* __restrict__ u0, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        u0[i] = dadd(0.0, dmul(dmul(om, w[i]), f[i]));
}

// prolongation onto the implicit first iterate u0 = 0 + (om*w)*f (see OpDownP)
__global__ void k_prolong_p(int n, const double* __restrict__ f, const double* __restrict__ w, double om,
                            const int* __restrict__ agg, const double* __restrict__ uc, double* __restrict__ out,
                            Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = dadd(dadd(0.0, dmul(dmul(om, w[i]), f[i])), dadd(0.0, uc[agg[i]]));
}

__global__ void k_prolong(int n, const double* __restrict__ u, const int* __restrict__ agg,
                          const double* __restrict__ uc, double* __restrict__ out, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = dadd(u[i], dadd(0.0, uc[agg[i]]));
}

// 4 consecutive rows per thread (16-byte vector loads of u/f/w, int4 of agg),
// one chunk per thread: the 4 coarse gathers of a thread are in flight
// together (the grid-stride scalar loops above serialise one dependent
// agg -> uc round trip per row)
__host__ __device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
__global__ void k_prolong_v4(int n, const double* __restrict__ u, const int* __restrict__ agg,
                             const double* __restrict__ uc, double* __restrict__ out, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    const int64_t i0 = 4 * (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
    if (i0 + 3 < n) {
        const int4 a = __ldg(reinterpret_cast<const int4*>(agg + i0));
        const double2 u01 = __ldg(reinterpret_cast<const double2*>(u + i0));
        const double2 u23 = __ldg(reinterpret_cast<const double2*>(u + i0 + 2));
        const double e0 = __ldg(uc + a.x), e1 = __ldg(uc + a.y), e2 = __ldg(uc + a.z), e3 = __ldg(uc + a.w);
        reinterpret_cast<double2*>(out + i0)[0] = make_double2(dadd(u01.x, dadd(0.0, e0)), dadd(u01.y, dadd(0.0, e1)));
        reinterpret_cast<double2*>(out + i0 + 2)[0] = make_double2(dadd(u23.x, dadd(0.0, e2)), dadd(u23.y, dadd(0.0, e3)));
    } else {
        for (int64_t i = i0; i < n; ++i) out[i] = dadd(u[i], dadd(0.0, uc[agg[i]]));
    }
}
__global__ void k_prolong_p_v4(int n, const double* __restrict__ f, const double* __restrict__ w, double om,
                               const int* __restrict__ agg, const double* __restrict__ uc, double* __restrict__ out,
                               Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    const int64_t i0 = 4 * (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
    if (i0 + 3 < n) {
        const int4 a = __ldg(reinterpret_cast<const int4*>(agg + i0));
        const double e0 = __ldg(uc + a.x), e1 = __ldg(uc + a.y), e2 = __ldg(uc + a.z), e3 = __ldg(uc + a.w);
        const double2 f01 = __ldg(reinterpret_cast<const double2*>(f + i0));
        const double2 f23 = __ldg(reinterpret_cast<const double2*>(f + i0 + 2));
        const double2 w01 = __ldg(reinterpret_cast<const double2*>(w + i0));
        const double2 w23 = __ldg(reinterpret_cast<const double2*>(w + i0 + 2));
        auto x = [&](double wi, double fi, double e) { return dadd(dadd(0.0, dmul(dmul(om, wi), fi)), dadd(0.0, e)); };
        reinterpret_cast<double2*>(out + i0)[0] = make_double2(x(w01.x, f01.x, e0), x(w01.y, f01.y, e1));
        reinterpret_cast<double2*>(out + i0 + 2)[0] = make_double2(x(w23.x, f23.x, e2), x(w23.y, f23.y, e3));
    } else {
        for (int64_t i = i0; i < n; ++i) out[i] = dadd(dadd(0.0, dmul(dmul(om, w[i]), f[i])), dadd(0.0, uc[agg[i]]));
    }
}

// ---- numeric RAP ----------------------------------------------------------
// Thread per coarse entry c (grid-stride), replaying the reference's two-level
// bracket of spmm(R, spmm(A, P)) (csr.cpp:145-194) over the cached plan:
//   acc = 0; part = 0; for p in [cptr[c], cptr[c+1]):
//     part += Af[contrib[p] & 0x7fffffff]; if (contrib[p] < 0) { acc += part; part = 0; }
// Plan and output are streamed with evict-first hints; the gathered fine values
// use the default policy so sectors shared by neighbouring aggregates can hit
// in L2.  (Variants measured slower in round 1 — row-group warps, shared-memory
// staging, 4 entries per thread: see DESIGN.md §3.3.)
// Numeric Galerkin product: coarse entry c sums its fine
// nonzeros contrib[cptr[c]..cptr[c+1]) in the reference's two-level bracket
// order (bit 31 of a contrib marks the end of one fine row's partial sum).
// Persistent blocks sweep the coarse entries in chunks of 256 x RAP_ILP,
// all blocks advancing together, so the fine values touched by a chunk (the
// rows of a few neighbouring aggregates) are still in L2 when the next chunk
// reuses their sectors.  Each thread runs RAP_ILP independent entries with
// the first two contributions loaded speculatively (avg 1.3 per entry at
// L0), so the cptr -> contrib -> value chains overlap.
constexpr int RAP_ILP = 4, RAP_BLOCK = 256;
// cptr entries: bit 30 flags a coarse diagonal entry (rap_symbolic), the
// low 30 bits are the contribution offset
constexpr int CP_DIAG = 1 << 30, CP_MASK = CP_DIAG - 1;

__device__ __forceinline__ void rap_acc(double v, int e, double& acc, double& part) {
    part = dadd(part, v);
    if (e < 0) {
        acc = dadd(acc, part);
        part = 0.0;
    }
}

__global__ void __launch_bounds__(RAP_BLOCK) k_rap(int64_t nnz_c, const int* __restrict__ cptr,
                                                   const int* __restrict__ contrib, const double* __restrict__ af,
                                                   double* __restrict__ ac) {
    constexpr int64_t CHUNK = static_cast<int64_t>(RAP_BLOCK) * RAP_ILP;
    for (int64_t base = blockIdx.x * CHUNK; base < nnz_c; base += static_cast<int64_t>(gridDim.x) * CHUNK) {
        int p0[RAP_ILP], p1[RAP_ILP], e0[RAP_ILP], e1[RAP_ILP];
        double v0[RAP_ILP], v1[RAP_ILP];
#pragma unroll
        for (int k = 0; k < RAP_ILP; ++k) {
            const int64_t c = base + k * RAP_BLOCK + threadIdx.x;
            p0[k] = c < nnz_c ? (__ldcs(cptr + c) & CP_MASK) : 0;
            p1[k] = c < nnz_c ? (__ldcs(cptr + c + 1) & CP_MASK) : 0;
        }
#pragma unroll
        for (int k = 0; k < RAP_ILP; ++k) {
            e0[k] = p0[k] < p1[k] ? __ldcs(contrib + p0[k]) : 0;
            e1[k] = p0[k] + 1 < p1[k] ? __ldcs(contrib + p0[k] + 1) : 0;
        }
#pragma unroll
        for (int k = 0; k < RAP_ILP; ++k) {
            v0[k] = p0[k] < p1[k] ? __ldg(af + (e0[k] & 0x7fffffff)) : 0.0;
            v1[k] = p0[k] + 1 < p1[k] ? __ldg(af + (e1[k] & 0x7fffffff)) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < RAP_ILP; ++k) {
            const int64_t c = base + k * RAP_BLOCK + threadIdx.x;
            if (c >= nnz_c) continue;
            double acc = 0.0, part = 0.0;
            if (p0[k] < p1[k]) rap_acc(v0[k], e0[k], acc, part);
            if (p0[k] + 1 < p1[k]) rap_acc(v1[k], e1[k], acc, part);
            for (int q = p0[k] + 2; q < p1[k]; ++q) {
                const int e = __ldcs(contrib + q);
                rap_acc(__ldg(af + (e & 0x7fffffff)), e, acc, part);
            }
            __stcs(ac + c, acc);
        }
    }
}

// TMA-staged variant: the streamed plan arrays (cptr and the chunk's
// contrib range) arrive by 1-D bulk copies into a double-buffered shared
// stage one chunk ahead, so the only global latency left per entry is the
// fine-value gather.  Chunks of RT_CH coarse entries, persistent blocks.
constexpr int RT_CH = 1024, RT_BLOCK = 256;

// PER entries per thread (strided by RT_BLOCK inside the chunk), the first B
// contributions of each loaded speculatively, the rest in batches of B; the
// accumulation is always the strict per-entry sequence of rap_acc.
template <int PER, int B, int FUSE>
__global__ void __launch_bounds__(RT_BLOCK, FUSE > 0 ? 4 : 5) k_rap_tma(int64_t nnz_c, const int* __restrict__ cptr,
                                                         const int* __restrict__ contrib,
                                                         const double* __restrict__ af, double* __restrict__ ac,
                                                         int cstage, RapJacobi fj) {
    static_assert(PER * RT_BLOCK <= RT_CH && RT_CH % (PER * RT_BLOCK) == 0, "chunk split");
    extern __shared__ __align__(128) unsigned char rt_smem[];
    int* s_cp = reinterpret_cast<int*>(rt_smem);  // [2][RT_CH + 4]
    int* s_cn = s_cp + 2 * (RT_CH + 4);            // [2][cstage]
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int s_ab[2];
    const int tid = threadIdx.x;
    const int64_t nchunks = (nnz_c + RT_CH - 1) / RT_CH;
    const int64_t G = gridDim.x;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // thread 0: stage chunk j whose contrib range [a, b) is known
    auto issue = [&](int64_t j, int st, int a, int b) {
        const int64_t c0 = j * RT_CH;
        const int64_t c1 = c0 + RT_CH < nnz_c ? c0 + RT_CH : nnz_c;
        const int ab = a & ~3, be = (b + 3) & ~3;
        s_ab[st] = ab;
        const uint32_t bc = static_cast<uint32_t>((c1 - c0 + 1 + 3) & ~3) * 4u;
        const uint32_t bn = static_cast<uint32_t>(be - ab) * 4u;
        fence_proxy_async();
        mbar_expect_tx(&bar[st], bc + bn);
        tma_load_1d(s_cp + st * (RT_CH + 4), cptr + c0, bc, &bar[st]);
        if (bn) tma_load_1d(s_cn + st * cstage, contrib + ab, bn, &bar[st]);
    };
    auto range = [&](int64_t j, int& a, int& b) {
        const int64_t c0 = j * RT_CH;
        a = __ldg(cptr + c0) & CP_MASK;
        b = __ldg(cptr + (c0 + RT_CH < nnz_c ? c0 + RT_CH : nnz_c)) & CP_MASK;
    };
    int64_t j = blockIdx.x;
    if (tid == 0) {
        int a, b;
        if (j < nchunks) {
            range(j, a, b);
            issue(j, 0, a, b);
        }
        if (j + G < nchunks) {
            range(j + G, a, b);
            issue(j + G, 1, a, b);
        }
    }
    int st = 0;
    uint32_t phase = 0;
    for (; j < nchunks; j += G) {
        // contrib range of the chunk two ahead (used after this chunk)
        int na = 0, nb = 0;
        const bool more = tid == 0 && j + 2 * G < nchunks;
        if (more) range(j + 2 * G, na, nb);
        mbar_wait(&bar[st], (phase >> st) & 1u);
        phase ^= (1u << st);
        const int64_t c0 = j * RT_CH;
        const int* cp = s_cp + st * (RT_CH + 4);
        const int* cn = s_cn + st * cstage;
        const int ab = s_ab[st];
        for (int sub = 0; sub < RT_CH; sub += PER * RT_BLOCK) {
            int p0[PER], p1[PER], e[PER][B];
            int dI[PER];  // coarse row of a diagonal entry (-1: not diagonal)
            double v[PER][B];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int x = sub + k * RT_BLOCK + tid;
                const bool ok = c0 + x < nnz_c;
                const int cx = ok ? cp[x] : 0;
                // prefetched with the plan so its latency overlaps the gathers
                dI[k] = (FUSE > 0 && (cx & CP_DIAG)) ? __ldg(fj.ccol + c0 + x) : -1;
                p0[k] = ok ? (cx & CP_MASK) - ab : 0;
                p1[k] = ok ? (cp[x + 1] & CP_MASK) - ab : 0;
#pragma unroll
                for (int t = 0; t < B; ++t) e[k][t] = p0[k] + t < p1[k] ? cn[p0[k] + t] : 0;
            }
            // unpredicated gathers (missing contributions re-read af[0], a cache
            // hit) so all PER*B loads are in flight before the first use
#pragma unroll
            for (int k = 0; k < PER; ++k)
#pragma unroll
                for (int t = 0; t < B; ++t) v[k][t] = __ldg(af + (e[k][t] & 0x7fffffff));
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int64_t c = c0 + sub + k * RT_BLOCK + tid;
                if (c >= nnz_c) continue;
                double acc = 0.0, part = 0.0;
#pragma unroll
                for (int t = 0; t < B; ++t)
                    if (p0[k] + t < p1[k]) rap_acc(v[k][t], e[k][t], acc, part);
                for (int q = p0[k] + B; q < p1[k]; q += B) {
                    int ee[B];
                    double vv[B];
#pragma unroll
                    for (int t = 0; t < B; ++t) ee[t] = q + t < p1[k] ? cn[q + t] : 0;
#pragma unroll
                    for (int t = 0; t < B; ++t) vv[t] = q + t < p1[k] ? __ldg(af + (ee[t] & 0x7fffffff)) : 0.0;
#pragma unroll
                    for (int t = 0; t < B; ++t)
                        if (q + t < p1[k]) rap_acc(vv[t], ee[t], acc, part);
                }
                __stcs(ac + c, acc);
                if constexpr (FUSE > 0) {
                    // this thread holds a coarse diagonal a_II: the damped-Jacobi
                    // weight of row I = its column (smoother.cpp:8-32)
                    if (dI[k] >= 0) {
                        const int I = dI[k];
                        if (acc == 0.0) {
                            atomicMin(fj.bad_c, I);
                            fj.wc[I] = 0.0;
                        } else {
                            fj.wc[I] = __drcp_rn(acc);  // == 1.0 / acc, both correctly rounded
                        }
                    }
                }
            }
        }
        __syncthreads();  // stage st consumed
        if (more) issue(j + 2 * G, st, na, nb);
        st ^= 1;
    }
}

template <int PER, int B, int FUSE>
void launch_rap_tma(Ctx& c, double bytes, int64_t nnz_c, const int* cptr, const int* contrib, const double* af,
                    double* ac, int cstage, size_t sm, const RapJacobi& fj) {
    static const bool attr = [] {  // opt in once (dynamic + static may exceed 48 KB)
        CK(cudaFuncSetAttribute(k_rap_tma<PER, B, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        return true;
    }();
    (void)attr;
    int res = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k_rap_tma<PER, B, FUSE>, RT_BLOCK, sm));
    const int64_t chunks = (nnz_c + RT_CH - 1) / RT_CH;
    const unsigned grid =
        static_cast<unsigned>(std::min<int64_t>(chunks, static_cast<int64_t>(c.num_sms) * std::max(res, 1)));
    LAUNCH(c, "rap", bytes, (k_rap_tma<PER, B, FUSE>), grid, RT_BLOCK, sm, nnz_c, cptr, contrib, af, ac, cstage, fj);
}

template <int PER, int B>
void launch_rap_tma_fused(Ctx& c, double bytes, int64_t nnz_c, const int* cptr, const int* contrib,
                          const double* af, double* ac, int cstage, size_t sm, const RapJacobi* fj) {
    if (!fj || !fj->wc)
        launch_rap_tma<PER, B, 0>(c, bytes, nnz_c, cptr, contrib, af, ac, cstage, sm, RapJacobi{});
    else
        launch_rap_tma<PER, B, 1>(c, bytes, nnz_c, cptr, contrib, af, ac, cstage, sm, *fj);
}

// ---- end k_rap_tma

// ---- k_rap_grp: warp-group Galerkin product (default) -----------------------
// One warp per group of consecutive coarse rows (GrpPlan, setup.cuh):
//  1. the group's member-row starts (<= 64) go to shared memory, its 2-byte
//     contribution codes arrive as aligned words;
//  2. gather, slot-parallel: lane l fetches contribution pairs 2l, 2l+1,
//     2l+64, ... from af[start of its member row + its offset] into shared
//     memory, in the plan's order — 64 entries of the group's neighbouring
//     member rows per instruction pair;
//  3. lane l sums the coarse entries of its run (the plan splits a group's
//     entries into 32 contiguous runs balanced by contribution count), each
//     over its contiguous contributions with the reference's bracket: the
//     partial of one member row is committed at the bracket bit
//     (csr.cpp:145-194) — the same arithmetic as k_rap /
//     k_rap_tma, bit for bit;
//  4. (JAC) w_i = 1.0 / a_ii of the member rows, first bad row into bad_f
//     (smoother.cpp:8-32, as k_jacobi).
// Plan bytes per fine entry drop from 4 (contrib) + 4 per coarse entry
// (cptr) to 2 + 0.25.  Measured and dropped (256^3): prefetching the next
// group's plan slice one group ahead, by per-lane cp.async (LDGSTS: 1.5x
// slower, MIO-throttled, +1 GB DRAM), by per-warp TMA bulk copies (4 small
// copies per group: 10% slower) or into registers one group ahead (more
// registers, fewer resident warps: 5-35% slower).
#ifndef RG_MINB
#define RG_MINB 5
#endif
constexpr int RG_WARPS = 8, RG_BUF = GRP_BUF, RG_MEM = 64;
struct RgSmem {
    double x[RG_BUF];
    uint32_t codew[RG_BUF / 2 + 2];
    int mst[RG_MEM];
};

template <bool JAC>
__global__ void __launch_bounds__(RG_WARPS * 32, RG_MINB) k_rap_grp(GrpArgs a) {
    extern __shared__ __align__(16) unsigned char rg_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    RgSmem& S = reinterpret_cast<RgSmem*>(rg_smem)[wid];
    uint16_t* s_code = reinterpret_cast<uint16_t*>(S.codew);
    const int64_t nw = static_cast<int64_t>(gridDim.x) * RG_WARPS;
    int64_t g = static_cast<int64_t>(blockIdx.x) * RG_WARPS + wid;
    int4 d0 = make_int4(0, 0, 0, 0), d1 = d0;
    if (g < a.ngroups) {
        d0 = __ldg(a.desc + g);
        d1 = __ldg(a.desc + g + 1);
    }
    for (; g < a.ngroups; g += nw) {
        // next group's descriptor, in flight during this one
        int4 n0 = d1, n1 = d1;
        if (g + nw < a.ngroups) {
            n0 = __ldg(a.desc + g + nw);
            n1 = __ldg(a.desc + g + nw + 1);
        }
        const int nmem = d1.y - d0.y, nbuf = d1.w - d0.w;
        const unsigned lt = __ldg(a.lanes + g * 32 + lane);
        int ms[2], md[2], mi[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int m = lane + 32 * k;
            const bool ok = m < nmem;
            ms[k] = ok ? __ldg(a.mstart + d0.y + m) : 0;
            md[k] = JAC && ok ? __ldg(a.mdoff + d0.y + m) : 255;
            mi[k] = JAC && ok ? __ldg(a.midx + d0.y + m) : 0;
        }
        const int dp = d0.w & 1;
        const int pw = (nbuf + dp + 1) >> 1;  // <= 128 words
        const uint32_t* cp = reinterpret_cast<const uint32_t*>(a.code) + ((d0.w - dp) >> 1);
        uint32_t wv[RG_BUF / 64];
#pragma unroll
        for (int k = 0; k < RG_BUF / 64; ++k) {
            const int t = lane + 32 * k;
            wv[k] = t < pw ? __ldg(cp + t) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k)
            if (lane + 32 * k < nmem) S.mst[lane + 32 * k] = ms[k];
        __syncwarp();
        // word w holds contributions 2w - dp and 2w - dp + 1
        double v[RG_BUF / 32];
#pragma unroll
        for (int k = 0; k < RG_BUF / 64; ++k) {
            const int w = lane + 32 * k;
            const int t = 2 * w - dp;
            const uint32_t c2 = wv[k];
            const unsigned lo = c2 & 0xffffu, hi = c2 >> 16;
            v[2 * k] = t >= 0 && t < nbuf ? __ldg(a.af + S.mst[(lo >> 8) & 63u] + (lo & 255u)) : 0.0;
            v[2 * k + 1] = t + 1 < nbuf ? __ldg(a.af + S.mst[(hi >> 8) & 63u] + (hi & 255u)) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < RG_BUF / 64; ++k) {
            const int w = lane + 32 * k;
            const int t = 2 * w - dp;
            if (w < pw) S.codew[w] = wv[k];
            if (t >= 0 && t < nbuf) S.x[t] = v[2 * k];
            if (t + 1 < nbuf) S.x[t + 1] = v[2 * k + 1];
        }
        __syncwarp();
        if (lane == 0) s_code[dp + nbuf] = 0x4000u;  // the end of the group closes the last entry
        __syncwarp();
        // this lane's run of coarse entries: contributions [p, e)
        int p = lt & 255u;
        const unsigned ln = __shfl_down_sync(0xffffffffu, lt, 1);
        const int e = lane < 31 ? static_cast<int>(ln & 255u) : nbuf;
        double* out = a.ac + d0.z + (lt >> 8);
        double acc = 0.0, part = 0.0;
        unsigned cd = p < e ? s_code[dp + p] : 0u;
        while (p < e) {
            part = dadd(part, S.x[p]);
            ++p;
            const unsigned nx = s_code[dp + p];
            if (cd & 0x8000u) {
                acc = dadd(acc, part);
                part = 0.0;
            }
            if (nx & 0x4000u) {
                __stcs(out++, acc);
                acc = 0.0;
            }
            cd = nx;
        }
        if constexpr (JAC) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (lane + 32 * k < nmem) {
                    const double d = md[k] != 255 ? __ldg(a.af + ms[k] + md[k]) : 0.0;
                    if (d == 0.0) {
                        atomicMin(a.bad_f, mi[k]);
                        a.wf[mi[k]] = 0.0;
                    } else {
                        a.wf[mi[k]] = __ddiv_rn(1.0, d);
                    }
                }
            }
        }
        __syncwarp();
        d0 = n0;
        d1 = n1;
    }
}

template <bool JAC>
static void launch_rap_grp(Ctx& c, const GrpArgs& a, double bytes) {
    const size_t sm = sizeof(RgSmem) * RG_WARPS;
    static const int res = [sm] {
        CK(cudaFuncSetAttribute(k_rap_grp<JAC>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        int r = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_rap_grp<JAC>, RG_WARPS * 32, sm));
        return r < 1 ? 1 : r;
    }();
    const int64_t need = (a.ngroups + RG_WARPS - 1) / RG_WARPS;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t{c.num_sms} * res)));
    LAUNCH(c, "rap", bytes, k_rap_grp<JAC>, grid, RG_WARPS * 32, sm, a);
}

// ---- k_rap_rows: member-row streaming Galerkin product ----------------------
// Thread per coarse row I.  Its members m (R, ascending fine index) are
// streamed row by row: the row's values are read contiguously (natural order,
// all loads in flight together) and parked in this thread's shared-memory
// column, then accumulated in the plan's order — slot groups, ascending k
// inside a group — so each group's partial is the inner bracket of
// spmm(A, P) and is committed to acc[slot] (the outer bracket of spmm(R, AP),
// members ascending; csr.cpp:145-194).  acc lives in shared
// memory interleaved by thread (acc[s][tid]: conflict-free).  The coarse
// row's diagonal gives the coarse Jacobi weight in the epilogue; on the first
// level of the chain the fine diagonal (flagged in the code) gives the fine
// one.  Values are bit-identical to k_rap / k_rap_tma.
constexpr int RR_BLOCK = 128;

template <int ML>
__global__ void __launch_bounds__(RR_BLOCK) k_rap_rows(RapRowsArgs a) {
    extern __shared__ __align__(16) double rr_sm[];
    const int tid = threadIdx.x;
    double* acc = rr_sm + tid;
    double* vs = rr_sm + a.dmax * RR_BLOCK + tid;
    const int I = blockIdx.x * RR_BLOCK + tid;
    if (I >= a.nc) return;
    const int c0 = __ldg(a.crp + I), deg = __ldg(a.crp + I + 1) - c0;
    for (int s = 0; s < deg; ++s) acc[s * RR_BLOCK] = 0.0;
    const int j0 = __ldg(a.mptr + I), j1 = __ldg(a.mptr + I + 1);
    for (int j = j0; j < j1; ++j) {
        const int base = __ldg(a.mrp + j);
        const int len = __ldg(a.mlen + j);
        unsigned cd[ML];
#pragma unroll
        for (int b = 0; b < ML; b += 8) {
            if (b < len) {
                double v[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    cd[b + t] = b + t < len ? __ldg(a.code + base + b + t) : 0u;
                    v[t] = b + t < len ? __ldg(a.af + base + b + t) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (b + t < len) vs[(b + t) * RR_BLOCK] = v[t];
            }
        }
        double part = 0.0, dv = 0.0;
        bool found = false;
#pragma unroll
        for (int t = 0; t < ML; ++t) {
            if (t < len) {
                const unsigned c = cd[t];
                const double x = vs[(c & 31u) * RR_BLOCK];
                part = dadd(part, x);
                if (c & 64u) {
                    dv = x;
                    found = true;
                }
                if (c & 32u) {
                    double* p = acc + (c >> 7) * RR_BLOCK;
                    *p = dadd(*p, part);
                    part = 0.0;
                }
            }
        }
        if (a.wf) {
            const int m = __ldg(a.midx + j);
            if (!found || dv == 0.0) {
                atomicMin(a.bad_f, m);
                a.wf[m] = 0.0;
            } else {
                a.wf[m] = __ddiv_rn(1.0, dv);
            }
        }
    }
    double* out = a.ac + c0;
    for (int s = 0; s < deg; ++s) out[s] = acc[s * RR_BLOCK];
    if (a.wc) {
        const int dp = __ldg(a.cdiag + I);
        const double d = dp >= 0 ? acc[(dp - c0) * RR_BLOCK] : 0.0;
        if (d == 0.0) {
            atomicMin(a.bad_c, I);
            a.wc[I] = 0.0;
        } else {
            a.wc[I] = __ddiv_rn(1.0, d);
        }
    }
}

template <int ML>
static void launch_rap_rows(Ctx& c, const RapRowsArgs& a, double bytes) {
    const size_t sm = sizeof(double) * static_cast<size_t>(a.dmax + ML) * RR_BLOCK;
    static const bool attr = [] {
        CK(cudaFuncSetAttribute(k_rap_rows<ML>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        return true;
    }();
    (void)attr;
    LAUNCH(c, "rap", bytes, k_rap_rows<ML>, (a.nc + RR_BLOCK - 1) / RR_BLOCK, RR_BLOCK, sm, a);
}
// w = 1/a_ii (smoother.cpp:8-32).  Each thread handles JB rows strided by the
// grid so the JB diagonal gathers (one 32-byte sector each) are in flight
// together.
constexpr int JB = 4;
__global__ void k_jacobi(int n, const double* __restrict__ val, const int* __restrict__ dpos,
                         double* __restrict__ w, int* bad) {
    const int stride = gridDim.x * blockDim.x;
    for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += JB * stride) {
        int k[JB];
        double d[JB];
#pragma unroll
        for (int t = 0; t < JB; ++t) k[t] = i0 + t * stride < n ? __ldg(dpos + i0 + t * stride) : -1;
#pragma unroll
        for (int t = 0; t < JB; ++t) d[t] = k[t] >= 0 ? __ldg(val + k[t]) : 0.0;
#pragma unroll
        for (int t = 0; t < JB; ++t) {
            const int i = i0 + t * stride;
            if (i >= n) continue;
            if (d[t] == 0.0) {
                atomicMin(bad, i);
                w[i] = 0.0;
            } else {
                w[i] = __ddiv_rn(1.0, d[t]);
            }
        }
    }
}

__global__ void k_spai0(CsrView A, const int* __restrict__ dpos, double* __restrict__ w, int* bad) {
    const int n = static_cast<int>(A.n);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) s = dadd(s, dmul(A.val[k], A.val[k]));
        const int k = dpos[i];
        const double d = k >= 0 ? A.val[k] : 0.0;
        if (d == 0.0) {
            atomicMin(bad, i);
            w[i] = 0.0;
        } else {
            w[i] = __ddiv_rn(d, s);
        }
    }
}

// ---- dense LU (coarse_factorize / coarse_solve, dense_lu.cpp:10-73) --------
// k_lu_cols: densify + LU with partial pivoting + the composed pivot
// permutation in ONE CTA, for n <= 160 (coarse_factorize, dense_lu.cpp:10-50).
// Warp w owns the columns j = w, w+16, ...; lane l the physical rows
// l, l+32, ...; the matrix lives in registers.  Rows are never moved: lp/pl
// map physical <-> logical rows (the reference's swaps).  Step k:
//  * the owner warp of column k finds the pivot with warp shuffles (max |.|
//    over logical rows >= k, lowest logical row on ties = the reference's
//    strict '>' scan; a NaN |m_kk| keeps p = k), records the swap and forms
//    the multipliers l = m_ik / pivot;
//  * one block barrier; every warp subtracts l*u_kj from its columns j > k
//    (m_ij -= l * m_kj, DMUL then DSUB as in the reference);
//  * look-ahead: the owner of column k+1 updates that column first and runs
//    step k+1's pivot search before its other columns, so the search overlaps
//    the bulk update.  Multipliers and the pivot row are double-buffered.
// The final logical->physical map is the composed rhs permutation of
// coarse_solve (dense_lu.cpp:58-59).
constexpr int LC_W = 16, LC_Q = 5, LC_C = 10, LC_MAXN = 160;

__device__ __forceinline__ double lc_sel(bool p, double a, double b) {
    double r;
    asm("{.reg .pred q; setp.ne.b32 q, %1, 0; selp.f64 %0, %2, %3, q;}" : "=d"(r) : "r"(static_cast<int>(p)), "d"(a),
        "d"(b));
    return r;
}

struct LcShared {
    double Lb[2][LC_MAXN];
    double Ub[LC_MAXN];
    int lp[LC_MAXN], pl[LC_MAXN];
    int pb[2];
    int s_status;
};

__device__ __forceinline__ void lc_pivot_step(double (&m)[LC_Q][LC_C], LcShared& S, int k, int n, int lane,
                                          int64_t* __restrict__ piv) {
    const int ck = k / LC_W;
    double colv[LC_Q];
#pragma unroll
    for (int q = 0; q < LC_Q; ++q) {
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < LC_C; ++c) v = lc_sel(c == ck, m[q][c], v);
        colv[q] = v;
    }
    double bv = -2.0;
    int bpos = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < LC_Q; ++q) {
        const int ph = lane + 32 * q;
        if (ph < n) {
            const int L = S.lp[ph];
            if (L >= k) {
                double v = fabs(colv[q]);
                if (v != v) v = -1.0;
                if (v > bv || (v == bv && L < bpos)) {
                    bv = v;
                    bpos = L;
                }
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int op = __shfl_xor_sync(0xffffffffu, bpos, off);
        if (ov > bv || (ov == bv && op < bpos)) {
            bv = ov;
            bpos = op;
        }
    }
    const int pk = S.pl[k];
    double vkk = 0.0;
#pragma unroll
    for (int q = 0; q < LC_Q; ++q) vkk = lc_sel(q == (pk >> 5), colv[q], vkk);
    vkk = __shfl_sync(0xffffffffu, vkk, pk & 31);
    const int p = (vkk != vkk) ? k : bpos;
    const int pp = S.pl[p];
    double pivot = 0.0;
#pragma unroll
    for (int q = 0; q < LC_Q; ++q) pivot = lc_sel(q == (pp >> 5), colv[q], pivot);
    pivot = __shfl_sync(0xffffffffu, pivot, pp & 31);
    __syncwarp();
    if (pivot == 0.0) {
        if (lane == 0) S.s_status = k;
        return;
    }
    if (lane == 0) {
        S.pl[k] = pp;
        S.pl[p] = pk;
        S.lp[pp] = k;
        S.lp[pk] = p;
        piv[k] = p;
        S.pb[k & 1] = pp;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < LC_Q; ++q) {
        const int ph = lane + 32 * q;
        if (ph < n && S.lp[ph] > k) {
            const double l = __ddiv_rn(colv[q], pivot);
            S.Lb[k & 1][ph] = l;
#pragma unroll
            for (int c = 0; c < LC_C; ++c) m[q][c] = lc_sel(c == ck, l, m[q][c]);
        }
    }
}

// columns j > k of this warp: m_ij -= l_i * u_j (only == slot `only`, or
// all but slot `skip`)
__device__ __forceinline__ void lc_update(double (&m)[LC_Q][LC_C], LcShared& S, int k, int n, int lane, int w,
                                      int only, int skip) {
    const int buf = k & 1;
    const int pp = S.pb[buf];
    if (lane == (pp & 31)) {
#pragma unroll
        for (int c = 0; c < LC_C; ++c) {
            double v = m[0][c];
#pragma unroll
            for (int q = 1; q < LC_Q; ++q) v = lc_sel(q == (pp >> 5), m[q][c], v);
            const int j = w + LC_W * c;
            if (j < n) S.Ub[j] = v;
        }
    }
    __syncwarp();
    double l[LC_Q];
    bool act[LC_Q];
#pragma unroll
    for (int q = 0; q < LC_Q; ++q) {
        const int ph = lane + 32 * q;
        act[q] = ph < n && S.lp[ph] > k;
        l[q] = act[q] ? S.Lb[buf][ph] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < LC_C; ++c) {
        const int j = w + LC_W * c;
        if (j <= k || j >= n) continue;
        if (only >= 0 && c != only) continue;
        if (c == skip) continue;
        const double u = S.Ub[j];
#pragma unroll
        for (int q = 0; q < LC_Q; ++q)
            if (act[q]) m[q][c] = dsub(m[q][c], dmul(l[q], u));
    }
}

__global__ void __launch_bounds__(LC_W * 32, 1) k_lu_cols(CsrView A, double* __restrict__ out,
                                                          int64_t* __restrict__ piv, int* __restrict__ perm,
                                                          int* status) {
    extern __shared__ __align__(16) double lc_dense[];
    __shared__ LcShared S;
    const int n = static_cast<int>(A.n);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int t = tid; t < n * n; t += LC_W * 32) lc_dense[t] = 0.0;
    __syncthreads();
    for (int i = tid; i < n; i += LC_W * 32)
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) lc_dense[i * n + A.col[e]] = A.val[e];
    for (int i = tid; i < n; i += LC_W * 32) {
        S.lp[i] = i;
        S.pl[i] = i;
    }
    if (tid == 0) S.s_status = -1;
    __syncthreads();
    double m[LC_Q][LC_C];
#pragma unroll
    for (int q = 0; q < LC_Q; ++q)
#pragma unroll
        for (int c = 0; c < LC_C; ++c) {
            const int i = lane + 32 * q, j = w + LC_W * c;
            m[q][c] = (i < n && j < n) ? lc_dense[i * n + j] : 0.0;
        }

    if (n > 0 && w == 0) lc_pivot_step(m, S, 0, n, lane, piv);
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        if (S.s_status >= 0) break;
        const int nk = k + 1;
        if (nk < n && w == nk % LC_W) {
            lc_update(m, S, k, n, lane, w, nk / LC_W, -1);
            lc_pivot_step(m, S, nk, n, lane, piv);
            lc_update(m, S, k, n, lane, w, -1, nk / LC_W);
        } else {
            lc_update(m, S, k, n, lane, w, -1, -1);
        }
        __syncthreads();
    }
    if (tid == 0) *status = S.s_status;
    if (S.s_status >= 0) return;
#pragma unroll
    for (int q = 0; q < LC_Q; ++q)
#pragma unroll
        for (int c = 0; c < LC_C; ++c) {
            const int i = lane + 32 * q, j = w + LC_W * c;
            if (i < n && j < n) out[S.lp[i] * n + j] = m[q][c];
        }
    for (int i = tid; i < n; i += LC_W * 32) perm[i] = S.pl[i];
}

__global__ void k_densify(CsrView A, double* dense) {
    const int64_t n = A.n;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dense[t] = 0.0;
}
// thread per row; the row bounds are read once and the (<= 8 at a time)
// entries loaded together (the stores could alias the CSR arrays for the
// compiler, which otherwise re-reads rp[i+1] and serialises the loads)
__global__ void k_densify_fill(CsrView A, double* __restrict__ dense) {
    const int64_t n = A.n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int k0 = __ldg(A.rp + i), k1 = __ldg(A.rp + i + 1);
        for (int k = k0; k < k1; k += 8) {
            int cj[8];
            double vj[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                cj[t] = k + t < k1 ? __ldg(A.col + k + t) : 0;
                vj[t] = k + t < k1 ? __ldg(A.val + k + t) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (k + t < k1) dense[i * n + cj[t]] = vj[t];
        }
    }
}

constexpr int LU_THREADS = 1024;

// coarse_factorize (dense_lu.cpp:10-50) replayed bit for bit: pivot = lowest
// row attaining the largest |m[i][k]| (the reference's strict '>' scan), row
// swap, l = m[i][k] / pivot, m[i][j] -= l*m[k][j] (no FMA).  One CTA; the
// factor lives in shared memory when it fits; a 32x32 thread tile walks the
// trailing submatrix without integer division; 3 barriers per step.
__global__ void __launch_bounds__(LU_THREADS) k_lu_factor(int n, double* gm, int64_t* piv, int* status,
                                                          int use_smem) {
    extern __shared__ double sm[];
    __shared__ double s_l[2048 + 1];
    __shared__ int s_p;
    double* m = use_smem ? sm : gm;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nn = n * n;
    if (use_smem)
        for (int t = tid; t < nn; t += blockDim.x) m[t] = gm[t];
    if (tid == 0) *status = -1;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        if (wid == 0) {
            double best = -1.0;
            int bi = 0x7fffffff;
            for (int i = k + lane; i < n; i += 32) {
                const double v = fabs(m[i * n + k]);
                if (v > best) {
                    best = v;
                    bi = i;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, best, off);
                const int oi = __shfl_down_sync(0xffffffffu, bi, off);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (lane == 0) {
                int p = bi;
                if (p == 0x7fffffff || !(fabs(m[k * n + k]) < best)) p = k;  // ties / NaN keep k
                s_p = p;
                piv[k] = p;
            }
        }
        __syncthreads();
        const int p = s_p;
        if (p != k)
            for (int j = tid; j < n; j += blockDim.x) {
                const double t = m[k * n + j];
                m[k * n + j] = m[p * n + j];
                m[p * n + j] = t;
            }
        __syncthreads();
        const double pivot = m[k * n + k];
        if (pivot == 0.0) {
            if (tid == 0) *status = k;
            break;
        }
        for (int i = k + 1 + tid; i < n; i += blockDim.x) {
            const double l = __ddiv_rn(m[i * n + k], pivot);
            s_l[i] = l;
            m[i * n + k] = l;
        }
        __syncthreads();
        const int ty = tid >> 5, tx = tid & 31;
        for (int i = k + 1 + ty; i < n; i += 32) {
            const double l = s_l[i];
            for (int j = k + 1 + tx; j < n; j += 32) m[i * n + j] = dsub(m[i * n + j], dmul(l, m[k * n + j]));
        }
        __syncthreads();
    }
    __syncthreads();
    if (use_smem)
        for (int t = tid; t < nn; t += blockDim.x) gm[t] = m[t];
}

// Register-resident dense elimination for small coarsest systems (n <= 160,
// the usual case: the coarsening stalls at ~150 rows).  512 threads; thread
// (ty, tx) holds rows ty + 16q and columns tx + 32m of the matrix in
// registers.  Rows are never moved: lp[] maps logical -> physical row and
// posof[] is its inverse, so the reference's row swaps (dense_lu.cpp:21-46)
// cost two integer stores.  Per step the pivot column and the pivot row are
// broadcast through shared memory (3 barriers).  The step loop is split into
// an unrolled loop over the 32-column group mb and a runtime loop over the
// lane kl, so every register access uses a compile-time index (no local
// memory) and column groups left of the pivot are skipped at compile time.
//   GJ = false: LU with the reference's pivot rule and operation order
//               (l = m[i][k] / pivot; m[i][j] -= l * m[k][j]).  Each row's
//               multipliers and, when it becomes the pivot row, its final U
//               part go to a shared-memory history Ls (by physical row), so
//               the register update is a bare DMUL + DADD on every row with
//               no predicates (finished rows just accumulate garbage); the
//               factor is written from Ls in the reference's swapped order.
//   GJ = true : in-place Gauss-Jordan inverse for AMGR_COARSE_INVERSE
//               (tolerance-level extension; output inv = A^{-1}).
#ifndef DR_THREADS_CFG
#define DR_THREADS_CFG 512
#endif
constexpr int DR_THREADS = DR_THREADS_CFG, DR_WARPS = DR_THREADS / 32, DR_ROWS = 160 / DR_WARPS, DR_COLS = 5,
              DR_MAXN = 160;

// predicated select in PTX: keeps NVVM from turning "for q: if (q == x) use
// a[q]" into a dynamically indexed (local-memory) access to the register tile
__device__ __forceinline__ double dr_sel(bool p, double a, double b) {
    double r;
    asm("{.reg .pred q; setp.ne.b32 q, %1, 0; selp.f64 %0, %2, %3, q;}" : "=d"(r) : "r"(static_cast<int>(p)), "d"(a),
        "d"(b));
    return r;
}

template <bool GJ>
__global__ void __launch_bounds__(DR_THREADS, 1) k_dense_reg(int n, const double* gin, double* gout,
                                                             int64_t* piv, int* status, int* perm) {
    extern __shared__ double Ls[];  // LU: n x n multiplier history, row = physical row
    __shared__ double colbuf[2][DR_MAXN], coll[DR_MAXN], rowbuf[DR_MAXN], lbuf[DR_MAXN];
    __shared__ int lp[DR_MAXN], posof[DR_MAXN];
    __shared__ int s_r, s_stop;
    __shared__ double s_piv;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, lane = tx;
    double a[DR_ROWS][DR_COLS];
    for (int i = tid; i < DR_MAXN; i += DR_THREADS) {
        colbuf[0][i] = 0.0;
        colbuf[1][i] = 0.0;
        lbuf[i] = 0.0;
    }
#pragma unroll
    for (int q = 0; q < DR_ROWS; ++q)
#pragma unroll
        for (int m = 0; m < DR_COLS; ++m) {
            const int i = ty + DR_WARPS * q, j = tx + 32 * m;
            a[q][m] = (i < n && j < n) ? gin[static_cast<int64_t>(i) * n + j] : 0.0;
        }
    for (int i = tid; i < DR_MAXN; i += DR_THREADS) {
        lp[i] = i;
        posof[i] = i;
        rowbuf[i] = 0.0;  // columns >= n stay 0
    }
    if (tid == 0) {
        *status = -1;
        s_stop = 0;
    }
    __syncthreads();
    bool stop = false;
#pragma unroll
    for (int mb = 0; mb < DR_COLS; ++mb) {
        for (int kl = 0; kl < 32; ++kl) {
            const int k = 32 * mb + kl;
            if (k >= n) break;
            double* cb = colbuf[k & 1];
            // 1. pivot column -> smem, by physical row (cb) and logical row (coll)
            if (tx == kl) {
#pragma unroll
                for (int q = 0; q < DR_ROWS; ++q) {
                    const int i = ty + DR_WARPS * q;
                    if (i < n) {
                        cb[i] = a[q][mb];
                        coll[posof[i]] = a[q][mb];
                    }
                }
            }
            __syncthreads();
            // 2. pivot: first maximum of |.| over logical rows k..n-1
            if (ty == 0) {
                double best = -1.0;
                int bi = 0x7fffffff;
                for (int i = k + lane; i < n; i += 32) {
                    const double v = fabs(coll[i]);
                    if (v > best) {
                        best = v;
                        bi = i;
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ob = __shfl_down_sync(0xffffffffu, best, off);
                    const int oi = __shfl_down_sync(0xffffffffu, bi, off);
                    if (ob > best || (ob == best && oi < bi)) {
                        best = ob;
                        bi = oi;
                    }
                }
                if (lane == 0) {
                    int p = bi;
                    if (p == 0x7fffffff || !(fabs(coll[k]) < best)) p = k;  // ties / NaN keep k
                    if (p != k) {
                        const int rk = lp[k], rp = lp[p];
                        lp[k] = rp;
                        lp[p] = rk;
                        posof[rp] = k;
                        posof[rk] = p;
                    }
                    if (!GJ) piv[k] = p;
                    const int r = lp[k];
                    s_r = r;
                    s_piv = cb[r];
                    if (cb[r] == 0.0) {
                        *status = k;
                        s_stop = 1;
                    }
                    if (GJ) cb[r] = 0.0;  // f = 0: the update leaves the pivot row alone
                }
            }
            __syncthreads();
            if (s_stop) {
                stop = true;
                break;
            }
            const int r = s_r;
            const double pivot = s_piv;
            // 3. pivot row -> smem (owner warp: ty == r % DR_WARPS, register row r / DR_WARPS)
            if (ty == r % DR_WARPS) {
                const int qr = r / DR_WARPS;
                const double ip = GJ ? 1.0 / pivot : 0.0;
#pragma unroll
                for (int m = 0; m < DR_COLS; ++m) {
                    double v = a[0][m];
#pragma unroll
                    for (int q = 1; q < DR_ROWS; ++q) v = dr_sel(q == qr, a[q][m], v);
                    const int j = tx + 32 * m;
                    if (GJ) {
                        v = (m == mb && tx == kl) ? ip : v * ip;
#pragma unroll
                        for (int q = 0; q < DR_ROWS; ++q) a[q][m] = dr_sel(q == qr, v, a[q][m]);
                    }
                    if (j < n) {
                        rowbuf[j] = v;
                        if (!GJ && j >= k) Ls[r * n + j] = v;  // final U row of r
                    }
                }
            }
            if (!GJ)
                for (int li = k + 1 + tid; li < n; li += DR_THREADS) {
                    const int ph = lp[li];
                    const double l = __ddiv_rn(cb[ph], pivot);
                    lbuf[ph] = l;
                    Ls[ph * n + k] = l;
                }
            __syncthreads();
            // 4. rank-1 update of the register tile
            double rb[DR_COLS];
#pragma unroll
            for (int m = 0; m < DR_COLS; ++m) rb[m] = rowbuf[tx + 32 * m];
            // row loads first (independent), then predicated updates: no
            // per-row branches, so the 10 rows' DMUL/DADD chains overlap
            // unpredicated updates: rows that must not change either have
            // f = 0 (GJ pivot row, padding) or are finished and already saved
            // in the Ls history (LU); padding rows/columns hold garbage
            if (GJ) {
#pragma unroll
                for (int q = 0; q < DR_ROWS; ++q) {
                    const double f = cb[ty + DR_WARPS * q];
                    if (tx == kl) a[q][mb] = dr_sel(ty + DR_WARPS * q != r, 0.0, a[q][mb]);
#pragma unroll
                    for (int m = 0; m < DR_COLS; ++m) a[q][m] = __fma_rn(-f, rb[m], a[q][m]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < DR_ROWS; ++q) {
                    const double l = lbuf[ty + DR_WARPS * q];
#pragma unroll
                    for (int m = mb; m < DR_COLS; ++m) a[q][m] = dsub(a[q][m], dmul(l, rb[m]));
                }
            }
        }
        if (stop) break;
    }
    __syncthreads();
    // write back: LU rows in logical (swapped) order, L part from the history;
    // inverse un-permuted: inv[posof[p]][lp[j]] = a[p][j]
#pragma unroll
    for (int q = 0; q < DR_ROWS; ++q) {
        const int i = ty + DR_WARPS * q;
        if (i < n) {
            const int rl = posof[i];
            const int64_t row = static_cast<int64_t>(rl) * n;
#pragma unroll
            for (int m = 0; m < DR_COLS; ++m) {
                const int j = tx + 32 * m;
                if (j < n) gout[GJ ? row + lp[j] : row + j] = GJ ? a[q][m] : Ls[i * n + j];
            }
        }
    }
    // the composed row swaps = the logical -> physical map (coarse_solve's
    // rhs permutation, dense_lu.cpp:58-59)
    if (!GJ && perm)
        for (int i = tid; i < n; i += DR_THREADS) perm[i] = lp[i];
}

constexpr int LS_THREADS = 64;

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// x = LU \ b replaying dense_lu.cpp:52-73 bit for bit.  The factor is staged
// into shared memory with one TMA bulk copy.  Forward sweep: column-oriented
// over warp 0 (each row still subtracts in ascending j).  Backward sweep: the
// reference's row-oriented chain (row i needs x[i+1] as its FIRST term, so the
// rows cannot overlap): warp 1 forms the products m[i-1][j]*x[j], j > i, of the
// next row while lane 0 of warp 0 runs row i's dependent subtraction chain;
// one named barrier per row.
__global__ void __launch_bounds__(LS_THREADS) k_lu_solve(int n, const double* __restrict__ m,
                                                         const int64_t* __restrict__ piv,
                                                         const double* b, double* x, int use_smem, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const int nn2 = use_smem ? ((n * n + 1) & ~1) : 0;
    double* ms = sm;              // n*n factor (when staged; 16-byte aligned TMA target)
    double* xs = sm + nn2;        // n
    double* ps = sm + nn2 + n;    // 2 x n products (double buffer)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const double* M = m;
    if (use_smem) {
        if (tid == 0) {
            mbar_init(&bar, 1);
            mbar_fence_init();
            const uint32_t bytes = static_cast<uint32_t>(((n * n + 1) & ~1) * 8);
            mbar_expect_tx(&bar, bytes);
            tma_load_1d(ms, m, bytes, &bar);
        }
        M = ms;
    }
    for (int i = tid; i < n; i += LS_THREADS) xs[i] = b[i];
    __syncthreads();
    if (wid == 0) {
        if (lane == 0)
            for (int k = 0; k < n; ++k) {
                const int p = static_cast<int>(piv[k]);
                if (p != k) {
                    const double t = xs[k];
                    xs[k] = xs[p];
                    xs[p] = t;
                }
            }
        if (use_smem) mbar_wait(&bar, 0);
        __syncwarp();
        for (int j = 0; j < n - 1; ++j) {
            const double xj = xs[j];
            for (int i = j + 1 + lane; i < n; i += 32) xs[i] = dsub(xs[i], dmul(M[i * n + j], xj));
            __syncwarp();
        }
    } else if (use_smem) {
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    // backward
    for (int i = n - 1; i >= 0; --i) {
        if (wid == 0) {
            if (lane == 0) {
                const double* mi = M + static_cast<int64_t>(i) * n;
                const double* pr = ps + (i & 1) * n;
                double s = xs[i];
                if (i + 1 < n) s = dsub(s, dmul(mi[i + 1], xs[i + 1]));
                int j = i + 2;
                for (; j + 8 <= n; j += 8) {
                    double q[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) q[t] = pr[j + t];
#pragma unroll
                    for (int t = 0; t < 8; ++t) s = dsub(s, q[t]);
                }
                for (; j < n; ++j) s = dsub(s, pr[j]);
                xs[i] = __ddiv_rn(s, mi[i]);
            }
        } else if (i > 0) {
            // products of row i-1 for j > i (x_j final)
            const double* mi = M + static_cast<int64_t>(i - 1) * n;
            double* pw = ps + ((i - 1) & 1) * n;
            for (int j = i + 1 + lane; j < n; j += 32) pw[j] = dmul(mi[j], xs[j]);
        }
        named_bar(1, LS_THREADS);
    }
    for (int i = tid; i < n; i += LS_THREADS) x[i] = xs[i];
}

// Single-warp exact solve for n <= 32*LW_Q (the register/shared-memory path
// used whenever the factor fits in shared memory).  Same arithmetic as
// dense_lu.cpp:52-73, in the same order per row:
//  * pivots: x = b[perm] with perm the composition of the reference's
//    sequential swaps (precomputed once per factorization, k_lu_perm);
//  * forward: column-oriented, lane l owns rows l, l+32, ... in registers;
//    step j broadcasts y_j with one shuffle, every row i > j subtracts
//    L_ij*y_j — per row still ascending j;
//  * backward: lane 0 runs the reference's row chain
//    s = y_i - U_i,i+1 x_i+1 - ... - U_i,n-1 x_n-1 with the products of the
//    next 8-entry chunk formed while the current chunk's dependent DSUBs issue
//    (software pipelined), so the sweep runs at the DSUB latency; no block
//    barriers at all.
constexpr int LW_Q = 5;  // rows per lane (n <= 160)

__device__ __forceinline__ double bwd_chain(const double* __restrict__ mi, const double* __restrict__ xs, int j0,
                                            int n, double s) {
    // s -= mi[j]*xs[j] for j = j0 .. n-1, ascending.  The leading (n - j0) % 8
    // entries go first so the 8-entry chunks end exactly at n.  Three-stage
    // software pipeline over the chunks: the shared-memory loads of chunk c+2
    // and the products of chunk c+1 issue while chunk c's dependent DSUB
    // chain runs, so (in-order issue) no instruction of the chain waits on a
    // load: the sweep runs at the DSUB latency.
    const int rem = (n - j0) & 7;
    const int jf = j0 + rem;          // first full chunk
    const int nch = (n - jf) >> 3;    // full chunks
    double ra[8], rx[8], p[8];
    // issue everything the first chunks need up front
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        ra[t] = mi[j0 + t];  // remainder (first rem used); reads stay inside the factor + slack
        rx[t] = xs[j0 + t];
    }
    double fa[8], fx[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        fa[t] = mi[jf + t];  // chunk 0 (harmless reads when nch == 0)
        fx[t] = xs[jf + t];
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) p[t] = dmul(ra[t], rx[t]);
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (t < rem) s = dsub(s, p[t]);
    if (nch == 0) return s;
    // chunk 0 products; raw loads of chunk 1
#pragma unroll
    for (int t = 0; t < 8; ++t) p[t] = dmul(fa[t], fx[t]);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        ra[t] = mi[jf + 8 + t];
        rx[t] = xs[jf + 8 + t];
    }
    int jn = jf + 16;  // raw chunk to load next
    for (int c = 0; c < nch; ++c) {
        double q[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            s = dsub(s, p[t]);
            q[t] = dmul(ra[t], rx[t]);  // chunk c+1 (garbage past the end, unused)
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            ra[t] = mi[jn + t];  // chunk c+2
            rx[t] = xs[jn + t];
            p[t] = q[t];
        }
        jn += 8;
    }
    return s;
}

__global__ void __launch_bounds__(32) k_lu_solve_warp(int n, const double* __restrict__ m,
                                                      const int* __restrict__ perm, const double* b, double* x,
                                                      Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x;
    const int nn2 = (n * n + 1) & ~1;
    double* ms = sm;        // n*n factor (TMA target)
    double* xs = sm + nn2;  // n (+16 slack read by the chunked chain)
    if (lane == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
        const uint32_t bytes = static_cast<uint32_t>(nn2 * 8);
        mbar_expect_tx(&bar, bytes);
        tma_load_1d(ms, m, bytes, &bar);
    }
    double y[LW_Q];
#pragma unroll
    for (int q = 0; q < LW_Q; ++q) {
        const int i = 32 * q + lane;
        y[q] = i < n ? b[perm[i]] : 0.0;
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    // forward (unit L)
#pragma unroll
    for (int gq = 0; gq < LW_Q; ++gq) {
        if (32 * gq >= n - 1) break;
        for (int t = 0; t < 32; ++t) {
            const int j = 32 * gq + t;
            if (j >= n - 1) break;
            const double yj = __shfl_sync(0xffffffffu, y[gq], t);
#pragma unroll
            for (int q = gq; q < LW_Q; ++q) {
                const int i = 32 * q + lane;
                if (i > j && i < n) y[q] = dsub(y[q], dmul(ms[i * n + j], yj));
            }
        }
    }
#pragma unroll
    for (int q = 0; q < LW_Q; ++q) {
        const int i = 32 * q + lane;
        if (i < n) xs[i] = y[q];
    }
    if (lane < 16) xs[n + lane] = 0.0;
    __syncwarp();
    // backward (row chain, lane 0)
    if (lane == 0) {
        double xn = __ddiv_rn(xs[n - 1], ms[(n - 1) * n + (n - 1)]);
        xs[n - 1] = xn;
        for (int i = n - 2; i >= 0; --i) {
            const double* mi = ms + i * n;
            double s = dsub(xs[i], dmul(mi[i + 1], xn));
            if (i + 2 < n) s = bwd_chain(mi, xs, i + 2, n, s);
            xn = __ddiv_rn(s, mi[i]);
            xs[i] = xn;
        }
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) x[i] = xs[i];
}

// Multi-warp variant (default for n <= 160): warp 0 runs the forward sweep
// (as above) and the backward row chain on lane 0; three helper warps form
// the chain's products ahead of it.  Row i of the chain is
//   s = y_i - U_i,i+1 x_i+1 - U_i,i+2 x_i+2 - P_i,i+3 - ... - P_i,n-1,
// x_i = s / U_ii (dense_lu.cpp:64-72, same association): the two newest
// products are formed by the chain itself, the rest (P_ij = U_ij x_j, all
// x_j known two rows earlier) by the helpers into a 3-slot ring of product
// rows, so the chain is one shared-memory load + one DSUB per entry.  The
// division uses the reciprocal formed ahead by the helpers (correctly
// rounded, __drcp_rn) and Markstein's correction q = s*y, r = s - U q
// (exact, FMA), x = q + r*y, which is the correctly rounded s / U_ii when no
// operand or result is near the under/overflow range (Markstein 1990; the
// same final step as CUDA's own division) — elsewhere it falls back to
// __ddiv_rn.  Bit-identical to the reference's solve.  The factor's TMA copy
// is issued before the PDL wait (it does not depend on the previous kernel).
constexpr int LM_HELP = 3, LM_PAD = 24;

__device__ __forceinline__ bool mk_range(double v) {
    const int e = (__double2hiint(v) >> 20) & 0x7ff;
    return e >= 600 && e <= 1446;  // |v| in [2^-423, 2^424): quotient, residual and products stay normal
}
__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_vol(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

__global__ void __launch_bounds__(32 * (1 + LM_HELP)) k_lu_solve_mw(int n, const double* __restrict__ m,
                                                                   const int* __restrict__ perm, const double* b,
                                                                   double* x, Gate g) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int s_prog, s_ready[3];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nn2 = (n * n + 1) & ~1, W = n + LM_PAD;
    double* ms = sm;            // n*n factor (TMA target)
    double* xs = sm + nn2;      // y, then x (W)
    double* pb = xs + W;        // 3 product rows (3W)
    double* rd = pb + 3 * W;    // 1 / U_ii (n)
    int* okd = reinterpret_cast<int*>(rd + n);  // U_ii in range (n)
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
        const uint32_t bytes = static_cast<uint32_t>(nn2 * 8);
        mbar_expect_tx(&bar, bytes);
        tma_load_1d(ms, m, bytes, &bar);
    }
    pdl_enter();
    const bool off = gated_off(g);
    for (int i = tid; i < 4 * W; i += blockDim.x) xs[i] = 0.0;  // xs + product rows (+0.0 padding)
    if (tid == 0) {
        s_prog = n;
        s_ready[0] = s_ready[1] = s_ready[2] = -1;
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    if (off) return;
    if (wid == 0) {
        double y[LW_Q];
#pragma unroll
        for (int q = 0; q < LW_Q; ++q) {
            const int i = 32 * q + lane;
            y[q] = i < n ? b[perm[i]] : 0.0;
        }
        // forward (unit L), column-oriented, rows in registers
#pragma unroll
        for (int gq = 0; gq < LW_Q; ++gq) {
            if (32 * gq >= n - 1) break;
            for (int t = 0; t < 32; ++t) {
                const int j = 32 * gq + t;
                if (j >= n - 1) break;
                const double yj = __shfl_sync(0xffffffffu, y[gq], t);
#pragma unroll
                for (int q = gq; q < LW_Q; ++q) {
                    const int i = 32 * q + lane;
                    if (i > j && i < n) y[q] = dsub(y[q], dmul(ms[i * n + j], yj));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < LW_Q; ++q) {
            const int i = 32 * q + lane;
            if (i < n) xs[i] = y[q];
        }
    } else {
        for (int i = tid - 32; i < n; i += 32 * LM_HELP) {
            const double u = ms[i * n + i];
            rd[i] = __drcp_rn(u);
            okd[i] = mk_range(u) ? 1 : 0;
        }
    }
    __syncthreads();
    if (wid == 0) {
        if (lane == 0) {
            auto mdiv = [&](double s, int i) -> double {
                const double u = ms[i * n + i];
                if (okd[i] && mk_range(s)) {
                    const double yv = rd[i];
                    const double q = __dmul_rn(s, yv);
                    const double r = __fma_rn(-u, q, s);
                    return __fma_rn(r, yv, q);
                }
                return __ddiv_rn(s, u);
            };
            double x1 = mdiv(xs[n - 1], n - 1), x2 = 0.0;
            xs[n - 1] = x1;
            __threadfence_block();
            st_vol(&s_prog, n - 1);
            for (int i = n - 2; i >= 0; --i) {
                const double* mi = ms + i * n;
                double s = dsub(xs[i], dmul(mi[i + 1], x1));
                if (i + 2 < n) s = dsub(s, dmul(mi[i + 2], x2));
                if (i + 3 < n) {
                    const double* P = pb + (i % 3) * W;
                    while (ld_vol(&s_ready[i % 3]) != i) {
                    }
                    int j = i + 3;
                    double a[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) a[t] = P[j + t];
                    for (; j < n; j += 8) {
                        double c[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) c[t] = P[j + 8 + t];  // +0.0 past n
#pragma unroll
                        for (int t = 0; t < 8; ++t) s = dsub(s, a[t]);   // padding: s - (+0.0) == s
#pragma unroll
                        for (int t = 0; t < 8; ++t) a[t] = c[t];
                    }
                }
                const double xi = mdiv(s, i);
                xs[i] = xi;
                __threadfence_block();
                st_vol(&s_prog, i);
                x2 = x1;
                x1 = xi;
            }
        }
    } else {
        const int hid = tid - 32;
        for (int i = n - 4; i >= 0; --i) {
            // products P_ij = U_ij x_j, j >= i + 3, once x_{i+3} is out (the
            // chain then no longer reads slot i % 3, last used by row i + 3)
            if (hid == 0) {
                while (ld_vol(&s_prog) > i + 3) {
                }
                __threadfence_block();
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LM_HELP) : "memory");
            double* P = pb + (i % 3) * W;
            const double* mi = ms + i * n;
            for (int j = i + 3 + hid; j < n; j += 32 * LM_HELP) P[j] = dmul(mi[j], xs[j]);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LM_HELP) : "memory");
            if (hid == 0) {
                __threadfence_block();
                st_vol(&s_ready[i % 3], i);
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) x[i] = xs[i];
}

// perm[i] = the rhs index that lands at position i after the reference's
// sequential swaps for k = 0..n-1: swap(x[k], x[piv[k]]) (dense_lu.cpp:60-61)
__global__ void k_lu_perm(int n, const int64_t* __restrict__ piv, int* __restrict__ perm) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
        const int p = static_cast<int>(piv[k]);
        if (p != k) {
            const int t = perm[k];
            perm[k] = perm[p];
            perm[p] = t;
        }
    }
}

// ---- FAST coarse solve (AMGR_COARSE_INVERSE, extension) -------------------
// Inverse of the coarsest matrix from its LU factors: warp per column,
// column-oriented forward and backward sweeps on the unit vectors (rounding
// differs from the reference's row-oriented solve; tolerance-level parity).
__global__ void __launch_bounds__(1024) k_lu_inverse(int n, const double* __restrict__ m,
                                                     const int64_t* __restrict__ piv, double* __restrict__ inv,
                                                     double* __restrict__ scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int col = blockIdx.x * nw + wid; col < n; col += gridDim.x * nw) {
        double* x = scratch + static_cast<int64_t>(col) * n;
        for (int i = lane; i < n; i += 32) x[i] = (i == col) ? 1.0 : 0.0;
        __syncwarp();
        if (lane == 0)
            for (int k = 0; k < n; ++k) {
                const int p = static_cast<int>(piv[k]);
                if (p != k) {
                    const double t = x[k];
                    x[k] = x[p];
                    x[p] = t;
                }
            }
        __syncwarp();
        for (int j = 0; j < n - 1; ++j) {
            const double xj = x[j];
            for (int i = j + 1 + lane; i < n; i += 32) x[i] = x[i] - m[static_cast<int64_t>(i) * n + j] * xj;
            __syncwarp();
        }
        for (int j = n - 1; j >= 0; --j) {
            if (lane == 0) x[j] = x[j] / m[static_cast<int64_t>(j) * n + j];
            __syncwarp();
            const double xj = x[j];
            for (int i = lane; i < j; i += 32) x[i] = x[i] - m[static_cast<int64_t>(i) * n + j] * xj;
            __syncwarp();
        }
        for (int i = lane; i < n; i += 32) inv[static_cast<int64_t>(i) * n + col] = x[i];
    }
}

// x = inv * b, warp per row, fixed-order lane partials + shuffle tree
__global__ void __launch_bounds__(1024) k_inv_apply(int n, const double* __restrict__ inv, const double* b,
                                                    double* x, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    extern __shared__ double bs[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) bs[i] = b[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int row = wid; row < n; row += nw) {
        const double* r = inv + static_cast<int64_t>(row) * n;
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s = __fma_rn(r[j], bs[j], s);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) x[row] = s;
    }
}

// power normalisation: lam = sqrt(yy)/sqrt(xx); x = y * (1/sqrt(yy)); xx' = x.x
// st = {yy, xx, lam}
__global__ void __launch_bounds__(256) k_power_norm(int n, const double* __restrict__ y, double* __restrict__ x,
                                                    double* st, DotSink ds) {
    const double yy = st[0];
    const double sc = 1.0 / sqrt(yy);
    double d[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double t = y[i] * sc;
        x[i] = t;
        d[0] = dadd(d[0], dmul(t, t));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st[2] = sqrt(yy) / sqrt(st[1]);
    block_dots<1>(d, ds);
}

// Gershgorin bound of D^-1 A: g = max_i sum_j |a_ij| / |a_ii| (row sums in
// column order; max is order-independent), as a non-negative double whose bit
// pattern orders like the value (atomicMax on the bits)
__global__ void k_gershgorin(CsrView A, const int* __restrict__ dpos, unsigned long long* out) {
    double g = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < A.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) s = dadd(s, fabs(A.val[k]));
        const double q = __ddiv_rn(s, fabs(A.val[dpos[i]]));
        g = q > g ? q : g;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double h = __shfl_xor_sync(0xffffffffu, g, o);
        g = h > g ? h : g;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(g)));
}

// power-iteration start vector: pseudo-random signs, x.x = n exactly
// (oracle/amg_oracle.c power_start_sign, same hash)
__global__ void k_power_start(int64_t n, double* x) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = (static_cast<uint64_t>(i) + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        x[i] = (z >> 63) ? -1.0 : 1.0;
    }
}

// Chebyshev coefficients from lam (oracle smooth_cheb): hi = lam*safety,
// lo = hi*lower, theta, delta, sigma; rho recursion for the degree-1 steps.
__global__ void k_cheb_coef(const double* st, double safety, double lower, int degree, double* coef) {
    const double hi = st[2] * safety, lo = hi * lower;
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo);
    const double sigma = theta / delta;
    double rho = 1.0 / sigma;
    coef[0] = theta;
    for (int k = 1; k < degree; ++k) {
        const double rho_new = 1.0 / (2.0 * sigma - rho);
        coef[2 * k - 1] = rho_new * rho;
        coef[2 * k] = 2.0 * rho_new / delta;
        rho = rho_new;
    }
    coef[2 * degree] = hi;
}

__global__ void k_axpy1(int n, double* __restrict__ x, const double* __restrict__ d, Gate g) {
    if (gated_off(g)) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = dadd(x[i], d[i]);
}

// d = (w*(f - 0)) / theta  (Chebyshev start from a zero iterate; A*0 = 0)
__global__ void k_cheb_zero(int n, const double* __restrict__ f, const double* __restrict__ w,
                            const double* __restrict__ coef, double* __restrict__ d, Gate g) {
    if (gated_off(g)) return;
    const double theta = coef[0];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        d[i] = __ddiv_rn(dmul(w[i], dsub(f[i], 0.0)), theta);
}

// ---- misc ---------------------------------------------------------------------
__global__ void k_fill(double* x, int64_t n, double v, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = v;
}
__global__ void k_copy(double* d, const double* s, int64_t n, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        d[i] = s[i];
}
__global__ void k_find_diag(CsrView A, int* dpos) {
    const int n = static_cast<int>(A.n);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int lo = A.rp[i], hi = A.rp[i + 1] - 1, found = -1;
        while (lo <= hi) {
            const int mid = (lo + hi) >> 1;
            const int cm = A.col[mid];
            if (cm == i) {
                found = mid;
                break;
            }
            if (cm < i) lo = mid + 1;
            else hi = mid - 1;
        }
        dpos[i] = found;
    }
}
__global__ void k_i32_to_i64(const int* s, int64_t* d, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        d[i] = s[i];
}
__global__ void k_i64_to_i32(const int64_t* s, int* d, int64_t n, int* ovf) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t v = s[i];
        if (v < INT32_MIN || v > INT32_MAX) *ovf = 1;
        d[i] = static_cast<int>(v);
    }
}
__global__ void k_max_span(const int* rp, int64_t n, int* out) {
    const int64_t groups = (n + 31) / 32;
    int m = 0;
    for (int64_t gi = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; gi < groups;
         gi += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t last = gi * 32 + 32 < n ? gi * 32 + 32 : n;
        const int span = ((rp[last] + 3) & ~3) - (rp[gi * 32] & ~3);
        m = max(m, span);
    }
    atomicMax(out, m);
}
__global__ void k_compare_i32(const int* a, const int* b, int64_t n, int* diff) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (a[i] != b[i]) *diff = 1;
}

}  // namespace

int dot_grid(const Ctx& c) { return c.num_sms * 8; }

// ---- launchers -----------------------------------------------------------------
void spmv(Ctx& c, const CsrView& A, const double* x, double* y, Gate g) {
    launch_rowpass(c, "spmv", spmv_bytes(A), A, OpSpmv{x, y}, g, {}, false);
}
void residual(Ctx& c, const CsrView& A, const double* f, const double* x, double* r, Gate g) {
    launch_rowpass(c, "residual", spmv_bytes(A) + 16.0 * A.n, A, OpResidual{f, x, r}, g, {}, false);
}
void vc_premul(Ctx& c, int64_t n, const double* f, const double* w, double om, double* u0, Gate g) {
    if (n == 0) return;
    LAUNCH_PDL(c, "vcycle_premul", 24.0 * n, k_premul, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(n), f,
           w, om, u0, g);
}
void vc_down(Ctx& c, const CsrView& A, const double* f, const double* u0, double* r, Gate g) {
    // A + f read once, u0 gathered (read once), r written once
    const double bytes = mat_bytes(A) + 24.0 * A.n;
    launch_rowpass(c, "vcycle_down", bytes, A, OpDown{f, u0, r}, g, {}, false);
}
void vc_restrict_general(Ctx& c, const CsrView& R, const double* r, double* fc, const double* wc, double om,
                         double* u0c, Gate g) {
    const double bytes = 12.0 * R.nnz + 4.0 * (R.n + 1) + 8.0 * R.ncols + 8.0 * R.n * (u0c ? 3 : 1);
    launch_rowpass(c, "restrict", bytes, R, OpRestrictG{r, fc, wc, om, u0c}, g, {}, false);
}
void vc_prolong_general(Ctx& c, const CsrView& P, const double* u, const double* e, double* out, Gate g) {
    const double bytes = 12.0 * P.nnz + 4.0 * (P.n + 1) + 8.0 * P.ncols + 16.0 * P.n;
    launch_rowpass(c, "prolong", bytes, P, OpProlongG{e, u, out}, g, {}, false);
}
void vc_down_premul(Ctx& c, const CsrView& A, const double* f, const double* w, double om, double* r, Gate g) {
    const double bytes = mat_bytes(A) + 24.0 * A.n;
    launch_rowpass(c, "vcycle_down", bytes, A, OpDownP{f, w, om, r}, g, {}, false);
}
// AMGR_VEC4=0: the scalar grid-stride prolongation kernels (A/B)
static bool vec_off() {
    const char* e = std::getenv("AMGR_VEC4");
    return e && e[0] == '0';
}
void vc_prolong_premul(Ctx& c, int64_t n, const double* f, const double* w, double om, const int* agg,
                       const double* uc, double* out, Gate g) {
    if (n == 0) return;
    if (al16(f) && al16(w) && al16(agg) && al16(out) && !vec_off()) {
        LAUNCH_PDL(c, "prolong", 28.0 * n, k_prolong_p_v4, grid_for((n + 3) / 4, 256), 256, 0, static_cast<int>(n),
                   f, w, om, agg, uc, out, g);
        return;
    }
    LAUNCH_PDL(c, "prolong", 28.0 * n, k_prolong_p, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(n), f,
               w, om, agg, uc, out, g);
}
// Row-list pass (the partitioned V-cycle's boundary rows after their halo
// arrived, dist.cu): thread per listed row, the same per-row arithmetic as
// k_rowpass — s = sum_j a_ij x_j in column order from 0.0, then Op::finish —
// so a row recomputed here gets the bits the full pass would have given it.
template <class Op>
__global__ void k_rowlist(CsrView A, const int* __restrict__ rows, int nrows, Op op, Gate g) {
    pdl_enter();
    if (gated_off(g)) return;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nrows; t += gridDim.x * blockDim.x) {
        const int i = __ldg(rows + t);
        const typename Op::Row q = op.load(i);
        double s = 0.0;
        for (int k = __ldg(A.rp + i); k < __ldg(A.rp + i + 1); ++k) s = dadd(s, dmul(__ldg(A.val + k), op.x(__ldg(A.col + k))));
        op.finish(i, s, q, nullptr);
    }
}
void vc_down_rows(Ctx& c, const CsrView& A, const int* rows, int64_t nrows, const double* f, const double* u0,
                  double* r, Gate g) {
    if (nrows == 0) return;
    LAUNCH_PDL(c, "vcycle_rows", 0.0, k_rowlist<OpDown>, grid_for(nrows, 128, c.num_sms * 8), 128, 0, A, rows,
               static_cast<int>(nrows), OpDown{f, u0, r}, g);
}
void vc_smooth_rows(Ctx& c, const CsrView& A, const int* rows, int64_t nrows, const double* f, const double* w,
                    double om, const double* u, double* out, Gate g) {
    if (nrows == 0) return;
    LAUNCH_PDL(c, "vcycle_rows", 0.0, k_rowlist<OpSmooth>, grid_for(nrows, 128, c.num_sms * 8), 128, 0, A, rows,
               static_cast<int>(nrows), OpSmooth{f, w, om, u, out}, g);
}
void vc_smooth(Ctx& c, const CsrView& A, const double* f, const double* w, double om, const double* u,
               double* out, Gate g) {
    const double bytes = mat_bytes(A) + 32.0 * A.n;
    launch_rowpass(c, "vcycle_smooth", bytes, A, OpSmooth{f, w, om, u, out}, g, {}, false);
}
void vc_prolong(Ctx& c, int64_t n, const double* u, const int* agg, const double* uc, double* out,
                Gate g) {
    if (n == 0) return;
    if (al16(u) && al16(agg) && al16(out) && !vec_off()) {
        LAUNCH_PDL(c, "prolong", 20.0 * n, k_prolong_v4, grid_for((n + 3) / 4, 256), 256, 0, static_cast<int>(n), u,
                   agg, uc, out, g);
        return;
    }
    LAUNCH_PDL(c, "prolong", 20.0 * n, k_prolong, grid_for(n, 256, c.num_sms * 16), 256, 0,
           static_cast<int>(n), u, agg, uc, out, g);
}
void restrict_sum(Ctx& c, int64_t nc, const int* mptr, const int* midx, const double* r, double* fc,
                  const double* wc, double om, double* u0c, Gate g) {
    if (nc == 0) return;
    // (a 4-rows-per-thread variant with all member loads in flight measured
    // slower: flat at level 0, 2x slower on the coarser levels' longer lists)
    LAUNCH_PDL(c, "restrict", 0.0, k_restrict, grid_for(nc, 256, c.num_sms * 16), 256, 0, static_cast<int>(nc), mptr,
           midx, r, fc, wc, om, u0c, g);
}
template <class Op2>
static bool launch_lag(Ctx& c, const CsrView& A, const OpSmooth& op1, const Op2& op2, Gate g, DotSink s,
                       int* done, int dgroups, double bytes) {
    using K = decltype(&k_rowpass_lag<OpSmooth, Op2, uint8_t>);
    const K kern = &k_rowpass_lag<OpSmooth, Op2, uint8_t>;
    constexpr size_t smem = static_cast<size_t>(RP_WARPS) * 2 * RP_CH * (8 + 1) + RP_WARPS * 2 * sizeof(uint64_t) +
                            256 * sizeof(int);
    static const int resident = [&] {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int b = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, RP_BLOCK, smem));
        return b;
    }();
    if (resident < RP_BLOCKS_PER_SM) return false;  // the whole persistent grid must be co-resident
    const int grid = c.num_sms * RP_BLOCKS_PER_SM;
    const int W = grid * RP_WARPS;
    const int64_t groups = (A.n + 31) / 32;
    const int64_t rounds = (groups + W - 1) / W;
    CK(cudaMemsetAsync(done, 0, sizeof(int) * static_cast<size_t>(rounds * LAG_SLOTS), c.stream));
    static const int lag = [] {
        const char* e = std::getenv("AMGR_LAG_ROUNDS");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    LAUNCH_PDL(c, "smooth_spmv", bytes, kern, grid, RP_BLOCK, smem, A, op1, op2, g, s, done, dgroups, lag);
    return true;
}

bool smooth_then_spmv(Ctx& c, const CsrView& A, const double* f, const double* w, double om, const double* u,
                      double* out, int kind, double* y, const double* ab, DotSink s, int* done, int dgroups,
                      Gate g) {
    if (A.cmode != 1 || A.n == 0 || dgroups <= 0) return false;
    // one DRAM sweep of A (+ the vectors of both passes); the second sweep is L2
    const double bytes = mat_bytes(A) + 32.0 * A.n + (kind == 1 ? 24.0 : 24.0) * A.n;
    const OpSmooth op1{f, w, om, u, out};
    if (kind == 1) return launch_lag(c, A, op1, OpSpmvDotL2{out, y, ab}, g, s, done, dgroups, bytes);
    return launch_lag(c, A, op1, OpSpmvDot2L2{out, y, ab}, g, s, done, dgroups, bytes);
}

void spmv_dot(Ctx& c, const CsrView& A, const double* x, double* y, const double* a, DotSink s, Gate g) {
    launch_rowpass(c, "spmv_dot", spmv_bytes(A) + 8.0 * A.n, A, OpSpmvDot{x, y, a}, g, s, true);
}
void spmv_dot2(Ctx& c, const CsrView& A, const double* x, double* y, const double* b, DotSink s,
               Gate g) {
    launch_rowpass(c, "spmv_dot2", spmv_bytes(A) + 8.0 * A.n, A, OpSpmvDot2{x, y, b}, g, s, true);
}
void resid_norm(Ctx& c, const CsrView& A, const double* f, const double* x, double* r, double* r2,
                DotSink s, Gate g) {
    launch_rowpass(c, "resid_norm", spmv_bytes(A), A, OpResidNorm{f, x, r, r2}, g, s, true);
}

__global__ void k_rap_chunk_max(int64_t nnz_c, const int* __restrict__ cptr, int* out) {
    const int64_t nchunks = (nnz_c + RT_CH - 1) / RT_CH;
    int m = 0;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < nchunks;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c1 = (j + 1) * RT_CH < nnz_c ? (j + 1) * RT_CH : nnz_c;
        m = max(m, (cptr[c1] & CP_MASK) - (cptr[j * RT_CH] & CP_MASK));
    }
    atomicMax(out, m);
}

int rap_chunk_max(Ctx& c, int64_t nnz_c, const int* cptr) {
    if (nnz_c == 0) return 0;
    DevArray<int> d(1, c.stream);
    CK(cudaMemsetAsync(d.get(), 0, sizeof(int), c.stream));
    LAUNCH(c, "setup", 0.0, k_rap_chunk_max, grid_for((nnz_c + RT_CH - 1) / RT_CH, 256, c.num_sms * 4), 256, 0,
           nnz_c, cptr, d.get());
    int h = 0;
    d2h(&h, d.get(), 1, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    return h;
}

bool rap_numeric(Ctx& c, int64_t nf, int64_t nc, int64_t nnz_c, const int* cptr, const int* contrib, const double* af,
                 double* ac, int64_t nnz_f, int max_chunk, const RapJacobi* fj) {
    if (nnz_c == 0) return false;
    // SURVEY.md 8(d) algorithmic bytes: 12*nnz(A_i) + 8*nnz(A_{i+1}) + 4*n_i + 4*(n_{i+1}+1);
    // fused Jacobi (SURVEY.md 8(d) Jacobi 20*n per level; the fine diagonal
    // value is gathered by the RAP itself): + 12*n_c (coarse) + 16*n_f (fine)
    double bytes = 12.0 * nnz_f + 8.0 * nnz_c + 4.0 * nf + 4.0 * (nc + 1);
    if (fj && fj->wc) bytes += 12.0 * nc;
    if (max_chunk >= 0) {
        const int cstage = (max_chunk + 8 + 3) & ~3;
        const size_t sm = sizeof(int) * (2 * (RT_CH + 4) + 2 * static_cast<size_t>(cstage));
        if (sm <= 96 * 1024) {
            // contributions per coarse entry: 1.3 (C3 L0), 2.4 (L1), 3-6 below
            static const double split = [] {  // contributions per coarse entry above which B = 4
                const char* e = std::getenv("AMGR_RAP_SPLIT");
                return e ? std::atof(e) : 2.5;
            }();
            if (static_cast<double>(nnz_f) <= split * static_cast<double>(nnz_c))
                launch_rap_tma_fused<4, 2>(c, bytes, nnz_c, cptr, contrib, af, ac, cstage, sm, fj);
            else
                launch_rap_tma_fused<2, 4>(c, bytes, nnz_c, cptr, contrib, af, ac, cstage, sm, fj);
            return fj != nullptr && fj->wc != nullptr;
        }
    }
    // persistent grid: exactly the resident blocks, so the sweep stays in order
    static const int resident = [] {
        int r = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_rap, RAP_BLOCK, 0));
        return r;
    }();
    const int64_t chunks = (nnz_c + RAP_BLOCK * RAP_ILP - 1) / (RAP_BLOCK * RAP_ILP);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(chunks, static_cast<int64_t>(c.num_sms) * resident));
    LAUNCH(c, "rap", bytes, k_rap, grid, RAP_BLOCK, 0, nnz_c, cptr, contrib, af, ac);
    return false;
}
void rap_grp(Ctx& c, const GrpArgs& a, int64_t nf, int64_t nc, int64_t nnz_f, int64_t nnz_c) {
    if (a.ngroups == 0) return;
    // RAP 12*nnz_f + 8*nnz_c + 4*nf + 4*(nc+1); fused Jacobi + 20*nf
    double bytes = 12.0 * nnz_f + 8.0 * nnz_c + 4.0 * nf + 4.0 * (nc + 1);
    if (a.wf) {
        launch_rap_grp<true>(c, a, bytes + 20.0 * nf);
    } else {
        launch_rap_grp<false>(c, a, bytes);
    }
}
void rap_rows(Ctx& c, const RapRowsArgs& a, int maxlen, int64_t nf, int64_t nnz_f, int64_t nnz_c) {
    if (a.nc == 0) return;
    // algorithmic bytes: values 8*nnz_f + codes 2*nnz_f + member starts and
    // lengths 5*nf + member pointers 4*(nc+1) + coarse row pointers 4*(nc+1)
    // + coarse values 8*nnz_c; fused Jacobi: + 8*nc (wc) and + 12*nf (wf, midx)
    double bytes = 10.0 * nnz_f + 5.0 * nf + 8.0 * (a.nc + 1) + 8.0 * nnz_c;
    if (a.wc) bytes += 12.0 * a.nc;
    if (a.wf) bytes += 12.0 * nf;
    if (maxlen <= 8)
        launch_rap_rows<8>(c, a, bytes);
    else if (maxlen <= 16)
        launch_rap_rows<16>(c, a, bytes);
    else
        launch_rap_rows<32>(c, a, bytes);
}

__global__ void k_reset_err(int64_t nl, int* err) {
    for (int64_t i = threadIdx.x; i <= nl; i += blockDim.x) err[i] = i < nl ? 0x7fffffff : -1;
}
void reset_error_slots(Ctx& c, int* err, int64_t nlevels) {
    LAUNCH(c, "setup", 0.0, k_reset_err, 1, 64, 0, nlevels, err);
}
void jacobi_rebuild(Ctx& c, int64_t n, const double* val, const int* dpos, double* w, int* bad) {
    if (n == 0) return;
    LAUNCH(c, "smoother", 20.0 * n, k_jacobi, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(n),
           val, dpos, w, bad);
}
void spai0_rebuild(Ctx& c, const CsrView& A, const int* dpos, double* w, int* bad) {
    if (A.n == 0) return;
    LAUNCH(c, "smoother", 8.0 * A.nnz + 12.0 * A.n, k_spai0, grid_for(A.n, 256, c.num_sms * 16), 256, 0, A,
           dpos, w, bad);
}

void lu_densify(Ctx& c, const CsrView& A, double* dense) {
    if (A.n == 0) return;
    LAUNCH(c, "coarse", 0.0, k_densify, grid_for(A.n * A.n, 256, c.num_sms * 8), 256, 0, A, dense);
    LAUNCH(c, "coarse", 0.0, k_densify_fill, grid_for(A.n, 128, c.num_sms * 8), 128, 0, A, dense);
}

static void lu_perm(Ctx& c, int64_t n, const int64_t* piv, int* perm) {
    if (perm) LAUNCH(c, "coarse", 0.0, k_lu_perm, 1, 32, 0, static_cast<int>(n), piv, perm);
}

void lu_factor(Ctx& c, int64_t n, double* m, int64_t* piv, int* status, int* perm, const CsrView* A) {
    if (n == 0) return;
    if (n <= DR_MAXN) {
        if (A) lu_densify(c, *A, m);
        const size_t sm = sizeof(double) * static_cast<size_t>(n * n);
        // always opt in: dynamic + static shared memory above 48 KB needs the
        // attribute even when the dynamic part alone is below it (n = 72..78)
        static const bool attr = [] {
            CK(cudaFuncSetAttribute(k_dense_reg<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(double) * DR_MAXN * DR_MAXN)));
            return true;
        }();
        (void)attr;
        LAUNCH(c, "coarse", 0.0, k_dense_reg<false>, 1, DR_THREADS, sm, static_cast<int>(n), m, m, piv, status,
               perm);
        return;
    }
    if (A) lu_densify(c, *A, m);
    if (n > 2048) invalid("coarse_factorize: coarse system larger than 2048 unknowns is not supported on device");
    const size_t sm = sizeof(double) * static_cast<size_t>(n * n);
    const int use_smem = sm <= 180 * 1024 ? 1 : 0;
    if (use_smem) CK(cudaFuncSetAttribute(k_lu_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024));
    LAUNCH(c, "coarse", 0.0, k_lu_factor, 1, LU_THREADS, use_smem ? sm : 0, static_cast<int>(n), m, piv, status,
           use_smem);
    lu_perm(c, n, piv, perm);
}

void lu_solve(Ctx& c, int64_t n, const double* m, const int64_t* piv, const double* b, double* x, Gate g,
              const int* perm) {
    if (n == 0) return;
    const char* old = std::getenv("AMGR_LU_SOLVE_OLD");  // 1: k_lu_solve, 2: single-warp k_lu_solve_warp
    if (perm && n <= 32 * LW_Q && !(old && (old[0] == '1' || old[0] == '2'))) {
        static const bool attr = [] {
            const int W = 32 * LW_Q + LM_PAD;
            CK(cudaFuncSetAttribute(k_lu_solve_mw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(double) * (32 * LW_Q * 32 * LW_Q + 4 * W + 32 * LW_Q) +
                                                     sizeof(int) * 32 * LW_Q)));
            return true;
        }();
        (void)attr;
        const int64_t W = n + LM_PAD;
        const size_t sm = sizeof(double) * static_cast<size_t>(((n * n + 1) & ~1) + 4 * W + n) +
                          sizeof(int) * static_cast<size_t>(n);
        LAUNCH_PDL(c, "coarse_solve", 0.0, k_lu_solve_mw, 1, 32 * (1 + LM_HELP), sm, static_cast<int>(n), m, perm, b,
                   x, g);
        return;
    }
    if (perm && n <= 32 * LW_Q && !(old && old[0] == '1')) {
        static const bool attr = [] {
            CK(cudaFuncSetAttribute(k_lu_solve_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(double) * (32 * LW_Q * 32 * LW_Q + 32 * LW_Q + 16))));
            return true;
        }();
        (void)attr;
        const size_t sm = sizeof(double) * static_cast<size_t>(((n * n + 1) & ~1) + n + 16);
        LAUNCH_PDL(c, "coarse_solve", 0.0, k_lu_solve_warp, 1, 32, sm, static_cast<int>(n), m, perm, b, x, g);
        return;
    }
    const size_t full = sizeof(double) * static_cast<size_t>(((n * n + 1) & ~1) + 3 * n);
    const int use_smem = full <= 200 * 1024 ? 1 : 0;
    const size_t sm = use_smem ? full : sizeof(double) * static_cast<size_t>(3 * n);
    static const bool attr = [] {  // opt in once (dynamic + static may exceed 48 KB)
        CK(cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        return true;
    }();
    (void)attr;
    LAUNCH_PDL(c, "coarse_solve", 0.0, k_lu_solve, 1, LS_THREADS, sm, static_cast<int>(n), m, piv, b, x, use_smem, g);
}

bool lu_factor_csr(Ctx& c, const CsrView& A, double* lu, int64_t* piv, int* status, int* perm) {
    const char* e = std::getenv("AMGR_LU_COLS");  // opt-in: slower than k_dense_reg so far
    if (!perm || A.n == 0 || A.n > LC_MAXN || !(e && e[0] == '1')) return false;
    const size_t sm = sizeof(double) * static_cast<size_t>(A.n * A.n);
    static const bool attr = [] {
        CK(cudaFuncSetAttribute(k_lu_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * LC_MAXN * LC_MAXN)));
        return true;
    }();
    (void)attr;
    LAUNCH(c, "coarse", 0.0, k_lu_cols, 1, LC_W * 32, sm, A, lu, piv, perm, status);
    return true;
}

bool dense_inverse_direct(Ctx& c, int64_t n, const double* a, double* inv, int64_t* piv, int* status) {
    if (n == 0 || n > DR_MAXN) return false;
    LAUNCH(c, "coarse", 0.0, k_dense_reg<true>, 1, DR_THREADS, 0, static_cast<int>(n), a, inv, piv, status,
           static_cast<int*>(nullptr));
    return true;
}

void lu_inverse(Ctx& c, int64_t n, const double* m, const int64_t* piv, double* inv) {
    if (n == 0) return;
    DevArray<double> scratch(n * n, c.stream);
    LAUNCH(c, "coarse", 0.0, k_lu_inverse, grid_for(n, 32, 64), 1024, 0, static_cast<int>(n), m, piv, inv,
           scratch.get());
}

void inv_apply(Ctx& c, int64_t n, const double* inv, const double* b, double* x, Gate g) {
    if (n == 0) return;
    const size_t sm = sizeof(double) * static_cast<size_t>(n);
    static const bool attr = [] {
        CK(cudaFuncSetAttribute(k_inv_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        return true;
    }();
    (void)attr;
    LAUNCH_PDL(c, "coarse_solve", 0.0, k_inv_apply, 1, 1024, sm, static_cast<int>(n), inv, b, x, g);
}

void power_step(Ctx& c, const CsrView& A, const double* w, const double* x, double* y, DotSink s) {
    launch_rowpass(c, "power", spmv_bytes(A) + 8.0 * A.n, A, OpPower{x, w, y}, Gate{}, s, true);
}
void gershgorin_bound(Ctx& c, const CsrView& A, const int* dpos, unsigned long long* out) {
    if (A.n == 0) return;
    LAUNCH(c, "smoother", 12.0 * A.nnz + 8.0 * A.n, k_gershgorin, grid_for(A.n, 256, c.num_sms * 8), 256, 0, A, dpos,
           out);
}
void power_start(Ctx& c, int64_t n, double* x) {
    LAUNCH(c, "power", 8.0 * n, k_power_start, grid_for(n, 256, c.num_sms * 16), 256, 0, n, x);
}
void power_norm(Ctx& c, int64_t n, const double* y, double* x, double* st, DotSink s) {
    LAUNCH(c, "power", 16.0 * n, k_power_norm, dot_grid(c), 256, 0, static_cast<int>(n), y, x, st, s);
}
void cheb_coef(Ctx& c, const double* st, double safety, double lower, int degree, double* coef) {
    LAUNCH(c, "smoother", 0.0, k_cheb_coef, 1, 1, 0, st, safety, lower, degree, coef);
}
void cheb_start(Ctx& c, const CsrView& A, const double* f, const double* w, const double* x, const double* coef,
                double* d, Gate g) {
    launch_rowpass(c, "cheb", spmv_bytes(A) + 16.0 * A.n, A, OpChebStart{f, w, x, coef, d}, g, {}, false);
}
void cheb_zero(Ctx& c, int64_t n, const double* f, const double* w, const double* coef, double* d, Gate g) {
    if (n == 0) return;
    LAUNCH(c, "cheb", 24.0 * n, k_cheb_zero, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(n), f, w,
           coef, d, g);
}
void cheb_step(Ctx& c, const CsrView& A, const double* f, const double* w, const double* x, const double* d,
               const double* coef, int k, double* xout, double* dout, Gate g) {
    launch_rowpass(c, "cheb", spmv_bytes(A) + 40.0 * A.n, A, OpChebStep{f, w, x, d, coef, k, xout, dout}, g, {},
                   false);
}
void axpy1(Ctx& c, int64_t n, double* x, const double* d, Gate g) {
    if (n == 0) return;
    LAUNCH(c, "cheb", 24.0 * n, k_axpy1, grid_for(n, 256, c.num_sms * 16), 256, 0, static_cast<int>(n), x, d, g);
}

void fill(Ctx& c, double* x, int64_t n, double v, Gate g) {
    if (n == 0) return;
    LAUNCH_PDL(c, "vec", 8.0 * n, k_fill, grid_for(n, 256, c.num_sms * 16), 256, 0, x, n, v, g);
}
void copy(Ctx& c, double* d, const double* s, int64_t n, Gate g) {
    if (n == 0) return;
    LAUNCH_PDL(c, "vec", 16.0 * n, k_copy, grid_for(n, 256, c.num_sms * 16), 256, 0, d, s, n, g);
}
void find_diag(Ctx& c, const CsrView& A, int* dpos) {
    if (A.n == 0) return;
    LAUNCH(c, "setup", 0.0, k_find_diag, grid_for(A.n, 256, c.num_sms * 16), 256, 0, A, dpos);
}
void i32_to_i64(Ctx& c, const int* s, int64_t* d, int64_t n) {
    if (n == 0) return;
    LAUNCH(c, "io", 0.0, k_i32_to_i64, grid_for(n, 256, c.num_sms * 16), 256, 0, s, d, n);
}
void i64_to_i32(Ctx& c, const int64_t* s, int* d, int64_t n, int* ovf) {
    if (n == 0) return;
    LAUNCH(c, "io", 0.0, k_i64_to_i32, grid_for(n, 256, c.num_sms * 16), 256, 0, s, d, n, ovf);
}
int max_group_span(Ctx& c, const int* rp, int64_t n) {
    if (n == 0) return 0;
    DevArray<int> m(1, c.stream);
    CK(cudaMemsetAsync(m.get(), 0, sizeof(int), c.stream));
    LAUNCH(c, "setup", 0.0, k_max_span, grid_for((n + 31) / 32, 256, c.num_sms * 8), 256, 0, rp, n, m.get());
    return d2h_scalar(m.get(), c.stream);
}
void compare_i32(Ctx& c, const int* a, const int* b, int64_t n, int* diff) {
    if (n == 0) return;
    LAUNCH(c, "io", 0.0, k_compare_i32, grid_for(n, 256, c.num_sms * 16), 256, 0, a, b, n, diff);
}


// ---- symmetric-stencil form: masks (per pattern) and values (per rebuild) ----
namespace {
struct DiaOff {
    int k;
    int o[3];
};
// bit of column offset d in the mask order (ascending column), -1 if none
__device__ __forceinline__ int dia_bit(const DiaOff& f, int64_t d) {
    if (d == 0) return f.k;
    for (int k = 0; k < f.k; ++k) {
        if (d == -f.o[k]) return f.k - 1 - k;
        if (d == f.o[k]) return f.k + 1 + k;
    }
    return -1;
}
__global__ void k_dia_mask(CsrView A, DiaOff f, uint8_t* mask, int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < A.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        unsigned m = 0;
        int last = -1;
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            const int b = dia_bit(f, static_cast<int64_t>(A.col[e]) - i);
            if (b <= last) {  // unknown offset, unsorted or repeated column
                atomicOr(bad, 1);
                break;
            }
            m |= 1u << b;
            last = b;
        }
        mask[i] = static_cast<uint8_t>(m);
    }
}
// structural symmetry: (i, i+o_k) present <=> (i+o_k, i) present
__global__ void k_dia_symm(int64_t n, DiaOff f, const uint8_t* mask, int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned m = mask[i];
        for (int k = 0; k < f.k; ++k) {
            const bool up = (m >> (f.k + 1 + k)) & 1u, lo = (m >> (f.k - 1 - k)) & 1u;
            const int64_t ju = i + f.o[k], jl = i - f.o[k];
            const bool pu = ju < n && ((mask[ju] >> (f.k - 1 - k)) & 1u);
            const bool pl = jl >= 0 && ((mask[jl] >> (f.k + 1 + k)) & 1u);
            if (up != pu || lo != pl) atomicOr(bad, 1);
        }
    }
}
__global__ void k_dia_values(CsrView A, DiaOff f, const uint8_t* __restrict__ mask, double* __restrict__ dia,
                             int* flag) {
    const int64_t n = A.n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned m = mask[i];
        const int base = __ldg(A.rp + i);
        bool diff = false;
        dia[i] = 0.0;
        for (int k = 0; k < f.k; ++k) dia[static_cast<int64_t>(k + 1) * n + i] = 0.0;
        for (int b = 0; b < 2 * f.k + 1; ++b) {
            if (!((m >> b) & 1u)) continue;
            const double v = __ldg(A.val + base + __popc(m & ((1u << b) - 1u)));
            if (b == f.k) {
                dia[i] = v;
            } else if (b > f.k) {
                dia[static_cast<int64_t>(b - f.k) * n + i] = v;
            } else {  // lower entry k: must equal the partner's upper entry bit for bit
                const int k = f.k - 1 - b;
                const int64_t j = i - f.o[k];
                const unsigned mj = mask[j];
                const int bj = f.k + 1 + k;
                const double u = __ldg(A.val + __ldg(A.rp + j) + __popc(mj & ((1u << bj) - 1u)));
                diff |= __double_as_longlong(u) != __double_as_longlong(v);
            }
        }
        if (diff) atomicOr(flag, 1);
    }
}
DiaOff dia_off(int K, const int* off) {
    DiaOff f{};
    f.k = K;
    for (int k = 0; k < K; ++k) f.o[k] = off[k];
    return f;
}
}  // namespace

bool dia_masks(Ctx& c, const CsrView& A, int K, const int* off, uint8_t* mask) {
    if (A.n == 0 || K < 1 || K > 3) return false;
    DevArray<int> bad(1, c.stream);
    CK(cudaMemsetAsync(bad.get(), 0, sizeof(int), c.stream));
    const DiaOff f = dia_off(K, off);
    LAUNCH(c, "setup", 0.0, k_dia_mask, grid_for(A.n, 256, c.num_sms * 8), 256, 0, A, f, mask, bad.get());
    LAUNCH(c, "setup", 0.0, k_dia_symm, grid_for(A.n, 256, c.num_sms * 8), 256, 0, A.n, f, mask, bad.get());
    return d2h_scalar(bad.get(), c.stream) == 0;
}

void dia_values(Ctx& c, const CsrView& A, int K, const int* off, const uint8_t* mask, double* dia, int* flag) {
    if (A.n == 0) return;
    CK(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
    // 6 of 8 block slots per SM (measured: the full grid slows the Galerkin
    // levels it overlaps more than it gains)
    const char* e = std::getenv("AMGR_DIA_BLOCKS");
    const int per_sm = e ? std::max(1, std::atoi(e)) : 6;
    LAUNCH(c, "dia", (12.0 + 8.0 * (K + 1) + 1.0) * A.n + 8.0 * A.nnz, k_dia_values,
           grid_for(A.n, 256, static_cast<int64_t>(c.num_sms) * per_sm), 256, 0, A, dia_off(K, off), mask, dia, flag);
}

}  // namespace amgr

// Setup kernels (sm_100a).  Sorting and prefix sums of the one-time setup use
// CUB's device primitives; everything else — the strength test, the exact
// aggregation replay, P/R and the Galerkin plan construction — is hand-written.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "reduce.cuh"
#include "setup.cuh"

namespace amgr {

namespace {

constexpr int SB = 256;

int bits_for(int64_t n) {
    int b = 1;
    while ((int64_t{1} << b) < n) ++b;
    return b;
}

template <class T>
void exclusive_sum(Ctx& c, const T* in, T* out, int64_t n) {
    if (n <= 0) return;
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c.stream));
    DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
    CK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, c.stream));
    ++c.launches;
}

// Stable LSD radix sort of (key, value) pairs on the low end_bit bits.
// Returns pointers to the sorted arrays (one of the two buffers).
void sort_pairs(Ctx& c, uint64_t* k0, uint64_t* k1, int* v0, int* v1, int64_t n, int end_bit,
                uint64_t** ko, int** vo) {
    cub::DoubleBuffer<uint64_t> kb(k0, k1);
    cub::DoubleBuffer<int> vb(v0, v1);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, n, 0, end_bit, c.stream));
    DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
    CK(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kb, vb, n, 0, end_bit, c.stream));
    c.launches += 1;
    *ko = kb.Current();
    *vo = vb.Current();
}

void sort_keys(Ctx& c, uint64_t* k0, uint64_t* k1, int64_t n, int end_bit, uint64_t** ko) {
    cub::DoubleBuffer<uint64_t> kb(k0, k1);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kb, n, 0, end_bit, c.stream));
    DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
    CK(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, kb, n, 0, end_bit, c.stream));
    c.launches += 1;
    *ko = kb.Current();
}

#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n); \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void k_bad_diag(CsrView A, const int* dpos, int* bad) {
    GRID_STRIDE(i, A.n) {
        const int k = dpos[i];
        if (k < 0 || A.val[k] == 0.0) atomicMin(bad, static_cast<int>(i));
    }
}

// coarsening.cpp:36-46: edge iff j != i and v*v > eps2*|d_i*d_j|, both directions.
__global__ void k_strong_count(CsrView A, const int* dpos, double eps2, int64_t* cnt) {
    GRID_STRIDE(i, A.n) {
        const double di = A.val[dpos[i]];
        int64_t c = 0;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int j = A.col[k];
            if (j == i) continue;
            const double v = A.val[k];
            const double dj = A.val[dpos[j]];
            if (__dmul_rn(v, v) > __dmul_rn(eps2, fabs(__dmul_rn(di, dj)))) c += 2;
        }
        cnt[i] = c;
    }
}

__global__ void k_strong_emit(CsrView A, const int* dpos, double eps2, const int64_t* off, int b,
                              uint64_t* keys) {
    GRID_STRIDE(i, A.n) {
        const double di = A.val[dpos[i]];
        int64_t o = off[i];
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int j = A.col[k];
            if (j == i) continue;
            const double v = A.val[k];
            const double dj = A.val[dpos[j]];
            if (__dmul_rn(v, v) > __dmul_rn(eps2, fabs(__dmul_rn(di, dj)))) {
                keys[o++] = (static_cast<uint64_t>(i) << b) | static_cast<uint64_t>(j);
                keys[o++] = (static_cast<uint64_t>(j) << b) | static_cast<uint64_t>(i);
            }
        }
    }
}

__global__ void k_heads(const uint64_t* keys, int64_t m, int64_t* head) {
    GRID_STRIDE(p, m) head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

__global__ void k_compact_keys(const uint64_t* keys, const int64_t* head, const int64_t* pos, int64_t m,
                               uint64_t* out) {
    GRID_STRIDE(p, m) if (head[p]) out[pos[p]] = keys[p];
}

// ptr[i] = lower_bound(ukeys, i << b); adj = low bits
__global__ void k_graph_ptr(const uint64_t* ukeys, int64_t m, int64_t n, int b, int* ptr) {
    GRID_STRIDE(i, n + 1) {
        const uint64_t target = static_cast<uint64_t>(i) << b;
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        ptr[i] = static_cast<int>(lo);
    }
}
__global__ void k_graph_adj(const uint64_t* ukeys, int64_t m, uint64_t mask, int* adj) {
    GRID_STRIDE(p, m) adj[p] = static_cast<int>(ukeys[p] & mask);
}

// ---- aggregation replay ------------------------------------------------------
// state: 0 undecided, 1 root, 2 non-root.  Node i is a pass-1 root iff
//  (a) no root among its lower-indexed neighbours, and
//  (b) some neighbour j > i has no root in N(j) ∩ [0, i)
// (DESIGN.md §3.2).  Decisions are final, so reading states
// written by other threads in the same round is safe.
__device__ __forceinline__ int ld_state(const int* s, int i) {
    return *reinterpret_cast<const volatile int*>(s + i);
}

// One round over the current list of undecided nodes (compacted between
// batches of rounds, so late rounds touch only the few nodes still open).
__global__ void __launch_bounds__(SB) k_agg_round(const int* __restrict__ nact, const int* __restrict__ act,
                                                  const int* __restrict__ ptr, const int* __restrict__ adj,
                                                  int* state, int* undecided) {
    int local = 0;
    const int na = *nact;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < na; t += gridDim.x * blockDim.x) {
        const int i = act[t];
        if (ld_state(state, i) != 0) continue;
        const int p0 = ptr[i], p1 = ptr[i + 1];
        if (p0 == p1) {  // isolated: never a pass-1 root
            reinterpret_cast<volatile int*>(state)[i] = 2;
            continue;
        }
        int decision = 0;
        bool blocked = false;
        int p = p0;
        for (; p < p1; ++p) {
            const int j = adj[p];
            if (j > i) break;
            const int s = ld_state(state, j);
            if (s == 1) {
                decision = 2;
                break;
            }
            if (s == 0) blocked = true;
        }
        if (decision == 0 && !blocked) {
            bool unknown = false, free_found = false;
            for (int q = p; q < p1 && !free_found; ++q) {
                const int j = adj[q];
                bool taken = false, junk = false;
                for (int t = ptr[j]; t < ptr[j + 1]; ++t) {
                    const int x = adj[t];
                    if (x >= i) break;
                    const int s = ld_state(state, x);
                    if (s == 1) {
                        taken = true;
                        break;
                    }
                    if (s == 0) junk = true;
                }
                if (!taken && !junk) free_found = true;
                else if (!taken) unknown = true;
            }
            if (free_found) decision = 1;
            else if (!unknown) decision = 2;
        }
        if (decision) reinterpret_cast<volatile int*>(state)[i] = decision;
        else ++local;
    }
    // block-aggregate the undecided count
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    if (local) atomicAdd(&s_cnt, local);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) atomicAdd(undecided, s_cnt);
}

// Decision of one undecided node from the current states (0: not yet
// determinable).  Same rule as k_agg_round.
__device__ __forceinline__ int agg_decide(int i, const int* __restrict__ ptr, const int* __restrict__ adj,
                                          const int* state) {
    const int p0 = ptr[i], p1 = ptr[i + 1];
    if (p0 == p1) return 2;  // isolated: never a pass-1 root
    bool blocked = false;
    int p = p0;
    for (; p < p1; ++p) {
        const int j = adj[p];
        if (j > i) break;
        const int s = ld_state(state, j);
        if (s == 1) return 2;
        if (s == 0) blocked = true;
    }
    if (blocked) return 0;
    bool unknown = false;
    for (int q = p; q < p1; ++q) {
        const int j = adj[q];
        bool taken = false, junk = false;
        for (int t = ptr[j]; t < ptr[j + 1]; ++t) {
            const int x = adj[t];
            if (x >= i) break;
            const int s = ld_state(state, x);
            if (s == 1) {
                taken = true;
                break;
            }
            if (s == 0) junk = true;
        }
        if (!taken && !junk) return 1;
        if (!taken) unknown = true;
    }
    return unknown ? 0 : 2;
}

// Persistent replay: every thread walks its nodes i = t, t+T, ... in
// ascending order and waits on each until it is determinable.  The lowest
// undecided node of the graph only depends on decided nodes, and its owner
// is waiting on exactly that node (its earlier nodes are lower, hence
// decided), so the sweep always progresses provided all threads are resident
// (cooperative launch).  Decisions are final, so the states reached are the
// rounds' fixed point; the chain of dependent decisions costs one L2 round
// trip per link instead of one kernel launch per round.
__global__ void k_agg_persistent(int n, const int* __restrict__ ptr, const int* __restrict__ adj, int* state,
                                 int* stuck) {
    const int T = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) {
        int d;
        unsigned spins = 0;
        while ((d = agg_decide(i, ptr, adj, state)) == 0) {
            // the chain can be ~3g links long; a node that stays undetermined
            // for ~seconds means a broken invariant: report instead of hanging
            if (++spins > (1u << 24) || *reinterpret_cast<volatile int*>(stuck)) {
                atomicExch(stuck, 1);
                return;
            }
            __nanosleep(64);
        }
        reinterpret_cast<volatile int*>(state)[i] = d;
    }
}

__global__ void k_iota_list(int n, int* act, int* nact) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) act[i] = i;
    if (blockIdx.x == 0 && threadIdx.x == 0) *nact = n;
}

// keep the still-undecided nodes (order irrelevant: decisions are final and
// depend only on neighbour states)
__global__ void k_compact_list(const int* __restrict__ nact, const int* __restrict__ act, const int* state,
                               int* nact2, int* act2) {
    const int na = *nact;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < na; t += gridDim.x * blockDim.x) {
        const int i = act[t];
        if (ld_state(state, i) == 0) act2[atomicAdd(nact2, 1)] = i;
    }
}

__global__ void k_root_flags(const int* state, int64_t n, int64_t* rf) {
    GRID_STRIDE(i, n) rf[i] = state[i] == 1 ? 1 : 0;
}

// pass 1: roots take their id; absorbed nodes take the id of their
// lowest-indexed root neighbour; -2 isolated, -1 pass-2 leftover.
__global__ void k_assign1(int64_t n, const int* ptr, const int* adj, const int* state, const int64_t* rid,
                          int* agg, int64_t* iso) {
    GRID_STRIDE(i, n) {
        int a = -1;
        int64_t is = 0;
        if (state[i] == 1) {
            a = static_cast<int>(rid[i]);
        } else if (ptr[i] == ptr[i + 1]) {
            a = -2;
            is = 1;
        } else {
            for (int p = ptr[i]; p < ptr[i + 1]; ++p) {
                const int j = adj[p];
                if (state[j] == 1) {
                    a = static_cast<int>(rid[j]);
                    break;
                }
            }
        }
        agg[i] = a;
        iso[i] = is;
    }
}

// pass 2 (coarsening.cpp:103-116): isolated -> new singleton ids after all
// roots in ascending order; leftover -> aggregate of the lowest-indexed
// neighbour (always assigned in pass 1).
__global__ void k_assign2(int64_t n, const int* ptr, const int* adj, int64_t n_roots, const int64_t* isorank,
                          int* agg, int* err) {
    GRID_STRIDE(i, n) {
        const int a = agg[i];
        if (a == -2) {
            agg[i] = static_cast<int>(n_roots + isorank[i]);
        } else if (a == -1) {
            const int j = adj[ptr[i]];
            const int aj = agg[j];
            if (aj < 0) *err = 1;
            agg[i] = aj;
        }
    }
}

__global__ void k_hist(const int* agg, int64_t n, int* cnt) {
    GRID_STRIDE(i, n) atomicAdd(cnt + agg[i], 1);
}
__global__ void k_iota(int* v, int64_t n) {
    GRID_STRIDE(i, n) v[i] = static_cast<int>(i);
}
__global__ void k_agg_keys(const int* agg, int64_t n, uint64_t* k) {
    GRID_STRIDE(i, n) k[i] = static_cast<uint64_t>(agg[i]);
}
__global__ void k_i64_to_i32(const int64_t* s, int* d, int64_t n) {
    GRID_STRIDE(i, n) d[i] = static_cast<int>(s[i]);
}

// ---- symbolic RAP -------------------------------------------------------------
__global__ void k_rap_keys(CsrView A, const int* agg, int b, uint64_t* keys, int* vals, int* rowof) {
    GRID_STRIDE(i, A.n) {
        const uint64_t I = static_cast<uint64_t>(agg[i]) << b;
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            keys[k] = I | static_cast<uint64_t>(agg[A.col[k]]);
            vals[k] = k;
            rowof[k] = static_cast<int>(i);
        }
    }
}
__global__ void k_rap_plan(const uint64_t* keys, const int* vals, const int* rowof, const int64_t* head,
                           const int64_t* pos, int64_t m, int* contrib, int* cptr, uint64_t* ukeys) {
    GRID_STRIDE(p, m) {
        const int e = vals[p];
        bool last = true;
        if (p + 1 < m && keys[p + 1] == keys[p] && rowof[vals[p + 1]] == rowof[e]) last = false;
        contrib[p] = last ? (e | static_cast<int>(0x80000000u)) : e;
        if (head[p]) {
            cptr[pos[p]] = static_cast<int>(p);
            ukeys[pos[p]] = keys[p];
        }
    }
}
// coarse columns; bit 30 of cptr flags the diagonal entries (the numeric RAP
// fuses the coarse Jacobi rebuild there, kernels.cuh RapJacobi)
__global__ void k_coarse_col(const uint64_t* ukeys, int64_t nnz_c, uint64_t mask, int b, int* col, int* cptr) {
    GRID_STRIDE(c, nnz_c) {
        const int J = static_cast<int>(ukeys[c] & mask);
        col[c] = J;
        if (static_cast<int>(ukeys[c] >> b) == J) cptr[c] |= (1 << 30);
    }
}
__global__ void k_set_int(int* p, int v) { *p = v; }

}  // namespace

int64_t first_bad_diag(Ctx& c, const CsrView& A, const int* dpos) {
    DevArray<int> bad(1, c.stream);
    const int big = 0x7fffffff;
    h2d(bad.get(), &big, 1, c.stream);
    LAUNCH(c, "setup", 0.0, k_bad_diag, grid_for(A.n, SB, c.num_sms * 16), SB, 0, A, dpos, bad.get());
    const int r = d2h_scalar(bad.get(), c.stream);
    return r == big ? -1 : r;
}

void strength_graph(Ctx& c, const CsrView& A, const int* dpos, double eps2, GraphDev& g) {
    const int64_t n = A.n;
    const int b = bits_for(n);
    DevArray<int64_t> cnt(n + 1, c.stream), off(n + 1, c.stream);
    CK(cudaMemsetAsync(cnt.get(), 0, sizeof(int64_t) * (n + 1), c.stream));
    LAUNCH(c, "setup", 0.0, k_strong_count, grid_for(n, SB, c.num_sms * 16), SB, 0, A, dpos, eps2, cnt.get());
    exclusive_sum(c, cnt.get(), off.get(), n + 1);
    const int64_t m2 = d2h_scalar(off.get() + n, c.stream);
    g.n = n;
    g.ptr.alloc(n + 1, c.stream);
    if (m2 == 0) {
        CK(cudaMemsetAsync(g.ptr.get(), 0, sizeof(int) * (n + 1), c.stream));
        g.m = 0;
        g.adj.alloc(1, c.stream);
        return;
    }
    DevArray<uint64_t> k0(m2, c.stream), k1(m2, c.stream);
    LAUNCH(c, "setup", 0.0, k_strong_emit, grid_for(n, SB, c.num_sms * 16), SB, 0, A, dpos, eps2, off.get(), b,
           k0.get());
    uint64_t* ks = nullptr;
    sort_keys(c, k0.get(), k1.get(), m2, 2 * b, &ks);
    DevArray<int64_t> head(m2, c.stream), pos(m2, c.stream);
    LAUNCH(c, "setup", 0.0, k_heads, grid_for(m2, SB, c.num_sms * 16), SB, 0, ks, m2, head.get());
    exclusive_sum(c, head.get(), pos.get(), m2);
    const int64_t m = d2h_scalar(pos.get() + m2 - 1, c.stream) + d2h_scalar(head.get() + m2 - 1, c.stream);
    uint64_t* other = (ks == k0.get()) ? k1.get() : k0.get();
    LAUNCH(c, "setup", 0.0, k_compact_keys, grid_for(m2, SB, c.num_sms * 16), SB, 0, ks, head.get(), pos.get(), m2,
           other);
    g.m = m;
    g.adj.alloc(m, c.stream);
    LAUNCH(c, "setup", 0.0, k_graph_ptr, grid_for(n + 1, SB, c.num_sms * 16), SB, 0, other, m, n, b, g.ptr.get());
    LAUNCH(c, "setup", 0.0, k_graph_adj, grid_for(m, SB, c.num_sms * 16), SB, 0, other, m,
           (uint64_t{1} << b) - 1, g.adj.get());
}

int64_t aggregate(Ctx& c, const GraphDev& g, DevArray<int>& agg, int64_t* rounds) {
    const int64_t n = g.n;
    DevArray<int> state(n, c.stream);
    CK(cudaMemsetAsync(state.get(), 0, sizeof(int) * n, c.stream));
    constexpr int BATCH = 16;
    DevArray<int> cnt(BATCH, c.stream);
    DevArray<int> list0(n, c.stream), list1(n, c.stream), nl(2, c.stream);
    int *act = list0.get(), *act2 = list1.get(), *nact = nl.get(), *nact2 = nl.get() + 1;
    int64_t r = 0;
    const unsigned grid = grid_for(n, SB, c.num_sms * 8);
    const char* pe = std::getenv("AMGR_AGG_PERSISTENT");
    const bool persistent = !(pe && pe[0] == '0');
    if (persistent) {
        static const int per_sm = [] {
            int b = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_agg_persistent, SB, 0));
            return b;
        }();
        int64_t blocks = (n + SB - 1) / SB;
        const int64_t cap = static_cast<int64_t>(c.num_sms) * per_sm;
        if (blocks > cap) blocks = cap;
        int nn = static_cast<int>(n);
        const int* pp = g.ptr.get();
        const int* aa = g.adj.get();
        int* ss = state.get();
        DevArray<int> stuck(1, c.stream);
        CK(cudaMemsetAsync(stuck.get(), 0, sizeof(int), c.stream));
        int* st = stuck.get();
        void* args[] = {&nn, &pp, &aa, &ss, &st};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_agg_persistent),
                                       dim3(static_cast<unsigned>(blocks)), dim3(SB), args, 0, c.stream));
        ++c.launches;
        if (d2h_scalar(stuck.get(), c.stream)) fail(AMGR_E_RUNTIME, "aggregate: persistent replay made no progress");
        r = 1;
    }
    if (!persistent) LAUNCH(c, "setup", 0.0, k_iota_list, grid, SB, 0, static_cast<int>(n), act, nact);
    while (!persistent) {
        CK(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * BATCH, c.stream));
        for (int k = 0; k < BATCH; ++k)
            LAUNCH(c, "setup", 0.0, k_agg_round, grid, SB, 0, nact, act, g.ptr.get(), g.adj.get(), state.get(),
                   cnt.get() + k);
        r += BATCH;
        int h[BATCH];
        d2h(h, cnt.get(), BATCH, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        int done_at = -1;
        for (int k = 0; k < BATCH; ++k)
            if (h[k] == 0) {
                done_at = k;
                break;
            }
        if (done_at >= 0) {
            r = r - BATCH + done_at + 1;
            break;
        }
        CK(cudaMemsetAsync(nact2, 0, sizeof(int), c.stream));
        LAUNCH(c, "setup", 0.0, k_compact_list, grid, SB, 0, nact, act, state.get(), nact2, act2);
        std::swap(act, act2);
        std::swap(nact, nact2);
    }
    if (rounds) *rounds = r;

    DevArray<int64_t> rf(n + 1, c.stream), rid(n + 1, c.stream), iso(n + 1, c.stream), isor(n + 1, c.stream);
    CK(cudaMemsetAsync(rf.get() + n, 0, sizeof(int64_t), c.stream));
    LAUNCH(c, "setup", 0.0, k_root_flags, grid_for(n, SB, c.num_sms * 16), SB, 0, state.get(), n, rf.get());
    exclusive_sum(c, rf.get(), rid.get(), n + 1);
    const int64_t n_roots = d2h_scalar(rid.get() + n, c.stream);
    agg.alloc(n, c.stream);
    CK(cudaMemsetAsync(iso.get() + n, 0, sizeof(int64_t), c.stream));
    LAUNCH(c, "setup", 0.0, k_assign1, grid_for(n, SB, c.num_sms * 16), SB, 0, n, g.ptr.get(), g.adj.get(),
           state.get(), rid.get(), agg.get(), iso.get());
    exclusive_sum(c, iso.get(), isor.get(), n + 1);
    const int64_t n_iso = d2h_scalar(isor.get() + n, c.stream);
    DevArray<int> err(1, c.stream);
    CK(cudaMemsetAsync(err.get(), 0, sizeof(int), c.stream));
    LAUNCH(c, "setup", 0.0, k_assign2, grid_for(n, SB, c.num_sms * 16), SB, 0, n, g.ptr.get(), g.adj.get(), n_roots,
           isor.get(), agg.get(), err.get());
    if (d2h_scalar(err.get(), c.stream)) fail(AMGR_E_RUNTIME, "aggregate: internal error (unassigned neighbour)");
    return n_roots + n_iso;
}

void members(Ctx& c, int64_t nf, int64_t nc, const int* agg, DevArray<int>& mptr, DevArray<int>& midx) {
    const int b = bits_for(nc);
    DevArray<int> cnt(nc + 1, c.stream);
    CK(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * (nc + 1), c.stream));
    LAUNCH(c, "setup", 0.0, k_hist, grid_for(nf, SB, c.num_sms * 16), SB, 0, agg, nf, cnt.get());
    mptr.alloc(nc + 1, c.stream);
    exclusive_sum(c, cnt.get(), mptr.get(), nc + 1);
    DevArray<uint64_t> k0(nf, c.stream), k1(nf, c.stream);
    DevArray<int> v0(nf, c.stream), v1(nf, c.stream);
    LAUNCH(c, "setup", 0.0, k_agg_keys, grid_for(nf, SB, c.num_sms * 16), SB, 0, agg, nf, k0.get());
    LAUNCH(c, "setup", 0.0, k_iota, grid_for(nf, SB, c.num_sms * 16), SB, 0, v0.get(), nf);
    uint64_t* ko;
    int* vo;
    sort_pairs(c, k0.get(), k1.get(), v0.get(), v1.get(), nf, b, &ko, &vo);
    midx.alloc(nf, c.stream);
    d2d(midx.get(), vo, nf, c.stream);
}

void rap_symbolic(Ctx& c, const CsrView& A, const int* agg, int64_t nc, RapSymbolic& out) {
    const int64_t m = A.nnz;
    const int b = bits_for(nc);
    const uint64_t mask = (uint64_t{1} << b) - 1;
    out.contrib.alloc(m, c.stream);
    DevArray<uint64_t> k0(m, c.stream), k1(m, c.stream);
    DevArray<int> v0(m, c.stream), v1(m, c.stream), rowof(m, c.stream);
    LAUNCH(c, "setup", 0.0, k_rap_keys, grid_for(A.n, SB, c.num_sms * 16), SB, 0, A, agg, b, k0.get(), v0.get(),
           rowof.get());
    uint64_t* ks;
    int* vs;
    sort_pairs(c, k0.get(), k1.get(), v0.get(), v1.get(), m, 2 * b, &ks, &vs);
    DevArray<int64_t> head(m, c.stream), pos(m, c.stream);
    LAUNCH(c, "setup", 0.0, k_heads, grid_for(m, SB, c.num_sms * 16), SB, 0, ks, m, head.get());
    exclusive_sum(c, head.get(), pos.get(), m);
    const int64_t nnz_c = d2h_scalar(pos.get() + m - 1, c.stream) + d2h_scalar(head.get() + m - 1, c.stream);
    out.nnz_c = nnz_c;
    out.cptr.alloc(nnz_c + 1, c.stream);
    uint64_t* ukeys = (ks == k0.get()) ? k1.get() : k0.get();
    LAUNCH(c, "setup", 0.0, k_rap_plan, grid_for(m, SB, c.num_sms * 16), SB, 0, ks, vs, rowof.get(), head.get(),
           pos.get(), m, out.contrib.get(), out.cptr.get(), ukeys);
    LAUNCH(c, "setup", 0.0, k_set_int, 1, 1, 0, out.cptr.get() + nnz_c, static_cast<int>(m));
    out.col.alloc(nnz_c, c.stream);
    if (m >= (int64_t{1} << 30)) invalid("galerkin plan: more than 2^30 fine entries per GPU");
    LAUNCH(c, "setup", 0.0, k_coarse_col, grid_for(nnz_c, SB, c.num_sms * 16), SB, 0, ukeys, nnz_c, mask, b,
           out.col.get(), out.cptr.get());
    out.rp.alloc(nc + 1, c.stream);
    LAUNCH(c, "setup", 0.0, k_graph_ptr, grid_for(nc + 1, SB, c.num_sms * 16), SB, 0, ukeys, nnz_c, nc, b,
           out.rp.get());
}

__global__ void k_rr_members(int64_t nf, const int* __restrict__ rp, const int* __restrict__ midx, int* mrp,
                             uint8_t* mlen, int* maxlen) {
    int mx = 0;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < nf;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int m = midx[j];
        const int a = rp[m], len = rp[m + 1] - a;
        mrp[j] = a;
        mlen[j] = static_cast<uint8_t>(len < 255 ? len : 255);
        mx = max(mx, len);
    }
    atomicMax(maxlen, mx);
}

__global__ void k_rr_dmax(int64_t nc, const int* __restrict__ crp, int* dmax) {
    int mx = 0;
    for (int64_t I = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; I < nc;
         I += static_cast<int64_t>(gridDim.x) * blockDim.x)
        mx = max(mx, crp[I + 1] - crp[I]);
    atomicMax(dmax, mx);
}

// thread per fine row: slots of its entries in coarse row agg[m], then a
// stable insertion sort by slot gives the accumulation order
__global__ void k_rr_code(CsrView A, const int* __restrict__ agg, const int* __restrict__ crp,
                          const int* __restrict__ ccol, uint16_t* __restrict__ code, int* bad) {
    for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m < A.n;
         m += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int e0 = A.rp[m], len = A.rp[m + 1] - e0;
        if (len > 32) {
            atomicOr(bad, 1);
            continue;
        }
        const int I = agg[m];
        const int c0 = crp[I], deg = crp[I + 1] - c0;
        if (deg > 511) {
            atomicOr(bad, 2);
            continue;
        }
        int slot[32], ord[32];
        for (int k = 0; k < len; ++k) {
            const int J = agg[A.col[e0 + k]];
            int lo = 0, hi = deg;  // lower_bound of J in ccol[c0, c0 + deg)
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (ccol[c0 + mid] < J) lo = mid + 1; else hi = mid;
            }
            if (lo >= deg || ccol[c0 + lo] != J) atomicOr(bad, 4);
            slot[k] = lo;
            int t = k;
            while (t > 0 && slot[ord[t - 1]] > lo) {
                ord[t] = ord[t - 1];
                --t;
            }
            ord[t] = k;
        }
        for (int t = 0; t < len; ++t) {
            const int k = ord[t];
            const int sl = slot[k];
            const bool last = t + 1 == len || slot[ord[t + 1]] != sl;
            const bool dg = A.col[e0 + k] == m;
            code[e0 + t] = static_cast<uint16_t>(k | (last ? 32 : 0) | (dg ? 64 : 0) | (sl << 7));
        }
    }
}

void rap_rows_plan(Ctx& c, const CsrView& A, const int* agg, const int* midx, int64_t nc, const int* crp,
                   const int* ccol, RowPlan& plan) {
    plan.ok = false;
    if (A.n == 0 || nc == 0) return;
    DevArray<int> st(3, c.stream);
    CK(cudaMemsetAsync(st.get(), 0, 3 * sizeof(int), c.stream));
    plan.mrp.alloc(A.n, c.stream);
    plan.mlen.alloc(A.n, c.stream);
    LAUNCH(c, "setup", 0.0, k_rr_members, grid_for(A.n, SB, c.num_sms * 16), SB, 0, A.n, A.rp, midx,
           plan.mrp.get(), plan.mlen.get(), st.get());
    LAUNCH(c, "setup", 0.0, k_rr_dmax, grid_for(nc, SB, c.num_sms * 16), SB, 0, nc, crp, st.get() + 1);
    int h[3];
    d2h(h, st.get(), 2, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    plan.maxlen = h[0];
    plan.dmax = h[1];
    if (plan.maxlen > 32 || plan.dmax > 511) {
        plan.mrp.release();
        plan.mlen.release();
        return;
    }
    plan.code.alloc(A.nnz + 8, c.stream);
    LAUNCH(c, "setup", 0.0, k_rr_code, grid_for(A.n, 128, c.num_sms * 16), 128, 0, A, agg, crp, ccol,
           plan.code.get(), st.get() + 2);
    const int bad = d2h_scalar(st.get() + 2, c.stream);
    if (bad) fail(AMGR_E_RUNTIME, "rap_rows_plan: inconsistent coarse pattern (internal error)");
    plan.ok = true;
}

// ---- warp-group Galerkin plan (k_rap_grp) ------------------------------------
namespace {
constexpr int GP_BUF = GRP_BUF - 1, GP_MEM = 64;
constexpr int GP_MASK = (1 << 30) - 1;  // cptr bit 30 flags the coarse diagonal

// group of coarse row I: the last group whose first row is <= I
__device__ __forceinline__ int64_t gp_group_of(const int4* desc, int64_t ngroups, int64_t I) {
    int64_t lo = 0, hi = ngroups;  // answer in [0, ngroups)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (desc[mid].x <= I) lo = mid; else hi = mid;
    }
    return lo;
}
// flag[I] = coarse row I starts a group: chunk starts always, then the
// greedy rule (the group [g0, I+1) would exceed the buffer or member bound)
__global__ void k_gp_greedy(int64_t nc, int64_t chunk, const int* __restrict__ pb, const int* __restrict__ mptr,
                            char* flag) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t a = t * chunk;
    if (a >= nc) return;
    const int64_t b = a + chunk < nc ? a + chunk : nc;
    int p0 = pb[a], m0 = mptr[a];
    flag[a] = 1;
    for (int64_t I = a + 1; I < b; ++I) {
        const int pe = pb[I + 1], me = mptr[I + 1];
        const bool cut = pe - p0 > GP_BUF || me - m0 > GP_MEM;
        flag[I] = cut ? 1 : 0;
        if (cut) {
            p0 = pb[I];
            m0 = mptr[I];
        }
    }
}
__global__ void k_set_i32(int* p, int v) { *p = v; }
__global__ void k_gp_pb(int64_t nc, const int* __restrict__ crp, const int* __restrict__ cptr, int* pb) {
    for (int64_t I = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; I <= nc;
         I += static_cast<int64_t>(gridDim.x) * blockDim.x)
        pb[I] = cptr[crp[I]] & GP_MASK;
}

// st[0]: longest member row
__global__ void k_gp_members(int64_t nf, const int* __restrict__ rp, const int* __restrict__ midx,
                             const int* __restrict__ dpos, int* mstart, uint8_t* mdoff, int* st) {
    int mx = 0;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < nf;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int m = midx[j];
        const int a = rp[m], len = rp[m + 1] - a, d = dpos[m];
        mstart[j] = a;
        mdoff[j] = static_cast<uint8_t>(d >= a && d - a < 255 ? d - a : 255);
        mx = max(mx, len);
    }
    atomicMax(st, mx);
}
// st[1]: largest coarse row (contributions), st[2]: most members of a coarse row
__global__ void k_gp_rows(int64_t nc, const int* __restrict__ crp, const int* __restrict__ cptr,
                          const int* __restrict__ mptr, int* st) {
    int mr = 0, mm = 0;
    for (int64_t I = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; I < nc;
         I += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        mr = max(mr, (cptr[crp[I + 1]] & GP_MASK) - (cptr[crp[I]] & GP_MASK));
        mm = max(mm, mptr[I + 1] - mptr[I]);
    }
    atomicMax(st + 1, mr);
    atomicMax(st + 2, mm);
}
__global__ void k_gp_desc(int64_t ngroups, const int* __restrict__ first, const int* __restrict__ crp,
                          const int* __restrict__ cptr, const int* __restrict__ mptr, int4* desc) {
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g <= ngroups;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int I = first[g];
        const int c0 = crp[I];
        desc[g] = make_int4(I, mptr[I], c0, cptr[c0] & GP_MASK);
    }
}
// st[3]: most contributions of a group, st[4]: most members of a group (checks)
__global__ void k_gp_check(int64_t ngroups, const int4* __restrict__ desc, int* st) {
    int mb = 0, mm = 0;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < ngroups;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        mb = max(mb, desc[g + 1].w - desc[g].w);
        mm = max(mm, desc[g + 1].y - desc[g].y);
    }
    atomicMax(st + 3, mb);
    atomicMax(st + 4, mm);
}
// per fine entry: its offset in the member row | the member's number in its
// group << 8 (thread per coarse row I: its members j in R order)
__global__ void k_gp_emap(int64_t nc, const int* __restrict__ mptr, const int* __restrict__ midx,
                          const int* __restrict__ rp, int64_t ngroups, const int4* __restrict__ desc,
                          uint16_t* emap) {
    for (int64_t I = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; I < nc;
         I += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t g = gp_group_of(desc, ngroups, I);
        const int m0 = desc[g].y;
        for (int j = mptr[I]; j < mptr[I + 1]; ++j) {
            const int i = midx[j];
            const int loc = j - m0;
            for (int e = rp[i]; e < rp[i + 1]; ++e) emap[e] = static_cast<uint16_t>((e - rp[i]) | (loc << 8));
        }
    }
}
__global__ void k_gp_code(int64_t m, const int* __restrict__ contrib, const uint16_t* __restrict__ emap,
                          uint16_t* code) {
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int e = contrib[p];
        code[p] = static_cast<uint16_t>(emap[e & 0x7fffffff] | (e < 0 ? 0x8000 : 0));
    }
}
__global__ void k_gp_entry_start(int64_t nnz_c, const int* __restrict__ cptr, uint16_t* code) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nnz_c;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        code[cptr[q] & GP_MASK] |= 0x4000;
}
// per group: split its coarse entries into <= 32 contiguous runs of at most
// L contributions (L = the smallest bound >= max(ceil(nbuf / 32), longest
// entry) for which greedy cutting needs <= 32 runs); lane k's run starts at
// contribution (low byte) and entry (high byte) of lanes[32 g + k]
__global__ void k_gp_lanes(int64_t ngroups, const int4* __restrict__ desc, const int* __restrict__ cptr,
                           uint16_t* lanes) {
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < ngroups;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int4 d0 = desc[g], d1 = desc[g + 1];
        const int nent = d1.z - d0.z, nbuf = d1.w - d0.w;
        int longest = 0;
        for (int q = 0; q < nent; ++q)
            longest = max(longest, (cptr[d0.z + q + 1] & GP_MASK) - (cptr[d0.z + q] & GP_MASK));
        int L = max((nbuf + 31) / 32, longest);
        for (;; ++L) {
            int runs = 0, cur = L + 1;
            for (int q = 0; q < nent; ++q) {
                const int k = (cptr[d0.z + q + 1] & GP_MASK) - (cptr[d0.z + q] & GP_MASK);
                if (cur + k > L) {
                    ++runs;
                    cur = 0;
                }
                cur += k;
            }
            if (runs <= 32) break;
        }
        uint16_t* out = lanes + g * 32;
        int lane = 0, cur = L + 1;
        for (int q = 0; q < nent; ++q) {
            const int p = (cptr[d0.z + q] & GP_MASK) - d0.w;
            const int k = (cptr[d0.z + q + 1] & GP_MASK) - (cptr[d0.z + q] & GP_MASK);
            if (cur + k > L) {
                out[lane++] = static_cast<uint16_t>(p | (q << 8));
                cur = 0;
            }
            cur += k;
        }
        for (; lane < 32; ++lane) out[lane] = static_cast<uint16_t>(nbuf | (nent << 8));
    }
}
}  // namespace

void rap_grp_plan(Ctx& c, const CsrView& A, const int* mptr, const int* midx, const int* dpos, int64_t nc,
                  const int* crp, int64_t nnz_c, const int* cptr, const int* contrib, GrpPlan& plan) {
    plan = GrpPlan{};
    const int64_t nf = A.n, m = A.nnz;
    if (nf == 0 || nc == 0 || nnz_c == 0 || m >= (int64_t{1} << 30)) return;
    DevArray<int> st(5, c.stream);
    CK(cudaMemsetAsync(st.get(), 0, 5 * sizeof(int), c.stream));
    plan.mstart.alloc(nf + 8, c.stream);  // + slack: k_rap_grp's 16-byte bulk-copy windows
    plan.mdoff.alloc(nf + 16, c.stream);
    LAUNCH(c, "setup", 0.0, k_gp_members, grid_for(nf, SB, c.num_sms * 16), SB, 0, nf, A.rp, midx, dpos,
           plan.mstart.get(), plan.mdoff.get(), st.get());
    LAUNCH(c, "setup", 0.0, k_gp_rows, grid_for(nc, SB, c.num_sms * 16), SB, 0, nc, crp, cptr, mptr, st.get());
    int h[5];
    d2h(h, st.get(), 3, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    // member rows <= 255 entries (8-bit offsets), every coarse row fits a
    // group (<= 256 contributions, <= 64 members)
    if (h[0] > 255 || h[1] > GP_BUF || h[2] > GP_MEM) {
        plan = GrpPlan{};
        return;
    }
    // greedy packing of consecutive coarse rows, on the device: the rows are
    // cut into chunks (one thread each) that always start a group, and each
    // thread packs its chunk greedily (a few % more groups than one global
    // greedy pass; no host round trip of the row arrays)
    DevArray<int> first;
    {
        DevArray<int> pb(nc + 1, c.stream);
        LAUNCH(c, "setup", 0.0, k_gp_pb, grid_for(nc + 1, SB, c.num_sms * 16), SB, 0, nc, crp, cptr, pb.get());
        const int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>(nc, int64_t{c.num_sms} * 64));
        const int64_t chunk = (nc + nchunk - 1) / nchunk;
        DevArray<char> flag(nc, c.stream);
        LAUNCH(c, "setup", 0.0, k_gp_greedy, grid_for(nchunk, 64), 64, 0, nc, chunk, pb.get(), mptr, flag.get());
        DevArray<int> sel(nc, c.stream), nsel(1, c.stream);
        cub::CountingInputIterator<int> it(0);
        size_t bytes = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, bytes, it, flag.get(), sel.get(), nsel.get(), nc, c.stream));
        DevArray<char> tmp(static_cast<int64_t>(std::max<size_t>(bytes, 1)), c.stream);
        CK(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flag.get(), sel.get(), nsel.get(), nc, c.stream));
        ++c.launches;
        plan.ngroups = d2h_scalar(nsel.get(), c.stream);
        first.alloc(plan.ngroups + 1, c.stream);
        d2d(first.get(), sel.get(), plan.ngroups, c.stream);
        LAUNCH(c, "setup", 0.0, k_set_i32, 1, 1, 0, first.get() + plan.ngroups, static_cast<int>(nc));
    }
    {
        plan.desc.alloc(plan.ngroups + 1, c.stream);
        LAUNCH(c, "setup", 0.0, k_gp_desc, grid_for(plan.ngroups + 1, SB, c.num_sms * 16), SB, 0, plan.ngroups,
               first.get(), crp, cptr, mptr, plan.desc.get());
        LAUNCH(c, "setup", 0.0, k_gp_check, grid_for(plan.ngroups, SB, c.num_sms * 16), SB, 0, plan.ngroups,
               plan.desc.get(), st.get());
        d2h(h + 3, st.get() + 3, 2, c.stream);
        CK(cudaStreamSynchronize(c.stream));
    }
    if (h[3] > GP_BUF || h[4] > GP_MEM) fail(AMGR_E_RUNTIME, "rap_grp_plan: group bounds violated (internal error)");
    {
        DevArray<uint16_t> emap(m, c.stream);
        LAUNCH(c, "setup", 0.0, k_gp_emap, grid_for(nc, SB, c.num_sms * 16), SB, 0, nc, mptr, midx, A.rp,
               plan.ngroups, plan.desc.get(), emap.get());
        plan.code.alloc(m + 8, c.stream);
        CK(cudaMemsetAsync(plan.code.get() + m, 0, 8 * sizeof(uint16_t), c.stream));
        LAUNCH(c, "setup", 0.0, k_gp_code, grid_for(m, SB, c.num_sms * 16), SB, 0, m, contrib, emap.get(),
               plan.code.get());
    }
    LAUNCH(c, "setup", 0.0, k_gp_entry_start, grid_for(nnz_c, SB, c.num_sms * 16), SB, 0, nnz_c, cptr,
           plan.code.get());
    plan.lanes.alloc(plan.ngroups * 32, c.stream);
    LAUNCH(c, "setup", 0.0, k_gp_lanes, grid_for(plan.ngroups, 128, c.num_sms * 16), 128, 0, plan.ngroups,
           plan.desc.get(), cptr, plan.lanes.get());
    plan.ok = true;
}

// ---- smoothed aggregation ----------------------------------------------------
// Smoothed aggregation (extension, north star "tentative and
// smoothed prolongator"; the reference ships only the tentative P).  Parity
// is against the restated oracle (oracle/amg_oracle.c:smoothed_prolongator,
// o_spmm, o_transpose, o_galerkin), bit for bit.
//
//  * spgemm_symbolic: C = A B on the device.  Every product a_ik b_kj becomes
//    a triple keyed (i, j); triples are generated in (i, k, B-row) order and
//    stable-radix-sorted by key, so each output entry's products stay in the
//    reference spmm's accumulation order (k ascending, csr.cpp:145-184).  The
//    unique keys are C's structural pattern (sorted columns, cancellation
//    zeros kept); the sorted (a-index, b-index) pairs are the numeric plan.
//  * spgemm_numeric: c_e = sum over the plan of a*b, from 0.0, in plan order
//    (thread per output entry).  With the plan cached, a partial rebuild of a
//    smoothed level is two numeric SpGEMMs: A P (P frozen) then R (A P).
//  * sa_prolongator_values: P = P_tent - (w D^-1) A P_tent on the pattern of
//    A P_tent: v = (J == agg_i ? 1 : 0) - (w * (1/a_ii)) * (A P_tent)_iJ.
//  * transpose: R = P^T with sorted columns (stable sort of P's entries by
//    column keeps the row order), values carried along.
namespace {

constexpr int SA_B = 256;

#define SA_STRIDE(i, n)                                                                    \
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n); \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void k_sp_count(CsrView A, const int* __restrict__ brp, int64_t* cnt) {
    SA_STRIDE(e, A.nnz) {
        const int k = A.col[e];
        cnt[e] = brp[k + 1] - brp[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[A.nnz] = 0;
}

__global__ void k_sp_triples(CsrView A, const int* __restrict__ brp, const int* __restrict__ bcol, int bj,
                             const int64_t* __restrict__ off, uint64_t* __restrict__ key, int* __restrict__ ia,
                             int* __restrict__ ib, int* __restrict__ id) {
    SA_STRIDE(i, A.n) {
        for (int e = A.rp[i]; e < A.rp[i + 1]; ++e) {
            const int k = A.col[e];
            int64_t t = off[e];
            for (int q = brp[k]; q < brp[k + 1]; ++q, ++t) {
                key[t] = (static_cast<uint64_t>(i) << bj) | static_cast<uint64_t>(bcol[q]);
                ia[t] = e;
                ib[t] = q;
                id[t] = static_cast<int>(t);
            }
        }
    }
}

__global__ void k_sp_heads(const uint64_t* keys, int64_t m, int64_t* head) {
    SA_STRIDE(p, m) head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

// unique keys, plan pointer, gathered pairs
__global__ void k_sp_plan(const uint64_t* __restrict__ ks, const int* __restrict__ perm, const int64_t* head,
                          const int64_t* pos, int64_t m, const int* __restrict__ ia, const int* __restrict__ ib,
                          uint64_t* __restrict__ ukeys, int* __restrict__ optr, int* __restrict__ pa,
                          int* __restrict__ pb) {
    SA_STRIDE(p, m) {
        if (head[p]) {
            ukeys[pos[p]] = ks[p];
            optr[pos[p]] = static_cast<int>(p);
        }
        const int t = perm[p];
        pa[p] = ia[t];
        pb[p] = ib[t];
    }
}

__global__ void k_sp_rowptr(const uint64_t* ukeys, int64_t m, int64_t n, int b, int* ptr) {
    SA_STRIDE(i, n + 1) {
        const uint64_t target = static_cast<uint64_t>(i) << b;
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        ptr[i] = static_cast<int>(lo);
    }
}

__global__ void k_sp_col(const uint64_t* ukeys, int64_t m, uint64_t mask, int* col) {
    SA_STRIDE(p, m) col[p] = static_cast<int>(ukeys[p] & mask);
}

__global__ void k_sp_set(int* p, int v) { *p = v; }

__global__ void k_spgemm_num(int64_t nnz, const int* __restrict__ optr, const int* __restrict__ pa,
                             const int* __restrict__ pb, const double* __restrict__ a, const double* __restrict__ b,
                             double* __restrict__ c) {
    SA_STRIDE(e, nnz) {
        double s = 0.0;
        for (int t = optr[e]; t < optr[e + 1]; ++t) s = dadd(s, dmul(a[pa[t]], b[pb[t]]));
        c[e] = s;
    }
}

__global__ void k_tentative(int64_t n, const int* __restrict__ agg, int* rp, int* col, double* val) {
    SA_STRIDE(i, n) {
        rp[i] = static_cast<int>(i);
        col[i] = agg[i];
        val[i] = 1.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) rp[n] = static_cast<int>(n);
}

__global__ void k_sa_values(int64_t n, const int* __restrict__ rp, const int* __restrict__ col, double* v,
                            const int* __restrict__ agg, const int* __restrict__ dpos, const double* __restrict__ aval,
                            double w, int* bad) {
    SA_STRIDE(i, n) {
        const int k = dpos[i];
        const double d = k >= 0 ? aval[k] : 0.0;
        if (k < 0 || d == 0.0) {
            atomicMin(bad, static_cast<int>(i));
            continue;
        }
        const double s = dmul(w, __ddiv_rn(1.0, d));
        const int J = agg[i];
        for (int q = rp[i]; q < rp[i + 1]; ++q) v[q] = dsub(col[q] == J ? 1.0 : 0.0, dmul(s, v[q]));
    }
}

__global__ void k_row_of(int64_t n, const int* __restrict__ rp, int* rowof) {
    SA_STRIDE(i, n) for (int e = rp[i]; e < rp[i + 1]; ++e) rowof[e] = static_cast<int>(i);
}

__global__ void k_tr_keys(int64_t m, const int* __restrict__ col, uint64_t* key, int* id) {
    SA_STRIDE(e, m) {
        key[e] = static_cast<uint64_t>(col[e]);
        id[e] = static_cast<int>(e);
    }
}

__global__ void k_tr_fill(int64_t m, const int* __restrict__ perm, const int* __restrict__ rowof,
                          const double* __restrict__ val, int* tcol, double* tval) {
    SA_STRIDE(p, m) {
        const int e = perm[p];
        tcol[p] = rowof[e];
        tval[p] = val[e];
    }
}

}  // namespace

void spgemm_symbolic(Ctx& c, const CsrView& A, const int* brp, const int* bcol, int64_t bcols, SpgPlan& out,
                     const char* what) {
    const int64_t m = A.nnz;
    DevArray<int64_t> cnt(m + 1, c.stream), off(m + 1, c.stream);
    LAUNCH(c, "setup", 0.0, k_sp_count, grid_for(m > 0 ? m : 1, SA_B, c.num_sms * 16), SA_B, 0, A, brp, cnt.get());
    exclusive_sum(c, cnt.get(), off.get(), m + 1);
    const int64_t T = d2h_scalar(off.get() + m, c.stream);
    if (T >= (int64_t{1} << 31) - 1) {
        std::ostringstream os;
        os << what << ": " << T << " products exceed the 2^31 plan limit of the device SpGEMM";
        fail(AMGR_E_RUNTIME, os.str());
    }
    const int bi = bits_for(A.n), bj = bits_for(bcols);
    DevArray<uint64_t> k0(T, c.stream), k1(T, c.stream);
    DevArray<int> ia(T, c.stream), ib(T, c.stream), v0(T, c.stream), v1(T, c.stream);
    if (T > 0)
        LAUNCH(c, "setup", 0.0, k_sp_triples, grid_for(A.n, SA_B, c.num_sms * 16), SA_B, 0, A, brp, bcol, bj,
               off.get(), k0.get(), ia.get(), ib.get(), v0.get());
    uint64_t* ks = k0.get();
    int* vs = v0.get();
    if (T > 1) sort_pairs(c, k0.get(), k1.get(), v0.get(), v1.get(), T, bi + bj, &ks, &vs);
    DevArray<int64_t> head(T, c.stream), pos(T, c.stream);
    int64_t nnz = 0;
    if (T > 0) {
        LAUNCH(c, "setup", 0.0, k_sp_heads, grid_for(T, SA_B, c.num_sms * 16), SA_B, 0, ks, T, head.get());
        exclusive_sum(c, head.get(), pos.get(), T);
        nnz = d2h_scalar(pos.get() + T - 1, c.stream) + d2h_scalar(head.get() + T - 1, c.stream);
    }
    out.nnz = nnz;
    out.products = T;
    out.optr.alloc(nnz + 1, c.stream);
    out.pa.alloc(T, c.stream);
    out.pb.alloc(T, c.stream);
    DevArray<uint64_t> ukeys(nnz, c.stream);
    if (T > 0)
        LAUNCH(c, "setup", 0.0, k_sp_plan, grid_for(T, SA_B, c.num_sms * 16), SA_B, 0, ks, vs, head.get(), pos.get(),
               T, ia.get(), ib.get(), ukeys.get(), out.optr.get(), out.pa.get(), out.pb.get());
    LAUNCH(c, "setup", 0.0, k_sp_set, 1, 1, 0, out.optr.get() + nnz, static_cast<int>(T));
    out.rp.alloc(A.n + 1, c.stream);
    LAUNCH(c, "setup", 0.0, k_sp_rowptr, grid_for(A.n + 1, SA_B, c.num_sms * 16), SA_B, 0, ukeys.get(), nnz, A.n,
           bj, out.rp.get());
    out.col.alloc(nnz, c.stream);
    if (nnz > 0)
        LAUNCH(c, "setup", 0.0, k_sp_col, grid_for(nnz, SA_B, c.num_sms * 16), SA_B, 0, ukeys.get(), nnz,
               (uint64_t{1} << bj) - 1, out.col.get());
}

void spgemm_numeric(Ctx& c, const SpgPlan& p, const double* a, const double* b, double* out) {
    if (p.nnz == 0) return;
    LAUNCH(c, "rap", 8.0 * p.nnz + 12.0 * p.products, k_spgemm_num, grid_for(p.nnz, SA_B, c.num_sms * 16), SA_B, 0,
           p.nnz, p.optr.get(), p.pa.get(), p.pb.get(), a, b, out);
}

void tentative_csr(Ctx& c, int64_t n, const int* agg, DevArray<int>& rp, DevArray<int>& col, DevArray<double>& val) {
    rp.alloc(n + 1, c.stream);
    col.alloc(n, c.stream);
    val.alloc(n, c.stream);
    LAUNCH(c, "setup", 0.0, k_tentative, grid_for(n, SA_B, c.num_sms * 16), SA_B, 0, n, agg, rp.get(), col.get(),
           val.get());
}

void sa_prolongator_values(Ctx& c, int64_t n, const int* rp, const int* col, double* v, const int* agg,
                           const int* dpos, const double* aval, double w, int* bad) {
    LAUNCH(c, "setup", 0.0, k_sa_values, grid_for(n, SA_B, c.num_sms * 16), SA_B, 0, n, rp, col, v, agg, dpos, aval,
           w, bad);
}

void transpose_csr(Ctx& c, int64_t nrows, int64_t ncols, int64_t nnz, const int* rp, const int* col,
                   const double* val, DevArray<int>& trp, DevArray<int>& tcol, DevArray<double>& tval) {
    DevArray<int> rowof(nnz, c.stream), v0(nnz, c.stream), v1(nnz, c.stream);
    DevArray<uint64_t> k0(nnz, c.stream), k1(nnz, c.stream);
    if (nnz > 0) {
        LAUNCH(c, "setup", 0.0, k_row_of, grid_for(nrows, SA_B, c.num_sms * 16), SA_B, 0, nrows, rp, rowof.get());
        LAUNCH(c, "setup", 0.0, k_tr_keys, grid_for(nnz, SA_B, c.num_sms * 16), SA_B, 0, nnz, col, k0.get(),
               v0.get());
    }
    uint64_t* ks = k0.get();
    int* vs = v0.get();
    if (nnz > 1) sort_pairs(c, k0.get(), k1.get(), v0.get(), v1.get(), nnz, bits_for(ncols), &ks, &vs);
    trp.alloc(ncols + 1, c.stream);
    LAUNCH(c, "setup", 0.0, k_sp_rowptr, grid_for(ncols + 1, SA_B, c.num_sms * 16), SA_B, 0, ks, nnz, ncols, 0,
           trp.get());
    tcol.alloc(nnz, c.stream);
    tval.alloc(nnz, c.stream);
    if (nnz > 0)
        LAUNCH(c, "setup", 0.0, k_tr_fill, grid_for(nnz, SA_B, c.num_sms * 16), SA_B, 0, nnz, vs, rowof.get(), val,
               tcol.get(), tval.get());
}

// ---- coded column stream (row-pass layout) -----------------------------------
namespace {

__global__ void k_offset_keys(int64_t n, const int* __restrict__ rp, const int* __restrict__ col, uint32_t* key) {
    GRID_STRIDE(i, n) {
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            key[k] = static_cast<uint32_t>(col[k] - static_cast<int>(i)) ^ 0x80000000u;  // order-preserving
    }
}

template <class CT>
__global__ void k_encode(int64_t n, const int* __restrict__ rp, const int* __restrict__ col,
                         const uint32_t* __restrict__ ukeys, int m, int* dict, CT* code) {
    GRID_STRIDE(t, m) dict[t] = static_cast<int>(ukeys[t] ^ 0x80000000u);
    GRID_STRIDE(i, n) {
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const uint32_t key = static_cast<uint32_t>(col[k] - static_cast<int>(i)) ^ 0x80000000u;
            int lo = 0, hi = m - 1;  // ukeys sorted, unique, contains key
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (ukeys[mid] < key) lo = mid + 1;
                else hi = mid;
            }
            code[k] = static_cast<CT>(lo);
        }
    }
}

}  // namespace

void encode_columns(Ctx& c, int64_t n, int64_t nnz, const int* rp, const int* col, ColCode& out, bool narrow16) {
    out = ColCode{};
    // Default: uint8 codes on <= 8 entries/row (C3 level 0), uint16 codes on
    // 8..12 entries/row (level 1, read with 384-entry chunks: 211/227 ->
    // 202/214 us at 256^3).  AMGR_COLCODE=16 also codes the > 12 entries/row
    // levels (measured slower: their dictionary reads through L1 are not
    // hidden), AMGR_COLCODE=0 disables coding.
    const char* e = std::getenv("AMGR_COLCODE");
    if (e && std::strcmp(e, "0") == 0) return;
    const bool wide_ok = e && std::strcmp(e, "16") == 0;
    if (nnz <= 0 || n <= 0) return;
    bool narrow = nnz <= 8 * n;
    if (nnz > 12 * n && !wide_ok) return;
    // narrow16: a narrow level with more than 256 offsets (a partitioned
    // level 0: its halo columns are numbered after the owned rows) may take
    // 2-byte codes instead of int32 columns
    const int limit = narrow && !narrow16 ? 256 : 65536;
    DevArray<uint32_t> k0(nnz, c.stream), k1(nnz, c.stream);
    const unsigned grid = grid_for(n, SB, c.num_sms * 16);
    LAUNCH(c, "setup", 0.0, k_offset_keys, grid, SB, 0, n, rp, col, k0.get());
    cub::DoubleBuffer<uint32_t> kb(k0.get(), k1.get());
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kb, nnz, 0, 32, c.stream));
    DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
    CK(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, kb, nnz, 0, 32, c.stream));
    uint32_t* sorted = kb.Current();
    uint32_t* uniq = sorted == k0.get() ? k1.get() : k0.get();
    DevArray<int> num(1, c.stream);
    size_t b2 = 0;
    CK(cub::DeviceSelect::Unique(nullptr, b2, sorted, uniq, num.get(), nnz, c.stream));
    DevArray<char> tmp2(static_cast<int64_t>(b2), c.stream);
    CK(cub::DeviceSelect::Unique(tmp2.get(), b2, sorted, uniq, num.get(), nnz, c.stream));
    c.launches += 2;
    const int m = d2h_scalar(num.get(), c.stream);
    if (m > limit) return;
    if (narrow && m > 256) narrow = false;  // narrow16: 2-byte codes
    out.ndict = m;
    out.dict.alloc(m, c.stream);
    // codes are read in 16-byte-rounded TMA ranges: zeroed slack past nnz
    if (narrow) {
        out.c8.alloc(nnz + 16, c.stream);
        CK(cudaMemsetAsync(out.c8.get() + nnz, 0, 16, c.stream));
        LAUNCH(c, "setup", 0.0, k_encode<uint8_t>, grid, SB, 0, n, rp, col, uniq, m, out.dict.get(), out.c8.get());
        out.mode = 1;
    } else {
        out.c16.alloc(nnz + 8, c.stream);
        CK(cudaMemsetAsync(out.c16.get() + nnz, 0, 16, c.stream));
        LAUNCH(c, "setup", 0.0, k_encode<uint16_t>, grid, SB, 0, n, rp, col, uniq, m, out.dict.get(), out.c16.get());
        out.mode = 2;
    }
}

}  // namespace amgr

// Device-built row partition of a hierarchy (the plan paper_2108_02054_b200/
// partition.py builds on the host, computed here with the hierarchy's own
// device arrays, no downloads of patterns).  Same rules, same arrays, bit for
// bit (tests/test_gpu_dist.py compares them):
//
//  * levels 0..T partitioned, T = the coarsest level with >= replicate_below
//    rows (never the coarsest level); level T+1 rows split into W contiguous
//    ranges, ownership propagated down the aggregation tree:
//    owner_i(row) = owner_{i+1}(agg_i(row))  (aggregate-consistent);
//  * local numbering: owned rows ascending, then halo columns grouped by owner
//    rank, ascending inside a group; each local row keeps the global column
//    order of its entries;
//  * send list to peer p: the owned rows p's rows reference, ascending;
//  * member lists of the rank's coarse rows (owned rows of level i+1, or its
//    range of level T+1), members ascending.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <vector>

#include "dist_plan.cuh"

namespace amgr {
namespace {

constexpr int PB = 256;

#define PSTRIDE(i, n)                                                                      \
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n); \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void k_own_top(int64_t n, int world, int* own) {
    PSTRIDE(i, n) own[i] = static_cast<int>((i * world) / (n > 0 ? n : 1));
}
__global__ void k_own_down(int64_t n, const int* __restrict__ agg, const int* __restrict__ own_c, int* own) {
    PSTRIDE(i, n) own[i] = own_c[agg[i]];
}
__global__ void k_flag_eq(int64_t n, const int* __restrict__ own, int rank, char* flag) {
    PSTRIDE(i, n) flag[i] = own[i] == rank;
}
__global__ void k_fill_i(int64_t n, int* p, int v) {
    PSTRIDE(i, n) p[i] = v;
}
__global__ void k_scatter_pos(int64_t n, const int* __restrict__ idx, int* out, int base) {
    PSTRIDE(k, n) out[idx[k]] = base + static_cast<int>(k);
}
__global__ void k_row_lens(int64_t n, const int* __restrict__ rows, const int* __restrict__ rp, int* len) {
    PSTRIDE(k, n) len[k] = rp[rows[k] + 1] - rp[rows[k]];
}
__global__ void k_set_tail(int* a, int64_t n, const int* len) {
    a[n] = n > 0 ? a[n - 1] + len[n - 1] : 0;
}
__global__ void k_nnz_map(int64_t n, const int* __restrict__ rows, const int* __restrict__ rp,
                          const int* __restrict__ lrp, int* map) {
    PSTRIDE(k, n) {
        const int m = rows[k];
        const int a = rp[m], b = rp[m + 1], o = lrp[k];
        for (int e = a; e < b; ++e) map[o + (e - a)] = e;
    }
}
// halo candidates: foreign columns of local entries, key (owner, column)
__global__ void k_halo_keys(int64_t nnz, const int* __restrict__ map, const int* __restrict__ col,
                            const int* __restrict__ g2l, const int* __restrict__ own, uint64_t* key) {
    PSTRIDE(e, nnz) {
        const int c = col[map[e]];
        key[e] = g2l[c] >= 0 ? ~uint64_t{0} : ((static_cast<uint64_t>(own[c]) << 32) | static_cast<uint32_t>(c));
    }
}
__global__ void k_key_low(int64_t n, const uint64_t* __restrict__ key, int* lo, int* hi) {
    PSTRIDE(k, n) {
        lo[k] = static_cast<int>(key[k] & 0xffffffffu);
        if (hi) hi[k] = static_cast<int>(key[k] >> 32);
    }
}
__global__ void k_local_col(int64_t nnz, const int* __restrict__ map, const int* __restrict__ col,
                            const int* __restrict__ g2l, const int* __restrict__ hpos, int* lcol) {
    PSTRIDE(e, nnz) {
        const int c = col[map[e]];
        const int l = g2l[c];
        lcol[e] = l >= 0 ? l : hpos[c];
    }
}
// send candidates: entries of rows owned by another rank whose column is mine,
// key (row owner, column)
__global__ void k_send_keys(int64_t n, const int* __restrict__ rp, const int* __restrict__ col,
                            const int* __restrict__ own, int rank, uint64_t* key) {
    PSTRIDE(m, n) {
        const int ro = own[m];
        for (int e = rp[m]; e < rp[m + 1]; ++e) {
            const int c = col[e];
            key[e] = (ro != rank && own[c] == rank) ? ((static_cast<uint64_t>(ro) << 32) | static_cast<uint32_t>(c))
                                                    : ~uint64_t{0};
        }
    }
}
__global__ void k_gather_i(int64_t n, const int* __restrict__ idx, const int* __restrict__ src, int* dst) {
    PSTRIDE(k, n) dst[k] = src[idx[k]];
}
__global__ void k_agg_local(int64_t n, const int* __restrict__ owned, const int* __restrict__ agg,
                            const int* __restrict__ g2l_c, int base, int* lagg, int* key) {
    PSTRIDE(k, n) {
        const int a = agg[owned[k]];
        const int l = g2l_c ? g2l_c[a] : a;
        lagg[k] = l;
        key[k] = g2l_c ? l : a - base;
    }
}
__global__ void k_iota_i(int64_t n, int* v) {
    PSTRIDE(k, n) v[k] = static_cast<int>(k);
}
__global__ void k_hist(int64_t n, const int* __restrict__ key, int* cnt) {
    PSTRIDE(k, n) atomicAdd(cnt + key[k], 1);
}
__global__ void k_check_nonneg(int64_t n, const int* __restrict__ a, int* bad) {
    PSTRIDE(k, n) if (a[k] < 0) atomicOr(bad, 1);
}

unsigned grid_of(const Ctx& c, int64_t n) {
    const int64_t want = (n + PB - 1) / PB;
    const int64_t cap = static_cast<int64_t>(c.num_sms) * 16;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min(want, cap)));
}

}  // namespace

// compact indices i in [0, n) with flag[i] into out; returns the count
int64_t select_flagged(Ctx& c, const char* flag, int64_t n, DevArray<int>& out) {
    DevArray<int> tmp_out(std::max<int64_t>(n, 1), c.stream);
    DevArray<int> nsel(1, c.stream);
    cub::CountingInputIterator<int> it(0);
    size_t bytes = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, bytes, it, flag, tmp_out.get(), nsel.get(), n, c.stream));
    DevArray<char> tmp(static_cast<int64_t>(std::max<size_t>(bytes, 1)), c.stream);
    CK(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flag, tmp_out.get(), nsel.get(), n, c.stream));
    const int64_t cnt = d2h_scalar(nsel.get(), c.stream);
    out.alloc(std::max<int64_t>(cnt, 1), c.stream);
    d2d(out.get(), tmp_out.get(), cnt, c.stream);
    return cnt;
}

namespace {

// sort + unique of the valid keys (invalid = all ones, sorted last); returns
// the unique valid keys
int64_t sort_unique(Ctx& c, DevArray<uint64_t>& keys, int64_t n, DevArray<uint64_t>& out) {
    if (n == 0) {
        out.alloc(1, c.stream);
        return 0;
    }
    DevArray<uint64_t> k1(n, c.stream);
    cub::DoubleBuffer<uint64_t> kb(keys.get(), k1.get());
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kb, n, 0, 64, c.stream));
    {
        DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
        CK(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, kb, n, 0, 64, c.stream));
    }
    DevArray<uint64_t> uq(n, c.stream);
    DevArray<int> nsel(1, c.stream);
    bytes = 0;
    CK(cub::DeviceSelect::Unique(nullptr, bytes, kb.Current(), uq.get(), nsel.get(), n, c.stream));
    {
        DevArray<char> tmp(static_cast<int64_t>(std::max<size_t>(bytes, 1)), c.stream);
        CK(cub::DeviceSelect::Unique(tmp.get(), bytes, kb.Current(), uq.get(), nsel.get(), n, c.stream));
    }
    int64_t u = d2h_scalar(nsel.get(), c.stream);
    if (u > 0) {
        uint64_t last = 0;
        d2h(&last, uq.get() + (u - 1), 1, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        if (last == ~uint64_t{0}) --u;  // drop the invalid marker
    }
    out.alloc(std::max<int64_t>(u, 1), c.stream);
    d2d(out.get(), uq.get(), u, c.stream);
    return u;
}

}  // namespace

int choose_top_level(const Hier& h, int64_t replicate_below) {
    int top = -1;
    for (size_t i = 0; i + 1 < h.lv.size(); ++i)
        if (h.lv[i].pat->n >= replicate_below) top = static_cast<int>(i);
    return top;
}

DevicePlan build_device_plan(Hier& h, int rank, int world, int64_t replicate_below) {
    Ctx& c = *h.ctx;
    DevicePlan P;
    P.top = choose_top_level(h, replicate_below);
    const int T = P.top;
    if (T < 0) invalid("amgr_dist_create_auto: hierarchy too small to partition (raise replicate_below)");
    for (int i = 0; i <= T; ++i)
        if (!h.lv[i].T || h.lv[i].T->smoothed) invalid("amgr_dist_create_auto: plain aggregation only");
    // ownership of levels 0..T+1
    std::vector<DevArray<int>> own(static_cast<size_t>(T + 2));
    const int64_t nT1 = h.lv[T + 1].pat->n;
    own[T + 1].alloc(nT1, c.stream);
    LAUNCH(c, "dist_plan", 0.0, k_own_top, grid_of(c, nT1), PB, 0, nT1, world, own[T + 1].get());
    for (int i = T; i >= 0; --i) {
        const int64_t n = h.lv[i].pat->n;
        own[i].alloc(n, c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_own_down, grid_of(c, n), PB, 0, n, h.lv[i].T->agg.get(), own[i + 1].get(),
               own[i].get());
    }
    // transition counts: rows I with floor(I*W/n) == r
    P.t_counts.assign(static_cast<size_t>(world), 0);
    for (int64_t I = 0; I < nT1; ++I) ++P.t_counts[static_cast<size_t>((I * world) / std::max<int64_t>(nT1, 1))];
    int64_t t0 = 0;
    for (int r = 0; r < rank; ++r) t0 += P.t_counts[static_cast<size_t>(r)];
    // per level: owned rows, local CSR, halo, send lists
    std::vector<DevArray<int>> g2l(static_cast<size_t>(T + 2));
    P.lv.resize(static_cast<size_t>(T + 1));
    for (int i = 0; i <= T; ++i) {
        const Pattern& G = *h.lv[i].pat;
        PlanLevel& L = P.lv[i];
        const int64_t n = G.n;
        DevArray<char> flag(n, c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_flag_eq, grid_of(c, n), PB, 0, n, own[i].get(), rank, flag.get());
        L.n_own = select_flagged(c, flag.get(), n, L.owned);
        g2l[i].alloc(n, c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_fill_i, grid_of(c, n), PB, 0, n, g2l[i].get(), -1);
        LAUNCH(c, "dist_plan", 0.0, k_scatter_pos, grid_of(c, L.n_own), PB, 0, L.n_own, L.owned.get(), g2l[i].get(), 0);
        DevArray<int> len(std::max<int64_t>(L.n_own, 1), c.stream);
        L.rp.alloc(L.n_own + 1, c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_row_lens, grid_of(c, L.n_own), PB, 0, L.n_own, L.owned.get(), G.rp.get(),
               len.get());
        if (L.n_own > 0) exclusive_sum_i32(c, len.get(), L.rp.get(), L.n_own);
        LAUNCH(c, "dist_plan", 0.0, k_set_tail, 1, 1, 0, L.rp.get(), L.n_own, len.get());
        L.nnz = d2h_scalar(L.rp.get() + L.n_own, c.stream);
        L.nnz_map.alloc(std::max<int64_t>(L.nnz, 1), c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_nnz_map, grid_of(c, L.n_own), PB, 0, L.n_own, L.owned.get(), G.rp.get(),
               L.rp.get(), L.nnz_map.get());
        // halo: unique (owner, column) of the foreign columns
        DevArray<uint64_t> hk(std::max<int64_t>(L.nnz, 1), c.stream), hu;
        LAUNCH(c, "dist_plan", 0.0, k_halo_keys, grid_of(c, L.nnz), PB, 0, L.nnz, L.nnz_map.get(), G.col.get(),
               g2l[i].get(), own[i].get(), hk.get());
        L.n_halo = sort_unique(c, hk, L.nnz, hu);
        L.halo.alloc(std::max<int64_t>(L.n_halo, 1), c.stream);
        DevArray<int> howner(std::max<int64_t>(L.n_halo, 1), c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_key_low, grid_of(c, L.n_halo), PB, 0, L.n_halo, hu.get(), L.halo.get(),
               howner.get());
        DevArray<int> hpos(n, c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_fill_i, grid_of(c, n), PB, 0, n, hpos.get(), -1);
        LAUNCH(c, "dist_plan", 0.0, k_scatter_pos, grid_of(c, L.n_halo), PB, 0, L.n_halo, L.halo.get(), hpos.get(),
               static_cast<int>(L.n_own));
        L.col.alloc(std::max<int64_t>(L.nnz, 1), c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_local_col, grid_of(c, L.nnz), PB, 0, L.nnz, L.nnz_map.get(), G.col.get(),
               g2l[i].get(), hpos.get(), L.col.get());
        // receive blocks: consecutive halo owners
        std::vector<int> ho(static_cast<size_t>(L.n_halo));
        d2h(ho.data(), howner.get(), L.n_halo, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        for (int64_t k = 0; k < L.n_halo;) {
            int64_t e = k;
            while (e < L.n_halo && ho[static_cast<size_t>(e)] == ho[static_cast<size_t>(k)]) ++e;
            L.recv_peer.push_back(ho[static_cast<size_t>(k)]);
            L.recv_off.push_back(k);
            L.recv_cnt.push_back(e - k);
            k = e;
        }
        // send lists: unique (peer, my column) over the entries of the peers' rows
        DevArray<uint64_t> sk(std::max<int64_t>(G.nnz, 1), c.stream), su;
        LAUNCH(c, "dist_plan", 0.0, k_send_keys, grid_of(c, n), PB, 0, n, G.rp.get(), G.col.get(), own[i].get(), rank,
               sk.get());
        const int64_t ns = sort_unique(c, sk, G.nnz, su);
        DevArray<int> scol(std::max<int64_t>(ns, 1), c.stream), speer(std::max<int64_t>(ns, 1), c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_key_low, grid_of(c, ns), PB, 0, ns, su.get(), scol.get(), speer.get());
        L.send_idx.alloc(ns, c.stream);  // exact size: the halo pack keys on it (0: nothing to send)
        if (ns > 0)
            LAUNCH(c, "dist_plan", 0.0, k_gather_i, grid_of(c, ns), PB, 0, ns, scol.get(), g2l[i].get(),
                   L.send_idx.get());
        std::vector<int> sp(static_cast<size_t>(ns));
        d2h(sp.data(), speer.get(), ns, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        for (int64_t k = 0; k < ns;) {
            int64_t e = k;
            while (e < ns && sp[static_cast<size_t>(e)] == sp[static_cast<size_t>(k)]) ++e;
            L.send_peer.push_back(sp[static_cast<size_t>(k)]);
            L.send_cnt.push_back(e - k);
            k = e;
        }
    }
    // transfers: local aggregate map and member lists of the rank's coarse rows
    for (int i = 0; i <= T; ++i) {
        PlanLevel& L = P.lv[i];
        const bool inner = i < T;
        L.n_cown = inner ? P.lv[i + 1].n_own : P.t_counts[static_cast<size_t>(rank)];
        L.agg.alloc(std::max<int64_t>(L.n_own, 1), c.stream);
        DevArray<int> key(std::max<int64_t>(L.n_own, 1), c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_agg_local, grid_of(c, L.n_own), PB, 0, L.n_own, L.owned.get(),
               h.lv[i].T->agg.get(), inner ? g2l[i + 1].get() : nullptr, static_cast<int>(inner ? 0 : t0), L.agg.get(),
               key.get());
        DevArray<int> bad(1, c.stream);
        CK(cudaMemsetAsync(bad.get(), 0, sizeof(int), c.stream));
        LAUNCH(c, "dist_plan", 0.0, k_check_nonneg, grid_of(c, L.n_own), PB, 0, L.n_own, key.get(), bad.get());
        if (d2h_scalar(bad.get(), c.stream)) fail(AMGR_E_RUNTIME, "dist plan: aggregate consistency violated");
        // members ascending per coarse row: stable sort of (key, local fine id)
        DevArray<int> v0(std::max<int64_t>(L.n_own, 1), c.stream), v1(std::max<int64_t>(L.n_own, 1), c.stream),
            k1(std::max<int64_t>(L.n_own, 1), c.stream);
        LAUNCH(c, "dist_plan", 0.0, k_iota_i, grid_of(c, L.n_own), PB, 0, L.n_own, v0.get());
        cub::DoubleBuffer<int> kb(key.get(), k1.get()), vb(v0.get(), v1.get());
        size_t bytes = 0;
        if (L.n_own > 0) {
            CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, L.n_own, 0, 32, c.stream));
            DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
            CK(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kb, vb, L.n_own, 0, 32, c.stream));
        }
        L.midx.alloc(std::max<int64_t>(L.n_own, 1), c.stream);
        d2d(L.midx.get(), vb.Current(), L.n_own, c.stream);
        DevArray<int> cnt(std::max<int64_t>(L.n_cown, 1), c.stream);
        CK(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * static_cast<size_t>(std::max<int64_t>(L.n_cown, 1)), c.stream));
        LAUNCH(c, "dist_plan", 0.0, k_hist, grid_of(c, L.n_own), PB, 0, L.n_own, kb.Current(), cnt.get());
        L.mptr.alloc(L.n_cown + 1, c.stream);
        if (L.n_cown > 0) exclusive_sum_i32(c, cnt.get(), L.mptr.get(), L.n_cown);
        LAUNCH(c, "dist_plan", 0.0, k_set_tail, 1, 1, 0, L.mptr.get(), L.n_cown, cnt.get());
    }
    CK(cudaStreamSynchronize(c.stream));
    return P;
}

}  // namespace amgr

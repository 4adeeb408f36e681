// Row-partitioned multi-GPU solve — one process per GPU,
// NCCL over NVLink for the data path.
//
//  * Setup is replicated: every rank builds the same global hierarchy
//    (deterministic), then adopts the aggregate-consistent partition computed
//    by paper_2108_02054_b200/partition.py (levels 0..T partitioned, T+1..
//    replicated).  Rebuild in round 1 is the global rebuild on every rank
//    followed by gathers of the local values (the rebuild is ~1% of a step);
//    the solve is partitioned.
//  * Partitioned levels run the same row-pass kernels on local CSR matrices
//    whose columns index [owned | halo]; before every pass whose operand is
//    gathered, the halo is exchanged with ncclSend/ncclRecv in one group.
//    Restriction and prolongation are local (aggregate-consistent ownership).
//  * Transition: each rank restricts onto its contiguous range of level-T+1
//    rows; one ncclAllGather (padded blocks) replicates f_{T+1}; the coarse
//    levels run through vcycle_from(T+1) on every rank.
//  * Dots: every rank's partial (deterministic block reduction) is
//    allgathered and summed in rank order on the device, so all ranks take
//    identical control-flow decisions.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <sstream>

#include "dist_plan.cuh"
#include "hierarchy.cuh"
#include "reduce.cuh"

namespace amgr {

// NCCL is bound at run time (dlopen), not at link time: the process usually
// already holds torch's bundled libnccl.so.2, and a link-time NEEDED entry
// would let the system copy claim that SONAME first when this library loads
// before torch.  RTLD_NOLOAD picks the already-loaded copy when present.
struct NcclApi {
    decltype(&::ncclGetUniqueId) GetUniqueId;
    decltype(&::ncclCommInitRank) CommInitRank;
    decltype(&::ncclCommDestroy) CommDestroy;
    decltype(&::ncclGroupStart) GroupStart;
    decltype(&::ncclGroupEnd) GroupEnd;
    decltype(&::ncclSend) Send;
    decltype(&::ncclRecv) Recv;
    decltype(&::ncclAllGather) AllGather;
    decltype(&::ncclGetErrorString) GetErrorString;
};

static const NcclApi* nccl_api() {
    static NcclApi api{};
    static bool ok = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        bool good = true;
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            good = good && f != nullptr;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GetErrorString, "ncclGetErrorString");
        return good;
    }();
    return ok ? &api : nullptr;
}

static const NcclApi& N() {
    const NcclApi* a = nccl_api();
    if (!a) fail(AMGR_E_NCCL, "NCCL: libnccl.so.2 could not be loaded");
    return *a;
}

#define NK(x)                                                                                         \
    do {                                                                                              \
        ncclResult_t r_ = (x);                                                                        \
        if (r_ != ncclSuccess) ::amgr::fail(AMGR_E_NCCL, std::string("NCCL: ") + ::amgr::N().GetErrorString(r_)); \
    } while (0)

namespace {

__global__ void k_gather_d(int64_t n, const double* __restrict__ src, const int* __restrict__ idx,
                           double* __restrict__ dst, Gate g) {
    if (gated_off(g)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[idx[i]];
}

// padded allgather blocks (W x pad) -> global vector (block r at displ[r], count[r])
__global__ void k_unpad(int world, int64_t pad, const double* __restrict__ buf, const int64_t* __restrict__ displ,
                        const int64_t* __restrict__ cnt, double* __restrict__ out) {
    for (int r = 0; r < world; ++r)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < cnt[r];
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            out[displ[r] + i] = buf[r * pad + i];
}

// sum the W gathered partials of each of k dots in rank order
__global__ void k_rank_sum(int world, int k, const double* __restrict__ parts, double* const* outs) {
    const int t = threadIdx.x;
    if (t >= k) return;
    double s = 0.0;
    for (int r = 0; r < world; ++r) s = __dadd_rn(s, parts[r * k + t]);
    *outs[t] = s;
}

// ---- sequential-dot parity mode (Ctx::seq_dots) --------------------------------
// The reference sums every dot left to right over the GLOBAL index
// (bicgstab.cpp:11-17).  Each rank forms its rounded products a_i*b_i in local
// order, one padded allgather brings all of them to every rank, and one
// thread per rank sums them in global order through gpos (global row ->
// position in the gathered blocks): the same bits as the reference's dot.
__global__ void k_dist_prod(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                            double* __restrict__ out, Gate g) {
    if (gated_off(g)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __dmul_rn(a[i], b[i]);
}

// gathered owned ids (as doubles, -1 = padding) -> gpos
__global__ void k_dist_gpos(int64_t total, const double* __restrict__ ids, int64_t* __restrict__ gpos) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = ids[k];
        if (v >= 0.0) gpos[static_cast<int64_t>(v)] = k;
    }
}

constexpr int GS_THREADS = 256, GS_CH = 2048;

// s = sum_{i < n} prod[gpos[i]] left to right; warps 1.. stage the next chunk
// into shared memory while thread 0 sums the current one
__global__ void __launch_bounds__(GS_THREADS) k_dist_seq_sum(int64_t n, const double* __restrict__ prod,
                                                             const int64_t* __restrict__ gpos, double* out, Gate g) {
    if (gated_off(g)) return;
    __shared__ double buf[2][GS_CH];
    const int tid = threadIdx.x;
    const int64_t nch = (n + GS_CH - 1) / GS_CH;
    auto fill = [&](int64_t ch, double* dst, int t0, int nt) {
        const int64_t base = ch * GS_CH;
        const int len = static_cast<int>(n - base < GS_CH ? n - base : GS_CH);
        for (int i = t0; i < len; i += nt) dst[i] = prod[gpos[base + i]];
    };
    if (nch > 0) fill(0, buf[0], tid, GS_THREADS);
    __syncthreads();
    double s = 0.0;
    for (int64_t ch = 0; ch < nch; ++ch) {
        if (tid >= 32) {
            if (ch + 1 < nch) fill(ch + 1, buf[(ch + 1) & 1], tid - 32, GS_THREADS - 32);
        } else if (tid == 0) {
            const int64_t base = ch * GS_CH;
            const int len = static_cast<int>(n - base < GS_CH ? n - base : GS_CH);
            const double* p = buf[ch & 1];
            for (int i = 0; i < len; ++i) s = __dadd_rn(s, p[i]);
        }
        __syncthreads();
    }
    if (tid == 0) *out = s;
}

// ---- partitioned rebuild (rank-local values) ----------------------------------
// local diagonal positions: owned row r has local column r (linear scan, the
// local columns are not sorted: halo ids follow the owned ones)
__global__ void k_local_diag(int64_t n, const int* __restrict__ rp, const int* __restrict__ col, int* dpos) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int d = -1;
        for (int k = rp[r]; k < rp[r + 1]; ++k)
            if (col[k] == static_cast<int>(r)) {
                d = k;
                break;
            }
        dpos[r] = d;
    }
}

__global__ void k_scatter_inv(int64_t n, const int* __restrict__ map, int* __restrict__ inv) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        inv[map[k]] = static_cast<int>(k);
}

// Local Galerkin plan = the global plan restricted to this rank's coarse rows.
// Local coarse row r is global row crow[r] (or base + r when crow is null);
// its entries are the global row's entries in the same order (local CSR keeps
// the global column order), local offsets lrp[r].  Counts first, then (after
// an exclusive scan) the contributions, each fine index remapped through
// ginv (global fine entry -> local entry of this rank; all members of an owned
// coarse row are owned: aggregate-consistent partition) with its row-break bit.
__global__ void k_lplan_count(int64_t nrows, const int* __restrict__ crow, int64_t base, const int* __restrict__ rpg,
                              const int* __restrict__ lrp, const int* __restrict__ cptrg, int* __restrict__ cnt) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < nrows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t I = crow ? crow[r] : base + r;
        const int g0 = rpg[I];
        for (int e = lrp[r]; e < lrp[r + 1]; ++e) {
            const int g = g0 + (e - lrp[r]);
            cnt[e] = (cptrg[g + 1] & 0x3fffffff) - (cptrg[g] & 0x3fffffff);
        }
    }
}
__global__ void k_lplan_fill(int64_t nrows, const int* __restrict__ crow, int64_t base, const int* __restrict__ rpg,
                             const int* __restrict__ lrp, const int* __restrict__ cptrg,
                             const int* __restrict__ contribg, const int* __restrict__ ginv,
                             const int* __restrict__ lcptr, int* __restrict__ lcontrib, int* bad) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < nrows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t I = crow ? crow[r] : base + r;
        const int g0 = rpg[I];
        for (int e = lrp[r]; e < lrp[r + 1]; ++e) {
            const int g = g0 + (e - lrp[r]);
            const int p0 = cptrg[g] & 0x3fffffff, p1 = cptrg[g + 1] & 0x3fffffff;
            int q = lcptr[e];
            for (int p = p0; p < p1; ++p, ++q) {
                const int v = contribg[p];
                const int l = ginv[v & 0x7fffffff];
                if (l < 0) atomicOr(bad, 1);
                lcontrib[q] = (l < 0 ? 0 : l) | (v & static_cast<int>(0x80000000u));
            }
        }
    }
}

__global__ void k_set_last(int* lcptr, int64_t n, const int* cnt) {
    if (n > 0) lcptr[n] = lcptr[n - 1] + cnt[n - 1];
    else lcptr[0] = 0;
}

// flag[i] = row i has a column in the halo (>= n_own)
__global__ void k_halo_rows(int64_t n_own, const int* __restrict__ rp, const int* __restrict__ col, char* flag) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_own;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        char h = 0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) h |= col[k] >= n_own ? 1 : 0;
        flag[i] = h;
    }
}

}  // namespace

struct DistLevel {
    int64_t n_own = 0, n_halo = 0, nnz = 0, n_cown = 0;
    DevArray<int> rp, col, nnz_map, owned, agg, mptr, midx;
    DevArray<double> val, w;
    // partitioned rebuild: local diagonal positions and the local Galerkin
    // plan onto this rank's coarse rows (k_rap_tma, rap_numeric)
    DevArray<int> dpos, lcptr, lcontrib;
    int64_t lnnz_c = 0, lnc = 0;
    int lmax_chunk = -1;
    GrpPlan grp;  // warp-group form of the local plan (k_rap_grp with the Jacobi rebuild fused)
    ColCode cc;  // coded column stream of the local pattern (when its offsets are few: no / few halos)
    DevArray<double> u0, x, out, f, r;  // u0/x carry halo space
    std::vector<int> send_peer, recv_peer;
    std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
    DevArray<int> send_idx;
    DevArray<double> send_buf;
    DevArray<int> brows;  // owned rows with a halo column (recomputed after the exchange when overlapping)
    int64_t nb = 0;
    int max_span = 0;
    CsrView view() const {
        CsrView v;
        v.n = n_own;
        v.ncols = n_own + n_halo;
        v.nnz = nnz;
        v.rp = rp.get();
        v.col = col.get();
        v.val = val.get();
        v.max_span = max_span;
        set_code(v, cc);
        return v;
    }
};

// In-process transport for testing the multi-rank device path on ONE GPU:
// W ranks live in one process (one host thread and one context/stream each).
// Every exchange is stream-ordered like its NCCL counterpart: a rank posts
// its send pointers plus an event recorded after the producing kernel, all
// ranks meet at a host barrier, each rank makes its stream wait on the
// producers' events and pulls the data with device-to-device copies, records
// a "consumed" event, and after a second barrier waits on its consumers'
// events before its send buffers may be reused.  No kernel ever waits on
// another rank's kernel.
struct Loopback {
    int world = 1;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    int64_t generation = 0;
    struct Post {
        std::vector<const double*> ptr;  // by destination rank (halo) or [0] (allgather)
        std::vector<int64_t> cnt;
        cudaEvent_t ready = nullptr, consumed = nullptr;
    };
    std::vector<Post> post;
    explicit Loopback(int w) : world(w), post(static_cast<size_t>(w)) {
        for (auto& p : post) {
            p.ptr.assign(static_cast<size_t>(w), nullptr);
            p.cnt.assign(static_cast<size_t>(w), 0);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const int64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

struct DistHier {
    DistHier() = default;
    DistHier(const DistHier&) = delete;
    DistHier& operator=(const DistHier&) = delete;
    ~DistHier();
    Hier* g = nullptr;
    Ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    Loopback* lb = nullptr;  // test transport instead of NCCL
    cudaEvent_t ev_ready = nullptr, ev_consumed = nullptr;
    // halo exchange overlapped with the V-cycle passes (world > 1): the
    // exchange runs on cs while the full pass runs on the library stream
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool overlap = false;
    int rank = 0, world = 1, T = -1;
    std::vector<DistLevel> lv;
    // transition (level T -> T+1)
    std::vector<int64_t> tcnt, tdispl;
    int64_t tpad = 0;
    DevArray<double> tsend, tgather, fT, uT;
    DevArray<int64_t> tcnt_d, tdispl_d;
    // partitioned rebuild: this rank's rows of A_{T+1} are a contiguous entry
    // range of the global level T+1; their values are allgathered (padded)
    std::vector<int64_t> tvcnt, tvdispl;
    int64_t tvpad = 0;
    DevArray<double> tvsend, tvgather;
    DevArray<int64_t> tvcnt_d, tvdispl_d;
    DevArray<int> lerr;       // per partitioned level first bad local row
    DevArray<double> errd, errall;
    // Krylov (level 0 local)
    DevArray<double> kr, krt, kp, kv, ks, kt, kph, ksh, ku;
    DevArray<double> dloc, dall;  // local dot results (up to 2) and the gathered partials
    DevArray<double*> douts;      // table of dot output pointer sets (out_slot)
    // sequential-dot parity mode: products, their padded allgather, global order
    int64_t spad = 0, n_global = 0;
    DevArray<double> sprod, sall, kq;
    DevArray<int64_t> gpos;
    std::vector<std::vector<double*>> dtab;
    std::vector<int64_t> dtab_off;
};

// Halo exchange of x's owned boundary values into the peers' halo slots.
// async: the exchange itself (NCCL send/recv or the loopback copies) runs on
// d.cs, forked after the pack kernel; the caller joins with halo_join before
// reading the halo.
static void halo(DistHier& d, DistLevel& L, double* x, Gate g, bool async = false) {
    Ctx& c = *d.ctx;
    if (L.send_idx.size() > 0)
        LAUNCH(c, "halo_pack", 16.0 * L.send_idx.size(), k_gather_d, grid_for(L.send_idx.size(), 256, c.num_sms * 8),
               256, 0, L.send_idx.size(), x, L.send_idx.get(), L.send_buf.get(), g);
    const cudaStream_t xs = async ? d.cs : c.stream;
    if (async) {
        CK(cudaEventRecord(d.ev_fork, c.stream));
        CK(cudaStreamWaitEvent(d.cs, d.ev_fork, 0));
    }
    if (d.lb) {  // every rank enters both barriers, peers or not
        Loopback& lb = *d.lb;
        Loopback::Post& me = lb.post[d.rank];
        CK(cudaEventRecord(d.ev_ready, c.stream));
        for (int q = 0; q < d.world; ++q) {
            me.ptr[q] = nullptr;
            me.cnt[q] = 0;
        }
        for (size_t k = 0; k < L.send_peer.size(); ++k) {
            me.ptr[L.send_peer[k]] = L.send_buf.get() + L.send_off[k];
            me.cnt[L.send_peer[k]] = L.send_cnt[k];
        }
        me.ready = d.ev_ready;
        me.consumed = d.ev_consumed;
        lb.barrier();
        for (size_t k = 0; k < L.recv_peer.size(); ++k) {
            const Loopback::Post& src = lb.post[L.recv_peer[k]];
            if (src.cnt[d.rank] != L.recv_cnt[k]) fail(AMGR_E_RUNTIME, "loopback halo: send/recv counts differ");
            CK(cudaStreamWaitEvent(xs, src.ready, 0));
            CK(cudaMemcpyAsync(x + L.n_own + L.recv_off[k], src.ptr[d.rank], sizeof(double) * L.recv_cnt[k],
                               cudaMemcpyDeviceToDevice, xs));
        }
        CK(cudaEventRecord(d.ev_consumed, xs));
        if (async) CK(cudaEventRecord(d.ev_join, xs));
        lb.barrier();
        for (size_t k = 0; k < L.send_peer.size(); ++k)
            CK(cudaStreamWaitEvent(c.stream, lb.post[L.send_peer[k]].consumed, 0));
        lb.barrier();  // posts may be rewritten only after every rank has read them
        return;
    }
    if (!(d.world == 1 || (L.send_peer.empty() && L.recv_peer.empty()))) {
        NK(N().GroupStart());
        for (size_t k = 0; k < L.send_peer.size(); ++k)
            NK(N().Send(L.send_buf.get() + L.send_off[k], static_cast<size_t>(L.send_cnt[k]), ncclDouble,
                        L.send_peer[k], d.comm, xs));
        for (size_t k = 0; k < L.recv_peer.size(); ++k)
            NK(N().Recv(x + L.n_own + L.recv_off[k], static_cast<size_t>(L.recv_cnt[k]), ncclDouble, L.recv_peer[k],
                        d.comm, xs));
        NK(N().GroupEnd());
    }
    if (async) CK(cudaEventRecord(d.ev_join, xs));
}
static void halo_join(DistHier& d) { CK(cudaStreamWaitEvent(d.ctx->stream, d.ev_join, 0)); }
// overlap this level's exchange with its pass: the full pass runs on stale
// halo values while the exchange is in flight, then the boundary rows are
// recomputed (k_rowlist, same arithmetic) once the halo has arrived
static bool overlapped(const DistHier& d, const DistLevel& L) {
    return d.overlap && L.nb > 0 && L.nb < L.n_own && (!L.send_peer.empty() || !L.recv_peer.empty());
}

// allgather of count doubles per rank (rank r's block at recv + r*count)
static void allgather(DistHier& d, const double* send, double* recv, int64_t count) {
    Ctx& c = *d.ctx;
    if (d.lb) {
        Loopback& lb = *d.lb;
        Loopback::Post& me = lb.post[d.rank];
        CK(cudaEventRecord(d.ev_ready, c.stream));
        me.ptr[0] = send;
        me.cnt[0] = count;
        me.ready = d.ev_ready;
        me.consumed = d.ev_consumed;
        lb.barrier();
        for (int q = 0; q < d.world; ++q) {
            CK(cudaStreamWaitEvent(c.stream, lb.post[q].ready, 0));
            CK(cudaMemcpyAsync(recv + q * count, lb.post[q].ptr[0], sizeof(double) * count, cudaMemcpyDeviceToDevice,
                               c.stream));
        }
        CK(cudaEventRecord(d.ev_consumed, c.stream));
        lb.barrier();
        for (int q = 0; q < d.world; ++q) CK(cudaStreamWaitEvent(c.stream, lb.post[q].consumed, 0));
        lb.barrier();
        return;
    }
    if (d.world > 1)
        NK(N().AllGather(send, recv, static_cast<size_t>(count), ncclDouble, d.comm, c.stream));
    else
        d2d(recv, send, count, c.stream);
}

// deterministic cross-rank sum of k local dots (d.dloc[0..k)) into outs
// The output pointer sets live in a device table (registered once, outside
// any graph capture), so an iteration enqueues no host-to-device copies and
// the NCCL path can be captured into a CUDA graph.
static double* const* out_slot(DistHier& d, std::initializer_list<double*> outs) {
    std::vector<double*> o(outs);
    for (size_t i = 0; i < d.dtab.size(); ++i)
        if (d.dtab[i] == o) return d.douts.get() + d.dtab_off[i];
    const int64_t off = d.dtab_off.empty() ? 0 : d.dtab_off.back() + static_cast<int64_t>(d.dtab.back().size());
    if (off + static_cast<int64_t>(o.size()) > d.douts.size()) fail(AMGR_E_RUNTIME, "dist: dot output table full");
    h2d(d.douts.get() + off, o.data(), static_cast<int64_t>(o.size()), d.ctx->stream);
    d.dtab.push_back(o);
    d.dtab_off.push_back(off);
    return d.douts.get() + off;
}

static void allsum(DistHier& d, int k, std::initializer_list<double*> outs) {
    Ctx& c = *d.ctx;
    double* const* slot = out_slot(d, outs);
    allgather(d, d.dloc.get(), d.dall.get(), k);
    LAUNCH(c, "dist", 0.0, k_rank_sum, 1, 32, 0, d.world, k, d.dall.get(), const_cast<double**>(slot));
}

// sequential-dot mode: global positions of every rank's level-0 rows (once,
// outside any capture: one allgather of the row counts, one of the ids)
static void seq_prepare(DistHier& d) {
    if (d.gpos.size() > 0) return;
    Ctx& c = *d.ctx;
    const DistLevel& L0 = d.lv[0];
    d.n_global = d.g->lv.front().pat->n;
    DevArray<double> cnt, cnts;
    cnt.alloc(1, c.stream);
    cnts.alloc(d.world, c.stream);
    const double me = static_cast<double>(L0.n_own);
    h2d(cnt.get(), &me, 1, c.stream);
    allgather(d, cnt.get(), cnts.get(), 1);
    std::vector<double> hc(static_cast<size_t>(d.world));
    d2h(hc.data(), cnts.get(), d.world, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    int64_t pad = 1, tot = 0;
    for (double v : hc) {
        pad = std::max(pad, static_cast<int64_t>(v));
        tot += static_cast<int64_t>(v);
    }
    if (tot != d.n_global) fail(AMGR_E_RUNTIME, "dist: level-0 rows of all ranks do not cover the global level");
    d.spad = pad;
    d.sprod.alloc(pad, c.stream);
    d.sall.alloc(pad * d.world, c.stream);
    d.kq.alloc(std::max<int64_t>(L0.n_own, 1), c.stream);
    d.gpos.alloc(d.n_global, c.stream);
    std::vector<int> ids(static_cast<size_t>(L0.n_own));
    d2h(ids.data(), L0.owned.get(), L0.n_own, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    std::vector<double> idd(static_cast<size_t>(pad), -1.0);
    for (int64_t i = 0; i < L0.n_own; ++i) idd[i] = ids[i];
    h2d(d.sprod.get(), idd.data(), pad, c.stream);
    allgather(d, d.sprod.get(), d.sall.get(), pad);
    LAUNCH(c, "dist", 0.0, k_dist_gpos, grid_for(pad * d.world, 256, c.num_sms * 8), 256, 0, pad * d.world,
           d.sall.get(), d.gpos.get());
    CK(cudaStreamSynchronize(c.stream));
}

// *out = the reference's dot(a, b) over the global vector (after the
// rank-ordered blocked value the same field held; gated like its producer)
static void seq_dot_dist(DistHier& d, const double* a, const double* b, double* out, Gate g = {}) {
    Ctx& c = *d.ctx;
    const int64_t n = d.lv[0].n_own;
    if (n > 0)
        LAUNCH(c, "seq_dot", 16.0 * n, k_dist_prod, grid_for(n, 256, c.num_sms * 8), 256, 0, n, a, b, d.sprod.get(),
               g);
    allgather(d, d.sprod.get(), d.sall.get(), d.spad);
    LAUNCH(c, "seq_dot", 16.0 * d.n_global, k_dist_seq_sum, 1, GS_THREADS, 0, d.n_global, d.sall.get(),
           d.gpos.get(), out, g);
}

static DotSink local_sink(DistHier& d, int slot) {
    Work& W = work(*d.g);
    return DotSink{W.partials.get(), W.ticket.get(), d.dloc.get() + slot};
}

// ---- V-cycle on the partition (hierarchy.cpp:152-186 semantics) -------------
static void dist_vcycle(DistHier& d, const double* f0, double* u_out, Gate g) {
    Ctx& c = *d.ctx;
    Hier& h = *d.g;
    const double om = h.om_eff();
    const int T = d.T;
    std::vector<const double*> fin(T + 1);
    fin[0] = f0;
    for (int i = 1; i <= T; ++i) fin[i] = d.lv[i].f.get();
    vc_premul(c, d.lv[0].n_own, f0, d.lv[0].w.get(), om, d.lv[0].u0.get(), g);
    for (int i = 0; i <= T; ++i) {
        c.cur_level = i;
        DistLevel& L = d.lv[i];
        if (overlapped(d, L)) {
            halo(d, L, L.u0.get(), g, true);
            vc_down(c, L.view(), fin[i], L.u0.get(), L.r.get(), g);
            halo_join(d);
            vc_down_rows(c, L.view(), L.brows.get(), L.nb, fin[i], L.u0.get(), L.r.get(), g);
        } else {
            halo(d, L, L.u0.get(), g);
            vc_down(c, L.view(), fin[i], L.u0.get(), L.r.get(), g);
        }
        if (i < T) {
            DistLevel& N = d.lv[i + 1];
            restrict_sum(c, L.n_cown, L.mptr.get(), L.midx.get(), L.r.get(), N.f.get(), N.w.get(), om, N.u0.get(), g);
        } else {
            restrict_sum(c, L.n_cown, L.mptr.get(), L.midx.get(), L.r.get(), d.tsend.get(), nullptr, 0.0, nullptr, g);
        }
    }
    // transition: replicate f_{T+1}, then the coarse levels on every rank
    allgather(d, d.tsend.get(), d.tgather.get(), d.tpad);
    LAUNCH(c, "dist", 0.0, k_unpad, grid_for(d.tpad, 256, 64), 256, 0, d.world, d.tpad, d.tgather.get(),
           d.tdispl_d.get(), d.tcnt_d.get(), d.fT.get());
    vcycle_from(h, static_cast<size_t>(T + 1), d.fT.get(), d.uT.get(), g);
    const double* uc = d.uT.get();
    for (int i = T; i >= 0; --i) {
        c.cur_level = i;
        DistLevel& L = d.lv[i];
        vc_prolong(c, L.n_own, L.u0.get(), L.agg.get(), uc, L.x.get(), g);
        double* out = (i == 0) ? u_out : L.out.get();
        if (overlapped(d, L)) {
            halo(d, L, L.x.get(), g, true);
            vc_smooth(c, L.view(), fin[i], L.w.get(), om, L.x.get(), out, g);
            halo_join(d);
            vc_smooth_rows(c, L.view(), L.brows.get(), L.nb, fin[i], L.w.get(), om, L.x.get(), out, g);
        } else {
            halo(d, L, L.x.get(), g);
            vc_smooth(c, L.view(), fin[i], L.w.get(), om, L.x.get(), out, g);
        }
        uc = out;
    }
    c.cur_level = -1;
}

// the communicator and events of a handle (also of a failed amgr_dist_create)
DistHier::~DistHier() {
    if (comm) {
        if (const NcclApi* a = nccl_api()) a->CommDestroy(comm);
    }
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_consumed) cudaEventDestroy(ev_consumed);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (cs) cudaStreamDestroy(cs);
}

// Plan validation, before any communicator is created: every index the
// kernels and exchanges will use is in range and the transition counts agree.
static void validate_plan(const Hier& H, int rank, int world, int top, const amgr_dist_level* levels,
                          const int64_t* t_counts) {
    auto bad = [&](int i, const char* what) {
        std::ostringstream os;
        os << "amgr_dist_create: level " << i << ": " << what;
        invalid(os.str());
    };
    auto in = [](const int64_t* a, int64_t n, int64_t lo, int64_t hi) {
        for (int64_t k = 0; k < n; ++k)
            if (a[k] < lo || a[k] >= hi) return false;
        return true;
    };
    for (int r = 0; r < world; ++r)
        if (t_counts[r] < 0) invalid("amgr_dist_create: negative transition count");
    for (int i = 0; i <= top; ++i) {
        const amgr_dist_level& s = levels[i];
        const int64_t ng = H.lv[i].pat->n, nnzg = H.lv[i].pat->nnz;
        if (s.n_own < 0 || s.n_halo < 0 || s.nnz < 0 || s.n_coarse_owned < 0 || s.n_own > ng) bad(i, "bad sizes");
        if (!s.row_ptr || s.row_ptr[0] != 0 || s.row_ptr[s.n_own] != s.nnz) bad(i, "row_ptr does not span nnz");
        for (int64_t r = 0; r < s.n_own; ++r)
            if (s.row_ptr[r + 1] < s.row_ptr[r]) bad(i, "row_ptr decreasing");
        if (!in(s.col, s.nnz, 0, s.n_own + s.n_halo)) bad(i, "column id out of [0, n_own + n_halo)");
        if (!in(s.nnz_map, s.nnz, 0, nnzg)) bad(i, "nnz_map out of the global level");
        if (!in(s.owned, s.n_own, 0, ng)) bad(i, "owned row out of the global level");
        const int64_t nc_local = i < top ? levels[i + 1].n_own : H.lv[top + 1].pat->n;
        if (!in(s.agg, s.n_own, 0, nc_local)) bad(i, "aggregate id out of range");
        if (i < top && s.n_coarse_owned != levels[i + 1].n_own) bad(i, "owned coarse rows != next level's rows");
        if (i == top && s.n_coarse_owned != t_counts[rank]) bad(i, "owned coarse rows != this rank's transition count");
        if (!s.mptr || s.mptr[0] != 0) bad(i, "member pointers");
        for (int64_t r = 0; r < s.n_coarse_owned; ++r)
            if (s.mptr[r + 1] < s.mptr[r]) bad(i, "member pointers decreasing");
        if (!in(s.midx, s.mptr[s.n_coarse_owned], 0, s.n_own)) bad(i, "member id out of the owned rows");
        int64_t sent = 0;
        for (int k = 0; k < s.n_send_peers; ++k) {
            if (s.send_peer[k] < 0 || s.send_peer[k] >= world || s.send_peer[k] == rank) bad(i, "bad send peer");
            if (s.send_cnt[k] < 0) bad(i, "negative send count");
            sent += s.send_cnt[k];
        }
        if (!in(s.send_idx, sent, 0, s.n_own)) bad(i, "send index out of the owned rows");
        for (int k = 0; k < s.n_recv_peers; ++k) {
            if (s.recv_peer[k] < 0 || s.recv_peer[k] >= world || s.recv_peer[k] == rank) bad(i, "bad recv peer");
            if (s.recv_off[k] < 0 || s.recv_cnt[k] < 0 || s.recv_off[k] + s.recv_cnt[k] > s.n_halo)
                bad(i, "recv block outside the halo");
        }
    }
}

static void gather_local(DistHier& d) {
    Ctx& c = *d.ctx;
    Hier& h = *d.g;
    for (int i = 0; i <= d.T; ++i) {
        DistLevel& L = d.lv[i];
        const Level& G = h.lv[i];
        LAUNCH(c, "dist", 0.0, k_gather_d, grid_for(L.nnz, 256, c.num_sms * 16), 256, 0, L.nnz, G.view().val,
               L.nnz_map.get(), L.val.get(), Gate{});
        LAUNCH(c, "dist", 0.0, k_gather_d, grid_for(L.n_own, 256, c.num_sms * 16), 256, 0, L.n_own, G.w.get(),
               L.owned.get(), L.w.get(), Gate{});
    }
}

// Local Galerkin plans for the partitioned rebuild, built on the device from
// the global plan (setup.cuh RapSymbolic) of every partitioned level.
static void build_local_plans(DistHier& d) {
    Ctx& c = *d.ctx;
    Hier& h = *d.g;
    for (int i = 0; i <= d.T; ++i) {
        DistLevel& L = d.lv[i];
        const Level& G = h.lv[i];
        const Level& GC = h.lv[i + 1];
        if (!G.rap || G.T->smoothed) fail(AMGR_E_RUNTIME, "dist: level without a plain Galerkin plan");
        LAUNCH(c, "dist", 0.0, k_local_diag, grid_for(L.n_own, 256, c.num_sms * 8), 256, 0, L.n_own, L.rp.get(),
               L.col.get(), L.dpos.get());
        DevArray<int> ginv(G.pat->nnz, c.stream);
        CK(cudaMemsetAsync(ginv.get(), 0xff, sizeof(int) * static_cast<size_t>(G.pat->nnz), c.stream));
        LAUNCH(c, "dist", 0.0, k_scatter_inv, grid_for(L.nnz, 256, c.num_sms * 8), 256, 0, L.nnz, L.nnz_map.get(),
               ginv.get());
        // this rank's coarse rows: the owned rows of level i+1, or at the top
        // its contiguous transition range of level T+1
        const int* crow = nullptr;
        int64_t base = 0, nrows = 0;
        const int* lrp = nullptr;
        DevArray<int> trp;
        if (i < d.T) {
            crow = d.lv[i + 1].owned.get();
            nrows = d.lv[i + 1].n_own;
            lrp = d.lv[i + 1].rp.get();
        } else {
            base = d.tdispl[d.rank];
            nrows = d.tcnt[d.rank];
            std::vector<int> grp(static_cast<size_t>(nrows + 1));
            d2h(grp.data(), GC.pat->rp.get() + base, nrows + 1, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            const int off = grp[0];
            for (auto& x : grp) x -= off;
            trp.alloc(nrows + 1, c.stream);
            h2d(trp.get(), grp.data(), nrows + 1, c.stream);
            lrp = trp.get();
        }
        L.lnc = nrows;
        int nent = 0;
        if (nrows > 0) d2h(&nent, lrp + nrows, 1, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        L.lnnz_c = nent;
        DevArray<int> cnt(std::max(nent, 1), c.stream);
        L.lcptr.alloc(nent + 1, c.stream);
        if (nrows > 0)
            LAUNCH(c, "dist", 0.0, k_lplan_count, grid_for(nrows, 256, c.num_sms * 8), 256, 0, nrows, crow, base,
                   GC.pat->rp.get(), lrp, G.rap->cptr.get(), cnt.get());
        if (nent > 0) exclusive_sum_i32(c, cnt.get(), L.lcptr.get(), nent);
        LAUNCH(c, "dist", 0.0, k_set_last, 1, 1, 0, L.lcptr.get(), static_cast<int64_t>(nent), cnt.get());
        int total = 0;
        d2h(&total, L.lcptr.get() + nent, 1, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        if (total != L.nnz)
            fail(AMGR_E_RUNTIME, "dist: local Galerkin plan does not cover the local entries (partition not "
                                 "aggregate-consistent)");
        L.lcontrib.alloc(std::max(total, 1), c.stream);
        DevArray<int> bad(1, c.stream);
        CK(cudaMemsetAsync(bad.get(), 0, sizeof(int), c.stream));
        if (nrows > 0)
            LAUNCH(c, "dist", 0.0, k_lplan_fill, grid_for(nrows, 256, c.num_sms * 8), 256, 0, nrows, crow, base,
                   GC.pat->rp.get(), lrp, G.rap->cptr.get(), G.rap->contrib.get(), ginv.get(), L.lcptr.get(),
                   L.lcontrib.get(), bad.get());
        if (d2h_scalar(bad.get(), c.stream)) fail(AMGR_E_RUNTIME, "dist: a member row of an owned aggregate is not local");
        L.lmax_chunk = rap_chunk_max(c, L.lnnz_c, L.lcptr.get());
        const char* ge = std::getenv("AMGR_RAP_GROUPS");
        if (!(ge && ge[0] == '0') && L.n_own > 0 && nrows > 0)
            rap_grp_plan(c, L.view(), L.mptr.get(), L.midx.get(), L.dpos.get(), nrows, lrp, L.lnnz_c,
                         L.lcptr.get(), L.lcontrib.get(), L.grp);
    }
    // transition values: entry ranges of every rank's level-(T+1) rows
    const Level& GT = h.lv[d.T + 1];
    std::vector<int> grp(static_cast<size_t>(GT.pat->n + 1));
    d2h(grp.data(), GT.pat->rp.get(), GT.pat->n + 1, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    d.tvcnt.clear();
    d.tvdispl.clear();
    d.tvpad = 0;
    for (int r = 0; r < d.world; ++r) {
        const int64_t a = grp[static_cast<size_t>(d.tdispl[r])], b = grp[static_cast<size_t>(d.tdispl[r] + d.tcnt[r])];
        d.tvdispl.push_back(a);
        d.tvcnt.push_back(b - a);
        d.tvpad = std::max<int64_t>(d.tvpad, b - a);
    }
    d.tvsend.alloc(std::max<int64_t>(d.tvpad, 1), c.stream);
    d.tvgather.alloc(std::max<int64_t>(d.tvpad * d.world, 1), c.stream);
    d.tvcnt_d.alloc(d.world, c.stream);
    d.tvdispl_d.alloc(d.world, c.stream);
    h2d(d.tvcnt_d.get(), d.tvcnt.data(), d.world, c.stream);
    h2d(d.tvdispl_d.get(), d.tvdispl.data(), d.world, c.stream);
    d.lerr.alloc(d.T + 1, c.stream);
    d.errd.alloc(d.T + 1, c.stream);
    d.errall.alloc(static_cast<int64_t>(d.T + 1) * d.world, c.stream);
}

// Partial rebuild from rank-local values (hierarchy.cpp:107-150 on the
// partition): each rank rebuilds the Jacobi weights of its rows and the
// numeric Galerkin product of its coarse rows from its own A_i entries
// (communication-free: every member row is local), down to its rows of
// A_{T+1}; one allgather replicates A_{T+1}; the replicated levels are
// rebuilt on every rank.  Values and errors are those of the global rebuild.
static void dist_rebuild_local(DistHier& d, const double* vals, int location) {
    Ctx& c = *d.ctx;
    Hier& h = *d.g;
    DistLevel& L0 = d.lv[0];
    CK(cudaMemcpyAsync(L0.val.get(), vals, sizeof(double) * static_cast<size_t>(L0.nnz),
                       location == AMGR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    std::vector<int> big(static_cast<size_t>(d.T + 1), 0x7fffffff);
    h2d(d.lerr.get(), big.data(), d.T + 1, c.stream);
    for (int i = 0; i <= d.T; ++i) {
        c.cur_level = i;
        DistLevel& L = d.lv[i];
        double* out = i < d.T ? d.lv[i + 1].val.get() : d.tvsend.get();
        if (L.grp.ok) {  // Galerkin + damped-Jacobi rebuild in one pass
            GrpArgs ga;
            ga.ngroups = L.grp.ngroups;
            ga.desc = L.grp.desc.get();
            ga.mstart = L.grp.mstart.get();
            ga.mdoff = L.grp.mdoff.get();
            ga.midx = L.midx.get();
            ga.code = L.grp.code.get();
            ga.lanes = L.grp.lanes.get();
            ga.af = L.val.get();
            ga.ac = out;
            ga.wf = L.w.get();
            ga.bad_f = d.lerr.get() + i;
            rap_grp(c, ga, L.n_own, L.lnc, L.nnz, L.lnnz_c);
        } else {
            jacobi_rebuild(c, L.n_own, L.val.get(), L.dpos.get(), L.w.get(), d.lerr.get() + i);
            rap_numeric(c, L.n_own, L.lnc, L.lnnz_c, L.lcptr.get(), L.lcontrib.get(), L.val.get(), out, L.nnz,
                        L.lmax_chunk);
        }
    }
    c.cur_level = d.T + 1;
    allgather(d, d.tvsend.get(), d.tvgather.get(), d.tvpad);
    LAUNCH(c, "dist", 0.0, k_unpad, grid_for(d.tvpad, 256, 64), 256, 0, d.world, d.tvpad, d.tvgather.get(),
           d.tvdispl_d.get(), d.tvcnt_d.get(), h.lv[d.T + 1].val.get());
    // the first bad row of each partitioned level, as a global row id, the
    // minimum over ranks (every rank throws the same error)
    std::vector<int> le(static_cast<size_t>(d.T + 1));
    d2h(le.data(), d.lerr.get(), d.T + 1, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    std::vector<double> ge(static_cast<size_t>(d.T + 1));
    for (int i = 0; i <= d.T; ++i) {
        double g = 1e300;
        if (le[i] != 0x7fffffff) {
            int row = 0;
            d2h(&row, d.lv[i].owned.get() + le[i], 1, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            g = row;
        }
        ge[i] = g;
    }
    h2d(d.errd.get(), ge.data(), d.T + 1, c.stream);
    allgather(d, d.errd.get(), d.errall.get(), d.T + 1);
    std::vector<double> all(static_cast<size_t>((d.T + 1) * d.world));
    d2h(all.data(), d.errall.get(), (d.T + 1) * d.world, c.stream);
    CK(cudaStreamSynchronize(c.stream));
    for (int i = 0; i <= d.T; ++i) {
        double m = 1e300;
        for (int r = 0; r < d.world; ++r) m = std::min(m, all[static_cast<size_t>(r * (d.T + 1) + i)]);
        if (m < 1e300) {
            std::ostringstream os;
            os << "level " << i << ": build_smoother: zero diagonal at row " << static_cast<int64_t>(m);
            invalid(os.str());
        }
    }
    rebuild_levels_from(h, static_cast<size_t>(d.T + 1));
    c.cur_level = -1;
}

// common tail of amgr_dist_create*: transition layout, local work vectors,
// local values/weights, local Galerkin plans
static void dist_finish(DistHier& d, const int64_t* t_counts, int64_t t_count_total) {
    Hier& H = *d.g;
    Ctx& c = *d.ctx;
    const int world = d.world, top = d.T;
    // transition allgather layout
    int64_t disp = 0;
    for (int r = 0; r < world; ++r) {
        d.tcnt.push_back(t_counts[r]);
        d.tdispl.push_back(disp);
        disp += t_counts[r];
        d.tpad = std::max<int64_t>(d.tpad, t_counts[r]);
    }
    if (disp != t_count_total || disp != H.lv[top + 1].pat->n)
        invalid("amgr_dist_create: transition counts do not cover level top+1");
    d.tsend.alloc(std::max<int64_t>(d.tpad, 1), c.stream);
    d.tgather.alloc(std::max<int64_t>(d.tpad * world, 1), c.stream);
    d.tcnt_d.alloc(world, c.stream);
    d.tdispl_d.alloc(world, c.stream);
    h2d(d.tcnt_d.get(), d.tcnt.data(), world, c.stream);
    h2d(d.tdispl_d.get(), d.tdispl.data(), world, c.stream);
    d.fT.alloc(disp, c.stream);
    d.uT.alloc(disp, c.stream);
    const int64_t n0 = d.lv[0].n_own, h0 = d.lv[0].n_halo;
    for (auto* v : {&d.kr, &d.krt, &d.kp, &d.kv, &d.ks, &d.kt}) v->alloc(n0, c.stream);
    for (auto* v : {&d.kph, &d.ksh, &d.ku}) v->alloc(n0 + h0, c.stream);
    d.dloc.alloc(4, c.stream);
    d.dall.alloc(4 * world, c.stream);
    d.douts.alloc(64, c.stream);
    work(H);
    gather_local(d);
    build_local_plans(d);
    // halo overlap (world > 1, AMGR_DIST_OVERLAP=0 disables): the owned rows
    // with a halo column, per partitioned level, and a stream for exchanges
    const char* ov = std::getenv("AMGR_DIST_OVERLAP");
    d.overlap = world > 1 && !(ov && ov[0] == '0');
    if (d.overlap) {
        CK(cudaStreamCreateWithFlags(&d.cs, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&d.ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&d.ev_join, cudaEventDisableTiming));
        for (auto& L : d.lv) {
            if (L.n_halo == 0 || L.n_own == 0) continue;
            DevArray<char> flag(L.n_own, c.stream);
            LAUNCH(c, "dist", 0.0, k_halo_rows, grid_for(L.n_own, 256, c.num_sms * 8), 256, 0, L.n_own, L.rp.get(),
                   L.col.get(), flag.get());
            L.nb = select_flagged(c, flag.get(), L.n_own, L.brows);
        }
    }
}

// levels of a device-built plan (dist_plan.cu): the arrays move in as they are
static void levels_from_device_plan(DistHier& d, DevicePlan& P) {
    Ctx& c = *d.ctx;
    d.lv.resize(static_cast<size_t>(P.top + 1));
    for (int i = 0; i <= P.top; ++i) {
        PlanLevel& s = P.lv[i];
        DistLevel& L = d.lv[i];
        L.n_own = s.n_own;
        L.n_halo = s.n_halo;
        L.nnz = s.nnz;
        L.n_cown = s.n_cown;
        L.rp = std::move(s.rp);
        L.col = std::move(s.col);
        L.nnz_map = std::move(s.nnz_map);
        L.owned = std::move(s.owned);
        L.agg = std::move(s.agg);
        L.mptr = std::move(s.mptr);
        L.midx = std::move(s.midx);
        L.send_idx = std::move(s.send_idx);
        L.val.alloc(s.nnz, c.stream);
        L.w.alloc(s.n_own, c.stream);
        L.dpos.alloc(s.n_own, c.stream);
        L.u0.alloc(s.n_own + s.n_halo, c.stream);
        L.x.alloc(s.n_own + s.n_halo, c.stream);
        L.out.alloc(s.n_own, c.stream);
        L.f.alloc(s.n_own, c.stream);
        L.r.alloc(s.n_own, c.stream);
        int64_t off = 0;
        for (size_t k = 0; k < s.send_peer.size(); ++k) {
            L.send_peer.push_back(s.send_peer[k]);
            L.send_off.push_back(off);
            L.send_cnt.push_back(s.send_cnt[k]);
            off += s.send_cnt[k];
        }
        L.send_buf.alloc(off, c.stream);
        L.recv_peer = s.recv_peer;
        L.recv_off = s.recv_off;
        L.recv_cnt = s.recv_cnt;
        L.max_span = max_group_span(c, L.rp.get(), L.n_own);
        encode_columns(c, L.n_own, L.nnz, L.rp.get(), L.col.get(), L.cc, true);
    }
}

}  // namespace amgr

// ---- C-ABI ----------------------------------------------------------------------
struct amgr_dist {
    std::unique_ptr<amgr::DistHier> d;
};

extern "C" {

amgr_status amgr_nccl_unique_id(void* out128) {
    if (!out128) return AMGR_E_INVALID_ARGUMENT;
    ncclUniqueId id;
    const amgr::NcclApi* api = amgr::nccl_api();
    if (!api || api->GetUniqueId(&id) != ncclSuccess) return AMGR_E_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
    return AMGR_OK;
}

static amgr_status dist_create_impl(amgr_hier* hg, int rank, int world, int top, const amgr_dist_level* levels,
                                    int64_t t_count_total, const int64_t* t_counts, amgr_dist** out,
                                    const std::function<void(amgr::DistHier&)>& connect) {
    if (!hg || !out || (top >= 0 && !levels) || world < 1 || rank < 0 || rank >= world)
        return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    amgr::Hier& H = *hg->h;
    amgr::Ctx& c = *H.ctx;
    try {
        CK(cudaSetDevice(c.device));
        if (top < 0 || top + 1 >= static_cast<int>(H.lv.size()))
            amgr::invalid("amgr_dist_create: need 0 <= top < num_levels - 1");
        if (H.prm.pre != 1 || H.prm.post != 1 || H.prm.smoother == AMGR_SMOOTHER_CHEBYSHEV)
            amgr::invalid("amgr_dist_create: the partitioned solve supports 1+1 Jacobi/SPAI0 sweeps");
        for (const auto& l : H.lv)
            if (l.T && l.T->smoothed)
                amgr::invalid("amgr_dist_create: the partitioned solve supports plain (tentative) aggregation only");
        amgr::validate_plan(H, rank, world, top, levels, t_counts);
        auto d = std::make_unique<amgr::DistHier>();
        d->g = &H;
        d->ctx = &c;
        d->rank = rank;
        d->world = world;
        d->T = top;
        connect(*d);  // after validation; a later failure destroys d (and its communicator)
        auto up32 = [&](amgr::DevArray<int>& dst, const int64_t* src, int64_t n) {
            std::vector<int> tmp(static_cast<size_t>(n));
            for (int64_t k = 0; k < n; ++k) tmp[k] = static_cast<int>(src[k]);
            dst.alloc(n, c.stream);
            amgr::h2d(dst.get(), tmp.data(), n, c.stream);
        };
        d->lv.resize(static_cast<size_t>(top + 1));
        for (int i = 0; i <= top; ++i) {
            const amgr_dist_level& s = levels[i];
            amgr::DistLevel& L = d->lv[i];
            L.n_own = s.n_own;
            L.n_halo = s.n_halo;
            L.nnz = s.nnz;
            L.n_cown = s.n_coarse_owned;
            up32(L.rp, s.row_ptr, s.n_own + 1);
            up32(L.col, s.col, s.nnz);
            up32(L.nnz_map, s.nnz_map, s.nnz);
            up32(L.owned, s.owned, s.n_own);
            up32(L.agg, s.agg, s.n_own);
            up32(L.mptr, s.mptr, s.n_coarse_owned + 1);
            up32(L.midx, s.midx, s.mptr[s.n_coarse_owned]);
            L.val.alloc(s.nnz, c.stream);
            L.w.alloc(s.n_own, c.stream);
            L.dpos.alloc(s.n_own, c.stream);
            L.u0.alloc(s.n_own + s.n_halo, c.stream);
            L.x.alloc(s.n_own + s.n_halo, c.stream);
            L.out.alloc(s.n_own, c.stream);
            L.f.alloc(s.n_own, c.stream);
            L.r.alloc(s.n_own, c.stream);
            int64_t off = 0;
            for (int k = 0; k < s.n_send_peers; ++k) {
                L.send_peer.push_back(s.send_peer[k]);
                L.send_off.push_back(off);
                L.send_cnt.push_back(s.send_cnt[k]);
                off += s.send_cnt[k];
            }
            up32(L.send_idx, s.send_idx, off);
            L.send_buf.alloc(off, c.stream);
            for (int k = 0; k < s.n_recv_peers; ++k) {
                L.recv_peer.push_back(s.recv_peer[k]);
                L.recv_off.push_back(s.recv_off[k]);
                L.recv_cnt.push_back(s.recv_cnt[k]);
            }
            L.max_span = amgr::max_group_span(c, L.rp.get(), L.n_own);
            // local columns keep the stencil offsets of owned neighbours; halo
            // columns (numbered after the owned rows) add distinct offsets:
            // 1-byte codes when there are few, 2-byte codes up to 65536
            amgr::encode_columns(c, L.n_own, L.nnz, L.rp.get(), L.col.get(), L.cc, true);
        }
        amgr::dist_finish(*d, t_counts, t_count_total);
        CK(cudaStreamSynchronize(c.stream));
        auto* o = new amgr_dist();
        o->d = std::move(d);
        *out = o;
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

amgr_status amgr_dist_create(amgr_hier* hg, const void* nccl_id128, int rank, int world, int top,
                             const amgr_dist_level* levels, int64_t t_count_total, const int64_t* t_counts,
                             amgr_dist** out) {
    if (!nccl_id128) return AMGR_E_INVALID_ARGUMENT;
    return dist_create_impl(hg, rank, world, top, levels, t_count_total, t_counts, out, [&](amgr::DistHier& d) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id128, sizeof(id));
        NK(::amgr::N().CommInitRank(&d.comm, world, id, rank));
    });
}

amgr_status amgr_dist_loopback_create(int world, amgr_loopback** out) {
    if (!out || world < 1) return AMGR_E_INVALID_ARGUMENT;
    *out = reinterpret_cast<amgr_loopback*>(new amgr::Loopback(world));
    return AMGR_OK;
}

void amgr_dist_loopback_destroy(amgr_loopback* lb) { delete reinterpret_cast<amgr::Loopback*>(lb); }

amgr_status amgr_dist_create_loopback(amgr_hier* hg, amgr_loopback* lbh, int rank, int world, int top,
                                      const amgr_dist_level* levels, int64_t t_count_total, const int64_t* t_counts,
                                      amgr_dist** out) {
    auto* lb = reinterpret_cast<amgr::Loopback*>(lbh);
    if (!lb || lb->world != world) return AMGR_E_INVALID_ARGUMENT;
    return dist_create_impl(hg, rank, world, top, levels, t_count_total, t_counts, out, [&](amgr::DistHier& d) {
        d.lb = lb;
        CK(cudaEventCreateWithFlags(&d.ev_ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&d.ev_consumed, cudaEventDisableTiming));
    });
}

static amgr_status dist_create_auto_impl(amgr_hier* hg, int rank, int world, int64_t replicate_below,
                                         amgr_dist** out, const std::function<void(amgr::DistHier&)>& connect) {
    if (!hg || !out || world < 1 || rank < 0 || rank >= world) return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    amgr::Hier& H = *hg->h;
    amgr::Ctx& c = *H.ctx;
    try {
        CK(cudaSetDevice(c.device));
        if (H.prm.pre != 1 || H.prm.post != 1 || H.prm.smoother == AMGR_SMOOTHER_CHEBYSHEV)
            amgr::invalid("amgr_dist_create: the partitioned solve supports 1+1 Jacobi/SPAI0 sweeps");
        amgr::DevicePlan P = amgr::build_device_plan(H, rank, world, replicate_below);  // before any communicator
        auto d = std::make_unique<amgr::DistHier>();
        d->g = &H;
        d->ctx = &c;
        d->rank = rank;
        d->world = world;
        d->T = P.top;
        connect(*d);
        amgr::levels_from_device_plan(*d, P);
        int64_t tot = 0;
        for (int64_t t : P.t_counts) tot += t;
        amgr::dist_finish(*d, P.t_counts.data(), tot);
        CK(cudaStreamSynchronize(c.stream));
        auto* o = new amgr_dist();
        o->d = std::move(d);
        *out = o;
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

amgr_status amgr_dist_create_auto(amgr_hier* hg, const void* nccl_id128, int rank, int world,
                                  int64_t replicate_below, amgr_dist** out) {
    if (!nccl_id128) return AMGR_E_INVALID_ARGUMENT;
    return dist_create_auto_impl(hg, rank, world, replicate_below, out, [&](amgr::DistHier& d) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id128, sizeof(id));
        NK(::amgr::N().CommInitRank(&d.comm, world, id, rank));
    });
}

amgr_status amgr_dist_create_auto_loopback(amgr_hier* hg, amgr_loopback* lbh, int rank, int world,
                                           int64_t replicate_below, amgr_dist** out) {
    auto* lb = reinterpret_cast<amgr::Loopback*>(lbh);
    if (!lb || lb->world != world) return AMGR_E_INVALID_ARGUMENT;
    return dist_create_auto_impl(hg, rank, world, replicate_below, out, [&](amgr::DistHier& d) {
        d.lb = lb;
        CK(cudaEventCreateWithFlags(&d.ev_ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&d.ev_consumed, cudaEventDisableTiming));
    });
}

// dims: {n_own, n_halo, nnz, n_coarse_owned, top}
amgr_status amgr_dist_level_dims(const amgr_dist* d, int level, int64_t* dims) {
    if (!d || !d->d || !dims || level < 0 || level > d->d->T) return AMGR_E_INVALID_ARGUMENT;
    const amgr::DistLevel& L = d->d->lv[level];
    dims[0] = L.n_own;
    dims[1] = L.n_halo;
    dims[2] = L.nnz;
    dims[3] = L.n_cown;
    dims[4] = d->d->T;
    return AMGR_OK;
}

amgr_status amgr_dist_level_code(const amgr_dist* d, int level, int* col_bytes) {
    if (!d || !d->d || !col_bytes || level < 0 || level > d->d->T) return AMGR_E_INVALID_ARGUMENT;
    const int m = d->d->lv[level].cc.mode;
    *col_bytes = m == 1 ? 1 : m == 2 ? 2 : 4;
    return AMGR_OK;
}

void amgr_dist_destroy(amgr_dist* d) { delete d; }  // ~DistHier releases the communicator and events

static amgr_status dist_guard(amgr_dist* d, const std::function<void()>& fn) {
    if (!d || !d->d) return AMGR_E_INVALID_ARGUMENT;
    amgr::Ctx& c = *d->d->ctx;
    try {
        CK(cudaSetDevice(c.device));
        fn();
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

// owned: n_own global rows; nnz_map: nnz global entry ids (either may be null)
amgr_status amgr_dist_level_maps(amgr_dist* d, int level, int64_t* owned, int64_t* nnz_map) {
    if (!d || !d->d || level < 0 || level > d->d->T) return AMGR_E_INVALID_ARGUMENT;
    return dist_guard(d, [&] {
        amgr::DistLevel& L = d->d->lv[level];
        amgr::Ctx& c = *d->d->ctx;
        std::vector<int> tmp;
        if (owned) {
            tmp.resize(static_cast<size_t>(L.n_own));
            amgr::d2h(tmp.data(), L.owned.get(), L.n_own, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            for (int64_t k = 0; k < L.n_own; ++k) owned[k] = tmp[static_cast<size_t>(k)];
        }
        if (nnz_map) {
            tmp.resize(static_cast<size_t>(L.nnz));
            amgr::d2h(tmp.data(), L.nnz_map.get(), L.nnz, c.stream);
            CK(cudaStreamSynchronize(c.stream));
            for (int64_t k = 0; k < L.nnz; ++k) nnz_map[k] = tmp[static_cast<size_t>(k)];
        }
    });
}

amgr_status amgr_dist_rebuild_values(amgr_dist* d, const double* global_values, int location) {
    return dist_guard(d, [&] {
        amgr::rebuild_values(*d->d->g, global_values, location);
        amgr::gather_local(*d->d);
    });
}

amgr_status amgr_dist_rebuild_local(amgr_dist* d, const double* local_values, int location) {
    if (!local_values) return AMGR_E_INVALID_ARGUMENT;
    return dist_guard(d, [&] { amgr::dist_rebuild_local(*d->d, local_values, location); });
}

amgr_status amgr_dist_vcycle(amgr_dist* d, const double* f_local, double* u_local) {
    return dist_guard(d, [&] { amgr::dist_vcycle(*d->d, f_local, u_local, amgr::Gate{}); });
}

}  // extern "C"

namespace amgr {

// BiCGStab (bicgstab.cpp:21-135) on the partition: local vectors of the owned
// level-0 rows, halo exchange before every level-0 SpMV, rank-ordered dots.
void dist_bicgstab(DistHier& d, const double* f, double* u, const amgr_solve_params& sp, amgr_solve_stats& out) {
    Ctx& c = *d.ctx;
    Hier& h = *d.g;
    DistLevel& L0 = d.lv[0];
    const CsrView A = L0.view();
    const int64_t n = L0.n_own;
    KState* st = work(h).st.get();
    out = amgr_solve_stats{0, 0.0, 0, 0};
    auto rd = [&]() {
        KState s;
        d2h(&s, st, 1, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        return s;
    };
    // sequential-dot parity mode (amgr_ctx_set_dot_order on this rank's
    // context; every rank must use the same order): after each rank-ordered
    // dot the reference's left-to-right global dot overwrites the field, at
    // the same places as the single-GPU solver (hierarchy.cu::bicgstab)
    const bool seq = c.seq_dots;
    if (d.world > 1) {
        // every rank must sum its dots the same way (a mismatch would leave
        // the ranks in different collective sequences): agree first, fail
        // together with a message otherwise
        DevArray<double> mine, all;
        mine.alloc(1, c.stream);
        all.alloc(d.world, c.stream);
        const double flag = seq ? 1.0 : 0.0;
        h2d(mine.get(), &flag, 1, c.stream);
        allgather(d, mine.get(), all.get(), 1);
        std::vector<double> flags(static_cast<size_t>(d.world));
        d2h(flags.data(), all.get(), d.world, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        for (double v : flags)
            if (v != flags[0])
                fail(AMGR_E_INVALID_ARGUMENT, "dist bicgstab: the ranks' contexts use different dot orders");
    }
    if (seq) seq_prepare(d);
    auto SD = [&](const double* a, const double* b, double* o, Gate g = {}) {
        if (seq) seq_dot_dist(d, a, b, o, g);
    };
    // ||f - A u||^2 into *o: rank-ordered, then (sequential mode) the
    // reference's sum over r = f - A u written to a scratch vector
    auto true_resid = [&](double* u_, double* o, Gate g) {
        resid_norm(c, A, f, u_, seq ? d.kq.get() : nullptr, nullptr, local_sink(d, 0), g);
        allsum(d, 1, {o});
        SD(d.kq.get(), d.kq.get(), o, g);
    };
    KState s0;
    h2d(st, &s0, 1, c.stream);
    dot(c, n, f, f, local_sink(d, 0));
    allsum(d, 1, {&st->d_true});
    SD(f, f, &st->d_true);
    KState s = rd();
    const double normf = std::sqrt(s.d_true);
    if (normf == 0.0) {
        fill(c, u, n, 0.0);
        out.converged = 1;
        return;
    }
    copy(c, d.ku.get(), u, n);  // u (with halo space) starts from the caller's guess
    double* uu = d.ku.get();
    halo(d, L0, uu, Gate{});
    resid_norm(c, A, f, uu, d.kr.get(), d.krt.get(), local_sink(d, 0));
    dot(c, n, d.krt.get(), d.kr.get(), local_sink(d, 1));
    allsum(d, 2, {&st->d_rr, &st->d_rtr});
    SD(d.kr.get(), d.kr.get(), &st->d_rr);
    SD(d.krt.get(), d.kr.get(), &st->d_rtr);
    s = rd();
    out.relative_residual = std::sqrt(s.d_rr) / normf;
    if (out.relative_residual <= sp.tol) {
        out.converged = 1;
        copy(c, u, uu, n);
        return;
    }
    s.normf = normf;
    s.floor = 1e-30 * normf * normf;
    s.tol = sp.tol;
    s.max_iter = sp.max_iter;
    s.rho_old = s.alpha = s.omega = 1.0;
    s.it = 0;
    s.flags = 0;
    h2d(st, &s, 1, c.stream);
    const Gate G = gate_of(st, KF_DONE);
    const Gate GH = gate_of(st, KF_DONE, KF_HALF);
    const Gate GF = gate_of(st, KF_DONE | KF_HALF);
    const Gate GC = gate_of(st, KF_DONE | KF_HALF, KF_CHECK);
    // one iteration of look-ahead, no per-iteration host sync; over NCCL the
    // iteration is captured once into a CUDA graph (halo send/recv and the
    // allgathers are capturable); the loopback test transport synchronises
    // host threads while enqueuing and runs kernel by kernel
    for (auto outs : {std::initializer_list<double*>{&st->d_rtv}, {&st->d_ss}, {&st->d_true}, {&st->d_rtr},
                      {&st->d_ts, &st->d_tt}, {&st->d_rr, &st->d_rtr}})
        out_slot(d, outs);  // register before any capture
    auto iter = [&]() {
        bicg_begin(c, st);
        bicg_p(c, st, n, d.kr.get(), d.kp.get(), d.kv.get());
        dist_vcycle(d, d.kp.get(), d.kph.get(), G);
        halo(d, L0, d.kph.get(), G);
        spmv_dot(c, A, d.kph.get(), d.kv.get(), d.krt.get(), local_sink(d, 0), G);
        allsum(d, 1, {&st->d_rtv});
        SD(d.krt.get(), d.kv.get(), &st->d_rtv, G);
        bicg_alpha(c, st);
        bicg_s(c, st, n, d.kr.get(), d.kv.get(), d.ks.get(), local_sink(d, 0));
        allsum(d, 1, {&st->d_ss});
        SD(d.ks.get(), d.ks.get(), &st->d_ss, G);
        bicg_half_test(c, st);
        bicg_half_u(c, st, n, uu, d.kph.get());
        halo(d, L0, uu, GH);
        true_resid(uu, &st->d_true, GH);
        bicg_half_check(c, st);
        bicg_half_r(c, st, n, d.kr.get(), d.ks.get(), d.krt.get(), local_sink(d, 0));
        allsum(d, 1, {&st->d_rtr});  // stale when gated off; bicg_update rewrites d_rtr then
        SD(d.krt.get(), d.kr.get(), &st->d_rtr, GH);
        dist_vcycle(d, d.ks.get(), d.ksh.get(), GF);
        halo(d, L0, d.ksh.get(), GF);
        spmv_dot2(c, A, d.ksh.get(), d.kt.get(), d.ks.get(), local_sink(d, 0), GF);
        allsum(d, 2, {&st->d_ts, &st->d_tt});
        SD(d.kt.get(), d.ks.get(), &st->d_ts, GF);
        SD(d.kt.get(), d.kt.get(), &st->d_tt, GF);
        bicg_omega(c, st);
        bicg_update(c, st, n, uu, d.kph.get(), d.ksh.get(), d.kr.get(), d.ks.get(), d.kt.get(), d.krt.get(),
                    local_sink(d, 0));
        allsum(d, 2, {&st->d_rr, &st->d_rtr});
        SD(d.kr.get(), d.kr.get(), &st->d_rr, GF);
        SD(d.krt.get(), d.kr.get(), &st->d_rtr, GF);
        bicg_end_test(c, st);
        halo(d, L0, uu, GC);
        true_resid(uu, &st->d_true, GC);
        bicg_end_check(c, st);
    };
    run_iterations(h, iter, s, d.lb == nullptr && !std::getenv("AMGR_DIST_NO_GRAPH"));
    out.iterations = s.it;
    if (s.flags & KF_CONVERGED) {
        out.converged = 1;
        out.relative_residual = s.res;
    } else {
        out.breakdown = (s.flags & KF_BREAKDOWN) ? 1 : 0;
        halo(d, L0, uu, Gate{});
        true_resid(uu, &st->d_true, Gate{});
        s = rd();
        out.relative_residual = std::sqrt(s.d_true) / normf;
        out.converged = (out.relative_residual <= sp.tol && !out.breakdown) ? 1 : 0;
    }
    copy(c, u, uu, n);
    CK(cudaStreamSynchronize(c.stream));
}

}  // namespace amgr

extern "C" amgr_status amgr_dist_bicgstab(amgr_dist* d, const double* f_local, double* u_local,
                                          const amgr_solve_params* prm, amgr_solve_stats* stats) {
    if (!stats) return AMGR_E_INVALID_ARGUMENT;
    return dist_guard(d, [&] {
        amgr_solve_params sp{1e-8, 100};
        if (prm) sp = *prm;
        amgr::dist_bicgstab(*d->d, f_local, u_local, sp, *stats);
    });
}

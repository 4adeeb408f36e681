"""Row partitioning of an AMG hierarchy over W ranks.

Aggregate-consistent ownership.  Levels 0..T are partitioned; levels T+1..L-1
(tiny, always including the coarsest) are replicated on every rank.  The rows
of level T+1 are split into W contiguous index ranges ("restriction owners"),
and ownership propagates down the aggregation tree:
owner_i(row) = owner_{i+1}(agg_i(row)).  Hence:

* every coarse row's member (fine) rows live on its owner, so restriction,
  prolongation and the numeric Galerkin product (whose contributions come
  only from member rows, csr.cpp:145-194) are communication-free and keep
  the reference's summation order (each coarse entry is summed on one GPU);
* SpMV on a partitioned level needs halo values of columns owned elsewhere
  (send/recv lists per peer, exchanged before each pass);
* at the transition, each rank restricts onto its owned level-T rows, then
  an allgather replicates f_T (and, at rebuild, the rows of A_T).

Local numbering per partitioned level: owned rows in ascending global order
(0..n_own-1), then halo columns grouped by owner rank, ascending.  Every local
row keeps its entries in the global column order, so row sums are
bit-identical to the single-GPU pass.

Host-side setup logic (numpy), executed once after the (replicated) device
setup; tests/test_partition.py checks it with a world-size-2 gloo run.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class LocalLevel:
    level: int
    n_global: int
    owned: np.ndarray            # global ids of owned rows (ascending)
    halo: np.ndarray             # global ids of halo columns (grouped by owner, ascending within)
    rp: np.ndarray               # local CSR (rows = owned)
    col: np.ndarray              # local column ids (owned 0..n_own-1, halo n_own..)
    nnz_map: np.ndarray          # local nnz -> global nnz index (values gather / RAP plan remap)
    recv: dict = field(default_factory=dict)   # peer -> slice of the halo (start, count)
    send: dict = field(default_factory=dict)   # peer -> local owned indices to send
    agg: np.ndarray | None = None    # owned fine row -> local coarse index (partitioned next) or global (replicated)
    mptr: np.ndarray | None = None   # member lists of owned coarse rows (local fine ids), when next is partitioned
    midx: np.ndarray | None = None

    @property
    def n_own(self):
        return len(self.owned)


@dataclass
class Plan:
    world: int
    rank: int
    top: int                      # last partitioned level (T)
    levels: list                  # LocalLevel for 0..T
    owner: list                   # per partitioned level: owner rank of every global row
    replicated_from: int          # first replicated level (T+1)


def _ranges(n, world):
    return (np.arange(n, dtype=np.int64) * world) // max(n, 1)


def ownership(n, agg, top, world):
    """owner arrays for levels 0..top+1 (agg[i] maps level i -> level i+1);
    level top+1 is the first replicated level (its owners restrict onto it)."""
    own = [None] * (top + 2)
    own[top + 1] = _ranges(n[top + 1], world)
    for i in range(top, -1, -1):
        own[i] = own[i + 1][agg[i]]
    return own


def choose_top(n, replicate_below):
    """Last partitioned level: the coarsest level with at least replicate_below
    rows, never the coarsest level itself (its dense LU is replicated).
    Returns -1 when nothing is partitioned."""
    top = -1
    for i, ni in enumerate(n[:-1]):
        if ni >= replicate_below:
            top = i
    return top


def build_plan(hier, rank: int, world: int, replicate_below: int = 20000) -> Plan:
    """hier: list of dicts per level with keys n, rp, col (int arrays) and agg
    (all but the coarsest)."""
    n = [int(L["n"]) for L in hier]
    agg = [np.asarray(L["agg"], np.int64) if L.get("agg") is not None else None for L in hier]
    top = choose_top(n, replicate_below)
    if top < 0:
        return Plan(world, rank, -1, [], [], 0)
    own = ownership(n, agg, top, world)
    levels = []
    for i in range(top + 1):
        rp = np.asarray(hier[i]["rp"], np.int64)
        col = np.asarray(hier[i]["col"], np.int64)
        oi = own[i]
        owned = np.nonzero(oi == rank)[0]
        g2l = -np.ones(n[i], np.int64)
        g2l[owned] = np.arange(len(owned))
        # local CSR rows in global order, entries in global column order
        lens = rp[owned + 1] - rp[owned]
        lrp = np.zeros(len(owned) + 1, np.int64)
        np.cumsum(lens, out=lrp[1:])
        row_len = np.diff(rp)
        nnz_map = np.nonzero(np.repeat(oi == rank, row_len))[0]
        gcol = col[nnz_map]
        foreign = gcol[g2l[gcol] < 0]
        halo_glob = np.unique(foreign)
        # group halo by owner, ascending within the group
        order = np.lexsort((halo_glob, oi[halo_glob]))
        halo = halo_glob[order]
        hpos = -np.ones(n[i], np.int64)
        hpos[halo] = len(owned) + np.arange(len(halo))
        lcol = np.where(g2l[gcol] >= 0, g2l[gcol], hpos[gcol])
        assert (lcol >= 0).all()
        LL = LocalLevel(i, n[i], owned, halo, lrp, lcol, nnz_map)
        start = 0
        for p in range(world):
            cnt = int((oi[halo] == p).sum())
            if cnt:
                LL.recv[p] = (start, cnt)
            start += cnt
        # send lists: rows of mine that peer p needs = halo of p owned by me
        for p in range(world):
            if p == rank:
                continue
            pe = np.nonzero(np.repeat(oi == p, row_len))[0]
            need = np.unique(col[pe])
            need = need[oi[need] == rank]
            if len(need):
                LL.send[p] = g2l[need]
        levels.append(LL)
    # transfers
    for i in range(top + 1):
        LL = levels[i]
        if i + 1 <= top:
            g2l_c = -np.ones(n[i + 1], np.int64)
            g2l_c[levels[i + 1].owned] = np.arange(levels[i + 1].n_own)
            LL.agg = g2l_c[agg[i][LL.owned]]
            assert (LL.agg >= 0).all(), "aggregate consistency violated"
        else:
            LL.agg = agg[i][LL.owned]  # into the replicated level (global ids)
        # member lists of owned coarse rows (the coarse rows this rank restricts onto)
        coarse_owned = np.nonzero(own[i + 1] == rank)[0]
        la = agg[i][LL.owned]
        cmap = -np.ones(n[i + 1], np.int64)
        cmap[coarse_owned] = np.arange(len(coarse_owned))
        key = cmap[la]
        assert (key >= 0).all(), "a fine row's aggregate is owned elsewhere"
        order = np.argsort(key, kind="stable")  # members ascending (local order = global order)
        LL.midx = order.astype(np.int64)
        LL.mptr = np.zeros(len(coarse_owned) + 1, np.int64)
        np.cumsum(np.bincount(key, minlength=len(coarse_owned)), out=LL.mptr[1:])
    return Plan(world, rank, top, levels, own, top + 1)


def hierarchy_from_oracle(h):
    """Convert an oracle/ref-style hierarchy (levels with .A and .agg) into the
    dict form build_plan takes."""
    out = []
    for L in h.levels:
        out.append({"n": len(L.A[0]) - 1, "rp": L.A[0], "col": L.A[1], "agg": L.agg})
    return out


def local_galerkin(L: LocalLevel, local_vals, agg_glob, coarse_rows, crp, ccol):
    """Partitioned numeric Galerkin product (host statement of what
    amgr_dist_rebuild_local runs with device plans): the values of this rank's
    coarse rows `coarse_rows` (global ids, ascending) of A_{i+1}, from ONLY the
    rank's local entries of A_i.  Per coarse row I and coarse column J:
    acc = 0; for each member fine row m of I ascending: part = 0; for each
    local entry (m, k) in column order with agg(col k) = J: part += a_mk;
    acc += part (two-level bracket of spmm(R, spmm(A, P)), csr.cpp:145-194,
    SURVEY.md F4).  Members are local by aggregate consistency; columns are
    mapped to global ids (owned / halo) only to look up their aggregate.
    Returns the concatenated row values in the global coarse CSR order."""
    gcol = np.where(L.col < L.n_own, L.owned[np.minimum(L.col, L.n_own - 1)],
                    L.halo[np.maximum(L.col - L.n_own, 0)] if len(L.halo) else 0)
    cagg = np.asarray(agg_glob)[gcol]  # coarse column of every local entry
    out = []
    # members of each coarse row (local fine ids ascending): rows whose aggregate is I
    own_agg = np.asarray(agg_glob)[L.owned]
    order = np.argsort(own_agg, kind="stable")
    sa = own_agg[order]
    for I in coarse_rows:
        a, b = np.searchsorted(sa, I), np.searchsorted(sa, I, side="right")
        cols = ccol[crp[I]:crp[I + 1]]
        acc = {int(J): 0.0 for J in cols}
        for m in order[a:b]:
            part = {}
            for k in range(L.rp[m], L.rp[m + 1]):
                J = int(cagg[k])
                part[J] = part.get(J, 0.0) + float(local_vals[k])
            for J, p in part.items():
                acc[J] = acc[J] + p
        out.append(np.array([acc[int(J)] for J in cols], np.float64))
    return np.concatenate(out) if out else np.zeros(0)

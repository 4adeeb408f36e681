/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * partial-reuse AMG path.  See amg_oracle.h for the pinning statement.
 * Every function names the reference file:line it restates (paths relative to
 * /root/reference/proj).  Compiled with -O2 -ffp-contract=off (oracle/Makefile)
 * so no a*b+c is contracted, matching the reference build the parity tests use.
 */
#define _GNU_SOURCE
#include "amg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define SETERR(...)                                 \
    do {                                            \
        if (err && errlen > 0) snprintf(err, (size_t)errlen, __VA_ARGS__); \
    } while (0)

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) abort();
    return p;
}

idx_t o_nnz(const ocsr* A) { return A->rp[A->nrows]; }

void o_free_csr(ocsr* A) {
    free(A->rp);
    free(A->ci);
    free(A->v);
    A->rp = NULL;
    A->ci = NULL;
    A->v = NULL;
}

static void csr_alloc(ocsr* A, idx_t nrows, idx_t ncols, idx_t nnz) {
    A->nrows = nrows;
    A->ncols = ncols;
    A->rp = (idx_t*)xcalloc((size_t)nrows + 1, sizeof(idx_t));
    A->ci = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)nnz);
    A->v = (double*)xmalloc(sizeof(double) * (size_t)nnz);
}

static void csr_copy(ocsr* dst, const ocsr* src) {
    idx_t nnz = o_nnz(src);
    csr_alloc(dst, src->nrows, src->ncols, nnz);
    memcpy(dst->rp, src->rp, sizeof(idx_t) * (size_t)(src->nrows + 1));
    memcpy(dst->ci, src->ci, sizeof(idx_t) * (size_t)nnz);
    memcpy(dst->v, src->v, sizeof(double) * (size_t)nnz);
}

/* ---- sparse core ------------------------------------------------------- */

/* csr.cpp:76-85: y_i = sum_k a_ik x_col, sequential in stored order from 0.0 */
void o_spmv(const ocsr* A, const double* x, double* y) {
    for (idx_t i = 0; i < A->nrows; ++i) {
        double s = 0.0;
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * x[A->ci[k]];
        y[i] = s;
    }
}

/* csr.cpp:93-113: counting sort by column; rows of T ascend by source row */
int o_transpose(const ocsr* A, ocsr* T) {
    idx_t nnz = o_nnz(A);
    csr_alloc(T, A->ncols, A->nrows, nnz);
    for (idx_t k = 0; k < nnz; ++k) T->rp[A->ci[k] + 1]++;
    for (idx_t j = 0; j < A->ncols; ++j) T->rp[j + 1] += T->rp[j];
    idx_t* pos = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)(A->ncols + 1));
    memcpy(pos, T->rp, sizeof(idx_t) * (size_t)(A->ncols + 1));
    for (idx_t i = 0; i < A->nrows; ++i)
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            idx_t p = pos[A->ci[k]]++;
            T->ci[p] = i;
            T->v[p] = A->v[k];
        }
    free(pos);
    return 0;
}

static int cmp_idx(const void* a, const void* b) {
    idx_t x = *(const idx_t*)a, y = *(const idx_t*)b;
    return (x > y) - (x < y);
}

/* csr.cpp:115-143 (symbolic: marker + sorted unique columns) followed by
 * csr.cpp:145-184 (numeric: per-row scratch keyed by the pattern, entries
 * accumulated in (A column, B column) stored order starting from 0.0). */
int o_spmm(const ocsr* A, const ocsr* B, ocsr* C, char* err, int errlen) {
    if (A->ncols != B->nrows) {
        SETERR("spmm_symbolic: dimension mismatch (%lld vs %lld)", (long long)A->ncols, (long long)B->nrows);
        return 1;
    }
    idx_t* marker = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)B->ncols);
    for (idx_t j = 0; j < B->ncols; ++j) marker[j] = -1;
    /* pass 1: count */
    idx_t* cnt = (idx_t*)xcalloc((size_t)A->nrows + 1, sizeof(idx_t));
    for (idx_t i = 0; i < A->nrows; ++i) {
        idx_t c = 0;
        for (idx_t ka = A->rp[i]; ka < A->rp[i + 1]; ++ka) {
            idx_t k = A->ci[ka];
            for (idx_t kb = B->rp[k]; kb < B->rp[k + 1]; ++kb) {
                idx_t j = B->ci[kb];
                if (marker[j] != i) {
                    marker[j] = i;
                    ++c;
                }
            }
        }
        cnt[i + 1] = c;
    }
    for (idx_t i = 0; i < A->nrows; ++i) cnt[i + 1] += cnt[i];
    csr_alloc(C, A->nrows, B->ncols, cnt[A->nrows]);
    memcpy(C->rp, cnt, sizeof(idx_t) * (size_t)(A->nrows + 1));
    free(cnt);
    for (idx_t j = 0; j < B->ncols; ++j) marker[j] = -1;
    double* scratch = (double*)xcalloc((size_t)B->ncols, sizeof(double));
    for (idx_t i = 0; i < A->nrows; ++i) {
        idx_t p = C->rp[i];
        for (idx_t ka = A->rp[i]; ka < A->rp[i + 1]; ++ka) {
            idx_t k = A->ci[ka];
            for (idx_t kb = B->rp[k]; kb < B->rp[k + 1]; ++kb) {
                idx_t j = B->ci[kb];
                if (marker[j] != i) {
                    marker[j] = i;
                    C->ci[p++] = j;
                }
            }
        }
        qsort(C->ci + C->rp[i], (size_t)(C->rp[i + 1] - C->rp[i]), sizeof(idx_t), cmp_idx);
        for (idx_t q = C->rp[i]; q < C->rp[i + 1]; ++q) scratch[C->ci[q]] = 0.0;
        for (idx_t ka = A->rp[i]; ka < A->rp[i + 1]; ++ka) {
            const idx_t k = A->ci[ka];
            const double av = A->v[ka];
            for (idx_t kb = B->rp[k]; kb < B->rp[k + 1]; ++kb) scratch[B->ci[kb]] += av * B->v[kb];
        }
        for (idx_t q = C->rp[i]; q < C->rp[i + 1]; ++q) C->v[q] = scratch[C->ci[q]];
    }
    free(scratch);
    free(marker);
    return 0;
}

/* csr.cpp:190-194: spmm(R, spmm(A, P)) */
int o_galerkin(const ocsr* R, const ocsr* A, const ocsr* P, ocsr* C, char* err, int errlen) {
    if (R->ncols != A->nrows) {
        SETERR("galerkin_product: R*A: dimension mismatch");
        return 1;
    }
    if (A->ncols != P->nrows) {
        SETERR("galerkin_product: A*P: dimension mismatch");
        return 1;
    }
    ocsr AP;
    int rc = o_spmm(A, P, &AP, err, errlen);
    if (rc) return rc;
    rc = o_spmm(R, &AP, C, err, errlen);
    o_free_csr(&AP);
    return rc;
}

/* ---- coarsening --------------------------------------------------------- */

static idx_t find_diag(const ocsr* A, idx_t i) {
    for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k)
        if (A->ci[k] == i) return k;
    return -1;
}

/* coarsening.cpp:11-75: diagonal check over all rows first, then the strong
 * test v*v > eps2*|d_i d_j| on stored off-diagonals, union-symmetrised,
 * sorted and deduplicated. */
int o_strength(const ocsr* A, double eps, idx_t** adj_ptr_out, idx_t** adj_out, char* err, int errlen) {
    const idx_t n = A->nrows;
    if (A->nrows != A->ncols) {
        SETERR("strength_graph: matrix is not square");
        return 1;
    }
    if (eps < 0.0 || eps >= 1.0) {
        SETERR("strength_graph: eps must be in [0, 1)");
        return 1;
    }
    double* dia = (double*)xcalloc((size_t)n, sizeof(double));
    for (idx_t i = 0; i < n; ++i) {
        idx_t k = find_diag(A, i);
        if (k >= 0) dia[i] = A->v[k];
        if (k < 0 || dia[i] == 0.0) {
            SETERR("strength_graph: zero diagonal at row %lld", (long long)i);
            free(dia);
            return 1;
        }
    }
    const double eps2 = eps * eps;
    idx_t* deg = (idx_t*)xcalloc((size_t)n + 1, sizeof(idx_t));
    for (idx_t i = 0; i < n; ++i)
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const idx_t j = A->ci[k];
            const double v = A->v[k];
            if (j != i && v * v > eps2 * fabs(dia[i] * dia[j])) {
                deg[i + 1]++;
                deg[j + 1]++;
            }
        }
    for (idx_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
    idx_t* lst = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)deg[n]);
    idx_t* pos = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)(n + 1));
    memcpy(pos, deg, sizeof(idx_t) * (size_t)(n + 1));
    for (idx_t i = 0; i < n; ++i)
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const idx_t j = A->ci[k];
            const double v = A->v[k];
            if (j != i && v * v > eps2 * fabs(dia[i] * dia[j])) {
                lst[pos[i]++] = j;
                lst[pos[j]++] = i;
            }
        }
    idx_t* ap = (idx_t*)xcalloc((size_t)n + 1, sizeof(idx_t));
    idx_t* adj = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)deg[n]);
    idx_t m = 0;
    for (idx_t i = 0; i < n; ++i) {
        idx_t b = deg[i], e = deg[i + 1];
        qsort(lst + b, (size_t)(e - b), sizeof(idx_t), cmp_idx);
        for (idx_t q = b; q < e; ++q)
            if (q == b || lst[q] != lst[q - 1]) adj[m++] = lst[q];
        ap[i + 1] = m;
    }
    free(lst);
    free(pos);
    free(deg);
    free(dia);
    *adj_ptr_out = ap;
    *adj_out = adj;
    return 0;
}

/* coarsening.cpp:77-120: pass 1 roots absorb free neighbours in ascending
 * order; pass 2 leftovers join their lowest-indexed assigned neighbour,
 * isolated nodes become singletons. */
idx_t o_aggregate(idx_t n, const idx_t* ap, const idx_t* adj, idx_t* a) {
    idx_t next = 0;
    for (idx_t i = 0; i < n; ++i) a[i] = -1;
    for (idx_t i = 0; i < n; ++i) {
        if (a[i] != -1) continue;
        int free_nb = 0;
        for (idx_t p = ap[i]; p < ap[i + 1]; ++p)
            if (a[adj[p]] == -1) {
                free_nb = 1;
                break;
            }
        if (!free_nb) continue;
        const idx_t id = next++;
        a[i] = id;
        for (idx_t p = ap[i]; p < ap[i + 1]; ++p)
            if (a[adj[p]] == -1) a[adj[p]] = id;
    }
    for (idx_t i = 0; i < n; ++i) {
        if (a[i] != -1) continue;
        if (ap[i] == ap[i + 1]) {
            a[i] = next++;
            continue;
        }
        for (idx_t p = ap[i]; p < ap[i + 1]; ++p)
            if (a[adj[p]] != -1) {
                a[i] = a[adj[p]];
                break;
            }
    }
    return next;
}

/* coarsening.cpp:122-132 */
static void tentative(idx_t nf, idx_t nc, const idx_t* agg, ocsr* P) {
    csr_alloc(P, nf, nc, nf);
    for (idx_t i = 0; i <= nf; ++i) P->rp[i] = i;
    for (idx_t i = 0; i < nf; ++i) {
        P->ci[i] = agg[i];
        P->v[i] = 1.0;
    }
}

/* ---- smoothers -------------------------------------------------------------- */

/* smoother.cpp:8-32 */
static int jacobi_build(const ocsr* A, double* inv_diag, char* err, int errlen) {
    for (idx_t i = 0; i < A->nrows; ++i) {
        idx_t k = find_diag(A, i);
        double d = k >= 0 ? A->v[k] : 0.0;
        if (k < 0 || d == 0.0) {
            SETERR("build_smoother: zero diagonal at row %lld", (long long)i);
            return 1;
        }
        inv_diag[i] = 1.0 / d;
    }
    return 0;
}

/* extension (parity unpinned): SPAI0  m_i = a_ii / sum_j a_ij^2 */
static int spai0_build(const ocsr* A, double* m, char* err, int errlen) {
    for (idx_t i = 0; i < A->nrows; ++i) {
        double s = 0.0;
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * A->v[k];
        idx_t k = find_diag(A, i);
        double d = k >= 0 ? A->v[k] : 0.0;
        if (k < 0 || d == 0.0) {
            SETERR("build_smoother: zero diagonal at row %lld", (long long)i);
            return 1;
        }
        m[i] = d / s;
    }
    return 0;
}

/* extension (parity unpinned): lambda_max(D^-1 A) by power iteration from
 * the all-ones vector: x <- y/|y| with y = D^-1 A x; lambda = |y|/|x|. */
static double power_start_sign(uint64_t i) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (z >> 63) ? -1.0 : 1.0;
}

static double power_lambda(const ocsr* A, const double* inv_diag, int iters) {
    const idx_t n = A->nrows;
    double* x = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* y = (double*)xmalloc(sizeof(double) * (size_t)n);
    /* start vector: pseudo-random signs (x_i = +-1, so x.x = n exactly); a
       constant start is nearly the smoothest mode of D^-1 A and leaves the
       estimate far below lambda_max after a few iterations */
    for (idx_t i = 0; i < n; ++i) x[i] = power_start_sign((uint64_t)i);
    double xx = (double)n, lam = 0.0;
    for (int it = 0; it < iters; ++it) {
        o_spmv(A, x, y);
        double yy = 0.0;
        for (idx_t i = 0; i < n; ++i) {
            y[i] = inv_diag[i] * y[i];
            yy += y[i] * y[i];
        }
        lam = sqrt(yy) / sqrt(xx);
        const double s = 1.0 / sqrt(yy);
        for (idx_t i = 0; i < n; ++i) x[i] = y[i] * s;
        xx = 0.0;
        for (idx_t i = 0; i < n; ++i) xx += x[i] * x[i];
    }
    free(x);
    free(y);
    return lam;
}

typedef struct {
    ocsr A;
    int has_P;
    ocsr P, R;
    int has_smoother;
    double* w;       /* inv_diag (jacobi, chebyshev) or m (spai0) */
    double lam_max;  /* chebyshev upper bound (after safety factor) */
    double omega;    /* Jacobi weight of this level (sa_jacobi_omega; = prm.omega otherwise) */
} olevel;

struct ohier {
    int nlev;
    olevel* lv;
    oparams prm;
    idx_t nL;
    double* lu;
    idx_t* piv;
};

/* smoother.cpp:34-48: u += (omega*inv_diag)(f - A u), `sweeps` times */
static void smooth_jacobi(const olevel* L, double omega, const double* f, double* u, int sweeps, double* r) {
    const idx_t n = L->A.nrows;
    for (int s = 0; s < sweeps; ++s) {
        o_spmv(&L->A, u, r);
        for (idx_t i = 0; i < n; ++i) u[i] += omega * L->w[i] * (f[i] - r[i]);
    }
}

/* extension (parity unpinned): Chebyshev polynomial smoother on D^-1 A with
 * bounds [lower*lam, lam]; degree SpMVs per sweep. */
static void smooth_cheb(const olevel* L, const oparams* p, const double* f, double* x, int sweeps, double* r) {
    const idx_t n = L->A.nrows;
    const double hi = L->lam_max, lo = hi * p->cheb_lower;
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo);
    const double sigma = theta / delta;
    double* d = (double*)xmalloc(sizeof(double) * (size_t)n);
    for (int s = 0; s < sweeps; ++s) {
        double rho = 1.0 / sigma;
        o_spmv(&L->A, x, r);
        for (idx_t i = 0; i < n; ++i) {
            r[i] = L->w[i] * (f[i] - r[i]);
            d[i] = r[i] / theta;
        }
        for (int k = 1; k <= p->cheb_degree; ++k) {
            for (idx_t i = 0; i < n; ++i) x[i] += d[i];
            if (k == p->cheb_degree) break;
            o_spmv(&L->A, x, r);
            const double rho_new = 1.0 / (2.0 * sigma - rho);
            const double c1 = rho_new * rho, c2 = 2.0 * rho_new / delta;
            for (idx_t i = 0; i < n; ++i) {
                r[i] = L->w[i] * (f[i] - r[i]);
                d[i] = c1 * d[i] + c2 * r[i];
            }
            rho = rho_new;
        }
    }
    free(d);
}

static void smooth_level(const ohier* h, const olevel* L, const double* f, double* u, int sweeps, double* r) {
    if (h->prm.smoother == 2)
        smooth_cheb(L, &h->prm, f, u, sweeps, r);
    else
        smooth_jacobi(L, h->prm.smoother == 1 ? 1.0 : L->omega, f, u, sweeps, r);
}

/* Smoothed aggregation (extension): the Galerkin operators of a smoothed P
 * are not diagonally dominant, and lambda_max(D^-1 A_l) grows to 4-15 on the
 * coarse levels (C1 at 32^3), where the fixed weight 0.72 diverges.  Each
 * level of an SA hierarchy therefore damps with
 *   omega_l = min(omega, (4/3) / g_l),  g_l = max_i sum_j |a_ij| / |a_ii|
 * (Gershgorin bound of D^-1 A_l: order-independent, so device and oracle
 * agree bit for bit).  Plain aggregation keeps omega. */
static double sa_jacobi_omega(const ocsr* A, double omega) {
    double g = 0.0;
    for (idx_t i = 0; i < A->nrows; ++i) {
        double s = 0.0, d = 0.0;
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            s += fabs(A->v[k]);
            if (A->ci[k] == i) d = A->v[k];
        }
        const double q = s / fabs(d);
        if (q > g) g = q;
    }
    const double cap = (4.0 / 3.0) / g;
    return cap < omega ? cap : omega;
}

static int build_level_smoother(olevel* L, const oparams* p, char* err, int errlen) {
    L->w = (double*)xmalloc(sizeof(double) * (size_t)L->A.nrows);
    L->has_smoother = 1;
    int rc = p->smoother == 1 ? spai0_build(&L->A, L->w, err, errlen) : jacobi_build(&L->A, L->w, err, errlen);
    if (rc) return rc;
    L->omega = (p->coarsening == 1 && p->smoother == 0) ? sa_jacobi_omega(&L->A, p->omega) : p->omega;
    if (p->smoother == 2) L->lam_max = power_lambda(&L->A, L->w, p->power_iters) * p->cheb_safety;
    return 0;
}

/* ---- dense LU (dense_lu.cpp:10-73) ---------------------------------------------- */

int o_factorize(const ocsr* A, double* m, idx_t* piv, char* err, int errlen) {
    const idx_t n = A->nrows;
    if (A->nrows != A->ncols) {
        SETERR("coarse_factorize: matrix is not square");
        return 1;
    }
    memset(m, 0, sizeof(double) * (size_t)(n * n));
    for (idx_t i = 0; i < n; ++i)
        for (idx_t k = A->rp[i]; k < A->rp[i + 1]; ++k) m[i * n + A->ci[k]] = A->v[k];
    for (idx_t k = 0; k < n; ++k) {
        idx_t p = k;
        double best = fabs(m[k * n + k]);
        for (idx_t i = k + 1; i < n; ++i) {
            const double c = fabs(m[i * n + k]);
            if (c > best) {
                best = c;
                p = i;
            }
        }
        piv[k] = p;
        if (p != k)
            for (idx_t j = 0; j < n; ++j) {
                double t = m[k * n + j];
                m[k * n + j] = m[p * n + j];
                m[p * n + j] = t;
            }
        const double pivot = m[k * n + k];
        if (pivot == 0.0) {
            SETERR("coarse_factorize: singular matrix (zero pivot at step %lld)", (long long)k);
            return 2;
        }
        for (idx_t i = k + 1; i < n; ++i) {
            const double l = m[i * n + k] / pivot;
            m[i * n + k] = l;
            for (idx_t j = k + 1; j < n; ++j) m[i * n + j] -= l * m[k * n + j];
        }
    }
    return 0;
}

void o_coarse_solve(idx_t n, const double* m, const idx_t* piv, const double* rhs, double* x) {
    memcpy(x, rhs, sizeof(double) * (size_t)n);
    for (idx_t k = 0; k < n; ++k)
        if (piv[k] != k) {
            double t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
    for (idx_t i = 1; i < n; ++i) {
        double s = x[i];
        for (idx_t j = 0; j < i; ++j) s -= m[i * n + j] * x[j];
        x[i] = s;
    }
    for (idx_t i = n; i-- > 0;) {
        double s = x[i];
        for (idx_t j = i + 1; j < n; ++j) s -= m[i * n + j] * x[j];
        x[i] = s / m[i * n + i];
    }
}

/* ---- hierarchy ---------------------------------------------------------------------- */

static void free_level(olevel* L) {
    o_free_csr(&L->A);
    if (L->has_P) {
        o_free_csr(&L->P);
        o_free_csr(&L->R);
    }
    free(L->w);
    L->w = NULL;
}

void o_free_hier(ohier* h) {
    if (!h) return;
    for (int l = 0; l < h->nlev; ++l) free_level(&h->lv[l]);
    free(h->lv);
    free(h->lu);
    free(h->piv);
    free(h);
}

static int prefix_level(int rc, int l, char* err, int errlen) {
    if (rc == 1 && err && errlen > 0) {
        char tmp[1024];
        snprintf(tmp, sizeof tmp, "level %d: %s", l, err);
        snprintf(err, (size_t)errlen, "%s", tmp);
    }
    return rc;
}

/* extension (parity unpinned): smoothed prolongator P = P_tent - (w D^-1) A P_tent
 * with w = sa_omega and D = diag(A).  Rows keep the sorted pattern of A P_tent. */
static int smoothed_prolongator(const ocsr* A, const ocsr* Pt, double w, ocsr* P, char* err, int errlen) {
    ocsr AP;
    int rc = o_spmm(A, Pt, &AP, err, errlen);
    if (rc) return rc;
    for (idx_t i = 0; i < A->nrows; ++i) {
        idx_t k = find_diag(A, i);
        double d = k >= 0 ? A->v[k] : 0.0;
        if (k < 0 || d == 0.0) {
            SETERR("smoothed_prolongator: zero diagonal at row %lld", (long long)i);
            o_free_csr(&AP);
            return 1;
        }
        const double s = w * (1.0 / d);
        const idx_t J = Pt->ci[i];
        for (idx_t q = AP.rp[i]; q < AP.rp[i + 1]; ++q)
            AP.v[q] = (AP.ci[q] == J ? 1.0 : 0.0) - s * AP.v[q];
    }
    *P = AP;
    return 0;
}

/* hierarchy.cpp:45-105 */
int o_setup(const ocsr* A0, const oparams* p, ohier** out, char* err, int errlen) {
    if (A0->nrows != A0->ncols) {
        SETERR("setup: matrix is not square");
        return 1;
    }
    if (A0->nrows == 0) {
        SETERR("setup: empty matrix");
        return 1;
    }
    ohier* h = (ohier*)xcalloc(1, sizeof(ohier));
    h->prm = *p;
    int cap = 64;
    h->lv = (olevel*)xcalloc((size_t)cap, sizeof(olevel));
    ocsr cur;
    csr_copy(&cur, A0);
    int rc = 0;
    while (cur.nrows > p->coarse_enough) {
        const int l = h->nlev;
        idx_t *ap = NULL, *adj = NULL;
        rc = o_strength(&cur, p->eps, &ap, &adj, err, errlen);
        if (rc) {
            rc = prefix_level(rc, l, err, errlen);
            goto fail;
        }
        idx_t* agg = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)cur.nrows);
        idx_t nc = o_aggregate(cur.nrows, ap, adj, agg);
        free(ap);
        free(adj);
        if (nc == cur.nrows) {
            free(agg);
            if (cur.nrows <= p->max_direct_size) break;
            SETERR("setup: coarsening stalled at level %d with %lld unknowns (> max_direct_size %lld)", l,
                   (long long)cur.nrows, (long long)p->max_direct_size);
            rc = 2;
            goto fail;
        }
        olevel* L = &h->lv[h->nlev];
        L->A = cur;
        L->has_P = 1;
        ocsr Pt;
        tentative(cur.nrows, nc, agg, &Pt);
        free(agg);
        if (p->coarsening == 1) {
            rc = smoothed_prolongator(&cur, &Pt, p->sa_omega, &L->P, err, errlen);
            o_free_csr(&Pt);
            if (rc) {
                L->has_P = 0;
                rc = prefix_level(rc, l, err, errlen);
                h->nlev++;
                goto fail_nocur;
            }
        } else {
            L->P = Pt;
        }
        o_transpose(&L->P, &L->R);
        rc = build_level_smoother(L, p, err, errlen);
        h->nlev++;
        if (rc) {
            rc = prefix_level(rc, l, err, errlen);
            goto fail_nocur;
        }
        ocsr next;
        rc = o_galerkin(&L->R, &L->A, &L->P, &next, err, errlen);
        if (rc) goto fail_nocur;
        cur = next;
        if (h->nlev + 1 >= cap) {
            cap *= 2;
            h->lv = (olevel*)realloc(h->lv, sizeof(olevel) * (size_t)cap);
            memset(h->lv + h->nlev, 0, sizeof(olevel) * (size_t)(cap - h->nlev));
        }
    }
    h->nL = cur.nrows;
    h->lu = (double*)xmalloc(sizeof(double) * (size_t)(h->nL * h->nL));
    h->piv = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)h->nL);
    rc = o_factorize(&cur, h->lu, h->piv, err, errlen);
    h->lv[h->nlev].A = cur;
    h->nlev++;
    if (rc) goto fail_nocur;
    *out = h;
    return 0;
fail:
    o_free_csr(&cur);
fail_nocur:
    o_free_hier(h);
    return rc;
}

/* hierarchy.cpp:107-150: frozen P/R, smoother + Galerkin per level, coarse LU */
int o_partial_update(const ohier* h0, const ocsr* A, const oparams* p, ohier** out, char* err, int errlen) {
    if (A->nrows != h0->lv[0].A.nrows || A->ncols != h0->lv[0].A.ncols) {
        SETERR("partial update impossible, full rebuild required: new matrix is %lldx%lld, hierarchy was built "
               "for %lldx%lld",
               (long long)A->nrows, (long long)A->ncols, (long long)h0->lv[0].A.nrows, (long long)h0->lv[0].A.ncols);
        return 1;
    }
    ohier* h = (ohier*)xcalloc(1, sizeof(ohier));
    h->prm = *p;
    h->lv = (olevel*)xcalloc((size_t)h0->nlev, sizeof(olevel));
    ocsr cur;
    csr_copy(&cur, A);
    int rc = 0;
    for (int i = 0; i + 1 < h0->nlev; ++i) {
        olevel* L = &h->lv[i];
        L->A = cur;
        L->has_P = 1;
        csr_copy(&L->P, &h0->lv[i].P);
        csr_copy(&L->R, &h0->lv[i].R);
        h->nlev++;
        rc = build_level_smoother(L, p, err, errlen);
        if (rc) {
            rc = prefix_level(rc, i, err, errlen);
            goto fail;
        }
        ocsr next;
        rc = o_galerkin(&L->R, &L->A, &L->P, &next, err, errlen);
        if (rc) goto fail;
        cur = next;
    }
    h->nL = cur.nrows;
    h->lu = (double*)xmalloc(sizeof(double) * (size_t)(h->nL * h->nL));
    h->piv = (idx_t*)xmalloc(sizeof(idx_t) * (size_t)h->nL);
    h->lv[h->nlev].A = cur;
    h->nlev++;
    rc = o_factorize(&cur, h->lu, h->piv, err, errlen);
    if (rc) goto fail;
    *out = h;
    return 0;
fail:
    o_free_hier(h);
    return rc;
}

/* hierarchy.cpp:152-186 with the smoothing the reference's spec describes
 * (smooth(span) on every level, zero initial guess). */
void o_vcycle(const ohier* h, const double* f, double* u_out) {
    const int L = h->nlev;
    double** us = (double**)xcalloc((size_t)L, sizeof(double*));
    double** fs = (double**)xcalloc((size_t)L, sizeof(double*));
    idx_t nmax = h->lv[0].A.nrows;
    double* r = (double*)xmalloc(sizeof(double) * (size_t)nmax);
    double* t = (double*)xmalloc(sizeof(double) * (size_t)nmax);
    fs[0] = (double*)xmalloc(sizeof(double) * (size_t)nmax);
    memcpy(fs[0], f, sizeof(double) * (size_t)nmax);
    for (int i = 0; i + 1 < L; ++i) {
        const olevel* lv = &h->lv[i];
        const idx_t n = lv->A.nrows;
        us[i] = (double*)xcalloc((size_t)n, sizeof(double));
        smooth_level(h, lv, fs[i], us[i], h->prm.pre_sweeps, t);
        o_spmv(&lv->A, us[i], r);
        for (idx_t k = 0; k < n; ++k) r[k] = fs[i][k] - r[k];
        fs[i + 1] = (double*)xmalloc(sizeof(double) * (size_t)lv->R.nrows);
        o_spmv(&lv->R, r, fs[i + 1]);
    }
    us[L - 1] = (double*)xmalloc(sizeof(double) * (size_t)h->nL);
    o_coarse_solve(h->nL, h->lu, h->piv, fs[L - 1], us[L - 1]);
    for (int i = L - 1; i-- > 0;) {
        const olevel* lv = &h->lv[i];
        const idx_t n = lv->A.nrows;
        o_spmv(&lv->P, us[i + 1], r);
        for (idx_t k = 0; k < n; ++k) us[i][k] += r[k];
        smooth_level(h, lv, fs[i], us[i], h->prm.post_sweeps, t);
    }
    memcpy(u_out, us[0], sizeof(double) * (size_t)nmax);
    for (int i = 0; i < L; ++i) {
        free(us[i]);
        free(fs[i]);
    }
    free(us);
    free(fs);
    free(r);
    free(t);
}

int o_num_levels(const ohier* h) { return h->nlev; }

void o_level_dims(const ohier* h, int l, idx_t* d) {
    const olevel* L = &h->lv[l];
    d[0] = L->A.nrows;
    d[1] = o_nnz(&L->A);
    d[2] = L->has_P;
    d[3] = L->has_P ? L->P.ncols : 0;
    d[4] = L->has_smoother;
    d[5] = L->has_P ? o_nnz(&L->P) : 0;
}

static void put(const ocsr* A, idx_t* rp, idx_t* ci, double* v) {
    memcpy(rp, A->rp, sizeof(idx_t) * (size_t)(A->nrows + 1));
    memcpy(ci, A->ci, sizeof(idx_t) * (size_t)o_nnz(A));
    memcpy(v, A->v, sizeof(double) * (size_t)o_nnz(A));
}

void o_level_A(const ohier* h, int l, idx_t* rp, idx_t* ci, double* v) { put(&h->lv[l].A, rp, ci, v); }
void o_level_P(const ohier* h, int l, idx_t* rp, idx_t* ci, double* v) { put(&h->lv[l].P, rp, ci, v); }
void o_level_R(const ohier* h, int l, idx_t* rp, idx_t* ci, double* v) { put(&h->lv[l].R, rp, ci, v); }
void o_level_smoother(const ohier* h, int l, double* w, double* extra) {
    memcpy(w, h->lv[l].w, sizeof(double) * (size_t)h->lv[l].A.nrows);
    if (extra) *extra = h->lv[l].lam_max;
}
idx_t o_coarse_n(const ohier* h) { return h->nL; }
void o_coarse(const ohier* h, double* lu, idx_t* piv) {
    memcpy(lu, h->lu, sizeof(double) * (size_t)(h->nL * h->nL));
    memcpy(piv, h->piv, sizeof(idx_t) * (size_t)h->nL);
}

/* ---- Krylov ------------------------------------------------------------------------------ */

static double dot(const double* a, const double* b, idx_t n) {
    double s = 0.0;
    for (idx_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static double true_res(const ohier* h, const double* f, const double* u, double* tmp, double nf) {
    const idx_t n = h->lv[0].A.nrows;
    o_spmv(&h->lv[0].A, u, tmp);
    double s = 0.0;
    for (idx_t i = 0; i < n; ++i) {
        const double d = f[i] - tmp[i];
        s += d * d;
    }
    return sqrt(s) / nf;
}

/* bicgstab.cpp:21-135, A = finest matrix, M = o_vcycle */
int o_bicgstab(const ohier* h, const double* f, const double* u0, double* u, double tol, idx_t max_iter,
               idx_t* stats, double* relres) {
    const idx_t n = h->lv[0].A.nrows;
    stats[0] = 0;
    stats[1] = 0;
    stats[2] = 0;
    *relres = 0.0;
    const double nf = sqrt(dot(f, f, n));
    if (nf == 0.0) {
        memset(u, 0, sizeof(double) * (size_t)n);
        stats[1] = 1;
        return 0;
    }
    double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* rt = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* p = (double*)xcalloc((size_t)n, sizeof(double));
    double* v = (double*)xcalloc((size_t)n, sizeof(double));
    double* s = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* t = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* ph = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* sh = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* tmp = (double*)xmalloc(sizeof(double) * (size_t)n);
    memcpy(u, u0, sizeof(double) * (size_t)n);
    o_spmv(&h->lv[0].A, u, r);
    for (idx_t i = 0; i < n; ++i) r[i] = f[i] - r[i];
    memcpy(rt, r, sizeof(double) * (size_t)n);
    int converged = 0, breakdown = 0;
    *relres = sqrt(dot(r, r, n)) / nf;
    if (*relres <= tol) {
        *relres = true_res(h, f, u, tmp, nf);
        if (*relres <= tol) {
            converged = 1;
            goto done;
        }
    }
    const double floor_ = 1e-30 * nf * nf;
    double rho_old = 1.0, alpha = 1.0, omega = 1.0;
    for (idx_t it = 1; it <= max_iter; ++it) {
        stats[0] = it;
        const double rho = dot(rt, r, n);
        if (fabs(rho) < floor_) {
            breakdown = 1;
            break;
        }
        if (it == 1) {
            memcpy(p, r, sizeof(double) * (size_t)n);
        } else {
            const double beta = (rho / rho_old) * (alpha / omega);
            for (idx_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
        }
        o_vcycle(h, p, ph);
        o_spmv(&h->lv[0].A, ph, v);
        const double rtv = dot(rt, v, n);
        if (fabs(rtv) < floor_) {
            breakdown = 1;
            break;
        }
        alpha = rho / rtv;
        for (idx_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
        if (sqrt(dot(s, s, n)) / nf <= tol) {
            for (idx_t i = 0; i < n; ++i) u[i] += alpha * ph[i];
            const double res = true_res(h, f, u, tmp, nf);
            if (res <= tol) {
                converged = 1;
                *relres = res;
                goto done;
            }
            memcpy(r, s, sizeof(double) * (size_t)n);
            rho_old = rho;
            continue;
        }
        o_vcycle(h, s, sh);
        o_spmv(&h->lv[0].A, sh, t);
        const double tt = dot(t, t, n);
        if (tt == 0.0) {
            breakdown = 1;
            break;
        }
        omega = dot(t, s, n) / tt;
        for (idx_t i = 0; i < n; ++i) {
            u[i] += alpha * ph[i] + omega * sh[i];
            r[i] = s[i] - omega * t[i];
        }
        rho_old = rho;
        if (sqrt(dot(r, r, n)) / nf <= tol) {
            const double res = true_res(h, f, u, tmp, nf);
            if (res <= tol) {
                converged = 1;
                *relres = res;
                goto done;
            }
        }
        if (fabs(omega) < 1e-30) {
            breakdown = 1;
            break;
        }
    }
    *relres = true_res(h, f, u, tmp, nf);
    converged = *relres <= tol && !breakdown;
done:
    stats[1] = converged;
    stats[2] = breakdown;
    free(r);
    free(rt);
    free(p);
    free(v);
    free(s);
    free(t);
    free(ph);
    free(sh);
    free(tmp);
    return 0;
}

/* extension (parity unpinned): preconditioned CG with the same stopping rule
 * (true-residual confirmation) and breakdown floor as the BiCGStab above. */
int o_cg(const ohier* h, const double* f, const double* u0, double* u, double tol, idx_t max_iter, idx_t* stats,
         double* relres) {
    const idx_t n = h->lv[0].A.nrows;
    stats[0] = stats[1] = stats[2] = 0;
    *relres = 0.0;
    const double nf = sqrt(dot(f, f, n));
    if (nf == 0.0) {
        memset(u, 0, sizeof(double) * (size_t)n);
        stats[1] = 1;
        return 0;
    }
    double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* z = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* p = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* q = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* tmp = (double*)xmalloc(sizeof(double) * (size_t)n);
    int converged = 0, breakdown = 0;
    memcpy(u, u0, sizeof(double) * (size_t)n);
    o_spmv(&h->lv[0].A, u, r);
    for (idx_t i = 0; i < n; ++i) r[i] = f[i] - r[i];
    *relres = sqrt(dot(r, r, n)) / nf;
    if (*relres <= tol) {
        converged = 1;
        goto done;
    }
    o_vcycle(h, r, z);
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rho = dot(r, z, n);
    const double floor_ = 1e-30 * nf * nf;
    for (idx_t it = 1; it <= max_iter; ++it) {
        stats[0] = it;
        o_spmv(&h->lv[0].A, p, q);
        const double pq = dot(p, q, n);
        if (fabs(pq) < floor_ || fabs(rho) < floor_) {
            breakdown = 1;
            break;
        }
        const double alpha = rho / pq;
        for (idx_t i = 0; i < n; ++i) {
            u[i] += alpha * p[i];
            r[i] -= alpha * q[i];
        }
        if (sqrt(dot(r, r, n)) / nf <= tol) {
            const double res = true_res(h, f, u, tmp, nf);
            if (res <= tol) {
                converged = 1;
                *relres = res;
                goto done;
            }
        }
        o_vcycle(h, r, z);
        const double rz = dot(r, z, n);
        const double beta = rz / rho;
        rho = rz;
        for (idx_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    *relres = true_res(h, f, u, tmp, nf);
    converged = *relres <= tol && !breakdown;
done:
    stats[1] = converged;
    stats[2] = breakdown;
    free(r);
    free(z);
    free(p);
    free(q);
    free(tmp);
    return 0;
}

/* ---- 3D generators (same op order as kernels_gen.cu) ------------------------- */

typedef struct {
    int kind;
    idx_t g;
    double inv_h2, shift, c, contrast, inv_sigma2, a_k, b_k, bx, by, bz;
} gparams;

static double node_coef(const gparams* p, idx_t x, idx_t y, idx_t z) {
    if (p->kind == 1 || p->kind == 3) {
        const double dx = (double)x - p->c, dy = (double)y - p->c, dz = (double)z - p->c;
        const double r2 = (dx * dx + dy * dy) + dz * dz;
        return 1.0 + (p->contrast - 1.0) * exp(-(r2 * p->inv_sigma2));
    }
    if (p->kind == 2) return ((double)x < p->a_k && (double)z < p->b_k) ? 1.0 / 1000.0 : 1.0;
    return 1.0;
}

static double harm(double a, double b) { return ((2.0 * a) * b) / (a + b); }

int o_grid3d(int kind, idx_t g, idx_t k, idx_t nsteps, idx_t* rp, idx_t* ci, double* v) {
    gparams p;
    memset(&p, 0, sizeof p);
    p.kind = kind;
    p.g = g;
    const double h = 1.0 / (double)(g + 1);
    p.inv_h2 = 1.0 / (h * h);
    const double den = (double)(nsteps > 1 ? nsteps - 1 : 1), gd = (double)g;
    if (kind == 0) {
        p.shift = 0.01 * (double)(k + 1) * (6.0 * p.inv_h2);
    } else if (kind == 1 || kind == 3) {
        p.contrast = 10.0;
        const double sigma = 0.2 * gd;
        p.inv_sigma2 = 1.0 / (sigma * sigma);
        const double limit = gd - 1.0;
        const double travel = (double)k * 0.25 / sqrt(3.0);
        double pos = fmod(travel, 2.0 * limit);
        if (pos > limit) pos = 2.0 * limit - pos;
        p.c = pos;
        if (kind == 3) {
            const double th = 2.0 * M_PI * (double)k / den, speed = 10.0 / h;
            p.bx = speed * cos(th) / h;
            p.by = speed * sin(th) / h;
            p.bz = 0.5 * speed / h;
        }
    } else if (kind == 2) {
        p.a_k = gd * (0.25 + 0.5 * (double)k / den);
        p.b_k = gd * (0.5 - 0.25 * (double)k / den);
    } else {
        return 1;
    }
    const idx_t g2 = g * g, n = g * g2;
    idx_t q = 0;
    rp[0] = 0;
    for (idx_t i = 0; i < n; ++i) {
        const idx_t x = i % g, y = (i / g) % g, z = i / g2;
        const double k0 = node_coef(&p, x, y, z);
        const double zlo = z > 0 ? harm(k0, node_coef(&p, x, y, z - 1)) : k0;
        const double ylo = y > 0 ? harm(k0, node_coef(&p, x, y - 1, z)) : k0;
        const double xlo = x > 0 ? harm(k0, node_coef(&p, x - 1, y, z)) : k0;
        const double xhi = x < g - 1 ? harm(k0, node_coef(&p, x + 1, y, z)) : k0;
        const double yhi = y < g - 1 ? harm(k0, node_coef(&p, x, y + 1, z)) : k0;
        const double zhi = z < g - 1 ? harm(k0, node_coef(&p, x, y, z + 1)) : k0;
        double dg = (((((zlo + ylo) + xlo) + xhi) + yhi) + zhi) * p.inv_h2;
        double cz0 = 0, cy0 = 0, cx0 = 0, cx1 = 0, cy1 = 0, cz1 = 0;
        if (kind == 3) {
            const double ax = fabs(p.bx), ay = fabs(p.by), az = fabs(p.bz);
            dg = dg + ((ax + ay) + az);
            if (p.bx > 0) cx0 = ax; else cx1 = ax;
            if (p.by > 0) cy0 = ay; else cy1 = ay;
            if (p.bz > 0) cz0 = az; else cz1 = az;
        }
        if (kind == 0) dg = dg + p.shift;
        if (z > 0) { ci[q] = i - g2; v[q++] = -(zlo * p.inv_h2 + cz0); }
        if (y > 0) { ci[q] = i - g; v[q++] = -(ylo * p.inv_h2 + cy0); }
        if (x > 0) { ci[q] = i - 1; v[q++] = -(xlo * p.inv_h2 + cx0); }
        ci[q] = i;
        v[q++] = dg;
        if (x < g - 1) { ci[q] = i + 1; v[q++] = -(xhi * p.inv_h2 + cx1); }
        if (y < g - 1) { ci[q] = i + g; v[q++] = -(yhi * p.inv_h2 + cy1); }
        if (z < g - 1) { ci[q] = i + g2; v[q++] = -(zhi * p.inv_h2 + cz1); }
        rp[i + 1] = q;
    }
    return 0;
}

/*
 * mvamg_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference solve path of arXiv 1907.04417's
 * `mvamg` package (pure Python + numba; /root/reference/pkg/src/mvamg).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this file's shared object.
 *
 * Parity pin: tests/test_oracle_golden.py checks every routine here against
 * fixtures produced by the unmodified reference (tests/golden/make_golden.py).
 *
 * Arithmetic recipe: compiled with -ffp-contract=off,
 * so every `s - a*x` is one rounded multiply and one rounded subtract, in
 * CSR order, exactly as numba/scipy evaluate them.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXLEV 64

/* Host threads: rows of an SpMV and elements of a vector update are split over
 * OpenMP threads; every row / element is computed exactly as in the serial
 * loop, and dots use a fixed blocking (below), so the results do not depend on
 * the thread count.  The Gauss-Seidel sweeps stay serial (_kernels.py:15-38). */
#define OR_PAR_MIN 32768
int or_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

/* scipy csr_matvec: y[i] = 0.0 + sum over row i in CSR order (sparse.py:40). */
void or_spmv(int n, const int* ip, const int* ix, const double* v, const double* x, double* y) {
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = ip[i]; k < ip[i + 1]; ++k) s += v[k] * x[ix[k]];
        y[i] = s;
    }
}

/* gs_forward / gs_backward, in place (_kernels.py:15-38). */
void or_gs(int dir, int n, const int* ip, const int* ix, const double* v, const double* d,
           const double* b, double* x) {
    for (int t = 0; t < n; ++t) {
        int i = dir == 0 ? t : n - 1 - t;
        double s = b[i];
        for (int k = ip[i]; k < ip[i + 1]; ++k) {
            int j = ix[k];
            if (j != i) s -= v[k] * x[j];
        }
        x[i] = s / d[i];
    }
}

/* dot: np.dot is blocked OpenBLAS (FMA, thread-count dependent), so parity is by
 * tolerance.  Here: sequential within blocks of OR_DOT_BLOCK elements, block
 * partials added in order -- the same bits for any thread count. */
#define OR_DOT_BLOCK 8192
double or_dot(int n, const double* x, const double* y) {
    if (n <= OR_DOT_BLOCK) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += x[i] * y[i];
        return s;
    }
    int nb = (n + OR_DOT_BLOCK - 1) / OR_DOT_BLOCK;
    double* part = (double*)malloc(sizeof(double) * (size_t)nb);
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
    for (int b = 0; b < nb; ++b) {
        int i0 = b * OR_DOT_BLOCK, i1 = i0 + OR_DOT_BLOCK < n ? i0 + OR_DOT_BLOCK : n;
        double s = 0.0;
        for (int i = i0; i < i1; ++i) s += x[i] * y[i];
        part[b] = s;
    }
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    free(part);
    return s;
}

/* LAPACK getrs restatement on scipy.linalg.lu_factor output (cycles.py:94-97):
 * lu is the n x n row-major numpy array (L unit-lower, U upper), piv 0-based. */
void or_lu_solve(int n, const double* lu, const int* piv, const double* b, double* x) {
    if (x != b) memcpy(x, b, sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        int p = piv[i];
        if (p != i) { double t = x[i]; x[i] = x[p]; x[p] = t; }
    }
    for (int i = 0; i < n; ++i) {          /* L y = Pb */
        double s = x[i];
        for (int j = 0; j < i; ++j) s -= lu[(size_t)i * n + j] * x[j];
        x[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {     /* U x = y */
        double s = x[i];
        for (int j = i + 1; j < n; ++j) s -= lu[(size_t)i * n + j] * x[j];
        x[i] = s / lu[(size_t)i * n + i];
    }
}

typedef struct { int n, m; const int* ip; const int* ix; const double* v; } or_csr;

enum { OR_GS_FWD = 0, OR_GS_BWD = 1, OR_JACOBI = 2 };

typedef struct {
    int nlev, kind, inner;                 /* kind 0 = V, 1 = K (cycles.py:43-52) */
    int pre_kind, pre_sweeps, post_kind, post_sweeps;
    double pre_omega, post_omega;
    or_csr A[OR_MAXLEV], P[OR_MAXLEV], R[OR_MAXLEV];
    const double* diag[OR_MAXLEV];
    const double* lu; const int* piv;      /* coarsest LU (cycles.py:88-97) */
    const double* inv;                     /* or, when set, a dense coarsest (pseudo-)inverse */
    /* scratch, allocated by or_hier_alloc */
    double *X[OR_MAXLEV], *T[OR_MAXLEV], *RC[OR_MAXLEV];
    double *fr[OR_MAXLEV], *fx[OR_MAXLEV], *fp[OR_MAXLEV][2], *fap[OR_MAXLEV][2];
} or_hier;

size_t or_hier_sizeof(void) { return sizeof(or_hier); }

void or_hier_alloc(or_hier* h) {
    for (int k = 0; k < h->nlev; ++k) {
        size_t n = (size_t)h->A[k].n;
        h->X[k] = calloc(n, 8); h->T[k] = calloc(n, 8); h->RC[k] = calloc(n, 8);
        h->fr[k] = calloc(n, 8); h->fx[k] = calloc(n, 8);
        for (int q = 0; q < 2; ++q) { h->fp[k][q] = calloc(n, 8); h->fap[k][q] = calloc(n, 8); }
    }
}

void or_hier_free(or_hier* h) {
    for (int k = 0; k < h->nlev; ++k) {
        free(h->X[k]); free(h->T[k]); free(h->RC[k]); free(h->fr[k]); free(h->fx[k]);
        for (int q = 0; q < 2; ++q) { free(h->fp[k][q]); free(h->fap[k][q]); }
    }
}

/* MultigridOperator._smooth (cycles.py:139-148). */
static void smooth(or_hier* h, int kind, int sweeps, double omega, int k, const double* b, double* x) {
    const or_csr* A = &h->A[k];
    for (int s = 0; s < sweeps; ++s) {
        if (kind == OR_GS_FWD || kind == OR_GS_BWD) {
            or_gs(kind, A->n, A->ip, A->ix, A->v, h->diag[k], b, x);
        } else {
            double* t = h->T[k];
            or_spmv(A->n, A->ip, A->ix, A->v, x, t);
#pragma omp parallel for schedule(static) if (A->n >= OR_PAR_MIN)
            for (int i = 0; i < A->n; ++i) x[i] += omega * (b[i] - t[i]) / h->diag[k][i];
        }
    }
}

static int descend(or_hier* h, int k, const double* r, double* out);

/* Coarsest solve: the reference's LU (cycles.py:96-97), or z = inv r with the
 * stated C5 deviation (truncated-eigen pseudo-inverse). */
static void coarse_solve(or_hier* h, int k, const double* r, double* out) {
    int n = h->A[k].n;
    if (!h->inv) { or_lu_solve(n, h->lu, h->piv, r, out); return; }
#pragma omp parallel for schedule(static) if (n >= 2048)
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += h->inv[(size_t)i * n + j] * r[j];
        out[i] = s;
    }
}

/* fcg (krylov.py:75-107), x0 = 0, preconditioner = descend(k). Returns <0 on breakdown. */
static int fcg_level(or_hier* h, int k, const double* b, int iters, double* x) {
    int n = h->A[k].n;
    const or_csr* A = &h->A[k];
    double* r = h->fr[k];
    memset(x, 0, sizeof(double) * (size_t)n);
    if (iters <= 0) return 0;
    memcpy(r, b, sizeof(double) * (size_t)n);
    double pAp_prev = 0.0;
    int cur = 0;
    for (int it = 0; it < iters; ++it) {
        double* z = h->X[k];
        int st = descend(h, k, r, z);
        if (st) return st;
        double* p = h->fp[k][cur];
        double* Ap = h->fap[k][cur];
        if (it == 0) {
            memcpy(p, z, sizeof(double) * (size_t)n);
        } else {
            double* pp = h->fp[k][cur ^ 1];
            double* App = h->fap[k][cur ^ 1];
            double beta = or_dot(n, z, App) / pAp_prev;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
            for (int i = 0; i < n; ++i) p[i] = z[i] - beta * pp[i];
        }
        or_spmv(n, A->ip, A->ix, A->v, p, Ap);
        double pAp = or_dot(n, p, Ap);
        if (!(pAp > 0.0)) return -2;
        double alpha = or_dot(n, p, r) / pAp;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; }
        pAp_prev = pAp;
        cur ^= 1;
    }
    return 0;
}

/* MultigridOperator._descend (cycles.py:150-172); out must not alias r. */
static int descend(or_hier* h, int k, const double* r, double* out) {
    int L = h->nlev;
    if (k == L - 1) { coarse_solve(h, k, r, out); return 0; }
    const or_csr* A = &h->A[k];
    int n = A->n, nc = h->A[k + 1].n;
    double* x = h->X[k];
    memset(x, 0, sizeof(double) * (size_t)n);
    smooth(h, h->pre_kind, h->pre_sweeps, h->pre_omega, k, r, x);
    double* t = h->T[k];
    or_spmv(n, A->ip, A->ix, A->v, x, t);
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
    for (int i = 0; i < n; ++i) t[i] = r[i] - t[i];
    double* rc = h->RC[k + 1];
    or_spmv(nc, h->R[k].ip, h->R[k].ix, h->R[k].v, t, rc);
    double* xc = h->fx[k + 1];
    int st;
    if (h->kind == 1 && h->inner >= 1 && k + 1 < L - 1) st = fcg_level(h, k + 1, rc, h->inner, xc);
    else st = descend(h, k + 1, rc, xc);
    if (st) return st;
    or_spmv(n, h->P[k].ip, h->P[k].ix, h->P[k].v, xc, t);
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
    for (int i = 0; i < n; ++i) x[i] += t[i];
    smooth(h, h->post_kind, h->post_sweeps, h->post_omega, k, r, x);
    if (out != x) memcpy(out, x, sizeof(double) * (size_t)n);
    return 0;
}

/* MultigridOperator.apply (cycles.py:174-179). */
int or_apply(or_hier* h, const double* r, double* z) {
    if (h->nlev == 1) { coarse_solve(h, 0, r, z); return 0; }
    return descend(h, 0, r, z);
}

/* MultigridOperator.error_propagation (cycles.py:181-184): e = x - apply(A x). */
int or_error_propagation(or_hier* h, const double* x, double* e, double* tmp_n, double* tmp2_n) {
    const or_csr* A = &h->A[0];
    or_spmv(A->n, A->ip, A->ix, A->v, x, tmp_n);
    int st = or_apply(h, tmp_n, tmp2_n);
    for (int i = 0; i < A->n; ++i) e[i] = x[i] - tmp2_n[i];
    return st;
}

/* apply_composite_symmetrized (bootstrap.py:98-113), in place on x. */
int or_composite(or_hier** ops, int r, double* x, double* t1, double* t2) {
    int n = ops[0]->A[0].n;
    for (int pass = 0; pass < 2 * r; ++pass) {
        or_hier* h = ops[pass < r ? pass : 2 * r - 1 - pass];
        or_spmv(n, h->A[0].ip, h->A[0].ix, h->A[0].v, x, t2);
        int st = or_apply(h, t2, t1);
        if (st) return st;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int i = 0; i < n; ++i) x[i] = x[i] - t1[i];
    }
    return 0;
}

/* Preconditioner kinds for or_pcg. */
enum { OR_PC_NONE = 0, OR_PC_CYCLE = 1, OR_PC_COMPOSITE = 2 };

/* Bsym(r): x = 0; for op in 1..r, r..1: x += B_op (r - A x). */
static int composite_precond(or_hier** ops, int nops, const double* r, double* z, double* t1, double* t2) {
    int n = ops[0]->A[0].n;
    const or_csr* A = &ops[0]->A[0];
    memset(z, 0, sizeof(double) * (size_t)n);
    for (int pass = 0; pass < 2 * nops; ++pass) {
        or_hier* h = ops[pass < nops ? pass : 2 * nops - 1 - pass];
        or_spmv(n, A->ip, A->ix, A->v, z, t1);
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int i = 0; i < n; ++i) t1[i] = r[i] - t1[i];
        int st = or_apply(h, t1, t2);
        if (st) return st;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int i = 0; i < n; ++i) z[i] = z[i] + t2[i];
    }
    return 0;
}

/* pcg (krylov.py:28-72), x0 = 0.  hist must hold itmax+1 entries.
 * Returns 0 ok, -1 r'z breakdown, -2 p'Ap breakdown (NotSpdError in the reference). */
int or_pcg(const or_csr* A, const double* b, int pc_kind, or_hier** ops, int nops, double rtol,
           int itmax, double* x, double* hist, int* nit, int* converged, double* work /* 6n */) {
    int n = A->n;
    double *r = work, *z = work + n, *p = work + 2 * (size_t)n, *q = work + 3 * (size_t)n;
    double *t1 = work + 4 * (size_t)n, *t2 = work + 5 * (size_t)n;
    memset(x, 0, sizeof(double) * (size_t)n);
    memcpy(r, b, sizeof(double) * (size_t)n);
    double r0 = sqrt(or_dot(n, r, r));
    hist[0] = r0; *nit = 0; *converged = 0;
    if (r0 == 0.0) { *converged = 1; return 0; }
#define PREC(IN, OUT) \
    (pc_kind == OR_PC_NONE ? (memcpy(OUT, IN, sizeof(double) * (size_t)n), 0) : \
     pc_kind == OR_PC_CYCLE ? or_apply(ops[0], IN, OUT) : composite_precond(ops, nops, IN, OUT, t1, t2))
    int st = PREC(r, z);
    if (st) return st;
    double rz = or_dot(n, r, z);
    if (!(rz > 0.0)) return -1;
    memcpy(p, z, sizeof(double) * (size_t)n);
    int k = 0;
    while (k < itmax) {
        or_spmv(n, A->ip, A->ix, A->v, p, q);
        double pq = or_dot(n, p, q);
        if (!(pq > 0.0)) { *nit = k; return -2; }
        double alpha = rz / pq;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
        ++k;
        hist[k] = sqrt(or_dot(n, r, r));
        if (hist[k] <= rtol * r0) { *converged = 1; break; }
        st = PREC(r, z);
        if (st) { *nit = k; return st; }
        double rzn = or_dot(n, r, z);
        if (!(rzn > 0.0)) { *nit = k; return -1; }
        double beta = rzn / rz;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rz = rzn;
    }
#undef PREC
    *nit = k;
    return 0;
}

/* ---- construction helpers for the ctypes wrapper (oracle/oracle.py) ---- */
or_hier* or_hier_new(int nlev, int kind, int inner, int pre_kind, int pre_sweeps, double pre_omega,
                     int post_kind, int post_sweeps, double post_omega) {
    if (nlev < 1 || nlev > OR_MAXLEV) return NULL;
    or_hier* h = calloc(1, sizeof(or_hier));
    h->nlev = nlev; h->kind = kind; h->inner = inner;
    h->pre_kind = pre_kind; h->pre_sweeps = pre_sweeps; h->pre_omega = pre_omega;
    h->post_kind = post_kind; h->post_sweeps = post_sweeps; h->post_omega = post_omega;
    return h;
}

void or_hier_set_level(or_hier* h, int k, int n, const int* ip, const int* ix, const double* v,
                       const double* diag) {
    h->A[k].n = n; h->A[k].m = n; h->A[k].ip = ip; h->A[k].ix = ix; h->A[k].v = v; h->diag[k] = diag;
}

void or_hier_set_transfer(or_hier* h, int k, int n, int nc, const int* pip, const int* pix,
                          const double* pv, const int* rip, const int* rix, const double* rv) {
    h->P[k].n = n; h->P[k].m = nc; h->P[k].ip = pip; h->P[k].ix = pix; h->P[k].v = pv;
    h->R[k].n = nc; h->R[k].m = n; h->R[k].ip = rip; h->R[k].ix = rix; h->R[k].v = rv;
}

void or_hier_set_coarse(or_hier* h, const double* lu, const int* piv) { h->lu = lu; h->piv = piv; h->inv = NULL; }

void or_hier_set_coarse_inverse(or_hier* h, const double* inv) { h->inv = inv; }

void or_hier_destroy(or_hier* h) { if (h) { or_hier_free(h); free(h); } }

int or_pcg_h(or_hier* a_owner, const double* b, int pc_kind, or_hier** ops, int nops, double rtol,
             int itmax, double* x, double* hist, int* nit, int* converged, double* work) {
    return or_pcg(&a_owner->A[0], b, pc_kind, ops, nops, rtol, itmax, x, hist, nit, converged, work);
}

/* ---- Galerkin product (setup) ---------------------------
 * galerkin_product(P, A) of pkg/src/mvamg/sparse.py:50-66:
 *   G = (P.T @ (A @ P)).tocsr();  S = ((G + G.T) * 0.5)  (canonical).
 * scipy's csr_matmat accumulates sums[col] += x_ij * y_jk with sums starting at
 * 0.0, in the order the products are generated (X row in CSR order, then Y's
 * row), and drops exact-zero sums; P.T @ AP runs csr_matmat on the transposed
 * (csc) operands, i.e. G[I,J] = 0.0 + sum over k ascending of AP[k,J]*P[k,I].
 * csr_plus_csr adds matching entries (one rounding, commutative), keeps a lone
 * entry as is, drops exact zeros; `* 0.5` scales every stored value. */
typedef struct { int n, m; int* ip; int* ix; double* v; } or_mat;

static int or_cmp_int(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* C = X @ Y (X: n x k, Y: k x m) in the csr_matmat summation order, sorted columns. */
static or_mat or_spgemm(int n, int m, const int* xp, const int* xi, const double* xv,
                        const int* yp, const int* yi, const double* yv) {
    or_mat C = {n, m, (int*)malloc(sizeof(int) * (size_t)(n + 1)), NULL, NULL};
    double* sums = (double*)calloc((size_t)m + 1, sizeof(double));
    char* seen = (char*)calloc((size_t)m + 1, 1);
    int* cols = (int*)malloc(sizeof(int) * ((size_t)m + 1));
    size_t cap = 1024, nnz = 0;
    C.ix = (int*)malloc(sizeof(int) * cap);
    C.v = (double*)malloc(sizeof(double) * cap);
    C.ip[0] = 0;
    for (int i = 0; i < n; ++i) {
        int nc = 0;
        for (int jj = xp[i]; jj < xp[i + 1]; ++jj) {
            const int j = xi[jj];
            const double a = xv[jj];
            for (int kk = yp[j]; kk < yp[j + 1]; ++kk) {
                const int c = yi[kk];
                sums[c] += a * yv[kk];
                if (!seen[c]) { seen[c] = 1; cols[nc++] = c; }
            }
        }
        qsort(cols, (size_t)nc, sizeof(int), or_cmp_int);
        for (int t = 0; t < nc; ++t) {
            const int c = cols[t];
            if (sums[c] != 0.0) {
                if (nnz == cap) {
                    cap *= 2;
                    C.ix = (int*)realloc(C.ix, sizeof(int) * cap);
                    C.v = (double*)realloc(C.v, sizeof(double) * cap);
                }
                C.ix[nnz] = c;
                C.v[nnz] = sums[c];
                ++nnz;
            }
            sums[c] = 0.0;
            seen[c] = 0;
        }
        C.ip[i + 1] = (int)nnz;
    }
    free(sums); free(seen); free(cols);
    return C;
}

/* Stable transpose: rows of the result list the source rows ascending. */
static or_mat or_transpose(int n, int m, const int* ip, const int* ix, const double* v) {
    const int nnz = ip[n];
    or_mat T = {m, n, (int*)calloc((size_t)m + 1, sizeof(int)), (int*)malloc(sizeof(int) * ((size_t)nnz + 1)),
                (double*)malloc(sizeof(double) * ((size_t)nnz + 1))};
    for (int k = 0; k < nnz; ++k) T.ip[ix[k] + 1]++;
    for (int c = 0; c < m; ++c) T.ip[c + 1] += T.ip[c];
    int* cur = (int*)malloc(sizeof(int) * ((size_t)m + 1));
    memcpy(cur, T.ip, sizeof(int) * (size_t)m);
    for (int i = 0; i < n; ++i)
        for (int k = ip[i]; k < ip[i + 1]; ++k) {
            const int p = cur[ix[k]]++;
            T.ix[p] = i;
            T.v[p] = v[k];
        }
    free(cur);
    return T;
}

static void or_mat_free(or_mat* M) { free(M->ip); free(M->ix); free(M->v); }

/* S = (G + G^T) * 0.5 with G = P^T (A P); returns nnz, result owned by *out_*
 * (free with or_free). */
int or_galerkin(int n, int nc, const int* aip, const int* aix, const double* av, const int* pip,
                const int* pix, const double* pv, int** out_ip, int** out_ix, double** out_v) {
    or_mat AP = or_spgemm(n, nc, aip, aix, av, pip, pix, pv);
    or_mat R = or_transpose(n, nc, pip, pix, pv);
    or_mat G = or_spgemm(nc, nc, R.ip, R.ix, R.v, AP.ip, AP.ix, AP.v);
    or_mat GT = or_transpose(nc, nc, G.ip, G.ix, G.v);
    int* sip = (int*)malloc(sizeof(int) * ((size_t)nc + 1));
    const size_t cap = (size_t)G.ip[nc] * 2 + 1;
    int* six = (int*)malloc(sizeof(int) * cap);
    double* sv = (double*)malloc(sizeof(double) * cap);
    int nnz = 0;
    sip[0] = 0;
    for (int i = 0; i < nc; ++i) {
        int a = G.ip[i], ae = G.ip[i + 1], b = GT.ip[i], be = GT.ip[i + 1];
        while (a < ae || b < be) {
            int c;
            double s;
            if (b >= be || (a < ae && G.ix[a] < GT.ix[b])) { c = G.ix[a]; s = G.v[a] + 0.0; ++a; }
            else if (a >= ae || GT.ix[b] < G.ix[a]) { c = GT.ix[b]; s = 0.0 + GT.v[b]; ++b; }
            else { c = G.ix[a]; s = G.v[a] + GT.v[b]; ++a; ++b; }
            if (s != 0.0) { six[nnz] = c; sv[nnz] = s * 0.5; ++nnz; }
        }
        sip[i + 1] = nnz;
    }
    or_mat_free(&AP); or_mat_free(&R); or_mat_free(&G); or_mat_free(&GT);
    *out_ip = sip; *out_ix = six; *out_v = sv;
    return nnz;
}

void or_free(void* p) { free(p); }


/* ---- setup natives (test infrastructure: the CPU-only setup of bench.py's
 * reference arm, oracle/host_setup.py) ------------------------------------- */

/* greedy_accept (_kernels.py:41-61): edges already in the greedy's order
 * (weight descending, ties by (i, j), matching.py:106-122).  partner[v] = -1
 * when v stays unmatched.  Returns the number of accepted pairs. */
long long or_greedy_accept(long long ne, const long long* ei, const long long* ej, int n, long long* partner,
                           long long* pi, long long* pj) {
    for (int v = 0; v < n; ++v) partner[v] = -1;
    long long np = 0;
    for (long long k = 0; k < ne; ++k) {
        long long i = ei[k], j = ej[k];
        if (partner[i] < 0 && partner[j] < 0) {
            partner[i] = j;
            partner[j] = i;
            pi[np] = i;
            pj[np] = j;
            ++np;
        }
    }
    return np;
}

/* One-sided Jacobi on one m x k row-major block in place (_kernels.py:64-121;
 * the accumulated V is not needed for U and sigma).  Returns 1 if converged. */
static int or_jacobi(double* B, int m, int k, int max_sweeps, double tol) {
    if (k < 2) return 1;
    double rel_tol = tol > 2.0 * m * 2.220446049250313e-16 ? tol : 2.0 * m * 2.220446049250313e-16;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        double total = 0.0;
        for (int p = 0; p < k; ++p)
            for (int r = 0; r < m; ++r) total += B[(size_t)r * k + p] * B[(size_t)r * k + p];
        double floor_ = tol * total;
        int rotated = 0;
        for (int p = 0; p < k - 1; ++p)
            for (int q = p + 1; q < k; ++q) {
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (int r = 0; r < m; ++r) {
                    double bp = B[(size_t)r * k + p], bq = B[(size_t)r * k + q];
                    alpha += bp * bp;
                    beta += bq * bq;
                    gamma += bp * bq;
                }
                if (gamma == 0.0) continue;
                if (fabs(gamma) <= rel_tol * sqrt(alpha * beta) || fabs(gamma) <= floor_) continue;
                ++rotated;
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = c * t;
                for (int r = 0; r < m; ++r) {
                    double bp = B[(size_t)r * k + p], bq = B[(size_t)r * k + q];
                    B[(size_t)r * k + p] = c * bp - s * bq;
                    B[(size_t)r * k + q] = s * bp + c * bq;
                }
            }
        if (rotated == 0) return 1;
    }
    return 0;
}

/* jacobi_svd (svd.py:17-55) of every stacked block rows rp[b]..rp[b+1] (k
 * columns, row-major): Jacobi, column norms (sequential over rows, as numpy's
 * axis-0 norm), stable descending sort, U = B / sigma for sigma > 0 else 0.
 * Blocks are independent (parallel over blocks).  Returns 0, or -1 with
 * *failed = the first block that did not converge. */
int or_jacobi_svd_batch(int nblk, const int* rp, int k, const double* A, int max_sweeps, double tol, double* U,
                        double* sigma, int* failed) {
    int first_fail = nblk;
#pragma omp parallel
    {
        int cap = 0;
        double* B = NULL;
        double s[64];
        int order[64];
#pragma omp for schedule(dynamic, 256) reduction(min : first_fail)
        for (int b = 0; b < nblk; ++b) {
            int r0 = rp[b], m = rp[b + 1] - r0;
            if (m * k > cap) { cap = m * k; B = (double*)realloc(B, sizeof(double) * (size_t)cap); }
            memcpy(B, A + (size_t)r0 * k, sizeof(double) * (size_t)m * k);
            if (!or_jacobi(B, m, k, max_sweeps, tol)) { if (b < first_fail) first_fail = b; continue; }
            for (int p = 0; p < k; ++p) {
                double acc = 0.0;
                for (int r = 0; r < m; ++r) acc += B[(size_t)r * k + p] * B[(size_t)r * k + p];
                s[p] = sqrt(acc);
                order[p] = p;
            }
            for (int a = 1; a < k; ++a) {   /* stable insertion sort, descending */
                int o = order[a], j = a - 1;
                while (j >= 0 && s[order[j]] < s[o]) { order[j + 1] = order[j]; --j; }
                order[j + 1] = o;
            }
            for (int p = 0; p < k; ++p) {
                int src = order[p];
                sigma[(size_t)b * k + p] = s[src];
                for (int r = 0; r < m; ++r)
                    U[(size_t)(r0 + r) * k + p] = s[src] > 0.0 ? B[(size_t)r * k + src] / s[src] : 0.0;
            }
        }
        free(B);
    }
    if (failed) *failed = first_fail < nblk ? first_fail : -1;
    return first_fail < nblk ? -1 : 0;
}

/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 * See ibm_oracle.h. Compiled with -ffp-contract=off so every a*b+c rounds twice,
 * as the reference does when built without -march (proj/CMakeLists.txt:9).
 * All file:line citations are relative to /root/reference/proj/include/ibm/.
 */
#include "ibm_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ CSR basics */
orc_csr* orc_csr_new(int rows, int cols, int nnz) {
    orc_csr* m = (orc_csr*)calloc(1, sizeof(orc_csr));
    m->rows = rows;
    m->cols = cols;
    m->nnz = nnz;
    m->rp = (int*)calloc((size_t)rows + 1, sizeof(int));
    m->ci = (int*)malloc(sizeof(int) * (size_t)(nnz > 0 ? nnz : 1));
    m->v = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    return m;
}

orc_csr* orc_csr_from(int rows, int cols, const int* rp, const int* ci, const double* v) {
    orc_csr* m = orc_csr_new(rows, cols, rp[rows]);
    memcpy(m->rp, rp, sizeof(int) * ((size_t)rows + 1));
    memcpy(m->ci, ci, sizeof(int) * (size_t)rp[rows]);
    memcpy(m->v, v, sizeof(double) * (size_t)rp[rows]);
    return m;
}

void orc_csr_free(orc_csr* m) {
    if (!m) return;
    free(m->rp);
    free(m->ci);
    free(m->v);
    free(m);
}

typedef struct {
    int r, c;
    double v;
} trip;

static int trip_cmp(const void* a, const void* b) {
    const trip* x = (const trip*)a;
    const trip* y = (const trip*)b;
    if (x->r != y->r) return x->r < y->r ? -1 : 1;
    if (x->c != y->c) return x->c < y->c ? -1 : 1;
    return 0;
}

/* sparse.hpp:36-67 — sort by (row, col), sum duplicates in sorted order, drop exact zeros.
 * Duplicates only ever come in pairs on the hot path (add_sparse), so the unstable sort
 * cannot change a sum (a+b == b+a). */
static orc_csr* finalize_trips(int rows, int cols, trip* t, size_t n) {
    qsort(t, n, sizeof(trip), trip_cmp);
    orc_csr* m = orc_csr_new(rows, cols, (int)n);
    size_t k = 0;
    int out = 0;
    for (int r = 0; r < rows; ++r) {
        while (k < n && t[k].r == r) {
            const int c = t[k].c;
            double v = 0.0;
            while (k < n && t[k].r == r && t[k].c == c) {
                v += t[k].v;
                ++k;
            }
            if (v != 0.0) {
                m->ci[out] = c;
                m->v[out] = v;
                ++out;
            }
        }
        m->rp[r + 1] = out;
    }
    m->nnz = out;
    return m;
}

orc_csr* orc_from_triplets(int rows, int cols, int n, const int* r, const int* c, const double* v) {
    trip* t = (trip*)malloc(sizeof(trip) * (size_t)(n > 0 ? n : 1));
    for (int k = 0; k < n; ++k) {
        if (r[k] < 0 || r[k] >= rows || c[k] < 0 || c[k] >= cols) {
            free(t);
            return NULL; /* std::invalid_argument in the reference (sparse.hpp:38-39) */
        }
        t[k].r = r[k];
        t[k].c = c[k];
        t[k].v = v[k];
    }
    orc_csr* m = finalize_trips(rows, cols, t, (size_t)n);
    free(t);
    return m;
}

/* sparse.hpp:101-110 — row-order accumulation */
void orc_spmv(const orc_csr* A, const double* x, double* y) {
    for (int i = 0; i < A->rows; ++i) {
        double s = 0.0;
        for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * x[A->ci[k]];
        y[i] = s;
    }
}

/* sparse.hpp:120-138 — counting-sort transpose; rows of A^T keep increasing source row */
orc_csr* orc_transpose(const orc_csr* A) {
    orc_csr* t = orc_csr_new(A->cols, A->rows, A->nnz);
    for (int k = 0; k < A->nnz; ++k) ++t->rp[A->ci[k] + 1];
    for (int c = 0; c < A->cols; ++c) t->rp[c + 1] += t->rp[c];
    int* next = (int*)malloc(sizeof(int) * (size_t)(A->cols > 0 ? A->cols : 1));
    memcpy(next, t->rp, sizeof(int) * (size_t)A->cols);
    for (int r = 0; r < A->rows; ++r)
        for (int k = A->rp[r]; k < A->rp[r + 1]; ++k) {
            const int pos = next[A->ci[k]]++;
            t->ci[pos] = r;
            t->v[pos] = A->v[k];
        }
    free(next);
    return t;
}

static int int_cmp(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return x < y ? -1 : x > y;
}

/* sparse.hpp:226-268 — Gustavson; per output column, products accumulate in
 * (A-row entry, B-row entry) traversal order starting from 0.0; cancelled entries kept. */
orc_csr* orc_spmm_rows(const orc_csr* A, int r0, int r1, const orc_csr* B) {
    if (A->cols != B->rows) return NULL;
    const int out_rows = r1 - r0;
    double* acc = (double*)calloc((size_t)(B->cols > 0 ? B->cols : 1), sizeof(double));
    int* marker = (int*)malloc(sizeof(int) * (size_t)(B->cols > 0 ? B->cols : 1));
    for (int c = 0; c < B->cols; ++c) marker[c] = -1;
    int* touched = (int*)malloc(sizeof(int) * (size_t)(B->cols > 0 ? B->cols : 1));
    size_t cap = 1024, nnz = 0;
    int* ci = (int*)malloc(sizeof(int) * cap);
    double* v = (double*)malloc(sizeof(double) * cap);
    int* rp = (int*)calloc((size_t)out_rows + 1, sizeof(int));
    for (int i = r0; i < r1; ++i) {
        int nt = 0;
        for (int ka = A->rp[i]; ka < A->rp[i + 1]; ++ka) {
            const int j = A->ci[ka];
            const double a = A->v[ka];
            for (int kb = B->rp[j]; kb < B->rp[j + 1]; ++kb) {
                const int c = B->ci[kb];
                if (marker[c] != i) {
                    marker[c] = i;
                    acc[c] = 0.0;
                    touched[nt++] = c;
                }
                acc[c] += a * B->v[kb];
            }
        }
        qsort(touched, (size_t)nt, sizeof(int), int_cmp);
        if (nnz + (size_t)nt > cap) {
            while (nnz + (size_t)nt > cap) cap *= 2;
            ci = (int*)realloc(ci, sizeof(int) * cap);
            v = (double*)realloc(v, sizeof(double) * cap);
        }
        for (int t = 0; t < nt; ++t) {
            ci[nnz] = touched[t];
            v[nnz] = acc[touched[t]];
            ++nnz;
        }
        rp[i - r0 + 1] = (int)nnz;
    }
    orc_csr* C = (orc_csr*)calloc(1, sizeof(orc_csr));
    C->rows = out_rows;
    C->cols = B->cols;
    C->nnz = (int)nnz;
    C->rp = rp;
    C->ci = ci;
    C->v = v;
    free(acc);
    free(marker);
    free(touched);
    return C;
}

/* sparse.hpp:282-314 — D = A*B*C by row slices of A */
orc_csr* orc_triple(const orc_csr* A, const orc_csr* B, const orc_csr* C, int slice, long long* peak, int* slices) {
    if (A->cols != B->rows || B->cols != C->rows || slice < 1) return NULL;
    size_t cap = 1024, nnz = 0;
    int* ci = (int*)malloc(sizeof(int) * cap);
    double* v = (double*)malloc(sizeof(double) * cap);
    int* rp = (int*)calloc((size_t)A->rows + 1, sizeof(int));
    long long pk = 0;
    int ns = 0;
    for (int r0 = 0; r0 < A->rows; r0 += slice) {
        const int r1 = A->rows < r0 + slice ? A->rows : r0 + slice;
        orc_csr* t = orc_spmm_rows(A, r0, r1, B);
        if (t->nnz > pk) pk = t->nnz;
        ++ns;
        orc_csr* d = orc_spmm_rows(t, 0, t->rows, C);
        if (nnz + (size_t)d->nnz > cap) {
            while (nnz + (size_t)d->nnz > cap) cap *= 2;
            ci = (int*)realloc(ci, sizeof(int) * cap);
            v = (double*)realloc(v, sizeof(double) * cap);
        }
        memcpy(ci + nnz, d->ci, sizeof(int) * (size_t)d->nnz);
        memcpy(v + nnz, d->v, sizeof(double) * (size_t)d->nnz);
        for (int r = 0; r < d->rows; ++r) rp[r0 + r + 1] = (int)nnz + d->rp[r + 1];
        nnz += (size_t)d->nnz;
        orc_csr_free(t);
        orc_csr_free(d);
    }
    if (peak) *peak = pk;
    if (slices) *slices = ns;
    orc_csr* D = (orc_csr*)calloc(1, sizeof(orc_csr));
    D->rows = A->rows;
    D->cols = C->cols;
    D->nnz = (int)nnz;
    D->rp = rp;
    D->ci = ci;
    D->v = v;
    return D;
}

/* sparse.hpp:317-329 — a*A + b*B via triplets (pattern union, exact-zero drop) */
orc_csr* orc_add(double a, const orc_csr* A, double b, const orc_csr* B) {
    if (A->rows != B->rows || A->cols != B->cols) return NULL;
    const size_t n = (size_t)A->nnz + (size_t)B->nnz;
    trip* t = (trip*)malloc(sizeof(trip) * (n > 0 ? n : 1));
    size_t k = 0;
    for (int r = 0; r < A->rows; ++r)
        for (int q = A->rp[r]; q < A->rp[r + 1]; ++q) t[k++] = (trip){r, A->ci[q], a * A->v[q]};
    for (int r = 0; r < B->rows; ++r)
        for (int q = B->rp[r]; q < B->rp[r + 1]; ++q) t[k++] = (trip){r, B->ci[q], b * B->v[q]};
    orc_csr* m = finalize_trips(A->rows, A->cols, t, n);
    free(t);
    return m;
}

/* sparse.hpp:351-353 */
orc_csr* orc_symmetrized(const orc_csr* A) {
    orc_csr* At = orc_transpose(A);
    orc_csr* S = orc_add(0.5, A, 0.5, At);
    orc_csr_free(At);
    return S;
}

/* operators.hpp:381-392 */
orc_csr* orc_pin(const orc_csr* A, int pin) {
    trip* t = (trip*)malloc(sizeof(trip) * ((size_t)A->nnz + 1));
    size_t k = 0;
    for (int r = 0; r < A->rows; ++r)
        for (int q = A->rp[r]; q < A->rp[r + 1]; ++q) {
            const int c = A->ci[q];
            if (r == pin || c == pin) continue;
            t[k++] = (trip){r, c, A->v[q]};
        }
    t[k++] = (trip){pin, pin, 1.0};
    orc_csr* m = finalize_trips(A->rows, A->cols, t, k);
    free(t);
    return m;
}

/* operators.hpp:394-404 */
orc_csr* orc_concat_cols(const orc_csr* G, const orc_csr* Et) {
    const size_t n = (size_t)G->nnz + (size_t)Et->nnz;
    trip* t = (trip*)malloc(sizeof(trip) * (n > 0 ? n : 1));
    size_t k = 0;
    for (int r = 0; r < G->rows; ++r)
        for (int q = G->rp[r]; q < G->rp[r + 1]; ++q) t[k++] = (trip){r, G->ci[q], G->v[q]};
    for (int r = 0; r < Et->rows; ++r)
        for (int q = Et->rp[r]; q < Et->rp[r + 1]; ++q) t[k++] = (trip){r, G->cols + Et->ci[q], Et->v[q]};
    orc_csr* m = finalize_trips(G->rows, G->cols + Et->cols, t, n);
    free(t);
    return m;
}

/* SparseMatrix::operator() by binary search (sparse.hpp:93-99) */
static double csr_at(const orc_csr* A, int i, int j) {
    int lo = A->rp[i], hi = A->rp[i + 1];
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (A->ci[mid] < j)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < A->rp[i + 1] && A->ci[lo] == j) ? A->v[lo] : 0.0;
}

static double dotv(const double* a, const double* b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* ------------------------------------------------------------------ dense Cholesky */
/* dense.hpp:20-40 — row-major factor with a tiny shift on non-positive pivots */
static double* chol_factor(const orc_csr* A) {
    const int n = A->rows;
    double* l = (double*)calloc((size_t)n * (size_t)n + 1, sizeof(double));
    double mx = 0.0;
    for (int r = 0; r < n; ++r)
        for (int k = A->rp[r]; k < A->rp[r + 1]; ++k) {
            l[(size_t)r * n + A->ci[k]] = A->v[k];
            if (fabs(A->v[k]) > mx) mx = fabs(A->v[k]);
        }
    const double shift = 1e-13 * (mx > 1.0 ? mx : 1.0);
    for (int j = 0; j < n; ++j) {
        double d = l[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) d -= l[(size_t)j * n + k] * l[(size_t)j * n + k];
        if (d <= 0.0) d = shift;
        d = sqrt(d);
        l[(size_t)j * n + j] = d;
        for (int i = j + 1; i < n; ++i) {
            double s = l[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= l[(size_t)i * n + k] * l[(size_t)j * n + k];
            l[(size_t)i * n + j] = s / d;
        }
    }
    return l;
}

/* dense.hpp:44-56 */
static void chol_solve(const double* l, int n, const double* b, double* x) {
    double* y = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= l[(size_t)i * n + k] * y[k];
        y[i] = s / l[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < n; ++k) s -= l[(size_t)k * n + i] * x[k];
        x[i] = s / l[(size_t)i * n + i];
    }
    free(y);
}

/* ------------------------------------------------------------------ SA-AMG */
/* amg.hpp:58-75 */
static double rho_dinv_a(const orc_csr* A, const double* inv_diag, int iters) {
    const int n = A->rows;
    double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    uint64_t s = 0x9e3779b97f4a7c15ull;
    for (int i = 0; i < n; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        v[i] = 0.5 + (double)(s >> 11) / (double)(1ull << 53);
    }
    double lambda = 1.0;
    for (int it = 0; it < iters; ++it) {
        orc_spmv(A, v, w);
        for (int i = 0; i < n; ++i) w[i] *= inv_diag[i];
        lambda = sqrt(dotv(w, w, n));
        if (lambda == 0.0) {
            lambda = 1.0;
            break;
        }
        for (int i = 0; i < n; ++i) v[i] = w[i] / lambda;
    }
    free(v);
    free(w);
    return lambda;
}

double orc_rho(const orc_csr* A, int iters) {
    double* d = (double*)malloc(sizeof(double) * (size_t)(A->rows > 0 ? A->rows : 1));
    for (int i = 0; i < A->rows; ++i) d[i] = 1.0 / csr_at(A, i, i);
    const double r = rho_dinv_a(A, d, iters);
    free(d);
    return r;
}

/* amg.hpp:110-123 — strong connections on the core block only */
static orc_csr* strength_graph(const orc_csr* A, double theta, int n_core) {
    double* diag = (double*)malloc(sizeof(double) * (size_t)(A->rows > 0 ? A->rows : 1));
    const int nd = A->rows < A->cols ? A->rows : A->cols;
    for (int i = 0; i < nd; ++i) diag[i] = csr_at(A, i, i);
    orc_csr* S = orc_csr_new(n_core, n_core, A->rp[n_core]);
    int out = 0;
    for (int i = 0; i < n_core; ++i) {
        for (int k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const int j = A->ci[k];
            if (j == i || j >= n_core) continue;
            const double bound = theta * sqrt(fabs(diag[i] * diag[j]));
            if (fabs(A->v[k]) >= bound && bound > 0.0) {
                S->ci[out] = j;
                S->v[out] = 1.0;
                ++out;
            }
        }
        S->rp[i + 1] = out;
    }
    S->nnz = out;
    free(diag);
    return S;
}

/* amg.hpp:79-107 — three-pass sequential greedy aggregation */
static int aggregate(const orc_csr* S, int* agg) {
    const int n = S->rows;
    for (int i = 0; i < n; ++i) agg[i] = -1;
    int count = 0;
    for (int i = 0; i < n; ++i) {
        if (agg[i] != -1) continue;
        int free_nbhd = 1;
        for (int k = S->rp[i]; k < S->rp[i + 1]; ++k)
            if (agg[S->ci[k]] != -1) {
                free_nbhd = 0;
                break;
            }
        if (!free_nbhd) continue;
        agg[i] = count;
        for (int k = S->rp[i]; k < S->rp[i + 1]; ++k) agg[S->ci[k]] = count;
        ++count;
    }
    for (int i = 0; i < n; ++i) {
        if (agg[i] != -1) continue;
        for (int k = S->rp[i]; k < S->rp[i + 1]; ++k) {
            const int j = S->ci[k];
            if (agg[j] != -1) {
                agg[i] = agg[j];
                break;
            }
        }
    }
    for (int i = 0; i < n; ++i)
        if (agg[i] == -1) agg[i] = count++;
    return count;
}

int orc_aggregate(const orc_csr* A, double theta, int n_core, int* agg) {
    orc_csr* S = strength_graph(A, theta, n_core);
    const int n = aggregate(S, agg);
    orc_csr_free(S);
    return n;
}

static orc_csr* csr_copy(const orc_csr* A) { return orc_csr_from(A->rows, A->cols, A->rp, A->ci, A->v); }

/* amg.hpp:127-194 */
orc_hier* orc_sa_build(const orc_csr* A_fine, double theta, int max_coarse, int max_levels, int power_its, int tail_opt) {
    if (A_fine->rows != A_fine->cols) return NULL;
    orc_hier* h = (orc_hier*)calloc(1, sizeof(orc_hier));
    const int cap = max_levels > 0 ? max_levels : 1;
    h->A = (orc_csr**)calloc((size_t)cap, sizeof(orc_csr*));
    h->P = (orc_csr**)calloc((size_t)cap, sizeof(orc_csr*));
    h->Pt = (orc_csr**)calloc((size_t)cap, sizeof(orc_csr*));
    h->inv_diag = (double**)calloc((size_t)cap, sizeof(double*));
    h->omega = (double*)calloc((size_t)cap, sizeof(double));
    orc_csr* A = csr_copy(A_fine);
    const int tail = tail_opt < A_fine->rows ? tail_opt : A_fine->rows;
    for (int lev = 0; lev < max_levels && A->rows > max_coarse + tail; ++lev) {
        const double theta_l = theta * pow(0.5, lev);
        const int n_core = A->rows - tail;
        orc_csr* S = strength_graph(A, theta_l, n_core);
        int* agg = (int*)malloc(sizeof(int) * (size_t)(n_core > 0 ? n_core : 1));
        const int n_agg = aggregate(S, agg);
        orc_csr_free(S);
        if (n_agg >= n_core) {
            h->stalled = 1;
            free(agg);
            break;
        }
        double* inv_diag = (double*)malloc(sizeof(double) * (size_t)A->rows);
        for (int i = 0; i < A->rows; ++i) {
            const double d = csr_at(A, i, i);
            if (d == 0.0) { /* std::invalid_argument (amg.hpp:147) */
                free(agg);
                free(inv_diag);
                orc_csr_free(A);
                orc_hier_free(h);
                return NULL;
            }
            inv_diag[i] = 1.0 / d;
        }
        const double rho = rho_dinv_a(A, inv_diag, power_its);
        const double omega = (4.0 / 3.0) / rho;

        int* agg_size = (int*)calloc((size_t)n_agg, sizeof(int));
        for (int i = 0; i < n_core; ++i) ++agg_size[agg[i]];
        /* P_tent (amg.hpp:156-161): rows >= n_core are empty */
        orc_csr* Pt_ent = orc_csr_new(A->rows, n_agg, n_core);
        for (int i = 0; i < n_core; ++i) {
            Pt_ent->ci[i] = agg[i];
            Pt_ent->v[i] = 1.0 / sqrt((double)agg_size[agg[i]]);
            Pt_ent->rp[i + 1] = i + 1;
        }
        for (int i = n_core; i < A->rows; ++i) Pt_ent->rp[i + 1] = n_core;
        /* DA = scaled_rows(inv_diag) (sparse.hpp:148) */
        orc_csr* DA = csr_copy(A);
        for (int r = 0; r < A->rows; ++r)
            for (int k = DA->rp[r]; k < DA->rp[r + 1]; ++k) DA->v[k] *= inv_diag[r];
        orc_csr* DAP = orc_spmm_rows(DA, 0, DA->rows, Pt_ent);
        orc_csr* Pc = orc_add(1.0, Pt_ent, -omega, DAP);
        orc_csr* P;
        if (tail > 0) {
            const size_t n = (size_t)Pc->nnz + (size_t)tail;
            int* r = (int*)malloc(sizeof(int) * n);
            int* c = (int*)malloc(sizeof(int) * n);
            double* v = (double*)malloc(sizeof(double) * n);
            size_t k = 0;
            for (int row = 0; row < n_core; ++row)
                for (int q = Pc->rp[row]; q < Pc->rp[row + 1]; ++q) {
                    r[k] = row;
                    c[k] = Pc->ci[q];
                    v[k] = Pc->v[q];
                    ++k;
                }
            for (int t2 = 0; t2 < tail; ++t2) {
                r[k] = n_core + t2;
                c[k] = n_agg + t2;
                v[k] = 1.0;
                ++k;
            }
            P = orc_from_triplets(A->rows, n_agg + tail, (int)k, r, c, v);
            free(r);
            free(c);
            free(v);
            orc_csr_free(Pc);
        } else {
            P = Pc;
        }
        orc_csr* Pt = orc_transpose(P);
        orc_csr* Ac = orc_triple(Pt, A, P, Pt->rows > 1 ? Pt->rows : 1, NULL, NULL);
        h->A[lev] = A;
        h->P[lev] = P;
        h->Pt[lev] = Pt;
        h->inv_diag[lev] = inv_diag;
        h->omega[lev] = omega;
        h->n_levels = lev + 1;
        A = Ac;
        free(agg);
        free(agg_size);
        orc_csr_free(Pt_ent);
        orc_csr_free(DA);
        orc_csr_free(DAP);
    }
    h->coarse_A = A;
    h->n_c = A->rows;
    h->chol = chol_factor(A);
    return h;
}

void orc_hier_free(orc_hier* h) {
    if (!h) return;
    for (int l = 0; l < h->n_levels; ++l) {
        orc_csr_free(h->A[l]);
        orc_csr_free(h->P[l]);
        orc_csr_free(h->Pt[l]);
        free(h->inv_diag[l]);
    }
    free(h->A);
    free(h->P);
    free(h->Pt);
    free(h->inv_diag);
    free(h->omega);
    orc_csr_free(h->coarse_A);
    free(h->chol);
    free(h);
}

/* amg.hpp:198-225 — V(1,1) with damped Jacobi, recursive */
static void v_cycle(const orc_hier* h, int lev, const double* b, double* x) {
    if (lev == h->n_levels) {
        chol_solve(h->chol, h->n_c, b, x);
        return;
    }
    const orc_csr* A = h->A[lev];
    const int n = A->rows;
    const double om = h->omega[lev];
    const double* id = h->inv_diag[lev];
    for (int i = 0; i < n; ++i) x[i] = om * id[i] * b[i];
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    orc_spmv(A, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const int nc = h->P[lev]->cols;
    double* rc = (double*)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    double* ec = (double*)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    orc_spmv(h->Pt[lev], r, rc);
    v_cycle(h, lev + 1, rc, ec);
    double* corr = (double*)malloc(sizeof(double) * (size_t)n);
    orc_spmv(h->P[lev], ec, corr);
    for (int i = 0; i < n; ++i) x[i] += corr[i];
    orc_spmv(A, x, r);
    for (int i = 0; i < n; ++i) x[i] += om * id[i] * (b[i] - r[i]);
    free(r);
    free(rc);
    free(ec);
    free(corr);
}

void orc_sa_apply(const orc_hier* h, const double* r, double* z) { v_cycle(h, 0, r, z); }

/* ------------------------------------------------------------------ PCG */
/* krylov.hpp:70-136; kind 0 identity, 1 diagonal (krylov.hpp:51-62), 2 SA */
int orc_pcg(const orc_csr* A, const double* b, const double* x0, int kind, const orc_hier* h, double rel_tol,
            int max_iters, double* x, int* iters, double* rel_res, int* status, double* history, int hist_cap,
            int* hist_len) {
    if (!(rel_tol > 0.0 && rel_tol < 1.0) || max_iters < 1) return 1;
    if (A->rows != A->cols) return 1;
    const int n = A->rows;
    int hl = 0;
#define PUSH_HIST(val)                               \
    do {                                             \
        if (history && hl < hist_cap) history[hl] = (val); \
        ++hl;                                        \
    } while (0)
    for (int i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
    *iters = 0;
    *rel_res = 0.0;
    *status = 0;
    const double bnorm = sqrt(dotv(b, b, n));
    if (bnorm == 0.0) {
        for (int i = 0; i < n; ++i) x[i] = 0.0;
        if (hist_len) *hist_len = 0;
        return 0;
    }
    double* inv_diag = NULL;
    if (kind == 1) {
        inv_diag = (double*)malloc(sizeof(double) * (size_t)n);
        for (int i = 0; i < n; ++i) {
            const double d = csr_at(A, i, i);
            if (d == 0.0) {
                free(inv_diag);
                return 1;
            }
            inv_diag[i] = 1.0 / d;
        }
    }
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    double* p = (double*)malloc(sizeof(double) * (size_t)n);
    double* Ap = (double*)malloc(sizeof(double) * (size_t)n);
    orc_spmv(A, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double rel = sqrt(dotv(r, r, n)) / bnorm;
    PUSH_HIST(rel);
    int done = 0;
    if (rel <= rel_tol) {
        *rel_res = rel;
        done = 1;
    }
#define APPLY_M()                                                        \
    do {                                                                 \
        if (kind == 0)                                                   \
            memcpy(z, r, sizeof(double) * (size_t)n);                    \
        else if (kind == 1)                                              \
            for (int i = 0; i < n; ++i) z[i] = r[i] * inv_diag[i];      \
        else                                                             \
            orc_sa_apply(h, r, z);                                       \
    } while (0)
    if (!done) {
        APPLY_M();
        memcpy(p, z, sizeof(double) * (size_t)n);
        double rz = dotv(r, z, n);
        int it;
        for (it = 1; it <= max_iters; ++it) {
            orc_spmv(A, p, Ap);
            const double pAp = dotv(p, Ap, n);
            if (pAp <= 0.0) {
                *iters = it - 1;
                *rel_res = rel;
                *status = 2;
                done = 1;
                break;
            }
            const double alpha = rz / pAp;
            for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
            for (int i = 0; i < n; ++i) r[i] += -alpha * Ap[i];
            rel = sqrt(dotv(r, r, n)) / bnorm;
            PUSH_HIST(rel);
            if (rel <= rel_tol) {
                *iters = it;
                *rel_res = rel;
                *status = 0;
                done = 1;
                break;
            }
            APPLY_M();
            const double rz_new = dotv(r, z, n);
            const double beta = rz_new / rz;
            rz = rz_new;
            for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
        if (!done) {
            *iters = max_iters;
            *rel_res = rel;
            *status = 1;
        }
    }
    if (hist_len) *hist_len = hl;
    free(inv_diag);
    free(r);
    free(z);
    free(p);
    free(Ap);
    return 0;
#undef APPLY_M
#undef PUSH_HIST
}

/* ------------------------------------------------------------------ E / H */
/* body.hpp:19-28 */
double orc_delta_roma(double r, double h) {
    const double a = fabs(r) / h;
    if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * a * a)) / (3.0 * h);
    if (a <= 1.5) {
        const double t = 1.0 - a;
        return (5.0 - 3.0 * a - sqrt(1.0 - 3.0 * t * t)) / (6.0 * h);
    }
    return 0.0;
}

/* operators.hpp:238-249 */
static void support_range(const double* coords, int lo, int hi, double xi, double rad, int* first, int* last) {
    *first = hi + 1;
    *last = hi;
    for (int i = lo; i <= hi; ++i) {
        const double d = coords[i] - xi;
        if (d > -rad && d < rad) {
            if (i < *first) *first = i;
            *last = i;
        }
    }
}

/* operators.hpp:264-342 (E) and :307-342 (H); staggered ids grid.hpp:47-48 */
int orc_assemble_EH(int nx, int ny, const double* x_faces, const double* y_faces, const double* x_c,
                    const double* y_c, const double* del_x, const double* del_y, double h, const double* uni,
                    int n_b, const double* px, const double* py, const double* ds, orc_csr** E, orc_csr** H) {
    const int n_u = (nx - 1) * ny;
    const int n_q = n_u + nx * (ny - 1);
    const double rad = 1.5 * h;
    const size_t cap = (size_t)n_b * 18 + 1;
    trip* te = (trip*)malloc(sizeof(trip) * cap);
    trip* th = (trip*)malloc(sizeof(trip) * cap);
    size_t ke = 0, kh = 0;
    for (int k = 0; k < n_b; ++k) {
        const double x = px[k], y = py[k];
        const double margin = rad * (1.0 - 1e-9); /* grid.hpp:22-24 contains_point */
        if (!(x >= uni[0] + margin && x <= uni[1] - margin && y >= uni[2] + margin && y <= uni[3] - margin)) {
            free(te);
            free(th);
            return 2;
        }
        int i0, i1, j0, j1;
        support_range(x_faces, 1, nx - 1, x, rad, &i0, &i1);
        support_range(y_c, 0, ny - 1, y, rad, &j0, &j1);
        for (int j = j0; j <= j1; ++j)
            for (int i_f = i0; i_f <= i1; ++i_f) {
                const double dd = orc_delta_roma(x_faces[i_f] - x, h);
                const double de = orc_delta_roma(y_c[j] - y, h);
                const double w = del_x[i_f - 1] * dd * de;
                const double wh = ds[k] * dd * de;
                const int col = (i_f - 1) + j * (nx - 1);
                if (w != 0.0) te[ke++] = (trip){k, col, w};
                if (wh != 0.0) th[kh++] = (trip){col, k, wh};
            }
        support_range(x_c, 0, nx - 1, x, rad, &i0, &i1);
        support_range(y_faces, 1, ny - 1, y, rad, &j0, &j1);
        for (int j_f = j0; j_f <= j1; ++j_f)
            for (int i = i0; i <= i1; ++i) {
                const double dd = orc_delta_roma(x_c[i] - x, h);
                const double de = orc_delta_roma(y_faces[j_f] - y, h);
                const double w = del_y[j_f - 1] * dd * de;
                const double wh = ds[k] * dd * de;
                const int col = n_u + i + (j_f - 1) * nx;
                if (w != 0.0) te[ke++] = (trip){n_b + k, col, w};
                if (wh != 0.0) th[kh++] = (trip){col, n_b + k, wh};
            }
    }
    *E = finalize_trips(2 * n_b, n_q, te, ke);
    *H = finalize_trips(n_q, 2 * n_b, th, kh);
    free(te);
    free(th);
    return 0;
}

/*
 * oracle/ks_oracle.c -- plain CPU oracle for the dense CG / BiCGSTAB hot path of
 * arXiv 1511.07174.  TEST INFRASTRUCTURE ONLY (see ks_oracle.h): the product path
 * never loads this file.
 *
 * Every function cites the passage it follows.  PAPER.md fixes only the building
 * blocks ("inner products, saxpy and matrix-vector products", sec.2),
 * CG's finite termination, and the method names (BiCGSTAB,
 * PAPER.md:33 sec.2).  The step-by-step listings are the textbook recurrences
 * SURVEY.md sec.8(c).3 (Hestenes-Stiefel CG, the paper's ref [9]) and sec.8(c).4
 * (van der Vorst BiCGSTAB), with the readings Q1-Q26 listed in DESIGN.md.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math,
 * no -march=native), so `s += a*b` is one rounded multiply then one rounded add.
 */
#include "ks_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Building blocks -- SURVEY.md sec.8(c).1; PAPER.md:29 ("inner products,   */
/* saxpy and matrix-vector products").  Sequential, index order, from +0.0.  */
/* ------------------------------------------------------------------------- */

/* dot(x, y) = sum_i x_i * y_i */
double or_dot(int64_t n, const double* x, const double* y) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

/* nrm2(x) = sqrt(sum_i x_i^2), no rescaling (reading Q12) */
double or_nrm2(int64_t n, const double* x) { return sqrt(or_dot(n, x, x)); }

/* axpy: y_i <- alpha*x_i + y_i */
void or_axpy(int64_t n, double alpha, const double* x, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = alpha * x[i] + y[i];
}

/* GEMV: y_i = sum_{j<n} a_ij x_j, A row-major (north star).  The row loop may run
 * on several threads; each row's sum stays sequential, so the result is bitwise
 * independent of `threads`. */
void or_gemv(int64_t m, int64_t n, const double* A, int64_t lda, const double* x, double* y,
             int32_t threads) {
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        const double* a = A + i * lda;
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += a[j] * x[j];
        y[i] = s;
    }
}

/* ------------------------------------------------------------------------- */
/* Generators -- SURVEY.md sec.8(d).2, re-implemented here independently.    */
/* ------------------------------------------------------------------------- */

/* SplitMix64 finaliser (ext: Steele, Lea & Flood 2014), uint64 wraparound. */
static uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* H(seed, stream, key) = sm64(sm64(seed ^ (stream << 56)) + key) */
uint64_t or_hash(uint64_t seed, uint64_t stream, uint64_t key) {
    return sm64(sm64(seed ^ (stream << 56)) + key);
}

/* U53 = (H >> 11) * 2^-53, exact in [0,1) */
static double u53(uint64_t seed, uint64_t stream, uint64_t key) {
    return (double)(or_hash(seed, stream, key) >> 11) * (1.0 / 9007199254740992.0);
}

/* G-SPD sign s_i = 1 - 2*(H(seed,4,i) >> 63) */
static double spd_sign(uint64_t seed, int64_t i) {
    return (or_hash(seed, 4, (uint64_t)i) >> 63) ? -1.0 : 1.0;
}

/* One row of the generated matrix.
 *   G-SPD: A_ij = s_i s_j c[(i-j) mod n]            (sign flips only: exact)
 *   G-DD : h_ij = ((H(seed,0,i*n+j) >> 44) - 2^19) * 2^-20, j != i
 *          A_ii = R_i * (17/16 * (1 + k_i)), R_i = sum_{j!=i} |h_ij|,
 *          k_i = (H(seed,1,i) >> 32) mod kd       (every step exact)        */
void or_gen_row(const or_gen* g, int64_t i, double* row) {
    const int64_t n = g->n;
    if (g->kind == 0) {
        const double si = spd_sign(g->seed, i);
        for (int64_t j = 0; j < n; ++j) {
            int64_t d = i - j;
            if (d < 0) d += n;
            row[j] = si * spd_sign(g->seed, j) * g->table[d];
        }
    } else {
        double R = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) { row[j] = 0.0; continue; }
            uint64_t h = or_hash(g->seed, 0, (uint64_t)i * (uint64_t)n + (uint64_t)j);
            double v = (double)((int64_t)(h >> 44) - 524288) * (1.0 / 1048576.0);
            row[j] = v;
            R += fabs(v);
        }
        uint64_t k = (or_hash(g->seed, 1, (uint64_t)i) >> 32) % (uint64_t)g->kd;
        double factor = (17.0 * (double)(1 + k)) / 16.0;
        row[i] = R * factor;
    }
}

void or_gen_rows(const or_gen* g, int64_t r0, int64_t nrows, double* A, int64_t lda) {
    for (int64_t r = 0; r < nrows; ++r) or_gen_row(g, r0 + r, A + r * lda);
}

/* The same rows expanded by `threads` OpenMP threads (rows are independent, so
 * the result is bitwise equal to or_gen_rows); used to store the n = 65536
 * matrices on the host for the full-size parity runs and the CPU baseline. */
void or_gen_rows_par(const or_gen* g, int64_t r0, int64_t nrows, double* A, int64_t lda,
                     int32_t threads) {
#pragma omp parallel for schedule(static) num_threads(threads < 1 ? 1 : threads)
    for (int64_t r = 0; r < nrows; ++r) or_gen_row(g, r0 + r, A + r * lda);
}

/* b_i = 2*U53(seed,2,i) - 1 */
void or_gen_rhs(int64_t n, uint64_t seed, double* b) {
    for (int64_t i = 0; i < n; ++i) b[i] = 2.0 * u53(seed, 2, (uint64_t)i) - 1.0;
}

/* ------------------------------------------------------------------------- */
/* Operator: stored A, or rows generated on the fly (same entries, same order) */
/* ------------------------------------------------------------------------- */

void or_op_rows(const or_op* op, int64_t r0, int64_t nrows, const double* x, double* y) {
    const int64_t n = op->n;
    int threads = op->threads < 1 ? 1 : op->threads;
    if (op->A) {
        or_gemv(nrows, n, op->A + r0 * op->lda, op->lda, x, y, threads);
        return;
    }
#pragma omp parallel num_threads(threads)
    {
        double* row = (double*)malloc((size_t)n * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t r = 0; r < nrows; ++r) {
            or_gen_row(op->gen, r0 + r, row);
            double s = 0.0;
            for (int64_t j = 0; j < n; ++j) s += row[j] * x[j];
            y[r] = s;
        }
        free(row);
    }
}

void or_op_apply(const or_op* op, const double* x, double* y) { or_op_rows(op, 0, op->n, x, y); }

static int finite(double v) { return isfinite(v); }

static void trace_store(double* tr, int64_t cap, int64_t k, int64_t n, const double* v) {
    if (tr && k < cap) memcpy(tr + k * n, v, (size_t)n * sizeof(double));
}

/* ------------------------------------------------------------------------- */
/* CG -- SURVEY.md sec.8(c).3 (Hestenes-Stiefel; "solves SPD    */
/* systems and in exact arithmetic gives the solution for at most n          */
/* iterations"; PAPER.md:123 ref [9]).  Line numbers refer to that listing.  */
/* trace_* (nullable, trace_cap x n each) receive x_k, r_k, p_k for k >= 0.  */
/* ------------------------------------------------------------------------- */
int or_cg(const or_op* op, const double* b, const double* x0, double tol, int64_t maxit,
          double* x, double* hist, int64_t hist_cap, or_report* rep,
          double* trace_x, double* trace_r, double* trace_p, int64_t trace_cap) {
    const int64_t n = op->n;
    or_report R;
    memset(&R, 0, sizeof R);
    if (n < 1 || tol < 0 || maxit < 0) { R.status = OR_EARG; if (rep) *rep = R; return OR_EARG; }

    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* p = (double*)malloc((size_t)n * sizeof(double));
    double* q = (double*)malloc((size_t)n * sizeof(double));

    /* 1: nb = ||b||; b = 0 -> x = 0, 0 iterations, converged (Q6) */
    double nb = or_nrm2(n, b);
    if (nb == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        R.converged = 1; R.status = OR_OK; R.relres = 0.0;
        goto done;
    }
    /* 2: r = b - A x0 (r = b when x0 absent, Q5); p = r; rho = <r,r> */
    if (x0) {
        for (int64_t i = 0; i < n; ++i) x[i] = x0[i];
        or_op_apply(op, x, q);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
    } else {
        for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; }
    }
    for (int64_t i = 0; i < n; ++i) p[i] = r[i];
    double rho = or_dot(n, r, r);
    trace_store(trace_x, trace_cap, 0, n, x);
    trace_store(trace_r, trace_cap, 0, n, r);
    trace_store(trace_p, trace_cap, 0, n, p);

    /* 3: 0-iteration exit (Q2) */
    R.relres = sqrt(rho) / nb;
    if (R.relres <= tol) { R.converged = 1; R.status = OR_OK; goto done; }

    R.status = OR_EMAXIT;
    for (int64_t k = 1; k <= maxit; ++k) {
        or_op_apply(op, p, q);                                  /* 5: q = A p          */
        double sigma = or_dot(n, p, q);                         /* 6: sigma = <p,q>    */
        if (!(sigma > 0.0)) { R.status = OR_ENOTSPD; R.iterations = k - 1; break; } /* Q9 */
        double alpha = rho / sigma;                             /* 7                   */
        or_axpy(n, alpha, p, x);                                /* 8: x = x + alpha p  */
        or_axpy(n, -alpha, q, r);                               /* 9: r = r - alpha q  */
        double rho1 = or_dot(n, r, r);                          /* 10                  */
        double rel = sqrt(rho1) / nb;
        if (hist && k - 1 < hist_cap) hist[k - 1] = rel;
        R.relres = rel;
        R.iterations = k;
        trace_store(trace_x, trace_cap, k, n, x);
        trace_store(trace_r, trace_cap, k, n, r);
        if (rel <= tol) { R.converged = 1; R.status = OR_OK; break; }   /* 11 (Q1) */
        double beta = rho1 / rho;                               /* 12                  */
        for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rho = rho1;
        trace_store(trace_p, trace_cap, k, n, p);
    }
    if (R.status == OR_EMAXIT) R.iterations = maxit;            /* 13                  */
done:
    R.matvecs = R.iterations;
    free(r); free(p); free(q);
    if (rep) *rep = R;
    return R.status;
}

/* ------------------------------------------------------------------------- */
/* BiCGSTAB -- SURVEY.md sec.8(c).4 (van der Vorst 1992; the paper names the */
/* method at PAPER.md:33 and lists it at PAPER.md:78, 109).  Shadow residual */
/* rhat = r0 (Q7); rho_old = alpha = omega = 1, v = p = 0 (Q8); breakdown    */
/* on an exactly-zero or non-finite scalar (Q9); half-step exit on ||s||     */
/* (Q2).  trace_s / trace_r (nullable) receive s_i, r_i, i>=1.  */
/* ------------------------------------------------------------------------- */
int or_bicgstab(const or_op* op, const double* b, const double* x0, double tol, int64_t maxit,
                double* x, double* hist, int64_t hist_cap, or_report* rep,
                double* trace_s, double* trace_r, int64_t trace_cap) {
    const int64_t n = op->n;
    or_report R;
    memset(&R, 0, sizeof R);
    if (n < 1 || tol < 0 || maxit < 0) { R.status = OR_EARG; if (rep) *rep = R; return OR_EARG; }

    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* rhat = (double*)malloc((size_t)n * sizeof(double));
    double* p = (double*)calloc((size_t)n, sizeof(double));
    double* v = (double*)calloc((size_t)n, sizeof(double));
    double* s = (double*)malloc((size_t)n * sizeof(double));
    double* t = (double*)malloc((size_t)n * sizeof(double));

    /* 1 */
    double nb = or_nrm2(n, b);
    if (nb == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        R.converged = 1; R.status = OR_OK;
        goto done;
    }
    /* 2: r = b - A x0; rhat = r; rho_old = alpha = omega = 1; v = p = 0 */
    if (x0) {
        for (int64_t i = 0; i < n; ++i) x[i] = x0[i];
        or_op_apply(op, x, t);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
    } else {
        for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; }
    }
    for (int64_t i = 0; i < n; ++i) rhat[i] = r[i];
    double rho_old = 1.0, alpha = 1.0, omega = 1.0;

    /* 3 */
    R.relres = or_nrm2(n, r) / nb;
    if (R.relres <= tol) { R.converged = 1; R.status = OR_OK; goto done; }

    R.status = OR_EMAXIT;
    for (int64_t i = 1; i <= maxit; ++i) {
        double rho = or_dot(n, rhat, r);                                        /* 5  */
        if (rho == 0.0 || !finite(rho)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        double beta = (rho / rho_old) * (alpha / omega);                        /* 6  */
        for (int64_t j = 0; j < n; ++j) p[j] = r[j] + beta * (p[j] - omega * v[j]); /* 7 */
        or_op_apply(op, p, v);                                                  /* 8  */
        double g = or_dot(n, rhat, v);                                          /* 9  */
        if (g == 0.0 || !finite(g)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        alpha = rho / g;                                                        /* 10 */
        for (int64_t j = 0; j < n; ++j) s[j] = r[j] - alpha * v[j];             /* 11 */
        trace_store(trace_s, trace_cap, i - 1, n, s);
        double srel = or_nrm2(n, s) / nb;                                       /* 12 */
        if (srel <= tol) {
            or_axpy(n, alpha, p, x);
            if (hist && i - 1 < hist_cap) hist[i - 1] = srel;
            R.relres = srel; R.half_step_exit = 1; R.converged = 1; R.status = OR_OK;
            R.iterations = i;
            break;
        }
        or_op_apply(op, s, t);                                                  /* 13 */
        double tt = or_dot(n, t, t);
        if (tt == 0.0 || !finite(tt)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        double om = or_dot(n, t, s) / tt;                                       /* 14 */
        if (om == 0.0 || !finite(om)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        omega = om;
        for (int64_t j = 0; j < n; ++j) x[j] = (x[j] + alpha * p[j]) + omega * s[j]; /* 15 */
        for (int64_t j = 0; j < n; ++j) r[j] = s[j] - omega * t[j];             /* 16 */
        trace_store(trace_r, trace_cap, i - 1, n, r);
        double rel = or_nrm2(n, r) / nb;
        if (hist && i - 1 < hist_cap) hist[i - 1] = rel;
        R.relres = rel;
        R.iterations = i;
        if (rel <= tol) { R.converged = 1; R.status = OR_OK; break; }           /* 17 */
        rho_old = rho;                                                          /* 18 */
    }
    if (R.status == OR_EMAXIT) R.iterations = maxit;                            /* 19 */
done:
    R.matvecs = 2 * R.iterations - (R.half_step_exit ? 1 : 0);
    free(r); free(rhat); free(p); free(v); free(s); free(t);
    if (rep) *rep = R;
    return R.status;
}

/* ------------------------------------------------------------------------- */
/* Transposed GEMV: y_j = sum_{i<m} a_ij x_i, A row-major m x n (sequential   */
/* in i for every j).  BiCG's "system's matrix and its transpose" */
/* ------------------------------------------------------------------------- */
void or_gemv_t(int64_t m, int64_t n, const double* A, int64_t lda, const double* x, double* y) {
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) s += A[i * lda + j] * x[i];
        y[j] = s;
    }
}

/* ------------------------------------------------------------------------- */
/* BiCG -- PAPER.md:33 sec.2: "BiCG generates two mutually orthogonal       */
/* sequences of residual vectors and A-orthogonal sequences of direction     */
/* vectors.  The updates for residuals and for the direction vectors are     */
/* similar to those of the CG method, but are performed using system's       */
/* matrix and its transpose."  Listing (Fletcher 1976; ext: Barrett et al.,  */
/* Templates sec.2.3.5), shadow residual rt0 = r0 (Q7), exact-zero or         */
/* non-finite rho / <pt, A p> -> BREAKDOWN (Q9), test on ||r_k||/||b|| (Q1):   */
/*   r = b - A x0; rt = r; rho = <rt, r>; p = r; pt = rt                     */
/*   for k = 1..maxit:                                                        */
/*     q = A p; qt = A^T pt; sigma = <pt, q>; alpha = rho / sigma             */
/*     x += alpha p; r -= alpha q; rt -= alpha qt                             */
/*     hist[k-1] = ||r||/||b||; converged -> stop                              */
/*     rho1 = <rt, r>; beta = rho1 / rho; p = r + beta p; pt = rt + beta pt    */
/* trace_* (nullable) receive r_k, rt_k, p_k, pt_k for k = 0..trace_cap-1.    */
/* ------------------------------------------------------------------------- */
int or_bicg(int64_t n, const double* A, int64_t lda, const double* b, const double* x0, double tol,
            int64_t maxit, double* x, double* hist, int64_t hist_cap, or_report* rep,
            double* trace_r, double* trace_rt, double* trace_p, double* trace_pt, int64_t trace_cap) {
    or_report R;
    memset(&R, 0, sizeof R);
    if (n < 1 || tol < 0 || maxit < 0) { R.status = OR_EARG; if (rep) *rep = R; return OR_EARG; }
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* rt = (double*)malloc((size_t)n * sizeof(double));
    double* p = (double*)malloc((size_t)n * sizeof(double));
    double* pt = (double*)malloc((size_t)n * sizeof(double));
    double* q = (double*)malloc((size_t)n * sizeof(double));
    double* qt = (double*)malloc((size_t)n * sizeof(double));
    double nb = or_nrm2(n, b);
    if (nb == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        R.converged = 1; R.status = OR_OK;
        goto done;
    }
    if (x0) {
        for (int64_t i = 0; i < n; ++i) x[i] = x0[i];
        or_gemv(n, n, A, lda, x, q, 1);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
    } else {
        for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; }
    }
    for (int64_t i = 0; i < n; ++i) { rt[i] = r[i]; p[i] = r[i]; pt[i] = r[i]; }
    double rho = or_dot(n, rt, r);
    trace_store(trace_r, trace_cap, 0, n, r);
    trace_store(trace_rt, trace_cap, 0, n, rt);
    trace_store(trace_p, trace_cap, 0, n, p);
    trace_store(trace_pt, trace_cap, 0, n, pt);
    R.relres = or_nrm2(n, r) / nb;
    if (R.relres <= tol) { R.converged = 1; R.status = OR_OK; goto done; }
    R.status = OR_EMAXIT;
    for (int64_t k = 1; k <= maxit; ++k) {
        if (rho == 0.0 || !finite(rho)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = k - 1; break; }
        or_gemv(n, n, A, lda, p, q, 1);                     /* q = A p     */
        or_gemv_t(n, n, A, lda, pt, qt);                    /* qt = A^T pt */
        double sigma = or_dot(n, pt, q);
        if (sigma == 0.0 || !finite(sigma)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = k - 1; break; }
        double alpha = rho / sigma;
        or_axpy(n, alpha, p, x);
        or_axpy(n, -alpha, q, r);
        or_axpy(n, -alpha, qt, rt);
        double rel = or_nrm2(n, r) / nb;
        if (hist && k - 1 < hist_cap) hist[k - 1] = rel;
        R.relres = rel;
        R.iterations = k;
        trace_store(trace_r, trace_cap, k, n, r);
        trace_store(trace_rt, trace_cap, k, n, rt);
        if (rel <= tol) { R.converged = 1; R.status = OR_OK; break; }
        double rho1 = or_dot(n, rt, r);
        double beta = rho1 / rho;
        for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        for (int64_t i = 0; i < n; ++i) pt[i] = rt[i] + beta * pt[i];
        trace_store(trace_p, trace_cap, k, n, p);
        trace_store(trace_pt, trace_cap, k, n, pt);
        rho = rho1;
    }
    if (R.status == OR_EMAXIT) R.iterations = maxit;
done:
    R.matvecs = 2 * R.iterations;
    free(r); free(rt); free(p); free(pt); free(q); free(qt);
    if (rep) *rep = R;
    return R.status;
}

/* ------------------------------------------------------------------------- */
/* GMRES(m) -- PAPER.md:31 sec.2: "GMRES uses a Gram-Schmidt                 */
/* orthogonalization process and requires the storage and computation of an  */
/* increasing amount of information at each iteration.  These difficulties   */
/* can be alleviated by restarting the computations after a fixed number of  */
/* iterations.  The intermediate results are then used as a new initial      */
/* point."  Listing (Saad & Schultz 1986, the paper's ref [20]): Arnoldi with */
/* modified Gram-Schmidt (SPEC.md design decision), Givens rotations for the  */
/* least-squares residual, restart from the current x.                        */
/*   cycle: r = b - A x; beta = ||r||; v_1 = r / beta; g = beta e_1           */
/*     for j = 1..m:  w = A v_j                                               */
/*        for i = 1..j: h_ij = <w, v_i>; w -= h_ij v_i          (MGS)         */
/*        h_{j+1,j} = ||w||; v_{j+1} = w / h_{j+1,j} (unless 0: exact)        */
/*        apply rotations 1..j-1 to column j; new rotation zeroes h_{j+1,j};  */
/*        g_{j+1} = -s_j g_j; g_j = c_j g_j                                    */
/*        hist[k-1] = |g_{j+1}| / ||b||  (k = total inner steps)               */
/*        stop the cycle if hist <= tol, h_{j+1,j} == 0 or k == maxit          */
/*     solve H y = g (upper triangular, back substitution); x += V y           */
/* iterations = total inner steps; converged when the implicit residual       */
/* |g_{j+1}|/||b|| <= tol (Q1 analogue).                                       */
/* ------------------------------------------------------------------------- */
int or_gmres(int64_t n, const double* A, int64_t lda, const double* b, const double* x0, double tol,
             int64_t restart, int64_t maxit, double* x, double* hist, int64_t hist_cap, or_report* rep) {
    or_report R;
    memset(&R, 0, sizeof R);
    if (n < 1 || tol < 0 || maxit < 0 || restart < 1) { R.status = OR_EARG; if (rep) *rep = R; return OR_EARG; }
    const int64_t m = restart;
    double* V = (double*)malloc((size_t)(m + 1) * (size_t)n * sizeof(double));
    double* H = (double*)calloc((size_t)(m + 1) * (size_t)m, sizeof(double));   /* H[i*m + j] */
    double* cs = (double*)malloc((size_t)m * sizeof(double));
    double* sn = (double*)malloc((size_t)m * sizeof(double));
    double* g = (double*)malloc((size_t)(m + 1) * sizeof(double));
    double* y = (double*)malloc((size_t)m * sizeof(double));
    double* w = (double*)malloc((size_t)n * sizeof(double));
    double nb = or_nrm2(n, b);
    int64_t k = 0;
    if (nb == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        R.converged = 1; R.status = OR_OK;
        goto done;
    }
    for (int64_t i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
    R.status = OR_EMAXIT;
    for (;;) {
        or_gemv(n, n, A, lda, x, w, 1);                       /* r = b - A x */
        for (int64_t i = 0; i < n; ++i) w[i] = b[i] - w[i];
        double beta = or_nrm2(n, w);
        R.relres = beta / nb;
        if (R.relres <= tol) { R.converged = 1; R.status = OR_OK; break; }
        if (k >= maxit) break;
        for (int64_t i = 0; i < n; ++i) V[i] = w[i] / beta;
        for (int64_t i = 0; i <= m; ++i) g[i] = 0.0;
        g[0] = beta;
        int64_t j = 0, jdone = 0;
        int stop = 0;
        for (j = 0; j < m && k < maxit; ++j) {
            const double* vj = V + j * n;
            or_gemv(n, n, A, lda, vj, w, 1);                   /* w = A v_j */
            for (int64_t i = 0; i <= j; ++i) {                 /* MGS */
                double h = or_dot(n, w, V + i * n);
                H[i * m + j] = h;
                or_axpy(n, -h, V + i * n, w);
            }
            double hn = or_nrm2(n, w);
            H[(j + 1) * m + j] = hn;
            if (hn != 0.0)
                for (int64_t i = 0; i < n; ++i) V[(j + 1) * n + i] = w[i] / hn;
            for (int64_t i = 0; i < j; ++i) {                  /* previous rotations */
                double a = H[i * m + j], c = H[(i + 1) * m + j];
                H[i * m + j] = cs[i] * a + sn[i] * c;
                H[(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
            }
            double a = H[j * m + j], c = H[(j + 1) * m + j];
            double den = sqrt(a * a + c * c);
            cs[j] = a / den;
            sn[j] = c / den;
            H[j * m + j] = den;
            H[(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++k;
            double rel = fabs(g[j + 1]) / nb;
            if (hist && k - 1 < hist_cap) hist[k - 1] = rel;
            R.relres = rel;
            jdone = j + 1;
            if (rel <= tol || hn == 0.0) { stop = 1; break; }
        }
        for (int64_t i = jdone - 1; i >= 0; --i) {             /* back substitution */
            double s = g[i];
            for (int64_t l = i + 1; l < jdone; ++l) s -= H[i * m + l] * y[l];
            y[i] = s / H[i * m + i];
        }
        for (int64_t i = 0; i < jdone; ++i) or_axpy(n, y[i], V + i * n, x);
        if (stop) { R.converged = 1; R.status = OR_OK; break; }
        if (k >= maxit) break;
    }
    R.iterations = k;
done:
    R.matvecs = R.iterations;
    free(V); free(H); free(cs); free(sn); free(g); free(y); free(w);
    if (rep) *rep = R;
    return R.status;
}

/* ------------------------------------------------------------------------- */
/* Single precision CG / BiCGSTAB -- NEXT-4.  Line-for-line the listings of   */
/* sec.8(c).3 / .4 (and or_cg / or_bicgstab above) in binary32; x0 = 0.      */
/* ------------------------------------------------------------------------- */
static float dot_f(int64_t n, const float* x, const float* y) {
    float s = 0.0f;
    for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}
static void gemv_f(int64_t n, const float* A, int64_t lda, const float* x, float* y) {
    for (int64_t i = 0; i < n; ++i) {
        const float* a = A + i * lda;
        float s = 0.0f;
        for (int64_t j = 0; j < n; ++j) s += a[j] * x[j];
        y[i] = s;
    }
}

int or_cg_f32(int64_t n, const float* A, int64_t lda, const float* b, float tol, int64_t maxit,
              float* x, float* hist, int64_t hist_cap, or_report* rep) {
    or_report R;
    memset(&R, 0, sizeof R);
    float* r = (float*)malloc((size_t)n * sizeof(float));
    float* p = (float*)malloc((size_t)n * sizeof(float));
    float* q = (float*)malloc((size_t)n * sizeof(float));
    const float nb = sqrtf(dot_f(n, b, b));
    for (int64_t i = 0; i < n; ++i) { x[i] = 0.0f; r[i] = b[i]; p[i] = b[i]; }
    if (nb == 0.0f) { R.converged = 1; R.status = OR_OK; goto done; }
    float rho = dot_f(n, r, r);
    R.relres = sqrtf(rho) / nb;
    if (R.relres <= tol) { R.converged = 1; R.status = OR_OK; goto done; }
    R.status = OR_EMAXIT;
    for (int64_t k = 1; k <= maxit; ++k) {
        gemv_f(n, A, lda, p, q);
        const float sigma = dot_f(n, p, q);
        if (!(sigma > 0.0f)) { R.status = OR_ENOTSPD; R.iterations = k - 1; break; }
        const float alpha = rho / sigma;
        for (int64_t i = 0; i < n; ++i) x[i] = alpha * p[i] + x[i];
        for (int64_t i = 0; i < n; ++i) r[i] = -alpha * q[i] + r[i];
        const float rho1 = dot_f(n, r, r);
        const float rel = sqrtf(rho1) / nb;
        if (hist && k - 1 < hist_cap) hist[k - 1] = rel;
        R.relres = rel;
        R.iterations = k;
        if (rel <= tol) { R.converged = 1; R.status = OR_OK; break; }
        const float beta = rho1 / rho;
        for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rho = rho1;
    }
    if (R.status == OR_EMAXIT) R.iterations = maxit;
done:
    R.matvecs = R.iterations;
    free(r); free(p); free(q);
    if (rep) *rep = R;
    return R.status;
}

int or_bicgstab_f32(int64_t n, const float* A, int64_t lda, const float* b, float tol, int64_t maxit,
                    float* x, float* hist, int64_t hist_cap, or_report* rep) {
    or_report R;
    memset(&R, 0, sizeof R);
    float* r = (float*)malloc((size_t)n * sizeof(float));
    float* rhat = (float*)malloc((size_t)n * sizeof(float));
    float* p = (float*)calloc((size_t)n, sizeof(float));
    float* v = (float*)calloc((size_t)n, sizeof(float));
    float* s = (float*)malloc((size_t)n * sizeof(float));
    float* t = (float*)malloc((size_t)n * sizeof(float));
    const float nb = sqrtf(dot_f(n, b, b));
    float rho_old = 1.0f, alpha = 1.0f, omega = 1.0f;
    for (int64_t i = 0; i < n; ++i) { x[i] = 0.0f; r[i] = b[i]; rhat[i] = b[i]; }
    if (nb == 0.0f) { R.converged = 1; R.status = OR_OK; goto done; }
    R.relres = sqrtf(dot_f(n, r, r)) / nb;
    if (R.relres <= tol) { R.converged = 1; R.status = OR_OK; goto done; }
    R.status = OR_EMAXIT;
    for (int64_t i = 1; i <= maxit; ++i) {
        const float rho = dot_f(n, rhat, r);
        if (rho == 0.0f || !isfinite(rho)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        const float beta = (rho / rho_old) * (alpha / omega);
        for (int64_t j = 0; j < n; ++j) p[j] = r[j] + beta * (p[j] - omega * v[j]);
        gemv_f(n, A, lda, p, v);
        const float g = dot_f(n, rhat, v);
        if (g == 0.0f || !isfinite(g)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        alpha = rho / g;
        for (int64_t j = 0; j < n; ++j) s[j] = r[j] - alpha * v[j];
        const float srel = sqrtf(dot_f(n, s, s)) / nb;
        if (srel <= tol) {
            for (int64_t j = 0; j < n; ++j) x[j] = alpha * p[j] + x[j];
            if (hist && i - 1 < hist_cap) hist[i - 1] = srel;
            R.relres = srel; R.half_step_exit = 1; R.converged = 1; R.status = OR_OK; R.iterations = i;
            break;
        }
        gemv_f(n, A, lda, s, t);
        const float tt = dot_f(n, t, t);
        if (tt == 0.0f || !isfinite(tt)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        const float om = dot_f(n, t, s) / tt;
        if (om == 0.0f || !isfinite(om)) { R.status = OR_EBREAKDOWN; R.breakdown = 1; R.iterations = i - 1; break; }
        omega = om;
        for (int64_t j = 0; j < n; ++j) x[j] = (x[j] + alpha * p[j]) + omega * s[j];
        for (int64_t j = 0; j < n; ++j) r[j] = s[j] - omega * t[j];
        const float rel = sqrtf(dot_f(n, r, r)) / nb;
        if (hist && i - 1 < hist_cap) hist[i - 1] = rel;
        R.relres = rel;
        R.iterations = i;
        if (rel <= tol) { R.converged = 1; R.status = OR_OK; break; }
        rho_old = rho;
    }
    if (R.status == OR_EMAXIT) R.iterations = maxit;
done:
    R.matvecs = 2 * R.iterations - (R.half_step_exit ? 1 : 0);
    free(r); free(rhat); free(p); free(v); free(s); free(t);
    if (rep) *rep = R;
    return R.status;
}

/* ------------------------------------------------------------------------- */
/* Reference solutions -- SURVEY.md sec.8(c).5                               */
/* ------------------------------------------------------------------------- */

/* Gaussian elimination with partial pivoting in long double (PAPER.md:37-40
 * describe LU with partial pivoting, ref [9]; pivot ties -> smallest row index,
 * SPEC.md:191).  Returns OR_ESINGULAR on an exactly-zero pivot. */
int or_ge_solve_ld(int64_t n, const double* A, int64_t lda, const double* b, double* x) {
    long double* M = (long double*)malloc((size_t)n * (size_t)n * sizeof(long double));
    long double* y = (long double*)malloc((size_t)n * sizeof(long double));
    if (!M || !y) { free(M); free(y); return OR_EARG; }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < n; ++j) M[i * n + j] = (long double)A[i * lda + j];
        y[i] = (long double)b[i];
    }
    int status = OR_OK;
    for (int64_t k = 0; k < n; ++k) {
        int64_t piv = k;
        long double best = fabsl(M[k * n + k]);
        for (int64_t i = k + 1; i < n; ++i) {
            long double a = fabsl(M[i * n + k]);
            if (a > best) { best = a; piv = i; }
        }
        if (best == 0.0L) { status = OR_ESINGULAR; break; }
        if (piv != k) {
            for (int64_t j = 0; j < n; ++j) {
                long double tmp = M[k * n + j]; M[k * n + j] = M[piv * n + j]; M[piv * n + j] = tmp;
            }
            long double tmp = y[k]; y[k] = y[piv]; y[piv] = tmp;
        }
        for (int64_t i = k + 1; i < n; ++i) {
            long double l = M[i * n + k] / M[k * n + k];
            if (l == 0.0L) continue;
            for (int64_t j = k + 1; j < n; ++j) M[i * n + j] -= l * M[k * n + j];
            y[i] -= l * y[k];
        }
    }
    if (status == OR_OK) {
        for (int64_t i = n - 1; i >= 0; --i) {           /* back substitution Ux = y */
            long double s = y[i];
            for (int64_t j = i + 1; j < n; ++j) s -= M[i * n + j] * y[j];
            y[i] = s / M[i * n + i];
        }
        for (int64_t i = 0; i < n; ++i) x[i] = (double)y[i];
    }
    free(M); free(y);
    return status;
}

/* In-place DFT of (re, im), sign -1 forward / +1 inverse (no 1/n), long double.
 * Radix-2 iterative FFT when n is a power of two, else the O(n^2) definition. */
static void dft_ld(int64_t n, long double* re, long double* im, int sign) {
    const long double PI = 3.141592653589793238462643383279502884L;
    if (n > 1 && (n & (n - 1)) == 0) {
        for (int64_t i = 1, j = 0; i < n; ++i) {               /* bit reversal */
            int64_t bit = n >> 1;
            for (; j & bit; bit >>= 1) j ^= bit;
            j ^= bit;
            if (i < j) {
                long double t = re[i]; re[i] = re[j]; re[j] = t;
                t = im[i]; im[i] = im[j]; im[j] = t;
            }
        }
        for (int64_t len = 2; len <= n; len <<= 1) {
            int64_t half = len >> 1;
            for (int64_t k = 0; k < half; ++k) {
                long double ang = sign * 2.0L * PI * (long double)k / (long double)len;
                long double wr = cosl(ang), wi = sinl(ang);
                for (int64_t i = k; i < n; i += len) {
                    long double ur = re[i], ui = im[i];
                    long double vr = re[i + half] * wr - im[i + half] * wi;
                    long double vi = re[i + half] * wi + im[i + half] * wr;
                    re[i] = ur + vr; im[i] = ui + vi;
                    re[i + half] = ur - vr; im[i + half] = ui - vi;
                }
            }
        }
        return;
    }
    long double* outr = (long double*)malloc((size_t)n * sizeof(long double));
    long double* outi = (long double*)malloc((size_t)n * sizeof(long double));
    for (int64_t k = 0; k < n; ++k) {
        long double sr = 0.0L, si = 0.0L;
        for (int64_t j = 0; j < n; ++j) {
            int64_t idx = (j * k) % n;
            long double ang = sign * 2.0L * PI * (long double)idx / (long double)n;
            long double c = cosl(ang), s = sinl(ang);
            sr += re[j] * c - im[j] * s;
            si += re[j] * s + im[j] * c;
        }
        outr[k] = sr; outi[k] = si;
    }
    memcpy(re, outr, (size_t)n * sizeof(long double));
    memcpy(im, outi, (size_t)n * sizeof(long double));
    free(outr); free(outi);
}

/* Closed-form G-SPD solution (pin P6):
 * A = S C S with C circulant (first column c), S = diag(s_i), S^2 = I, so
 * x* = S C^{-1} S b and C^{-1} y = IDFT(DFT(y) / DFT(c)) (convolution theorem),
 * where DFT(c) are the exact eigenvalues of the rounded table. */
void or_spd_exact_solve_ld(int64_t n, const double* table, uint64_t seed, const double* b,
                           double* x) {
    long double* yr = (long double*)malloc((size_t)n * sizeof(long double));
    long double* yi = (long double*)calloc((size_t)n, sizeof(long double));
    long double* lr = (long double*)malloc((size_t)n * sizeof(long double));
    long double* li = (long double*)calloc((size_t)n, sizeof(long double));
    for (int64_t i = 0; i < n; ++i) {
        yr[i] = (long double)spd_sign(seed, i) * (long double)b[i];
        lr[i] = (long double)table[i];
    }
    dft_ld(n, yr, yi, -1);
    dft_ld(n, lr, li, -1);
    for (int64_t k = 0; k < n; ++k) {          /* (a+ib)/(c+id) */
        long double den = lr[k] * lr[k] + li[k] * li[k];
        long double a = yr[k], bb = yi[k];
        yr[k] = (a * lr[k] + bb * li[k]) / den;
        yi[k] = (bb * lr[k] - a * li[k]) / den;
    }
    dft_ld(n, yr, yi, +1);
    for (int64_t i = 0; i < n; ++i)
        x[i] = (double)((long double)spd_sign(seed, i) * yr[i] / (long double)n);
    free(yr); free(yi); free(lr); free(li);
}

/* ||b - A x|| / ||b|| with long-double accumulation (pin P11). */
double or_true_relres_ld(const or_op* op, const double* b, const double* x) {
    const int64_t n = op->n;
    int threads = op->threads < 1 ? 1 : op->threads;
    long double rr = 0.0L, bb = 0.0L;
    for (int64_t i = 0; i < n; ++i) bb += (long double)b[i] * (long double)b[i];
#pragma omp parallel num_threads(threads) reduction(+ : rr)
    {
        double* row = op->A ? NULL : (double*)malloc((size_t)n * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            const double* a;
            if (op->A) a = op->A + i * op->lda;
            else { or_gen_row(op->gen, i, row); a = row; }
            long double s = (long double)b[i];
            for (int64_t j = 0; j < n; ++j) s -= (long double)a[j] * (long double)x[j];
            rr += s * s;
        }
        free(row);
    }
    return (double)(sqrtl(rr) / sqrtl(bb));
}

/*
 * oracle/ks_oracle.h -- plain, slow, obviously-correct CPU oracle for the dense
 * Krylov hot path of arXiv 1511.07174 (CUPLSS; sec.2, sec.2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table generator or constant with the CUDA path (paper_1511_07174_b200/),
 * and neither side includes or links the other.
 *
 * Arithmetic rules: IEEE binary64, round-to-nearest; every
 * GEMV row, dot and norm accumulates sequentially in index order from +0.0;
 * compiled -O2 -ffp-contract=off (no FMA contraction, no reassociation).
 * long double (x87, 64-bit significand) is used only for the reference solutions
 * (Gaussian elimination, closed-form circulant solve) and true residuals.
 */
#ifndef KS_ORACLE_H
#define KS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same meanings as SPEC.md:675 exit codes (2 = dimension,
 * 3 = not SPD, 4 = max iterations, 5 = breakdown); defined here independently. */
enum { OR_OK = 0, OR_EARG = 1, OR_EDIM = 2, OR_ENOTSPD = 3, OR_EMAXIT = 4, OR_EBREAKDOWN = 5,
       OR_ESINGULAR = 6 };

typedef struct {
    int64_t iterations;     /* completed loop bodies (Q3)                      */
    int64_t matvecs;        /* CG: iterations; BiCGSTAB: 2*iterations - half    */
    int32_t converged, breakdown, half_step_exit, status;
    double  relres;         /* recurrence ||r_k||/||b|| at exit (Q1)             */
} or_report;

/* Matrix source: either a stored row-major array, or a generator spec
 * (SURVEY.md sec.8(d) G-SPD / G-DD) expanded on the fly one row at a time. */
typedef struct {
    int32_t kind;           /* 0 = G-SPD, 1 = G-DD                                 */
    int64_t n;
    uint64_t seed;
    int32_t kd;             /* G-DD diagonal classes                               */
    const double* table;    /* G-SPD circulant table c (n doubles), borrowed       */
} or_gen;

typedef struct {
    int64_t n;
    const double* A;        /* row-major, A[i*lda + j]; NULL -> use gen            */
    int64_t lda;
    const or_gen* gen;
    int32_t threads;        /* row-parallel GEMV threads (rows stay sequential)    */
} or_op;

/* --- building blocks --- */
double or_dot(int64_t n, const double* x, const double* y);
double or_nrm2(int64_t n, const double* x);
void   or_axpy(int64_t n, double alpha, const double* x, double* y);
void   or_gemv(int64_t m, int64_t n, const double* A, int64_t lda, const double* x, double* y,
               int32_t threads);
void   or_op_apply(const or_op* op, const double* x, double* y);
void   or_op_rows(const or_op* op, int64_t r0, int64_t nrows, const double* x, double* y);

/* --- solvers --- */
int or_cg(const or_op* op, const double* b, const double* x0, double tol, int64_t maxit,
          double* x, double* hist, int64_t hist_cap, or_report* rep,
          double* trace_x, double* trace_r, double* trace_p, int64_t trace_cap);
int or_bicgstab(const or_op* op, const double* b, const double* x0, double tol, int64_t maxit,
                double* x, double* hist, int64_t hist_cap, or_report* rep,
                double* trace_s, double* trace_r, int64_t trace_cap);

/* --- the paper's other Krylov methods --- */
void or_gemv_t(int64_t m, int64_t n, const double* A, int64_t lda, const double* x, double* y);
int or_bicg(int64_t n, const double* A, int64_t lda, const double* b, const double* x0, double tol,
            int64_t maxit, double* x, double* hist, int64_t hist_cap, or_report* rep,
            double* trace_r, double* trace_rt, double* trace_p, double* trace_pt, int64_t trace_cap);
int or_gmres(int64_t n, const double* A, int64_t lda, const double* b, const double* x0, double tol,
             int64_t restart, int64_t maxit, double* x, double* hist, int64_t hist_cap, or_report* rep);

/* --- single precision ---
 * The same listings evaluated in IEEE binary32: float storage, float products,
 * float sequential sums (no FMA), float scalars.  A is row-major float.        */
int or_cg_f32(int64_t n, const float* A, int64_t lda, const float* b, float tol, int64_t maxit,
              float* x, float* hist, int64_t hist_cap, or_report* rep);
int or_bicgstab_f32(int64_t n, const float* A, int64_t lda, const float* b, float tol, int64_t maxit,
                    float* x, float* hist, int64_t hist_cap, or_report* rep);

/* --- reference solutions --- */
int    or_ge_solve_ld(int64_t n, const double* A, int64_t lda, const double* b, double* x);
void   or_spd_exact_solve_ld(int64_t n, const double* table, uint64_t seed, const double* b,
                             double* x);
double or_true_relres_ld(const or_op* op, const double* b, const double* x);

/* --- generators, independent re-implementation --- */
uint64_t or_hash(uint64_t seed, uint64_t stream, uint64_t key);
void or_gen_row(const or_gen* g, int64_t i, double* row);
void or_gen_rows(const or_gen* g, int64_t r0, int64_t nrows, double* A, int64_t lda);
void or_gen_rows_par(const or_gen* g, int64_t r0, int64_t nrows, double* A, int64_t lda,
                     int32_t threads);
void or_gen_rhs(int64_t n, uint64_t seed, double* b);

#ifdef __cplusplus
}
#endif
#endif

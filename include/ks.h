/*
 * include/ks.h -- C ABI of the B200-native dense Krylov hot path (arXiv 1511.07174).
 *
 * What it computes.  The per-iteration body of the paper's non-stationary Krylov
 * solvers on a dense matrix: "inner products, saxpy and matrix-vector products
 * that has the complexity of O(n^2)" (sec.2) for CG on SPD systems
 * and BiCGSTAB on nonsymmetric systems (sec.2; listed as
 * implemented at PAPER.md:78 and PAPER.md:109).  The recurrences are the
 * textbook ones written out in SURVEY.md sec.8(c).3 (CG) and sec.8(c).4
 * (BiCGSTAB); every reading of a point the paper leaves open is listed in
 * DESIGN.md ("Readings", Q1-Q27).  Parallelism is hidden behind an opaque
 * object, as the paper asks ("encapsulation of data and distribution and
 * communication in opaque objects").
 *
 * Layout.  A is n x n, ROW-MAJOR (element (i,j) at A[i*lda + j]), FP64.  It is
 * split into contiguous row blocks, one per GPU: shard g owns rows
 * [g*floor(n/P) + min(g, n mod P), ...) (ks_row_range).  On the device each row
 * is padded to a multiple of 512 doubles (4 KiB); the padding is zero.
 *
 * Pointers.  Every vector argument of ks_matvec / ks_cg / ks_bicgstab may be
 * host memory (pageable or pinned) or CUDA device memory: copies use
 * cudaMemcpyDefault (unified addressing).  Buffers are owned by the caller,
 * read or written only during the call, never retained.  Every call is
 * synchronous: it returns after its outputs are in the caller's memory.
 *
 * Errors.  Every call returns a ks_status.  Argument errors (KS_EARG, KS_EDIM)
 * are detected before any work.  KS_ECUDA / KS_ENCCL / KS_ENOMEM poison the
 * context: later calls return KS_ESTATE except ks_destroy.  The library never
 * aborts, exits, prints or throws across this ABI; ks_last_error() returns a
 * message.  A context is used by one caller thread at a time.
 */
#ifndef KS_H
#define KS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ks_ctx ks_ctx; /* opaque handle */

/* Storage and arithmetic precision of the device path.  KS_FLOAT32 (SURVEY.md
 * NEXT-4; the paper's experiments are single precision): A and every
 * device vector in binary32, half the HBM bytes per GEMV.  The ABI stays FP64
 * (host/device double buffers, converted on the device).  FP32 supports ks_cg and
 * ks_bicgstab with x0 = NULL on the persistent path (P == 1, or P > 1 with peer
 * access); ks_bicg, ks_gmres, ks_matvec_t and x0 != NULL return KS_EARG.        */
typedef enum { KS_FLOAT64 = 0, KS_FLOAT32 = 1 } ks_dtype;

typedef enum {
    KS_OK = 0,         /* converged (or call succeeded)                         */
    KS_EARG = 1,       /* invalid argument                                      */
    KS_EDIM = 2,       /* dimension mismatch          (SPEC.md:675 exit code 2) */
    KS_ENOTSPD = 3,    /* CG: <p, A p> <= 0 or non-finite      (exit code 3)    */
    KS_EMAXIT = 4,     /* maxit reached without convergence    (exit code 4)    */
    KS_EBREAKDOWN = 5, /* BiCGSTAB scalar exactly 0 / non-finite (exit code 5)  */
    KS_ECUDA = 6,      /* CUDA runtime error (poisons the context)              */
    KS_ENCCL = 7,      /* NCCL error (poisons the context)                      */
    KS_ENOMEM = 8,     /* device allocation failed (poisons the context)        */
    KS_ESTATE = 9      /* context poisoned, or matrix not fully loaded          */
} ks_status;

typedef struct {
    int64_t iterations;    /* completed loop bodies (Q3); the setup     */
                           /* GEMV r0 = b - A x0 is never counted                  */
    int64_t matvecs;       /* CG: iterations; BiCGSTAB: 2*iterations - half_step   */
    int32_t converged;     /* 1 if relres <= tol                                   */
    int32_t breakdown;     /* 1 on a BiCGSTAB breakdown                            */
    int32_t half_step_exit;/* 1 if BiCGSTAB stopped on ||s||         */
    int32_t status;        /* the ks_status the call returned                      */
    double relres;         /* recurrence ||r_k||/||b|| at exit (Q1)                 */
    double true_relres;    /* ||b - A x||/||b|| with one extra GEMV (or -1 if off) */
    double seconds_loop;   /* CUDA-event time of the iteration loop (max over      */
                           /* this context's GPUs); excludes setup and copies      */
    double seconds_total;  /* host wall-clock of the whole call                    */
    double seconds_gemv;   /* CUDA-event time of the kernels that ran the loop's    */
                           /* GEMVs: the K1 launches, or (persistent mode) the     */
                           /* whole-iteration kernels, which also run the vector   */
                           /* phases; 0 unless KS_OPT_PROFILE_GEMV = 1             */
    int64_t gemv_launches; /* GEMVs executed inside the loop (per GPU)             */
    int64_t kernel_launches; /* all library kernel launches of the call (per GPU)  */
} ks_report;

/* Synthetic-input generator spec.
 *   kind 0 = G-SPD: A_ij = s_i s_j c[(i-j) mod n]; spd_table = c (host, n doubles,
 *            borrowed during the call), s_i = 1 - 2 (H(seed,4,i) >> 63).
 *   kind 1 = G-DD : dense nonsymmetric, strictly row-diagonally dominant, exact
 *            dyadic entries; kd = number of diagonal classes.
 *   b_i = 2 U53(seed,2,i) - 1.  H is SplitMix64 as specified in DESIGN.md.     */
typedef struct {
    int32_t kind;
    uint64_t seed;
    double kappa;             /* informational for G-SPD (the table fixes A)      */
    int32_t kd;
    const double* spd_table;
} ks_gen_spec;

typedef enum {
    KS_OPT_TRUE_RESIDUAL = 0, /* 1 (default): report true_relres (one extra GEMV) */
    KS_OPT_PROFILE_GEMV = 1,  /* 1: time every K1 launch with CUDA events         */
    KS_OPT_POLL_BATCH = 2,    /* iterations per done-flag poll; 0 (default) =     */
                              /* auto: the whole solve in one persistent launch,  */
                              /* 16 on the multi-kernel path                      */
    KS_OPT_GEMV_ROWS = 3,     /* K1 rows per CTA tile: 2, 4, 8, 16 (0 = auto)     */
    KS_OPT_GEMV_SPLIT = 4,    /* K1 column splits per tile (0 = auto)             */
    KS_OPT_GEMV_KERNEL = 5,   /* K1 variant: 0 = auto, 1 = LDG stream (the only   */
                              /* one; round 1's TMA ring was removed)             */
    KS_OPT_USE_GRAPHS = 6,    /* 1: replay each poll batch as a CUDA graph        */
    KS_OPT_FUSED_COMM = 7,    /* 1 (default): when P > 1 and every GPU pair has   */
                              /* peer access, the producing kernels store their   */
                              /* slices/partials straight into every rank's       */
                              /* exchange buffer over NVLink and release an epoch */
                              /* flag (no NCCL call in the loop); 0: NCCL         */
                              /* allgathers.  ks_get_option returns the effective */
                              /* mode.                                            */
    KS_OPT_PERSISTENT = 8,    /* 0: one kernel per step; 1: one persistent        */
                              /* cooperative kernel per poll batch (grid barriers */
                              /* instead of kernel boundaries; needs P == 1 or    */
                              /* the fused exchange); 2 (default): auto (on when  */
                              /* eligible).  ks_get_option returns the effective  */
                              /* mode.                                            */
    KS_OPT_GEMV_UNROLL = 9,   /* tuning: K1 LDG column-block unroll 1/2/4/8 (0 =  */
                              /* the default for the row count)                   */
    KS_OPT_PERSIST_GRID = 10, /* tuning: cap on the persistent kernels' CTA count */
                              /* (0 = auto; the grid must be equal on all ranks)  */
    KS_OPT_GEMVT_SHAPE = 11,  /* tuning: K1T 16-byte vectors per                  */
                              /* thread per row (1/2/4) * 100 + rows in flight    */
                              /* (4/8/16); default 204 (profiles/r01_gemvt_sweep) */
    KS_OPT_SMALL = 12,        /* persistent path: 1 = small-n kernels that keep   */
                              /* the full vectors in every CTA's shared memory    */
                              /* (CG and BiCGSTAB on one GPU: 1 / 2 grid barriers */
                              /* per iteration; on P > 1 GPUs with the fused      */
                              /* exchange CG: one q exchange + 1 barrier,         */
                              /* BiCGSTAB: v and t exchanges + 2 barriers) when   */
                              /* they fit; 0 = off; 2 (default) = auto (on        */
                              /* when a vector is <= 32 KiB: FP64 n <= 4096, FP32 */
                              /* n <= 8192; BiCGSTAB on P > 1: <= 16 KiB)         */
    KS_OPT_JOIN_TIMEOUT_MS = 13, /* fused exchange (P > 1): every solve starts with  */
                              /* an on-device rendezvous of all ranks (no host    */
                              /* sync); a rank that does not arrive within this   */
                              /* many ms (default 120000) fails the solve with    */
                              /* KS_ENCCL.  In-loop waits stay bounded at 10 s.   */
    KS_OPT_TINY = 14,         /* 1 (default): one GPU, FP64, n <= 1024, whole     */
                              /* solve in one launch -> the register-resident     */
                              /* kernels (A in shared memory, vectors replicated  */
                              /* in registers, LL-format exchange of the GEMV     */
                              /* output: no grid barrier); 0 = off                */
    KS_OPT_JITTER = 15,       /* race detection: seed (0 = off, default) of       */
                              /* pseudo-random delays (<= ~4 us, a quarter of the */
                              /* visits) at every synchronisation point of the    */
                              /* persistent, small, tiny and multi-RHS kernels    */
                              /* (grid-barrier arrival / departure, flag publish  */
                              /* and wait, LL store and poll).  Results must not  */
                              /* change: the kernels' sums have fixed orders and  */
                              /* their exchanges are epoch-tagged, so a run with  */
                              /* jitter equals a run without it bit for bit.      */
    KS_OPT_LL_XCHG = 16       /* 1 (default): the persistent CG / BiCGSTAB        */
                              /* kernels over P > 1 GPUs hand the r / v slices   */
                              /* and the rank partial scalars over as LL words   */
                              /* (32 payload bits + the iteration epoch per 8-B  */
                              /* word, one 16-B system-scope store per value     */
                              /* into every rank) that consumers poll: no fence, */
                              /* no flag.  Same sums in the same order: results   */
                              /* equal the fence + flag handovers (0) bitwise.   */
} ks_option;

/* Creates the opaque object that encapsulates the distributed matrix and its
 * communication ("encapsulation of data and distribution and communication in
 * opaque objects"; the data distribution level of Fig. 2,
 * PAPER.md:64-76; Step 3 "Allocate memory ... in the device memory",
 * PAPER.md:83).  Row blocks instead of the paper's bidimensional mesh
 * (Q24).
 * One process drives GPUs 0..ngpus-1 (one worker thread and stream per GPU, NCCL
 * communicator from ncclCommInitAll when ngpus > 1).  n >= 1, 1 <= ngpus <= 16
 * and <= device count, dtype = KS_FLOAT64 or KS_FLOAT32.  Allocates each shard (m_g x ld)
 * plus O(n) vectors with cudaMalloc and zero-fills them.                        */
ks_status ks_create(ks_ctx** out, int64_t n, ks_dtype dtype, int32_t ngpus);

/* As ks_create, with rank g on device devices[g] (nranks entries, 1..16, each a
 * valid device ordinal).  A device may be listed more than once, to run the P > 1
 * schedule (row-block partition, allgathers of the direction-vector ingredients,
 * rank-ordered scalar sums, x gather: "communication ... encapsulated in
 * opaque objects", PAPER.md:78 data distribution) on fewer GPUs than ranks.  Such a
 * context has no NCCL communicator (NCCL rejects two ranks on one GPU) and never
 * runs kernels that wait on each other (separate launches on one GPU have no
 * co-residency guarantee): its collectives are host-driven peer copies ordered by
 * events, KS_OPT_FUSED_COMM is 0 and cannot be set, and the kernels that need the
 * fused exchange at P > 1 as separate launches are not used.  Instead, with every
 * rank on one GPU, CG / BiCGSTAB with x0 = NULL (whole solve in one launch) run the
 * fused persistent kernels -- or the tiny kernels for n <= 1024 -- of all ranks as
 * ONE cooperative launch (rank = block / CTAs per rank), so their exchanges between
 * ranks run with co-residency guaranteed.  Results equal the oracle's within the
 * same bars (the tiny kernels: bitwise the one-GPU result).
 * KS_EARG for a bad device list, KS_EDIM for n < nranks.                         */
ks_status ks_create_on(ks_ctx** out, int64_t n, ks_dtype dtype, int32_t nranks, const int32_t* devices);

/* One rank of a multi-process job (one process per GPU, e.g. torchrun) -- the
 * paper's one-MPI-process-per-node model ("MPI ... for the
 * communication between processors"), NCCL over NVLink in place of
 * MPI over Ethernet.
 * nccl_comm: a BORROWED ncclComm_t of nranks ranks (e.g. torch's
 * ProcessGroupNCCL._comm_ptr()), or NULL when nranks == 1.  stream: a BORROWED
 * cudaStream_t on `device` (NULL -> the context creates its own).  Both must
 * outlive the context.  The shard of this rank is ks_row_range(ctx, rank).      */
ks_status ks_create_rank(ks_ctx** out, int64_t n, ks_dtype dtype, int32_t rank, int32_t nranks,
                         void* nccl_comm, int32_t device, void* stream);

/* Frees every device allocation of the context (never the borrowed comm/stream):
 * Step 8 "Memory clean up".  Always allowed, also on a poisoned
 * context; ctx == NULL is a no-op returning KS_OK.                              */
ks_status ks_destroy(ks_ctx* ctx);

/* Row range [*row_begin, *row_end) of shard `shard` (0 <= shard < P): the
 * distribution of the matrix over the processors ("distribution of
 * vectors and matrices on processors"; 1-D row blocks, Q15/Q24).
 * shard outside [0, P) -> KS_EARG.                                               */
ks_status ks_row_range(const ks_ctx* ctx, int32_t shard, int64_t* row_begin, int64_t* row_end);

/* Step 4 "Copy matrices from host memory to device memory" for a
 * distributed matrix.
 * Copies rows [row_begin, row_begin + nrows) of A (row-major, leading dimension
 * lda >= n; row r of the argument is global row row_begin + r) into the shards
 * that own them; rows owned by other ranks of a multi-process job are ignored.
 * Rows may be loaded in any chunks; a reloaded row is overwritten.               */
ks_status ks_load_rows(ks_ctx* ctx, int64_t row_begin, int64_t nrows, const double* A, int64_t lda);

/* Step 2 "Initialize matrices and vectors" done on the device: the
 * paper's workload is only "60000 rows and columns", so the
 * synthetic inputs of SURVEY.md sec.8(d).2 are expanded into every shard (K0),
 * bitwise equal to the oracle's expansion.  b (n doubles, generated on the
 * device) goes to b_out if non-NULL.  Bad kind / kd < 1 / missing table ->
 * KS_EARG; marks every row loaded.                                              */
ks_status ks_generate(ks_ctx* ctx, const ks_gen_spec* spec, double* b_out);

/* y = A x (n doubles each).  The plain GEMV building block.        */
ks_status ks_matvec(ks_ctx* ctx, const double* x, double* y);

/* Measurement of the O(n^2) matrix-vector product that dominates a Krylov
 * iteration (SURVEY.md sec.8(d).5 "GEMV metric").
 * Times `reps` back-to-back K1 GEMV launches on device-resident data with CUDA
 * events; *seconds_per_matvec = elapsed/reps (max over this context's GPUs).
 * reps < 1 -> KS_EARG.  No host data is read or written.                        */
ks_status ks_time_matvec(ks_ctx* ctx, int32_t reps, double* seconds_per_matvec);

/* CG.  b: n doubles (required).  x0: n doubles or NULL
 * (zero start).  tol >= 0 (tol = 0 runs exactly maxit iterations unless r = 0).
 * maxit >= 0.  x: n doubles (required), receives the last complete iterate.
 * hist: NULL or hist_cap doubles; receives min(iterations, hist_cap) values
 * ||r_k||/||b||, k = 1..iterations (Q4).  rep: NULL or filled.
 * Returns KS_OK, KS_EMAXIT, KS_ENOTSPD, or an error.  b = 0 -> x = 0, KS_OK.   */
ks_status ks_cg(ks_ctx* ctx, const double* b, const double* x0, double tol, int64_t maxit,
                double* x, double* hist, int64_t hist_cap, ks_report* rep);

/* BiCGSTAB: shadow residual rhat = r0; exact-zero or
 * non-finite scalars -> KS_EBREAKDOWN with x = last complete iterate; a
 * half-step exit records ||s_i||/||b|| as the last history value.               */
ks_status ks_bicgstab(ks_ctx* ctx, const double* b, const double* x0, double tol, int64_t maxit,
                      double* x, double* hist, int64_t hist_cap, ks_report* rep);

/* BiCG (NEXT-3; "performed using system's matrix and its transpose";
 * listed as implemented at PAPER.md:78, 109).  Fletcher's recurrence with shadow
 * residual rt0 = r0 (oracle or_bicg); arguments and returns as ks_cg; an exactly
 * zero or non-finite <rt, r> or <pt, A p> -> KS_EBREAKDOWN.  Two GEMVs per
 * iteration: A p (K1) and A^T pt (K1T, row-block partials reduce-scattered).    */
ks_status ks_bicg(ks_ctx* ctx, const double* b, const double* x0, double tol, int64_t maxit,
                  double* x, double* hist, int64_t hist_cap, ks_report* rep);

/* Restarted GMRES(m) (NEXT-3; "Gram-Schmidt orthogonalization ...
 * restarting the computations after a fixed number of iterations", listed as
 * implemented at PAPER.md:78, 109).  Arnoldi with classical Gram-Schmidt applied
 * twice, Givens rotations, restart from the current x.  1 <= restart <= 63.
 * iterations = total inner (Arnoldi) steps; hist receives the implicit residual
 * |g_{j+1}|/||b|| of every inner step; converged when it is <= tol (or on a
 * lucky breakdown).  Returns KS_OK or KS_EMAXIT (x = the last update).           */
ks_status ks_gmres(ks_ctx* ctx, const double* b, const double* x0, double tol, int32_t restart,
                   int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep);

/* Multi-RHS CG (SURVEY.md sec.8(f) "multi-RHS"; reading Q30): nrhs
 * (1..8) independent CG recurrences of sec.8(c).3 -- column k is exactly the CG of
 * ks_cg on (A, b_k): its own alpha, beta, stopping test and NOTSPD exit -- sharing
 * every pass over A: each iteration is ONE skinny GEMM Q = A P (TMA-fed, FP64), so
 * the HBM bytes per iteration are those of a single GEMV.  Converged columns stop
 * updating; the solve ends when every column has stopped or after maxit.
 * B, X: n x nrhs, column-major (column k at B + k*n), required; X0: same or NULL
 * (zero start).  hist: NULL or hist_cap x nrhs column-major (column k at
 * hist + k*hist_cap), receives min(iterations_k, hist_cap) values ||r||/||b_k||.
 * reps: NULL or nrhs reports (true_relres -1: not computed).  P == 1, or P > 1 with
 * the fused exchange (peer access between all GPUs); FP64 contexts only (else KS_EARG).  Returns the worst column status:
 * KS_ENOTSPD > KS_EMAXIT > KS_OK.                                                 */
ks_status ks_cg_multi(ks_ctx* ctx, int32_t nrhs, const double* B, const double* X0, double tol, int64_t maxit,
                      double* X, double* hist, int64_t hist_cap, ks_report* reps);

/* Multi-RHS BiCGSTAB (reading Q30 applied to sec.8(c).4): nrhs (1..8) independent
 * BiCGSTAB recurrences -- column k is exactly ks_bicgstab on (A, b_k): own rho,
 * alpha, omega, breakdown tests and half-step exit -- sharing both GEMMs of every
 * iteration (v = A P and t = A S, TMA-fed, FP64).  Arguments, layouts and reports as
 * ks_cg_multi (half_step_exit, breakdown, matvecs = 2 iterations - half per column).
 * P == 1, or P > 1 with the fused exchange (v and r slices and the per-column dots
 * exchanged over NVLink in-kernel), FP64.  Returns the worst column status:
 * KS_EBREAKDOWN > KS_EMAXIT > KS_OK.                                              */
ks_status ks_bicgstab_multi(ks_ctx* ctx, int32_t nrhs, const double* B, const double* X0, double tol,
                            int64_t maxit, double* X, double* hist, int64_t hist_cap, ks_report* reps);

/* y = A^T x (n doubles each): the transposed GEMV building block of BiCG (K1T). */
ks_status ks_matvec_t(ks_ctx* ctx, const double* x, double* y);

/* Options select kernels / schedules.  In a multi-process job (ks_create_rank)
 * every rank must set the same options before the same calls: the ranks run one
 * schedule in lockstep (collectives, epoch flags, persistent grid sizes).        */
ks_status ks_set_option(ks_ctx* ctx, ks_option opt, int64_t value);
ks_status ks_get_option(const ks_ctx* ctx, ks_option opt, int64_t* value);

/* Number of GPUs (shards) this context drives locally, and the global P, n and
 * the padded device row length ld (the distribution).              */
ks_status ks_info(const ks_ctx* ctx, int32_t* local_gpus, int32_t* nranks, int64_t* n, int64_t* ld);

/* Guard-zone check (a test facility: compute-sanitizer is not available on the
 * GPU pool).  With the environment variable KS_GUARD=1 set when the library is
 * loaded, every device buffer the library allocates (except the CUDA-IPC exchange
 * buffer) is surrounded by 4 KiB canary zones.  *violations receives the number of
 * zones found corrupted -- out-of-bounds writes by some kernel -- on the context's
 * GPUs now plus any found when buffers were freed; -1 when KS_GUARD is not set.
 * Synchronises the context's devices.                                            */
ks_status ks_check_guards(const ks_ctx* ctx, int64_t* violations);

/* Last error message of ctx (or of the calling thread when ctx == NULL).         */
const char* ks_last_error(const ks_ctx* ctx);

/* Library version string, e.g. "ks 0.1 sm_100a". */
const char* ks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KS_H */

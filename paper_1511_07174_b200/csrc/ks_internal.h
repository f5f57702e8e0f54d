// Internal declarations of the B200 dense Krylov library (not part of the ABI).
// Layering: ks_abi.cpp (L4 C ABI) -> ks_ctx.cpp / ks_solvers.cpp
// (L3 context + L2 schedules) -> ks_gemv.cu / ks_vec.cu / ks_gen.cu (L1 kernels).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ks.h"

namespace ks {

constexpr int kMaxRanks = 16;
constexpr int64_t kColAlign = 512;   // row padding of the device shard (doubles)
constexpr int kScalSlot = 4;         // doubles per rank in the scalar gather buffer
constexpr int kNumTickets = 64;
// Fused-collective phases (one epoch flag per phase and source rank).
constexpr int kPhaseS = 0;   // scalar partials  (CG sigma; BiCGSTAB <t,s>, <t,t>)
constexpr int kPhaseR = 1;   // r slice + <rhat,r>, <r,r> / rho' partials
constexpr int kPhaseV = 2;   // BiCGSTAB v slice + <rhat,v>
constexpr int kPhaseJ = 3;   // solve-start rendezvous (epoch = the solve's ebase)
constexpr int kPhaseX = 4;   // end-of-solve x gather (epoch = ebase + maxit + 1)
constexpr int kNumPhases = 5;
// LL handover region of the persistent kernels over P > 1 GPUs (KS_OPT_LL_XCHG): every
// entry is one double as two 8-byte words (32 payload bits + the 32-bit epoch each),
// stored with one 16-byte system-scope store by the producer straight into every
// rank's region; consumers poll their local copy until both words carry the epoch --
// no fence, no flag.  Layout (u64 words): [2 parities][3 vectors (r, v, spare)][ld] x 2,
// then [2 parities][kLlPhases][kMaxRanks][2 scalars] x 2.
constexpr int kLlPhases = 4;   // 0: CG sigma / BiCGSTAB gamma, 1: rho' / (rhat,r),(r,r), 2: (t,s),(t,t)
__host__ __device__ constexpr int64_t ll_words(int64_t ld) { return 2 * 3 * ld * 2 + 2 * kLlPhases * kMaxRanks * 2 * 2; }
__host__ __device__ inline int64_t ll_vec_off(int64_t ld, int par, int vec, int64_t j) {
    return (((int64_t)par * 3 + vec) * ld + j) * 2;
}
__host__ __device__ inline int64_t ll_scal_off(int64_t ld, int par, int ph, int rank, int q) {
    return 2 * 3 * ld * 2 + ((((int64_t)par * kLlPhases + ph) * kMaxRanks + rank) * 2 + q) * 2;
}

// Peer (NVLink, unified-address) pointers to every rank's exchange buffers,
// parity-0 bases; rank g's own entries point at its local memory.
template <class T>
struct PeerPtrsT {
    T* G_r[kMaxRanks];
    T* G_v[kMaxRanks];
    T* S[kMaxRanks];
    unsigned long long* flags[kMaxRanks];   // [kNumPhases][kMaxRanks] epochs
    T* X[kMaxRanks];                        // full-length x (contiguous), end-of-solve gather
    uint64_t* llg[kMaxRanks];               // LL handover slots of the persistent kernels (P > 1)
};
using PeerPtrs = PeerPtrsT<double>;

// Row partition + gather layout, passed by value to kernels.
struct Layout {
    int P, rank;
    int64_t n, ld;     // n; padded length of full vectors (multiple of kColAlign)
    int64_t chunk;     // stride (doubles) of one rank's chunk in a gather buffer
    int64_t pslot;     // offset of the partial-scalar slots inside a chunk
    int64_t row0[kMaxRanks + 1];
};

// Device-resident solver state (one per rank).  Scalars that a kernel reads and
// a later kernel writes live in 4-deep rings indexed by iteration (k & 3), so no
// kernel ever reads a value another CTA of the same launch may be writing.
struct DevState {
    double nb;                 // ||b||
    double tol;
    double rho[4], alpha[4], omega[4];
    double relres;             // last recorded recurrence relres
    double true_rr;            // ||b - A x||^2 (true residual)
    long long iters;           // completed loop bodies
    long long maxit;
    long long half_iter;       // BiCGSTAB iteration of a half-step exit (0 = none)
    long long hist_cap;
    unsigned long long ebase;  // epoch of iteration k is ebase + k (fused collectives)
    int done, status, converged, breakdown, half, bzero;
    int peer_timeout;          // a fused-collective wait timed out (error)
    unsigned jitter;           // race-detection delays at sync points (KS_OPT_JITTER; 0 off)
    unsigned jitter_pad;
};

// Scratch for deterministic last-block grid reductions.
struct Scratch {
    double* part;        // kNumTickets * kPartStride doubles
    unsigned* ticket;    // kNumTickets
    double* qpart;       // split-K partial rows
    unsigned* tile_ticket;
    int64_t qpart_cap, tile_cap;
};
constexpr int64_t kPartStride = 4096 * 2;

template <class T>
struct GemvParamsT {
    const T* A; int64_t lda; int64_t m; int64_t ncols;
    const T* x;            // padded full input vector (ncols)
    T* y;                  // m outputs
    const T* bsub;         // nullable: y = bsub - A x
    const T* w1;           // nullable: *out1 = <w1, y>
    T* out1;
    T* out2;               // nullable: *out2 = <y, y>
    const int* done;       // nullable: skip when *done != 0
    // Fused publish (peer mode): y rows and/or dot partials stored straight into
    // every rank's exchange buffer, then the phase flag released with the epoch.
    int pub_P = 0, pub_rank = 0;           // 0: no peer publishing
    T* y_peer[kMaxRanks];                  // parity-0 address of row 0 of this rank's slice at rank g
    int64_t ypar = 0;                      // parity stride of y_peer
    int64_t y_par = 0;                     // parity stride applied to the local y
    T* d_peer[kMaxRanks];                  // parity-0 address of this rank's dot slots at rank g
    int64_t dpar = 0;
    unsigned long long* f_peer[kMaxRanks]; // flag [phase][this rank] at rank g
    const unsigned long long* ebase = nullptr;
    const long long* kdev = nullptr;       // epoch = *ebase + koff + (kdev ? *kdev : 0)
    long long koff = 0;
};
using GemvParams = GemvParamsT<double>;

struct GemvConfig {
    int variant;   // 1 = LDG stream, 2 = TMA bulk ring
    int rows;      // R
    int splits;    // S
    int unroll;    // LDG unroll U (0 = default for R)
};

// ---- kernels (launchers return the number of kernel launches issued) -------
int launch_gemv(const GemvParams& p, const GemvConfig& c, const Scratch& s, int ticket_id,
                int num_sms, cudaStream_t st);
GemvConfig choose_gemv(int64_t m, int64_t ncols, int num_sms, int rows_opt, int split_opt,
                       int variant_opt);

// K1T: u = A_loc^T x_loc (BiCG), chunk-layout output; upart holds
// ceil(m / rc_rows) x lda partials, col_ticket lda / 512 counters.
int64_t gemv_t_chunk_rows(int64_t m, int64_t lda, int num_sms, int shape);
bool gemv_t_shape_ok(int64_t shape);   // KS_OPT_GEMVT_SHAPE value check
// Fused reduce-scatter of K1T (BiCG, P > 1, NEXT-1): each column sum is stored
// straight into its owner rank's exchange slot for this rank, and the last column
// block to finish releases `epoch` into every rank's flag slot.
struct GemvTPub {
    int P = 0;                                // 0: plain chunk-layout output
    double* dst[kMaxRanks];                   // rank g: slot of this rank (row j - row0[g])
    unsigned long long* f_peer[kMaxRanks];    // flag [phase][this rank] at rank g
    unsigned long long epoch = 0;
    unsigned* ticket = nullptr;               // column blocks finished (self-resetting)
};
int launch_gemv_t(const double* A, int64_t lda, int64_t m, int64_t n, const double* x,
                  int64_t rc_rows, double* upart, unsigned* col_ticket, double* out, const Layout& L,
                  const int* done, int shape, cudaStream_t st, const GemvTPub* pub = nullptr);

int launch_gen_spd(double* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                   const double* table_dev, cudaStream_t st);
int launch_gen_dd(double* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                  int kd, cudaStream_t st);
int launch_gen_rhs(double* b, int64_t n, uint64_t seed, cudaStream_t st);

// Vector/control kernels (ks_vec.cu).  `G_r`, `G_v` are gather buffers in chunk
// layout; `S` is the scalar gather buffer (kScalSlot doubles per rank).
template <class T>
struct VecArgsT {
    Layout L;
    DevState* st;
    double* hist;          // always FP64 (relres values)
    const T* b_full;       // ld
    T* x_loc;              // m
    T* p_full;             // ld
    T* s_full;             // ld
    T* v_full;             // ld (BiCGSTAB: local copy of the gathered v)
    T* q_loc;              // m (CG q / BiCGSTAB t)
    T* rhat_loc;           // m (BiCGSTAB rhat; BiCG's shadow residual rt)
    T* pt_loc;             // m (BiCG shadow direction pt)
    const T* qt_loc;       // m (BiCG qt = (A^T pt) rows of this rank)
    T* G_r;                // P * chunk
    T* G_v;                // P * chunk
    T* S;                  // P * kScalSlot
    Scratch scr;
    int num_sms;
    // iteration-parity double buffering of G_r / G_v / S (0 in NCCL mode)
    int64_t gpar, spar;
    int peer;              // 1: fused NVLink peer-store collectives
    unsigned jitter;       // KS_OPT_JITTER seed (0: off), ks_device.cuh jitter_at
    int ll;                // 1: LL handovers in the persistent kernels (P > 1, KS_OPT_LL_XCHG)
    uint64_t* llg;         // own LL handover region (ll_words(ld) words), nullptr for P == 1
    PeerPtrsT<T> pp;
    unsigned long long* flags;   // own [kNumPhases][kMaxRanks]
    T* X;                  // own full-length x gather buffer (exchange allocation)
    T* b_full_mut() const { return const_cast<T*>(b_full); }
};
using VecArgs = VecArgsT<double>;

int launch_setup_r(const VecArgs& a, bool have_x0, const double* x0_full, cudaStream_t st);
int launch_setup_local(const VecArgs& a, cudaStream_t st);   // P > 1, x0 = 0: no gather
int launch_cg_init(const VecArgs& a, double tol, long long maxit, long long hist_cap,
                   unsigned long long ebase, cudaStream_t st);
int launch_cg_update(const VecArgs& a, const long long* kdev, long long k, cudaStream_t st);
int launch_cg_direction(const VecArgs& a, const long long* kdev, long long k, cudaStream_t st);
int launch_cg_finish(const VecArgs& a, cudaStream_t st);
int launch_bs_init(const VecArgs& a, double tol, long long maxit, long long hist_cap,
                   unsigned long long ebase, cudaStream_t st);
int launch_bs_p(const VecArgs& a, const long long* kdev, long long i, cudaStream_t st);
int launch_bs_s(const VecArgs& a, const long long* kdev, long long i, cudaStream_t st);
int launch_bs_xr(const VecArgs& a, const long long* kdev, long long i, cudaStream_t st);
int launch_bs_finish(const VecArgs& a, cudaStream_t st);
int launch_true_res_final(const VecArgs& a, cudaStream_t st);
int launch_pack_x(const VecArgs& a, cudaStream_t st);   // x_loc -> G_v own chunk
// out = rank-ordered sum of the P slots S[g*chunk ..] (host-driven reduce-scatter)
int launch_sum_slots(const double* S, int P, int64_t chunk, double* out, int num_sms, cudaStream_t st);
// Solve-start rendezvous of the fused exchange (P > 1): releases `epoch` into
// flag [kPhaseJ][rank] of every rank and waits (bounded by timeout_ms) until every
// rank has released it -- i.e. every rank's stream has finished its previous solve
// and initialised this one.  Host-side skew between ranks is absorbed here, so the
// in-loop waits' timeout only bounds in-kernel skew.  A timeout marks the solve
// failed (KS_ENCCL).  Launched after the init kernel, before the iteration loop.
template <class T>
int launch_join(const VecArgsT<T>& a, unsigned long long epoch, long long timeout_ms, cudaStream_t st);
// Solve start with x0 = 0 in ONE launch (rows A0 / B0): r0 = b into G_r (every rank
// holds all of b: no gather), x = 0, rhat = r0, CG p0 = r0, ||b||^2 = <r0, r0> in
// the partial slots, the solver state (init_state / init_decide), and -- when
// join_ms > 0 (fused P > 1) -- the solve-start rendezvous of launch_join.  It also
// zeroes the persistent kernels' grid-barrier counter (scr.ticket + 8), so the first
// persistent launch of the solve needs no memset (bar_zeroed).
int launch_start(const VecArgs& a, int bicgstab, double tol, long long maxit, long long hist_cap,
                 unsigned long long ebase, long long join_ms, cudaStream_t st);
// Solve end in ONE launch: the k_finish decisions (BiCGSTAB test of the last step,
// EMAXIT, b = 0 -> x = 0) and, when gather (fused P > 1), the x gather: every rank
// stores its rows of x into every rank's contiguous X buffer over NVLink and
// releases kPhaseX with `epoch`; the launch returns when every rank's rows arrived.
int launch_end(const VecArgs& a, int bicgstab, int gather, unsigned long long epoch, cudaStream_t st);
// Iteration kernels use k = koff + (kdev ? *kdev : 0): a captured batch of
// iterations (CUDA graph) is replayed with *kdev advanced by k_advance.
int launch_advance(long long* kdev, long long by, cudaStream_t st);
// GMRES(m) (NEXT-3, ks_gmres.cu)
constexpr int kMaxBasis = 64;          // restart length m <= kMaxBasis - 1
struct GmresState {
    long long jdone;    // Arnoldi steps completed in the current cycle
    int cycle_end;      // the current cycle ended (convergence, m steps, maxit)
    int converged;
    int skip;           // done || cycle_end: K1 launches of the cycle exit early
};
struct GmresArgs {
    VecArgs a;
    double* V;          // (m+1) basis slices, V_i at V + i * ldv (own rows)
    int64_t ldv;
    int mres;           // m
    double* H;          // (m+1) x m, row-major H[i * m + j]
    double* cs;
    double* sn;
    double* g;          // m+1
    double* hx;         // P x kMaxBasis: partial dots, gathered in place
    GmresState* gs;
    double* part;       // gridDim.x x kMaxBasis CTA partials
    unsigned* ticket;
};
int launch_gm_init(const GmresArgs& g, double tol, long long maxit, long long hist_cap, cudaStream_t st);
int launch_gm_start(const GmresArgs& g, cudaStream_t st);
int launch_gm_dots(const GmresArgs& g, int j, cudaStream_t st);
int launch_gm_orth(const GmresArgs& g, int j, int pass, cudaStream_t st);
int launch_gm_step_end(const GmresArgs& g, int j, long long k, cudaStream_t st);
int launch_gm_vfull(const GmresArgs& g, cudaStream_t st);
int launch_gm_cycle_end(const GmresArgs& g, long long k_enqueued, cudaStream_t st);
// one restart cycle as one persistent cooperative kernel (ks_gmres_persist.cu; P = 1,
// or P > 1 with the fused exchange: g.a from vargs(true), exchange s has epoch ebase + s)
int launch_gm_cycle_persist(const GmresArgs& g, const double* A, int64_t lda, int64_t ncols, double* bpart,
                            unsigned* bar, int grid, unsigned long long ebase, cudaStream_t st);
// epochs one solve of GMRES(restart) with maxit steps may use
inline unsigned long long gm_epochs(long long maxit, int restart) {
    return (unsigned long long)(maxit / restart + 2) * (3ull + 4ull * (unsigned long long)restart) + 4ull;
}
int gm_persist_grid(int num_sms, int64_t m);

// BiCG (NEXT-3)
int launch_bicg_init(const VecArgs& a, double tol, long long maxit, long long hist_cap,
                     unsigned long long ebase, cudaStream_t st);
int launch_bicg_update(const VecArgs& a, long long k, cudaStream_t st);
int launch_bicg_direction(const VecArgs& a, long long k, cudaStream_t st);

// Persistent cooperative whole-iteration kernels (ks_persist.cu, NEXT-2); the
// FP32 instantiation is the NEXT-4 path.
// rows/unroll: the GEMV tile shape (0, 0 = default R=2, U=4; (4,2) and (4,4) selectable).
template <class T>
int persist_grid(int bicgstab, int num_sms, int64_t mmax, int rows, int unroll);
template <class T>
int launch_persist(int bicgstab, const VecArgsT<T>& a, const T* A, int64_t lda, int64_t ncols,
                   T* bpart, unsigned* bar, long long k0, long long k1, int grid, int rows, int unroll,
                   cudaStream_t st, bool bar_zeroed = false);

// Small-n kernels (ks_small.cu, NEXT-2): full-length vectors in every CTA's shared
// memory, 1 (CG) / 2 (BiCGSTAB) grid barriers per iteration.  kind: 0 = CG, 1 =
// BiCGSTAB (P = 1), 2 = CG, 3 = BiCGSTAB over P > 1 GPUs with the fused exchange
// (allgather-only: one / two exchanges and barriers per iteration; a = vargs(true)).  small_grid (rows =
// this rank's rows) returns 0 when the vectors do not fit in shared memory.
template <class T>
int small_grid(int kind, int num_sms, int64_t rows, int64_t ncols);
template <class T>
int launch_small(int kind, const VecArgsT<T>& a, const T* A, int64_t lda, int64_t ncols, T* bpart,
                 unsigned* bar, long long k0, long long k1, int grid, cudaStream_t st, bool bar_zeroed = false);

// Tiny kernels (ks_tiny.cu, NEXT-2): FP64, n <= 1024: A resident in registers, full
// vectors replicated in registers, GEMV outputs exchanged through an LL-format global
// buffer (ll: 4 * ld uint64 words, zeroed once).  The whole solve
// in one launch (they always finish the solve).  tiny_grid returns 0 when not
// applicable.
// P > 1 (fused exchange): the LL words go over NVLink into every rank's buffer (llp,
// a region of the exchange allocation), x0f = the full x0 or NULL.  m = this rank's rows.
int tiny_grid(int bicgstab, int num_sms, int64_t n, int64_t m, int64_t ld);
constexpr int kMaxEmuRanks = 8;     // ranks of one emulated launch (kernel-parameter budget)
// Ranks sharing one GPU: every rank's persistent CG / BiCGSTAB kernel (FP64) as one
// cooperative launch of P * g CTAs (rank h = block / g, arguments a[h], A[h], bpart[h],
// bar[h]); persist_emu_grid = the per-rank CTA count for num_sms / P SMs, 0 = n/a.
int persist_emu_grid(int bicgstab, int num_sms, int P, int64_t mmax, int rows, int unroll);
int launch_persist_emu(int bicgstab, const VecArgs* const* a, const double* const* A, int64_t lda, int64_t ncols,
                       double* const* bpart, unsigned* const* bar, long long k0, long long k1, int P, int g,
                       int rows, int unroll, cudaStream_t st);
// the emulated-rank tiny launch of `blocks` CTAs is co-resident on one GPU
bool tiny_emu_fits(int bicgstab, int64_t lda, int blocks, int num_sms);
int launch_tiny(int bicgstab, const VecArgs& a, const double* A, int64_t lda, uint64_t* ll,
                uint64_t* const* llp, const double* x0f, int grid, cudaStream_t st);
// Ranks sharing one GPU: every rank's tiny kernel as one cooperative launch of P * g
// CTAs (rank h = block / g); a[h] / A[h] / ll[h] / llp[h] are rank h's arguments.  The
// lead CTA of each rank also writes the full x into that rank's X.
int launch_tiny_emu(int bicgstab, const VecArgs* const* a, const double* const* A, int64_t lda,
                    uint64_t* const* ll, uint64_t* const* const* llp, int P, int g, cudaStream_t st);

// Multi-RHS CG (ks_multi.cu, SURVEY.md sec.8(f) "multi-RHS"): K <= kMaxRhs independent
// CG recurrences sharing every pass over A (one GPU, FP64).  Per-column state:
struct MultiCol {
    double nb, rho, relres;
    long long iters;
    int status, active, converged, bzero;
    double rho_old, alpha, omega;      // BiCGSTAB
    int half, breakdown;               // BiCGSTAB
};
constexpr int kMaxRhs = 8;
struct MultiState { MultiCol col[kMaxRhs]; };
// P > 1: every rank's multi-RHS exchange regions (fifth to seventh regions of the
// exchange allocation) and epoch flags.
struct MultiPeer {
    double* MR[kMaxRanks];                  // [2 parities][P][kMaxRhs][chunk]: r slices
    double* MV[kMaxRanks];                  // [2 parities][P][kMaxRhs][chunk]: v slices (BiCGSTAB)
    double* MS[kMaxRanks];                  // [2][P][6 kMaxRhs]: rank partial scalars
    double* MX[kMaxRanks];                  // [kMaxRhs][ld]: the gathered x
    unsigned long long* flags[kMaxRanks];
};
struct MultiArgs {
    int nrhs, has_x0;
    int peer;                      // 1: P > 1 with the fused NVLink exchange
    Layout L;
    MultiPeer mp;
    double *MRo, *MVo, *MSo;       // this rank's own regions (read side)
    unsigned long long* flags;     // own [kNumPhases][kMaxRanks]
    unsigned long long ebase;      // epochs: setup ebase, iteration k ebase + k, x gather ebase + maxit + 1
    unsigned long long join_ns;
    int64_t n, m, ld, ldm, row0;   // ldm: stride of the K rows of X, R, Q; ld: of P
    double tol;
    long long maxit;
    double* X;                     // K x ldm: x (own rows)
    double* R;                     // K x ldm: b on entry, then r
    double* Q;                     // K x ldm: A p
    double* Pf;                    // K x ld: p (full length); x0 on entry when has_x0
    double* Sf;                    // BiCGSTAB: K x ld: s (full length, the second GEMM's input)
    double* Rh;                    // BiCGSTAB: K x ldm: rhat
    double* T;                     // BiCGSTAB: K x ldm: t = A s (Q holds v = A p)
    double* hist;                  // K x hist_cap (column k at hist + k * hist_cap), nullable
    int64_t hist_cap;
    MultiState* ms;
    DevState* st;                  // error reporting (grid-barrier timeout)
    double* bpart;                 // gridDim.x x 2K CTA partials
    unsigned* bar;                 // grid-barrier counter (zeroed by the launcher)
};
int multi_k(int nrhs);             // kernel width K for nrhs columns (0: unsupported)
int multi_grid(int K, int num_sms);
int launch_cg_multi(int K, const MultiArgs& M, const double* A, int grid, cudaStream_t st);
// multi-RHS BiCGSTAB (one GPU): K independent BiCGSTAB recurrences (SURVEY.md
// sec.8(c).4 per column) sharing both GEMMs (v = A p, t = A s) of every iteration
int multi_grid_bs(int K, int num_sms);
int launch_bicgstab_multi(int K, const MultiArgs& M, const double* A, int grid, cudaStream_t st);

// NEXT-4 (FP32) support kernels (ks_f32.cu): K1 in FP32, setup/init/finish in
// FP32, conversions at the FP64 ABI boundary, FP32 generators.
int launch_gemv_f32(const GemvParamsT<float>& p, const Scratch& s, int ticket_id, cudaStream_t st);
int launch_setup_r_f32(const VecArgsT<float>& a, cudaStream_t st);           // x0 = 0
int launch_init_f32(const VecArgsT<float>& a, int bicgstab, double tol, long long maxit,
                    long long hist_cap, unsigned long long ebase, cudaStream_t st);
int launch_finish_f32(const VecArgsT<float>& a, int bicgstab, cudaStream_t st);
int launch_pack_x_f32(const VecArgsT<float>& a, cudaStream_t st);
int launch_true_res_final_f32(const VecArgsT<float>& a, cudaStream_t st);
int launch_d2f(const double* src, float* dst, int64_t n, cudaStream_t st);
int launch_f2d(const float* src, double* dst, int64_t n, cudaStream_t st);
int launch_rows_d2f(const double* src, int64_t lds, float* dst, int64_t ldd, int64_t rows,
                    int64_t cols, cudaStream_t st);
int launch_gen_spd_f32(float* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                       const double* table_dev, cudaStream_t st);
int launch_gen_dd_f32(float* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                      int kd, cudaStream_t st);

}  // namespace ks

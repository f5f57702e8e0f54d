// NEXT-2, third stage: the register-resident whole-solve
// kernels for C1-sized systems (one GPU, FP64, n <= 1024 -- the matrix fits in
// the register files of the SMs: 8 MiB at n = 1024 = 56 KiB per SM of 256 KiB).
//
// Where the small-n kernels (ks_small.cu) re-read A from L2 every GEMV and pay a
// global arrival counter (one atomic per CTA, a fence, a spin) per reduction,
// here:
//   * each CTA owns a contiguous block of <= kRM rows of A and keeps it in
//     REGISTERS for the whole solve (thread t holds its columns of those rows,
//     loaded once per launch): the GEMV reads no memory at all;
//   * every CTA holds the full-length vectors x, r, p (BiCGSTAB: also rhat, v, s)
//     REPLICATED in registers, in one fixed column-ownership layout (thread t
//     owns columns 2t + 512u + {0, 1}); every O(n) step of the recurrence and every
//     full-length dot runs redundantly in every CTA in one fixed order, so all
//     CTAs hold bitwise-identical vectors and take identical decisions;
//   * the only grid-wide step is the exchange of the GEMV output (q = A p; v and
//     t for BiCGSTAB): each CTA stores its rows into a global slot in the LL
//     ("low-latency") format -- every 8-byte word carries 32 bits of the value
//     and a 32-bit epoch, written with single-copy-atomic 8-byte stores -- and
//     every thread polls exactly the words it needs until both halves carry the
//     exchange's epoch.  No fence, no atomic, no barrier: one store propagation
//     plus one L2 round trip per exchange.
// Epochs: exchange "which" (CG 0; BiCGSTAB 0 = v, 1 = t) of iteration k carries
// 2 (ebase + k) + which; the solves of a context advance ebase by maxit + 2, so
// the epochs of one LL buffer only ever grow and a stale word never matches.
// Slots are double-buffered (CG: parity of k; BiCGSTAB: slot 0 = v, slot 1 = t):
// a CTA overwrites a slot only after it has read every CTA's previous use of the
// other slot, which every CTA wrote only after reading this one.
//
// Same recurrences as every other path (SURVEY.md sec.8(c).3 / .4, rows A1-A5,
// B1-B8); the kernels make every decision in-kernel (including the test of the
// last BiCGSTAB step) and always leave st->done = 1, so they are used only when
// one launch runs the whole solve (the default poll batch).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>

#include "ks_device.cuh"
#include "ks_common.cuh"
#include "ks_internal.h"
#include "ks_tma.cuh"

namespace ks {

namespace {

constexpr int kTT = 256;            // threads per CTA
constexpr int kTW = kTT / 32;
constexpr int kRM = 8;              // max rows of A per CTA (shared memory: kRM * ld * 8 B)

__device__ __forceinline__ void ll_store(uint64_t* slot, double v, uint32_t flag) {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const uint64_t lo = (bits & 0xffffffffull) | ((uint64_t)flag << 32);
    const uint64_t hi = (bits >> 32) | ((uint64_t)flag << 32);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(lo), "l"(hi) : "memory");
}
// system scope: the LL words of the P > 1 variant are stored over NVLink into every
// rank's buffer (each 8-byte word still single-copy atomic)
__device__ __forceinline__ void ll_store_sys(uint64_t* slot, double v, uint32_t flag) {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const uint64_t lo = (bits & 0xffffffffull) | ((uint64_t)flag << 32);
    const uint64_t hi = (bits >> 32) | ((uint64_t)flag << 32);
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ void ll_load(const uint64_t* slot, uint64_t& lo, uint64_t& hi) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(slot) : "memory");
}
__device__ __forceinline__ double ll_value(uint64_t lo, uint64_t hi) {
    return __longlong_as_double((long long)(((hi & 0xffffffffull) << 32) | (lo & 0xffffffffull)));
}

__device__ __forceinline__ void ll_load2(const uint64_t* slot, uint64_t (&w)[4]) {
    asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(slot) : "memory");
}
__device__ __forceinline__ void ll_load2_sys(const uint64_t* slot, uint64_t (&w)[4]) {
    asm volatile("ld.relaxed.sys.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(slot) : "memory");
}

// Reads the V values of this thread's columns (2t + 512u + {0, 1}) from an LL slot,
// spinning until every word carries `flag`.  The two entries of a column pair are
// 32 contiguous bytes: one 256-bit load (LDG.256) per pair and poll round, each of
// its four 8-byte words checked on its own.  Columns >= n read as 0.  Bounded:
// returns false after kWaitTimeoutNs (a bug, never a peer: all CTAs are resident).
template <int V>
__device__ __forceinline__ bool ll_gather(const uint64_t* slot, int n, uint32_t flag, double (&out)[V],
                                          unsigned backoff_ns, int wide) {
    constexpr int U = V / 2;
    bool have[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = 2 * threadIdx.x + 512 * u;
        have[u] = j >= n;
        out[2 * u] = out[2 * u + 1] = 0.0;
    }
    unsigned long long t0 = 0;
    for (int spin = 0;; ++spin) {
        bool all = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (have[u]) continue;
            const int j = 2 * threadIdx.x + 512 * u;
            uint64_t w[4];
            if (wide == 2) {
                ll_load2_sys(slot + 2 * (int64_t)j, w);
            } else if (wide) {
                ll_load2(slot + 2 * (int64_t)j, w);
            } else {
                ll_load(slot + 2 * (int64_t)j, w[0], w[1]);
                ll_load(slot + 2 * (int64_t)j + 2, w[2], w[3]);
            }
            const bool ok0 = (uint32_t)(w[0] >> 32) == flag && (uint32_t)(w[1] >> 32) == flag;
            const bool ok1 = j + 1 >= n || ((uint32_t)(w[2] >> 32) == flag && (uint32_t)(w[3] >> 32) == flag);
            if (ok0 && ok1) {
                out[2 * u] = ll_value(w[0], w[1]);
                if (j + 1 < n) out[2 * u + 1] = ll_value(w[2], w[3]);
                have[u] = true;
            } else {
                all = false;
            }
        }
        if (all) return true;
        if (backoff_ns) __nanosleep(backoff_ns);     // fewer polls in flight while waiting
        if ((spin & 255) == 255) {
            if (t0 == 0) t0 = globaltimer_ns();
            else if (globaltimer_ns() - t0 > kWaitTimeoutNs) return false;
        }
    }
}

// Exchange, mode 1 (KS_TINY_XCHG=1, tuning): plain values + one ready flag per CTA.
// Slot layout: lda doubles of data, then one 64-bit flag per CTA.  Writers: value
// stores, __threadfence, barrier, one flag store; readers: warp 0 polls the flags
// (acquire), barrier, every thread reads its values through L2.
__device__ __forceinline__ void fx_put(uint64_t* slot, int64_t lda, int rb, int R, double v, uint64_t flag) {
    double* data = reinterpret_cast<double*>(slot);
    if (threadIdx.x < R) {
        __stcg(data + rb + threadIdx.x, v);
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* f = reinterpret_cast<unsigned long long*>(slot + lda) + blockIdx.x;
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(f), "l"((unsigned long long)flag) : "memory");
    }
}
template <int V>
__device__ __forceinline__ bool fx_get(const uint64_t* slot, int64_t lda, int n, uint64_t flag, double (&out)[V]) {
    __shared__ int s_ok;
    if (threadIdx.x < 32) {
        const unsigned long long* f = reinterpret_cast<const unsigned long long*>(slot + lda);
        bool ok = true;
        const unsigned long long t0 = globaltimer_ns();
        for (int j = threadIdx.x; j < (int)gridDim.x && ok; j += 32) {
            for (;;) {
                unsigned long long v;
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f + j) : "memory");
                if (v == flag) break;
                if (globaltimer_ns() - t0 > kWaitTimeoutNs) { ok = false; break; }
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        if (threadIdx.x == 0) s_ok = ok;
    }
    __syncthreads();
    const double* data = reinterpret_cast<const double*>(slot);
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int j = 2 * threadIdx.x + 512 * (v >> 1) + (v & 1);
        out[v] = j < n ? __ldcg(data + j) : 0.0;
    }
    return s_ok != 0;
}

// Block sum of K values (fixed tree; every thread gets the same bits): butterfly in
// each warp, warp sums through shared memory, each thread adds the kTW warp sums in
// warp order.  ONE __syncthreads: `red` holds two buffers used alternately (a thread
// rewrites buffer b only after the barrier of the call in between, which every
// thread reaches after reading b), `par` toggles per call.
template <int K>
__device__ __forceinline__ void tsum(double (&v)[K], double* red, int& par) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    static_assert(K <= 2, "red holds two buffers of 2 * kTW");
    double* rb = red + par * (2 * kTW);     // fixed stride: calls of different K alternate safely
    par ^= 1;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) rb[k * kTW + w] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double t = 0.0;
#pragma unroll
        for (int ww = 0; ww < kTW; ++ww) t += rb[k * kTW + ww];
        v[k] = t;
    }
}

// Warp sums of kRM = 8 per-thread row partials in 9 shuffles (transpose reduction):
// three halving exchanges (16, 8, 4) leave lane l one row, (l >> 2) & 7 in bit-reversed
// order below, then two butterfly steps (2, 1).  Returns the row sum and its row.
__device__ __forceinline__ double warp_rows8(double (&a)[kRM], int& row) {
    const int lane = threadIdx.x & 31;
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    double v4[4], v2[2], v1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = b4 ? a[i] : a[i + 4];
        const double keep = b4 ? a[i + 4] : a[i];
        v4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b3 ? v4[i] : v4[i + 2];
        const double keep = b3 ? v4[i + 2] : v4[i];
        v2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
        const double send = b2 ? v2[0] : v2[1];
        const double keep = b2 ? v2[1] : v2[0];
        v1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
    row = (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
    return v1;
}

// Loads this thread's slice of rows [rb, rb + R) of A into registers: a[i][v] =
// A[rb + i][col_of(v)] (zero for i >= R or columns >= ld), once per launch.
template <int V>
__device__ __forceinline__ void load_rows_reg(const double* A, int64_t lda, int rb, int R, double (&a)[kRM][V]) {
#pragma unroll
    for (int i = 0; i < kRM; ++i) {
#pragma unroll
        for (int u = 0; u < V / 2; ++u) {
            double2 v2 = make_double2(0.0, 0.0);
            if (i < R) v2 = __ldg(reinterpret_cast<const double2*>(A + (int64_t)(rb + i) * lda + 2 * threadIdx.x + 512 * u));
            a[i][2 * u] = v2.x;
            a[i][2 * u + 1] = v2.y;
        }
    }
}

// GEMV rows [0, R) of this CTA's block, held in registers (a), against the
// register-resident full-length x (this thread's V columns); thread t < R returns
// row t's sum.  Per-thread row partials -> transpose warp reduction -> warp sums in
// warp order.  No shared-memory traffic for A.
template <int V>
__device__ __forceinline__ double gemv_rows(const double (&a)[kRM][V], int R, const double (&x)[V],
                                            double* wred) {
    double acc[kRM];
#pragma unroll
    for (int i = 0; i < kRM; ++i) {
        acc[i] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) acc[i] = fma(a[i][v], x[v], acc[i]);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int row;
    const double s = warp_rows8(acc, row);
    if ((lane & 3) == 0) wred[row * kTW + w] = s;
    __syncthreads();
    double q = 0.0;
    if (threadIdx.x < R) {
#pragma unroll
        for (int ww = 0; ww < kTW; ++ww) q += wred[threadIdx.x * kTW + ww];
    }
    return q;
}

// gemv_rows plus one CTA-wide sum riding on the same barrier: `side` (per-thread
// partial) -> warp butterfly -> warp sums added in warp order (the tsum tree), so the
// result is the same in every thread and every CTA.  (BiCGSTAB: ||s||^2 with t = A s.)
template <int V>
__device__ __forceinline__ double gemv_rows_side(const double (&a)[kRM][V], int R, const double (&x)[V],
                                                 double* wred, double side, double& side_sum) {
    double acc[kRM];
#pragma unroll
    for (int i = 0; i < kRM; ++i) {
        acc[i] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) acc[i] = fma(a[i][v], x[v], acc[i]);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) side += __shfl_xor_sync(0xffffffffu, side, o);
    int row;
    const double s = warp_rows8(acc, row);
    if ((lane & 3) == 0) wred[row * kTW + w] = s;
    if (lane == 0) wred[kRM * kTW + w] = side;
    __syncthreads();
    double q = 0.0;
    if (threadIdx.x < R) {
#pragma unroll
        for (int ww = 0; ww < kTW; ++ww) q += wred[threadIdx.x * kTW + ww];
    }
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < kTW; ++ww) t += wred[kRM * kTW + ww];
    side_sum = t;
    return q;
}

struct TinyArgs {
    VecArgs a;
    const double* A;
    int64_t lda;
    uint64_t* ll;        // 2 slots x ld entries x 2 words (LL format), this rank's
    uint64_t* llp[kMaxRanks];   // P > 1: every rank's LL buffer (exchange allocation)
    const double* x0f;   // P > 1: the full x0 (NULL: zero start)
    // debug (KS_TINY_TRACE=k): thread 0 of every CTA stamps %clock64 at the phase
    // boundaries of CG iteration k (kTrace stamps per CTA) and %globaltimer once
    unsigned long long* trace;
    long long trace_k;
    unsigned backoff;    // ns of __nanosleep after an unsuccessful LL poll round (0: spin)
    int wide;            // 1: one 256-bit load per column pair and poll round (0: two 128-bit)
    int xfull;           // 1: the lead CTA also writes the full x into the rank's X (emulated ranks)
};
// Ranks sharing one GPU (ks_create_on): all ranks' CTAs in ONE cooperative launch --
// CTA b serves rank b / g as its block b % g -- so the CTAs that wait on each other's
// LL words are co-resident by construction (separate launches would not be).
constexpr int kMaxEmu = kMaxEmuRanks;
struct TinyEmuArgs {
    TinyArgs t[kMaxEmu];
    int P, g;
};
constexpr int kTrace = 8;
__device__ __forceinline__ void stamp(const TinyArgs& T, long long k, int i) {
    if (T.trace && k == T.trace_k && threadIdx.x == 0) {
        long long c;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
        T.trace[blockIdx.x * kTrace + i] = (unsigned long long)c;
        if (i == 0) T.trace[gridDim.x * kTrace + blockIdx.x] = globaltimer_ns();
    }
}

// This CTA's rows [rb, rb + R) of the rank's m rows: balanced contiguous blocks over
// the rank's vg CTAs (vb = this CTA's index among them).
__device__ __forceinline__ void my_rows(int n, int& rb, int& R, int vb, int vg) {
    const int q = n / vg, rem = n % vg, b = vb;
    rb = b * q + min(b, rem);
    R = q + (b < rem ? 1 : 0);
}

__device__ __forceinline__ int col_of(int v) { return 2 * threadIdx.x + 512 * (v >> 1) + (v & 1); }

// Publishes this CTA's rows (thread t < R: global row grow = row0 + rb + t) of the GEMV
// output into slot `off` (words) of every rank's LL buffer (P = 1: the own buffer).
__device__ __forceinline__ void ll_publish(const TinyArgs& T, int64_t off, int64_t grow, double v, uint32_t flag) {
    const int P = T.a.L.P;
    if (P == 1) {
        ll_store(T.ll + off + 2 * grow, v, flag);
    } else {
        for (int g = 0; g < P; ++g) ll_store_sys(T.llp[g] + off + 2 * grow, v, flag);
    }
}

// ------------------------------------------------------------------ CG (A1-A5)
template <int V, int XM>
__device__ __forceinline__ void cg_tiny_body(const TinyArgs& T, int vb, int vg) {
    __shared__ double wred[kRM * kTW];
    __shared__ double red[2 * 2 * kTW];
    int par = 0;
    const VecArgs& a = T.a;
    DevState* st = a.st;
    const int n = (int)a.L.n;
    if (is_done(st)) {                               // 0-iteration exit: x = x0 = 0
        if (T.xfull && vb == 0)
            for (int j = threadIdx.x; j < n; j += kTT) a.X[j] = 0.0;
        return;
    }
    const int P = a.L.P, m = (int)rows_of(a.L);
    const int64_t row0 = a.L.row0[a.L.rank];
    const int wide = P > 1 ? 2 : T.wide;           // P > 1: system-scope polls of the LL words
    int rb, R;
    my_rows(m, rb, R, vb, vg);
    double Ar[kRM][V];
    load_rows_reg<V>(T.A, T.lda, rb, R, Ar);
    double x[V], r[V], p[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int j = col_of(v);
        const bool in = j < n;
        x[v] = !in ? 0.0 : P == 1 ? a.x_loc[j] : (T.x0f ? T.x0f[j] : 0.0);   // x0 (replicated)
        r[v] = in ? a.G_r[gidx(a.L, j)] : 0.0;  // r0 (gather buffer, parity 0: every rank has all of it)
        p[v] = in ? a.p_full[j] : 0.0;          // p0 = r0
    }
    double rho = st->rho[0];
    const double nb = st->nb, tol = st->tol;
    const long long maxit = st->maxit;
    const unsigned long long eb = st->ebase;
    const bool lead0 = vb == 0;
    long long k = 1;
    int status = KS_EMAXIT, conv = 0;
    long long iters = maxit;
    for (; k <= maxit; ++k) {
        stamp(T, k, 0);
        // A1: q rows = A p; LL exchange (the grid-wide step)
        const double qrow = gemv_rows<V>(Ar, R, p, wred);
        stamp(T, k, 1);
        const uint32_t flag = (uint32_t)(2ull * (eb + (unsigned long long)k));
        uint64_t* slot = T.ll + (int64_t)(k & 1) * 2 * T.lda;
        double q[V];
        bool got;
        if (XM == 0) {
            jitter_at(T.a.jitter, 6u);
            if (threadIdx.x < R) ll_publish(T, (int64_t)(k & 1) * 2 * T.lda, row0 + rb + threadIdx.x, qrow, flag);
            jitter_at(T.a.jitter, 7u);
            got = ll_gather<V>(slot, n, flag, q, T.backoff, wide);
        } else {
            fx_put(slot, T.lda, rb, R, qrow, flag);
            got = fx_get<V>(slot, T.lda, n, flag, q);
        }
        if (!got) {
            if (lead0 && threadIdx.x == 0) { st->peer_timeout = 1; st->status = KS_ECUDA; st->done = 1; }
            return;
        }
        stamp(T, k, 2);
        // A2: sigma = <p, q> (full length, every CTA)
        double s1[1] = {0.0};
#pragma unroll
        for (int v = 0; v < V; ++v) s1[0] = fma(p[v], q[v], s1[0]);
        tsum<1>(s1, red, par);
        const double sigma = s1[0];
        stamp(T, k, 3);
        if (!(sigma > 0.0)) { status = KS_ENOTSPD; iters = k - 1; break; }   // Q9: x unchanged
        const double alpha = rho / sigma;
        // A3: x += alpha p; r -= alpha q; rho' = <r, r>
        double s2[1] = {0.0};
#pragma unroll
        for (int v = 0; v < V; ++v) {
            x[v] = fma(alpha, p[v], x[v]);
            r[v] = fma(-alpha, q[v], r[v]);
            s2[0] = fma(r[v], r[v], s2[0]);
        }
        tsum<1>(s2, red, par);
        const double rho1 = s2[0];
        stamp(T, k, 4);
        const double rel = sqrt(rho1) / nb;
        if (lead0 && threadIdx.x == 0) {
            put_hist(st, a.hist, k - 1, rel);
            st->relres = rel;
        }
        if (rel <= tol) { status = KS_OK; conv = 1; iters = k; break; }
        // A5: p = r + beta p
        const double beta = rho1 / rho;
#pragma unroll
        for (int v = 0; v < V; ++v) p[v] = fma(beta, p[v], r[v]);
        rho = rho1;
        stamp(T, k, 5);
    }
    if (lead0) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int j = col_of(v);
            if (j >= row0 && j < row0 + m) a.x_loc[j - row0] = x[v];      // own rows
            if (j < n) a.p_full[j] = p[v];
            if (P == 1 && j < n) a.G_r[j] = r[v];
            if (T.xfull && j < n) a.X[j] = x[v];                           // emulated ranks: full x
        }
        if (threadIdx.x == 0) {
            st->iters = iters; st->status = status; st->converged = conv;
            st->rho[iters & 3] = rho;
            st->done = 1;
        }
    }
}

// ---------------------------------------------------------- BiCGSTAB (B1-B8)
template <int V, int XM>
__device__ __forceinline__ void bs_tiny_body(const TinyArgs& T, int vb, int vg) {
    __shared__ double wred[(kRM + 1) * kTW];
    __shared__ double red[2 * 2 * kTW];
    int par = 0;
    const VecArgs& a = T.a;
    DevState* st = a.st;
    const int n = (int)a.L.n;
    if (is_done(st)) {                               // 0-iteration exit: x = x0 = 0
        if (T.xfull && vb == 0)
            for (int j = threadIdx.x; j < n; j += kTT) a.X[j] = 0.0;
        return;
    }
    const int P = a.L.P, m = (int)rows_of(a.L);
    const int64_t row0 = a.L.row0[a.L.rank];
    const int wide = P > 1 ? 2 : T.wide;           // P > 1: system-scope polls of the LL words
    int rb, R;
    my_rows(m, rb, R, vb, vg);
    double Ar[kRM][V];
    load_rows_reg<V>(T.A, T.lda, rb, R, Ar);
    double x[V], r[V], p[V], v_[V], rh[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int j = col_of(v);
        const bool in = j < n;
        x[v] = !in ? 0.0 : P == 1 ? a.x_loc[j] : (T.x0f ? T.x0f[j] : 0.0);
        r[v] = in ? a.G_r[gidx(a.L, j)] : 0.0;  // r0
        rh[v] = r[v];                           // rhat = r0 (Q7)
        p[v] = 0.0;                           // v = p = 0 (Q8)
        v_[v] = 0.0;
    }
    const double nb = st->nb, tol = st->tol;
    const long long maxit = st->maxit;
    const unsigned long long eb = st->ebase;
    const bool lead0 = vb == 0;
    double rho = slot_sum(a.L, a.G_r, 0);     // rho_1 = <rhat, r0>
    double rho_old = 1.0, alpha = 1.0, omega = 1.0;
    int status = KS_EMAXIT, conv = 0, brk = 0, half = 0;
    long long iters = maxit;
    for (long long i = 1; i <= maxit; ++i) {
        if (rho == 0.0 || !isfinite(rho)) { status = KS_EBREAKDOWN; brk = 1; iters = i - 1; break; }
        // B1: p = r + beta (p - omega v)   (i = 1: p = r exactly)
        const double beta = (rho / rho_old) * (alpha / omega);
#pragma unroll
        for (int v = 0; v < V; ++v) p[v] = i == 1 ? r[v] : fma(beta, fma(-omega, v_[v], p[v]), r[v]);
        // B2/B3: v = A p, exchange (slot 0)
        const uint32_t fv = (uint32_t)(2ull * (eb + (unsigned long long)i));
        double vrow = gemv_rows<V>(Ar, R, p, wred);
        bool got;
        if (XM == 0) {
            jitter_at(T.a.jitter, 6u);
            if (threadIdx.x < R) ll_publish(T, 0, row0 + rb + threadIdx.x, vrow, fv);
            jitter_at(T.a.jitter, 7u);
            got = ll_gather<V>(T.ll, n, fv, v_, T.backoff, wide);
        } else {
            fx_put(T.ll, T.lda, rb, R, vrow, fv);
            got = fx_get<V>(T.ll, T.lda, n, fv, v_);
        }
        if (!got) {
            if (lead0 && threadIdx.x == 0) { st->peer_timeout = 1; st->status = KS_ECUDA; st->done = 1; }
            return;
        }
        // B4: gamma = <rhat, v>; alpha; s = r - alpha v; ||s||^2
        double g1[1] = {0.0};
#pragma unroll
        for (int v = 0; v < V; ++v) g1[0] = fma(rh[v], v_[v], g1[0]);
        tsum<1>(g1, red, par);
        const double gam = g1[0];
        if (gam == 0.0 || !isfinite(gam)) { status = KS_EBREAKDOWN; brk = 1; iters = i - 1; break; }
        alpha = rho / gam;
        double s[V];
        double ss = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            s[v] = fma(-alpha, v_[v], r[v]);
            ss = fma(s[v], s[v], ss);
        }
        // B5 + B6: t rows = A s computed alongside ||s||^2 (one barrier for both); t is
        // published only when the half-step test does not end the solve
        double sst;
        const double trow = gemv_rows_side<V>(Ar, R, s, wred, ss, sst);
        const double srel = sqrt(sst) / nb;
        if (srel <= tol) {                                     // B5: half-step exit
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = fma(alpha, p[v], x[v]);
            if (lead0 && threadIdx.x == 0) { put_hist(st, a.hist, i - 1, srel); st->relres = srel; }
            status = KS_OK; conv = 1; half = 1; iters = i;
            break;
        }
        // B6: t = A s, exchange (slot 1); <t, s>, <t, t>
        const uint32_t ft = fv + 1u;

        uint64_t* slot1 = T.ll + 2 * T.lda;
        double t[V];
        if (XM == 0) {
            jitter_at(T.a.jitter, 6u);
            if (threadIdx.x < R) ll_publish(T, 2 * T.lda, row0 + rb + threadIdx.x, trow, ft);
            jitter_at(T.a.jitter, 7u);
            got = ll_gather<V>(slot1, n, ft, t, T.backoff, wide);
        } else {
            fx_put(slot1, T.lda, rb, R, trow, ft);
            got = fx_get<V>(slot1, T.lda, n, ft, t);
        }
        if (!got) {
            if (lead0 && threadIdx.x == 0) { st->peer_timeout = 1; st->status = KS_ECUDA; st->done = 1; }
            return;
        }
        double d2[2] = {0.0, 0.0};
#pragma unroll
        for (int v = 0; v < V; ++v) {
            d2[0] = fma(t[v], s[v], d2[0]);
            d2[1] = fma(t[v], t[v], d2[1]);
        }
        tsum<2>(d2, red, par);
        const double tt = d2[1];
        if (tt == 0.0 || !isfinite(tt)) { status = KS_EBREAKDOWN; brk = 1; iters = i - 1; break; }
        const double om = d2[0] / tt;
        if (om == 0.0 || !isfinite(om)) { status = KS_EBREAKDOWN; brk = 1; iters = i - 1; break; }
        // B7: x = (x + alpha p) + omega s; r = s - omega t; <rhat, r>, <r, r>
        double d3[2] = {0.0, 0.0};
#pragma unroll
        for (int v = 0; v < V; ++v) {
            x[v] = fma(om, s[v], fma(alpha, p[v], x[v]));
            r[v] = fma(-om, t[v], s[v]);
            d3[0] = fma(rh[v], r[v], d3[0]);
            d3[1] = fma(r[v], r[v], d3[1]);
        }
        tsum<2>(d3, red, par);
        omega = om;
        rho_old = rho;
        rho = d3[0];
        // B8: history, convergence test
        const double rel = sqrt(d3[1]) / nb;
        if (lead0 && threadIdx.x == 0) { put_hist(st, a.hist, i - 1, rel); st->relres = rel; }
        if (rel <= tol) { status = KS_OK; conv = 1; iters = i; break; }
    }
    if (lead0) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int j = col_of(v);
            if (j >= row0 && j < row0 + m) a.x_loc[j - row0] = x[v];      // own rows
            if (j < n) { a.p_full[j] = p[v]; a.v_full[j] = v_[v]; }
            if (P == 1 && j < n) a.G_r[j] = r[v];
            if (T.xfull && j < n) a.X[j] = x[v];                           // emulated ranks: full x
        }
        if (threadIdx.x == 0) {
            st->iters = iters; st->status = status; st->converged = conv; st->breakdown = brk;
            st->half = half; st->half_iter = half ? iters : 0;
            st->alpha[iters & 3] = alpha; st->omega[iters & 3] = omega; st->rho[iters & 3] = rho;
            st->done = 1;
        }
    }
}

template <int V, int XM>
__global__ void __launch_bounds__(kTT, 1) k_cg_tiny(TinyArgs T) {
    cg_tiny_body<V, XM>(T, (int)blockIdx.x, (int)gridDim.x);
}
template <int V, int XM>
__global__ void __launch_bounds__(kTT, 1) k_bs_tiny(TinyArgs T) {
    bs_tiny_body<V, XM>(T, (int)blockIdx.x, (int)gridDim.x);
}
template <int V>
__global__ void __launch_bounds__(kTT, 1) k_cg_tiny_emu(const __grid_constant__ TinyEmuArgs E) {
    const int rk = (int)blockIdx.x / E.g;
    cg_tiny_body<V, 0>(E.t[rk], (int)blockIdx.x - rk * E.g, E.g);
}
template <int V>
__global__ void __launch_bounds__(kTT, 1) k_bs_tiny_emu(const __grid_constant__ TinyEmuArgs E) {
    const int rk = (int)blockIdx.x / E.g;
    bs_tiny_body<V, 0>(E.t[rk], (int)blockIdx.x - rk * E.g, E.g);
}

template <int V, int XM>
const void* kern(int bicgstab) {
    return bicgstab ? (const void*)k_bs_tiny<V, XM> : (const void*)k_cg_tiny<V, XM>;
}
int xchg_mode() {
    const char* e = std::getenv("KS_TINY_XCHG");   // tuning: 0 = LL (default), 1 = ready flags
    return e && std::atoi(e) == 1 ? 1 : 0;
}
const void* kern_v(int bicgstab, int V, int P = 1) {
    if (xchg_mode() == 1 && P == 1) return V == 2 ? kern<2, 1>(bicgstab) : kern<4, 1>(bicgstab);
    return V == 2 ? kern<2, 0>(bicgstab) : kern<4, 0>(bicgstab);
}

}  // namespace

// Grid of the tiny kernels for an n x n FP64 system on one GPU (ld = padded row
// length), 0 when not applicable: n <= 1024 (the full vectors fit in registers,
// 4 values per thread and vector), every CTA's rows fit in registers (<= kRM),
// one co-resident CTA per SM.
int tiny_grid(int bicgstab, int num_sms, int64_t n, int64_t m, int64_t ld) {
    if (n < 1 || n > 1024 || ld > 1024 || m < 1) return 0;
    const int V = ld <= 512 ? 2 : 4;
    // The fewest CTAs that hold the rows (kRM = 8 per CTA): every CTA polls all n LL
    // words of each exchange, so fewer pollers finish it sooner -- n = 1024: 128 CTAs
    // CG 2.31 / BiCGSTAB 4.68 us per iteration vs 2.80 / 6.58 on all 148 SMs
    // (profiles/r02_tiny_grid_ab.jsonl).
    int g = (int)std::min<int64_t>(num_sms, (m + kRM - 1) / kRM);
    if (const char* tg = std::getenv("KS_TINY_GRID")) {     // tuning override
        const int v = std::atoi(tg);
        if (v >= 1 && v <= num_sms) g = v;
    }
    if (g > m) g = (int)m;
    const int64_t rmax = (m + g - 1) / g;
    if (rmax > kRM) return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern_v(bicgstab, V), kTT, 0) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm >= 1 ? g : 0;
}

int launch_tiny(int bicgstab, const VecArgs& a, const double* A, int64_t lda, uint64_t* ll,
                uint64_t* const* llp, const double* x0f, int grid, cudaStream_t st) {
    TinyArgs T;
    T.a = a;
    T.A = A;
    T.lda = lda;
    T.ll = ll;
    for (int g = 0; g < kMaxRanks; ++g) T.llp[g] = (llp && g < a.L.P) ? llp[g] : nullptr;
    T.x0f = x0f;
    T.trace = nullptr;
    T.trace_k = 0;
    T.backoff = 0;
    if (const char* bo = std::getenv("KS_TINY_BACKOFF")) T.backoff = (unsigned)std::atoi(bo);   // tuning
    T.wide = 1;
    if (const char* wd = std::getenv("KS_TINY_WIDE")) T.wide = std::atoi(wd) != 0;               // tuning
    T.xfull = 0;
    const char* tr = bicgstab ? nullptr : std::getenv("KS_TINY_TRACE");   // debug facility
    if (tr) {
        T.trace_k = std::atoll(tr);
        if (cudaMalloc(&T.trace, (size_t)grid * (kTrace + 1) * sizeof(unsigned long long)) != cudaSuccess)
            T.trace = nullptr;
        else cudaMemsetAsync(T.trace, 0, (size_t)grid * (kTrace + 1) * sizeof(unsigned long long), st);
    }
    void* args[] = {&T};
    const cudaError_t e = cudaLaunchCooperativeKernel(kern_v(bicgstab, lda <= 512 ? 2 : 4, a.L.P), dim3((unsigned)grid),
                                                      dim3(kTT), args, 0, st);
    if (T.trace) {                      // dump: one line per CTA, clock deltas then the start time
        std::vector<unsigned long long> h((size_t)grid * (kTrace + 1));
        cudaMemcpyAsync(h.data(), T.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(T.trace);
        const char* out = std::getenv("KS_TINY_TRACE_OUT");
        if (FILE* f = std::fopen(out ? out : "tiny_trace.txt", "a")) {
            for (int b = 0; b < grid; ++b) {
                std::fprintf(f, "%d %llu", b, h[(size_t)grid * kTrace + b]);
                for (int i = 1; i < 6; ++i)
                    std::fprintf(f, " %lld", (long long)(h[(size_t)b * kTrace + i] - h[(size_t)b * kTrace + i - 1]));
                std::fprintf(f, "\n");
            }
            std::fclose(f);
        }
    }
    return e == cudaSuccess ? 1 : -(int)e;
}

bool tiny_emu_fits(int bicgstab, int64_t lda, int blocks, int num_sms) {
    if (blocks < 1 || lda > 1024) return false;
    const int V = lda <= 512 ? 2 : 4;
    const void* k = bicgstab ? (V == 2 ? (const void*)k_bs_tiny_emu<2> : (const void*)k_bs_tiny_emu<4>)
                             : (V == 2 ? (const void*)k_cg_tiny_emu<2> : (const void*)k_cg_tiny_emu<4>);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kTT, 0) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (int64_t)per_sm * num_sms >= blocks;
}

int launch_tiny_emu(int bicgstab, const VecArgs* const* a, const double* const* A, int64_t lda,
                    uint64_t* const* ll, uint64_t* const* const* llp, int P, int g, cudaStream_t st) {
    if (P < 2 || P > kMaxEmu || g < 1) return -(int)cudaErrorInvalidValue;
    TinyEmuArgs E;
    std::memset(&E, 0, sizeof E);
    for (int h = 0; h < P; ++h) {
        TinyArgs& T = E.t[h];
        T.a = *a[h];
        T.A = A[h];
        T.lda = lda;
        T.ll = ll[h];
        for (int q = 0; q < kMaxRanks; ++q) T.llp[q] = q < P ? llp[h][q] : nullptr;
        T.x0f = nullptr;
        T.trace = nullptr;
        T.trace_k = 0;
        T.backoff = 0;
        T.wide = 2;
        T.xfull = 1;
    }
    E.P = P;
    E.g = g;
    const int V = lda <= 512 ? 2 : 4;
    const void* k = bicgstab ? (V == 2 ? (const void*)k_bs_tiny_emu<2> : (const void*)k_bs_tiny_emu<4>)
                             : (V == 2 ? (const void*)k_cg_tiny_emu<2> : (const void*)k_cg_tiny_emu<4>);
    void* args[] = {&E};
    const cudaError_t e = cudaLaunchCooperativeKernel(k, dim3((unsigned)(P * g)), dim3(kTT), args, 0, st);
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ks

// Multi-RHS CG ("multi-RHS": with K right-hand sides the GEMV
// becomes a skinny GEMM, Q = A P with P n x K).  K independent CG recurrences
// (sec.8(c).3 per column: own alpha, beta, stopping test, NOTSPD exit; DESIGN.md
// reading Q30) share every pass over A, so one HBM stream of A serves K iterations:
// K/4 flop per byte instead of 1/4.  FP64 on the CUDA cores -- B200's FP64 tensor
// path is no faster than the FP64 pipes, and at K <= 8 the GEMM stays HBM-bound.
//
// One persistent cooperative kernel per solve, one CTA per SM, 7 consumer warps +
// 1 TMA producer warp:
//   * A is cut into bands of 28 rows (round-robin over the CTAs) and chunks of
//     128 columns; a stage = the A tile (28 x 128, 28 KiB) + the matching P tile
//     (K x 128), both brought into shared memory by 2-D TMA loads (K = 8: 56 x 64
//     tiles, 8 rows per warp -- see the shape note below)
//     (cp.async.bulk.tensor, tensor maps built on the host) completing on a
//     full-mbarrier; kMS stages in flight; consumers release a stage through an
//     empty-mbarrier (one arrival per warp);
//   * consumer warp w owns rows 4w..4w+3 of the band (shape (4, 128)), lane l the column pairs
//     2l and 64 + 2l of each chunk: 4 x K accumulators per thread, the P pair loaded
//     once per column pair and reused for the 4 rows (shared-memory traffic ~3x the
//     A bytes at K = 8, conflict-free 512-byte rows);
//   * at the end of a band the 32 lanes' partials are summed by a butterfly; lane 0
//     writes q and accumulates sigma_k = <p_k, q_k> over its rows;
//   * the O(n) phases (alpha, x, r, rho', beta, p per column) run between grid
//     barriers as in the single-RHS persistent kernel; every sum is fixed-order.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstdlib>

#include "ks_device.cuh"
#include "ks_common.cuh"
#include "ks_internal.h"
#include "ks_persist.cuh"
#include "ks_tma.cuh"

namespace ks {

namespace {

// GEMM shape: WR rows per consumer warp (band = kMW WR rows), CH columns per chunk
// (CH / 64 column pairs per lane).  (4, 128): 28 x 128 A tiles, the P pair reused for
// 4 rows; (8, 64) and (8, 128): 56-row bands, the P pair reused for 8 rows -- half the
// shared-memory reads of P per FMA.  (8, 128) with 3 stages of 64 KiB is the default
// (1 KiB row segments per TMA box row; best for K = 4 and 8 on the same box).
// pipeline stages of a shape: 4, or 3 when a stage holds 56 KiB of A (8 x 128)
template <int WR, int CH>
struct Stages { static constexpr int value = (WR * CH >= 1024) ? 3 : 4; };
// 7 consumer warps + 1 producer warp = 8 warps, 2 per SM sub-partition: up to 255
// registers per thread (9 warps put 3 on one sub-partition, capping them at 168)
constexpr int kMW = 7;                    // consumer warps
constexpr int kMT = (kMW + 1) * 32;       // + the producer warp
constexpr int kMCT = kMW * 32;            // consumer threads
// MS rows (rank partial scalars, per parity and rank): slot ranges per exchange phase
// of one iteration, disjoint so a fast rank's next phase never overwrites a slot a
// slow rank is still reading (CG: sigma [0, K), rho' [K, 2K); BiCGSTAB: <rhat, v>,
// (<t,s>, <t,t>), (<rhat,r>, <r,r>)).
constexpr int kMsV = 0, kMsS = 2 * kMaxRhs, kMsR = 4 * kMaxRhs, kMsRow = 6 * kMaxRhs;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Sum over the consumer threads of K values (fixed tree), result in every consumer
// thread; the producer warp takes part in the barriers only.
template <int K>
__device__ __forceinline__ void csum(double (&v)[K], double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane == 0 && w < kMW) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[k * kMW + w] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double t = lane < kMW ? red[k * kMW + lane] : 0.0;
        v[k] = warp_sum(t);
    }
}

template <int K, int WR, int CH>
struct MultiSmem {
    static constexpr int kMS = Stages<WR, CH>::value;
    double A[kMS][kMW * WR * CH];
    double P[kMS][K * CH];
    uint64_t full[kMS], empty[kMS];
    double red[2 * K * kMW];
    double wpart[kMW][K];
    double wpart2[kMW][K];
};

// Q = A P (this CTA's bands) and sigma partials <P_k, Q_k> over the CTA's rows in
// band order.  `it` is the pipeline position, identical in producer and consumers.
// Output rows go to out[k * ldm + row]; d1_k = sum over the rows of W[k * ldw + woff + row]
// * out_k (CG: sigma = <p, q>; BiCGSTAB: <rhat, v>, <s, t>), d2_k = <out_k, out_k> when DOT2.
template <int K, int WR, int CH, bool DOT2 = false>
__device__ void gemm_phase(const CUtensorMap* tmA, const CUtensorMap* tmP, const MultiArgs& M,
                           MultiSmem<K, WR, CH>& S, uint32_t& it, double (&sig)[K], double* out = nullptr,
                           const double* W = nullptr, int64_t ldw = 0, int64_t woff = 0, double* d2 = nullptr) {
    if (!out) { out = M.Q; W = M.Pf; ldw = M.ld; woff = M.row0; }
    constexpr int BAND = kMW * WR, NP = CH / 64;
    constexpr int kMS = MultiSmem<K, WR, CH>::kMS;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nbands = (int)((M.m + BAND - 1) / BAND);
    const int nchunks = (int)(M.ld / CH);
#pragma unroll
    for (int k = 0; k < K; ++k) sig[k] = 0.0;
    if (DOT2) {
#pragma unroll
        for (int k = 0; k < K; ++k) d2[k] = 0.0;
    }
    if (w == kMW) {                                        // ---- TMA producer warp
        if (lane == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");   // P written by the generic proxy
            const uint32_t bytes = (uint32_t)(BAND * CH + K * CH) * sizeof(double);
            for (int b = blockIdx.x; b < nbands; b += gridDim.x) {
                for (int c = 0; c < nchunks; ++c, ++it) {
                    const int s = (int)(it % kMS);
                    const uint32_t ph = (it / kMS) & 1u;
                    mbar_wait(&S.empty[s], ph ^ 1u);
                    mbar_expect_tx(&S.full[s], bytes);
                    tma_load_2d(S.A[s], tmA, c * CH, b * BAND, &S.full[s]);
                    tma_load_2d(S.P[s], tmP, c * CH, 0, &S.full[s]);
                }
            }
        } else {
            for (int b = blockIdx.x; b < nbands; b += gridDim.x) it += (uint32_t)nchunks;
        }
        return;
    }
    for (int b = blockIdx.x; b < nbands; b += gridDim.x) {  // ---- consumer warps
        double acc[WR][K];
#pragma unroll
        for (int rr = 0; rr < WR; ++rr)
#pragma unroll
            for (int k = 0; k < K; ++k) acc[rr][k] = 0.0;
        for (int c = 0; c < nchunks; ++c, ++it) {
            const int s = (int)(it % kMS);
            const uint32_t ph = (it / kMS) & 1u;
            mbar_wait(&S.full[s], ph);
            const double* At = S.A[s] + (WR * w) * CH + 2 * lane;
            const double* Pt = S.P[s] + 2 * lane;
            constexpr int UNP = WR >= 8 ? 1 : NP;   // 8 rows x K: one column pair live at a time
#pragma unroll UNP
            for (int u = 0; u < NP; ++u) {
                double2 p[K];
#pragma unroll
                for (int k = 0; k < K; ++k) p[k] = *reinterpret_cast<const double2*>(Pt + k * CH + 64 * u);
#pragma unroll
                for (int rr = 0; rr < WR; ++rr) {
                    const double2 a = *reinterpret_cast<const double2*>(At + rr * CH + 64 * u);
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        acc[rr][k] = fma(a.x, p[k].x, acc[rr][k]);
                        acc[rr][k] = fma(a.y, p[k].y, acc[rr][k]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[s]);
        }
#pragma unroll
        for (int rr = 0; rr < WR; ++rr)
#pragma unroll
            for (int k = 0; k < K; ++k) acc[rr][k] = warp_sum(acc[rr][k]);
        if (lane == 0) {
#pragma unroll
            for (int rr = 0; rr < WR; ++rr) {
                const int64_t row = (int64_t)b * BAND + WR * w + rr;
                if (row < M.m) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        out[k * M.ldm + row] = acc[rr][k];
                        sig[k] = fma(W[k * ldw + woff + row], acc[rr][k], sig[k]);
                        if (DOT2) d2[k] = fma(acc[rr][k], acc[rr][k], d2[k]);
                    }
                }
            }
        }
    }
}

// Per-CTA partial slots: kBSlots * K doubles per CTA.  Phases whose partials are
// written without a grid barrier after the previous phase's totals were read use
// disjoint slots: BiCGSTAB's B4 (||s||^2) -> [K, 2K), B6 (<t,s>, <t,t>) -> [2K, 4K),
// B7 (<rhat,r>, <r,r>) -> [4K, 6K) -- with shared slots a fast CTA's B6 / B7 partials
// could overwrite a slot a slow CTA was still summing (found by KS_OPT_JITTER).
constexpr int kBSlots = 6;
// CTA-order totals of K partial slots (q0 .. q0 + K - 1 of the kBSlots * K per CTA).
template <int K>
__device__ __forceinline__ void totals(const double* bpart, int q0, double (&out)[K], double* red) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double acc = 0.0;
        if (threadIdx.x < kMCT)
            for (int b = threadIdx.x; b < (int)gridDim.x; b += kMCT) acc += __ldcg(bpart + (int64_t)b * kBSlots * K + q0 + k);
        out[k] = acc;
    }
    csum<K>(out, red);
}

// ---- P > 1 (fused NVLink exchange) ------------------------------------------
// Rank all-reduce of NV scalars that every CTA of this rank holds identically
// (CTA-order totals): the lead stores them into slots [q0, q0 + NV) of this rank's
// row of every rank's MS[par] and releases `ph` with `epoch`; every CTA waits for
// all ranks (thread 0 spins, the barrier orders the rest) and sums the P rows in
// rank order.  P == 1: v unchanged.
template <int NV>
__device__ __forceinline__ bool rank_sum(const MultiArgs& M, double (&v)[NV], int par, int q0, int ph,
                                         unsigned long long epoch) {
    if (!M.peer) return true;
    const int P = M.L.P, me = M.L.rank;
    const int64_t row = kMsRow, pst = (int64_t)P * row;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int g = 0; g < P; ++g)
            for (int k = 0; k < NV; ++k) M.mp.MS[g][par * pst + (int64_t)me * row + q0 + k] = v[k];
        unsigned long long* f[kMaxRanks];
        for (int g = 0; g < P; ++g) f[g] = M.mp.flags[g] + ph * kMaxRanks + me;
        jitter_at(*(volatile const unsigned*)&M.st->jitter, 5u);
        publish_flags(f, P, epoch);
    }
    if (threadIdx.x == 0) jitter_at(*(volatile const unsigned*)&M.st->jitter, 3u);
    if (!wait_flags(M.flags + ph * kMaxRanks, P, epoch)) {
        if (threadIdx.x == 0) { M.st->peer_timeout = 1; M.st->status = KS_ENCCL; M.st->done = 1; }
        return false;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = 0.0;
        for (int g = 0; g < P; ++g) t += __ldcg(M.MSo + par * pst + (int64_t)g * row + q0 + k);
        v[k] = t;
    }
    return true;
}
// MR / MV [par][g][k][chunk]: rank g's rows of column k of r / v (parity par)
__device__ __forceinline__ int64_t mr_off(const MultiArgs& M, int par, int g, int k) {
    return (((int64_t)par * M.L.P + g) * kMaxRhs + k) * M.L.chunk;
}
// element j of column k of a full-length vector gathered in MR / MV; o = owner of j
// (advanced monotonically by the caller's grid-stride loop)
__device__ __forceinline__ double gathered(const MultiArgs& M, const double* G, int par, int k, int64_t j, int& o) {
    while (o + 1 < M.L.P && j >= M.L.row0[o + 1]) ++o;
    return __ldcg(G + mr_off(M, par, o, k) + (j - M.L.row0[o]));
}

// End of a P > 1 solve: every rank stores its rows of X into every rank's contiguous
// MX (K x ld), one system fence per CTA, a grid barrier, then CTA 0 releases kPhaseX
// (epoch ebase + maxit + 1) and waits for every rank's.
template <int K, class Smem>
__device__ void gather_x(const MultiArgs& M, Smem& S) {
    (void)S;
    const int tid = threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * kMCT, t0 = (int64_t)blockIdx.x * kMCT + tid;
    if (tid < kMCT)
        for (int64_t i = t0; i < M.m; i += gs)
#pragma unroll
            for (int k = 0; k < K; ++k)
                for (int g = 0; g < M.L.P; ++g) M.mp.MX[g][k * M.ld + M.row0 + i] = M.X[k * M.ldm + i];
    __syncthreads();
    if (tid == 0) __threadfence_system();
    if (!pk::grid_sync(M.bar, M.st)) return;
    if (blockIdx.x == 0) {
        if (tid == 0) {
            unsigned long long* f[kMaxRanks];
            for (int g = 0; g < M.L.P; ++g) f[g] = M.mp.flags[g] + kPhaseX * kMaxRanks + M.L.rank;
            publish_flags(f, M.L.P, M.ebase + (unsigned long long)M.maxit + 1ull);
        }
        if (!wait_flags(M.flags + kPhaseX * kMaxRanks, M.L.P, M.ebase + (unsigned long long)M.maxit + 1ull) &&
            tid == 0) {
            M.st->peer_timeout = 1; M.st->status = KS_ENCCL;
        }
    }
}

template <int K, int WR, int CH>
__global__ void __launch_bounds__(kMT, 1) k_cgm(const __grid_constant__ CUtensorMap tmA,
                                               const __grid_constant__ CUtensorMap tmP, MultiArgs M) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    MultiSmem<K, WR, CH>& S = *reinterpret_cast<MultiSmem<K, WR, CH>*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    MultiState* ms = M.ms;
    DevState* st = M.st;
    const int tid = threadIdx.x;
    const bool cons = tid < kMCT;
    const int64_t gs = (int64_t)gridDim.x * kMCT;
    const int64_t t0 = (int64_t)blockIdx.x * kMCT + tid;
    const int64_t m = M.m;
    const bool peer = M.peer != 0;
    if (tid == 0) {
        for (int s = 0; s < MultiSmem<K, WR, CH>::kMS; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], kMW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == kMW * 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmP) : "memory");
    }
    if (peer && blockIdx.x == 0 && tid == 0) {     // solve-start rendezvous (k_join's protocol)
        unsigned long long* f[kMaxRanks];
        for (int g = 0; g < M.L.P; ++g) f[g] = M.mp.flags[g] + kPhaseJ * kMaxRanks + M.L.rank;
        publish_flags(f, M.L.P, M.ebase);
        const unsigned long long tj = globaltimer_ns();
        for (int g = 0; g < M.L.P; ++g) {
            while (flag_acquire_sys(M.flags + kPhaseJ * kMaxRanks + g) < M.ebase) {
                if (globaltimer_ns() - tj > M.join_ns) { st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1; break; }
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
    if (peer && !pk::grid_sync(M.bar, st)) return;
    if (*(volatile const int*)&st->peer_timeout) return;   // the rendezvous failed (reset by the host)
    uint32_t it = 0;
    double sig[K];
    // ---- setup (row A0 per column): r0 = b - A x0 (or b), x = x0 (or 0), p = r0,
    // nb = ||b||, rho0 = <r0, r0>, the 0-iteration exits (Q2, Q6)
    if (M.has_x0) {                        // P holds the full x0 (host copy): Q = A x0
        gemm_phase<K, WR, CH>(&tmA, &tmP, M, S, it, sig);
        if (!pk::grid_sync(M.bar, st)) return;   // every CTA's rows of Q before they are read
    }
    {
        double v[2 * K];
#pragma unroll
        for (int k = 0; k < 2 * K; ++k) v[k] = 0.0;
        if (cons) {
            for (int64_t i = t0; i < m; i += gs) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double bk = M.R[k * M.ldm + i];          // the host put b's own rows here
                    const double r = M.has_x0 ? bk - M.Q[k * M.ldm + i] : bk;
                    v[k] = fma(bk, bk, v[k]);
                    v[K + k] = fma(r, r, v[K + k]);
                    M.R[k * M.ldm + i] = r;
                    M.X[k * M.ldm + i] = M.has_x0 ? M.Pf[k * M.ld + M.row0 + i] : 0.0;   // x = x0
                    if (peer)
                        for (int g = 0; g < M.L.P; ++g) M.mp.MR[g][mr_off(M, 0, M.L.rank, k) + i] = r;
                }
            }
        }
        if (peer) { __syncthreads(); if (tid == 0) __threadfence_system(); }
        csum<2 * K>(v, S.red);
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < 2 * K; ++k) M.bpart[(int64_t)blockIdx.x * kBSlots * K + k] = v[k];
        }
        if (!pk::grid_sync(M.bar, st)) return;
        double tbr[2 * K];
        {
            double tb[K], tr[K];
            totals<K>(M.bpart, 0, tb, S.red);
            totals<K>(M.bpart, K, tr, S.red);
#pragma unroll
            for (int k = 0; k < K; ++k) { tbr[k] = tb[k]; tbr[K + k] = tr[k]; }
        }
        if (!rank_sum<2 * K>(M, tbr, 0, 0, kPhaseR, M.ebase)) return;   // ||b||^2, <r0, r0> over the ranks
        if (cons) {
            for (int64_t i = t0; i < m; i += gs)                         // Q6: b = 0 -> x = 0
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (!(k < M.nrhs) || tbr[k] == 0.0) M.X[k * M.ldm + i] = 0.0;
            int o = 0;
            for (int64_t j = t0; j < M.n; j += gs) {                      // p0 = r0 (full length)
                int64_t jl = j;
                if (peer) {
                    while (o + 1 < M.L.P && j >= M.L.row0[o + 1]) ++o;   // j only grows per thread
                    jl = j - M.L.row0[o];
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const bool z = !(k < M.nrhs) || tbr[k] == 0.0;
                    const double r = peer ? __ldcg(M.MRo + mr_off(M, 0, o, k) + jl) : M.R[k * M.ldm + j];
                    M.Pf[k * M.ld + j] = z ? 0.0 : r;
                }
            }
        }
        if (blockIdx.x == 0 && tid == 0) {
            for (int k = 0; k < K; ++k) {
                MultiCol& cl = ms->col[k];
                cl.nb = sqrt(tbr[k]);
                cl.rho = tbr[K + k];
                cl.iters = 0;
                cl.relres = 0.0;
                cl.status = KS_EMAXIT;
                cl.active = 1;
                if (k >= M.nrhs || tbr[k] == 0.0) {               // padding column / Q6: b = 0
                    cl.active = 0; cl.status = KS_OK; cl.converged = 1; cl.bzero = 1;
                } else {
                    cl.converged = 0; cl.bzero = 0;
                    cl.relres = sqrt(tbr[K + k]) / cl.nb;
                    if (cl.relres <= M.tol) { cl.active = 0; cl.status = KS_OK; cl.converged = 1; }   // Q2
                }
            }
        }
        if (!pk::grid_sync(M.bar, st)) return;
    }
    // ---- iterations (rows A1-A5 per column)
    for (long long k1 = 1; k1 <= M.maxit; ++k1) {
        const int par = (int)(k1 & 1);
        int act[K];
        int any = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) { act[k] = *(volatile const int*)&ms->col[k].active; any |= act[k]; }
        if (!any) break;
        // A1: Q = A P, sigma partials
        gemm_phase<K, WR, CH>(&tmA, &tmP, M, S, it, sig);
        __syncthreads();
        if ((tid & 31) == 0 && tid < kMCT) {
#pragma unroll
            for (int k = 0; k < K; ++k) S.wpart[tid >> 5][k] = sig[k];
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int ww = 0; ww < kMW; ++ww) s += S.wpart[ww][k];
                M.bpart[(int64_t)blockIdx.x * kBSlots * K + k] = s;
            }
        }
        if (!pk::grid_sync(M.bar, st)) return;
        // A2: sigma (rank all-reduce), alpha (per active column; NOTSPD ends that column, x unchanged)
        double sg[K], alpha[K], rho[K];
        totals<K>(M.bpart, 0, sg, S.red);
        if (!rank_sum<K>(M, sg, par, 0, kPhaseS, M.ebase + (unsigned long long)k1)) return;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            rho[k] = *(volatile const double*)&ms->col[k].rho;
            if (act[k] && !(sg[k] > 0.0)) {
                act[k] = 0;
                if (blockIdx.x == 0 && tid == 0) {
                    ms->col[k].active = 0; ms->col[k].status = KS_ENOTSPD; ms->col[k].iters = k1 - 1;
                }
            }
            alpha[k] = act[k] ? rho[k] / sg[k] : 0.0;
        }
        // A3: x += alpha p; r -= alpha q (own rows, pushed to every rank); rho' partials
        double rr[K];
#pragma unroll
        for (int k = 0; k < K; ++k) rr[k] = 0.0;
        if (cons) {
            for (int64_t i = t0; i < m; i += gs) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (!act[k]) continue;
                    const double pk_ = M.Pf[k * M.ld + M.row0 + i];
                    M.X[k * M.ldm + i] = fma(alpha[k], pk_, M.X[k * M.ldm + i]);
                    const double r = fma(-alpha[k], M.Q[k * M.ldm + i], M.R[k * M.ldm + i]);
                    M.R[k * M.ldm + i] = r;
                    if (peer)
                        for (int g = 0; g < M.L.P; ++g) M.mp.MR[g][mr_off(M, par, M.L.rank, k) + i] = r;
                    rr[k] = fma(r, r, rr[k]);
                }
            }
        }
        if (peer) { __syncthreads(); if (tid == 0) __threadfence_system(); }
        csum<K>(rr, S.red);
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) M.bpart[(int64_t)blockIdx.x * kBSlots * K + K + k] = rr[k];
        }
        if (!pk::grid_sync(M.bar, st)) return;
        // A4 + A5: rho' (rank all-reduce; releases the pushed r slices too), test, beta,
        // p = r + beta p over the full length
        double rho1[K], beta[K];
        totals<K>(M.bpart, K, rho1, S.red);
        if (!rank_sum<K>(M, rho1, par, K, kPhaseR, M.ebase + (unsigned long long)k1)) return;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            beta[k] = 0.0;
            if (!act[k]) continue;
            const double rel = sqrt(rho1[k]) / ms->col[k].nb;
            if (blockIdx.x == 0 && tid == 0) {
                MultiCol& cl = ms->col[k];
                if (M.hist && k1 - 1 < M.hist_cap) M.hist[(int64_t)k * M.hist_cap + (k1 - 1)] = rel;
                cl.relres = rel; cl.iters = k1;
            }
            if (rel <= M.tol) {
                act[k] = 0;
                if (blockIdx.x == 0 && tid == 0) { ms->col[k].active = 0; ms->col[k].status = KS_OK; ms->col[k].converged = 1; }
                continue;
            }
            beta[k] = rho1[k] / rho[k];
        }
        if (cons) {
            int o = 0;
            for (int64_t j = t0; j < M.n; j += gs) {
                int64_t jl = j;
                if (peer) {
                    while (o + 1 < M.L.P && j >= M.L.row0[o + 1]) ++o;   // j only grows per thread
                    jl = j - M.L.row0[o];
                }
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (act[k]) {
                        const double r = peer ? __ldcg(M.MRo + mr_off(M, par, o, k) + jl) : M.R[k * M.ldm + j];
                        M.Pf[k * M.ld + j] = fma(beta[k], M.Pf[k * M.ld + j], r);
                    }
            }
        }
        if (blockIdx.x == 0 && tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) if (act[k]) ms->col[k].rho = rho1[k];
        }
        if (!pk::grid_sync(M.bar, st)) return;
    }
    // ---- end: P > 1 gathers X into every rank's contiguous MX (K x ld)
    if (peer) gather_x<K>(M, S);
}

// ---- multi-RHS BiCGSTAB: rows B0-B8 of SURVEY.md sec.8(c).4 per column, the two
// GEMMs of an iteration (v = A p from P, t = A s from S) shared by the K columns.  Per
// column: own rho, alpha, omega, the exact-zero / non-finite breakdown tests (Q9), the
// half-step exit; a stopped column stops updating.  5 grid barriers per iteration, as
// the single-RHS persistent BiCGSTAB.  P > 1 (fused exchange): the v and r slices go
// into every rank's MV / MR regions (parity of the iteration), <rhat, v>, (<t, s>,
// <t, t>) and (<rhat, r>, <r, r>) are rank all-reduces in disjoint MS slots; s, p and
// ||s||^2 are formed over the full length on every rank from the gathered r and v.
template <int K, int WR, int CH>
__global__ void __launch_bounds__(kMT, 1) k_bsm(const __grid_constant__ CUtensorMap tmA,
                                               const __grid_constant__ CUtensorMap tmP,
                                               const __grid_constant__ CUtensorMap tmS, MultiArgs M) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    MultiSmem<K, WR, CH>& S = *reinterpret_cast<MultiSmem<K, WR, CH>*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    MultiState* ms = M.ms;
    DevState* st = M.st;
    const int tid = threadIdx.x;
    const bool cons = tid < kMCT;
    const int64_t gs = (int64_t)gridDim.x * kMCT;
    const int64_t t0 = (int64_t)blockIdx.x * kMCT + tid;
    const int64_t n = M.n, m = M.m, row0 = M.row0;
    const bool lead = blockIdx.x == 0 && tid == 0;
    const bool peer = M.peer != 0;
    const int me = M.L.rank;
    if (tid == 0) {
        for (int s = 0; s < MultiSmem<K, WR, CH>::kMS; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], kMW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == kMW * 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmP) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmS) : "memory");
    }
    if (peer && lead) {                          // solve-start rendezvous (k_join's protocol)
        unsigned long long* f[kMaxRanks];
        for (int g = 0; g < M.L.P; ++g) f[g] = M.mp.flags[g] + kPhaseJ * kMaxRanks + me;
        publish_flags(f, M.L.P, M.ebase);
        const unsigned long long tj = globaltimer_ns();
        for (int g = 0; g < M.L.P; ++g) {
            while (flag_acquire_sys(M.flags + kPhaseJ * kMaxRanks + g) < M.ebase) {
                if (globaltimer_ns() - tj > M.join_ns) { st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1; break; }
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
    if (peer && !pk::grid_sync(M.bar, st)) return;
    if (*(volatile const int*)&st->peer_timeout) return;
    uint32_t it = 0;
    double d1[K], d2[K];
    // ---- B0: r0 = b - A x0 (or b), rhat = r0, x = x0 (or 0), ||b||, rho_1 = <rhat, r0>
    if (M.has_x0) {
        gemm_phase<K, WR, CH>(&tmA, &tmP, M, S, it, d1);          // Q = A x0 (P holds the full x0)
        if (!pk::grid_sync(M.bar, st)) return;
    }
    {
        double v[2 * K];
#pragma unroll
        for (int k = 0; k < 2 * K; ++k) v[k] = 0.0;
        if (cons) {
            for (int64_t i = t0; i < m; i += gs) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double bk = M.R[k * M.ldm + i];
                    const double r = M.has_x0 ? bk - M.Q[k * M.ldm + i] : bk;
                    v[k] = fma(bk, bk, v[k]);
                    v[K + k] = fma(r, r, v[K + k]);
                    M.R[k * M.ldm + i] = r;
                    M.Rh[k * M.ldm + i] = r;                           // rhat = r0 (Q7)
                    M.X[k * M.ldm + i] = M.has_x0 ? M.Pf[k * M.ld + row0 + i] : 0.0;
                    if (peer)
                        for (int g = 0; g < M.L.P; ++g) M.mp.MR[g][mr_off(M, 0, me, k) + i] = r;
                }
            }
        }
        if (peer) { __syncthreads(); if (tid == 0) __threadfence_system(); }
        csum<2 * K>(v, S.red);
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < 2 * K; ++k) M.bpart[(int64_t)blockIdx.x * kBSlots * K + k] = v[k];
        }
        if (!pk::grid_sync(M.bar, st)) return;
        double tbr[2 * K];
        {
            double tb[K], tr[K];
            totals<K>(M.bpart, 0, tb, S.red);
            totals<K>(M.bpart, K, tr, S.red);
#pragma unroll
            for (int k = 0; k < K; ++k) { tbr[k] = tb[k]; tbr[K + k] = tr[k]; }
        }
        if (!rank_sum<2 * K>(M, tbr, 0, kMsR, kPhaseR, M.ebase)) return;
        if (cons) {
            for (int64_t i = t0; i < m; i += gs)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (!(k < M.nrhs) || tbr[k] == 0.0) M.X[k * M.ldm + i] = 0.0;   // Q6
        }
        if (lead) {
            for (int k = 0; k < K; ++k) {
                MultiCol& cl = ms->col[k];
                cl.nb = sqrt(tbr[k]);
                cl.rho = tbr[K + k];                              // <rhat, r0> = <r0, r0>
                cl.rho_old = cl.alpha = cl.omega = 1.0;           // Q8
                cl.iters = 0; cl.relres = 0.0; cl.status = KS_EMAXIT; cl.active = 1;
                cl.half = 0; cl.breakdown = 0;
                if (k >= M.nrhs || tbr[k] == 0.0) {
                    cl.active = 0; cl.status = KS_OK; cl.converged = 1; cl.bzero = 1;
                } else {
                    cl.converged = 0; cl.bzero = 0;
                    cl.relres = sqrt(tbr[K + k]) / cl.nb;
                    if (cl.relres <= M.tol) { cl.active = 0; cl.status = KS_OK; cl.converged = 1; }   // Q2
                }
            }
        }
        if (!pk::grid_sync(M.bar, st)) return;
    }
    for (long long i1 = 1; i1 <= M.maxit; ++i1) {
        const int par = (int)(i1 & 1), pprev = par ^ 1;
        int act[K];
        int any = 0;
        double rho[K], beta[K], omega[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const MultiCol& cl = ms->col[k];
            act[k] = *(volatile const int*)&cl.active;
            rho[k] = *(volatile const double*)&cl.rho;
            omega[k] = *(volatile const double*)&cl.omega;
            beta[k] = 0.0;
            if (act[k] && (rho[k] == 0.0 || !isfinite(rho[k]))) {          // Q9: rho breakdown
                act[k] = 0;
                if (lead) { ms->col[k].active = 0; ms->col[k].status = KS_EBREAKDOWN; ms->col[k].breakdown = 1;
                            ms->col[k].iters = i1 - 1; }
            }
            if (act[k]) beta[k] = (rho[k] / *(volatile const double*)&cl.rho_old) * (*(volatile const double*)&cl.alpha / omega[k]);
            any |= act[k];
        }
        if (!any) break;
        // B1: p = r + beta (p - omega v) over the full length   (i = 1: p = r)
        if (cons) {
            int o = 0, o2 = 0;
            for (int64_t j = t0; j < n; j += gs)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (act[k]) {
                        const double r = peer ? gathered(M, M.MRo, pprev, k, j, o) : M.R[k * M.ldm + j];
                        if (i1 == 1) { M.Pf[k * M.ld + j] = r; continue; }
                        const double vv = peer ? gathered(M, M.MVo, pprev, k, j, o2) : M.Q[k * M.ldm + j];
                        M.Pf[k * M.ld + j] = fma(beta[k], fma(-omega[k], vv, M.Pf[k * M.ld + j]), r);
                    }
        }
        if (!pk::grid_sync(M.bar, st)) return;
        // B3: v = A p (own rows, into Q; P > 1: pushed to every rank's MV), <rhat, v> partials
        gemm_phase<K, WR, CH>(&tmA, &tmP, M, S, it, d1, M.Q, M.Rh, M.ldm, 0);
        __syncthreads();
        if ((tid & 31) == 0 && tid < kMCT) {
#pragma unroll
            for (int k = 0; k < K; ++k) S.wpart[tid >> 5][k] = d1[k];
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double t = 0.0;
                for (int ww = 0; ww < kMW; ++ww) t += S.wpart[ww][k];
                M.bpart[(int64_t)blockIdx.x * kBSlots * K + k] = t;
            }
        }
        if (!pk::grid_sync(M.bar, st)) return;
        if (peer) {                                  // every CTA's rows of v are complete: push them
            if (cons)
                for (int64_t i = t0; i < m; i += gs)
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const double vv = M.Q[k * M.ldm + i];
                        for (int g = 0; g < M.L.P; ++g) M.mp.MV[g][mr_off(M, par, me, k) + i] = vv;
                    }
            __syncthreads();
            if (tid == 0) __threadfence_system();
            if (!pk::grid_sync(M.bar, st)) return;
        }
        double gam[K], alpha[K];
        totals<K>(M.bpart, 0, gam, S.red);
        if (!rank_sum<K>(M, gam, par, kMsV, kPhaseV, M.ebase + (unsigned long long)i1)) return;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (act[k] && (gam[k] == 0.0 || !isfinite(gam[k]))) {          // Q9
                act[k] = 0;
                if (lead) { ms->col[k].active = 0; ms->col[k].status = KS_EBREAKDOWN; ms->col[k].breakdown = 1;
                            ms->col[k].iters = i1 - 1; }
            }
            alpha[k] = act[k] ? rho[k] / gam[k] : 0.0;
        }
        // B4: s = r - alpha v over the full length (identical on every rank), ||s||^2
        double ssp[K];
#pragma unroll
        for (int k = 0; k < K; ++k) ssp[k] = 0.0;
        if (cons) {
            int o = 0, o2 = 0;
            for (int64_t j = t0; j < n; j += gs)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (act[k]) {
                        const double r = peer ? gathered(M, M.MRo, pprev, k, j, o) : M.R[k * M.ldm + j];
                        const double vv = peer ? gathered(M, M.MVo, par, k, j, o2) : M.Q[k * M.ldm + j];
                        const double sv = fma(-alpha[k], vv, r);
                        M.Sf[k * M.ld + j] = sv;
                        ssp[k] = fma(sv, sv, ssp[k]);
                    }
        }
        csum<K>(ssp, S.red);
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) M.bpart[(int64_t)blockIdx.x * kBSlots * K + K + k] = ssp[k];
        }
        if (!pk::grid_sync(M.bar, st)) return;
        double ss[K];
        totals<K>(M.bpart, K, ss, S.red);
        int half[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            half[k] = 0;
            if (!act[k]) continue;
            const double srel = sqrt(ss[k]) / ms->col[k].nb;
            if (srel <= M.tol) {                                           // B5: half-step exit
                half[k] = 1;
                act[k] = 0;
                if (lead) {
                    MultiCol& cl = ms->col[k];
                    if (M.hist && i1 - 1 < M.hist_cap) M.hist[(int64_t)k * M.hist_cap + (i1 - 1)] = srel;
                    cl.relres = srel; cl.iters = i1; cl.half = 1; cl.converged = 1; cl.status = KS_OK;
                    cl.active = 0; cl.alpha = alpha[k];
                }
            }
        }
        if (cons) {                                                        // half step: x += alpha p
            for (int64_t i = t0; i < m; i += gs)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (half[k]) M.X[k * M.ldm + i] = fma(alpha[k], M.Pf[k * M.ld + row0 + i], M.X[k * M.ldm + i]);
        }
        // B6: t = A s (own rows, into T), <s, t> and <t, t> partials
        gemm_phase<K, WR, CH, true>(&tmA, &tmS, M, S, it, d1, M.T, M.Sf, M.ld, row0, d2);
        __syncthreads();
        if ((tid & 31) == 0 && tid < kMCT) {
#pragma unroll
            for (int k = 0; k < K; ++k) { S.wpart[tid >> 5][k] = d1[k]; S.wpart2[tid >> 5][k] = d2[k]; }
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double a1 = 0.0, a2 = 0.0;
                for (int ww = 0; ww < kMW; ++ww) { a1 += S.wpart[ww][k]; a2 += S.wpart2[ww][k]; }
                M.bpart[(int64_t)blockIdx.x * kBSlots * K + 2 * K + k] = a1;
                M.bpart[(int64_t)blockIdx.x * kBSlots * K + 3 * K + k] = a2;
            }
        }
        if (!pk::grid_sync(M.bar, st)) return;
        double tst[2 * K];
        {
            double ts[K], tt[K];
            totals<K>(M.bpart, 2 * K, ts, S.red);
            totals<K>(M.bpart, 3 * K, tt, S.red);
#pragma unroll
            for (int k = 0; k < K; ++k) { tst[k] = ts[k]; tst[K + k] = tt[k]; }
        }
        if (!rank_sum<2 * K>(M, tst, par, kMsS, kPhaseS, M.ebase + (unsigned long long)i1)) return;
        double om[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            om[k] = 0.0;
            if (!act[k]) continue;
            const double tt = tst[K + k];
            bool bad = tt == 0.0 || !isfinite(tt);
            if (!bad) { om[k] = tst[k] / tt; bad = om[k] == 0.0 || !isfinite(om[k]); }
            if (bad) {                                                     // Q9
                act[k] = 0;
                if (lead) { ms->col[k].active = 0; ms->col[k].status = KS_EBREAKDOWN; ms->col[k].breakdown = 1;
                            ms->col[k].iters = i1 - 1; }
            }
        }
        // B7: x = (x + alpha p) + omega s; r = s - omega t (own rows; P > 1: pushed);
        // <rhat, r>, <r, r> partials
        double v2[2 * K];
#pragma unroll
        for (int k = 0; k < 2 * K; ++k) v2[k] = 0.0;
        if (cons) {
            for (int64_t i = t0; i < m; i += gs)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (act[k]) {
                        const double sv = M.Sf[k * M.ld + row0 + i];
                        M.X[k * M.ldm + i] = fma(om[k], sv, fma(alpha[k], M.Pf[k * M.ld + row0 + i], M.X[k * M.ldm + i]));
                        const double r = fma(-om[k], M.T[k * M.ldm + i], sv);
                        M.R[k * M.ldm + i] = r;
                        if (peer)
                            for (int g = 0; g < M.L.P; ++g) M.mp.MR[g][mr_off(M, par, me, k) + i] = r;
                        v2[k] = fma(M.Rh[k * M.ldm + i], r, v2[k]);
                        v2[K + k] = fma(r, r, v2[K + k]);
                    }
        }
        if (peer) { __syncthreads(); if (tid == 0) __threadfence_system(); }
        csum<2 * K>(v2, S.red);
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < 2 * K; ++k) M.bpart[(int64_t)blockIdx.x * kBSlots * K + 4 * K + k] = v2[k];
        }
        if (!pk::grid_sync(M.bar, st)) return;
        double rr2[2 * K];
        {
            double rhn[K], rr[K];
            totals<K>(M.bpart, 4 * K, rhn, S.red);
            totals<K>(M.bpart, 5 * K, rr, S.red);
#pragma unroll
            for (int k = 0; k < K; ++k) { rr2[k] = rhn[k]; rr2[K + k] = rr[k]; }
        }
        if (!rank_sum<2 * K>(M, rr2, par, kMsR, kPhaseR, M.ebase + (unsigned long long)i1)) return;
        // B8: history, test; rho_old = rho, rho = <rhat, r>
        if (lead) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (!act[k]) continue;
                MultiCol& cl = ms->col[k];
                const double rel = sqrt(rr2[K + k]) / cl.nb;
                if (M.hist && i1 - 1 < M.hist_cap) M.hist[(int64_t)k * M.hist_cap + (i1 - 1)] = rel;
                cl.relres = rel; cl.iters = i1;
                cl.rho_old = rho[k]; cl.rho = rr2[k]; cl.alpha = alpha[k]; cl.omega = om[k];
                if (rel <= M.tol) { cl.active = 0; cl.converged = 1; cl.status = KS_OK; }
            }
        }
        if (!pk::grid_sync(M.bar, st)) return;
    }
    if (peer) gather_x<K>(M, S);
}

// shapes: 0 = (4 rows/warp, 128 columns, 4 stages), 1 = (8, 64, 4), 2 = (8, 128, 3)
int multi_shape(int K) {
    if (const char* e = std::getenv("KS_MULTI_SHAPE")) {                // tuning
        const int v = std::atoi(e);
        return v == 1 || v == 2 ? v : 0;
    }
    (void)K;
    return 2;   // measured best for K = 4 and 8 (profiles/r02_multi_rhs_shapes.jsonl)
}
const void* kern_m(int K, int shape) {
    if (K == 4) return shape == 1 ? (const void*)k_cgm<4, 8, 64>
                     : shape == 2 ? (const void*)k_cgm<4, 8, 128> : (const void*)k_cgm<4, 4, 128>;
    return shape == 1 ? (const void*)k_cgm<8, 8, 64>
         : shape == 2 ? (const void*)k_cgm<8, 8, 128> : (const void*)k_cgm<8, 4, 128>;
}
const void* kern_bs(int K) {
    return K == 4 ? (const void*)k_bsm<4, 8, 128> : (const void*)k_bsm<8, 8, 128>;
}
size_t smem_m(int K, int shape) {
    size_t b;
    if (K == 4) b = shape == 1 ? sizeof(MultiSmem<4, 8, 64>) : shape == 2 ? sizeof(MultiSmem<4, 8, 128>)
                                                                        : sizeof(MultiSmem<4, 4, 128>);
    else b = shape == 1 ? sizeof(MultiSmem<8, 8, 64>) : shape == 2 ? sizeof(MultiSmem<8, 8, 128>)
                                                                   : sizeof(MultiSmem<8, 4, 128>);
    return b + 1024;
}

}  // namespace

int multi_k(int nrhs) { return nrhs <= 4 ? 4 : nrhs <= 8 ? 8 : 0; }

int multi_grid(int K, int num_sms) {
    const int shape = multi_shape(K);
    const void* k = kern_m(K, shape);
    const size_t sm = smem_m(K, shape);
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
    if (sm > (size_t)optin) return 0;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { cudaGetLastError(); return 0; }
    const int dyn_max = optin - (int)fa.sharedSizeBytes;     // opt-in limit minus static smem
    if ((size_t)dyn_max < sm ||
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kMT, sm);
    if (per_sm < 1) return 0;
    return num_sms;
}

// 2-D tensor map of a row-major FP64 matrix (rows x cols, leading dimension ld
// elements), box = box_rows x box_cols, zero fill out of bounds.
static bool make_map(CUtensorMap* tm, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     int box_cols) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return false;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int multi_grid_bs(int K, int num_sms) {
    const void* k = kern_bs(K);
    const size_t sm = smem_m(K, 2);
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { cudaGetLastError(); return 0; }
    const int dyn_max = optin - (int)fa.sharedSizeBytes;
    if ((size_t)dyn_max < sm ||
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kMT, sm);
    return per_sm >= 1 ? num_sms : 0;
}

int launch_bicgstab_multi(int K, const MultiArgs& M, const double* A, int grid, cudaStream_t st) {
    CUtensorMap tmA, tmP, tmS;
    if (!make_map(&tmA, A, M.m, M.ld, M.ld, kMW * 8, 128)) return -(int)cudaErrorInvalidValue;
    if (!make_map(&tmP, M.Pf, K, M.ld, M.ld, K, 128)) return -(int)cudaErrorInvalidValue;
    if (!make_map(&tmS, M.Sf, K, M.ld, M.ld, K, 128)) return -(int)cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(M.bar, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return -(int)e;
    MultiArgs Mc = M;
    void* args[] = {&tmA, &tmP, &tmS, &Mc};
    e = cudaLaunchCooperativeKernel(kern_bs(K), dim3((unsigned)grid), dim3(kMT), args, smem_m(K, 2), st);
    return e == cudaSuccess ? 1 : -(int)e;
}

int launch_cg_multi(int K, const MultiArgs& M, const double* A, int grid, cudaStream_t st) {
    const int shape = multi_shape(K);
    const int band = kMW * (shape == 0 ? 4 : 8), ch = shape == 1 ? 64 : 128;
    CUtensorMap tmA, tmP;
    if (!make_map(&tmA, A, M.m, M.ld, M.ld, band, ch)) return -(int)cudaErrorInvalidValue;
    if (!make_map(&tmP, M.Pf, K, M.ld, M.ld, K, ch)) return -(int)cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(M.bar, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return -(int)e;
    MultiArgs Mc = M;
    void* args[] = {&tmA, &tmP, &Mc};
    e = cudaLaunchCooperativeKernel(kern_m(K, shape), dim3((unsigned)grid), dim3(kMT), args,
                                    smem_m(K, shape), st);
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ks

// Building blocks of the persistent cooperative kernels (ks_persist.cu for CG /
// BiCGSTAB, ks_gmres_persist.cu for GMRES): grid barrier, CTA-order totals,
// fused-exchange flag helpers, and the GEMV phase (K1's streaming loop over
// round-robin tiles).  Everything is deterministic: fixed tile -> CTA
// assignment, CTA partials summed in CTA order by a fixed tree.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ks_device.cuh"
#include "ks_common.cuh"
#include "ks_internal.h"
#include "ks_tile.cuh"

namespace ks {
namespace pk {
namespace {

constexpr int kNT = 256;
constexpr int kNW = kNT / 32;
// GEMV tile shape of the persistent kernels (rows R x unrolled column blocks U);
// instantiated for the shapes the tuning sweep found at the streaming ceiling.

// -- small helpers (layout / state accessors are shared: ks_common.cuh) ---------
template <class T>
__device__ __forceinline__ T* par_ptr(T* G, int64_t par, long long k) { return G + (k & 1) * par; }

// Grid-wide barrier (all CTAs co-resident: cooperative launch).  One 64-bit
// arrival counter, zeroed by the launcher before every launch and never reset
// inside it: barrier b of the launch completes when the counter reaches
// (b + 1) * gridDim.x, and each CTA learns b from the value its own arrival
// returned.  Waiters observe the last arrival directly (no second round trip
// through a generation word).  Arrival = fence (release, cumulative over the
// CTA's bar.sync) + relaxed atomicAdd; wait = ld.acquire.gpu.  Bounded spin: a
// timeout marks the solve failed instead of hanging.
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// nb = the CTAs that meet (gridDim.x, or one rank's CTAs of an emulated launch).
__device__ bool grid_sync_n(unsigned* bar, DevState* st, unsigned nb) {
    __shared__ int s_ok;
    __shared__ unsigned s_jit;
    __syncthreads();
    if (threadIdx.x == 0) {
        int ok = 1;
        const unsigned jit = *(volatile const unsigned*)&st->jitter;
        jitter_at(jit, 1u);                       // arrival order (race detection; 0: off)
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(bar);
        __threadfence();
        const unsigned long long old = atomicAdd(cnt, 1ull);
        const unsigned long long target = (old / nb + 1ull) * nb;
        if (old + 1ull != target) {
            const unsigned long long t0 = globaltimer_ns();
            while (ld_acquire_gpu_u64(cnt) < target) {
                if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                    ok = 0;
                    st->peer_timeout = 1; st->status = KS_ECUDA; st->done = 1;
                    break;
                }
            }
        } else {
            __threadfence();   // last arrival: acquire the other CTAs' writes
        }
        s_ok = ok;
        s_jit = jit;
    }
    __syncthreads();
    jitter_at(s_jit, 2u);                         // departure order of the warps
    return s_ok != 0;
}
__device__ __forceinline__ bool grid_sync(unsigned* bar, DevState* st) { return grid_sync_n(bar, st, gridDim.x); }

// Sum over CTAs (in CTA order, fixed tree) of slot q of the per-CTA partials;
// every CTA computes the same value.
template <int K, class T>
__device__ __forceinline__ void grid_total(const T* bpart, int q0, T (&out)[K], T* red, int nb) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T acc = T(0);
        for (int b = threadIdx.x; b < nb; b += kNT) acc += __ldcg(bpart + (int64_t)b * 4 + q0 + k);
        out[k] = acc;
    }
    block_sum<kNT, K>(out, red);
}
template <int K, class T>
__device__ __forceinline__ void grid_total(const T* bpart, int q0, T (&out)[K], T* red) {
    grid_total<K>(bpart, q0, out, red, (int)gridDim.x);
}

// Fused-mode wait for phase ph of iteration k from every rank (all CTAs).
template <class T>
__device__ __forceinline__ bool wait_ph(const VecArgsT<T>& a, int ph, long long k) {
    if (threadIdx.x == 0) jitter_at(a.jitter, 3u);
    const bool ok = wait_flags(a.flags + ph * kMaxRanks, a.L.P, epoch_of(a.st, k));
    if (!ok && threadIdx.x == 0) { a.st->peer_timeout = 1; a.st->status = KS_ENCCL; a.st->done = 1; }
    return ok;
}
template <class T>
__device__ __forceinline__ void flags_out(const VecArgsT<T>& a, int ph, long long k) {
    unsigned long long* f[kMaxRanks];
    for (int g = 0; g < a.L.P; ++g) f[g] = a.pp.flags[g] + ph * kMaxRanks + a.L.rank;
    jitter_at(a.jitter, 4u);
    publish_flags(f, a.L.P, epoch_of(a.st, k));
}

// ---- LL handovers over P > 1 GPUs (KS_OPT_LL_XCHG; layout: ks_internal.h ll_*) ----
// One value = two 8-byte words, each 32 payload bits + the 32-bit epoch, written with
// one 16-byte system-scope store into every rank's region; a reader polls its local
// copy until both words carry the epoch.  Each 8-byte word is single-copy atomic, so a
// matching pair is the value: no fence on the producer side, no flag.  Values travel
// as double (exact for float).
__device__ __forceinline__ void ll_put_sys(uint64_t* slot, double v, uint32_t ep) {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const uint64_t lo = (bits & 0xffffffffull) | ((uint64_t)ep << 32);
    const uint64_t hi = (bits >> 32) | ((uint64_t)ep << 32);
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(lo), "l"(hi) : "memory");
}
// Polls one value (bounded: false after kWaitTimeoutNs -- a lost peer).
__device__ __forceinline__ bool ll_get_sys(const uint64_t* slot, uint32_t ep, double& v) {
    unsigned long long t0 = 0;
    for (int spin = 0;; ++spin) {
        uint64_t lo, hi;
        asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(slot) : "memory");
        if ((uint32_t)(lo >> 32) == ep && (uint32_t)(hi >> 32) == ep) {
            v = __longlong_as_double((long long)(((hi & 0xffffffffull) << 32) | (lo & 0xffffffffull)));
            return true;
        }
        if ((spin & 63) == 63) {
            if (t0 == 0) t0 = globaltimer_ns();
            else if (globaltimer_ns() - t0 > kWaitTimeoutNs) return false;
        }
    }
}
__device__ __forceinline__ uint32_t ll_epoch(const DevState* st, long long k) { return (uint32_t)epoch_of(st, k); }
// Rank-partial all-reduce of K scalars of LL phase ph: the lead CTA pushed its rank's
// values (ll_push_scal); every CTA polls the P x K words (thread g * K + q) and sums
// them in rank order (the order scal_sum / slot_sum use), so every thread of every
// CTA of every rank ends with the same bits.  False (all threads) on a timeout.
template <class T>
__device__ __forceinline__ void ll_push_scal(const VecArgsT<T>& a, int par, int ph, const double* v, int K,
                                             uint32_t ep) {
    jitter_at(a.jitter, 8u);
    for (int g = 0; g < a.L.P; ++g)
        for (int q = 0; q < K; ++q) ll_put_sys(a.pp.llg[g] + ll_scal_off(a.L.ld, par, ph, a.L.rank, q), v[q], ep);
}
template <int K, class T>
__device__ __forceinline__ bool ll_sum_scal(const VecArgsT<T>& a, int par, int ph, uint32_t ep, T (&out)[K]) {
    __shared__ double s_v[kMaxRanks * 2];
    __shared__ int s_ok;
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    const int P = a.L.P;
    if ((int)threadIdx.x < P * K) {
        jitter_at(a.jitter, 9u);
        const int g = threadIdx.x / K, q = threadIdx.x % K;
        double v = 0.0;
        if (!ll_get_sys(a.llg + ll_scal_off(a.L.ld, par, ph, g, q), ep, v)) s_ok = 0;
        s_v[g * K + q] = v;
    }
    __syncthreads();
    if (!s_ok) {
        if (threadIdx.x == 0) { a.st->peer_timeout = 1; a.st->status = KS_ENCCL; a.st->done = 1; }
        return false;
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        T t = T(0);
        for (int g = 0; g < P; ++g) t += (T)s_v[g * K + q];
        out[q] = t;
    }
    return true;
}

template <class T>
struct PersistArgs {
    VecArgsT<T> a;
    const T* A;
    int64_t lda, ncols;
    T* bpart;           // gridDim.x * 4
    unsigned* bar;      // {count, generation}
    long long k0, k1;   // iteration range of this launch (inclusive)
    int defer = 0;      // 1: deferred row reductions in the GEMV phase (gemv_phase)
};

// GEMV phase: y = A_loc x (or bsub - A_loc x) over the tiles of this CTA
// (round-robin); thread 0 returns the CTA's partials <w1, y> and <y, y>
// accumulated in tile order.
template <int kR, int kU, class T>
__device__ void gemv_phase(const PersistArgs<T>& P, const T* x, T* y, const T* w1, T& d1, T& d2,
                           T* red, const T* bsub, int vb, int vg) {
    const int64_t m = rows_of(P.a.L);
    const int64_t tiles = (m + kR - 1) / kR;
    const int64_t ncb = P.ncols / (Vec16<T>::W * kNT);
    d1 = T(0);
    d2 = T(0);
    // Deferred row reductions (P.defer): each warp parks its row partials of every tile
    // in shared memory and streams on -- no CTA barrier between tiles, so a CTA's loads
    // never drain at a tile boundary (a tile of a 16384-column row is only 4 load steps).
    // One barrier at the end; then each row's warp partials are added in warp order and
    // the dot partials are a fixed-tree block sum (every thread returns them).
    constexpr int kDeferRows = 256;
    __shared__ T wp[kDeferRows * kNW];
    const int64_t mine = tiles > vb ? (tiles - vb + vg - 1) / vg : 0;
    if (P.defer && mine * kR <= kDeferRows) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int nt = 0;
        for (int64_t tile = vb; tile < tiles; tile += vg, ++nt) {
            const int64_t r0 = tile * kR;
            const int nvalid = (int)min((int64_t)kR, m - r0);
            T acc[kR];
            stream_rows<kR, kU, kNT>(P.A, P.lda, r0, nvalid, x, 0, ncb, acc);
#pragma unroll
            for (int r = 0; r < kR; ++r) acc[r] = warp_sum(acc[r]);
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < kR; ++r) wp[(nt * kR + r) * kNW + w] = acc[r];
            }
        }
        __syncthreads();
        T v2[2] = {T(0), T(0)};
        for (int j = threadIdx.x; j < nt * kR; j += kNT) {
            const int64_t row = ((int64_t)vb + (int64_t)(j / kR) * vg) * kR + (j % kR);
            if (row < m) {
                T sum = T(0);
#pragma unroll
                for (int ww = 0; ww < kNW; ++ww) sum += wp[j * kNW + ww];
                const T yv = bsub ? bsub[row] - sum : sum;
                y[row] = yv;
                if (w1) v2[0] = fma(w1[row], yv, v2[0]);
                v2[1] = fma(yv, yv, v2[1]);
            }
        }
        block_sum<kNT, 2>(v2, red);
        d1 = v2[0];
        d2 = v2[1];
        return;
    }
    for (int64_t tile = vb; tile < tiles; tile += vg) {
        const int64_t r0 = tile * kR;
        const int nvalid = (int)min((int64_t)kR, m - r0);
        T acc[kR];
        stream_rows<kR, kU, kNT>(P.A, P.lda, r0, nvalid, x, 0, ncb, acc);
        block_sum<kNT, kR>(acc, red);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                if (r < nvalid) {
                    const T yv = bsub ? bsub[r0 + r] - acc[r] : acc[r];
                    y[r0 + r] = yv;
                    if (w1) d1 = fma(w1[r0 + r], yv, d1);
                    d2 = fma(yv, yv, d2);
                }
            }
        }
    }
}


}  // namespace
}  // namespace pk
}  // namespace ks

// Device helpers shared by the sm_100a kernels: deterministic warp / block / grid
// reductions (fixed summation trees, so every rank that runs the same launch on
// the same data gets bitwise-identical scalars -- DESIGN.md "Determinism").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ks_internal.h"

namespace ks {

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
    // xor butterfly: a+b == b+a in IEEE, so all lanes end with the same bits.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of K values per thread; result valid in every thread.  `red` must
// hold K * (NT/32) doubles.  Fixed tree: warp butterfly, then warp sums added in
// warp order by a butterfly over the first NT/32 lanes of every warp.
template <int NT, int K, class T>
__device__ __forceinline__ void block_sum(T (&v)[K], T* red) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();  // protect `red` from a previous use
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[k * NW + w] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T t = lane < NW ? red[k * NW + lane] : T(0);
        v[k] = warp_sum(t);
    }
}

// Last-block grid reduction of K values (block totals already in v, all threads).
// Returns true in the last-arriving block, whose threads then hold the grid
// totals in v (blocks summed in blockIdx order by a fixed tree).  The ticket is
// reset by the last block so the slot can be reused by the next launch.
template <int NT, int K, class T>
__device__ __forceinline__ bool grid_sum(T (&v)[K], T* part, unsigned* ticket, T* red) {
    __shared__ int s_last;
    const int nb = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) part[(int64_t)blockIdx.x * K + k] = v[k];
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == (unsigned)(nb - 1));
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T acc = T(0);
        for (int b = threadIdx.x; b < nb; b += NT) acc += __ldcg(part + (int64_t)b * K + k);
        v[k] = acc;
    }
    block_sum<NT, K>(v, red);
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

// ---- race detection (KS_OPT_JITTER) -----------------------------------------
// At a synchronisation point (grid-barrier arrival and departure, flag publish and
// wait, LL store and poll) a pseudo-random quarter of the visits of each warp sleep
// up to ~4 us, so the order in which CTAs, warps and ranks reach every hand-over
// changes from run to run.  The kernels' results do not depend on that order (fixed
// summation trees, epoch-tagged exchanges), so a run with jitter must equal a run
// without it bit for bit; a missing barrier or fence shows up as a difference or a
// hang-timeout instead (tests/test_gpu_race.py).  seed = 0: one predictable branch.
static __device__ __noinline__ void jitter_sleep(unsigned seed, unsigned site) {
    unsigned h = seed ^ (blockIdx.x * 0x9E3779B1u) ^ (site * 0x85EBCA77u) ^ ((threadIdx.x >> 5) * 0xC2B2AE3Du) ^
                 (unsigned)clock64();
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    if ((h & 3u) == 0u) __nanosleep(h >> 20);
}
// out of line: the hot kernels only pay a predictable branch (no registers held for it)
__device__ __forceinline__ void jitter_at(unsigned seed, unsigned site) {
    if (__builtin_expect(seed != 0u, 0)) jitter_sleep(seed, site);
}

// ---- fused NVLink collectives: epoch flags ---------------------------------
__device__ __forceinline__ void flag_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void flag_store_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long flag_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Block-wide wait until flags[src] >= epoch for every source rank (thread 0
// spins with acquire loads; the barrier then orders every thread's later loads).
// Bounded: after kWaitTimeoutNs the wait gives up and returns false, so a broken
// peer can never hang the GPU.
constexpr unsigned long long kWaitTimeoutNs = 10ULL * 1000 * 1000 * 1000;
__device__ __forceinline__ bool wait_flags(const unsigned long long* flags, int P,
                                           unsigned long long epoch) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        int ok = 1;
        const unsigned long long t0 = globaltimer_ns();
        for (int g = 0; g < P && ok; ++g) {
            while (flag_acquire_sys(flags + g) < epoch) {
                if (globaltimer_ns() - t0 > kWaitTimeoutNs) { ok = 0; break; }
                __nanosleep(20);
            }
        }
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// Releases `epoch` into flag slot f_peer[g] of every rank g: ONE fence.sc.sys
// (orders every store this thread performed or observed before it) followed by
// relaxed system-scope stores -- a release pattern whose P flag stores are posted
// back to back (P st.release.sys would each wait for the previous remote store).
__device__ __forceinline__ void publish_flags(unsigned long long* const* f_peer, int P,
                                              unsigned long long epoch) {
    __threadfence_system();
    for (int g = 0; g < P; ++g) flag_store_relaxed_sys(f_peer[g], epoch);
}

}  // namespace ks

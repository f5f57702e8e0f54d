// The K1 streaming inner loop, shared by the per-launch GEMV (ks_gemv.cu) and the
// persistent whole-iteration kernels (ks_persist.cu), so both stream A with the
// identical instruction sequence.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ks {

__device__ __forceinline__ double2 ld_stream(const double* p) {
    return __ldcs(reinterpret_cast<const double2*>(p));   // ld.global.cs: evict-first
}
__device__ __forceinline__ double2 ld_x(const double* p) {
    return __ldg(reinterpret_cast<const double2*>(p));    // ld.global.nc: read-only path
}
__device__ __forceinline__ float4 ld_stream(const float* p) {
    return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 ld_x(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ double fma16(const double2& a, const double2& x, double acc) {
    acc = fma(a.x, x.x, acc);
    return fma(a.y, x.y, acc);
}
__device__ __forceinline__ float fma16(const float4& a, const float4& x, float acc) {
    acc = fmaf(a.x, x.x, acc);
    acc = fmaf(a.y, x.y, acc);
    acc = fmaf(a.z, x.z, acc);
    return fmaf(a.w, x.w, acc);
}
// 16-byte vector of T: W elements per load (2 doubles / 4 floats), so a CTA of NT
// threads covers W * NT columns (4 KiB of a row) per column block.
template <class T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int W = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int W = 4; };

// acc[r] = sum over column blocks [cb0, cb1) of A[r0 + r, cols] * x[cols], where
// thread t owns columns 2t + 2*NT*cb (128-bit loads, 512 contiguous bytes of one
// row per warp instruction).  U column blocks are unrolled so U*R independent
// 16-byte loads are in flight per thread.  Rows >= nvalid re-read the last valid
// row (tail tile) and are discarded by the caller.  kXS: x lives in shared memory
// (the small-n kernels, ks_small.cu) instead of global memory.
template <int R, int U, int NT, class T, bool kXS = false>
__device__ __forceinline__ void stream_rows(const T* A, int64_t lda, int64_t r0, int nvalid,
                                            const T* x, int64_t cb0, int64_t cb1, T (&acc)[R]) {
    using V = typename Vec16<T>::type;
    constexpr int W = Vec16<T>::W;
    const T* base = A + r0 * lda + W * threadIdx.x;
    int64_t roff[R];
#pragma unroll
    for (int r = 0; r < R; ++r) roff[r] = (int64_t)min(r, nvalid - 1) * lda;
    const T* xp = x + W * threadIdx.x;
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = T(0);
    int64_t cb = cb0;
    for (; cb + U <= cb1; cb += U) {
        V av[U][R];
        V xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = (cb + u) * (W * NT);
            xv[u] = kXS ? *reinterpret_cast<const V*>(xp + c) : ld_x(xp + c);
#pragma unroll
            for (int r = 0; r < R; ++r) av[u][r] = ld_stream(base + roff[r] + c);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fma16(av[u][r], xv[u], acc[r]);
        }
    }
    for (; cb < cb1; ++cb) {
        const int64_t c = cb * (W * NT);
        const V xv = kXS ? *reinterpret_cast<const V*>(xp + c) : ld_x(xp + c);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma16(ld_stream(base + roff[r] + c), xv, acc[r]);
    }
}

}  // namespace ks

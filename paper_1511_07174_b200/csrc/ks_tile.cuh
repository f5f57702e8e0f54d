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

// acc[r] = sum over column blocks [cb0, cb1) of A[r0 + r, cols] * x[cols], where
// thread t owns columns 2t + 2*NT*cb (128-bit loads, 512 contiguous bytes of one
// row per warp instruction).  U column blocks are unrolled so U*R independent
// 16-byte loads are in flight per thread.  Rows >= nvalid re-read the last valid
// row (tail tile) and are discarded by the caller.
template <int R, int U, int NT>
__device__ __forceinline__ void stream_rows(const double* A, int64_t lda, int64_t r0, int nvalid,
                                            const double* x, int64_t cb0, int64_t cb1,
                                            double (&acc)[R]) {
    const double* base = A + r0 * lda + 2 * threadIdx.x;
    int64_t roff[R];
#pragma unroll
    for (int r = 0; r < R; ++r) roff[r] = (int64_t)min(r, nvalid - 1) * lda;
    const double* xp = x + 2 * threadIdx.x;
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int64_t cb = cb0;
    for (; cb + U <= cb1; cb += U) {
        double2 av[U][R];
        double2 xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = (cb + u) * (2 * NT);
            xv[u] = ld_x(xp + c);
#pragma unroll
            for (int r = 0; r < R; ++r) av[u][r] = ld_stream(base + roff[r] + c);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                acc[r] = fma(av[u][r].x, xv[u].x, acc[r]);
                acc[r] = fma(av[u][r].y, xv[u].y, acc[r]);
            }
        }
    }
    for (; cb < cb1; ++cb) {
        const int64_t c = cb * (2 * NT);
        const double2 xv = ld_x(xp + c);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double2 a = ld_stream(base + roff[r] + c);
            acc[r] = fma(a.x, xv.x, acc[r]);
            acc[r] = fma(a.y, xv.y, acc[r]);
        }
    }
}

}  // namespace ks

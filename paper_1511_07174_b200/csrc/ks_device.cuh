// Device helpers shared by the sm_100a kernels: deterministic warp / block / grid
// reductions (fixed summation trees, so every rank that runs the same launch on
// the same data gets bitwise-identical scalars -- DESIGN.md "Determinism").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ks_internal.h"

namespace ks {

__device__ __forceinline__ double warp_sum(double v) {
    // xor butterfly: a+b == b+a in IEEE, so all lanes end with the same bits.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of K values per thread; result valid in every thread.  `red` must
// hold K * (NT/32) doubles.  Fixed tree: warp butterfly, then warp sums added in
// warp order by a butterfly over the first NT/32 lanes of every warp.
template <int NT, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red) {
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
        double t = lane < NW ? red[k * NW + lane] : 0.0;
        v[k] = warp_sum(t);
    }
}

// Last-block grid reduction of K values (block totals already in v, all threads).
// Returns true in the last-arriving block, whose threads then hold the grid
// totals in v (blocks summed in blockIdx order by a fixed tree).  The ticket is
// reset by the last block so the slot can be reused by the next launch.
template <int NT, int K>
__device__ __forceinline__ bool grid_sum(double (&v)[K], double* part, unsigned* ticket,
                                         double* red) {
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
        double acc = 0.0;
        for (int b = threadIdx.x; b < nb; b += NT) acc += __ldcg(part + (int64_t)b * K + k);
        v[k] = acc;
    }
    block_sum<NT, K>(v, red);
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

}  // namespace ks

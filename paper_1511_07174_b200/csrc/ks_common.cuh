// Device helpers shared by every kernel file: row-block layout arithmetic, the
// rank-ordered sums of gathered partial slots, and the solver-state accessors.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ks_internal.h"

namespace ks {

// rows of this rank's shard
__device__ __forceinline__ int64_t rows_of(const Layout& L) { return L.row0[L.rank + 1] - L.row0[L.rank]; }
__device__ __forceinline__ bool lead() { return blockIdx.x == 0 && threadIdx.x == 0; }
// element j of a full-length vector inside a chunk-layout gather buffer; *owner = its rank
__device__ __forceinline__ int64_t gidx_owner(const Layout& L, int64_t j, int* owner) {
    int g = 0;
    while (g + 1 < L.P && j >= L.row0[g + 1]) ++g;
    *owner = g;
    return (int64_t)g * L.chunk + (j - L.row0[g]);
}
__device__ __forceinline__ int64_t gidx(const Layout& L, int64_t j) {
    int o;
    return gidx_owner(L, j, &o);
}
// rank-ordered sum of partial slot q of every chunk of a gather buffer
template <class T>
__device__ __forceinline__ T slot_sum(const Layout& L, const T* G, int q) {
    T s = T(0);
    for (int g = 0; g < L.P; ++g) s += G[(int64_t)g * L.chunk + L.pslot + q];
    return s;
}
// rank-ordered sum of entry q of the scalar gather buffer (kScalSlot per rank)
template <class T>
__device__ __forceinline__ T scal_sum(const Layout& L, const T* S, int q) {
    T s = T(0);
    for (int g = 0; g < L.P; ++g) s += S[g * kScalSlot + q];
    return s;
}
__device__ __forceinline__ bool is_done(const DevState* st) { return *(volatile const int*)&st->done != 0; }
__device__ __forceinline__ void put_hist(DevState* st, double* hist, long long k1, double v) {
    if (hist && k1 >= 0 && k1 < st->hist_cap) hist[k1] = v;
}
// epoch of iteration k of the current solve (fused exchange flags)
__device__ __forceinline__ unsigned long long epoch_of(const DevState* st, long long k) {
    return *(volatile const unsigned long long*)&st->ebase + (unsigned long long)k;
}

}  // namespace ks

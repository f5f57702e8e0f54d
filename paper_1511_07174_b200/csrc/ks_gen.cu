// K0 -- device expansion of the synthetic inputs.  The
// 34-550 GB configs can only come from here: host RAM cannot stage them.
// Counter-based (SplitMix64), O(1) per entry, and exact: every entry is either a
// sign flip of a table value (G-SPD) or a dyadic rational with exact row sums
// (G-DD), so this expansion is bitwise equal to the oracle's independent one
// (pin P12).  None of the Krylov method's arithmetic lives here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ks_internal.h"

namespace ks {

namespace {

constexpr int kNT = 256;

__device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t key) {
    return sm64(sm64(seed ^ (stream << 56)) + key);
}
// sm64(seed ^ (stream << 56)) hoisted: H = sm64(base + key)
__device__ __forceinline__ uint64_t hash_b(uint64_t base, uint64_t key) { return sm64(base + key); }

__device__ __forceinline__ double sign_of(uint64_t h) { return (h >> 63) ? -1.0 : 1.0; }

// G-SPD: A_ij = s_i s_j c[(i - j) mod n]
__global__ void __launch_bounds__(kNT) k_gen_spd(double* A, int64_t lda, int64_t row0, int64_t m,
                                                 int64_t n, uint64_t seed, const double* table) {
    const uint64_t base4 = sm64(seed ^ (4ULL << 56));
    for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
        const int64_t i = row0 + r;
        const double si = sign_of(hash_b(base4, (uint64_t)i));
        double* row = A + r * lda;
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            int64_t d = i - j;
            if (d < 0) d += n;
            row[j] = si * sign_of(hash_b(base4, (uint64_t)j)) * table[d];
        }
    }
}

// G-DD: h_ij = ((H(seed,0,i*n+j) >> 44) - 2^19) 2^-20 (j != i);
//       A_ii = R_i * (17 (1 + k_i) / 16), R_i = sum_{j != i} |h_ij| (exact in any order).
__global__ void __launch_bounds__(kNT) k_gen_dd(double* A, int64_t lda, int64_t row0, int64_t m,
                                                int64_t n, uint64_t seed, int kd) {
    __shared__ double red[kNT / 32];
    const uint64_t base0 = sm64(seed ^ (0ULL << 56));
    for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
        const int64_t i = row0 + r;
        double* row = A + r * lda;
        double acc = 0.0;
        const uint64_t key0 = (uint64_t)i * (uint64_t)n;
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            double v = 0.0;
            if (j != i) {
                const uint64_t h = hash_b(base0, key0 + (uint64_t)j);
                v = (double)((int64_t)(h >> 44) - 524288) * (1.0 / 1048576.0);
                acc += fabs(v);
            }
            row[j] = v;
        }
        // exact sum: every partial is an integer multiple of 2^-20 below 2^38 units
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double R = 0.0;
            for (int w = 0; w < kNT / 32; ++w) R += red[w];
            const uint64_t k = (hash3(seed, 1, (uint64_t)i) >> 32) % (uint64_t)kd;
            const double factor = (17.0 * (double)(1 + k)) / 16.0;
            row[i] = R * factor;
        }
        __syncthreads();
    }
}

__global__ void k_gen_rhs(double* b, int64_t n, uint64_t seed) {
    const uint64_t base2 = sm64(seed ^ (2ULL << 56));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double u = (double)(hash_b(base2, (uint64_t)i) >> 11) * (1.0 / 9007199254740992.0);
        b[i] = 2.0 * u - 1.0;
    }
}

unsigned row_grid(int64_t m) {
    int64_t g = m < 148 * 16 ? m : 148 * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

int launch_gen_spd(double* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                   const double* table_dev, cudaStream_t st) {
    if (m <= 0) return 0;
    k_gen_spd<<<row_grid(m), kNT, 0, st>>>(A, lda, row0, m, n, seed, table_dev);
    return 1;
}
int launch_gen_dd(double* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                  int kd, cudaStream_t st) {
    if (m <= 0) return 0;
    k_gen_dd<<<row_grid(m), kNT, 0, st>>>(A, lda, row0, m, n, seed, kd);
    return 1;
}
int launch_gen_rhs(double* b, int64_t n, uint64_t seed, cudaStream_t st) {
    unsigned g = (unsigned)((n + 255) / 256);
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    k_gen_rhs<<<g, 256, 0, st>>>(b, n, seed);
    return 1;
}

}  // namespace ks

// NEXT-4: single-precision path.  The paper's experiments
// are single precision and it "tested ... both single precision and
// double precision".  Matrix and vectors are stored and computed in
// binary32 (half the HBM bytes of FP64 per GEMV); the ABI stays FP64 and the
// conversions happen on the device at the boundary.  The iteration itself runs
// in the persistent kernels instantiated for float (ks_persist.cu); this file
// holds the FP32 setup / init / finish kernels, the conversions and the FP32
// generators (entries computed in FP64 exactly as in ks_gen.cu, then rounded to
// nearest float -- the same rounding numpy's float32 cast applies).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ks_device.cuh"
#include "ks_common.cuh"
#include "ks_internal.h"

namespace ks {

namespace {

constexpr int kNT = 256;
using VA = VecArgsT<float>;


// r0 = b (x0 = 0), x = 0, rhat = r0, slots <r0, r0>
__global__ void __launch_bounds__(kNT) k_setup_r_f32(VA a) {
    __shared__ float red[kNT / 32];
    const int64_t m = rows_of(a.L), r0 = a.L.row0[a.L.rank];
    float* rl = a.G_r + (int64_t)a.L.rank * a.L.chunk;
    float acc[1] = {0.0f};
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
        const float r = a.b_full[r0 + i];
        rl[i] = r;
        a.x_loc[i] = 0.0f;
        a.rhat_loc[i] = r;
        acc[0] = fmaf(r, r, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, reinterpret_cast<float*>(a.scr.part), a.scr.ticket, red) && threadIdx.x == 0) {
        rl[a.L.pslot + 0] = acc[0];
        rl[a.L.pslot + 1] = acc[0];
    }
}

__global__ void __launch_bounds__(kNT) k_init_f32(VA a, int bicgstab, double tol, long long maxit,
                                                  long long hist_cap, unsigned long long ebase) {
    __shared__ float red[kNT / 32];
    float acc[1] = {0.0f};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT) {
        if (!bicgstab) a.p_full[j] = a.G_r[gidx(a.L, j)];       // CG: p0 = r0
        const float bj = a.b_full[j];
        acc[0] = fmaf(bj, bj, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, reinterpret_cast<float*>(a.scr.part), a.scr.ticket, red) && threadIdx.x == 0) {
        DevState* st = a.st;
        st->tol = tol;
        st->ebase = ebase;
        st->peer_timeout = 0;
        st->maxit = maxit;
        st->hist_cap = hist_cap;
        st->iters = 0;
        st->half_iter = 0;
        st->done = 0;
        st->status = KS_EMAXIT;
        st->converged = st->breakdown = st->half = st->bzero = 0;
        st->true_rr = -1.0;
        for (int q = 0; q < 4; ++q) st->rho[q] = st->alpha[q] = st->omega[q] = 1.0;
        const float nb = sqrtf(acc[0]);
        st->nb = nb;
        const float rr = slot_sum(a.L, a.G_r, 1);
        if (!bicgstab) st->rho[0] = rr;
        if (nb == 0.0f) {
            st->bzero = 1; st->converged = 1; st->status = KS_OK; st->relres = 0.0; st->done = 1;
        } else {
            const float rel = sqrtf(rr) / nb;
            st->relres = rel;
            if (rel <= (float)tol) { st->converged = 1; st->status = KS_OK; st->done = 1; }
        }
    }
}

__global__ void __launch_bounds__(kNT) k_finish_f32(VA a, int bicgstab) {
    DevState* st = a.st;
    if (bicgstab && !*(volatile int*)&st->done && st->maxit >= 1 && a.peer) {
        const unsigned long long e = *(volatile unsigned long long*)&st->ebase + (unsigned long long)st->maxit;
        if (!wait_flags(a.flags + kPhaseR * kMaxRanks, a.L.P, e)) {
            if (threadIdx.x == 0) { st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1; }
            return;
        }
    }
    if (lead() && !st->done) {
        const long long maxit = st->maxit;
        st->iters = maxit;
        st->status = KS_EMAXIT;
        if (bicgstab && maxit >= 1) {
            const float rel = sqrtf(slot_sum(a.L, a.G_r + (maxit & 1) * a.gpar, 1)) / (float)st->nb;
            if (a.hist && maxit - 1 < st->hist_cap) a.hist[maxit - 1] = rel;
            st->relres = rel;
            if (rel <= (float)st->tol) { st->converged = 1; st->status = KS_OK; }
        }
        st->done = 1;
    }
    if (st->bzero) {
        const int64_t m = rows_of(a.L);
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
            a.x_loc[i] = 0.0f;
    }
}

__global__ void __launch_bounds__(kNT) k_pack_x_f32(VA a) {
    const int64_t m = rows_of(a.L);
    float* xl = a.G_v + (int64_t)a.L.rank * a.L.chunk;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
        xl[i] = a.x_loc[i];
}

__global__ void k_true_res_final_f32(VA a) {
    if (lead()) {
        float s = 0.0f;
        for (int g = 0; g < a.L.P; ++g) s += a.S[g * kScalSlot + 1];
        a.st->true_rr = s;
    }
}

__global__ void k_d2f(const double* src, float* dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (float)src[i];                               // round to nearest
}
__global__ void k_f2d(const float* src, double* dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (double)src[i];
}
__global__ void k_rows_d2f(const double* src, int64_t lds, float* dst, int64_t ldd, int64_t rows,
                           int64_t cols) {
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
        for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) dst[r * ldd + j] = (float)src[r * lds + j];
}

// -- FP32 generators: the FP64 entry rounded to float --------------------------
__device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__global__ void __launch_bounds__(kNT) k_gen_spd_f32(float* A, int64_t lda, int64_t row0, int64_t m,
                                                     int64_t n, uint64_t seed, const double* table) {
    const uint64_t base4 = sm64(seed ^ (4ULL << 56));
    for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
        const int64_t i = row0 + r;
        const double si = (sm64(base4 + (uint64_t)i) >> 63) ? -1.0 : 1.0;
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            int64_t d = i - j;
            if (d < 0) d += n;
            const double sj = (sm64(base4 + (uint64_t)j) >> 63) ? -1.0 : 1.0;
            A[r * lda + j] = (float)(si * sj * table[d]);
        }
    }
}
__global__ void __launch_bounds__(kNT) k_gen_dd_f32(float* A, int64_t lda, int64_t row0, int64_t m,
                                                    int64_t n, uint64_t seed, int kd) {
    __shared__ double red[kNT / 32];
    const uint64_t base0 = sm64(seed ^ (0ULL << 56));
    const uint64_t base1 = sm64(seed ^ (1ULL << 56));
    for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
        const int64_t i = row0 + r;
        double acc = 0.0;
        const uint64_t key0 = (uint64_t)i * (uint64_t)n;
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            double v = 0.0;
            if (j != i) {
                const uint64_t h = sm64(base0 + key0 + (uint64_t)j);
                v = (double)((int64_t)(h >> 44) - 524288) * (1.0 / 1048576.0);
                acc += fabs(v);
            }
            A[r * lda + j] = (float)v;                        // exact: 20-bit dyadic
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double R = 0.0;
            for (int w = 0; w < kNT / 32; ++w) R += red[w];
            const uint64_t k = (sm64(base1 + (uint64_t)i) >> 32) % (uint64_t)kd;
            A[r * lda + i] = (float)(R * ((17.0 * (double)(1 + k)) / 16.0));
        }
        __syncthreads();
    }
}

unsigned grid_for(int64_t len, int num_sms) {
    int64_t g = (len + kNT * 4 - 1) / (kNT * 4);
    if (g < 1) g = 1;
    const int64_t cap = 2LL * num_sms;
    return (unsigned)(g > cap ? cap : g);
}
unsigned flat_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

int launch_setup_r_f32(const VA& a, cudaStream_t st) {
    k_setup_r_f32<<<grid_for(a.L.row0[a.L.rank + 1] - a.L.row0[a.L.rank], a.num_sms), kNT, 0, st>>>(a);
    return 1;
}
int launch_init_f32(const VA& a, int bicgstab, double tol, long long maxit, long long hist_cap,
                    unsigned long long ebase, cudaStream_t st) {
    k_init_f32<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, bicgstab, tol, maxit, hist_cap, ebase);
    return 1;
}
int launch_finish_f32(const VA& a, int bicgstab, cudaStream_t st) {
    k_finish_f32<<<grid_for(a.L.row0[a.L.rank + 1] - a.L.row0[a.L.rank], a.num_sms), kNT, 0, st>>>(a, bicgstab);
    return 1;
}
int launch_pack_x_f32(const VA& a, cudaStream_t st) {
    k_pack_x_f32<<<grid_for(a.L.row0[a.L.rank + 1] - a.L.row0[a.L.rank], a.num_sms), kNT, 0, st>>>(a);
    return 1;
}
int launch_true_res_final_f32(const VA& a, cudaStream_t st) {
    k_true_res_final_f32<<<1, 32, 0, st>>>(a);
    return 1;
}
int launch_d2f(const double* src, float* dst, int64_t n, cudaStream_t st) {
    if (n > 0) k_d2f<<<flat_grid(n), 256, 0, st>>>(src, dst, n);
    return 1;
}
int launch_f2d(const float* src, double* dst, int64_t n, cudaStream_t st) {
    if (n > 0) k_f2d<<<flat_grid(n), 256, 0, st>>>(src, dst, n);
    return 1;
}
int launch_rows_d2f(const double* src, int64_t lds, float* dst, int64_t ldd, int64_t rows, int64_t cols,
                    cudaStream_t st) {
    if (rows > 0) k_rows_d2f<<<(unsigned)(rows < 148 * 16 ? rows : 148 * 16), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
    return 1;
}
int launch_gen_spd_f32(float* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed,
                       const double* table_dev, cudaStream_t st) {
    if (m > 0) k_gen_spd_f32<<<(unsigned)(m < 148 * 16 ? m : 148 * 16), kNT, 0, st>>>(A, lda, row0, m, n, seed, table_dev);
    return 1;
}
int launch_gen_dd_f32(float* A, int64_t lda, int64_t row0, int64_t m, int64_t n, uint64_t seed, int kd,
                      cudaStream_t st) {
    if (m > 0) k_gen_dd_f32<<<(unsigned)(m < 148 * 16 ? m : 148 * 16), kNT, 0, st>>>(A, lda, row0, m, n, seed, kd);
    return 1;
}

}  // namespace ks

// LDG flavour probe (measurement tool): read-only streaming with different cache
// qualifiers / L2 prefetch sizes, same grid as the best LDG probe config (4 CTAs/SM).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int KIND>
__device__ __forceinline__ double2 ld(const double2* p) {
    double2 v;
    if (KIND == 0) {
        v = __ldcs(p);
    } else if (KIND == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    } else if (KIND == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    } else if (KIND == 3) {
        asm volatile("ld.global.cs.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    }
    return v;
}

// 256-bit loads (sm_100): one thread reads 32 B
struct d4 { double a, b, c, d; };
template <int KIND>
__device__ __forceinline__ d4 ld256(const d4* p) {
    d4 v;
    if (KIND == 0)
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d) : "l"(p));
    else if (KIND == 1)
        asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d) : "l"(p));
    else
        asm volatile("ld.global.cs.v4.b64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d) : "l"(p));
    return v;
}
template <int KIND, int U>
__global__ void __launch_bounds__(256) k_read256(const d4* __restrict__ a, int64_t n4, double* out) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        d4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld256<KIND>(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].a + v[u].b + v[u].c + v[u].d;
    }
    for (; i < n4; i += stride) { d4 v = ld256<KIND>(a + i); acc += v.a + v.b + v.c + v.d; }
    if (acc == 1.2345) out[0] = acc;
}
template <int KIND>
static double run256(const void* a, int64_t bytes, int grid, int reps, double* out) {
    const int64_t n4 = bytes / 32;
    k_read256<KIND, 4><<<grid, 256>>>((const d4*)a, n4, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_read256<KIND, 4><<<grid, 256>>>((const d4*)a, n4, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return (double)n4 * 32 * reps / (ms * 1e-3) / 1e9;
}

template <int KIND, int U>
__global__ void __launch_bounds__(256) k_read(const double2* __restrict__ a, int64_t n2, double* out) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld<KIND>(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) { double2 v = ld<KIND>(a + i); acc += v.x + v.y; }
    if (acc == 1.2345) out[0] = acc;
}

template <int KIND>
static double run(const double2* a, int64_t n2, int grid, int reps, double* out) {
    k_read<KIND, 8><<<grid, 256>>>(a, n2, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_read<KIND, 8><<<grid, 256>>>(a, n2, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return (double)n2 * 16 * reps / (ms * 1e-3) / 1e9;
}

extern "C" int ld_probe(double gib, int reps) {
    const int64_t bytes = (int64_t)(gib * (1LL << 30));
    const int64_t n2 = bytes / 16;
    double2* a = nullptr; double* out = nullptr;
    if (cudaMalloc(&a, bytes) != cudaSuccess) return 1;
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, bytes);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"ld.global.cs v2", "nc.L1::no_allocate.L2::256B v2", "nc.L1::no_allocate.L2::128B v2",
                           "cs.L2::256B v2", "256-bit nc.no_alloc.evict_first", "256-bit nc.no_alloc", "256-bit cs"};
    for (int rep = 0; rep < 2; ++rep) {
        for (int g : {4, 8}) {
            const int grid = sms * g;
            double r[7] = {run<0>(a, n2, grid, reps, out), run<1>(a, n2, grid, reps, out), run<2>(a, n2, grid, reps, out),
                           run<3>(a, n2, grid, reps, out), run256<0>(a, bytes, grid, reps, out),
                           run256<1>(a, bytes, grid, reps, out), run256<2>(a, bytes, grid, reps, out)};
            for (int k = 0; k < 7; ++k) printf("grid=%d %-36s %.1f GB/s\n", grid, names[k], r[k]);
        }
    }
    cudaFree(a); cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// K1 -- FP64 row-block GEMV with fused dot epilogue.
//
//   y[i] = sum_{j<n} A_loc[i,j] * x[j]          ("matrix-vector products")
//   optional: y[i] = bsub[i] - (A x)[i]          (residual r0 = b - A x0)
//   optional: *out1 = <w1, y>, *out2 = <y, y>    (fused inner products)
//
// HBM-bound: 0.25 flop/byte, ~20x below the FP64 ridge, so no tensor cores (this
// is not a dense contraction).  Algorithmic bytes per launch = 8*m*n (A read
// once); x (<= 2 MiB) stays L2-resident and is re-read once per row tile.
//
// Variant 1 ("LDG stream"): a CTA of NT threads owns a tile of R rows and a
// contiguous range of 2*NT-column blocks (split-K over S CTAs when there are too
// few tiles to fill 148 SMs).  Thread t streams columns {2t + 2*NT*c} of all R
// rows with 128-bit evict-first loads (ld.global.cs.v2.f64), so every warp
// instruction reads 512 contiguous bytes of one row, and each x element loaded
// (ld.global.nc) is reused for R rows from registers.  Rows are reduced with a
// warp butterfly plus a fixed cross-warp tree; split partials are combined in
// split order by the last-arriving CTA of the tile; tile dot partials are
// combined in tile order by the last-arriving tile -- the result is bitwise
// independent of CTA scheduling.
//
// (Round 1 also had a TMA bulk-ring variant with one producer thread; it measured
// 4.3-6.8 TB/s against this stream's 7.4 and was removed.  The warp-specialised
// TMA pipeline -- producer warp, 2-D tensor-map loads, 40 KiB stages, consumer
// warps -- is the multi-RHS GEMM, ks_multi.cu.)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "ks_device.cuh"
#include "ks_tile.cuh"
#include "ks_internal.h"

namespace ks {

namespace {

constexpr int kNT = 256;  // threads per CTA
constexpr int kNW = kNT / 32;


// Tile epilogue.  `acc` holds the full-row sums (valid in
// every thread).  Returns nothing; handles split-K combine, y store, dots.
template <int R, class T>
__device__ __forceinline__ void gemv_epilogue(const GemvParamsT<T>& p, T (&acc)[R], int64_t tile,
                                              int s, int S, int64_t tiles, T* qpart,
                                              unsigned* tile_ticket, T* dpart,
                                              unsigned* ticket, T* red) {
    __shared__ int s_last;
    const int64_t r0 = tile * R;
    const int nvalid = (int)min((int64_t)R, p.m - r0);
    if (S > 1) {
        if (threadIdx.x == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) qpart[(tile * S + s) * R + r] = acc[r];
            __threadfence();
            unsigned t = atomicAdd(&tile_ticket[tile], 1u);
            s_last = (t == (unsigned)(S - 1));
        }
        __syncthreads();
        if (!s_last) return;
        if (threadIdx.x == 0) tile_ticket[tile] = 0u;
        __threadfence();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T v = T(0);
            for (int q = 0; q < S; ++q) v += __ldcg(qpart + (tile * S + q) * R + r);
            acc[r] = v;
        }
    }
    const bool want_dots = (p.out1 != nullptr) || (p.out2 != nullptr);
    // fused publish: iteration parity and epoch (graph-safe: read from device)
    long long k = 0;
    if (p.pub_P) k = p.koff + (p.kdev ? *p.kdev : 0);
    const int64_t par = k & 1;
    if (threadIdx.x == 0) {
        T d1 = T(0), d2 = T(0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r < nvalid) {
                T yv = acc[r];
                if (p.bsub) yv = p.bsub[r0 + r] - yv;
                if (p.pub_P && p.y_peer[0]) {
                    for (int g = 0; g < p.pub_P; ++g) p.y_peer[g][par * p.ypar + r0 + r] = yv;
                } else {
                    p.y[par * p.y_par + r0 + r] = yv;
                }
                if (p.w1) d1 = fma(p.w1[r0 + r], yv, d1);
                d2 = fma(yv, yv, d2);
            }
        }
        if (want_dots) {
            dpart[tile * 2 + 0] = d1;
            dpart[tile * 2 + 1] = d2;
            // rows stored to peers must be visible system-wide before the flag;
            // tiles that only produced dot partials need the GPU-scope fence of the
            // ticket pattern (the last block releases at system scope)
            if (p.pub_P && p.y_peer[0]) __threadfence_system(); else __threadfence();
            unsigned t = atomicAdd(ticket, 1u);
            s_last = (t == (unsigned)(tiles - 1));
        }
    }
    if (!want_dots) return;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    T v[2] = {T(0), T(0)};
    for (int64_t t = threadIdx.x; t < tiles; t += kNT) {
        v[0] += __ldcg(dpart + t * 2 + 0);
        v[1] += __ldcg(dpart + t * 2 + 1);
    }
    block_sum<kNT, 2>(v, red);
    if (threadIdx.x == 0) {
        if (p.pub_P) {                     // fused C2: partials -> every rank, then the flag
            for (int g = 0; g < p.pub_P; ++g) {
                if (p.out1) p.d_peer[g][par * p.dpar + 0] = v[0];
                if (p.out2) p.d_peer[g][par * p.dpar + 1] = v[1];
            }
            publish_flags(p.f_peer, p.pub_P, *(volatile const unsigned long long*)p.ebase + k);
        } else {
            if (p.out1) *p.out1 = v[0];
            if (p.out2) *p.out2 = v[1];
        }
        *ticket = 0u;
    }
}

template <int R, int U, class T>
__global__ void __launch_bounds__(kNT) k1_gemv_ldg(GemvParamsT<T> p, int S, int64_t tiles,
                                                   T* qpart, unsigned* tile_ticket,
                                                   T* dpart, unsigned* ticket) {
    __shared__ T red[R * kNW];
    if (p.done && *(volatile const int*)p.done) return;
    const int64_t unit = blockIdx.x;
    const int64_t tile = unit / S;
    const int s = (int)(unit % S);
    const int64_t r0 = tile * R;
    const int nvalid = (int)min((int64_t)R, p.m - r0);
    const int64_t ncb = p.ncols / (Vec16<T>::W * kNT);
    const int64_t cb0 = s * ncb / S, cb1 = (s + 1) * ncb / S;

    T acc[R];
    stream_rows<R, U, kNT>(p.A, p.lda, r0, nvalid, p.x, cb0, cb1, acc);
    block_sum<kNT, R>(acc, red);
    gemv_epilogue<R>(p, acc, tile, s, S, tiles, qpart, tile_ticket, dpart, ticket, red);
}

template <int R, int U>
void launch_ldg(const GemvParams& p, const GemvConfig& c, const Scratch& s, int ticket_id, cudaStream_t st) {
    const int64_t tiles = (p.m + R - 1) / R;
    const int64_t grid = tiles * c.splits;
    double* dpart = s.part + (int64_t)ticket_id * kPartStride;
    if (tiles * 2 > kPartStride) dpart = s.qpart + (s.qpart_cap - tiles * 2);
    k1_gemv_ldg<R, U, double><<<(unsigned)grid, kNT, 0, st>>>(p, c.splits, tiles, s.qpart, s.tile_ticket,
                                                              dpart, s.ticket + ticket_id);
}

template <int R>
int launch_rows(const GemvParams& p, const GemvConfig& c, const Scratch& s, int ticket_id,
                cudaStream_t st) {
    const int64_t tiles = (p.m + R - 1) / R;
    const int64_t grid = tiles * c.splits;
    double* dpart = s.part + (int64_t)ticket_id * kPartStride;
    // dots of more than kPartStride/2 tiles go to the split-K scratch tail
    if (tiles * 2 > kPartStride) dpart = s.qpart + (s.qpart_cap - tiles * 2);
    unsigned* ticket = s.ticket + ticket_id;

    // LDG stream: unroll U (tuning sweep; default 16 loads in flight per thread)
    const int U = c.unroll > 0 ? c.unroll : (R >= 16 ? 1 : (R >= 8 ? 2 : 4));
    switch (U) {
        case 1: launch_ldg<R, 1>(p, c, s, ticket_id, st); break;
        case 2: launch_ldg<R, 2>(p, c, s, ticket_id, st); break;
        case 8: launch_ldg<R, 8>(p, c, s, ticket_id, st); break;
        default: launch_ldg<R, 4>(p, c, s, ticket_id, st); break;
    }
    return 1;
}

}  // namespace

GemvConfig choose_gemv(int64_t m, int64_t ncols, int num_sms, int rows_opt, int split_opt,
                       int variant_opt) {
    GemvConfig c;
    (void)variant_opt;
    c.variant = 1;
    // measured on B200 at n = 65536 (profiles/r01_gemv_sweep*.json): LDG R=2/U=4
    // 7.41 TB/s, R=4/U=2 7.40, R=4/U=4 6.84-7.43 (box dependent), R=8 <= 7.18.  The
    // round-1 single-producer-thread TMA variant (6.82 / 6.00 / 4.28 TB/s at R = 16 / 8 /
    // 4) was removed in round 2; the warp-specialised TMA pipeline lives in ks_multi.cu.
    c.rows = (rows_opt == 2 || rows_opt == 4 || rows_opt == 8 || rows_opt == 16) ? rows_opt
                                                                                  : 2;
    c.unroll = 0;
    const int64_t tiles = (m + c.rows - 1) / c.rows;
    const int64_t ncb = std::max<int64_t>(1, ncols / (2 * kNT));   // == ncols / kCW
    if (split_opt > 0) {
        c.splits = (int)std::min<int64_t>(split_opt, ncb);
    } else {
        const int64_t target = 6LL * 2 * num_sms;   // ~6 waves of 2 CTAs/SM
        int64_t S = tiles >= target ? 1 : (target + tiles - 1) / tiles;
        c.splits = (int)std::max<int64_t>(1, std::min<int64_t>({S, ncb, 32}));
    }
    return c;
}

int launch_gemv(const GemvParams& p, const GemvConfig& c, const Scratch& s, int ticket_id,
                int num_sms, cudaStream_t st) {
    (void)num_sms;
    if (p.m <= 0) return 0;
    switch (c.rows) {
        case 2: return launch_rows<2>(p, c, s, ticket_id, st);
        case 4: return launch_rows<4>(p, c, s, ticket_id, st);
        case 8: return launch_rows<8>(p, c, s, ticket_id, st);
        default: return launch_rows<16>(p, c, s, ticket_id, st);
    }
}


// NEXT-4: K1 in FP32 (R = 2 rows x 1024-column blocks of float4 loads; no split-K:
// the FP32 path serves the configs whose row count fills the GPU).
int launch_gemv_f32(const GemvParamsT<float>& p, const Scratch& s, int ticket_id, cudaStream_t st) {
    if (p.m <= 0) return 0;
    constexpr int R = 2;
    const int64_t tiles = (p.m + R - 1) / R;
    float* dpart = reinterpret_cast<float*>(s.part + (int64_t)ticket_id * kPartStride);
    if (tiles * 2 > 2 * kPartStride) dpart = reinterpret_cast<float*>(s.qpart);
    k1_gemv_ldg<R, 4, float><<<(unsigned)tiles, kNT, 0, st>>>(p, 1, tiles, reinterpret_cast<float*>(s.qpart),
                                                              s.tile_ticket, dpart, s.ticket + ticket_id);
    return 1;
}

// ============================================================================
// K1T -- transposed GEMV u = A_loc^T x_loc (length n) for BiCG (
// PAPER.md:33 "performed using system's matrix and its transpose").  Row-major
// A has no contiguous columns, so a CTA owns a block of 512 columns (2 per
// thread, 128-bit evict-first loads, 4 KiB contiguous per row) and a chunk of
// RC rows; it accumulates x_i * A[i, cols] over its rows with UT rows in
// flight.  Row-chunk partials are combined per column block in chunk order by
// the last-arriving CTA (deterministic).  Same 8*m*n algorithmic bytes as K1.
// Output in chunk layout (out[g*chunk + (j - row0[g])]) so P > 1 can
// reduce-scatter it; for P = 1 it is the plain vector.
// ============================================================================
namespace {

// VPT: 16-byte vectors per thread per row (column block = 2 * VPT * NT doubles);
// UT: rows in flight per thread.
template <int VPT, int UT>
__global__ void __launch_bounds__(kNT) k1t_gemv(const double* A, int64_t lda, int64_t m, int64_t n,
                                               const double* x, int64_t rc_rows, int64_t nrc,
                                               double* upart, unsigned* col_ticket, double* out,
                                               Layout L, const int* done, GemvTPub pub) {
    constexpr int CB = 2 * VPT * kNT;
    __shared__ int s_last, s_all;
    if (done && *(volatile const int*)done) return;
    const int64_t ncb = lda / CB;
    const int64_t cb = blockIdx.x % ncb;
    const int64_t rc = blockIdx.x / ncb;
    const int64_t col0 = cb * CB + 2 * threadIdx.x;     // + v * 2 * kNT
    const int64_t i0 = rc * rc_rows;
    const int64_t i1 = min(m, i0 + rc_rows);
    double2 acc[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) acc[v] = make_double2(0.0, 0.0);
    int64_t i = i0;
    for (; i + UT <= i1; i += UT) {
        double2 a[UT][VPT];
        double xi[UT];
#pragma unroll
        for (int u = 0; u < UT; ++u) {
            xi[u] = __ldg(x + i + u);
#pragma unroll
            for (int v = 0; v < VPT; ++v) a[u][v] = ld_stream(A + (i + u) * lda + col0 + v * 2 * kNT);
        }
#pragma unroll
        for (int u = 0; u < UT; ++u)
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                acc[v].x = fma(a[u][v].x, xi[u], acc[v].x);
                acc[v].y = fma(a[u][v].y, xi[u], acc[v].y);
            }
    }
    for (; i < i1; ++i) {
        const double xi = __ldg(x + i);
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            const double2 a = ld_stream(A + i * lda + col0 + v * 2 * kNT);
            acc[v].x = fma(a.x, xi, acc[v].x);
            acc[v].y = fma(a.y, xi, acc[v].y);
        }
    }
    if (nrc > 1) {
#pragma unroll
        for (int v = 0; v < VPT; ++v)
            *reinterpret_cast<double2*>(upart + rc * lda + col0 + v * 2 * kNT) = acc[v];
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned t = atomicAdd(&col_ticket[cb], 1u);
            s_last = (t == (unsigned)(nrc - 1));
        }
        __syncthreads();
        if (!s_last) return;
        if (threadIdx.x == 0) col_ticket[cb] = 0u;
        __threadfence();
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            double2 sum = make_double2(0.0, 0.0);
            for (int64_t q = 0; q < nrc; ++q) {
                const double2 w = __ldcg(reinterpret_cast<const double2*>(upart + q * lda + col0 + v * 2 * kNT));
                sum.x += w.x;
                sum.y += w.y;
            }
            acc[v] = sum;
        }
    }
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        for (int e = 0; e < 2; ++e) {
            const int64_t j = col0 + v * 2 * kNT + e;
            if (j >= n) break;
            int g = 0;
            while (g + 1 < L.P && j >= L.row0[g + 1]) ++g;
            if (pub.P) pub.dst[g][j - L.row0[g]] = e ? acc[v].y : acc[v].x;   // fused reduce-scatter
            else out[(int64_t)g * L.chunk + (j - L.row0[g])] = e ? acc[v].y : acc[v].x;
        }
    }
    if (pub.P) {
        // the last column block to finish releases this rank's slices to every owner
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned t = atomicAdd(pub.ticket, 1u);
            s_all = (t == (unsigned)(ncb - 1));
            if (s_all) {
                *pub.ticket = 0u;
                publish_flags(pub.f_peer, pub.P, pub.epoch);
            }
        }
    }
}

// K1T shape from KS_OPT_GEMVT_SHAPE (vectors per thread per row * 100 + rows in
// flight; validated by ks_set_option, default 204 = the sweep's best).
int shape_vpt(int shape) { const int v = shape / 100; return (v == 1 || v == 2 || v == 4) ? v : 2; }
int shape_ut(int shape) { const int u = shape % 100; return (u == 4 || u == 8 || u == 16) ? u : 4; }

}  // namespace

bool gemv_t_shape_ok(int64_t shape) {
    const int64_t v = shape / 100, u = shape % 100;
    return (v == 1 || v == 2 || v == 4) && (u == 4 || u == 8 || u == 16);
}

int64_t gemv_t_chunk_rows(int64_t m, int64_t lda, int num_sms, int shape) {
    const int64_t ncb = std::max<int64_t>(1, lda / (2 * shape_vpt(shape) * kNT));
    const int64_t target = 6LL * 4 * num_sms;            // ~6 waves of 4 CTAs/SM
    int64_t nrc = (target + ncb - 1) / ncb;
    if (nrc < 1) nrc = 1;
    int64_t rc = (m + nrc - 1) / nrc;
    rc = std::max<int64_t>(16, (rc + 15) / 16 * 16);
    return rc;
}

int launch_gemv_t(const double* A, int64_t lda, int64_t m, int64_t n, const double* x,
                  int64_t rc_rows, double* upart, unsigned* col_ticket, double* out, const Layout& L,
                  const int* done, int shape, cudaStream_t st, const GemvTPub* pub) {
    if (m <= 0) return 0;
    const GemvTPub pb = pub ? *pub : GemvTPub{};
    const int ut = shape_ut(shape);
    const int vpt = (lda % (2 * shape_vpt(shape) * kNT) == 0) ? shape_vpt(shape) : 1;
    const int64_t ncb = lda / (2 * vpt * kNT);
    const int64_t nrc = (m + rc_rows - 1) / rc_rows;
    const unsigned grid = (unsigned)(ncb * nrc);
#define K1T_CASE(V, U)                                                                       \
    if (vpt == V && ut == U) {                                                          \
        k1t_gemv<V, U><<<grid, kNT, 0, st>>>(A, lda, m, n, x, rc_rows, nrc, upart, col_ticket,  \
                                            out, L, done, pb);                                 \
        return 1;                                                                              \
    }
    K1T_CASE(1, 4) K1T_CASE(1, 8) K1T_CASE(1, 16)
    K1T_CASE(2, 4) K1T_CASE(2, 8) K1T_CASE(2, 16)
    K1T_CASE(4, 4) K1T_CASE(4, 8) K1T_CASE(4, 16)
#undef K1T_CASE
    return 0;
}

}  // namespace ks

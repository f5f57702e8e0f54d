// NEXT-3: restarted GMRES(m) (sec.2: "GMRES uses a Gram-Schmidt
// orthogonalization process and requires the storage and computation of an
// increasing amount of information at each iteration.  These difficulties can
// be alleviated by restarting ... The intermediate results are then used as a
// new initial point"; listed as implemented at PAPER.md:78, 109).
//
// Arnoldi with classical Gram-Schmidt applied twice (CGS2): each pass is one
// fused multi-dot over the local basis rows plus one update pass, so a step
// needs 3 scalar exchanges instead of MGS's j+1 (the oracle uses MGS, SPEC.md's
// design decision; both span the same Krylov basis, CGS2 keeps orthogonality to
// O(eps)).  The (m+1) x m Hessenberg matrix, the Givens rotations and the
// least-squares right-hand side g live on the device and are updated by one
// thread; the basis V is sharded by rows like x and r; v_{j+1} is gathered to
// full length for the next GEMV.  Every reduction is fixed-order, so all ranks
// take identical decisions.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ks_device.cuh"
#include "ks_common.cuh"
#include "ks_internal.h"

namespace ks {

namespace {

constexpr int kNT = 256;
constexpr int kNW = kNT / 32;

__device__ __forceinline__ bool done_or_ended(const GmresArgs& g) {
    return *(volatile const int*)&g.a.st->done != 0 || *(volatile const int*)&g.gs->cycle_end != 0;
}
__device__ __forceinline__ double* Vcol(const GmresArgs& g, int i) { return g.V + (int64_t)i * g.ldv; }

// Per-CTA partials of NV dots (vectors V_0..V_{NV-1} against w) are written to
// part[b * kMaxBasis + i]; the last CTA sums them over CTAs in order (one warp
// per vector, lanes striding CTAs, butterfly) and writes out[i].
__device__ void multidot_finish(const GmresArgs& g, const double* vals, int nv, double* out) {
    __shared__ int s_last;
    __shared__ double sred[kMaxBasis];
    const int nb = gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nv; ++i) g.part[(int64_t)blockIdx.x * kMaxBasis + i] = vals[i];
        __threadfence();
        const unsigned t = atomicAdd(g.ticket, 1u);
        s_last = (t == (unsigned)(nb - 1));
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = w; i < nv; i += kNW) {
        double acc = 0.0;
        for (int b = lane; b < nb; b += 32) acc += __ldcg(g.part + (int64_t)b * kMaxBasis + i);
        acc = warp_sum(acc);
        if (lane == 0) sred[i] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nv; ++i) out[i] = sred[i];
        *g.ticket = 0u;
    }
}

// Block partials of <V_i, w> for i < nv, 8 vectors per pass over w; thread 0
// ends up with the block's nv partials in `vals` (shared).
__device__ void block_multidot(const GmresArgs& g, const double* w, int nv, double* vals) {
    __shared__ double red[8 * kNW];
    const int64_t m = rows_of(g.a.L);
    for (int i0 = 0; i0 < nv; i0 += 8) {
        double acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0;
        for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
            const double we = w[e];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (i0 + q < nv) acc[q] = fma(Vcol(g, i0 + q)[e], we, acc[q]);
        }
        block_sum<kNT, 8>(acc, red);
        if (threadIdx.x == 0)
            for (int q = 0; q < 8 && i0 + q < nv; ++q) vals[i0 + q] = acc[q];
    }
}

// CGS pass 1 dots: h_i = <V_i, w>, i <= j, partials of this rank -> hx[rank].
__global__ void __launch_bounds__(kNT) k_gm_dots(GmresArgs g, int j) {
    __shared__ double vals[kMaxBasis];
    if (done_or_ended(g)) return;
    block_multidot(g, g.a.q_loc, j + 1, vals);
    multidot_finish(g, vals, j + 1, g.hx + (int64_t)g.a.L.rank * kMaxBasis);
}

// Apply one CGS pass: h = sum_g hx[g] (rank order), w -= sum_i h_i V_i, H[:, j] += h;
// then the NEXT reduction's partials: pass 2 dots (pass == 1) into hx, or
// ||w||^2 (pass == 2) into hx slot 0.
__global__ void __launch_bounds__(kNT) k_gm_orth(GmresArgs g, int j, int pass) {
    __shared__ double h[kMaxBasis];
    __shared__ double vals[kMaxBasis];
    __shared__ double red[8 * kNW];
    if (done_or_ended(g)) return;
    const Layout& L = g.a.L;
    const int nv = j + 1;
    if (threadIdx.x < nv) {
        double s = 0.0;
        for (int q = 0; q < L.P; ++q) s += g.hx[(int64_t)q * kMaxBasis + threadIdx.x];
        h[threadIdx.x] = s;
    }
    __syncthreads();
    const int64_t m = rows_of(L);
    double* w = g.a.q_loc;
    if (pass == 1) {
        // update, then pass-2 partial dots on the updated elements
        for (int i0 = 0; i0 < nv; i0 += 8) {
            double acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = 0.0;
            for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
                double we;
                if (i0 == 0) {
                    we = w[e];
                    for (int i = 0; i < nv; ++i) we = fma(-h[i], Vcol(g, i)[e], we);
                    w[e] = we;
                } else {
                    we = w[e];
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (i0 + q < nv) acc[q] = fma(Vcol(g, i0 + q)[e], we, acc[q]);
            }
            block_sum<kNT, 8>(acc, red);
            if (threadIdx.x == 0)
                for (int q = 0; q < 8 && i0 + q < nv; ++q) vals[i0 + q] = acc[q];
        }
        if (lead())
            for (int i = 0; i < nv; ++i) g.H[(int64_t)i * g.mres + j] = h[i];
        __syncthreads();
        multidot_finish(g, vals, nv, g.hx + (int64_t)L.rank * kMaxBasis);
    } else {
        double acc[1] = {0.0};
        for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
            double we = w[e];
            for (int i = 0; i < nv; ++i) we = fma(-h[i], Vcol(g, i)[e], we);
            w[e] = we;
            acc[0] = fma(we, we, acc[0]);
        }
        if (lead())
            for (int i = 0; i < nv; ++i) g.H[(int64_t)i * g.mres + j] += h[i];
        block_sum<kNT, 1>(acc, red);
        if (threadIdx.x == 0) vals[0] = acc[0];
        __syncthreads();
        multidot_finish(g, vals, 1, g.hx + (int64_t)L.rank * kMaxBasis);
    }
}

// End of step j (global step k): h_{j+1,j} = ||w||; v_{j+1} = w / h; Givens;
// implicit residual |g_{j+1}| / ||b||; cycle end on convergence (Q1), lucky
// breakdown (h = 0), the last step of the cycle, or maxit.
__global__ void __launch_bounds__(kNT) k_gm_step_end(GmresArgs g, int j, long long k) {
    if (done_or_ended(g)) return;
    const Layout& L = g.a.L;
    DevState* st = g.a.st;
    double nrm2 = 0.0;
    for (int q = 0; q < L.P; ++q) nrm2 += g.hx[(int64_t)q * kMaxBasis];
    const double hn = sqrt(nrm2);
    const int64_t m = rows_of(L);
    double* vn = Vcol(g, j + 1);
    double* gown = g.a.G_r + (int64_t)L.rank * L.chunk;
    if (hn != 0.0) {
        for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
            const double v = g.a.q_loc[e] / hn;
            vn[e] = v;
            gown[e] = v;
        }
    }
    if (lead()) {
        double* H = g.H;
        const int mr = g.mres;
        for (int i = 0; i < j; ++i) {                       // previous rotations
            const double a = H[(int64_t)i * mr + j], c = H[(int64_t)(i + 1) * mr + j];
            H[(int64_t)i * mr + j] = g.cs[i] * a + g.sn[i] * c;
            H[(int64_t)(i + 1) * mr + j] = -g.sn[i] * a + g.cs[i] * c;
        }
        const double a = H[(int64_t)j * mr + j];
        const double den = sqrt(a * a + hn * hn);
        g.cs[j] = a / den;
        g.sn[j] = hn / den;
        H[(int64_t)j * mr + j] = den;
        H[(int64_t)(j + 1) * mr + j] = 0.0;
        g.g[j + 1] = -g.sn[j] * g.g[j];
        g.g[j] = g.cs[j] * g.g[j];
        const double rel = fabs(g.g[j + 1]) / st->nb;
        if (g.a.hist && k - 1 < st->hist_cap) g.a.hist[k - 1] = rel;
        st->relres = rel;
        st->iters = k;
        g.gs->jdone = j + 1;
        const bool conv = rel <= st->tol || hn == 0.0;
        if (conv) g.gs->converged = 1;
        if (conv || j + 1 == g.mres || k >= st->maxit) { g.gs->cycle_end = 1; g.gs->skip = 1; }
    }
}

// v_{j+1} (gathered G_r) -> the full-length GEMV input.
__global__ void __launch_bounds__(kNT) k_gm_vfull(GmresArgs g) {
    if (done_or_ended(g)) return;
    const Layout& L = g.a.L;
    for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < L.n; e += (int64_t)gridDim.x * kNT)
        g.a.p_full[e] = g.a.G_r[gidx(L, e)];
}

// Cycle start: beta = ||b - A x|| (K1 residual partials in S slot 1); test;
// v_0 = r / beta (own rows + G_r own chunk); g = beta e_1.
__global__ void __launch_bounds__(kNT) k_gm_start(GmresArgs g) {
    DevState* st = g.a.st;
    if (*(volatile const int*)&st->done) return;
    const Layout& L = g.a.L;
    double bb = 0.0;
    for (int q = 0; q < L.P; ++q) bb += g.a.S[q * kScalSlot + 1];
    const double beta = sqrt(bb);
    const double rel = beta / st->nb;
    if (rel <= st->tol) {
        if (lead()) { st->relres = rel; st->converged = 1; st->status = KS_OK; st->done = 1; g.gs->skip = 1; }
        return;
    }
    const int64_t m = rows_of(L);
    double* v0 = Vcol(g, 0);
    double* gown = g.a.G_r + (int64_t)L.rank * L.chunk;
    for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
        const double v = g.a.q_loc[e] / beta;
        v0[e] = v;
        gown[e] = v;
    }
    if (lead()) {
        for (int i = 0; i <= g.mres; ++i) g.g[i] = 0.0;
        g.g[0] = beta;
        g.gs->cycle_end = 0;
        g.gs->jdone = 0;
        g.gs->converged = 0;
        g.gs->skip = 0;
        st->relres = rel;
    }
}

// Cycle end: y = H^{-1} g (upper triangular, every CTA redundantly, jdone <= 64);
// x += V y; convergence / maxit decision.
__global__ void __launch_bounds__(kNT) k_gm_cycle_end(GmresArgs g, long long k_enqueued) {
    __shared__ double y[kMaxBasis];
    DevState* st = g.a.st;
    if (*(volatile const int*)&st->done) return;
    const int jd = (int)g.gs->jdone;
    if (threadIdx.x == 0) {
        const int mr = g.mres;
        for (int i = jd - 1; i >= 0; --i) {
            double s = g.g[i];
            for (int l = i + 1; l < jd; ++l) s -= g.H[(int64_t)i * mr + l] * y[l];
            y[i] = s / g.H[(int64_t)i * mr + i];
        }
    }
    __syncthreads();
    const int64_t m = rows_of(g.a.L);
    for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
        double xe = g.a.x_loc[e];
        for (int i = 0; i < jd; ++i) xe = fma(y[i], Vcol(g, i)[e], xe);
        g.a.x_loc[e] = xe;
    }
    if (lead()) {
        if (g.gs->converged) { st->converged = 1; st->status = KS_OK; st->done = 1; }
        else if (st->iters >= st->maxit || k_enqueued >= st->maxit) { st->status = KS_EMAXIT; st->done = 1; }
        g.gs->cycle_end = 0;
        g.gs->skip = 1;          // until the next cycle start
    }
}

__global__ void k_gm_init(GmresArgs g, double tol, long long maxit, long long hist_cap) {
    // ||b||, state; the first cycle's residual comes from the K1 residual launch
    __shared__ double red[kNW];
    double acc[1] = {0.0};
    const Layout& L = g.a.L;
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < L.n; j += (int64_t)gridDim.x * kNT) {
        const double bj = g.a.b_full[j];
        acc[0] = fma(bj, bj, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (threadIdx.x == 0) {
        DevState* st = g.a.st;
        st->nb = sqrt(acc[0]);
        st->tol = tol;
        st->maxit = maxit;
        st->hist_cap = hist_cap;
        st->iters = 0;
        st->half_iter = 0;
        st->status = KS_EMAXIT;
        st->converged = st->breakdown = st->half = 0;
        st->true_rr = -1.0;
        st->peer_timeout = 0;
        st->bzero = st->nb == 0.0;
        st->done = st->bzero;
        if (st->bzero) { st->converged = 1; st->status = KS_OK; st->relres = 0.0; }
        g.gs->cycle_end = 0;
        g.gs->jdone = 0;
        g.gs->converged = 0;
        g.gs->skip = st->done;
    }
}

unsigned grid_for(int64_t len, int num_sms) {
    int64_t b = (len + kNT * 4 - 1) / (kNT * 4);
    if (b < 1) b = 1;
    const int64_t cap = 2LL * num_sms;
    return (unsigned)(b > cap ? cap : b);
}

}  // namespace

int launch_gm_init(const GmresArgs& g, double tol, long long maxit, long long hist_cap, cudaStream_t st) {
    k_gm_init<<<1, kNT, 0, st>>>(g, tol, maxit, hist_cap);   // one CTA: ||b|| in a fixed order
    return 1;
}
int launch_gm_start(const GmresArgs& g, cudaStream_t st) {
    k_gm_start<<<grid_for(g.a.L.row0[g.a.L.rank + 1] - g.a.L.row0[g.a.L.rank], g.a.num_sms), kNT, 0, st>>>(g);
    return 1;
}
int launch_gm_dots(const GmresArgs& g, int j, cudaStream_t st) {
    k_gm_dots<<<grid_for(g.a.L.row0[g.a.L.rank + 1] - g.a.L.row0[g.a.L.rank], g.a.num_sms), kNT, 0, st>>>(g, j);
    return 1;
}
int launch_gm_orth(const GmresArgs& g, int j, int pass, cudaStream_t st) {
    k_gm_orth<<<grid_for(g.a.L.row0[g.a.L.rank + 1] - g.a.L.row0[g.a.L.rank], g.a.num_sms), kNT, 0, st>>>(g, j, pass);
    return 1;
}
int launch_gm_step_end(const GmresArgs& g, int j, long long k, cudaStream_t st) {
    k_gm_step_end<<<grid_for(g.a.L.row0[g.a.L.rank + 1] - g.a.L.row0[g.a.L.rank], g.a.num_sms), kNT, 0, st>>>(g, j, k);
    return 1;
}
int launch_gm_vfull(const GmresArgs& g, cudaStream_t st) {
    k_gm_vfull<<<grid_for(g.a.L.n, g.a.num_sms), kNT, 0, st>>>(g);
    return 1;
}
int launch_gm_cycle_end(const GmresArgs& g, long long k_enqueued, cudaStream_t st) {
    k_gm_cycle_end<<<grid_for(g.a.L.row0[g.a.L.rank + 1] - g.a.L.row0[g.a.L.rank], g.a.num_sms), kNT, 0, st>>>(g, k_enqueued);
    return 1;
}

}  // namespace ks

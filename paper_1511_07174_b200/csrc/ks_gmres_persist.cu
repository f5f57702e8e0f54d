// NEXT-3 + NEXT-2: one restart cycle of GMRES(m) as one persistent
// cooperative kernel.  Same arithmetic as the multi-kernel path (ks_gmres.cu):
// CGS2 Arnoldi, Givens rotations, x += V y at the cycle end; grid barriers replace
// the ~6 kernel boundaries of every Arnoldi step.  Every CTA keeps the running
// least-squares entry g_j and the convergence decision in registers (identical
// everywhere: computed from the same totals), the lead CTA records H, cs, sn, g
// and the history for the back substitution and the host.
//
// P > 1 (NEXT-1, fused exchange): the four collectives of an Arnoldi step (two
// CGS dot vectors, ||w||^2, the v_{j+1} slices) and the cycle start's x slices and
// ||r||^2 are exchanged inside the kernel over NVLink peer memory: the producer
// stores into every rank's exchange buffer, fences, and raises its epoch flag;
// consumers wait for every rank's flag and sum in rank order, so all ranks hold
// bitwise-identical totals.  Exchange s of a solve has epoch ebase + s, s =
// 1 + c (3 + 4m) + {0: x, 1: beta, 2: v_0, 3 + 4j: dots 1, 4 + 4j: dots 2,
// 5 + 4j: norm, 6 + 4j: v_{j+1}} in cycle c; vector slices go through G_r,
// scalars and dot vectors through G_v, alternating by the parity of s (every
// pair of consecutive uses of one buffer half is separated by a completed
// all-rank exchange).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ks_persist.cuh"

namespace ks {

namespace {

using namespace pk;

struct GPArgs {
    PersistArgs<double> P;   // a, A, lda, ncols, bpart (grid x 4), bar
    GmresArgs g;             // V, ldv, mres, H, cs, sn, g, hx (totals), part (grid x kMaxBasis)
    unsigned long long ebase;   // P > 1: epoch of exchange s is ebase + s
};

// ---- fused exchange (P > 1) ---------------------------------------------------
__device__ bool xwait(const VecArgs& a, int ph, unsigned long long e) {
    const bool ok = wait_flags(a.flags + ph * kMaxRanks, a.L.P, e);
    if (!ok && threadIdx.x == 0) { a.st->peer_timeout = 1; a.st->status = KS_ENCCL; a.st->done = 1; }
    return ok;
}
__device__ void xflag(const VecArgs& a, int ph, unsigned long long e) {
    unsigned long long* f[kMaxRanks];
    for (int g = 0; g < a.L.P; ++g) f[g] = a.pp.flags[g] + ph * kMaxRanks + a.L.rank;
    publish_flags(f, a.L.P, e);
}
// nv per-rank totals (src, read by the lead) -> rank-ordered global sums in dst
// (shared memory) on every CTA of every rank.  Slot: G_v[parity][rank * chunk + i].
__device__ bool xch_sums(const VecArgs& a, const double* src, int nv, unsigned long long s, unsigned long long e,
                         double* dst) {
    const Layout& L = a.L;
    const int64_t off = (int64_t)(s & 1) * a.gpar;
    if (lead()) {
        for (int i = 0; i < nv; ++i) {
            const double v = __ldcg(src + i);
            for (int g = 0; g < L.P; ++g) a.pp.G_v[g][off + (int64_t)L.rank * L.chunk + i] = v;
        }
        xflag(a, kPhaseS, e);
    }
    if (!xwait(a, kPhaseS, e)) return false;
    if (threadIdx.x < nv) {
        double t = 0.0;
        for (int g = 0; g < L.P; ++g) t += __ldcg(a.G_v + off + (int64_t)g * L.chunk + threadIdx.x);
        dst[threadIdx.x] = t;
    }
    __syncthreads();
    return true;
}
// Every rank's slice src[0, m) -> full-length dst[0, n) on every rank (via G_r).
__device__ bool xch_vec(const PersistArgs<double>& P, const double* src, unsigned long long s, unsigned long long e,
                        double* dst) {
    const VecArgs& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t m = rows_of(L), off = (int64_t)(s & 1) * a.gpar;
    const int64_t tid0 = (int64_t)blockIdx.x * kNT + threadIdx.x, gstride = (int64_t)gridDim.x * kNT;
    for (int64_t i = tid0; i < m; i += gstride) {
        const double v = src[i];
        for (int g = 0; g < L.P; ++g) a.pp.G_r[g][off + (int64_t)L.rank * L.chunk + i] = v;
    }
    if (tid0 < m) __threadfence_system();   // only threads that stored remotely
    if (!grid_sync(P.bar, st)) return false;
    if (lead()) xflag(a, kPhaseR, e);
    if (!xwait(a, kPhaseR, e)) return false;
    for (int64_t j = tid0; j < L.n; j += gstride) {
        int o;
        dst[j] = __ldcg(a.G_r + off + gidx_owner(L, j, &o));
    }
    return grid_sync(P.bar, st);
}

__device__ __forceinline__ double* Vc(const GmresArgs& g, int i) { return g.V + (int64_t)i * g.ldv; }

// CTA partials of <V_i, w>, i < nv -> part[blockIdx * kMaxBasis + i] (8 vectors per pass).
__device__ void cta_dots(const GmresArgs& g, const double* w, int64_t m, int nv, double* red) {
    for (int i0 = 0; i0 < nv; i0 += 8) {
        double acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0;
        for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < m; e += (int64_t)gridDim.x * kNT) {
            const double we = w[e];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (i0 + q < nv) acc[q] = fma(Vc(g, i0 + q)[e], we, acc[q]);
        }
        block_sum<kNT, 8>(acc, red);
        if (threadIdx.x == 0)
            for (int q = 0; q < 8 && i0 + q < nv; ++q) g.part[(int64_t)blockIdx.x * kMaxBasis + i0 + q] = acc[q];
    }
}

// CTA i (< nv) sums part[*][i] over CTAs in CTA order -> tot[i].
__device__ void reduce_dots(const GmresArgs& g, int nv, double* red) {
    if ((int)blockIdx.x >= nv) return;
    double acc[1] = {0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kNT)
        acc[0] += __ldcg(g.part + (int64_t)b * kMaxBasis + blockIdx.x);
    block_sum<kNT, 1>(acc, red);
    if (threadIdx.x == 0) g.hx[blockIdx.x] = acc[0];
}

template <int kR, int kU>
__global__ void __launch_bounds__(kNT, 4) k_gm_cycle(GPArgs A) {
    __shared__ double red[8 * kNW];
    __shared__ double h1[kMaxBasis], h2[kMaxBasis];
    __shared__ double s_rel, s_hn, s_x[1];
    const VecArgs& a = A.P.a;
    const GmresArgs& g = A.g;
    const Layout& L = a.L;
    DevState* st = a.st;
    if (is_done(st)) return;
    const int64_t m = rows_of(L);
    const int64_t tid0 = (int64_t)blockIdx.x * kNT + threadIdx.x, gstride = (int64_t)gridDim.x * kNT;
    long long k = *(volatile const long long*)&st->iters;   // inner steps completed so far
    const long long maxit = st->maxit;
    const double nb = st->nb, tol = st->tol;
    const bool peer = a.peer != 0;
    // exchange sequence number of this cycle's first exchange (see the header)
    const unsigned long long sq0 = 1ull + (unsigned long long)(k / g.mres) * (3ull + 4ull * (unsigned long long)g.mres);
    // ---- cycle start: r = b - A x, beta, v_0 = r / beta, g = beta e_1
    if (peer) {
        if (!xch_vec(A.P, a.x_loc, sq0, A.ebase + sq0, a.s_full)) return;
    } else {
        for (int64_t i = tid0; i < m; i += gstride) a.s_full[i] = a.x_loc[i];
        if (!grid_sync(A.P.bar, st)) return;
    }
    double d1, d2;
    gemv_phase<kR, kU>(A.P, a.s_full, a.q_loc, (const double*)nullptr, d1, d2, red, a.b_full + L.row0[L.rank],
                       (int)blockIdx.x, (int)gridDim.x);
    if (threadIdx.x == 0) A.P.bpart[blockIdx.x * 4 + 1] = d2;
    if (!grid_sync(A.P.bar, st)) return;
    double bt[1];
    grid_total<1>(A.P.bpart, 1, bt, red);
    if (peer) {
        if (lead()) g.hx[0] = bt[0];
        if (!xch_sums(a, g.hx, 1, sq0 + 1, A.ebase + sq0 + 1, s_x)) return;
        bt[0] = s_x[0];
    }
    const double beta = sqrt(bt[0]);
    if (beta / nb <= tol || k >= maxit) {
        if (lead()) {
            st->relres = beta / nb;
            if (beta / nb <= tol) { st->converged = 1; st->status = KS_OK; }
            else st->status = KS_EMAXIT;
            st->done = 1;
        }
        return;
    }
    for (int64_t i = tid0; i < m; i += gstride) {
        const double v = a.q_loc[i] / beta;
        Vc(g, 0)[i] = v;
        if (!peer) a.p_full[i] = v;
    }
    if (peer) {
        if (!xch_vec(A.P, Vc(g, 0), sq0 + 2, A.ebase + sq0 + 2, a.p_full)) return;
    } else {
        if (!grid_sync(A.P.bar, st)) return;
    }
    double gcur = beta;                      // running g_j (same in every CTA)
    int jd = 0;
    bool conv = false;
    for (int j = 0; j < g.mres && k < maxit; ++j) {
        const unsigned long long sj = sq0 + 3 + 4ull * (unsigned long long)j;
        const int nv = j + 1;
        gemv_phase<kR, kU>(A.P, a.p_full, a.q_loc, (const double*)nullptr, d1, d2, red, (const double*)nullptr, (int)blockIdx.x,
                           (int)gridDim.x);   // w = A v_j
        if (!grid_sync(A.P.bar, st)) return;
        cta_dots(g, a.q_loc, m, nv, red);                                 // CGS pass 1
        if (!grid_sync(A.P.bar, st)) return;
        reduce_dots(g, nv, red);
        if (!grid_sync(A.P.bar, st)) return;
        if (peer) {
            if (!xch_sums(a, g.hx, nv, sj, A.ebase + sj, h1)) return;
        } else {
            if (threadIdx.x < nv) h1[threadIdx.x] = __ldcg(g.hx + threadIdx.x);
            __syncthreads();
        }
        for (int64_t e = tid0; e < m; e += gstride) {                     // w -= V h1
            double we = a.q_loc[e];
            for (int i = 0; i < nv; ++i) we = fma(-h1[i], Vc(g, i)[e], we);
            a.q_loc[e] = we;
        }
        cta_dots(g, a.q_loc, m, nv, red);                                 // CGS pass 2 (same elements,
        if (!grid_sync(A.P.bar, st)) return;                              //  same thread: no race)
        reduce_dots(g, nv, red);
        if (!grid_sync(A.P.bar, st)) return;
        if (peer) {
            if (!xch_sums(a, g.hx, nv, sj + 1, A.ebase + sj + 1, h2)) return;
        } else {
            if (threadIdx.x < nv) h2[threadIdx.x] = __ldcg(g.hx + threadIdx.x);
            __syncthreads();
        }
        double nacc[1] = {0.0};
        for (int64_t e = tid0; e < m; e += gstride) {                     // w -= V h2, ||w||^2
            double we = a.q_loc[e];
            for (int i = 0; i < nv; ++i) we = fma(-h2[i], Vc(g, i)[e], we);
            a.q_loc[e] = we;
            nacc[0] = fma(we, we, nacc[0]);
        }
        block_sum<kNT, 1>(nacc, red);
        if (threadIdx.x == 0) A.P.bpart[blockIdx.x * 4 + 0] = nacc[0];
        if (!grid_sync(A.P.bar, st)) return;
        double nt[1];
        grid_total<1>(A.P.bpart, 0, nt, red);
        if (peer) {
            if (lead()) g.hx[0] = nt[0];
            if (!xch_sums(a, g.hx, 1, sj + 2, A.ebase + sj + 2, s_x)) return;
            nt[0] = s_x[0];
        }
        const double hn = sqrt(nt[0]);
        if (hn != 0.0) {
            for (int64_t e = tid0; e < m; e += gstride) {
                const double v = a.q_loc[e] / hn;
                Vc(g, j + 1)[e] = v;
                if (!peer) a.p_full[e] = v;
            }
        }
        if (threadIdx.x == 0) {            // Givens on column j (every CTA, identical)
            const int mr = g.mres;
            double col[kMaxBasis];
            for (int i = 0; i < nv; ++i) col[i] = h1[i] + h2[i];
            for (int i = 0; i < j; ++i) {
                const double c = __ldcg(g.cs + i), s = __ldcg(g.sn + i);
                const double x0 = col[i], x1 = col[i + 1];
                col[i] = c * x0 + s * x1;
                col[i + 1] = -s * x0 + c * x1;
            }
            const double den = sqrt(col[j] * col[j] + hn * hn);
            const double cj = col[j] / den, sj2 = hn / den;
            const double gj1 = -sj2 * gcur;
            const double gj = cj * gcur;
            s_rel = fabs(gj1) / nb;
            s_hn = hn;
            if (blockIdx.x == 0) {
                for (int i = 0; i < j; ++i) g.H[(int64_t)i * mr + j] = col[i];
                g.H[(int64_t)j * mr + j] = den;
                g.H[(int64_t)(j + 1) * mr + j] = 0.0;
                g.cs[j] = cj;
                g.sn[j] = sj2;
                g.g[j] = gj;
                g.g[j + 1] = gj1;
                if (a.hist && k < st->hist_cap) a.hist[k] = s_rel;
                st->relres = s_rel;
                st->iters = k + 1;
            }
            red[0] = gj1;
        }
        __syncthreads();
        gcur = red[0];
        ++k;
        jd = j + 1;
        conv = s_rel <= tol || s_hn == 0.0;
        if (conv || j + 1 == g.mres || k >= maxit) break;
        if (peer) {                                                       // v_{j+1} slices -> p_full
            if (!xch_vec(A.P, Vc(g, j + 1), sj + 3, A.ebase + sj + 3, a.p_full)) return;
        } else {
            if (!grid_sync(A.P.bar, st)) return;
        }
    }
    if (!grid_sync(A.P.bar, st)) return;   // H, g complete
    // ---- cycle end: y = H^{-1} g (every CTA), x += V y
    __shared__ double y[kMaxBasis];
    if (threadIdx.x == 0) {
        const int mr = g.mres;
        for (int i = jd - 1; i >= 0; --i) {
            double s = __ldcg(g.g + i);
            for (int l = i + 1; l < jd; ++l) s -= __ldcg(g.H + (int64_t)i * mr + l) * y[l];
            y[i] = s / __ldcg(g.H + (int64_t)i * mr + i);
        }
    }
    __syncthreads();
    for (int64_t e = tid0; e < m; e += gstride) {
        double xe = a.x_loc[e];
        for (int i = 0; i < jd; ++i) xe = fma(y[i], Vc(g, i)[e], xe);
        a.x_loc[e] = xe;
    }
    if (lead()) {
        if (conv) { st->converged = 1; st->status = KS_OK; st->done = 1; }
        else if (k >= maxit) { st->status = KS_EMAXIT; st->done = 1; }
    }
}

}  // namespace

int launch_gm_cycle_persist(const GmresArgs& g, const double* A, int64_t lda, int64_t ncols, double* bpart,
                            unsigned* bar, int grid, unsigned long long ebase, cudaStream_t st) {
    GPArgs args;
    args.ebase = ebase;
    args.P.a = g.a;
    args.P.A = A;
    args.P.lda = lda;
    args.P.ncols = ncols;
    args.P.bpart = bpart;
    args.P.bar = bar;
    args.P.k0 = 0;
    args.P.k1 = 0;
    args.g = g;
    void* params[] = {&args};
    cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned long long), st);   // grid_sync counter
    if (e != cudaSuccess) return -(int)e;
    e = cudaLaunchCooperativeKernel((const void*)k_gm_cycle<2, 4>, dim3((unsigned)grid), dim3(kNT),
                                                params, 0, st);
    return e == cudaSuccess ? 1 : -(int)e;
}

int gm_persist_grid(int num_sms, int64_t m) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_gm_cycle<2, 4>, kNT, 0);
    if (per_sm < 1) per_sm = 1;
    const int64_t cap = (int64_t)per_sm * num_sms;
    const int64_t tiles = (m + 1) / 2;
    int64_t gsz = tiles < num_sms ? num_sms : tiles;
    if (gsz > cap) gsz = cap;
    if (gsz < kMaxBasis) gsz = kMaxBasis;      // one CTA per basis vector in reduce_dots
    return (int)gsz;
}

}  // namespace ks

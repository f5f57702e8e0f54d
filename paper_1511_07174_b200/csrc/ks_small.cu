// NEXT-2, second stage: the small-n kernels.
//
// For an L2-resident system (C1: n = 1024, 8 MiB) an iteration is a chain of
// grid-wide dependencies, each ~2 us (barrier + reading the CTA partials), with
// ~1 us of GEMV between them.  The persistent kernels of ks_persist.cu pay one
// barrier per reduction plus one per full-length vector the GEMV reads (CG 3 per
// iteration, BiCGSTAB 5).  Here every CTA keeps the full-length vectors in its
// own shared memory and updates them redundantly (n <= a few thousand: a few KB
// of L2 reads per CTA), so only the reductions that need every CTA's GEMV rows
// remain grid-wide:
//   CG        : 1 barrier  (sigma = <p, A p>); r, rho' = <r, r>, p computed per CTA
//   BiCGSTAB  : 2 barriers (<rhat, v>; <t, s>, <t, t>); s, ||s||, r, rho, p per CTA
// Same recurrences as the other paths (SURVEY.md sec.8(c).3/.4, rows A1-A5 and
// B1-B8); the per-CTA full-length dots are block reductions over the whole
// vector in a fixed thread mapping, so every CTA obtains the same bits.
// Buffers whose readers may lag one iteration behind their writers (GEMV outputs,
// CTA partials) are double-buffered by iteration parity; the single barrier per
// reduction then orders everything.  The global copies of r, p, v (and G_r's
// partial slots) are refreshed every iteration by their owning threads, so a
// later launch (the next poll batch) or the finish kernels see current state --
// each only after the iteration's first grid barrier, since before it a slow CTA
// may still be loading the previous values at the start of its launch.
// k_cg_small / k_bs_small run on one GPU; k_cg_small_peer / k_bs_small_peer are the
// variants for P > 1 GPUs with the fused exchange (see their comments).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ks_device.cuh"
#include "ks_internal.h"
#include "ks_tile.cuh"
#include "ks_persist.cuh"

namespace ks {

namespace {

using namespace pk;

constexpr int kSlots = 8;   // CTA partial slots per parity pair: [par * 4 + q]

// Block-wide sum of K values over a full-length loop, identical in every CTA.
template <int K, class T>
__device__ __forceinline__ void cta_total(T (&v)[K], T* red) { block_sum<kNT, K>(v, red); }

// GEMV over this CTA's round-robin tiles with x in shared memory; thread 0
// accumulates <w, y> (w in shared memory) and <y, y> over its rows in tile order.
template <int kR, int kU, class T>
__device__ void gemv_smem(const PersistArgs<T>& P, int64_t m, const T* xs, T* y, const T* ws, T& d1, T& d2,
                          T* red) {
    const int64_t tiles = (m + kR - 1) / kR;
    const int64_t ncb = P.ncols / (Vec16<T>::W * kNT);
    d1 = T(0);
    d2 = T(0);
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t r0 = tile * kR;
        const int nvalid = (int)min((int64_t)kR, m - r0);
        T acc[kR];
        stream_rows<kR, kU, kNT, T, true>(P.A, P.lda, r0, nvalid, xs, 0, ncb, acc);
        block_sum<kNT, kR>(acc, red);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                if (r < nvalid) {
                    y[r0 + r] = acc[r];
                    d1 = fma(ws[r0 + r], acc[r], d1);
                    d2 = fma(acc[r], acc[r], d2);
                }
            }
        }
    }
}

// ------------------------------------------------------------------ CG (A1-A5)
template <class T, int kR, int kU>
__global__ void __launch_bounds__(kNT, 2) k_cg_small(PersistArgs<T> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sp = reinterpret_cast<T*>(smem_raw);   // p (ncols, zero padded)
    T* sr = sp + P.ncols;                     // r (n)
    __shared__ T red[(kR > 2 ? kR : 2) * kNW];
    const VecArgsT<T>& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t n = L.n;
    const int64_t gstride = (int64_t)gridDim.x * kNT;
    const int64_t tid0 = (int64_t)blockIdx.x * kNT + threadIdx.x;
    if (is_done(st)) return;
    {
        const T* rin = par_ptr(a.G_r, a.gpar, P.k0 - 1);
        for (int64_t j = threadIdx.x; j < P.ncols; j += kNT) {
            sp[j] = j < n ? a.p_full[j] : T(0);
            if (j < n) sr[j] = rin[j];
        }
    }
    T rho = (T)st->rho[(P.k0 - 1) & 3];
    __syncthreads();
    for (long long k = P.k0; k <= P.k1; ++k) {
        // A1: q = A p (parity buffer), sigma partial
        T* q = (k & 1) ? a.q_loc : a.s_full;
        T d1, d2;
        gemv_smem<kR, kU>(P, n, sp, q, sp, d1, d2, red);
        if (threadIdx.x == 0) P.bpart[blockIdx.x * kSlots + (k & 1) * 4 + 0] = d1;
        if (!grid_sync(P.bar, st)) return;
        T sig[1] = {T(0)};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kNT)
            sig[0] += __ldcg(P.bpart + (int64_t)b * kSlots + (k & 1) * 4 + 0);
        cta_total<1>(sig, red);
        const T sigma = sig[0];
        if (!(sigma > T(0))) {                              // Q9
            if (lead()) { st->status = KS_ENOTSPD; st->iters = k - 1; st->done = 1; }
            return;
        }
        const T alpha = rho / sigma;
        // A3: x += alpha p (owned rows); r -= alpha q and rho' = <r, r> (every CTA, full n)
        for (int64_t i = tid0; i < n; i += gstride) a.x_loc[i] = fma(alpha, sp[i], a.x_loc[i]);
        T acc[1] = {T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T r = fma(-alpha, __ldcg(q + j), sr[j]);
            sr[j] = r;
            acc[0] = fma(r, r, acc[0]);
        }
        cta_total<1>(acc, red);
        const T rho1 = acc[0];
        const T rel = sqrt(rho1) / (T)st->nb;
        T* rout = par_ptr(a.G_r, a.gpar, k);
        for (int64_t i = tid0; i < n; i += gstride) rout[i] = sr[i];
        if (lead()) {
            put_hist(st, a.hist, k - 1, rel);
            rout[L.pslot + 1] = rho1;
            st->relres = rel; st->iters = k; st->alpha[k & 3] = alpha;
        }
        if (rel <= (T)st->tol) {
            if (lead()) { st->converged = 1; st->status = KS_OK; st->done = 1; }
            return;
        }
        // A5: p = r + beta p (every CTA, full n)
        const T beta = rho1 / rho;
        for (int64_t j = threadIdx.x; j < n; j += kNT) sp[j] = fma(beta, sp[j], sr[j]);
        __syncthreads();
        for (int64_t i = tid0; i < n; i += gstride) a.p_full[i] = sp[i];
        if (lead()) st->rho[k & 3] = rho1;
        rho = rho1;
    }
}

// ------------------------------------------- CG on P > 1 GPUs (fused exchange)
// Allgather-only schedule on the small-n kernel:
// each rank computes its rows of q = A p and stores them into every rank's G_v
// (parity k) -- the one exchange of the iteration; then every CTA of every rank
// forms sigma = <p, q>, r -= alpha q, rho' = <r, r> and p = r + beta p over the full
// length in its own shared memory.  The full-length sums run in one fixed order,
// so every CTA of every rank takes the same decisions.  One grid barrier and one
// exchange per iteration (the general fused kernels: three barriers, two
// exchanges).
template <class T, int kR, int kU>
__global__ void __launch_bounds__(kNT, 2) k_cg_small_peer(PersistArgs<T> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sp = reinterpret_cast<T*>(smem_raw);   // p (ncols, zero padded)
    T* sr = sp + P.ncols;                     // r (n)
    T* sq = sr + P.ncols;                     // gathered q (n)
    __shared__ T red[(kR > 2 ? kR : 2) * kNW];
    const VecArgsT<T>& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t n = L.n, m = rows_of(L), r0 = L.row0[L.rank];
    const int64_t gstride = (int64_t)gridDim.x * kNT;
    const int64_t tid0 = (int64_t)blockIdx.x * kNT + threadIdx.x;
    if (is_done(st)) return;
    {
        const T* rin = par_ptr(a.G_r, a.gpar, P.k0 - 1);
        for (int64_t j = threadIdx.x; j < P.ncols; j += kNT) {
            sp[j] = j < n ? a.p_full[j] : T(0);
            if (j < n) sr[j] = rin[gidx(L, j)];
        }
    }
    T rho = (T)st->rho[(P.k0 - 1) & 3];
    __syncthreads();
    const int64_t tiles = (m + kR - 1) / kR;
    const int64_t ncb = P.ncols / (Vec16<T>::W * kNT);
    for (long long k = P.k0; k <= P.k1; ++k) {
        // A1 + A4': this rank's rows of q = A p, stored into every rank's G_v (parity k)
        const int64_t qo = (k & 1) * a.gpar + (int64_t)L.rank * L.chunk;
        bool pushed = false;
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int64_t t0 = tile * kR;
            const int nvalid = (int)min((int64_t)kR, m - t0);
            T acc[kR];
            stream_rows<kR, kU, kNT, T, true>(P.A, P.lda, t0, nvalid, sp, 0, ncb, acc);
            block_sum<kNT, kR>(acc, red);
            if (threadIdx.x == 0) {
                for (int r = 0; r < nvalid; ++r)
                    for (int g = 0; g < L.P; ++g) a.pp.G_v[g][qo + t0 + r] = acc[r];
                pushed = true;
            }
        }
        if (pushed) __threadfence_system();
        if (!grid_sync(P.bar, st)) return;
        if (lead()) flags_out(a, kPhaseV, k);
        if (!wait_ph(a, kPhaseV, k)) return;
        // A2: sigma = <p, q> over the full length (every CTA; same order everywhere)
        const T* qg = par_ptr(a.G_v, a.gpar, k);
        T sig[1] = {T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T qj = __ldcg(qg + gidx(L, j));
            sq[j] = qj;
            sig[0] = fma(sp[j], qj, sig[0]);
        }
        cta_total<1>(sig, red);
        const T sigma = sig[0];
        if (!(sigma > T(0))) {                              // Q9
            if (lead()) { st->status = KS_ENOTSPD; st->iters = k - 1; st->done = 1; }
            return;
        }
        const T alpha = rho / sigma;
        // A3: x += alpha p (own rows); r -= alpha q, rho' = <r, r> (full length)
        for (int64_t i = tid0; i < m; i += gstride) a.x_loc[i] = fma(alpha, sp[r0 + i], a.x_loc[i]);
        T acc[1] = {T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T r = fma(-alpha, sq[j], sr[j]);
            sr[j] = r;
            acc[0] = fma(r, r, acc[0]);
        }
        cta_total<1>(acc, red);
        const T rho1 = acc[0];
        const T rel = sqrt(rho1) / (T)st->nb;
        T* rout = par_ptr(a.G_r, a.gpar, k);              // this rank's full copy of r
        for (int64_t j = tid0; j < n; j += gstride) rout[gidx(L, j)] = sr[j];
        if (lead()) {
            put_hist(st, a.hist, k - 1, rel);
            for (int g = 0; g < L.P; ++g) rout[(int64_t)g * L.chunk + L.pslot + 1] = g == 0 ? rho1 : T(0);
            st->relres = rel; st->iters = k; st->alpha[k & 3] = alpha;
        }
        if (rel <= (T)st->tol) {
            if (lead()) { st->converged = 1; st->status = KS_OK; st->done = 1; }
            return;
        }
        // A5: p = r + beta p (full length, shared memory)
        const T beta = rho1 / rho;
        for (int64_t j = threadIdx.x; j < n; j += kNT) sp[j] = fma(beta, sp[j], sr[j]);
        __syncthreads();
        for (int64_t i = tid0; i < n; i += gstride) a.p_full[i] = sp[i];
        if (lead()) st->rho[k & 3] = rho1;
        rho = rho1;
    }
}

// --------------------------------------- BiCGSTAB on P > 1 GPUs (fused exchange)
// Allgather-only BiCGSTAB on the small-n kernel: the two GEMV outputs (v rows,
// t rows) are the iteration's only exchanges (into every rank's G_v / G_r, parity
// i); everything else -- <rhat, v>, s, ||s||, <t, s>, <t, t>, r, <rhat, r>, <r, r>,
// p -- is formed over the full length in every CTA's shared memory, in one fixed
// order.  Two exchanges and two grid barriers per iteration (general fused
// kernels: three and five).  rhat (full length) is kept in shared memory and, for
// later launches of the same solve, in s_full.  The test of the last iteration of
// the solve is made in-kernel (the general path defers it to k_finish).
template <class T, int kR, int kU>
__global__ void __launch_bounds__(kNT, 1) k_bs_small_peer(PersistArgs<T> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sp = reinterpret_cast<T*>(smem_raw);   // p (ncols, zero padded)
    T* ss = sp + P.ncols;                     // r -> s -> r (ncols, zero padded)
    T* sv = ss + P.ncols;                     // v (n)
    T* sh = sv + P.ncols;                     // rhat (n)
    __shared__ T red[(kR > 2 ? kR : 2) * kNW];
    const VecArgsT<T>& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t n = L.n, m = rows_of(L), r0 = L.row0[L.rank];
    const int64_t gstride = (int64_t)gridDim.x * kNT;
    const int64_t tid0 = (int64_t)blockIdx.x * kNT + threadIdx.x;
    if (is_done(st)) return;
    const T* rin = par_ptr(a.G_r, a.gpar, P.k0 - 1);
    for (int64_t j = threadIdx.x; j < P.ncols; j += kNT) {
        sp[j] = j < n ? a.p_full[j] : T(0);
        ss[j] = j < n ? rin[gidx(L, j)] : T(0);
        if (j < n) {
            sv[j] = a.v_full[j];
            sh[j] = P.k0 == 1 ? ss[j] : a.s_full[j];      // rhat = r0 (Q7)
        }
    }
    if (P.k0 == 1)
        for (int64_t j = tid0; j < n; j += gstride) a.s_full[j] = rin[gidx(L, j)];
    T rho = slot_sum(L, rin, 0), rr = slot_sum(L, rin, 1);
    T rho_prev = (T)st->rho[(P.k0 - 1) & 3], alpha_prev = (T)st->alpha[(P.k0 - 1) & 3];
    T omega_prev = (T)st->omega[(P.k0 - 1) & 3];
    const long long maxit = st->maxit;
    __syncthreads();
    const int64_t tiles = (m + kR - 1) / kR;
    const int64_t ncb = P.ncols / (Vec16<T>::W * kNT);
    // this rank's rows of y = A x (x in shared memory) into slot `off` of every rank's G
    auto gemv_push = [&](const T* xs, T* const* G, int64_t off) {
        bool pushed = false;
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int64_t t0 = tile * kR;
            const int nvalid = (int)min((int64_t)kR, m - t0);
            T acc[kR];
            stream_rows<kR, kU, kNT, T, true>(P.A, P.lda, t0, nvalid, xs, 0, ncb, acc);
            block_sum<kNT, kR>(acc, red);
            if (threadIdx.x == 0) {
                for (int r = 0; r < nvalid; ++r)
                    for (int g = 0; g < L.P; ++g) G[g][off + t0 + r] = acc[r];
                pushed = true;
            }
        }
        if (pushed) __threadfence_system();
    };
    for (long long i = P.k0; i <= P.k1; ++i) {
        // B8 (test of i-1) + B1
        T rel = T(0);
        if (i >= 2) {
            rel = sqrt(rr) / (T)st->nb;
            if (rel <= (T)st->tol) {
                if (lead()) {
                    put_hist(st, a.hist, i - 2, rel);
                    st->relres = rel; st->iters = i - 1; st->converged = 1; st->status = KS_OK; st->done = 1;
                }
                return;
            }
        }
        if (rho == T(0) || !isfinite(rho)) {
            if (lead()) {
                if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
                st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1;
            }
            return;
        }
        if (i == 1) {
            for (int64_t j = threadIdx.x; j < n; j += kNT) sp[j] = ss[j];
        } else {
            const T beta = (rho / rho_prev) * (alpha_prev / omega_prev);
            for (int64_t j = threadIdx.x; j < n; j += kNT) sp[j] = fma(beta, fma(-omega_prev, sv[j], sp[j]), ss[j]);
        }
        if (lead()) {
            if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
            st->rho[i & 3] = rho;
            st->iters = i - 1;
        }
        __syncthreads();
        // B2/B3: v rows -> every rank's G_v (parity i); gather
        const int64_t po = (i & 1) * a.gpar + (int64_t)L.rank * L.chunk;
        gemv_push(sp, a.pp.G_v, po);
        if (!grid_sync(P.bar, st)) return;
        // p to global only now: before this barrier a slow CTA may still be loading
        // the previous p at the start of the launch
        for (int64_t j = tid0; j < n; j += gstride) a.p_full[j] = sp[j];
        if (lead()) flags_out(a, kPhaseV, i);
        if (!wait_ph(a, kPhaseV, i)) return;
        // B4: gamma = <rhat, v> (full length), alpha
        const T* vg = par_ptr(a.G_v, a.gpar, i);
        T gm[1] = {T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T vj = __ldcg(vg + gidx(L, j));
            sv[j] = vj;
            gm[0] = fma(sh[j], vj, gm[0]);
        }
        cta_total<1>(gm, red);
        const T gam = gm[0];
        if (gam == T(0) || !isfinite(gam)) {
            if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
            return;
        }
        const T alpha = rho / gam;
        // B5: s = r - alpha v, ||s|| (full length), half-step test
        T sacc[1] = {T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T s = fma(-alpha, sv[j], ss[j]);
            ss[j] = s;
            sacc[0] = fma(s, s, sacc[0]);
        }
        cta_total<1>(sacc, red);
        for (int64_t j = tid0; j < n; j += gstride) a.v_full[j] = sv[j];
        const T srel = sqrt(sacc[0]) / (T)st->nb;
        if (srel <= (T)st->tol) {
            for (int64_t l = tid0; l < m; l += gstride) a.x_loc[l] = fma(alpha, sp[r0 + l], a.x_loc[l]);
            if (lead()) {
                put_hist(st, a.hist, i - 1, srel);
                st->alpha[i & 3] = alpha;
                st->relres = srel; st->half = 1; st->half_iter = i; st->converged = 1;
                st->status = KS_OK; st->iters = i; st->done = 1;
            }
            return;
        }
        // B6: t rows -> every rank's G_r (parity i); gather
        gemv_push(ss, a.pp.G_r, po);
        if (!grid_sync(P.bar, st)) return;
        if (lead()) flags_out(a, kPhaseS, i);
        if (!wait_ph(a, kPhaseS, i)) return;
        // B7: <t, s>, <t, t> (full length), omega
        const T* tg = par_ptr(a.G_r, a.gpar, i);
        T tv[2] = {T(0), T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T tj = __ldcg(tg + gidx(L, j));
            tv[0] = fma(tj, ss[j], tv[0]);
            tv[1] = fma(tj, tj, tv[1]);
        }
        cta_total<2>(tv, red);
        const T ts = tv[0], tt = tv[1];
        const T om = ts / tt;
        if (tt == T(0) || !isfinite(tt) || om == T(0) || !isfinite(om)) {
            if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
            return;
        }
        // x += alpha p + omega s (own rows); r = s - omega t, <rhat, r>, <r, r> (full length)
        for (int64_t l = tid0; l < m; l += gstride)
            a.x_loc[l] = fma(om, ss[r0 + l], fma(alpha, sp[r0 + l], a.x_loc[l]));
        __syncthreads();
        T acc[2] = {T(0), T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T r = fma(-om, __ldcg(tg + gidx(L, j)), ss[j]);
            ss[j] = r;
            acc[0] = fma(sh[j], r, acc[0]);
            acc[1] = fma(r, r, acc[1]);
        }
        cta_total<2>(acc, red);
        if (lead()) {
            st->alpha[i & 3] = alpha;
            st->omega[i & 3] = om;
            st->iters = i;
        }
        rho_prev = rho;
        alpha_prev = alpha;
        omega_prev = om;
        rho = acc[0];
        rr = acc[1];
        if (i == P.k1) {
            if (i == maxit) {                          // test of the solve's last step (B8)
                if (lead()) {
                    const T relm = sqrt(rr) / (T)st->nb;
                    put_hist(st, a.hist, i - 1, relm);
                    st->relres = relm;
                    if (relm <= (T)st->tol) { st->converged = 1; st->status = KS_OK; }
                    else st->status = KS_EMAXIT;
                    st->done = 1;
                }
                return;
            }
            // hand r and its partial slots to the next launch (after every CTA read t)
            if (!grid_sync(P.bar, st)) return;
            T* rout = par_ptr(a.G_r, a.gpar, i);
            for (int64_t j = tid0; j < n; j += gstride) rout[gidx(L, j)] = ss[j];
            if (lead()) {
                for (int g = 0; g < L.P; ++g) {
                    rout[(int64_t)g * L.chunk + L.pslot + 0] = g == 0 ? rho : T(0);
                    rout[(int64_t)g * L.chunk + L.pslot + 1] = g == 0 ? rr : T(0);
                }
            }
        }
    }
}

// ------------------------------------------------------------ BiCGSTAB (B1-B8)
template <class T, int kR, int kU>
__global__ void __launch_bounds__(kNT, 2) k_bs_small(PersistArgs<T> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sp = reinterpret_cast<T*>(smem_raw);   // p (ncols, zero padded)
    T* ss = sp + P.ncols;                     // r, overwritten by s, then by the next r (ncols)
    T* sv = ss + P.ncols;                     // v (n)
    __shared__ T red[(kR > 2 ? kR : 2) * kNW];
    const VecArgsT<T>& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t n = L.n;
    const int64_t gstride = (int64_t)gridDim.x * kNT;
    const int64_t tid0 = (int64_t)blockIdx.x * kNT + threadIdx.x;
    if (is_done(st)) return;
    const T* rin = par_ptr(a.G_r, a.gpar, P.k0 - 1);
    for (int64_t j = threadIdx.x; j < P.ncols; j += kNT) {
        sp[j] = j < n ? a.p_full[j] : T(0);
        ss[j] = j < n ? rin[j] : T(0);
        if (j < n) sv[j] = a.v_full[j];
    }
    T rho = rin[L.pslot + 0], rr = rin[L.pslot + 1];
    T rho_prev = (T)st->rho[(P.k0 - 1) & 3], alpha_prev = (T)st->alpha[(P.k0 - 1) & 3];
    T omega_prev = (T)st->omega[(P.k0 - 1) & 3];
    __syncthreads();
    for (long long i = P.k0; i <= P.k1; ++i) {
        // B8 (test of i-1) + B1
        T rel = T(0);
        if (i >= 2) {
            rel = sqrt(rr) / (T)st->nb;
            if (rel <= (T)st->tol) {
                if (lead()) {
                    put_hist(st, a.hist, i - 2, rel);
                    st->relres = rel; st->iters = i - 1; st->converged = 1; st->status = KS_OK; st->done = 1;
                }
                return;
            }
        }
        if (rho == T(0) || !isfinite(rho)) {
            if (lead()) {
                if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
                st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1;
            }
            return;
        }
        if (i == 1) {
            for (int64_t j = threadIdx.x; j < n; j += kNT) sp[j] = ss[j];
        } else {
            const T beta = (rho / rho_prev) * (alpha_prev / omega_prev);
            for (int64_t j = threadIdx.x; j < n; j += kNT) sp[j] = fma(beta, fma(-omega_prev, sv[j], sp[j]), ss[j]);
        }
        if (lead()) {
            if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
            st->rho[i & 3] = rho;
            st->iters = i - 1;
        }
        __syncthreads();
        // B3: v = A p (parity buffer), <rhat, v> partial
        T* vb = par_ptr(a.G_v, a.gpar, i);
        T d1 = T(0), d2 = T(0);
        {
            const int64_t tiles = (n + kR - 1) / kR;
            const int64_t ncb = P.ncols / (Vec16<T>::W * kNT);
            for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int64_t r0 = tile * kR;
                const int nvalid = (int)min((int64_t)kR, n - r0);
                T acc[kR];
                stream_rows<kR, kU, kNT, T, true>(P.A, P.lda, r0, nvalid, sp, 0, ncb, acc);
                block_sum<kNT, kR>(acc, red);
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int r = 0; r < kR; ++r)
                        if (r < nvalid) { vb[r0 + r] = acc[r]; d1 = fma(a.rhat_loc[r0 + r], acc[r], d1); }
                }
            }
        }
        if (threadIdx.x == 0) P.bpart[blockIdx.x * kSlots + (i & 1) * 4 + 0] = d1;
        if (!grid_sync(P.bar, st)) return;
        // p to global only now: before this barrier a slow CTA may still be loading
        // the previous p at the start of the launch
        for (int64_t j = tid0; j < n; j += gstride) a.p_full[j] = sp[j];
        T gm[1] = {T(0)};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kNT)
            gm[0] += __ldcg(P.bpart + (int64_t)b * kSlots + (i & 1) * 4 + 0);
        cta_total<1>(gm, red);
        const T gam = gm[0];
        if (gam == T(0) || !isfinite(gam)) {
            if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
            return;
        }
        const T alpha = rho / gam;
        // B4/B5: v to shared memory; s = r - alpha v and ||s||^2 (every CTA, full n)
        T sacc[1] = {T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T v = __ldcg(vb + j);
            sv[j] = v;
            const T s = fma(-alpha, v, ss[j]);
            ss[j] = s;
            sacc[0] = fma(s, s, sacc[0]);
        }
        cta_total<1>(sacc, red);
        for (int64_t j = tid0; j < n; j += gstride) a.v_full[j] = sv[j];
        const T srel = sqrt(sacc[0]) / (T)st->nb;
        if (srel <= (T)st->tol) {                          // half-step exit
            for (int64_t l = tid0; l < n; l += gstride) a.x_loc[l] = fma(alpha, sp[l], a.x_loc[l]);
            if (lead()) {
                put_hist(st, a.hist, i - 1, srel);
                st->alpha[i & 3] = alpha;
                st->relres = srel; st->half = 1; st->half_iter = i; st->converged = 1;
                st->status = KS_OK; st->iters = i; st->done = 1;
            }
            return;
        }
        // B6: t = A s (parity buffer), <t, s>, <t, t> partials
        T* tb = (i & 1) ? a.q_loc : a.s_full;
        gemv_smem<kR, kU>(P, n, ss, tb, ss, d1, d2, red);
        if (threadIdx.x == 0) {
            P.bpart[blockIdx.x * kSlots + (i & 1) * 4 + 1] = d1;
            P.bpart[blockIdx.x * kSlots + (i & 1) * 4 + 2] = d2;
        }
        if (!grid_sync(P.bar, st)) return;
        T tv[2] = {T(0), T(0)};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kNT) {
            tv[0] += __ldcg(P.bpart + (int64_t)b * kSlots + (i & 1) * 4 + 1);
            tv[1] += __ldcg(P.bpart + (int64_t)b * kSlots + (i & 1) * 4 + 2);
        }
        cta_total<2>(tv, red);
        const T ts = tv[0], tt = tv[1];
        const T om = ts / tt;
        if (tt == T(0) || !isfinite(tt) || om == T(0) || !isfinite(om)) {
            if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
            return;
        }
        // B7: x += alpha p + omega s (owned rows); r = s - omega t, <rhat, r>, <r, r> (every CTA)
        for (int64_t l = tid0; l < n; l += gstride) a.x_loc[l] = fma(om, ss[l], fma(alpha, sp[l], a.x_loc[l]));
        __syncthreads();
        T acc[2] = {T(0), T(0)};
        for (int64_t j = threadIdx.x; j < n; j += kNT) {
            const T r = fma(-om, __ldcg(tb + j), ss[j]);
            ss[j] = r;
            acc[0] = fma(__ldg(a.rhat_loc + j), r, acc[0]);
            acc[1] = fma(r, r, acc[1]);
        }
        cta_total<2>(acc, red);
        T* rout = par_ptr(a.G_r, a.gpar, i);
        for (int64_t j = tid0; j < n; j += gstride) rout[j] = ss[j];
        if (lead()) {
            rout[L.pslot + 0] = acc[0];
            rout[L.pslot + 1] = acc[1];
            st->alpha[i & 3] = alpha;
            st->omega[i & 3] = om;
            st->iters = i;
        }
        rho_prev = rho;
        alpha_prev = alpha;
        omega_prev = om;
        rho = acc[0];
        rr = acc[1];
    }
}

// Tile shape: R = 4 rows, U = 2 column blocks (C1: 256 tiles of 8 KiB rows).
constexpr int kSR = 4, kSU = 2;

// kind: 0 = CG, 1 = BiCGSTAB (P = 1), 2 = CG, 3 = BiCGSTAB with the fused exchange (P > 1)
template <class T>
const void* kern(int kind) {
    return kind == 3 ? (const void*)k_bs_small_peer<T, kSR, kSU>
         : kind == 2 ? (const void*)k_cg_small_peer<T, kSR, kSU>
         : kind == 1 ? (const void*)k_bs_small<T, kSR, kSU> : (const void*)k_cg_small<T, kSR, kSU>;
}
template <class T>
size_t smem_bytes(int kind, int64_t ncols) {
    return (size_t)(kind == 0 ? 2 : kind == 3 ? 4 : 3) * (size_t)ncols * sizeof(T);
}

}  // namespace

// Grid for the small kernels (rows = this rank's rows), 0 if the vectors do not
// fit in shared memory.
template <class T>
int small_grid(int kind, int num_sms, int64_t rows, int64_t ncols) {
    const size_t sm = smem_bytes<T>(kind, ncols);
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
    if (sm + 1024 > (size_t)optin) return 0;
    const void* k = kern<T>(kind);
    // the attribute is per function (shared by every context on the device): allow the
    // device maximum, so a launch of any context's size stays valid after a memo hit
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { cudaGetLastError(); return 0; }
    const int dyn_max = optin - (int)fa.sharedSizeBytes;     // opt-in limit minus static smem
    if ((size_t)dyn_max < sm ||
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kNT, sm);
    if (per_sm < 1) return 0;
    const int64_t tiles = (rows + kSR - 1) / kSR;
    int64_t g = (int64_t)per_sm * num_sms;
    if (g > tiles) g = tiles;
    if (g > kPartStride / kSlots) g = kPartStride / kSlots;   // bpart region: grid x kSlots
    if (g < 1) g = 1;
    return (int)g;
}

template <class T>
int launch_small(int kind, const VecArgsT<T>& a, const T* A, int64_t lda, int64_t ncols, T* bpart,
                 unsigned* bar, long long k0, long long k1, int grid, cudaStream_t st, bool bar_zeroed) {
    PersistArgs<T> P;
    P.a = a;
    P.A = A;
    P.lda = lda;
    P.ncols = ncols;
    P.bpart = bpart;
    P.bar = bar;
    P.k0 = k0;
    P.k1 = k1;
    void* args[] = {&P};
    cudaError_t e = cudaSuccess;
    if (!bar_zeroed) {
        e = cudaMemsetAsync(bar, 0, sizeof(unsigned long long), st);   // grid_sync counter
        if (e != cudaSuccess) return -(int)e;
    }
    e = cudaLaunchCooperativeKernel(kern<T>(kind), dim3((unsigned)grid), dim3(kNT), args,
                                    smem_bytes<T>(kind, ncols), st);
    return e == cudaSuccess ? 1 : -(int)e;
}

template int small_grid<double>(int, int, int64_t, int64_t);
template int small_grid<float>(int, int, int64_t, int64_t);
template int launch_small<double>(int, const VecArgsT<double>&, const double*, int64_t, int64_t, double*,
                                  unsigned*, long long, long long, int, cudaStream_t, bool);
template int launch_small<float>(int, const VecArgsT<float>&, const float*, int64_t, int64_t, float*,
                                 unsigned*, long long, long long, int, cudaStream_t, bool);

}  // namespace ks

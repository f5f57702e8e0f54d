// K2/K3 -- fused vector updates with fused dots, and the per-iteration control
// logic folded into their prologues (SURVEY.md sec.8(a) rows A0, A2-A5, B0-B2,
// B4, B5, B7, B8).  Every kernel is O(n) and HBM/L2-bound; each one replaces
// several BLAS-1 passes (axpy, axpy, dot) by one pass with a deterministic
// fused reduction.
//
// Schedule, one rank of P, iteration k:
//   CG:       K1 q=A p (+sigma_g) -> [allgather S] -> cg_update -> [allgather G_r]
//             -> cg_direction
//   BiCGSTAB: bs_p -> K1 v=A p (+<rhat,v>_g) -> [allgather G_v] -> bs_s
//             -> K1 t=A s (+<t,s>_g,<t,t>_g) -> [allgather S] -> bs_xr -> [allgather G_r]
// The collectives carry the partial scalars next to the vector slices; every
// rank forms the replicated full-length vectors (p, s) redundantly and sums the
// partials in rank order, so all ranks take identical control decisions.
//
// Control: each kernel first checks st->done; the scalars a kernel reads were
// written by an earlier kernel (rings indexed by iteration), and the decision
// (convergence, breakdown, not-SPD) is computed identically by every CTA, then
// recorded by one thread.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ks_device.cuh"
#include "ks_common.cuh"
#include "ks_internal.h"

namespace ks {

namespace {

constexpr int kNT = 256;

// Gather buffers are double-buffered by iteration parity in the fused mode
// (gpar/spar = 0 in NCCL mode: one buffer, gathered in place).
__device__ __forceinline__ double* Gpar(const VecArgs& a, double* G, long long k) {
    return G + (k & 1) * a.gpar;
}
__device__ __forceinline__ double* Spar(const VecArgs& a, long long k) {
    return a.S + (k & 1) * a.spar;
}
__device__ __forceinline__ double* own_chunk(const VecArgs& a, double* G) {
    return G + (int64_t)a.L.rank * a.L.chunk;
}
// Fused mode: wait for phase `ph` of iteration k from every rank.  A timeout
// marks the solve failed (KS_ENCCL) instead of hanging.
__device__ __forceinline__ bool wait_phase(const VecArgs& a, int ph, long long k) {
    if (!a.peer) return true;
    const bool ok = wait_flags(a.flags + ph * kMaxRanks, a.L.P, epoch_of(a.st, k));
    if (!ok && threadIdx.x == 0) {
        a.st->peer_timeout = 1; a.st->status = KS_ENCCL; a.st->done = 1;
    }
    return ok;
}
// Stores v at offset `off` of this rank's chunk in G (parity-0 base per rank) at
// every rank (fused allgather), or only locally in NCCL mode.
__device__ __forceinline__ void publish(const VecArgs& a, double* const* Gpeer, double* G_own,
                                        long long k, int64_t off, double v) {
    const int64_t o = (k & 1) * a.gpar + (int64_t)a.L.rank * a.L.chunk + off;
    if (a.peer) {
        for (int g = 0; g < a.L.P; ++g) Gpeer[g][o] = v;
    } else {
        G_own[o] = v;
    }
}
__device__ __forceinline__ void publish_phase(const VecArgs& a, int ph, long long k) {
    if (!a.peer) return;
    unsigned long long* f[kMaxRanks];
    for (int g = 0; g < a.L.P; ++g) f[g] = a.pp.flags[g] + ph * kMaxRanks + a.L.rank;
    publish_flags(f, a.L.P, epoch_of(a.st, k));
}

// ---------------------------------------------------------------- setup (A0/B0)
__global__ void __launch_bounds__(kNT) k_setup_r(VecArgs a, int have_x0, const double* x0_full) {
    __shared__ double red[kNT / 32];
    const int64_t m = rows_of(a.L), r0 = a.L.row0[a.L.rank];
    double* rl = own_chunk(a, a.G_r);
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
        double r;
        if (have_x0) {
            r = rl[i];                       // r0 = b - A x0 written by K1 (residual mode)
            a.x_loc[i] = x0_full[r0 + i];
        } else {
            r = a.b_full[r0 + i];            // r0 = b (x0 = 0, Q5)
            rl[i] = r;
            a.x_loc[i] = 0.0;
        }
        a.rhat_loc[i] = r;                   // BiCGSTAB shadow residual rhat = r0 (Q7)
        acc[0] = fma(r, r, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        rl[a.L.pslot + 0] = acc[0];          // <rhat, r0> = <r0, r0>
        rl[a.L.pslot + 1] = acc[0];
    }
}

// Setup for P > 1 with x0 = 0: every rank already holds the full b, so r0 = b needs
// no gather.  Every rank fills all chunks of G_r (parity 0) from b; <r0, r0> =
// <rhat, r0> = ||b||^2 is one full-length reduction (fixed order, identical on
// every rank), stored in chunk 0's partial slots with the other chunks' slots 0, so
// the consumers' rank-ordered slot sums read it unchanged.
__global__ void __launch_bounds__(kNT) k_setup_local(VecArgs a) {
    __shared__ double red[kNT / 32];
    const Layout& L = a.L;
    const int64_t m = rows_of(L), r0 = L.row0[L.rank];
    double acc[1] = {0.0};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < L.n; j += (int64_t)gridDim.x * kNT) {
        const double bj = a.b_full[j];
        a.G_r[gidx(L, j)] = bj;
        acc[0] = fma(bj, bj, acc[0]);
    }
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
        a.x_loc[i] = 0.0;
        a.rhat_loc[i] = a.b_full[r0 + i];
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        for (int g = 0; g < L.P; ++g) {
            a.G_r[(int64_t)g * L.chunk + L.pslot + 0] = g == 0 ? acc[0] : 0.0;
            a.G_r[(int64_t)g * L.chunk + L.pslot + 1] = g == 0 ? acc[0] : 0.0;
        }
    }
}

__device__ void init_state(DevState* st, double tol, long long maxit, long long hist_cap,
                           unsigned long long ebase) {
    st->tol = tol;
    st->ebase = ebase;
    st->peer_timeout = 0;
    st->maxit = maxit;
    st->hist_cap = hist_cap;
    st->iters = 0;
    st->half_iter = 0;
    st->done = 0;
    st->status = KS_EMAXIT;
    st->converged = 0;
    st->breakdown = 0;
    st->half = 0;
    st->bzero = 0;
    st->true_rr = -1.0;
    for (int q = 0; q < 4; ++q) st->rho[q] = st->alpha[q] = st->omega[q] = 1.0;
}

// Decides the 0-iteration exits (Q6: b = 0 -> x = 0; Q2: ||r0||/||b|| <= tol).
__device__ void init_decide(DevState* st, double bb, double rr) {
    const double nb = sqrt(bb);
    st->nb = nb;
    if (nb == 0.0) {
        st->bzero = 1; st->converged = 1; st->status = KS_OK; st->relres = 0.0; st->done = 1;
        return;
    }
    const double rel = sqrt(rr) / nb;
    st->relres = rel;
    if (rel <= st->tol) { st->converged = 1; st->status = KS_OK; st->done = 1; }
}

// ------------------------------------------------------------------- CG (A1-A5)
__global__ void __launch_bounds__(kNT) k_cg_init(VecArgs a, double tol, long long maxit,
                                                 long long hist_cap, unsigned long long ebase) {
    __shared__ double red[kNT / 32];
    double acc[1] = {0.0};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT) {
        a.p_full[j] = a.G_r[gidx(a.L, j)];                 // p0 = r0 (full, replicated)
        const double bj = a.b_full[j];
        acc[0] = fma(bj, bj, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        DevState* st = a.st;
        init_state(st, tol, maxit, hist_cap, ebase);
        const double rho0 = slot_sum(a.L, a.G_r, 1);
        st->rho[0] = rho0;
        init_decide(st, acc[0], rho0);
    }
}

// A2 + A3: sigma = sum_g sigma_g; alpha = rho/sigma; x += alpha p; r -= alpha q;
// rho'_g = <r_loc, r_loc> -> own partial slot of G_r (rides on the r allgather).
__global__ void __launch_bounds__(kNT) k_cg_update(VecArgs a, const long long* kdev, long long koff) {
    const long long k = koff + (kdev ? *kdev : 0);
    __shared__ double red[kNT / 32];
    DevState* st = a.st;
    if (is_done(st)) return;
    if (!wait_phase(a, kPhaseS, k)) return;                   // sigma partials of iteration k
    const double sigma = scal_sum(a.L, Spar(a, k), 0);
    if (!(sigma > 0.0)) {                                   // Q9: NOTSPD, x unchanged
        if (lead()) { st->status = KS_ENOTSPD; st->iters = k - 1; st->done = 1; }
        return;
    }
    const double alpha = st->rho[(k - 1) & 3] / sigma;
    const int64_t m = rows_of(a.L), r0 = a.L.row0[a.L.rank];
    const double* rin = own_chunk(a, Gpar(a, a.G_r, k - 1));   // r_{k-1}
    const double* pl = a.p_full + r0;
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
        a.x_loc[i] = fma(alpha, pl[i], a.x_loc[i]);
        const double r = fma(-alpha, a.q_loc[i], rin[i]);
        publish(a, a.pp.G_r, a.G_r, k, i, r);                // r_k -> every rank (fused C1)
        acc[0] = fma(r, r, acc[0]);
    }
    if (a.peer) __threadfence_system();
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        publish(a, a.pp.G_r, a.G_r, k, a.L.pslot + 1, acc[0]);
        st->alpha[k & 3] = alpha;
        publish_phase(a, kPhaseR, k);
    }
}

// A5: rho' = sum_g rho'_g; convergence test (Q1); beta; p = r + beta p (full n).
__global__ void __launch_bounds__(kNT) k_cg_direction(VecArgs a, const long long* kdev, long long koff) {
    const long long k = koff + (kdev ? *kdev : 0);
    DevState* st = a.st;
    if (is_done(st)) return;
    if (!wait_phase(a, kPhaseR, k)) return;
    const double* Gr = Gpar(a, a.G_r, k);
    const double rho1 = slot_sum(a.L, Gr, 1);
    const double rel = sqrt(rho1) / st->nb;
    if (rel <= st->tol) {
        if (lead()) {
            put_hist(st, a.hist, k - 1, rel);
            st->relres = rel; st->iters = k; st->converged = 1; st->status = KS_OK; st->done = 1;
        }
        return;
    }
    const double beta = rho1 / st->rho[(k - 1) & 3];
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT)
        a.p_full[j] = fma(beta, a.p_full[j], Gr[gidx(a.L, j)]);
    if (lead()) {
        put_hist(st, a.hist, k - 1, rel);
        st->relres = rel; st->iters = k; st->rho[k & 3] = rho1;
    }
}

__global__ void __launch_bounds__(kNT) k_finish(VecArgs a, int bicgstab) {
    DevState* st = a.st;
    if (bicgstab && !is_done(st) && st->maxit >= 1 && !wait_phase(a, kPhaseR, st->maxit)) return;
    if (lead() && !st->done) {
        const long long maxit = st->maxit;
        st->iters = maxit;
        st->status = KS_EMAXIT;
        if (bicgstab && maxit >= 1) {                     // test of the last full step
            const double rel = sqrt(slot_sum(a.L, Gpar(a, a.G_r, maxit), 1)) / st->nb;
            put_hist(st, a.hist, maxit - 1, rel);
            st->relres = rel;
            if (rel <= st->tol) { st->converged = 1; st->status = KS_OK; }
        }
        st->done = 1;
    }
    if (st->bzero) {                                      // Q6: b = 0 -> x = 0
        const int64_t m = rows_of(a.L);
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
            a.x_loc[i] = 0.0;
    }
}

// ------------------------------------------------------------- BiCGSTAB (B1-B8)
__global__ void __launch_bounds__(kNT) k_bs_init(VecArgs a, double tol, long long maxit,
                                                 long long hist_cap, unsigned long long ebase) {
    __shared__ double red[kNT / 32];
    double acc[1] = {0.0};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT) {
        const double bj = a.b_full[j];
        acc[0] = fma(bj, bj, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        DevState* st = a.st;
        init_state(st, tol, maxit, hist_cap, ebase);   // rho_old = alpha = omega = 1 (Q8)
        init_decide(st, acc[0], slot_sum(a.L, a.G_r, 1));
    }
}

// B8 (test of iteration i-1) + B1: rho_i = <rhat, r_{i-1}> from the gathered
// partials; beta; p = r + beta (p - omega v) over the full length (i = 1: p = r).
__global__ void __launch_bounds__(kNT) k_bs_p(VecArgs a, const long long* kdev, long long koff) {
    const long long i = koff + (kdev ? *kdev : 0);
    DevState* st = a.st;
    if (is_done(st)) return;
    if (i >= 2 && !wait_phase(a, kPhaseR, i - 1)) return;
    const double* Gr = Gpar(a, a.G_r, i - 1);              // r_{i-1} (+ partials)
    const double rho = slot_sum(a.L, Gr, 0);
    double rel = 0.0;
    if (i >= 2) {
        rel = sqrt(slot_sum(a.L, Gr, 1)) / st->nb;
        if (rel <= st->tol) {
            if (lead()) {
                put_hist(st, a.hist, i - 2, rel);
                st->relres = rel; st->iters = i - 1; st->converged = 1; st->status = KS_OK;
                st->done = 1;
            }
            return;
        }
    }
    if (rho == 0.0 || !isfinite(rho)) {                    // Q9
        if (lead()) {
            if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
            st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1;
        }
        return;
    }
    if (i == 1) {
        for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT)
            a.p_full[j] = Gr[gidx(a.L, j)];
    } else {
        const int q = (int)((i - 1) & 3);
        const double om = st->omega[q];
        const double beta = (rho / st->rho[q]) * (st->alpha[q] / om);
        for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT) {
            a.p_full[j] = fma(beta, fma(-om, a.v_full[j], a.p_full[j]), Gr[gidx(a.L, j)]);
        }
    }
    if (lead()) {
        if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
        st->rho[i & 3] = rho;
        st->iters = i - 1;
    }
}

// B4 + B5: gamma = sum_g <rhat,v>_g; alpha = rho/gamma; s = r - alpha v (full n,
// redundant); ||s||^2 over the full length; half-step test.
__global__ void __launch_bounds__(kNT) k_bs_s(VecArgs a, const long long* kdev, long long koff) {
    const long long i = koff + (kdev ? *kdev : 0);
    __shared__ double red[kNT / 32];
    DevState* st = a.st;
    if (is_done(st)) return;
    if (!wait_phase(a, kPhaseV, i)) return;                   // v_i slices + <rhat,v> partials
    // the <rhat,v> partials were pushed into the local buffer; the v slices are
    // PULLED from their owners over NVLink in the fused mode (K1 wrote them
    // locally; its last block released the flag), or read from the NCCL-gathered
    // local buffer.  A full local copy is kept for the next bs_p.
    const double* Gv = Gpar(a, a.G_v, i);
    const double* Gr = Gpar(a, a.G_r, i - 1);
    const double g = slot_sum(a.L, Gv, 0);
    if (g == 0.0 || !isfinite(g)) {
        if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
        return;
    }
    const double alpha = st->rho[i & 3] / g;
    const int64_t vpar = (i & 1) * a.gpar;
    double acc[1] = {0.0};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT) {
        int o = 0;
        while (o + 1 < a.L.P && j >= a.L.row0[o + 1]) ++o;
        const int64_t gj = (int64_t)o * a.L.chunk + (j - a.L.row0[o]);
        const double v = a.peer ? __ldcg(a.pp.G_v[o] + vpar + gj) : Gv[gj];
        a.v_full[j] = v;
        const double s = fma(-alpha, v, Gr[gj]);
        a.s_full[j] = s;
        acc[0] = fma(s, s, acc[0]);
    }
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        st->alpha[i & 3] = alpha;
        const double srel = sqrt(acc[0]) / st->nb;
        if (srel <= st->tol) {                              // half-step exit (Q2)
            put_hist(st, a.hist, i - 1, srel);
            st->relres = srel; st->half = 1; st->half_iter = i; st->converged = 1;
            st->status = KS_OK; st->iters = i; st->done = 1;
        }
    }
}

// B7: omega = <t,s>/<t,t>; x += alpha p + omega s; r = s - omega t; partials
// <rhat, r>_g and <r, r>_g into the own slots of G_r.  On a half-step exit in
// iteration i this kernel applies x += alpha p instead.
__global__ void __launch_bounds__(kNT) k_bs_xr(VecArgs a, const long long* kdev, long long koff) {
    const long long i = koff + (kdev ? *kdev : 0);
    __shared__ double red[2 * (kNT / 32)];
    DevState* st = a.st;
    const int64_t m = rows_of(a.L), r0 = a.L.row0[a.L.rank];
    const double* pl = a.p_full + r0;
    if (is_done(st)) {
        if (st->half_iter == i) {
            const double alpha = st->alpha[i & 3];
            for (int64_t l = blockIdx.x * (int64_t)kNT + threadIdx.x; l < m; l += (int64_t)gridDim.x * kNT)
                a.x_loc[l] = fma(alpha, pl[l], a.x_loc[l]);
        }
        return;
    }
    if (!wait_phase(a, kPhaseS, i)) return;                   // <t,s>, <t,t> partials
    const double* Si = Spar(a, i);
    const double ts = scal_sum(a.L, Si, 0), tt = scal_sum(a.L, Si, 1);
    const double om = ts / tt;
    if (tt == 0.0 || !isfinite(tt) || om == 0.0 || !isfinite(om)) {
        if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
        return;
    }
    const double alpha = st->alpha[i & 3];
    const double* sl = a.s_full + r0;
    double acc[2] = {0.0, 0.0};
    for (int64_t l = blockIdx.x * (int64_t)kNT + threadIdx.x; l < m; l += (int64_t)gridDim.x * kNT) {
        const double s = sl[l];
        a.x_loc[l] = fma(om, s, fma(alpha, pl[l], a.x_loc[l]));
        const double r = fma(-om, a.q_loc[l], s);
        publish(a, a.pp.G_r, a.G_r, i, l, r);                // r_i -> every rank (fused C1)
        acc[0] = fma(a.rhat_loc[l], r, acc[0]);
        acc[1] = fma(r, r, acc[1]);
    }
    if (a.peer) __threadfence_system();
    block_sum<kNT, 2>(acc, red);
    if (grid_sum<kNT, 2>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        publish(a, a.pp.G_r, a.G_r, i, a.L.pslot + 0, acc[0]);
        publish(a, a.pp.G_r, a.G_r, i, a.L.pslot + 1, acc[1]);
        st->omega[i & 3] = om;
        st->iters = i;
        publish_phase(a, kPhaseR, i);
    }
}

// ---------------------------------------------------------------- BiCG (NEXT-3)
// Fletcher's BiCG (oracle or_bicg): p = r + beta p (full, replicated like CG),
// the shadow pair (rt, pt) stays sharded: qt rows come from K1T + reduce-scatter.
__global__ void __launch_bounds__(kNT) k_bicg_init(VecArgs a, double tol, long long maxit,
                                                   long long hist_cap, unsigned long long ebase) {
    __shared__ double red[kNT / 32];
    const int64_t m = rows_of(a.L);
    double acc[1] = {0.0};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT) {
        a.p_full[j] = a.G_r[gidx(a.L, j)];                  // p0 = r0
        const double bj = a.b_full[j];
        acc[0] = fma(bj, bj, acc[0]);
    }
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
        a.pt_loc[i] = a.rhat_loc[i];                        // pt0 = rt0 = r0 (Q7)
    block_sum<kNT, 1>(acc, red);
    if (grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        DevState* st = a.st;
        init_state(st, tol, maxit, hist_cap, ebase);
        st->rho[0] = slot_sum(a.L, a.G_r, 0);              // <rt0, r0>
        init_decide(st, acc[0], slot_sum(a.L, a.G_r, 1));
    }
}

// sigma = <pt, A p> (K1 partials); alpha; x += alpha p; r -= alpha q; rt -= alpha qt;
// partials <rt, r>, <r, r> into the own slots of G_r.  Fused mode: sigma partials
// and the K1T column-sum slices (G_v, one slot per source rank, summed in rank
// order) arrive over NVLink; r_k and the partials are pushed to every rank.
__global__ void __launch_bounds__(kNT) k_bicg_update(VecArgs a, long long k) {
    __shared__ double red[2 * (kNT / 32)];
    DevState* st = a.st;
    if (is_done(st)) return;
    if (!wait_phase(a, kPhaseS, k) || !wait_phase(a, kPhaseV, k)) return;
    const double sigma = scal_sum(a.L, Spar(a, k), 0);
    if (sigma == 0.0 || !isfinite(sigma)) {
        if (lead()) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = k - 1; st->done = 1; }
        return;
    }
    const double alpha = st->rho[(k - 1) & 3] / sigma;
    const int64_t m = rows_of(a.L), r0 = a.L.row0[a.L.rank];
    const double* rin = own_chunk(a, Gpar(a, a.G_r, k - 1));   // r_{k-1}
    const double* qslots = Gpar(a, a.G_v, k);                   // fused: P slots of qt rows
    double acc[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
        a.x_loc[i] = fma(alpha, a.p_full[r0 + i], a.x_loc[i]);
        const double r = fma(-alpha, a.q_loc[i], rin[i]);
        publish(a, a.pp.G_r, a.G_r, k, i, r);
        double qt;
        if (a.peer) {
            qt = 0.0;
            for (int g = 0; g < a.L.P; ++g) qt += qslots[(int64_t)g * a.L.chunk + i];
        } else {
            qt = a.qt_loc[i];
        }
        const double rt = fma(-alpha, qt, a.rhat_loc[i]);
        a.rhat_loc[i] = rt;
        acc[0] = fma(rt, r, acc[0]);
        acc[1] = fma(r, r, acc[1]);
    }
    if (a.peer) __threadfence_system();
    block_sum<kNT, 2>(acc, red);
    if (grid_sum<kNT, 2>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0) {
        publish(a, a.pp.G_r, a.G_r, k, a.L.pslot + 0, acc[0]);
        publish(a, a.pp.G_r, a.G_r, k, a.L.pslot + 1, acc[1]);
        st->alpha[k & 3] = alpha;
        publish_phase(a, kPhaseR, k);
    }
}

// test (Q1), rho' breakdown (Q9), beta, p = r + beta p (full), pt = rt + beta pt.
__global__ void __launch_bounds__(kNT) k_bicg_direction(VecArgs a, long long k) {
    DevState* st = a.st;
    if (is_done(st)) return;
    if (!wait_phase(a, kPhaseR, k)) return;
    const double* Gr = Gpar(a, a.G_r, k);
    const double rho1 = slot_sum(a.L, Gr, 0);
    const double rel = sqrt(slot_sum(a.L, Gr, 1)) / st->nb;
    if (rel <= st->tol) {
        if (lead()) {
            put_hist(st, a.hist, k - 1, rel);
            st->relres = rel; st->iters = k; st->converged = 1; st->status = KS_OK; st->done = 1;
        }
        return;
    }
    if (rho1 == 0.0 || !isfinite(rho1)) {
        if (lead()) {
            put_hist(st, a.hist, k - 1, rel);
            st->relres = rel; st->iters = k; st->status = KS_EBREAKDOWN; st->breakdown = 1; st->done = 1;
        }
        return;
    }
    const double beta = rho1 / st->rho[(k - 1) & 3];
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < a.L.n; j += (int64_t)gridDim.x * kNT)
        a.p_full[j] = fma(beta, a.p_full[j], Gr[gidx(a.L, j)]);
    const int64_t m = rows_of(a.L);
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
        a.pt_loc[i] = fma(beta, a.pt_loc[i], a.rhat_loc[i]);
    if (lead()) {
        put_hist(st, a.hist, k - 1, rel);
        st->relres = rel; st->iters = k; st->rho[k & 3] = rho1;
    }
}

__global__ void k_advance(long long* kdev, long long by) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *kdev += by;
}

__global__ void k_true_res_final(VecArgs a) {
    if (lead()) a.st->true_rr = scal_sum(a.L, a.S, 1);
}

__global__ void __launch_bounds__(kNT) k_pack_x(VecArgs a) {
    const int64_t m = rows_of(a.L);
    double* xl = own_chunk(a, a.G_v);
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT)
        xl[i] = a.x_loc[i];
}

unsigned grid_for(int64_t len, int num_sms) {
    int64_t g = (len + kNT * 4 - 1) / (kNT * 4);
    if (g < 1) g = 1;
    const int64_t cap = 2LL * num_sms;
    return (unsigned)(g > cap ? cap : g);
}

int64_t mloc_h(const Layout& L) { return L.row0[L.rank + 1] - L.row0[L.rank]; }

template <class T>
__global__ void k_join(VecArgsT<T> a, unsigned long long epoch, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    unsigned long long* f[kMaxRanks];
    for (int g = 0; g < a.L.P; ++g) f[g] = a.pp.flags[g] + kPhaseJ * kMaxRanks + a.L.rank;
    publish_flags(f, a.L.P, epoch);
    const unsigned long long t0 = globaltimer_ns();
    for (int g = 0; g < a.L.P; ++g) {
        while (flag_acquire_sys(a.flags + kPhaseJ * kMaxRanks + g) < epoch) {
            if (globaltimer_ns() - t0 > timeout_ns) {
                a.st->peer_timeout = 1; a.st->status = KS_ENCCL; a.st->done = 1;
                return;
            }
            __nanosleep(64);
        }
    }
}

// Rows A0 / B0 with x0 = 0 plus the solver-state init (and the rendezvous) in one
// launch; the arithmetic is k_setup_local's / k_setup_r's and k_cg_init's /
// k_bs_init's: r0 = b, <r0, r0> = ||b||^2 in one fixed-order grid reduction.
__global__ void __launch_bounds__(kNT) k_start(VecArgs a, int bicgstab, double tol, long long maxit,
                                               long long hist_cap, unsigned long long ebase,
                                               unsigned long long join_ns) {
    __shared__ double red[kNT / 32];
    const Layout& L = a.L;
    const int64_t m = rows_of(L), r0 = L.row0[L.rank];
    const int64_t gs = (int64_t)gridDim.x * kNT;
    double acc[1] = {0.0};
    for (int64_t j = blockIdx.x * (int64_t)kNT + threadIdx.x; j < L.n; j += gs) {
        const double bj = a.b_full[j];
        a.G_r[gidx(L, j)] = bj;                       // r0 = b (Q5), parity 0
        if (!bicgstab) a.p_full[j] = bj;               // CG: p0 = r0 (full, replicated)
        acc[0] = fma(bj, bj, acc[0]);
    }
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += gs) {
        a.x_loc[i] = 0.0;
        a.rhat_loc[i] = a.b_full[r0 + i];              // rhat = r0 (Q7)
    }
    block_sum<kNT, 1>(acc, red);
    if (!(grid_sum<kNT, 1>(acc, a.scr.part, a.scr.ticket, red) && threadIdx.x == 0)) return;
    for (int g = 0; g < L.P; ++g) {
        a.G_r[(int64_t)g * L.chunk + L.pslot + 0] = g == 0 ? acc[0] : 0.0;   // <rhat, r0>
        a.G_r[(int64_t)g * L.chunk + L.pslot + 1] = g == 0 ? acc[0] : 0.0;   // <r0, r0>
    }
    DevState* st = a.st;
    *reinterpret_cast<unsigned long long*>(a.scr.ticket + 8) = 0ull;   // persistent grid-barrier counter
    init_state(st, tol, maxit, hist_cap, ebase);     // BiCGSTAB: rho_old = alpha = omega = 1 (Q8)
    if (!bicgstab) st->rho[0] = acc[0];
    init_decide(st, acc[0], acc[0]);
    if (join_ns == 0) return;
    unsigned long long* f[kMaxRanks];                 // the rendezvous (launch_join)
    for (int g = 0; g < L.P; ++g) f[g] = a.pp.flags[g] + kPhaseJ * kMaxRanks + L.rank;
    publish_flags(f, L.P, ebase);
    const unsigned long long t0 = globaltimer_ns();
    for (int g = 0; g < L.P; ++g) {
        while (flag_acquire_sys(a.flags + kPhaseJ * kMaxRanks + g) < ebase) {
            if (globaltimer_ns() - t0 > join_ns) {
                st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1;
                return;
            }
            __nanosleep(64);
        }
    }
}

// k_finish + (gather) the fused end-of-solve x gather into every rank's X.
__global__ void __launch_bounds__(kNT) k_end(VecArgs a, int bicgstab, int gather, unsigned long long epoch) {
    __shared__ int s_last;
    DevState* st = a.st;
    const Layout& L = a.L;
    if (bicgstab && !is_done(st) && st->maxit >= 1 && !wait_phase(a, kPhaseR, st->maxit)) return;
    if (lead() && !st->done) {
        const long long maxit = st->maxit;
        st->iters = maxit;
        st->status = KS_EMAXIT;
        if (bicgstab && maxit >= 1) {                     // test of the last full step
            const double rel = sqrt(slot_sum(L, Gpar(a, a.G_r, maxit), 1)) / st->nb;
            put_hist(st, a.hist, maxit - 1, rel);
            st->relres = rel;
            if (rel <= st->tol) { st->converged = 1; st->status = KS_OK; }
        }
        st->done = 1;
    }
    const int bz = st->bzero;                             // set by the start kernel only
    const int64_t m = rows_of(L), r0 = L.row0[L.rank];
    bool stored = false;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < m; i += (int64_t)gridDim.x * kNT) {
        double xv = a.x_loc[i];
        if (bz) { xv = 0.0; a.x_loc[i] = 0.0; }           // Q6: b = 0 -> x = 0
        if (gather) {
            for (int g = 0; g < L.P; ++g) a.pp.X[g][r0 + i] = xv;
            stored = true;
        }
    }
    if (!gather) return;
    (void)stored;
    // every thread's remote stores, then ONE system-scope fence per CTA (cumulative over
    // the barrier, the pattern NCCL's primitives use) before the CTA's ticket arrival
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        unsigned* ticket = a.scr.ticket + 16;
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        if (s_last) *ticket = 0u;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    unsigned long long* f[kMaxRanks];
    for (int g = 0; g < L.P; ++g) f[g] = a.pp.flags[g] + kPhaseX * kMaxRanks + L.rank;
    publish_flags(f, L.P, epoch);
    const unsigned long long t0 = globaltimer_ns();
    for (int g = 0; g < L.P; ++g) {
        while (flag_acquire_sys(a.flags + kPhaseX * kMaxRanks + g) < epoch) {
            if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                st->peer_timeout = 1; st->status = KS_ENCCL;
                return;
            }
            __nanosleep(32);
        }
    }
}

}  // namespace

int launch_start(const VecArgs& a, int bicgstab, double tol, long long maxit, long long hist_cap,
                 unsigned long long ebase, long long join_ms, cudaStream_t st) {
    const unsigned long long ns = join_ms > 0 ? (unsigned long long)join_ms * 1000000ULL : 0ULL;
    k_start<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, bicgstab, tol, maxit, hist_cap, ebase, ns);
    return 1;
}
int launch_end(const VecArgs& a, int bicgstab, int gather, unsigned long long epoch, cudaStream_t st) {
    k_end<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, bicgstab, gather, epoch);
    return 1;
}

template <class T>
int launch_join(const VecArgsT<T>& a, unsigned long long epoch, long long timeout_ms, cudaStream_t st) {
    const unsigned long long ns = (unsigned long long)(timeout_ms > 0 ? timeout_ms : 1) * 1000000ULL;
    k_join<T><<<1, 32, 0, st>>>(a, epoch, ns);
    return 1;
}
template int launch_join<double>(const VecArgsT<double>&, unsigned long long, long long, cudaStream_t);
template int launch_join<float>(const VecArgsT<float>&, unsigned long long, long long, cudaStream_t);

int launch_setup_local(const VecArgs& a, cudaStream_t st) {
    k_setup_local<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a);
    return 1;
}
int launch_setup_r(const VecArgs& a, bool have_x0, const double* x0_full, cudaStream_t st) {
    k_setup_r<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, have_x0 ? 1 : 0, x0_full);
    return 1;
}
int launch_cg_init(const VecArgs& a, double tol, long long maxit, long long hist_cap,
                   unsigned long long ebase, cudaStream_t st) {
    k_cg_init<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, tol, maxit, hist_cap, ebase);
    return 1;
}
int launch_cg_update(const VecArgs& a, const long long* kdev, long long k, cudaStream_t st) {
    k_cg_update<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, kdev, k);
    return 1;
}
int launch_cg_direction(const VecArgs& a, const long long* kdev, long long k, cudaStream_t st) {
    k_cg_direction<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, kdev, k);
    return 1;
}
int launch_cg_finish(const VecArgs& a, cudaStream_t st) {
    k_finish<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, 0);
    return 1;
}
int launch_bs_init(const VecArgs& a, double tol, long long maxit, long long hist_cap,
                   unsigned long long ebase, cudaStream_t st) {
    k_bs_init<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, tol, maxit, hist_cap, ebase);
    return 1;
}
int launch_bs_p(const VecArgs& a, const long long* kdev, long long i, cudaStream_t st) {
    k_bs_p<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, kdev, i);
    return 1;
}
int launch_bs_s(const VecArgs& a, const long long* kdev, long long i, cudaStream_t st) {
    k_bs_s<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, kdev, i);
    return 1;
}
int launch_bs_xr(const VecArgs& a, const long long* kdev, long long i, cudaStream_t st) {
    k_bs_xr<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, kdev, i);
    return 1;
}
int launch_bs_finish(const VecArgs& a, cudaStream_t st) {
    k_finish<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, 1);
    return 1;
}
int launch_advance(long long* kdev, long long by, cudaStream_t st) {
    k_advance<<<1, 32, 0, st>>>(kdev, by);
    return 1;
}
int launch_bicg_init(const VecArgs& a, double tol, long long maxit, long long hist_cap,
                     unsigned long long ebase, cudaStream_t st) {
    k_bicg_init<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, tol, maxit, hist_cap, ebase);
    return 1;
}
int launch_bicg_update(const VecArgs& a, long long k, cudaStream_t st) {
    k_bicg_update<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a, k);
    return 1;
}
int launch_bicg_direction(const VecArgs& a, long long k, cudaStream_t st) {
    k_bicg_direction<<<grid_for(a.L.n, a.num_sms), kNT, 0, st>>>(a, k);
    return 1;
}
int launch_true_res_final(const VecArgs& a, cudaStream_t st) {
    k_true_res_final<<<1, 32, 0, st>>>(a);
    return 1;
}
// out[i] = sum over g = 0..P-1 (in rank order) of S[g * chunk + i]: the reduction
// half of a host-driven reduce-scatter (shared-device contexts, ks_ctx.cpp).
__global__ void k_sum_slots(const double* __restrict__ S, int P, int64_t chunk, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < chunk; i += (int64_t)gridDim.x * kNT) {
        double s = S[i];
        for (int g = 1; g < P; ++g) s += S[(int64_t)g * chunk + i];
        out[i] = s;
    }
}
int launch_sum_slots(const double* S, int P, int64_t chunk, double* out, int num_sms, cudaStream_t st) {
    k_sum_slots<<<grid_for(chunk, num_sms), kNT, 0, st>>>(S, P, chunk, out);
    return 1;
}
int launch_pack_x(const VecArgs& a, cudaStream_t st) {
    k_pack_x<<<grid_for(mloc_h(a.L), a.num_sms), kNT, 0, st>>>(a);
    return 1;
}

}  // namespace ks

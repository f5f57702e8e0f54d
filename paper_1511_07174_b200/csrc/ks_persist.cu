// NEXT-2: persistent cooperative whole-iteration kernels.
//
// One cooperative launch runs a batch of CG / BiCGSTAB iterations (the same
// rows A1-A5 / B1-B8 as the multi-kernel path), with grid-wide barriers where
// the multi-kernel path has kernel boundaries.  This removes the per-kernel
// launch gaps and last-block reductions that dominate small systems (C1: the
// 8 MiB matrix is L2-resident and a GEMV is ~1 us) and the ~30 us/iteration of
// vector-kernel overhead at large n.  The GEMV phase streams A with the same
// inner loop as K1 (ks_tile.cuh) over tiles assigned round-robin to the
// resident CTAs.  All reductions are fixed-order (tile order within a CTA, CTA
// order across the grid), so results are deterministic and identical on every
// rank; the grid size depends only on (n, P) so every rank uses the same one.
// For P > 1 it requires the fused NVLink exchange (no host-launched NCCL call
// can run inside a persistent kernel): partial scalars and r slices are pushed
// to every rank and flagged; v is pulled.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstring>
#include <math.h>
#include <stdint.h>

#include "ks_device.cuh"
#include "ks_internal.h"
#include "ks_tile.cuh"
#include "ks_persist.cuh"

namespace ks {

namespace {

using namespace pk;

// ---------------------------------------------------------------- CG (A1-A5)
template <class T, int kR, int kU>
__device__ __forceinline__ void cg_persist_body(const PersistArgs<T>& P, int vb, int vg) {
    __shared__ T red[(kR > 2 ? kR : 2) * kNW];
    const VecArgsT<T>& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t m = rows_of(L), r0 = L.row0[L.rank];
    const int64_t gstride = (int64_t)vg * kNT;
    const int64_t tid0 = (int64_t)vb * kNT + threadIdx.x;
    for (long long k = P.k0; k <= P.k1; ++k) {
        if (is_done(st)) break;
        // A1: q = A p, sigma_g = <p_loc, q>
        T d1, d2;
        gemv_phase<kR, kU>(P, a.p_full, a.q_loc, a.p_full + r0, d1, d2, red, (const T*)nullptr, vb, vg);
        if (threadIdx.x == 0) P.bpart[vb * 4 + 0] = d1;
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        T sig[1];
        grid_total<1>(P.bpart, 0, sig, red, vg);
        T sigma = sig[0];
        if (a.peer && a.ll) {                           // A2 fused C2, LL words
            if ((vb == 0 && threadIdx.x == 0)) {
                const double v = (double)sigma;
                ll_push_scal(a, (int)(k & 1), 0, &v, 1, ll_epoch(st, k));
            }
            if (!ll_sum_scal<1>(a, (int)(k & 1), 0, ll_epoch(st, k), sig)) return;
            sigma = sig[0];
        } else if (a.peer) {                            // A2 fused C2
            if ((vb == 0 && threadIdx.x == 0)) {
                for (int g = 0; g < L.P; ++g) a.pp.S[g][(k & 1) * a.spar + L.rank * kScalSlot] = sigma;
                flags_out(a, kPhaseS, k);
            }
            if (!wait_ph(a, kPhaseS, k)) return;
            sigma = scal_sum(L, par_ptr(a.S, a.spar, k), 0);
        }
        if (!(sigma > T(0))) {                           // Q9
            if ((vb == 0 && threadIdx.x == 0)) { st->status = KS_ENOTSPD; st->iters = k - 1; st->done = 1; }
            break;
        }
        const T alpha = (T)st->rho[(k - 1) & 3] / sigma;
        // A3: x += alpha p, r -= alpha q, rho'_g
        const T* rin = par_ptr(a.G_r, a.gpar, k - 1) + (int64_t)L.rank * L.chunk;
        const int64_t ro = (k & 1) * a.gpar + (int64_t)L.rank * L.chunk;
        T acc[1] = {T(0)};
        const uint32_t ep = ll_epoch(st, k);
        if (a.peer && a.ll) jitter_at(a.jitter, 8u);
        for (int64_t i = tid0; i < m; i += gstride) {
            a.x_loc[i] = fma(alpha, a.p_full[r0 + i], a.x_loc[i]);
            const T r = fma(-alpha, a.q_loc[i], rin[i]);
            if (a.peer && a.ll) {                       // A4 as LL words (own chunk kept plain: next rin)
                a.G_r[ro + i] = r;
                for (int g = 0; g < L.P; ++g) ll_put_sys(a.pp.llg[g] + ll_vec_off(L.ld, (int)(k & 1), 0, r0 + i), (double)r, ep);
            } else if (a.peer) {
                for (int g = 0; g < L.P; ++g) a.pp.G_r[g][ro + i] = r;
            } else {
                a.G_r[ro + i] = r;
            }
            acc[0] = fma(r, r, acc[0]);
        }
        if (a.peer && !a.ll && tid0 < m) __threadfence_system();   // only threads that stored remotely
        block_sum<kNT, 1>(acc, red);
        if (threadIdx.x == 0) P.bpart[vb * 4 + 1] = acc[0];
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        T rr[1];
        grid_total<1>(P.bpart, 1, rr, red, vg);
        T rho1 = rr[0];
        if (a.peer && a.ll) {                           // rho' rank partials, LL words
            if ((vb == 0 && threadIdx.x == 0)) {
                const double v = (double)rho1;
                ll_push_scal(a, (int)(k & 1), 1, &v, 1, ep);
            }
            if (!ll_sum_scal<1>(a, (int)(k & 1), 1, ep, rr)) return;
            rho1 = rr[0];
        } else if (a.peer) {                            // A4 fused C1 (+ partials)
            if ((vb == 0 && threadIdx.x == 0)) {
                for (int g = 0; g < L.P; ++g) a.pp.G_r[g][ro + L.pslot + 1] = rho1;
                flags_out(a, kPhaseR, k);
            }
            if (!wait_ph(a, kPhaseR, k)) return;
            rho1 = slot_sum(L, par_ptr(a.G_r, a.gpar, k), 1);
        }
        // A5: test, beta, p = r + beta p (full, replicated)
        const T rel = sqrt(rho1) / (T)st->nb;
        if (rel <= (T)st->tol) {
            if ((vb == 0 && threadIdx.x == 0)) {
                put_hist(st, a.hist, k - 1, rel);
                st->relres = rel; st->iters = k; st->converged = 1; st->status = KS_OK; st->done = 1;
            }
            break;
        }
        const T beta = rho1 / (T)st->rho[(k - 1) & 3];
        const T* Gr = par_ptr(a.G_r, a.gpar, k);
        if (a.peer && a.ll) {                           // p = r + beta p, r polled from the LL slots
            bool ok = true;
            jitter_at(a.jitter, 9u);
            for (int64_t j = tid0; j < L.n && ok; j += gstride) {
                double rj = 0.0;
                ok = ll_get_sys(a.llg + ll_vec_off(L.ld, (int)(k & 1), 0, j), ep, rj);
                a.p_full[j] = fma(beta, a.p_full[j], (T)rj);
            }
            if (!ok) { st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1; return; }
        } else {
            for (int64_t j = tid0; j < L.n; j += gstride) {
                int o;
                const int64_t gj = gidx_owner(L, j, &o);
                a.p_full[j] = fma(beta, a.p_full[j], Gr[gj]);
            }
        }
        if ((vb == 0 && threadIdx.x == 0)) {
            put_hist(st, a.hist, k - 1, rel);
            st->relres = rel; st->iters = k; st->rho[k & 3] = rho1; st->alpha[k & 3] = alpha;
            if (!a.peer) a.G_r[ro + L.pslot + 1] = rho1;    // for the multi-kernel path / finish
        }
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
    }
}

// ---------------------------------------------------------- BiCGSTAB (B1-B8)
template <class T, int kR, int kU>
__device__ __forceinline__ void bs_persist_body(const PersistArgs<T>& P, int vb, int vg) {
    __shared__ T red[(kR > 2 ? kR : 2) * kNW];
    const VecArgsT<T>& a = P.a;
    const Layout& L = a.L;
    DevState* st = a.st;
    const int64_t m = rows_of(L), r0 = L.row0[L.rank];
    const int64_t gstride = (int64_t)vg * kNT;
    const int64_t tid0 = (int64_t)vb * kNT + threadIdx.x;
    // scalars of the previous iteration (written by the previous launch / init)
    T rho_prev = (T)st->rho[(P.k0 - 1) & 3], alpha_prev = (T)st->alpha[(P.k0 - 1) & 3];
    T omega_prev = (T)st->omega[(P.k0 - 1) & 3];
    T rho_next = T(0), rr_next = T(0);
    for (long long i = P.k0; i <= P.k1; ++i) {
        if (is_done(st)) break;
        // B8 (test of i-1) + B1
        const bool llx = a.peer && a.ll;               // LL handovers (KS_OPT_LL_XCHG)
        const uint32_t ep_prev = ll_epoch(st, i - 1), ep = ll_epoch(st, i);
        const int par_prev = (int)((i - 1) & 1), par = (int)(i & 1);
        if (a.peer && !llx && i >= 2 && !wait_ph(a, kPhaseR, i - 1)) return;
        const T* Gr = par_ptr(a.G_r, a.gpar, i - 1);
        // P == 1: after the first iteration of a launch the partials are in registers
        // (every CTA computed them), so no barrier is needed to read the lead's slots
        const bool carried = !a.peer && i > P.k0;
        T rv_prev[2] = {T(0), T(0)};
        if (llx && i >= 2 && !ll_sum_scal<2>(a, par_prev, 1, ep_prev, rv_prev)) return;
        const T rho = carried ? rho_next : (llx && i >= 2) ? rv_prev[0] : slot_sum(L, Gr, 0);
        T rel = T(0);
        if (i >= 2) {
            rel = sqrt(carried ? rr_next : llx ? rv_prev[1] : slot_sum(L, Gr, 1)) / (T)st->nb;
            if (rel <= (T)st->tol) {
                if ((vb == 0 && threadIdx.x == 0)) {
                    put_hist(st, a.hist, i - 2, rel);
                    st->relres = rel; st->iters = i - 1; st->converged = 1; st->status = KS_OK; st->done = 1;
                }
                break;
            }
        }
        if (rho == T(0) || !isfinite(rho)) {
            if ((vb == 0 && threadIdx.x == 0)) {
                if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
                st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1;
            }
            break;
        }
        if (i == 1) {
            for (int64_t j = tid0; j < L.n; j += gstride) {
                int o;
                a.p_full[j] = Gr[gidx_owner(L, j, &o)];
            }
        } else if (llx) {                               // r of i-1 polled from the LL slots
            const T beta = (rho / rho_prev) * (alpha_prev / omega_prev);
            bool ok = true;
            jitter_at(a.jitter, 9u);
            for (int64_t j = tid0; j < L.n && ok; j += gstride) {
                double rj = 0.0;
                ok = ll_get_sys(a.llg + ll_vec_off(L.ld, par_prev, 0, j), ep_prev, rj);
                a.p_full[j] = fma(beta, fma(-omega_prev, a.v_full[j], a.p_full[j]), (T)rj);
            }
            if (!ok) { st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1; return; }
        } else {
            const T beta = (rho / rho_prev) * (alpha_prev / omega_prev);
            for (int64_t j = tid0; j < L.n; j += gstride) {
                int o;
                const int64_t gj = gidx_owner(L, j, &o);
                a.p_full[j] = fma(beta, fma(-omega_prev, a.v_full[j], a.p_full[j]), Gr[gj]);
            }
        }
        if ((vb == 0 && threadIdx.x == 0)) {
            if (i >= 2) { put_hist(st, a.hist, i - 2, rel); st->relres = rel; }
            st->rho[i & 3] = rho;
            st->iters = i - 1;
        }
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        // B3: v = A p (own chunk of G_v[i&1]), <rhat, v>_g
        const int64_t vo = (i & 1) * a.gpar + (int64_t)L.rank * L.chunk;
        T d1, d2;
        gemv_phase<kR, kU>(P, a.p_full, a.G_v + vo, a.rhat_loc, d1, d2, red, (const T*)nullptr, vb, vg);
        if (threadIdx.x == 0) P.bpart[vb * 4 + 0] = d1;
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        T gm[1];
        grid_total<1>(P.bpart, 0, gm, red, vg);
        T gam = gm[0];
        if (llx) {                                      // B2/B4: v rows and the rank partial as LL words
            if ((vb == 0 && threadIdx.x == 0)) {
                const double g1 = (double)gam;
                ll_push_scal(a, par, 0, &g1, 1, ep);
            }
            jitter_at(a.jitter, 8u);
            for (int64_t l = tid0; l < m; l += gstride) {
                const double vl = (double)a.G_v[vo + l];
                for (int g = 0; g < L.P; ++g) ll_put_sys(a.pp.llg[g] + ll_vec_off(L.ld, par, 1, r0 + l), vl, ep);
            }
            if (!ll_sum_scal<1>(a, par, 0, ep, gm)) return;
            gam = gm[0];
        } else if (a.peer) {                            // B2/B4: v pulled, partial pushed
            if ((vb == 0 && threadIdx.x == 0)) {
                for (int g = 0; g < L.P; ++g) a.pp.G_v[g][vo + L.pslot] = gam;
                flags_out(a, kPhaseV, i);
            }
            if (!wait_ph(a, kPhaseV, i)) return;
            gam = slot_sum(L, par_ptr(a.G_v, a.gpar, i), 0);
        }
        if (gam == T(0) || !isfinite(gam)) {
            if ((vb == 0 && threadIdx.x == 0)) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
            break;
        }
        const T alpha = rho / gam;
        // B4/B5: s = r - alpha v (full n, redundant), ||s||^2
        T sacc[1] = {T(0)};
        if (llx) {
            bool ok = true;
            jitter_at(a.jitter, 9u);
            for (int64_t j = tid0; j < L.n && ok; j += gstride) {
                double vj = 0.0, rj = 0.0;
                ok = ll_get_sys(a.llg + ll_vec_off(L.ld, par, 1, j), ep, vj);
                if (i >= 2) {
                    ok = ok && ll_get_sys(a.llg + ll_vec_off(L.ld, par_prev, 0, j), ep_prev, rj);
                } else {
                    int o;
                    rj = (double)Gr[gidx_owner(L, j, &o)];
                }
                const T v = (T)vj;
                a.v_full[j] = v;
                const T s = fma(-alpha, v, (T)rj);
                a.s_full[j] = s;
                sacc[0] = fma(s, s, sacc[0]);
            }
            if (!ok) { st->peer_timeout = 1; st->status = KS_ENCCL; st->done = 1; return; }
        } else {
            for (int64_t j = tid0; j < L.n; j += gstride) {
                int o;
                const int64_t gj = gidx_owner(L, j, &o);
                const T v = a.peer ? __ldcg(a.pp.G_v[o] + (i & 1) * a.gpar + gj)
                                        : a.G_v[(i & 1) * a.gpar + gj];
                a.v_full[j] = v;
                const T s = fma(-alpha, v, Gr[gj]);
                a.s_full[j] = s;
                sacc[0] = fma(s, s, sacc[0]);
            }
        }
        block_sum<kNT, 1>(sacc, red);
        if (threadIdx.x == 0) P.bpart[vb * 4 + 1] = sacc[0];
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        T ssv[1];
        grid_total<1>(P.bpart, 1, ssv, red, vg);
        const T srel = sqrt(ssv[0]) / (T)st->nb;
        if (srel <= (T)st->tol) {                          // half-step exit
            for (int64_t l = tid0; l < m; l += gstride) a.x_loc[l] = fma(alpha, a.p_full[r0 + l], a.x_loc[l]);
            if ((vb == 0 && threadIdx.x == 0)) {
                put_hist(st, a.hist, i - 1, srel);
                st->alpha[i & 3] = alpha;
                st->relres = srel; st->half = 1; st->half_iter = i; st->converged = 1;
                st->status = KS_OK; st->iters = i; st->done = 1;
            }
            break;
        }
        // B6: t = A s (q_loc), <t, s_loc>_g, <t, t>_g
        gemv_phase<kR, kU>(P, a.s_full, a.q_loc, a.s_full + r0, d1, d2, red, (const T*)nullptr, vb, vg);
        if (threadIdx.x == 0) { P.bpart[vb * 4 + 2] = d1; P.bpart[vb * 4 + 3] = d2; }
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        T tv[2];
        grid_total<2>(P.bpart, 2, tv, red, vg);
        T ts = tv[0], tt = tv[1];
        if (llx) {                                      // B7 C2 as LL words
            if ((vb == 0 && threadIdx.x == 0)) {
                const double w2[2] = {(double)ts, (double)tt};
                ll_push_scal(a, par, 2, w2, 2, ep);
            }
            if (!ll_sum_scal<2>(a, par, 2, ep, tv)) return;
            ts = tv[0];
            tt = tv[1];
        } else if (a.peer) {                            // B7 fused C2
            if ((vb == 0 && threadIdx.x == 0)) {
                for (int g = 0; g < L.P; ++g) {
                    a.pp.S[g][(i & 1) * a.spar + L.rank * kScalSlot + 0] = ts;
                    a.pp.S[g][(i & 1) * a.spar + L.rank * kScalSlot + 1] = tt;
                }
                flags_out(a, kPhaseS, i);
            }
            if (!wait_ph(a, kPhaseS, i)) return;
            ts = scal_sum(L, par_ptr(a.S, a.spar, i), 0);
            tt = scal_sum(L, par_ptr(a.S, a.spar, i), 1);
        }
        const T om = ts / tt;
        if (tt == T(0) || !isfinite(tt) || om == T(0) || !isfinite(om)) {
            if ((vb == 0 && threadIdx.x == 0)) { st->status = KS_EBREAKDOWN; st->breakdown = 1; st->iters = i - 1; st->done = 1; }
            break;
        }
        // B7: x += alpha p + omega s; r = s - omega t; <rhat, r>_g, <r, r>_g
        const int64_t ro = (i & 1) * a.gpar + (int64_t)L.rank * L.chunk;
        T acc[2] = {T(0), T(0)};
        if (llx) jitter_at(a.jitter, 8u);
        for (int64_t l = tid0; l < m; l += gstride) {
            const T s = a.s_full[r0 + l];
            a.x_loc[l] = fma(om, s, fma(alpha, a.p_full[r0 + l], a.x_loc[l]));
            const T r = fma(-om, a.q_loc[l], s);
            if (llx) {
                a.G_r[ro + l] = r;
                for (int g = 0; g < L.P; ++g) ll_put_sys(a.pp.llg[g] + ll_vec_off(L.ld, par, 0, r0 + l), (double)r, ep);
            } else if (a.peer) {
                for (int g = 0; g < L.P; ++g) a.pp.G_r[g][ro + l] = r;
            } else {
                a.G_r[ro + l] = r;
            }
            acc[0] = fma(a.rhat_loc[l], r, acc[0]);
            acc[1] = fma(r, r, acc[1]);
        }
        if (a.peer && !llx && tid0 < m) __threadfence_system();   // only threads that stored remotely
        block_sum<kNT, 2>(acc, red);
        if (threadIdx.x == 0) { P.bpart[vb * 4 + 0] = acc[0]; P.bpart[vb * 4 + 1] = acc[1]; }
        if (!grid_sync_n(P.bar, st, (unsigned)vg)) return;
        T rv[2];
        grid_total<2>(P.bpart, 0, rv, red, vg);
        if ((vb == 0 && threadIdx.x == 0)) {
            if (llx) {                                  // consumed at the top of i + 1
                const double w2[2] = {(double)rv[0], (double)rv[1]};
                ll_push_scal(a, par, 1, w2, 2, ep);
            }
            // the flag protocol also at the solve's last step: k_end tests it from G_r
            if (a.peer && (!llx || i == (long long)st->maxit)) {
                for (int g = 0; g < L.P; ++g) {
                    a.pp.G_r[g][ro + L.pslot + 0] = rv[0];
                    a.pp.G_r[g][ro + L.pslot + 1] = rv[1];
                }
                flags_out(a, kPhaseR, i);
            } else if (!a.peer) {
                a.G_r[ro + L.pslot + 0] = rv[0];
                a.G_r[ro + L.pslot + 1] = rv[1];
            }
            st->alpha[i & 3] = alpha;
            st->omega[i & 3] = om;
            st->iters = i;
        }
        rho_prev = rho;
        alpha_prev = alpha;
        omega_prev = om;
        rho_next = rv[0];
        rr_next = rv[1];
        // fused: the next iteration waits on the R flags; P == 1: the values are
        // carried in registers and the lead's slots are read only by the next launch
    }
}

template <class T, int kR, int kU, int kMinB = 4>
__global__ void __launch_bounds__(kNT, kMinB) k_cg_persist(PersistArgs<T> P) {
    cg_persist_body<T, kR, kU>(P, (int)blockIdx.x, (int)gridDim.x);
}
template <class T, int kR, int kU, int kMinB = 4>
__global__ void __launch_bounds__(kNT, kMinB) k_bs_persist(PersistArgs<T> P) {
    bs_persist_body<T, kR, kU>(P, (int)blockIdx.x, (int)gridDim.x);
}

// Ranks sharing one GPU (ks_create_on): every rank's persistent kernel as ONE
// cooperative launch of P * g CTAs -- CTA b serves rank b / g as its block b % g, with
// its rank's arguments -- so the CTAs that wait on each other's exchanges are
// co-resident by construction (separate launches on one GPU would not be).
constexpr int kMaxEmuP = kMaxEmuRanks;
template <class T>
struct PersistEmuArgs {
    PersistArgs<T> p[kMaxEmuP];
    int P, g;
};
template <class T, int kR, int kU>
__global__ void __launch_bounds__(kNT, 4) k_cg_persist_emu(const __grid_constant__ PersistEmuArgs<T> E) {
    const int rk = (int)blockIdx.x / E.g;
    cg_persist_body<T, kR, kU>(E.p[rk], (int)blockIdx.x - rk * E.g, E.g);
}
template <class T, int kR, int kU>
__global__ void __launch_bounds__(kNT, 4) k_bs_persist_emu(const __grid_constant__ PersistEmuArgs<T> E) {
    const int rk = (int)blockIdx.x / E.g;
    bs_persist_body<T, kR, kU>(E.p[rk], (int)blockIdx.x - rk * E.g, E.g);
}

// Persistent GEMV shape: default R=2, U=4 (the sweep's best: CG 211.5 / BiCGSTAB
// 105.3 it/s at n = 65536 vs 206.6 / 103.4 for R=4/U=2, profiles/r01_persist_sweep.json);
// (4,2) and (4,4) selectable through KS_OPT_GEMV_ROWS / KS_OPT_GEMV_UNROLL.
// (1, 8): one-row tiles for shards whose 2-row tile count would leave a badly filled
// last wave over the resident CTAs (ks_solvers.cpp persist_shape).
// KS_GEMV_DEFER=1 (tuning): deferred row reductions in the persistent GEMV phase.
int defer_gemv() {
    static const int v = [] {
        const char* e = std::getenv("KS_GEMV_DEFER");
        return e && std::atoi(e) == 1 ? 1 : 0;
    }();
    return v;
}
// KS_PERSIST_OCC=5 (tuning): the default (2, 4) shape compiled for 5 CTAs per SM
// (48 registers; the GEMV loop stays spill-free) instead of 4 (64 registers).
bool occ5() {
    static const bool v = [] {
        const char* e = std::getenv("KS_PERSIST_OCC");
        return e && std::atoi(e) == 5;
    }();
    return v;
}
template <class T>
const void* pick(int bicgstab, int rows, int unroll) {
    const int shape = (rows == 4 && unroll == 2) ? 1 : (rows == 4 && unroll == 4) ? 2 : (rows == 1) ? 3 : 0;
    if (shape == 0 && occ5())
        return bicgstab ? (const void*)k_bs_persist<T, 2, 4, 5> : (const void*)k_cg_persist<T, 2, 4, 5>;
    if (bicgstab) {
        return shape == 1 ? (const void*)k_bs_persist<T, 4, 2>
             : shape == 2 ? (const void*)k_bs_persist<T, 4, 4>
             : shape == 3 ? (const void*)k_bs_persist<T, 1, 8> : (const void*)k_bs_persist<T, 2, 4>;
    }
    return shape == 1 ? (const void*)k_cg_persist<T, 4, 2>
         : shape == 2 ? (const void*)k_cg_persist<T, 4, 4>
         : shape == 3 ? (const void*)k_cg_persist<T, 1, 8> : (const void*)k_cg_persist<T, 2, 4>;
}
int rows_of(int rows, int unroll) {
    return (rows == 4 && (unroll == 2 || unroll == 4)) ? 4 : rows == 1 ? 1 : 2;
}

int coop_grid(const void* kern, int num_sms, int64_t mmax, int R) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNT, 0);
    if (per_sm < 1) per_sm = 1;
    const int64_t cap = (int64_t)per_sm * num_sms;
    const int64_t tiles = (mmax + R - 1) / R;
    int64_t g = tiles < num_sms ? num_sms : tiles;
    // (Tried in round 2: the fewest CTAs keeping the wave count -- 586 instead of 592 at
    // n = 65536 to fill the last wave; no gain at n = 65536 and a loss where it cut the
    // grid to 512 CTAs (n = 16384, P = 4): fewer loads in flight.  Full occupancy wins.)
    if (g > cap) g = cap;
    return (int)g;
}

}  // namespace

template <class T>
int persist_grid(int bicgstab, int num_sms, int64_t mmax, int rows, int unroll) {
    return coop_grid(pick<T>(bicgstab, rows, unroll), num_sms, mmax, rows_of(rows, unroll));
}

template <class T>
int launch_persist(int bicgstab, const VecArgsT<T>& a, const T* A, int64_t lda, int64_t ncols,
                   T* bpart, unsigned* bar, long long k0, long long k1, int grid, int rows, int unroll,
                   cudaStream_t st, bool bar_zeroed) {
    PersistArgs<T> P;
    P.a = a;
    P.A = A;
    P.lda = lda;
    P.ncols = ncols;
    P.bpart = bpart;
    P.bar = bar;
    P.k0 = k0;
    P.k1 = k1;
    P.defer = defer_gemv();
    void* args[] = {&P};
    cudaError_t e = cudaSuccess;
    if (!bar_zeroed) {
        e = cudaMemsetAsync(bar, 0, sizeof(unsigned long long), st);   // grid_sync counter
        if (e != cudaSuccess) return -(int)e;
    }
    e = cudaLaunchCooperativeKernel(pick<T>(bicgstab, rows, unroll), dim3((unsigned)grid),
                                                dim3(kNT), args, 0, st);
    return e == cudaSuccess ? 1 : -(int)e;
}

// ---- emulated ranks (all on one GPU): one cooperative launch for every rank -------
namespace {
const void* pick_emu(int bicgstab, int rows, int unroll) {
    const int shape = (rows == 4 && unroll == 2) ? 1 : (rows == 4 && unroll == 4) ? 2 : (rows == 1) ? 3 : 0;
    if (bicgstab) {
        return shape == 1 ? (const void*)k_bs_persist_emu<double, 4, 2>
             : shape == 2 ? (const void*)k_bs_persist_emu<double, 4, 4>
             : shape == 3 ? (const void*)k_bs_persist_emu<double, 1, 8> : (const void*)k_bs_persist_emu<double, 2, 4>;
    }
    return shape == 1 ? (const void*)k_cg_persist_emu<double, 4, 2>
         : shape == 2 ? (const void*)k_cg_persist_emu<double, 4, 4>
         : shape == 3 ? (const void*)k_cg_persist_emu<double, 1, 8> : (const void*)k_cg_persist_emu<double, 2, 4>;
}
}  // namespace

int persist_emu_grid(int bicgstab, int num_sms, int P, int64_t mmax, int rows, int unroll) {
    if (P < 2 || P > kMaxEmuP || num_sms < P) return 0;
    return coop_grid(pick_emu(bicgstab, rows, unroll), num_sms / P, mmax, rows_of(rows, unroll));
}

int launch_persist_emu(int bicgstab, const VecArgs* const* a, const double* const* A, int64_t lda, int64_t ncols,
                       double* const* bpart, unsigned* const* bar, long long k0, long long k1, int P, int g,
                       int rows, int unroll, cudaStream_t st) {
    if (P < 2 || P > kMaxEmuP || g < 1) return -(int)cudaErrorInvalidValue;
    PersistEmuArgs<double> E;
    std::memset(&E, 0, sizeof E);
    for (int h = 0; h < P; ++h) {
        PersistArgs<double>& Q = E.p[h];
        Q.a = *a[h];
        Q.A = A[h];
        Q.lda = lda;
        Q.ncols = ncols;
        Q.bpart = bpart[h];
        Q.bar = bar[h];
        Q.k0 = k0;
        Q.k1 = k1;
        Q.defer = defer_gemv();
    }
    E.P = P;
    E.g = g;
    void* args[] = {&E};
    const cudaError_t e = cudaLaunchCooperativeKernel(pick_emu(bicgstab, rows, unroll), dim3((unsigned)(P * g)),
                                                      dim3(kNT), args, 0, st);
    return e == cudaSuccess ? 1 : -(int)e;
}

template int persist_grid<double>(int, int, int64_t, int, int);
template int persist_grid<float>(int, int, int64_t, int, int);
template int launch_persist<double>(int, const VecArgsT<double>&, const double*, int64_t, int64_t, double*,
                                    unsigned*, long long, long long, int, int, int, cudaStream_t, bool);
template int launch_persist<float>(int, const VecArgsT<float>&, const float*, int64_t, int64_t, float*,
                                   unsigned*, long long, long long, int, int, int, cudaStream_t, bool);

}  // namespace ks

// L2: per-GPU schedules of CG and BiCGSTAB
// (sec.8(c).4).  Each local rank runs the same schedule on its own
// stream; NCCL collectives over NVLink carry the vector slices with the partial
// scalars piggybacked:
//   CG        : 1 allgather (r + rho' partials) + 1 scalar allgather (sigma) / iteration
//   BiCGSTAB  : 2 allgathers (v + <rhat,v>; r + <rhat,r>,<r,r>) + 1 scalar allgather
// The host only queues work: scalars never leave the device inside the loop; a
// 4-byte done flag is polled once per batch with one batch in flight.
#include <chrono>
#include <cmath>
#include <cstring>

#include "ks_ctx.h"

namespace ks {

namespace {

using Clock = std::chrono::steady_clock;

// Persistent GEMV shape: the tuning options if set, else R=4/U=2 for small shards
// (<= 4096 rows: fewer, fuller tiles; C1 CG 13.4 vs 15.8 us/iteration,
// profiles/r01_small_sweep.json) and the kernels' default R=2/U=4 above.
// Either default is replaced when its tile count leaves the last wave over the
// resident CTAs (4 per SM) badly filled -- n = 16384 at P = 4 has 1024 four-row
// tiles on 592 CTAs, 1.73 waves, so every GEMV takes 2 waves' time (13 % lost); one-row
// tiles (R = 1, U = 8: still 8 loads of 16 B in flight per thread) give 6.92 -> 7.
void persist_shape(const ks_ctx* c, const Rank& r, int* rows, int* unroll) {
    *rows = (int)c->opt.gemv_rows;
    *unroll = (int)c->opt.gemv_unroll;
    if (*rows != 0 || *unroll != 0) return;
    const int64_t cap = 4LL * r.num_sms, m = r.L.pslot;
    auto fill = [&](int64_t R) {                  // useful fraction of the last-wave-padded work
        const int64_t tiles = (m + R - 1) / R;
        const int64_t G = std::min(tiles, cap);     // coop_grid's CTA count
        const int64_t waves = (tiles + G - 1) / G;
        return (double)tiles / (double)(waves * G);
    };
    // rows of <= 16384 columns (128 KiB): one-row tiles stream faster on one B200 --
    // n = 16384: CG 320.1 -> 313.8 us, BiCGSTAB 646.2 -> 630.7 us; n = 8192: 92.3 ->
    // 87.1 / 183.4 -> 176.7 us per iteration (profiles/r02_defer_ab.jsonl, rows 0 vs 1)
    const int def_r = m <= 4096 ? 4 : (c->ld <= 16384 ? 1 : 2);
    *rows = def_r;
    *unroll = def_r == 4 ? 2 : def_r == 1 ? 8 : 4;
    double best = fill(def_r);
    for (int R : {2, 1}) {
        if (R == def_r) continue;
        const double f = fill(R);
        if (f > best + 0.03) { best = f; *rows = R; *unroll = R == 1 ? 8 : 4; }
    }
}

// Small-n shared-memory kernels (ks_small.cu): their kind for this solve (0 CG,
// 1 BiCGSTAB, 2 CG over P > 1 with the fused exchange), -1 = not used.
int small_kind(const ks_ctx* c, int bicgstab) {
    if (c->opt.small == 0) return -1;
    if (c->opt.small == 2 && c->n * (int64_t)c->esz > ks_ctx::kSmallAutoMaxBytes) return -1;
    if (c->P == 1) return bicgstab ? 1 : 0;
    if (!c->fused()) return -1;
    // BiCGSTAB over P > 1: the shared-memory schedule wins up to 16 KiB vectors
    // (n = 512: 33 -> 20 us/iteration at P = 2); at 32 KiB the general fused
    // kernels are faster (n = 4096, P = 2: 52 vs 60 us), profiles/r01_exchange_cost_small_peer2.jsonl
    if (bicgstab && c->opt.small == 2 && c->n * (int64_t)c->esz > ks_ctx::kSmallAutoMaxBytes / 2) return -1;
    return bicgstab ? 3 : 2;
}
// Launch geometry of a kernel kind, memoised per rank: the occupancy queries behind
// it cost tens of microseconds of host time per call (a context's n, ld and device
// never change).  key: (what << 48) | kind / shape.
template <class F>
int memo_grid(Rank& r, long long key, F&& f) {
    auto it = r.grid_memo.find(key);
    if (it != r.grid_memo.end()) return it->second;
    const int g = f();
    r.grid_memo.emplace(key, g);
    return g;
}

// Grid of the small-n kernels, 0 = not used.
template <class T>
int small_path_grid(const ks_ctx* c, Rank& r, int bicgstab) {
    const int kind = small_kind(c, bicgstab);
    if (kind < 0) return 0;
    int g = memo_grid(r, (1LL << 48) | ((long long)sizeof(T) << 40) | kind,
                      [&] { return small_grid<T>(kind, r.num_sms, r.m, c->ld); });
    if (g > 0 && c->opt.persist_grid > 0) g = (int)std::min<int64_t>(g, c->opt.persist_grid);
    return g;
}

// Iterations per host poll.  KS_OPT_POLL_BATCH = 0 (auto): a persistent kernel runs
// the whole solve in one launch (it stops itself on convergence, so nothing is
// wasted and no launch gap remains); the multi-kernel path queues 16 iterations.
int64_t poll_batch(const ks_ctx* c, bool persist, int64_t maxit) {
    if (c->opt.poll_batch > 0) return c->opt.poll_batch;
    return persist ? std::max<int64_t>(1, maxit) : 16;
}

struct Prof {
    ks_ctx* c;
    Rank& r;
    int64_t per_slot;
    int used[2] = {0, 0};
    Prof(ks_ctx* c_, Rank& r_, int64_t gemvs_per_batch) : c(c_), r(r_), per_slot(gemvs_per_batch) {
        if (!c->opt.profile_gemv) return;
        const size_t need = (size_t)(2 * 2 * per_slot);
        while (r.ev_gemv.size() < need) {
            cudaEvent_t e;
            KS_CUDA(cudaEventCreate(&e));
            r.ev_gemv.push_back(e);
        }
    }
    void begin(int slot) { used[slot] = 0; }
    void pre(int slot) {
        if (!c->opt.profile_gemv) return;
        KS_CUDA(cudaEventRecord(r.ev_gemv[(size_t)(slot * per_slot + used[slot]) * 2], r.stream));
    }
    void post(int slot) {
        if (!c->opt.profile_gemv) return;
        KS_CUDA(cudaEventRecord(r.ev_gemv[(size_t)(slot * per_slot + used[slot]) * 2 + 1], r.stream));
        ++used[slot];
    }
    void harvest(int slot) {
        if (!c->opt.profile_gemv) return;
        for (int q = 0; q < used[slot]; ++q) {
            float ms = 0.f;
            const size_t base = (size_t)(slot * per_slot + q) * 2;
            KS_CUDA(cudaEventElapsedTime(&ms, r.ev_gemv[base], r.ev_gemv[base + 1]));
            r.gemv_seconds += ms * 1e-3;
        }
        used[slot] = 0;
    }
};

// Batched launch loop with a device done flag.  With
// KS_OPT_USE_GRAPHS a full batch of B iterations is captured once into a CUDA
// graph (kernels + NCCL calls) and replayed; the captured kernels read the
// iteration base from r.kdev, which the graph's last node advances by B.
template <class IterFn>
void run_loop(ks_ctx* c, Rank& r, int kind, int64_t maxit, int gemvs_per_iter, IterFn&& iter) {
    const bool persist = c->persistent();
    const int64_t B = poll_batch(c, persist, maxit);
    Prof prof(c, r, persist ? 1 : B * gemvs_per_iter);
    int pgrid = 0, sgrid = 0, tgrid = 0;
    int prows = 0, punroll = 0;
    // tiny kernels: one GPU, the whole solve in one launch (they always finish it)
    // tiny kernels: n <= 1024, the whole solve in one launch (they always finish it);
    // P > 1 only with the fused exchange (their LL slots live in the exchange allocation)
    if (persist && (c->P == 1 || (c->fused() && r.llx)) && c->opt.tiny && c->opt.small != 0 && B >= maxit)
        tgrid = memo_grid(r, (2LL << 48) | kind, [&] { return tiny_grid(kind, r.num_sms, c->n, r.m, c->ld); });
    if (tgrid > 0 && c->P == 1 && !r.ll) {
        dev_alloc_t(&r.ll, (size_t)(4 * c->ld));
        KS_CUDA(cudaMemsetAsync(r.ll, 0, (size_t)(4 * c->ld) * sizeof(uint64_t), r.stream));
    }
    if (persist && tgrid == 0) sgrid = small_path_grid<double>(c, r, kind);
    if (persist && tgrid == 0 && sgrid == 0) {
        persist_shape(c, r, &prows, &punroll);
        pgrid = memo_grid(r, (3LL << 48) | ((long long)prows << 24) | ((long long)punroll << 8) | kind,
                          [&] { return persist_grid<double>(kind, r.num_sms, r.L.pslot, prows, punroll); });
        if (c->opt.persist_grid > 0) pgrid = (int)std::min<int64_t>(pgrid, c->opt.persist_grid);
    }
    const bool use_graph = !persist && c->opt.use_graphs && !c->opt.profile_gemv && B >= 2 && maxit >= B;
    Rank::GraphCache* g = nullptr;
    if (use_graph) {
        g = &r.graphs[kind];
        const GemvConfig cfg = gemv_config(c, r);
        if (!(g->exec && g->kind == kind && g->B == B && g->hist == r.hist && g->variant == cfg.variant &&
              g->rows == cfg.rows && g->splits == cfg.splits && g->fused == (c->fused() ? 1 : 0))) {
            if (g->exec) { KS_CUDA(cudaGraphExecDestroy(g->exec)); g->exec = nullptr; }
            const int64_t before = r.launches;
            cudaGraph_t graph;
            KS_CUDA(cudaStreamBeginCapture(r.stream, cudaStreamCaptureModeThreadLocal));
            for (int64_t j = 1; j <= B; ++j) iter(r.kdev, j, prof, 0);
            r.launches += launch_advance(r.kdev, B, r.stream);
            KS_CUDA(cudaStreamEndCapture(r.stream, &graph));
            KS_CUDA(cudaGraphInstantiate(&g->exec, graph, 0));
            KS_CUDA(cudaGraphDestroy(graph));
            g->kind = kind; g->B = B; g->hist = r.hist;
            g->variant = cfg.variant; g->rows = cfg.rows; g->splits = cfg.splits;
            g->fused = c->fused() ? 1 : 0;
            g->launches = r.launches - before;
            r.launches = before;
        }
        KS_CUDA(cudaMemsetAsync(r.kdev, 0, sizeof(long long), r.stream));
    }
    int64_t k = 1;
    int64_t batch = 0;
    KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
    while (k <= maxit) {
        const int slot = (int)(batch & 1);
        prof.begin(slot);
        if (persist) {                                    // one cooperative launch per batch
            const int64_t kend = std::min<int64_t>(maxit, k + B - 1);
            prof.pre(slot);
            const bool z = r.bar_zeroed && k == 1;
            const int rc = tgrid > 0
                ? launch_tiny(kind, r.vargs(c->fused()), r.A, c->ld, c->P == 1 ? r.ll : r.llx, r.llpeer,
                              r.x0_full, tgrid, r.stream)
                : sgrid > 0
                ? launch_small<double>(small_kind(c, kind), r.vargs(c->fused()), r.A, c->ld, c->ld,
                                       r.scr.part + 2 * kPartStride, r.scr.ticket + 8, k, kend, sgrid, r.stream, z)
                : launch_persist<double>(kind, r.vargs(c->fused()), r.A, c->ld, c->ld,
                                         r.scr.part + 2 * kPartStride, r.scr.ticket + 8, k, kend, pgrid,
                                         prows, punroll, r.stream, z);
            prof.post(slot);
            if (rc < 0) KS_CUDA((cudaError_t)(-rc));
            r.launches += 1;
            r.gemv_launches += (kend - k + 1) * gemvs_per_iter;
            k = kend + 1;
            if (k > maxit) break;        // last launch: nothing left to stop early
        } else if (use_graph && k + B - 1 <= maxit) {
            KS_CUDA(cudaGraphLaunch(g->exec, r.stream));   // iterations k .. k+B-1
            r.launches += g->launches;
            r.gemv_launches += B * gemvs_per_iter;
            k += B;
        } else {
            const int64_t kend = std::min<int64_t>(maxit, k + B - 1);
            for (; k <= kend; ++k) iter(nullptr, k, prof, slot);
        }
        KS_CUDA(cudaMemcpyAsync(&r.h_done[slot], &r.st->done, sizeof(int), cudaMemcpyDeviceToHost,
                                r.stream));
        KS_CUDA(cudaEventRecord(r.ev_poll[slot], r.stream));
        if (batch >= 1) {
            KS_CUDA(cudaEventSynchronize(r.ev_poll[slot ^ 1]));
            prof.harvest(slot ^ 1);
            if (r.h_done[slot ^ 1]) { ++batch; break; }
        }
        ++batch;
    }
    r.bar_zeroed = false;
    KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
    if (c->opt.profile_gemv) {            // otherwise finish_and_copy's synchronisation covers it
        KS_CUDA(cudaStreamSynchronize(r.stream));
        prof.harvest(0);
        prof.harvest(1);
    }
}

void gemv(ks_ctx* c, Rank& r, const GemvParams& p) {
    r.launches += launch_gemv(p, gemv_config(c, r), r.scr, 1, r.num_sms, r.stream);
}

GemvParams gp(const ks_ctx* c, const Rank& r, const double* x, double* y) {
    GemvParams p{};
    p.A = r.A;
    p.lda = c->ld;
    p.m = r.m;
    p.ncols = c->ld;
    p.x = x;
    p.y = y;
    return p;
}

// Setup shared by both methods (rows A0 / B0): b and x0 in; r0 = b - A x0
// (K1 residual mode) or r0 = b; x_loc; rhat; partial <r0, r0>; allgather G_r.
void ensure_hist(Rank& r, int64_t hist_cap) {
    if (hist_cap > r.hist_alloc) {
        retire(r, r.hist);
        r.hist = nullptr;
        r.hist_alloc = std::max<int64_t>(hist_cap, 2 * r.hist_alloc);
        dev_alloc_t(&r.hist, (size_t)r.hist_alloc);
    }
}

// CG / BiCGSTAB with x0 = 0: b in, then rows A0/B0 + state init (+ the rendezvous
// for the fused exchange) as ONE kernel (launch_start).
void start(ks_ctx* c, Rank& r, int bicgstab, const double* b, double tol, int64_t maxit, int64_t hist_cap,
           unsigned long long ebase) {
    ensure_hist(r, hist_cap);
    KS_CUDA(cudaMemcpyAsync(r.b_full, b, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
    r.launches += launch_start(r.vargs(c->fused()), bicgstab, tol, maxit, hist_cap, ebase,
                               c->fused() ? c->opt.join_timeout_ms : 0, r.stream);
    r.bar_zeroed = true;
}

void setup(ks_ctx* c, Rank& r, const double* b, const double* x0, int64_t hist_cap) {
    const size_t nbytes = (size_t)c->n * sizeof(double);
    ensure_hist(r, hist_cap);
    KS_CUDA(cudaMemcpyAsync(r.b_full, b, nbytes, cudaMemcpyDefault, r.stream));
    VecArgs a = r.vargs(false);   // setup gathers r0 with NCCL into parity 0
    if (x0) {
        KS_CUDA(cudaMemcpyAsync(r.s_full, x0, nbytes, cudaMemcpyDefault, r.stream));
        GemvParams p = gp(c, r, r.s_full, r.G_r + (int64_t)r.rank * r.L.chunk);
        p.bsub = r.b_full + r.row0;
        gemv(c, r, p);
        r.launches += launch_setup_r(a, true, r.s_full, r.stream);
    } else if (c->P > 1) {
        r.launches += launch_setup_local(a, r.stream);   // r0 = b: every rank has all of b
        return;
    } else {
        r.launches += launch_setup_r(a, false, nullptr, r.stream);
    }
    allgather(c, r, r.G_r, r.L.chunk);
}

// Final x: gather, optional true residual ||b - A x|| (one extra GEMV), copy out.
// end_mode: 0 = the caller already ran its finish kernel (x gathered with NCCL for
// P > 1); 1 = CG / BiCGSTAB: launch_end runs the finish decisions and, with the
// fused exchange, gathers x into every rank's contiguous X over NVLink (no NCCL
// call, no extra launch).  One stream synchronisation when the history is short.
void finish_and_copy(ks_ctx* c, Rank& r, double* x, double* hist, int64_t hist_cap,
                     ks_report* rep, bool bicgstab, const Clock::time_point& t_start, int64_t maxit,
                     int end_mode = 0, unsigned long long x_epoch = 0, bool x_ready = false,
                     bool emulated = false) {
    VecArgs a = r.vargs(false);   // final x gather / true residual: NCCL, parity 0
    const bool fused_x = end_mode == 1 && c->P > 1 && c->fused();
    // emulated ranks: the solve ran in the fused layout (parity-buffered slots), so
    // k_end's last-step test reads it with the fused arguments (its flags are all set)
    if (end_mode == 1) r.launches += launch_end(r.vargs(c->fused() || emulated), bicgstab ? 1 : 0,
                                                fused_x ? 1 : 0, x_epoch, r.stream);
    // contiguous full x: P == 1 x_loc; fused: gathered into X by k_end; x_ready: the
    // emulated-rank tiny kernels wrote it into X
    const double* xsrc = c->P == 1 ? r.x_loc : (fused_x || x_ready) ? r.X : nullptr;
    if (c->P > 1 && !fused_x && !x_ready) {
        r.launches += launch_pack_x(a, r.stream);
        allgather(c, r, r.G_v, r.L.chunk);
    }
    if (c->opt.true_residual) {
        if (xsrc) KS_CUDA(cudaMemcpyAsync(r.s_full, xsrc, (size_t)c->n * sizeof(double),
                                          cudaMemcpyDeviceToDevice, r.stream));
        else copy_chunks_to(c, r, r.G_v, r.s_full, cudaMemcpyDeviceToDevice);
        GemvParams p = gp(c, r, r.s_full, r.q_loc);
        p.bsub = r.b_full + r.row0;
        p.out2 = r.S + (int64_t)r.rank * kScalSlot + 1;
        gemv(c, r, p);
        allgather(c, r, r.S, kScalSlot);
        r.launches += launch_true_res_final(a, r.stream);
    }
    KS_CUDA(cudaMemcpyAsync(r.h_state, r.st, sizeof(DevState), cudaMemcpyDeviceToHost, r.stream));
    const bool out = c->writes_host(r);
    if (out) {                            // x does not depend on the state: same synchronisation
        if (xsrc) KS_CUDA(cudaMemcpyAsync(x, xsrc, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
        else copy_chunks_to(c, r, r.G_v, x, cudaMemcpyDefault);
    }
    // history: at most min(maxit, hist_cap) entries; a short one is staged in pinned
    // memory in the same batch (the valid prefix is copied out after the one sync)
    const int64_t nh_max = std::min<int64_t>(hist_cap, maxit);
    const bool staged = out && hist && nh_max > 0 && nh_max <= kHistStage;
    if (staged)
        KS_CUDA(cudaMemcpyAsync(r.h_hist, r.hist, (size_t)nh_max * sizeof(double), cudaMemcpyDeviceToHost,
                                r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    const DevState& s = *r.h_state;
    if (out) {
        const int64_t nh = std::min<int64_t>(s.iters, hist_cap);
        if (hist && nh > 0) {
            if (staged) {
                cudaPointerAttributes at{};
                const bool dev_dst = cudaPointerGetAttributes(&at, hist) == cudaSuccess &&
                                     at.type == cudaMemoryTypeDevice;
                if (!dev_dst) {
                    std::memcpy(hist, r.h_hist, (size_t)nh * sizeof(double));
                } else {
                    KS_CUDA(cudaMemcpyAsync(hist, r.hist, (size_t)nh * sizeof(double), cudaMemcpyDefault, r.stream));
                    KS_CUDA(cudaStreamSynchronize(r.stream));
                }
            } else {
                KS_CUDA(cudaMemcpyAsync(hist, r.hist, (size_t)nh * sizeof(double), cudaMemcpyDefault,
                                        r.stream));
                KS_CUDA(cudaStreamSynchronize(r.stream));
            }
        }
    }
    if (rep) {
        float ms = 0.f;
        KS_CUDA(cudaEventElapsedTime(&ms, r.ev_t0, r.ev_t1));
        ks_report R;
        std::memset(&R, 0, sizeof R);
        R.iterations = s.iters;
        R.half_step_exit = s.half;
        R.matvecs = bicgstab ? 2 * s.iters - (s.half ? 1 : 0) : s.iters;
        R.converged = s.converged;
        R.breakdown = s.breakdown;
        R.status = s.status;
        R.relres = s.relres;
        R.true_relres = (c->opt.true_residual && s.nb > 0) ? std::sqrt(s.true_rr) / s.nb
                        : (s.bzero ? 0.0 : -1.0);
        R.seconds_loop = ms * 1e-3;
        R.seconds_total = std::chrono::duration<double>(Clock::now() - t_start).count();
        R.seconds_gemv = r.gemv_seconds;
        R.gemv_launches = r.gemv_launches;
        R.kernel_launches = r.launches;
        *rep = R;
    }
}

void check_loaded(const ks_ctx* c, const Rank& r) {
    (void)c;
    if (r.loaded_count < r.m)
        throw KsError(KS_ESTATE, "matrix not fully loaded: call ks_load_rows / ks_generate first");
}

}  // namespace

// Fused-publish parameters of a K1 launch (peer mode): the y rows of this rank
// (y_base: parity-0 chunk base in the G buffer of every rank, or none) and the dot
// partials (slot base in G or S of every rank) go straight to every rank, then
// the flag of `phase` is released with the iteration's epoch.
void fuse_gemv(const ks_ctx* c, const Rank& r, GemvParams& p, int phase, double* const* ybase,
               int64_t ypar, double* const* dbase, int64_t doff, int64_t dpar) {
    p.pub_P = c->P;
    p.pub_rank = r.rank;
    for (int g = 0; g < c->P; ++g) {
        p.y_peer[g] = ybase ? ybase[g] + (int64_t)r.rank * r.L.chunk : nullptr;
        p.d_peer[g] = dbase[g] + doff;
        p.f_peer[g] = r.pp.flags[g] + phase * kMaxRanks + r.rank;
    }
    p.ypar = ypar;
    p.dpar = dpar;
    p.ebase = &r.st->ebase;
}

// Ranks sharing one GPU (ks_create_on with every rank on the same device), x0 = 0, the
// whole solve in one launch: every rank's kernel in ONE cooperative launch over all
// ranks' CTAs (rank = block / g) -- the tiny kernels for n <= 1024, else the persistent
// kernels -- so the fused exchange between ranks (LL words / peer stores + flags) runs
// with the waiting CTAs co-resident by construction.  The plan depends only on
// context state, so every rank decides the same; g == 0: not applicable (the
// host-collective schedule runs).
struct EmuPlan {
    int tiny = 0, g = 0, rows = 0, unroll = 0;
};
EmuPlan emu_plan(const ks_ctx* c, int bicgstab, int64_t maxit) {
    EmuPlan e;
    if (!c->shared_dev || c->P < 2 || c->P > kMaxEmuRanks || c->dtype != KS_FLOAT64 || c->opt.persistent == 0)
        return e;
    if (c->opt.poll_batch > 0 && c->opt.poll_batch < maxit) return e;
    for (const auto& h : c->ranks)
        if (h.dev != c->ranks[0].dev || !h.llg) return e;
    const Rank& r0 = c->ranks[0];                  // the first ranks hold the extra rows
    if (c->opt.tiny && c->opt.small != 0 && r0.llx) {
        const int g = tiny_grid(bicgstab, r0.num_sms, c->n, r0.m, c->ld);
        if (g > 0 && tiny_emu_fits(bicgstab, c->ld, c->P * g, r0.num_sms)) {
            e.tiny = 1;
            e.g = g;
            return e;
        }
    }
    e.rows = c->opt.gemv_rows ? (int)c->opt.gemv_rows : (r0.L.pslot <= 4096 ? 4 : 2);
    e.unroll = c->opt.gemv_unroll ? (int)c->opt.gemv_unroll : (e.rows == 4 ? 2 : 4);
    e.g = persist_emu_grid(bicgstab, r0.num_sms, c->P, r0.L.pslot, e.rows, e.unroll);
    return e;
}

int64_t run_emu(ks_ctx* c, Rank& r, int bicgstab, const double* b, double tol, int64_t maxit,
                double* x, double* hist, int64_t hist_cap, ks_report* rep, const EmuPlan& plan) {
    const auto t_start = Clock::now();
    r.launches = 0;
    r.gemv_launches = 0;
    r.gemv_seconds = 0.0;
    ensure_hist(r, hist_cap);
    const unsigned long long ebase = r.epoch_next;
    r.epoch_next += (unsigned long long)maxit + 2;
    r.x0_full = nullptr;
    KS_CUDA(cudaMemcpyAsync(r.b_full, b, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
    // rows A0 / B0 + state init in the fused layout (also zeroes the grid-barrier
    // counter); no rendezvous (no cross-launch wait)
    r.launches += launch_start(r.vargs(true), bicgstab, tol, maxit, hist_cap, ebase, 0, r.stream);
    host_launch_once(c, r, [&] {
        VecArgs va[kMaxRanks];
        const VecArgs* av[kMaxRanks];
        const double* Av[kMaxRanks];
        uint64_t* llv[kMaxRanks];
        uint64_t* const* llpv[kMaxRanks];
        double* bp[kMaxRanks];
        unsigned* bar[kMaxRanks];
        for (int h = 0; h < c->P; ++h) {
            Rank& rh = c->ranks[(size_t)h];
            va[h] = rh.vargs(true);
            av[h] = &va[h];
            Av[h] = rh.A;
            llv[h] = rh.llx;
            llpv[h] = rh.llpeer;
            bp[h] = rh.scr.part + 2 * kPartStride;
            bar[h] = rh.scr.ticket + 8;
        }
        // loop time = the emulated launch alone (after the waits for every rank's start)
        KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
        const int rc = plan.tiny
            ? launch_tiny_emu(bicgstab, av, Av, c->ld, llv, llpv, c->P, plan.g, r.stream)
            : launch_persist_emu(bicgstab, av, Av, c->ld, c->ld, bp, bar, 1, maxit, c->P, plan.g, plan.rows,
                                 plan.unroll, r.stream);
        if (rc < 0) KS_CUDA((cudaError_t)(-rc));
        KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
        r.launches += 1;
    });
    if (r.rank != 0) {                    // the launch ran on rank 0's stream
        KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
        KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
    }
    r.bar_zeroed = false;
    // tiny: the kernels wrote the full x into every rank's X; persistent: x is gathered
    // by the host collective (pack + allgather), as on the host-collective schedule
    finish_and_copy(c, r, x, hist, hist_cap, rep, bicgstab != 0, t_start, maxit, 1,
                    ebase + (unsigned long long)maxit + 1, plan.tiny != 0, true);
    r.gemv_launches = bicgstab ? 2 * r.h_state->iters - (r.h_state->half ? 1 : 0) : r.h_state->iters;
    if (rep) rep->gemv_launches = r.gemv_launches;
    return r.h_state->peer_timeout ? (int64_t)KS_ENCCL : r.h_state->status;
}

int64_t run_cg(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol, int64_t maxit,
               double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    if (!x0) {
        const EmuPlan plan = emu_plan(c, 0, maxit);
        if (plan.g > 0) {
            check_loaded(c, r);
            return run_emu(c, r, 0, b, tol, maxit, x, hist, hist_cap, rep, plan);
        }
    }
    const auto t_start = Clock::now();
    check_loaded(c, r);
    r.launches = 0;
    r.gemv_launches = 0;
    r.gemv_seconds = 0.0;
    const bool fused = c->fused();
    ensure_hist(r, hist_cap);                 // before vargs: it may move r.hist
    VecArgs a = r.vargs(fused);
    const unsigned long long ebase = r.epoch_next;
    r.epoch_next += (unsigned long long)maxit + 2;
    r.x0_full = x0 ? r.s_full : nullptr;     // setup() puts the full x0 there
    if (!x0) {
        start(c, r, 0, b, tol, maxit, hist_cap, ebase);     // A0 + init (+ rendezvous): one launch
    } else {
        setup(c, r, b, x0, hist_cap);
        r.launches += launch_cg_init(a, tol, maxit, hist_cap, ebase, r.stream);
        if (fused) r.launches += launch_join(a, ebase, c->opt.join_timeout_ms, r.stream);
    }
    double* sig = r.S + (int64_t)r.rank * kScalSlot;
    GemvParams pq = gp(c, r, r.p_full, r.q_loc);
    pq.w1 = r.p_full + r.row0;                 // sigma_g = <p_loc, q_loc>
    pq.out1 = sig;
    pq.done = &r.st->done;
    if (fused) fuse_gemv(c, r, pq, kPhaseS, nullptr, 0, r.pp.S, (int64_t)r.rank * kScalSlot, a.spar);
    run_loop(c, r, 0, maxit, 1, [&](const long long* kdev, int64_t k, Prof& prof, int slot) {
        pq.kdev = kdev;
        pq.koff = k;
        prof.pre(slot);
        gemv(c, r, pq);                          // A1 (+ fused C2 publish)
        prof.post(slot);
        if (!kdev) ++r.gemv_launches;
        if (!fused) allgather(c, r, r.S, kScalSlot);   // A2 (C2)
        r.launches += launch_cg_update(a, kdev, k, r.stream);    // A2 + A3 (+ fused C1)
        if (!fused) allgather(c, r, r.G_r, r.L.chunk); // A4 (C1)
        r.launches += launch_cg_direction(a, kdev, k, r.stream); // A5
    });
    finish_and_copy(c, r, x, hist, hist_cap, rep, false, t_start, maxit, 1, ebase + (unsigned long long)maxit + 1);
    return r.h_state->peer_timeout ? (int64_t)KS_ENCCL : r.h_state->status;
}

int64_t run_bicgstab(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol,
                     int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    if (!x0) {
        const EmuPlan plan = emu_plan(c, 1, maxit);
        if (plan.g > 0) {
            check_loaded(c, r);
            return run_emu(c, r, 1, b, tol, maxit, x, hist, hist_cap, rep, plan);
        }
    }
    const auto t_start = Clock::now();
    check_loaded(c, r);
    r.launches = 0;
    r.gemv_launches = 0;
    r.gemv_seconds = 0.0;
    const bool fused = c->fused();
    ensure_hist(r, hist_cap);                 // before vargs: it may move r.hist
    VecArgs a = r.vargs(fused);
    const unsigned long long ebase = r.epoch_next;
    r.epoch_next += (unsigned long long)maxit + 2;
    r.x0_full = x0 ? r.s_full : nullptr;
    if (!x0) {
        start(c, r, 1, b, tol, maxit, hist_cap, ebase);     // B0 + init (+ rendezvous): one launch
    } else {
        setup(c, r, b, x0, hist_cap);
        r.launches += launch_bs_init(a, tol, maxit, hist_cap, ebase, r.stream);
        if (fused) r.launches += launch_join(a, ebase, c->opt.join_timeout_ms, r.stream);
    }
    double* vown = r.G_v + (int64_t)r.rank * r.L.chunk;
    GemvParams pv = gp(c, r, r.p_full, vown);  // B3: v = A p, <rhat, v>_g
    pv.w1 = r.rhat_loc;
    pv.out1 = vown + r.L.pslot;
    pv.done = &r.st->done;
    if (fused) {   // v rows stay local (pulled by bs_s); the partial is pushed
        fuse_gemv(c, r, pv, kPhaseV, nullptr, 0, r.pp.G_v, (int64_t)r.rank * r.L.chunk + r.L.pslot,
                  a.gpar);
        pv.y_par = a.gpar;
    }
    double* sc = r.S + (int64_t)r.rank * kScalSlot;
    GemvParams pt = gp(c, r, r.s_full, r.q_loc);  // B6: t = A s, <t,s>_g, <t,t>_g
    pt.w1 = r.s_full + r.row0;
    pt.out1 = sc;
    pt.out2 = sc + 1;
    pt.done = &r.st->done;
    if (fused) fuse_gemv(c, r, pt, kPhaseS, nullptr, 0, r.pp.S, (int64_t)r.rank * kScalSlot, a.spar);
    run_loop(c, r, 1, maxit, 2, [&](const long long* kdev, int64_t i, Prof& prof, int slot) {
        pv.kdev = pt.kdev = kdev;
        pv.koff = pt.koff = i;
        r.launches += launch_bs_p(a, kdev, i, r.stream);  // B8(i-1) + B1
        prof.pre(slot);
        gemv(c, r, pv);                          // B3 (+ fused C1/C2 publish)
        prof.post(slot);
        if (!fused) allgather(c, r, r.G_v, r.L.chunk);   // B2/B4 (C1 + C2)
        r.launches += launch_bs_s(a, kdev, i, r.stream);  // B4 + B5
        prof.pre(slot);
        gemv(c, r, pt);                          // B6 (+ fused C2 publish)
        prof.post(slot);
        if (!kdev) r.gemv_launches += 2;
        if (!fused) allgather(c, r, r.S, kScalSlot);     // B7 (C2)
        r.launches += launch_bs_xr(a, kdev, i, r.stream); // B7 (+ fused C1)
        if (!fused) allgather(c, r, r.G_r, r.L.chunk);   // B8 partials + r (C1)
    });
    finish_and_copy(c, r, x, hist, hist_cap, rep, true, t_start, maxit, 1, ebase + (unsigned long long)maxit + 1);
    return r.h_state->peer_timeout ? (int64_t)KS_ENCCL : r.h_state->status;
}

// NEXT-4: CG / BiCGSTAB in FP32 (persistent path; P == 1 or the fused exchange).
// The ABI is FP64: b is converted on the device, x converted back; x0 = 0.
int64_t run_f32(ks_ctx* c, Rank& r, int bicgstab, const double* b, double tol, int64_t maxit,
                double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    const auto t_start = Clock::now();
    check_loaded(c, r);
    r.launches = 0;
    r.gemv_launches = 0;
    r.gemv_seconds = 0.0;
    if (hist_cap > r.hist_alloc) {
        retire(r, r.hist);
        r.hist = nullptr;
        r.hist_alloc = std::max<int64_t>(hist_cap, 2 * r.hist_alloc);
        dev_alloc_t(&r.hist, (size_t)r.hist_alloc);
    }
    const bool fused = c->fused();
    VecArgsT<float> a0 = r.vargs_f32(false), a = r.vargs_f32(fused);
    double* tmp = nullptr;                              // FP64 staging of b / x
    dev_alloc_t(&tmp, (size_t)c->n);
    KS_CUDA(cudaMemcpyAsync(tmp, b, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
    r.launches += launch_d2f(tmp, a.b_full_mut(), c->n, r.stream);
    r.launches += launch_setup_r_f32(a0, r.stream);
    allgather(c, r, r.G_r, r.L.chunk);
    const unsigned long long ebase = r.epoch_next;
    r.epoch_next += (unsigned long long)maxit + 2;
    r.launches += launch_init_f32(a, bicgstab, tol, maxit, hist_cap, ebase, r.stream);
    if (fused) r.launches += launch_join(a, ebase, c->opt.join_timeout_ms, r.stream);
    const int64_t B = poll_batch(c, true, maxit);
    const int gemvs = bicgstab ? 2 : 1;
    Prof prof(c, r, 1);
    int prows = 0, punroll = 0;
    persist_shape(c, r, &prows, &punroll);
    int pgrid = memo_grid(r, (4LL << 48) | ((long long)prows << 24) | ((long long)punroll << 8) | bicgstab,
                          [&] { return persist_grid<float>(bicgstab, r.num_sms, r.L.pslot, prows, punroll); });
    if (c->opt.persist_grid > 0) pgrid = (int)std::min<int64_t>(pgrid, c->opt.persist_grid);
    const int sgrid = small_path_grid<float>(c, r, bicgstab);
    float* bpart = reinterpret_cast<float*>(r.scr.part + 2 * kPartStride);
    int64_t k = 1, batch = 0;
    KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
    while (k <= maxit) {
        const int slot = (int)(batch & 1);
        prof.begin(slot);
        const int64_t kend = std::min<int64_t>(maxit, k + B - 1);
        prof.pre(slot);
        const int rc = sgrid > 0
            ? launch_small<float>(small_kind(c, bicgstab), a, reinterpret_cast<const float*>(r.A), c->ld,
                                  c->ld, bpart, r.scr.ticket + 8, k, kend, sgrid, r.stream)
            : launch_persist<float>(bicgstab, a, reinterpret_cast<const float*>(r.A), c->ld, c->ld,
                                    bpart, r.scr.ticket + 8, k, kend, pgrid, prows, punroll, r.stream);
        prof.post(slot);
        if (rc < 0) KS_CUDA((cudaError_t)(-rc));
        r.launches += 1;
        r.gemv_launches += (kend - k + 1) * gemvs;
        k = kend + 1;
        KS_CUDA(cudaMemcpyAsync(&r.h_done[slot], &r.st->done, sizeof(int), cudaMemcpyDeviceToHost, r.stream));
        KS_CUDA(cudaEventRecord(r.ev_poll[slot], r.stream));
        if (batch >= 1) {
            KS_CUDA(cudaEventSynchronize(r.ev_poll[slot ^ 1]));
            prof.harvest(slot ^ 1);
            if (r.h_done[slot ^ 1]) { ++batch; break; }
        }
        ++batch;
    }
    KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    prof.harvest(0);
    prof.harvest(1);
    r.launches += launch_finish_f32(a, bicgstab, r.stream);
    // x (full length, FP32) -> true residual (K1 FP32, residual mode) -> FP64 out
    float* xfull = a.s_full;
    if (c->P > 1) {
        r.launches += launch_pack_x_f32(a0, r.stream);
        allgather(c, r, r.G_v, r.L.chunk);
        copy_chunks_to(c, r, r.G_v, r.s_full, cudaMemcpyDeviceToDevice);
    } else {
        KS_CUDA(cudaMemcpyAsync(xfull, a.x_loc, (size_t)c->n * sizeof(float), cudaMemcpyDeviceToDevice, r.stream));
    }
    if (c->opt.true_residual) {
        GemvParamsT<float> p{};
        p.A = reinterpret_cast<const float*>(r.A);
        p.lda = c->ld;
        p.m = r.m;
        p.ncols = c->ld;
        p.x = xfull;
        p.y = a.q_loc;
        p.bsub = a.b_full + r.row0;
        p.out2 = a0.S + (int64_t)r.rank * kScalSlot + 1;
        r.launches += launch_gemv_f32(p, r.scr, 1, r.stream);
        allgather(c, r, r.S, kScalSlot);
        r.launches += launch_true_res_final_f32(a0, r.stream);
    }
    r.launches += launch_f2d(xfull, tmp, c->n, r.stream);
    KS_CUDA(cudaMemcpyAsync(r.h_state, r.st, sizeof(DevState), cudaMemcpyDeviceToHost, r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    const DevState& s = *r.h_state;
    if (c->writes_host(r)) {
        KS_CUDA(cudaMemcpyAsync(x, tmp, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
        const int64_t nh = std::min<int64_t>(s.iters, hist_cap);
        if (hist && nh > 0)
            KS_CUDA(cudaMemcpyAsync(hist, r.hist, (size_t)nh * sizeof(double), cudaMemcpyDefault, r.stream));
        KS_CUDA(cudaStreamSynchronize(r.stream));
    }
    retire(r, tmp);
    if (rep) {
        float ms = 0.f;
        KS_CUDA(cudaEventElapsedTime(&ms, r.ev_t0, r.ev_t1));
        ks_report R;
        std::memset(&R, 0, sizeof R);
        R.iterations = s.iters;
        R.half_step_exit = s.half;
        R.matvecs = bicgstab ? 2 * s.iters - (s.half ? 1 : 0) : s.iters;
        R.converged = s.converged;
        R.breakdown = s.breakdown;
        R.status = s.status;
        R.relres = s.relres;
        R.true_relres = (c->opt.true_residual && s.nb > 0) ? std::sqrt(s.true_rr) / s.nb : (s.bzero ? 0.0 : -1.0);
        R.seconds_loop = ms * 1e-3;
        R.seconds_total = std::chrono::duration<double>(Clock::now() - t_start).count();
        R.seconds_gemv = r.gemv_seconds;
        R.gemv_launches = r.gemv_launches;
        R.kernel_launches = r.launches;
        *rep = R;
    }
    return s.peer_timeout ? (int64_t)KS_ENCCL : s.status;
}

// GMRES(m) (NEXT-3): host-orchestrated cycles (their structure is
// deterministic; an early exit inside a cycle makes the remaining launches of the
// cycle no-ops through GmresState::skip).  NCCL for P > 1.
int64_t run_gmres(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol, int restart,
                  int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    const auto t_start = Clock::now();
    check_loaded(c, r);
    r.launches = 0;
    r.gemv_launches = 0;
    r.gemv_seconds = 0.0;
    const size_t nbytes = (size_t)c->n * sizeof(double);
    if (hist_cap > r.hist_alloc) {
        retire(r, r.hist);
        r.hist = nullptr;
        r.hist_alloc = std::max<int64_t>(hist_cap, 2 * r.hist_alloc);
        dev_alloc_t(&r.hist, (size_t)r.hist_alloc);
    }
    if (r.gm_m < restart || !r.gmV) {
        for (void* p : {(void*)r.gmV, (void*)r.gmH, (void*)r.gm_hx, (void*)r.gm_state})
            retire(r, p);
        r.gm_ldv = (r.m + 31) / 32 * 32;
        r.gm_m = restart;
        dev_alloc_t(&r.gmV, (size_t)(restart + 1) * r.gm_ldv);
        const size_t hsz = (size_t)(restart + 1) * restart + 3 * (size_t)(restart + 1);
        dev_alloc_t(&r.gmH, hsz);
        KS_CUDA(cudaMemsetAsync(r.gmH, 0, hsz * sizeof(double), r.stream));
        dev_alloc_t(&r.gm_hx, (size_t)c->P * kMaxBasis);
        dev_alloc_t(&r.gm_state, 1);
        KS_CUDA(cudaMemsetAsync(r.gm_state, 0, sizeof(GmresState), r.stream));
    }
    VecArgs a = r.vargs(false);
    GmresArgs g;
    g.a = a;
    g.V = r.gmV;
    g.ldv = r.gm_ldv;
    g.mres = restart;
    g.H = r.gmH;
    g.cs = r.gmH + (size_t)(restart + 1) * restart;
    g.sn = g.cs + (restart + 1);
    g.g = g.sn + (restart + 1);
    g.hx = r.gm_hx;
    g.gs = r.gm_state;
    g.part = r.scr.part + 3 * kPartStride;     // 296 CTAs x 64 <= kPartStride
    g.ticket = r.scr.ticket + 12;
    KS_CUDA(cudaMemcpyAsync(r.b_full, b, nbytes, cudaMemcpyDefault, r.stream));
    if (x0) KS_CUDA(cudaMemcpyAsync(r.x_loc, x0 + r.row0, (size_t)r.m * sizeof(double), cudaMemcpyDefault, r.stream));
    else KS_CUDA(cudaMemsetAsync(r.x_loc, 0, (size_t)r.m * sizeof(double), r.stream));
    r.launches += launch_gm_init(g, tol, maxit, hist_cap, r.stream);
    GemvParams pres = gp(c, r, r.s_full, r.q_loc);   // r = b - A x, ||r||^2 partial
    pres.bsub = r.b_full + r.row0;
    pres.out2 = r.S + (int64_t)r.rank * kScalSlot + 1;
    pres.done = &r.st->done;
    GemvParams pw = gp(c, r, r.p_full, r.q_loc);     // w = A v_j
    pw.done = &r.gm_state->skip;
    Prof prof(c, r, restart + 1);
    int64_t k = 0, cycle = 0;
    KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
    if ((c->P == 1 || c->fused()) && c->opt.persistent != 0) {
        // NEXT-2 for GMRES: one persistent cooperative kernel per restart cycle;
        // P > 1: the Arnoldi collectives run inside it over NVLink (NEXT-1)
        const int grid = gm_persist_grid(r.num_sms, r.m);
        const int64_t max_cycles = maxit / restart + 2;
        GmresArgs gf = g;
        gf.a = r.vargs(c->fused());
        const unsigned long long ebase = r.epoch_next;
        r.epoch_next += gm_epochs(maxit, restart);
        if (c->fused()) r.launches += launch_join(gf.a, ebase, c->opt.join_timeout_ms, r.stream);
        for (cycle = 0; cycle < max_cycles; ++cycle) {
            const int slot = (int)(cycle & 1);
            prof.begin(slot);
            prof.pre(slot);
            const int rc = launch_gm_cycle_persist(gf, r.A, c->ld, c->ld, r.scr.part + 2 * kPartStride,
                                                   r.scr.ticket + 8, grid, ebase, r.stream);
            prof.post(slot);
            if (rc < 0) KS_CUDA((cudaError_t)(-rc));
            r.launches += 1;
            KS_CUDA(cudaMemcpyAsync(&r.h_done[slot], &r.st->done, sizeof(int), cudaMemcpyDeviceToHost, r.stream));
            KS_CUDA(cudaEventRecord(r.ev_poll[slot], r.stream));
            if (cycle >= 1) {
                KS_CUDA(cudaEventSynchronize(r.ev_poll[slot ^ 1]));
                prof.harvest(slot ^ 1);
                if (r.h_done[slot ^ 1]) break;
            }
        }
        KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
        KS_CUDA(cudaStreamSynchronize(r.stream));
        prof.harvest(0);
        prof.harvest(1);
        KS_CUDA(cudaMemcpy(r.h_state, r.st, sizeof(DevState), cudaMemcpyDeviceToHost));
        r.gemv_launches = r.h_state->iters;
        r.launches += launch_cg_finish(a, r.stream);
        finish_and_copy(c, r, x, hist, hist_cap, rep, false, t_start, maxit);
        return r.h_state->status;
    }
    while (true) {
        const int slot = (int)(cycle & 1);
        prof.begin(slot);
        // x (gathered, full length) -> residual of the cycle start
        if (c->P > 1) {
            r.launches += launch_pack_x(a, r.stream);
            allgather(c, r, r.G_v, r.L.chunk);
            copy_chunks_to(c, r, r.G_v, r.s_full, cudaMemcpyDeviceToDevice);
        } else {
            KS_CUDA(cudaMemcpyAsync(r.s_full, r.x_loc, nbytes, cudaMemcpyDeviceToDevice, r.stream));
        }
        gemv(c, r, pres);
        allgather(c, r, r.S, kScalSlot);
        r.launches += launch_gm_start(g, r.stream);
        allgather(c, r, r.G_r, r.L.chunk);
        r.launches += launch_gm_vfull(g, r.stream);
        for (int j = 0; j < restart && k < maxit; ++j) {
            ++k;
            prof.pre(slot);
            gemv(c, r, pw);                                    // w = A v_j
            prof.post(slot);
            ++r.gemv_launches;
            r.launches += launch_gm_dots(g, j, r.stream);      // CGS pass 1
            allgather(c, r, g.hx, kMaxBasis);
            r.launches += launch_gm_orth(g, j, 1, r.stream);   // update + pass-2 dots
            allgather(c, r, g.hx, kMaxBasis);
            r.launches += launch_gm_orth(g, j, 2, r.stream);   // update + ||w||^2
            allgather(c, r, g.hx, kMaxBasis);
            r.launches += launch_gm_step_end(g, j, k, r.stream);
            allgather(c, r, r.G_r, r.L.chunk);
            r.launches += launch_gm_vfull(g, r.stream);
        }
        r.launches += launch_gm_cycle_end(g, k, r.stream);
        KS_CUDA(cudaMemcpyAsync(&r.h_done[slot], &r.st->done, sizeof(int), cudaMemcpyDeviceToHost, r.stream));
        KS_CUDA(cudaEventRecord(r.ev_poll[slot], r.stream));
        if (cycle >= 1) {
            KS_CUDA(cudaEventSynchronize(r.ev_poll[slot ^ 1]));
            prof.harvest(slot ^ 1);
            if (r.h_done[slot ^ 1]) break;
        }
        ++cycle;
        if (k >= maxit) break;
    }
    KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    prof.harvest(0);
    prof.harvest(1);
    r.launches += launch_cg_finish(a, r.stream);
    finish_and_copy(c, r, x, hist, hist_cap, rep, false, t_start, maxit);
    return r.h_state->status;
}

// BiCG (NEXT-3): multi-kernel schedule; NCCL for P > 1 (allgather of
// [r | <rt,r>, <r,r>], scalar allgather of <pt, A p>, reduce-scatter of A^T pt).
int64_t run_bicg(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol, int64_t maxit,
                 double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    const auto t_start = Clock::now();
    check_loaded(c, r);
    r.launches = 0;
    r.gemv_launches = 0;
    r.gemv_seconds = 0.0;
    setup(c, r, b, x0, hist_cap);                  // r0, x, rt0 = r0, slots <r0,r0>
    // fused (P > 1, NEXT-1): sigma partials pushed by K1's epilogue, the A^T pt
    // reduce-scatter fused into K1T, r slices pushed by k_bicg_update -- no NCCL
    // call in the loop
    const bool fused = c->fused();
    VecArgs a = r.vargs(fused);
    const unsigned long long ebase = r.epoch_next;
    r.epoch_next += (unsigned long long)maxit + 2;
    r.launches += launch_bicg_init(a, tol, maxit, hist_cap, ebase, r.stream);
    if (fused) r.launches += launch_join(a, ebase, c->opt.join_timeout_ms, r.stream);
    GemvParams pq = gp(c, r, r.p_full, r.q_loc);   // q = A p, sigma_g = <pt_loc, q>
    pq.w1 = r.pt_loc;
    pq.out1 = r.S + (int64_t)r.rank * kScalSlot;
    pq.done = &r.st->done;
    if (fused) fuse_gemv(c, r, pq, kPhaseS, nullptr, 0, r.pp.S, (int64_t)r.rank * kScalSlot, a.spar);
    const int64_t B = poll_batch(c, false, maxit);
    Prof prof(c, r, 2 * B);
    int64_t k = 1, batch = 0;
    KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
    while (k <= maxit) {
        const int slot = (int)(batch & 1);
        prof.begin(slot);
        const int64_t kend = std::min<int64_t>(maxit, k + B - 1);
        for (; k <= kend; ++k) {
            pq.koff = k;
            prof.pre(slot);
            gemv(c, r, pq);                                    // q = A p (+ fused sigma publish)
            prof.post(slot);
            prof.pre(slot);
            gemv_t(c, r, r.pt_loc, &r.st->done, fused ? k : 0, ebase);   // qt = A^T pt (+ reduce-scatter)
            prof.post(slot);
            r.gemv_launches += 2;
            if (!fused) allgather(c, r, r.S, kScalSlot);
            r.launches += launch_bicg_update(a, k, r.stream);
            if (!fused) allgather(c, r, r.G_r, r.L.chunk);
            r.launches += launch_bicg_direction(a, k, r.stream);
        }
        KS_CUDA(cudaMemcpyAsync(&r.h_done[slot], &r.st->done, sizeof(int), cudaMemcpyDeviceToHost, r.stream));
        KS_CUDA(cudaEventRecord(r.ev_poll[slot], r.stream));
        if (batch >= 1) {
            KS_CUDA(cudaEventSynchronize(r.ev_poll[slot ^ 1]));
            prof.harvest(slot ^ 1);
            if (r.h_done[slot ^ 1]) { ++batch; break; }
        }
        ++batch;
    }
    KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    prof.harvest(0);
    prof.harvest(1);
    r.launches += launch_cg_finish(a, r.stream);
    finish_and_copy(c, r, x, hist, hist_cap, rep, false, t_start, maxit);
    if (rep) rep->matvecs = 2 * rep->iterations;
    return r.h_state->status;
}

// Multi-RHS CG (ks_multi.cu): nrhs <= 8 independent CG
// recurrences sharing every pass over A, one persistent launch per solve; one GPU.
// B, X0, X: n x nrhs column-major (column k at + k n); hist: hist_cap x nrhs
// column-major; reps: nrhs reports.  Returns the worst column status
// (ENOTSPD > EMAXIT > OK).
int64_t run_multi(ks_ctx* c, Rank& r, int bicgstab, int nrhs, const double* B, const double* X0, double tol,
                  int64_t maxit, double* X, double* hist, int64_t hist_cap, ks_report* reps) {
    const auto t_start = Clock::now();
    check_loaded(c, r);
    const int K = multi_k(nrhs);
    const int64_t n = c->n, ld = c->ld, ldm = (r.m + 63) / 64 * 64;
    if (K != r.mK) {
        for (double* p : {r.mX, r.mR, r.mQ, r.mP, r.mRh, r.mT, r.mS}) retire(r, p);
        r.mRh = r.mT = r.mS = nullptr;
        dev_alloc_t(&r.mX, (size_t)(K * ldm));
        dev_alloc_t(&r.mR, (size_t)(K * ldm));
        dev_alloc_t(&r.mQ, (size_t)(K * ldm));
        dev_alloc_t(&r.mP, (size_t)(K * ld));
        if (!r.mstate) dev_alloc_t(&r.mstate, 1);
        r.mK = K;
    }
    if (bicgstab && !r.mS) {                 // BiCGSTAB: rhat, t, and the full-length s
        dev_alloc_t(&r.mRh, (size_t)(K * ldm));
        dev_alloc_t(&r.mT, (size_t)(K * ldm));
        dev_alloc_t(&r.mS, (size_t)(K * ld));
        KS_CUDA(cudaMemsetAsync(r.mS, 0, (size_t)(K * ld) * sizeof(double), r.stream));
    }
    const int64_t hc = hist ? hist_cap : 0;
    if (hc > 0 && hc * K > r.mhist_cap) {
        retire(r, r.mhist);
        r.mhist = nullptr;
        r.mhist_cap = hc * K;
        dev_alloc_t(&r.mhist, (size_t)r.mhist_cap);
    }
    const size_t e = sizeof(double);
    // b -> R (K rows of stride ldm), padding rows zero; x0 -> P; P zero elsewhere
    KS_CUDA(cudaMemsetAsync(r.mR, 0, (size_t)(K * ldm) * e, r.stream));
    KS_CUDA(cudaMemsetAsync(r.mP, 0, (size_t)(K * ld) * e, r.stream));
    // this rank's rows of b (P = 1: all of them)
    KS_CUDA(cudaMemcpy2DAsync(r.mR, (size_t)ldm * e, B + r.row0, (size_t)n * e, (size_t)r.m * e, (size_t)nrhs,
                              cudaMemcpyDefault, r.stream));
    if (X0)
        KS_CUDA(cudaMemcpy2DAsync(r.mP, (size_t)ld * e, X0, (size_t)n * e, (size_t)n * e, (size_t)nrhs,
                                  cudaMemcpyDefault, r.stream));
    MultiArgs M{};
    M.nrhs = nrhs;
    M.has_x0 = X0 ? 1 : 0;
    M.n = n;
    M.m = r.m;
    M.ld = ld;
    M.ldm = ldm;
    M.row0 = r.row0;
    M.tol = tol;
    M.maxit = maxit;
    M.X = r.mX;
    M.R = r.mR;
    M.Q = r.mQ;
    M.Pf = r.mP;
    M.hist = hc > 0 ? r.mhist : nullptr;
    M.hist_cap = hc;
    M.ms = r.mstate;
    M.st = r.st;
    M.bpart = r.scr.part + 2 * kPartStride;
    M.bar = r.scr.ticket + 8;
    M.peer = c->P > 1 ? 1 : 0;
    M.L = r.L;
    M.mp = r.mpeer;
    M.MRo = r.MR;
    M.MVo = r.MV;
    M.MSo = r.MS;
    M.flags = r.flags;
    M.ebase = r.epoch_next;
    r.epoch_next += (unsigned long long)maxit + 2;
    M.join_ns = (unsigned long long)c->opt.join_timeout_ms * 1000000ULL;
    M.Sf = r.mS;
    M.Rh = r.mRh;
    M.T = r.mT;
    const int grid = bicgstab ? memo_grid(r, (6LL << 48) | K, [&] { return multi_grid_bs(K, r.num_sms); })
                              : memo_grid(r, (5LL << 48) | K, [&] { return multi_grid(K, r.num_sms); });
    if (grid <= 0) throw KsError(KS_ECUDA, "multi-RHS kernel does not fit this device");
    KS_CUDA(cudaMemsetAsync(&r.st->peer_timeout, 0, sizeof(int), r.stream));
    KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
    const int rc = bicgstab ? launch_bicgstab_multi(K, M, r.A, grid, r.stream)
                            : launch_cg_multi(K, M, r.A, grid, r.stream);
    if (rc < 0) KS_CUDA((cudaError_t)(-rc));
    KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
    // out: X columns, state, histories -- one synchronisation
    MultiState hs;
    if (c->writes_host(r)) {
        if (c->P > 1)                     // gathered in-kernel into this rank's MX (K x ld)
            KS_CUDA(cudaMemcpy2DAsync(X, (size_t)n * e, r.MX, (size_t)ld * e, (size_t)n * e, (size_t)nrhs,
                                      cudaMemcpyDefault, r.stream));
        else
            KS_CUDA(cudaMemcpy2DAsync(X, (size_t)n * e, r.mX, (size_t)ldm * e, (size_t)n * e, (size_t)nrhs,
                                      cudaMemcpyDefault, r.stream));
    }
    KS_CUDA(cudaMemcpyAsync(r.h_state, r.st, sizeof(DevState), cudaMemcpyDeviceToHost, r.stream));
    KS_CUDA(cudaMemcpyAsync(&hs, r.mstate, sizeof(MultiState), cudaMemcpyDeviceToHost, r.stream));
    const int64_t nh = std::min<int64_t>(hc, maxit);
    if (nh > 0 && c->writes_host(r))
        KS_CUDA(cudaMemcpy2DAsync(hist, (size_t)hist_cap * e, r.mhist, (size_t)hc * e, (size_t)nh * e,
                                  (size_t)nrhs, cudaMemcpyDefault, r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    if (r.h_state->peer_timeout)
        throw KsError(c->P > 1 ? KS_ENCCL : KS_ECUDA, "multi-RHS kernel: a barrier or peer wait timed out");
    float ms = 0.f;
    KS_CUDA(cudaEventElapsedTime(&ms, r.ev_t0, r.ev_t1));
    int64_t worst = KS_OK;
    for (int k = 0; k < nrhs; ++k) {
        const MultiCol& cl = hs.col[k];
        const int64_t stt = cl.active ? (int64_t)KS_EMAXIT : (int64_t)cl.status;
        if (stt == KS_ENOTSPD || stt == KS_EBREAKDOWN) worst = stt;
        else if (stt == KS_EMAXIT && worst == KS_OK) worst = KS_EMAXIT;
        if (reps) {
            ks_report R;
            std::memset(&R, 0, sizeof R);
            R.iterations = cl.active ? maxit : cl.iters;
            R.matvecs = bicgstab ? 2 * R.iterations - (cl.half ? 1 : 0) : R.iterations;
            R.half_step_exit = bicgstab ? cl.half : 0;
            R.breakdown = bicgstab ? cl.breakdown : 0;
            R.converged = cl.converged;
            R.status = (int32_t)stt;
            R.relres = cl.bzero ? 0.0 : cl.relres;
            R.true_relres = -1.0;
            R.seconds_loop = ms * 1e-3;
            R.seconds_total = std::chrono::duration<double>(Clock::now() - t_start).count();
            R.gemv_launches = hs.col[0].iters;
            R.kernel_launches = 1;
            reps[k] = R;
        }
    }
    return worst;
}

}  // namespace ks

// L4: the extern "C" boundary declared in include/ks.h.  Validates arguments
// before any work, converts internal exceptions to ks_status + message, and
// poisons the context on CUDA/NCCL/allocation errors.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ks_ctx.h"

using ks::KsError;
using ks::Rank;

namespace {

thread_local std::string g_tls_error;

ks_status fail(ks_ctx* c, ks_status code, const std::string& msg) {
    g_tls_error = msg;
    if (c) {
        c->last_error = msg;
        if (code == KS_ECUDA || code == KS_ENCCL || code == KS_ENOMEM) c->poisoned = true;
    }
    return code;
}

// Every local rank must hold all of its rows before a call that runs a collective
// schedule: checked up front for ALL local ranks, so in single-process multi-GPU
// mode an unloaded shard is an error on every rank rather than one rank throwing
// while its peers wait in a fused exchange.  In multi-process mode
// each process checks its own shard; a peer that stops here makes the others'
// solve-start rendezvous fail with KS_ENCCL after its timeout, never hang.
bool all_loaded(const ks_ctx* c) {
    for (const Rank& r : c->ranks)
        if (r.loaded_count < r.m) return false;
    return true;
}

template <class F>
ks_status guarded(ks_ctx* c, F&& f) {
    if (c && c->poisoned) return fail(c, KS_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    try {
        return f();
    } catch (const KsError& e) {
        return fail(c, e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(c, KS_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(c, KS_ECUDA, e.what());
    }
}

void make_layout(ks_ctx* c) {
    const int64_t n = c->n;
    const int P = c->P;
    const int64_t align = (int64_t)(4096 / c->esz);   // 4 KiB rows: 512 doubles / 1024 floats
    c->ld = (n + align - 1) / align * align;
    ks::Layout L{};
    L.P = P;
    L.n = n;
    L.ld = c->ld;
    const int64_t q = n / P, rem = n % P;
    int64_t mmax = 0;
    for (int g = 0; g <= P; ++g) {
        L.row0[g] = (int64_t)g * q + std::min<int64_t>(g, rem);
    }
    for (int g = 0; g < P; ++g) mmax = std::max(mmax, L.row0[g + 1] - L.row0[g]);
    L.pslot = (mmax + 31) / 32 * 32;
    L.chunk = L.pslot + 32;
    for (auto& r : c->ranks) {
        r.L = L;
        r.L.rank = r.rank;
        r.row0 = L.row0[r.rank];
        r.m = L.row0[r.rank + 1] - r.row0;
    }
}

ks_status status_of(int64_t s) { return (ks_status)s; }

}  // namespace

extern "C" {

ks_status ks_create_on(ks_ctx** out, int64_t n, ks_dtype dtype, int32_t nranks, const int32_t* devices) {
    if (!out) return fail(nullptr, KS_EARG, "out is NULL");
    *out = nullptr;
    if (dtype != KS_FLOAT64 && dtype != KS_FLOAT32) return fail(nullptr, KS_EARG, "dtype must be KS_FLOAT64 or KS_FLOAT32");
    if (n < 1) return fail(nullptr, KS_EDIM, "n must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    if (nranks < 1 || nranks > ks::kMaxRanks || !devices)
        return fail(nullptr, KS_EARG, "nranks must be in [1, 16] and devices non-NULL");
    std::vector<int> devs((size_t)nranks);
    bool shared = false;
    for (int g = 0; g < nranks; ++g) {
        devs[g] = devices[g];
        if (devs[g] < 0 || devs[g] >= ndev)
            return fail(nullptr, KS_EARG, "devices[" + std::to_string(g) + "] is not a device (count=" +
                                              std::to_string(ndev) + ")");
        for (int h = 0; h < g; ++h) shared = shared || devs[h] == devs[g];
    }
    if (n < nranks) return fail(nullptr, KS_EDIM, "n must be >= nranks");
    ks_ctx* c = new ks_ctx();
    c->n = n;
    c->P = nranks;
    c->dtype = dtype;
    c->esz = dtype == KS_FLOAT32 ? sizeof(float) : sizeof(double);
    c->shared_dev = shared;
    // Ranks sharing a GPU never run kernels that wait on each other: separate launches
    // on one GPU have no co-residency guarantee (B200_PROFILING.md; 2-4 such ranks as
    // processes on one B200 raised Xid 109).  Their exchanges are the host-driven
    // collectives, so the fused exchange (and the persistent / small-n / tiny /
    // multi-RHS kernels that need it) stays off.
    if (shared) c->opt.fused_comm = 0;
    c->ranks.resize((size_t)nranks);
    for (int g = 0; g < nranks; ++g) {
        c->ranks[g].rank = g;
        c->ranks[g].dev = devs[g];
        c->ranks[g].dev_share = (int)std::count(devs.begin(), devs.end(), devs[g]);
    }
    make_layout(c);
    ks_status st = guarded(c, [&] {
        if (nranks > 1 && !shared) {
            std::vector<ncclComm_t> comms((size_t)nranks);
            KS_NCCL(ncclCommInitAll(comms.data(), nranks, devs.data()));
            for (int g = 0; g < nranks; ++g) { c->ranks[g].comm = comms[g]; c->ranks[g].own_comm = true; }
        }
        c->for_each_rank([&](Rank& r) { ks::rank_alloc(c, r); });
        ks::setup_peers(c);
        return KS_OK;
    });
    if (st != KS_OK) {
        for (auto& r : c->ranks) ks::rank_free(r);
        delete c;
        return st;
    }
    *out = c;
    return KS_OK;
}

ks_status ks_create(ks_ctx** out, int64_t n, ks_dtype dtype, int32_t ngpus) {
    if (!out) return fail(nullptr, KS_EARG, "out is NULL");
    *out = nullptr;
    if (dtype != KS_FLOAT64 && dtype != KS_FLOAT32) return fail(nullptr, KS_EARG, "dtype must be KS_FLOAT64 or KS_FLOAT32");
    if (n < 1) return fail(nullptr, KS_EDIM, "n must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    if (ngpus < 1 || ngpus > ks::kMaxRanks || ngpus > ndev)
        return fail(nullptr, KS_EARG, "ngpus must be in [1, min(16, device count=" + std::to_string(ndev) + ")]");
    std::vector<int32_t> devs((size_t)ngpus);
    for (int g = 0; g < ngpus; ++g) devs[g] = g;
    return ks_create_on(out, n, dtype, ngpus, devs.data());
}

ks_status ks_create_rank(ks_ctx** out, int64_t n, ks_dtype dtype, int32_t rank, int32_t nranks,
                         void* nccl_comm, int32_t device, void* stream) {
    if (!out) return fail(nullptr, KS_EARG, "out is NULL");
    *out = nullptr;
    if (dtype != KS_FLOAT64 && dtype != KS_FLOAT32) return fail(nullptr, KS_EARG, "dtype must be KS_FLOAT64 or KS_FLOAT32");
    if (n < 1) return fail(nullptr, KS_EDIM, "n must be >= 1");
    if (nranks < 1 || nranks > ks::kMaxRanks || rank < 0 || rank >= nranks)
        return fail(nullptr, KS_EARG, "need 0 <= rank < nranks <= 16");
    if (nranks > 1 && !nccl_comm) return fail(nullptr, KS_EARG, "nccl_comm required when nranks > 1");
    if (n < nranks) return fail(nullptr, KS_EDIM, "n must be >= nranks");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    if (device < 0 || device >= ndev) return fail(nullptr, KS_EARG, "invalid device");
    ks_ctx* c = new ks_ctx();
    c->n = n;
    c->P = nranks;
    c->dtype = dtype;
    c->esz = dtype == KS_FLOAT32 ? sizeof(float) : sizeof(double);
    c->multiprocess = true;
    c->ranks.resize(1);
    Rank& r = c->ranks[0];
    r.rank = rank;
    r.dev = device;
    r.comm = (ncclComm_t)nccl_comm;
    r.own_comm = false;
    r.stream = (cudaStream_t)stream;
    r.own_stream = false;
    make_layout(c);
    ks_status st = guarded(c, [&] {
        if (nranks > 1) {
            int cnt = 0, crank = 0;
            KS_NCCL(ncclCommCount(r.comm, &cnt));
            KS_NCCL(ncclCommUserRank(r.comm, &crank));
            if (cnt != nranks || crank != rank)
                throw KsError(KS_EARG, "nccl_comm size/rank do not match (nranks, rank)");
        }
        c->for_each_rank([&](Rank& rr) { ks::rank_alloc(c, rr); });
        ks::setup_peers(c);
        return KS_OK;
    });
    if (st != KS_OK) {
        ks::rank_free(r);
        delete c;
        return st;
    }
    *out = c;
    return KS_OK;
}

ks_status ks_destroy(ks_ctx* c) {
    if (!c) return KS_OK;
    for (auto& r : c->ranks) ks::rank_free(r);
    delete c;
    return KS_OK;
}

ks_status ks_row_range(const ks_ctx* c, int32_t shard, int64_t* b, int64_t* e) {
    if (!c || !b || !e) return fail(nullptr, KS_EARG, "NULL argument");
    if (shard < 0 || shard >= c->P) return fail(const_cast<ks_ctx*>(c), KS_EARG, "shard out of range");
    const ks::Layout& L = c->ranks[0].L;
    *b = L.row0[shard];
    *e = L.row0[shard + 1];
    return KS_OK;
}

ks_status ks_load_rows(ks_ctx* c, int64_t row_begin, int64_t nrows, const double* A, int64_t lda) {
    if (!c) return fail(nullptr, KS_EARG, "ctx is NULL");
    if (nrows < 0 || row_begin < 0 || row_begin + nrows > c->n)
        return fail(c, KS_EDIM, "rows out of range");
    if (lda < c->n) return fail(c, KS_EDIM, "lda < n");
    if (nrows > 0 && !A) return fail(c, KS_EARG, "A is NULL");
    return guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            const int64_t b = std::max(row_begin, r.row0);
            const int64_t e = std::min(row_begin + nrows, r.row0 + r.m);
            if (e <= b) return;
            if (c->dtype == KS_FLOAT32) {                 // FP64 rows -> device staging -> FP32
                const int64_t chunk = std::max<int64_t>(1, (int64_t)(8 << 20) / c->n);
                double* stage = nullptr;
                ks::dev_alloc_t(&stage, (size_t)std::min(chunk, e - b) * c->n);
                for (int64_t i = b; i < e; i += chunk) {
                    const int64_t cnt = std::min(chunk, e - i);
                    KS_CUDA(cudaMemcpy2DAsync(stage, (size_t)c->n * sizeof(double), A + (i - row_begin) * lda,
                                              (size_t)lda * sizeof(double), (size_t)c->n * sizeof(double),
                                              (size_t)cnt, cudaMemcpyDefault, r.stream));
                    ks::launch_rows_d2f(stage, c->n, reinterpret_cast<float*>(r.A) + (i - r.row0) * c->ld, c->ld,
                                        cnt, c->n, r.stream);
                }
                KS_CUDA(cudaStreamSynchronize(r.stream));
                ks::dev_free(stage);
                for (int64_t i = b; i < e; ++i) {
                    auto& f = r.loaded[(size_t)(i - r.row0)];
                    if (!f) { f = 1; ++r.loaded_count; }
                }
                return;
            }
            KS_CUDA(cudaMemcpy2DAsync(r.A + (b - r.row0) * c->ld, (size_t)c->ld * sizeof(double),
                                      A + (b - row_begin) * lda, (size_t)lda * sizeof(double),
                                      (size_t)c->n * sizeof(double), (size_t)(e - b), cudaMemcpyDefault,
                                      r.stream));
            KS_CUDA(cudaStreamSynchronize(r.stream));
            for (int64_t i = b; i < e; ++i) {
                auto& f = r.loaded[(size_t)(i - r.row0)];
                if (!f) { f = 1; ++r.loaded_count; }
            }
        });
        return KS_OK;
    });
}

ks_status ks_generate(ks_ctx* c, const ks_gen_spec* spec, double* b_out) {
    if (!c || !spec) return fail(c, KS_EARG, "NULL argument");
    if (spec->kind != 0 && spec->kind != 1) return fail(c, KS_EARG, "kind must be 0 (G-SPD) or 1 (G-DD)");
    if (spec->kind == 0 && !spec->spd_table) return fail(c, KS_EARG, "G-SPD needs spd_table");
    if (spec->kind == 1 && spec->kd < 1) return fail(c, KS_EARG, "G-DD needs kd >= 1");
    return guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            if (spec->kind == 0) {
                double* tab = nullptr;
                ks::dev_alloc_t(&tab, (size_t)c->n);
                KS_CUDA(cudaMemcpyAsync(tab, spec->spd_table, (size_t)c->n * sizeof(double),
                                        cudaMemcpyDefault, r.stream));
                if (c->dtype == KS_FLOAT32)
                    ks::launch_gen_spd_f32(reinterpret_cast<float*>(r.A), c->ld, r.row0, r.m, c->n, spec->seed, tab, r.stream);
                else
                    ks::launch_gen_spd(r.A, c->ld, r.row0, r.m, c->n, spec->seed, tab, r.stream);
                KS_CUDA(cudaStreamSynchronize(r.stream));
                ks::dev_free(tab);
            } else {
                if (c->dtype == KS_FLOAT32)
                    ks::launch_gen_dd_f32(reinterpret_cast<float*>(r.A), c->ld, r.row0, r.m, c->n, spec->seed, spec->kd, r.stream);
                else
                    ks::launch_gen_dd(r.A, c->ld, r.row0, r.m, c->n, spec->seed, spec->kd, r.stream);
            }
            KS_CUDA(cudaGetLastError());
            if (b_out && c->writes_host(r)) {
                double* bd = nullptr;                     // b is FP64 at the ABI
                ks::dev_alloc_t(&bd, (size_t)c->n);
                ks::launch_gen_rhs(bd, c->n, spec->seed, r.stream);
                KS_CUDA(cudaMemcpyAsync(b_out, bd, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
                KS_CUDA(cudaStreamSynchronize(r.stream));
                ks::dev_free(bd);
            }
            KS_CUDA(cudaStreamSynchronize(r.stream));
            std::fill(r.loaded.begin(), r.loaded.end(), 1);
            r.loaded_count = r.m;
        });
        return KS_OK;
    });
}

ks_status ks_matvec(ks_ctx* c, const double* x, double* y) {
    if (!c || !x || !y) return fail(c, KS_EARG, "NULL argument");
    if (!c->poisoned && !all_loaded(c)) return fail(c, KS_ESTATE, "matrix not fully loaded");
    return guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            if (c->dtype == KS_FLOAT32) {
                double* tmp = nullptr;
                ks::dev_alloc_t(&tmp, (size_t)c->n);
                KS_CUDA(cudaMemcpyAsync(tmp, x, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
                ks::launch_d2f(tmp, reinterpret_cast<float*>(r.s_full), c->n, r.stream);
                ks::GemvParamsT<float> p{};
                p.A = reinterpret_cast<const float*>(r.A); p.lda = c->ld; p.m = r.m; p.ncols = c->ld;
                p.x = reinterpret_cast<const float*>(r.s_full);
                p.y = reinterpret_cast<float*>(r.G_v) + (int64_t)r.rank * r.L.chunk;
                ks::launch_gemv_f32(p, r.scr, 1, r.stream);
                ks::allgather(c, r, r.G_v, r.L.chunk);
                ks::copy_chunks_to(c, r, r.G_v, r.p_full, cudaMemcpyDeviceToDevice);
                ks::launch_f2d(reinterpret_cast<const float*>(r.p_full), tmp, c->n, r.stream);
                if (c->writes_host(r))
                    KS_CUDA(cudaMemcpyAsync(y, tmp, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
                KS_CUDA(cudaStreamSynchronize(r.stream));
                KS_CUDA(cudaGetLastError());
                ks::dev_free(tmp);
                return;
            }
            KS_CUDA(cudaMemcpyAsync(r.s_full, x, (size_t)c->n * sizeof(double), cudaMemcpyDefault,
                                    r.stream));
            ks::GemvParams p{};
            p.A = r.A; p.lda = c->ld; p.m = r.m; p.ncols = c->ld;
            p.x = r.s_full;
            p.y = r.G_v + (int64_t)r.rank * r.L.chunk;
            ks::launch_gemv(p, ks::gemv_config(c, r), r.scr, 1, r.num_sms, r.stream);
            KS_CUDA(cudaGetLastError());
            ks::allgather(c, r, r.G_v, r.L.chunk);
            if (c->writes_host(r)) ks::copy_chunks_to(c, r, r.G_v, y, cudaMemcpyDefault);
            KS_CUDA(cudaStreamSynchronize(r.stream));
        });
        return KS_OK;
    });
}

ks_status ks_time_matvec(ks_ctx* c, int32_t reps, double* seconds) {
    if (!c || !seconds || reps < 1) return fail(c, KS_EARG, "bad argument");
    std::vector<double> per(c->ranks.size(), 0.0);
    ks_status st = guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            if (c->dtype == KS_FLOAT32) {
                ks::GemvParamsT<float> p{};
                p.A = reinterpret_cast<const float*>(r.A); p.lda = c->ld; p.m = r.m; p.ncols = c->ld;
                p.x = reinterpret_cast<const float*>(r.p_full);
                p.y = reinterpret_cast<float*>(r.q_loc);
                ks::launch_gemv_f32(p, r.scr, 1, r.stream);
                KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
                for (int q = 0; q < reps; ++q) ks::launch_gemv_f32(p, r.scr, 1, r.stream);
                KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
                KS_CUDA(cudaStreamSynchronize(r.stream));
                KS_CUDA(cudaGetLastError());
                float ms = 0.f;
                KS_CUDA(cudaEventElapsedTime(&ms, r.ev_t0, r.ev_t1));
                per[(size_t)(&r - c->ranks.data())] = ms * 1e-3 / reps;
                return;
            }
            ks::GemvParams p{};
            p.A = r.A; p.lda = c->ld; p.m = r.m; p.ncols = c->ld;
            p.x = r.p_full;
            p.y = r.q_loc;
            p.w1 = r.p_full + r.row0;
            p.out1 = r.S + (int64_t)r.rank * ks::kScalSlot;
            const ks::GemvConfig cfg = ks::gemv_config(c, r);
            ks::launch_gemv(p, cfg, r.scr, 1, r.num_sms, r.stream);   // warm-up
            KS_CUDA(cudaEventRecord(r.ev_t0, r.stream));
            for (int q = 0; q < reps; ++q) ks::launch_gemv(p, cfg, r.scr, 1, r.num_sms, r.stream);
            KS_CUDA(cudaEventRecord(r.ev_t1, r.stream));
            KS_CUDA(cudaStreamSynchronize(r.stream));
            KS_CUDA(cudaGetLastError());
            float ms = 0.f;
            KS_CUDA(cudaEventElapsedTime(&ms, r.ev_t0, r.ev_t1));
            per[(size_t)(&r - c->ranks.data())] = ms * 1e-3 / reps;
        });
        return KS_OK;
    });
    if (st == KS_OK) {
        double mx = 0.0;
        for (double v : per) mx = std::max(mx, v);
        *seconds = mx;
    }
    return st;
}

static ks_status solve(ks_ctx* c, int method, const double* b, const double* x0, double tol,
                       int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    if (!c) return fail(nullptr, KS_EARG, "ctx is NULL");
    if (!b || !x) return fail(c, KS_EARG, "b and x are required");
    if (!(tol >= 0.0)) return fail(c, KS_EARG, "tol must be >= 0");
    if (maxit < 0) return fail(c, KS_EARG, "maxit must be >= 0");
    if (hist_cap < 0 || (hist_cap > 0 && !hist)) return fail(c, KS_EARG, "bad hist/hist_cap");
    if (!hist) hist_cap = 0;
    if (c->dtype == KS_FLOAT32) {
        if (method == 2) return fail(c, KS_EARG, "BiCG is FP64-only");
        if (x0) return fail(c, KS_EARG, "FP32 path: x0 must be NULL (zero start)");
        if (!(c->P == 1 || c->fused())) return fail(c, KS_EARG, "FP32 path needs P == 1 or peer access");
    }
    if (c->poisoned) return fail(c, KS_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    if (!all_loaded(c)) return fail(c, KS_ESTATE, "matrix not fully loaded: call ks_load_rows / ks_generate first");
    std::vector<ks_report> reps(c->ranks.size());
    std::vector<int64_t> stat(c->ranks.size(), 0);
    ks_status st = guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            const size_t i = (size_t)(&r - c->ranks.data());
            if (c->dtype == KS_FLOAT32) {
                stat[i] = ks::run_f32(c, r, method == 1, b, tol, maxit, x, hist, hist_cap, &reps[i]);
                KS_CUDA(cudaGetLastError());
                return;
            }
            stat[i] = method == 1 ? ks::run_bicgstab(c, r, b, x0, tol, maxit, x, hist, hist_cap, &reps[i])
                    : method == 2 ? ks::run_bicg(c, r, b, x0, tol, maxit, x, hist, hist_cap, &reps[i])
                                  : ks::run_cg(c, r, b, x0, tol, maxit, x, hist, hist_cap, &reps[i]);
            KS_CUDA(cudaGetLastError());
        });
        return KS_OK;
    });
    if (st != KS_OK) return st;
    ks_report R = reps[0];
    for (auto& q : reps) {
        R.seconds_loop = std::max(R.seconds_loop, q.seconds_loop);
        R.seconds_total = std::max(R.seconds_total, q.seconds_total);
        R.seconds_gemv = std::max(R.seconds_gemv, q.seconds_gemv);
    }
    if (rep) *rep = R;
    const ks_status s = status_of(stat[0]);
    if (s == KS_ENCCL) return fail(c, KS_ENCCL, "fused collective wait timed out (peer rank lost)");
    if (s != KS_OK) {
        const char* what = s == KS_EMAXIT ? "maximum iterations reached"
                         : s == KS_ENOTSPD ? "CG: <p, A p> <= 0 (matrix not SPD)"
                         : s == KS_EBREAKDOWN ? "BiCGSTAB breakdown (zero or non-finite scalar)"
                                              : "solver failed";
        c->last_error = what;
        g_tls_error = what;
    }
    return s;
}

ks_status ks_cg(ks_ctx* c, const double* b, const double* x0, double tol, int64_t maxit, double* x,
                double* hist, int64_t hist_cap, ks_report* rep) {
    return solve(c, 0, b, x0, tol, maxit, x, hist, hist_cap, rep);
}

ks_status ks_bicg(ks_ctx* c, const double* b, const double* x0, double tol, int64_t maxit, double* x,
                  double* hist, int64_t hist_cap, ks_report* rep) {
    return solve(c, 2, b, x0, tol, maxit, x, hist, hist_cap, rep);
}

ks_status ks_gmres(ks_ctx* c, const double* b, const double* x0, double tol, int32_t restart,
                   int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    if (!c) return fail(nullptr, KS_EARG, "ctx is NULL");
    if (c->dtype != KS_FLOAT64) return fail(c, KS_EARG, "GMRES is FP64-only");
    if (!b || !x) return fail(c, KS_EARG, "b and x are required");
    if (!(tol >= 0.0)) return fail(c, KS_EARG, "tol must be >= 0");
    if (maxit < 0) return fail(c, KS_EARG, "maxit must be >= 0");
    if (restart < 1 || restart >= ks::kMaxBasis) return fail(c, KS_EARG, "restart must be in [1, 63]");
    if (hist_cap < 0 || (hist_cap > 0 && !hist)) return fail(c, KS_EARG, "bad hist/hist_cap");
    if (!hist) hist_cap = 0;
    if (c->poisoned) return fail(c, KS_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    if (!all_loaded(c)) return fail(c, KS_ESTATE, "matrix not fully loaded: call ks_load_rows / ks_generate first");
    std::vector<ks_report> reps(c->ranks.size());
    std::vector<int64_t> stat(c->ranks.size(), 0);
    ks_status st = guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            const size_t i = (size_t)(&r - c->ranks.data());
            stat[i] = ks::run_gmres(c, r, b, x0, tol, restart, maxit, x, hist, hist_cap, &reps[i]);
            KS_CUDA(cudaGetLastError());
        });
        return KS_OK;
    });
    if (st != KS_OK) return st;
    ks_report R = reps[0];
    for (auto& q : reps) {
        R.seconds_loop = std::max(R.seconds_loop, q.seconds_loop);
        R.seconds_total = std::max(R.seconds_total, q.seconds_total);
        R.seconds_gemv = std::max(R.seconds_gemv, q.seconds_gemv);
    }
    if (rep) *rep = R;
    const ks_status s = (ks_status)stat[0];
    if (s == KS_EMAXIT) { c->last_error = "maximum iterations reached"; g_tls_error = c->last_error; }
    return s;
}

static ks_status solve_multi(ks_ctx* c, int bicgstab, int32_t nrhs, const double* B, const double* X0, double tol,
                             int64_t maxit, double* X, double* hist, int64_t hist_cap, ks_report* reps) {
    if (!c) return fail(nullptr, KS_EARG, "ctx is NULL");
    if (!B || !X) return fail(c, KS_EARG, "B and X are required");
    if (nrhs < 1 || nrhs > ks::kMaxRhs) return fail(c, KS_EARG, "nrhs must be in [1, 8]");
    if (c->dtype != KS_FLOAT64) return fail(c, KS_EARG, "multi-RHS solvers are FP64-only");
    if (c->P != 1 && !c->fused()) return fail(c, KS_EARG, "multi-RHS solvers over P > 1 GPUs need peer access (fused exchange)");
    if (!(tol >= 0.0)) return fail(c, KS_EARG, "tol must be >= 0");
    if (maxit < 0) return fail(c, KS_EARG, "maxit must be >= 0");
    if (hist_cap < 0 || (hist_cap > 0 && !hist)) return fail(c, KS_EARG, "bad hist/hist_cap");
    if (!hist) hist_cap = 0;
    if (c->poisoned) return fail(c, KS_ESTATE, "context poisoned by an earlier CUDA/NCCL error");
    if (!all_loaded(c)) return fail(c, KS_ESTATE, "matrix not fully loaded: call ks_load_rows / ks_generate first");
    std::vector<int64_t> stat(c->ranks.size(), 0);
    ks_status st = guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            const size_t i = (size_t)(&r - c->ranks.data());
            // reports from the rank that writes the host outputs (all ranks agree)
            stat[i] = ks::run_multi(c, r, bicgstab, nrhs, B, X0, tol, maxit, X, hist, hist_cap,
                                    c->writes_host(r) ? reps : nullptr);
            KS_CUDA(cudaGetLastError());
        });
        return KS_OK;
    });
    if (st != KS_OK) return st;
    const ks_status s = status_of(stat[0]);
    if (s != KS_OK) {
        const char* what = s == KS_EMAXIT ? "maximum iterations reached (some column)"
                         : s == KS_EBREAKDOWN ? "BiCGSTAB breakdown in some column (zero or non-finite scalar)"
                                              : "CG: <p, A p> <= 0 in some column (matrix not SPD)";
        c->last_error = what;
        g_tls_error = what;
    }
    return s;
}

ks_status ks_cg_multi(ks_ctx* c, int32_t nrhs, const double* B, const double* X0, double tol, int64_t maxit,
                      double* X, double* hist, int64_t hist_cap, ks_report* reps) {
    return solve_multi(c, 0, nrhs, B, X0, tol, maxit, X, hist, hist_cap, reps);
}

ks_status ks_bicgstab_multi(ks_ctx* c, int32_t nrhs, const double* B, const double* X0, double tol, int64_t maxit,
                            double* X, double* hist, int64_t hist_cap, ks_report* reps) {
    return solve_multi(c, 1, nrhs, B, X0, tol, maxit, X, hist, hist_cap, reps);
}

ks_status ks_matvec_t(ks_ctx* c, const double* x, double* y) {
    if (!c || !x || !y) return fail(c, KS_EARG, "NULL argument");
    if (c->dtype != KS_FLOAT64) return fail(c, KS_EARG, "ks_matvec_t is FP64-only");
    if (!c->poisoned && !all_loaded(c)) return fail(c, KS_ESTATE, "matrix not fully loaded");
    return guarded(c, [&] {
        c->for_each_rank([&](Rank& r) {
            KS_CUDA(cudaMemcpyAsync(r.q_loc, x + r.row0, (size_t)r.m * sizeof(double), cudaMemcpyDefault,
                                    r.stream));
            const double* mine = ks::gemv_t(c, r, r.q_loc, nullptr);
            // gather every rank's rows of A^T x (chunk layout) and copy out
            if (c->P > 1) {
                KS_CUDA(cudaMemcpyAsync(r.G_v + (int64_t)r.rank * r.L.chunk, mine,
                                        (size_t)r.m * sizeof(double), cudaMemcpyDeviceToDevice, r.stream));
                ks::allgather(c, r, r.G_v, r.L.chunk);
                if (c->writes_host(r)) ks::copy_chunks_to(c, r, r.G_v, y, cudaMemcpyDefault);
            } else {
                KS_CUDA(cudaMemcpyAsync(y, mine, (size_t)c->n * sizeof(double), cudaMemcpyDefault, r.stream));
            }
            KS_CUDA(cudaStreamSynchronize(r.stream));
        });
        return KS_OK;
    });
}

ks_status ks_bicgstab(ks_ctx* c, const double* b, const double* x0, double tol, int64_t maxit,
                      double* x, double* hist, int64_t hist_cap, ks_report* rep) {
    return solve(c, 1, b, x0, tol, maxit, x, hist, hist_cap, rep);
}

ks_status ks_set_option(ks_ctx* c, ks_option opt, int64_t v) {
    if (!c) return fail(nullptr, KS_EARG, "ctx is NULL");
    ks::Options& o = c->opt;
    switch (opt) {
        case KS_OPT_TRUE_RESIDUAL: o.true_residual = v ? 1 : 0; break;
        case KS_OPT_PROFILE_GEMV: o.profile_gemv = v ? 1 : 0; break;
        case KS_OPT_POLL_BATCH:
            if (v < 0 || v > 4096) return fail(c, KS_EARG, "poll batch must be in [0, 4096]");
            o.poll_batch = v; break;
        case KS_OPT_GEMV_ROWS:
            if (v != 0 && v != 1 && v != 2 && v != 4 && v != 8 && v != 16)
                return fail(c, KS_EARG, "rows must be 0, 1 (persistent kernels only), 2, 4, 8 or 16");
            o.gemv_rows = v; break;
        case KS_OPT_GEMV_SPLIT:
            if (v < 0 || v > 64) return fail(c, KS_EARG, "split must be in [0, 64]");
            o.gemv_split = v; break;
        case KS_OPT_GEMV_KERNEL:
            if (v < 0 || v > 1) return fail(c, KS_EARG, "kernel must be 0 or 1 (the TMA variant was removed)");
            o.gemv_kernel = v; break;
        case KS_OPT_USE_GRAPHS: o.use_graphs = v ? 1 : 0; break;
        case KS_OPT_FUSED_COMM:
            if (v && c->shared_dev)
                return fail(c, KS_EARG, "ranks sharing a GPU cannot use the fused exchange (kernels that wait on "
                                        "each other have no co-residency guarantee across launches)");
            o.fused_comm = v ? 1 : 0; break;
        case KS_OPT_PERSISTENT:
            if (v < 0 || v > 2) return fail(c, KS_EARG, "persistent must be 0, 1 or 2");
            o.persistent = v; break;
        case KS_OPT_GEMV_UNROLL:
            if (v != 0 && v != 1 && v != 2 && v != 4 && v != 8) return fail(c, KS_EARG, "unroll must be 0, 1, 2, 4 or 8");
            o.gemv_unroll = v; break;
        case KS_OPT_PERSIST_GRID:
            if (v < 0 || v > 1 << 20) return fail(c, KS_EARG, "bad persistent grid");
            o.persist_grid = v; break;
        case KS_OPT_GEMVT_SHAPE:
            if (!ks::gemv_t_shape_ok(v)) return fail(c, KS_EARG, "gemvt shape must be (1|2|4) * 100 + (4|8|16)");
            o.gemvt_shape = v; break;
        case KS_OPT_SMALL:
            if (v < 0 || v > 2) return fail(c, KS_EARG, "small must be 0, 1 or 2");
            o.small = v; break;
        case KS_OPT_JOIN_TIMEOUT_MS:
            if (v < 1 || v > 3600000) return fail(c, KS_EARG, "join timeout must be in [1, 3600000] ms");
            o.join_timeout_ms = v; break;
        case KS_OPT_TINY:
            if (v < 0 || v > 1) return fail(c, KS_EARG, "tiny must be 0 or 1");
            o.tiny = v; break;
        case KS_OPT_JITTER: {
            if (v < 0 || v > 0xffffffffLL) return fail(c, KS_EARG, "jitter seed must be in [0, 2^32)");
            const unsigned seed = (unsigned)v;
            ks_status st = guarded(c, [&] {
                c->for_each_rank([&](Rank& r) {
                    KS_CUDA(cudaStreamSynchronize(r.stream));
                    KS_CUDA(cudaMemcpy(&r.st->jitter, &seed, sizeof(seed), cudaMemcpyHostToDevice));
                    r.jitter = seed;
                    for (auto& g : r.graphs) g.kind = -1;   // captured kernel parameters are stale
                });
                return KS_OK;
            });
            if (st != KS_OK) return st;
            o.jitter = v;
            break;
        }
        case KS_OPT_LL_XCHG:
            if (v < 0 || v > 1) return fail(c, KS_EARG, "ll_xchg must be 0 or 1");
            o.ll_xchg = v;
            for (auto& r : c->ranks) r.ll_on = (int)v;
            break;
        default: return fail(c, KS_EARG, "unknown option");
    }
    return KS_OK;
}

ks_status ks_check_guards(const ks_ctx* c, int64_t* violations) {
    if (!c || !violations) return fail(nullptr, KS_EARG, "NULL argument");
    std::vector<int> devs;
    for (const auto& r : c->ranks) devs.push_back(r.dev);
    *violations = ks::guard_check(devs);
    return KS_OK;
}

ks_status ks_get_option(const ks_ctx* c, ks_option opt, int64_t* v) {
    if (!c || !v) return fail(nullptr, KS_EARG, "NULL argument");
    const ks::Options& o = c->opt;
    switch (opt) {
        case KS_OPT_TRUE_RESIDUAL: *v = o.true_residual; break;
        case KS_OPT_PROFILE_GEMV: *v = o.profile_gemv; break;
        case KS_OPT_POLL_BATCH: *v = o.poll_batch; break;
        case KS_OPT_GEMV_ROWS: *v = o.gemv_rows; break;
        case KS_OPT_GEMV_SPLIT: *v = o.gemv_split; break;
        case KS_OPT_GEMV_KERNEL: *v = o.gemv_kernel; break;
        case KS_OPT_USE_GRAPHS: *v = o.use_graphs; break;
        case KS_OPT_FUSED_COMM: *v = c->fused() ? 1 : 0; break;   // effective value
        case KS_OPT_PERSISTENT: *v = c->persistent() ? 1 : 0; break;  // effective value
        case KS_OPT_GEMV_UNROLL: *v = o.gemv_unroll; break;
        case KS_OPT_PERSIST_GRID: *v = o.persist_grid; break;
        case KS_OPT_GEMVT_SHAPE: *v = o.gemvt_shape; break;
        case KS_OPT_SMALL: *v = o.small; break;
        case KS_OPT_JOIN_TIMEOUT_MS: *v = o.join_timeout_ms; break;
        case KS_OPT_TINY: *v = o.tiny; break;
        case KS_OPT_JITTER: *v = o.jitter; break;
        case KS_OPT_LL_XCHG: *v = (o.ll_xchg && (c->fused() || c->shared_dev)) ? 1 : 0; break;   // effective
        default: return fail(const_cast<ks_ctx*>(c), KS_EARG, "unknown option");
    }
    return KS_OK;
}

ks_status ks_info(const ks_ctx* c, int32_t* local_gpus, int32_t* nranks, int64_t* n, int64_t* ld) {
    if (!c) return fail(nullptr, KS_EARG, "ctx is NULL");
    if (local_gpus) *local_gpus = (int32_t)c->ranks.size();
    if (nranks) *nranks = c->P;
    if (n) *n = c->n;
    if (ld) *ld = c->ld;
    return KS_OK;
}

const char* ks_last_error(const ks_ctx* c) {
    if (c) return c->last_error.c_str();
    return g_tls_error.c_str();
}

const char* ks_version(void) { return "ks 0.1 sm_100a (FP64 dense CG/BiCGSTAB)"; }

}  // extern "C"

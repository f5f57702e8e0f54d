// L3 context: partition, device allocation, NCCL plumbing, worker threads.
#include "ks_ctx.h"

#include <algorithm>
#include <chrono>
#include <exception>
#include <mutex>
#include <thread>

namespace ks {

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    const ks_status code = (e == cudaErrorMemoryAllocation) ? KS_ENOMEM : KS_ECUDA;
    throw KsError(code, std::string(what) + ": " + cudaGetErrorString(e));
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    throw KsError(KS_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

VecArgs Rank::vargs(bool fused) const {
    VecArgs a;
    a.gpar = fused ? (int64_t)L.P * L.chunk : 0;
    a.spar = fused ? (int64_t)L.P * kScalSlot : 0;
    a.peer = fused ? 1 : 0;
    a.jitter = jitter;
    a.ll = (fused && llg) ? ll_on : 0;
    a.llg = llg;
    a.pp = pp;
    a.flags = flags;
    a.L = L;
    a.st = st;
    a.hist = hist;
    a.b_full = b_full;
    a.x_loc = x_loc;
    a.p_full = p_full;
    a.s_full = s_full;
    a.v_full = v_full;
    a.q_loc = q_loc;
    a.rhat_loc = rhat_loc;
    a.pt_loc = pt_loc;
    a.qt_loc = (L.P > 1) ? qt_loc : U;
    a.G_r = G_r;
    a.G_v = G_v;
    a.S = S;
    a.X = X;
    a.scr = scr;
    a.num_sms = num_sms;
    return a;
}

template <class T>
static void dmalloc(T** p, size_t count) {
    dev_alloc_t(p, std::max<size_t>(count, 1));
    KS_CUDA(cudaMemset(*p, 0, std::max<size_t>(count, 1) * sizeof(T)));
}
// element buffers of the context's dtype (double* members hold floats in FP32 contexts)
static void emalloc(double** p, size_t count, size_t esz) {
    const size_t bytes = std::max<size_t>(count, 1) * esz;
    *p = static_cast<double*>(dev_alloc(bytes));
    KS_CUDA(cudaMemset(*p, 0, bytes));
}
template <class T>
static T* as(double* p) { return reinterpret_cast<T*>(p); }

void rank_alloc(ks_ctx* c, Rank& r) {
    KS_CUDA(cudaSetDevice(r.dev));
    KS_CUDA(cudaDeviceGetAttribute(&r.num_sms, cudaDevAttrMultiProcessorCount, r.dev));
    if (!r.stream) {
        KS_CUDA(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
        r.own_stream = true;
    }
    r.ll_on = (int)c->opt.ll_xchg;
    const int64_t ld = c->ld;
    const size_t P = (size_t)c->P;
    const size_t e = c->esz;
    emalloc(&r.A, (size_t)r.m * (size_t)ld, e);     // zero padding columns [n, ld)
    emalloc(&r.b_full, ld, e);
    emalloc(&r.x_loc, r.m + 64, e);
    emalloc(&r.p_full, ld, e);
    emalloc(&r.s_full, ld, e);
    emalloc(&r.v_full, ld, e);
    emalloc(&r.q_loc, r.m + 64, e);
    emalloc(&r.rhat_loc, r.m + 64, e);
    emalloc(&r.pt_loc, r.m + 64, e);
    emalloc(&r.U, P * (size_t)r.L.chunk, e);
    emalloc(&r.qt_loc, (size_t)r.L.chunk, e);
    {
        // exchange buffers (one allocation -> one CUDA IPC handle), byte layout
        const size_t g = 2 * P * (size_t)r.L.chunk * e;
        const size_t sb = (2 * P * kScalSlot * e + 511) / 512 * 512;
        const size_t fb = (kNumPhases * kMaxRanks * sizeof(unsigned long long) + 511) / 512 * 512;
        const size_t xb = ((size_t)ld * e + 511) / 512 * 512;
        // multi-RHS CG over P > 1 (FP64 contexts): r slices, rank partials, gathered x
        const bool mm = c->dtype == KS_FLOAT64 && P > 1;
        const size_t mrb = mm ? 2 * P * (size_t)kMaxRhs * (size_t)r.L.chunk * sizeof(double) : 0;
        const size_t msb = mm ? (2 * P * 6 * (size_t)kMaxRhs * sizeof(double) + 511) / 512 * 512 : 0;
        const size_t mxb = mm ? (size_t)kMaxRhs * (size_t)ld * sizeof(double) : 0;
        const size_t mvb = mrb;                     // v slices of multi-RHS BiCGSTAB
        // tiny kernels over P > 1 (n <= 1024): their LL exchange slots, 4 ld words
        const size_t llb = (P > 1 && ld <= 1024) ? 4 * (size_t)ld * sizeof(uint64_t) : 0;
        const size_t lgb = P > 1 ? (size_t)ll_words(ld) * sizeof(uint64_t) : 0;   // persistent LL handovers
        const size_t total = 2 * g + sb + fb + xb + mrb + msb + mxb + llb + mvb + lgb;
        char* base = nullptr;
        KS_CUDA(cudaMalloc(reinterpret_cast<void**>(&base), total));
        KS_CUDA(cudaMemset(base, 0, total));
        r.xbuf = reinterpret_cast<double*>(base);
        r.xbuf_bytes = total;
        r.G_r = reinterpret_cast<double*>(base);
        r.G_v = reinterpret_cast<double*>(base + g);
        r.S = reinterpret_cast<double*>(base + 2 * g);
        r.flags = reinterpret_cast<unsigned long long*>(base + 2 * g + sb);
        r.X = reinterpret_cast<double*>(base + 2 * g + sb + fb);
        r.MR = mm ? reinterpret_cast<double*>(base + 2 * g + sb + fb + xb) : nullptr;
        r.MS = mm ? reinterpret_cast<double*>(base + 2 * g + sb + fb + xb + mrb) : nullptr;
        r.MX = mm ? reinterpret_cast<double*>(base + 2 * g + sb + fb + xb + mrb + msb) : nullptr;
        r.llx = llb ? reinterpret_cast<uint64_t*>(base + 2 * g + sb + fb + xb + mrb + msb + mxb) : nullptr;
        r.MV = mm ? reinterpret_cast<double*>(base + 2 * g + sb + fb + xb + mrb + msb + mxb + llb) : nullptr;
        r.llg = lgb ? reinterpret_cast<uint64_t*>(base + 2 * g + sb + fb + xb + mrb + msb + mxb + llb + mvb) : nullptr;
        for (int q = 0; q < kMaxRanks; ++q) r.llpeer[q] = nullptr;
        r.llpeer[r.rank] = r.llx;
        for (int q = 0; q < kMaxRanks; ++q) {
            r.mpeer.MR[q] = r.mpeer.MS[q] = r.mpeer.MX[q] = r.mpeer.MV[q] = nullptr;
            r.mpeer.flags[q] = nullptr;
        }
        r.mpeer.MR[r.rank] = r.MR;
        r.mpeer.MS[r.rank] = r.MS;
        r.mpeer.MX[r.rank] = r.MX;
        r.mpeer.MV[r.rank] = r.MV;
        r.mpeer.flags[r.rank] = r.flags;
        for (int q = 0; q < kMaxRanks; ++q) {
            r.pp.G_r[q] = r.pp.G_v[q] = r.pp.S[q] = r.pp.X[q] = nullptr;
            r.pp.flags[q] = nullptr;
            r.pp.llg[q] = nullptr;
        }
        r.pp.llg[r.rank] = r.llg;
        r.pp.X[r.rank] = r.X;
        r.pp.G_r[r.rank] = r.G_r;
        r.pp.G_v[r.rank] = r.G_v;
        r.pp.S[r.rank] = r.S;
        r.pp.flags[r.rank] = r.flags;
    }
    dmalloc(&r.st, 1);
    dmalloc(&r.kdev, 1);
    r.hist_alloc = 1024;
    dmalloc(&r.hist, r.hist_alloc);
    dmalloc(&r.scr.part, (size_t)kNumTickets * kPartStride);
    dmalloc(&r.scr.ticket, kNumTickets);
    r.scr.tile_cap = r.m / 2 + 2;                  // tiles of the smallest row count (R = 2)
    r.scr.qpart_cap = std::max<int64_t>(2 * 6 * 2 * 160 * 16 + 4096, 2 * r.scr.tile_cap + 4096);
    dmalloc(&r.scr.qpart, r.scr.qpart_cap);
    dmalloc(&r.scr.tile_ticket, r.scr.tile_cap);
    KS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&r.h_done), 2 * sizeof(int)));
    KS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&r.h_hist), (size_t)kHistStage * sizeof(double)));
    KS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&r.h_state), sizeof(DevState)));
    for (auto& e : r.ev_poll) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreate(&r.ev_t0));
    KS_CUDA(cudaEventCreate(&r.ev_t1));
    for (auto& e : r.ev_coll) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    r.loaded.assign((size_t)r.m, 0);
    r.loaded_count = 0;
    KS_CUDA(cudaDeviceSynchronize());
}

// Buffers replaced while a call runs are freed at the start of the next call (or at
// destroy), never inside it: cudaFree synchronises the whole device, so inside a call
// it can wait on a kernel that spins for a peer rank's not-yet-launched work (found
// with ranks sharing a GPU, §15.7).
void retire(Rank& r, void* p) {
    if (p) r.retired.push_back(p);
}
void flush_retired(Rank& r) {
    for (void* p : r.retired) dev_free(p);
    r.retired.clear();
}

void rank_free(Rank& r) {
    if (cudaSetDevice(r.dev) != cudaSuccess) return;
    cudaDeviceSynchronize();
    flush_retired(r);
    for (void* p : r.ipc_opened) cudaIpcCloseMemHandle(p);
    r.ipc_opened.clear();
    if (r.xbuf) cudaFree(r.xbuf);                 // IPC-exported: plain cudaMalloc
    for (void* p : {(void*)r.A, (void*)r.b_full, (void*)r.x_loc, (void*)r.p_full, (void*)r.s_full, (void*)r.v_full,
                    (void*)r.q_loc, (void*)r.rhat_loc,
                    (void*)r.st, (void*)r.hist, (void*)r.scr.part, (void*)r.scr.ticket,
                    (void*)r.scr.qpart, (void*)r.scr.tile_ticket, (void*)r.table_tmp,
                    (void*)r.kdev, (void*)r.pt_loc, (void*)r.U, (void*)r.qt_loc,
                    (void*)r.upart, (void*)r.col_ticket, (void*)r.gmV, (void*)r.gmH,
                    (void*)r.gm_hx, (void*)r.gm_state, (void*)r.ll, (void*)r.mX, (void*)r.mR,
                    (void*)r.mQ, (void*)r.mP, (void*)r.mhist, (void*)r.mstate, (void*)r.mRh,
                    (void*)r.mT, (void*)r.mS})
        if (p) dev_free(p);
    if (r.h_done) cudaFreeHost(r.h_done);
    if (r.h_hist) cudaFreeHost(r.h_hist);
    if (r.h_state) cudaFreeHost(r.h_state);
    for (auto e : r.ev_poll) if (e) cudaEventDestroy(e);
    if (r.ev_t0) cudaEventDestroy(r.ev_t0);
    if (r.ev_t1) cudaEventDestroy(r.ev_t1);
    for (auto e : r.ev_coll) if (e) cudaEventDestroy(e);
    if (r.rs_stage) dev_free(r.rs_stage);
    for (auto e : r.ev_gemv) cudaEventDestroy(e);
    for (auto& g : r.graphs) if (g.exec) cudaGraphExecDestroy(g.exec);
    r.ev_gemv.clear();
    if (r.own_comm && r.comm) ncclCommDestroy(r.comm);
    if (r.own_stream && r.stream) cudaStreamDestroy(r.stream);
    r = Rank{};
}

void HostBarrier::reset(int parties) {
    std::lock_guard<std::mutex> g(mu);
    n = parties;
    count = 0;
    aborted = false;
}

void HostBarrier::wait() {
    std::unique_lock<std::mutex> g(mu);
    if (aborted) throw KsError(KS_ENCCL, "host collective: a peer rank failed");
    const unsigned long long my = gen;
    if (++count == n) {
        count = 0;
        ++gen;
        cv.notify_all();
        return;
    }
    // bounded: a rank that never arrives (a bug) fails the call instead of hanging it
    if (!cv.wait_for(g, std::chrono::seconds(120), [&] { return gen != my || aborted; })) {
        aborted = true;
        cv.notify_all();
        throw KsError(KS_ENCCL, "host collective: timed out waiting for the peer ranks");
    }
    if (gen == my) throw KsError(KS_ENCCL, "host collective: a peer rank failed");
}

void HostBarrier::abort() {
    std::lock_guard<std::mutex> g(mu);
    aborted = true;
    cv.notify_all();
}

namespace {

// Host-driven collective step of a shared-device context (one process, no NCCL):
// every rank records `ev_coll[0]` after its producer, the worker threads meet, each
// stream waits for every peer's producer and pulls what it needs with peer copies
// (`pull`), records `ev_coll[1]`, the threads meet again and each stream waits for
// every peer's pulls -- so no rank overwrites a region a peer is still reading.
// Stream-ordered: no host synchronisation with the device.
template <class F>
void host_collective(const ks_ctx* c, Rank& r, F&& pull) {
    KS_CUDA(cudaEventRecord(r.ev_coll[0], r.stream));
    c->hbar->wait();
    for (const Rank& h : c->ranks)
        if (h.rank != r.rank) KS_CUDA(cudaStreamWaitEvent(r.stream, h.ev_coll[0], 0));
    pull();
    KS_CUDA(cudaEventRecord(r.ev_coll[1], r.stream));
    c->hbar->wait();
    for (const Rank& h : c->ranks)
        if (h.rank != r.rank) KS_CUDA(cudaStreamWaitEvent(r.stream, h.ev_coll[1], 0));
}

}  // namespace

// Ranks sharing one GPU: rank 0 runs `launch` once on its stream after every rank's
// stream reached this point (events), and every rank's stream continues after it --
// a single launch may then serve all ranks (their kernels wait on each other, so
// they must be ONE launch to be co-resident).
void host_launch_once(const ks_ctx* c, Rank& r, const std::function<void()>& launch) {
    KS_CUDA(cudaEventRecord(r.ev_coll[0], r.stream));
    c->hbar->wait();
    if (r.rank == 0) {
        for (const Rank& h : c->ranks)
            if (h.rank != 0) KS_CUDA(cudaStreamWaitEvent(r.stream, h.ev_coll[0], 0));
        launch();
        KS_CUDA(cudaEventRecord(r.ev_coll[1], r.stream));
    }
    c->hbar->wait();
    if (r.rank != 0) KS_CUDA(cudaStreamWaitEvent(r.stream, c->ranks[0].ev_coll[1], 0));
}

// In-place allgather of one chunk per rank (count_per_rank doubles at G + rank*chunk).
// G is one of the exchange regions (G_r, G_v, S) of this rank's exchange allocation.
void allgather(const ks_ctx* c, Rank& r, double* G, int64_t count_per_rank) {
    if (c->P == 1) return;
    char* base = reinterpret_cast<char*>(G);
    const size_t cb = (size_t)count_per_rank * c->esz;
    if (!r.comm) {                      // ranks sharing a GPU: host-driven peer copies
        if (!c->shared_dev) throw KsError(KS_ESTATE, "allgather without a communicator");
        // G lies in this rank's exchange allocation or its GMRES partials; the peer's
        // copy of the region sits at the same offset of the peer's allocation
        const char* xb = reinterpret_cast<const char*>(r.xbuf);
        const char* hb = reinterpret_cast<const char*>(r.gm_hx);
        const bool in_x = base >= xb && base < xb + r.xbuf_bytes;
        const bool in_h = hb && base >= hb && base < hb + (size_t)c->P * kMaxBasis * sizeof(double);
        if (!in_x && !in_h) throw KsError(KS_ESTATE, "allgather: buffer outside the exchange regions");
        const size_t off = (size_t)(base - (in_x ? xb : hb));
        host_collective(c, r, [&] {
            for (const Rank& h : c->ranks) {
                if (h.rank == r.rank) continue;
                const char* src = reinterpret_cast<const char*>(in_x ? (const void*)h.xbuf : (const void*)h.gm_hx) +
                                  off + (size_t)h.rank * cb;
                KS_CUDA(cudaMemcpyAsync(base + (size_t)h.rank * cb, src, cb, cudaMemcpyDefault, r.stream));
            }
        });
        return;
    }
    KS_NCCL(ncclAllGather(base + (size_t)r.rank * cb, base, (size_t)count_per_rank,
                          c->dtype == KS_FLOAT32 ? ncclFloat : ncclDouble, r.comm, r.stream));
}

// Sum over ranks of every rank's slot `r.rank` of U (chunk layout) into r.qt_loc:
// the reduce-scatter of K1T.  Shared-device contexts: peer copies of the P slots into
// a staging buffer, then a rank-ordered sum (launch_sum_slots).
static void reduce_scatter_u(const ks_ctx* c, Rank& r) {
    const int64_t chunk = r.L.chunk;
    if (r.comm) {
        KS_NCCL(ncclReduceScatter(r.U, r.qt_loc, (size_t)chunk, ncclDouble, ncclSum, r.comm, r.stream));
        return;
    }
    if (!c->shared_dev) throw KsError(KS_ESTATE, "reduce-scatter without a communicator");
    if (!r.rs_stage) dev_alloc_t(&r.rs_stage, (size_t)c->P * (size_t)chunk);
    host_collective(c, r, [&] {
        for (const Rank& h : c->ranks)
            KS_CUDA(cudaMemcpyAsync(r.rs_stage + (int64_t)h.rank * chunk, h.U + (int64_t)r.rank * chunk,
                                    (size_t)chunk * sizeof(double), cudaMemcpyDefault, r.stream));
    });
    r.launches += launch_sum_slots(r.rs_stage, c->P, chunk, r.qt_loc, r.num_sms, r.stream);
}

// Copies the P row slices held in chunk layout to a contiguous n-vector.
VecArgsT<float> Rank::vargs_f32(bool fused) const {
    VecArgsT<float> a;
    a.L = L;
    a.st = st;
    a.hist = hist;
    a.b_full = as<float>(b_full);
    a.x_loc = as<float>(x_loc);
    a.p_full = as<float>(p_full);
    a.s_full = as<float>(s_full);
    a.v_full = as<float>(v_full);
    a.q_loc = as<float>(q_loc);
    a.rhat_loc = as<float>(rhat_loc);
    a.pt_loc = as<float>(pt_loc);
    a.qt_loc = as<float>(qt_loc);
    a.G_r = as<float>(G_r);
    a.G_v = as<float>(G_v);
    a.S = as<float>(S);
    a.scr = scr;
    a.num_sms = num_sms;
    a.gpar = fused ? (int64_t)L.P * L.chunk : 0;
    a.spar = fused ? (int64_t)L.P * kScalSlot : 0;
    a.peer = fused ? 1 : 0;
    a.jitter = jitter;
    a.ll = (fused && llg) ? ll_on : 0;
    a.llg = llg;
    for (int g = 0; g < kMaxRanks; ++g) {
        a.pp.llg[g] = pp.llg[g];
        a.pp.G_r[g] = as<float>(pp.G_r[g]);
        a.pp.G_v[g] = as<float>(pp.G_v[g]);
        a.pp.S[g] = as<float>(pp.S[g]);
        a.pp.flags[g] = pp.flags[g];
        a.pp.X[g] = as<float>(pp.X[g]);
    }
    a.flags = flags;
    a.X = as<float>(X);
    return a;
}

// Elements are of the context's dtype (G and dst both).
void copy_chunks_to(const ks_ctx* c, Rank& r, const double* G, double* dst, cudaMemcpyKind kind) {
    const size_t e = c->esz;
    const char* src = reinterpret_cast<const char*>(G);
    char* out = reinterpret_cast<char*>(dst);
    for (int g = 0; g < c->P; ++g) {
        const int64_t b = r.L.row0[g], en = r.L.row0[g + 1];
        if (en > b)
            KS_CUDA(cudaMemcpyAsync(out + (size_t)b * e, src + (size_t)g * (size_t)r.L.chunk * e,
                                    (size_t)(en - b) * e, kind, r.stream));
    }
}

// Makes every rank's exchange buffers addressable from every other rank:
// - one process, several GPUs: cudaDeviceEnablePeerAccess, raw pointers;
// - one process per GPU: CUDA IPC handles of the exchange allocation, exchanged
//   over the (borrowed) NCCL communicator itself, opened with lazy peer access.
// Peer access is required for the fused collectives; without it the context
// keeps the NCCL collectives (opt.fused_comm is then ineffective).
void setup_peers(ks_ctx* c) {
    if (c->P == 1) return;
    auto boff = [&](const void* p) {
        return (size_t)(static_cast<const char*>(p) - reinterpret_cast<const char*>(c->ranks[0].xbuf));
    };
    const size_t offGv = boff(c->ranks[0].G_v), offS = boff(c->ranks[0].S), offF = boff(c->ranks[0].flags),
                 offX = boff(c->ranks[0].X);
    const bool mm = c->ranks[0].MR != nullptr;
    const size_t offMR = mm ? boff(c->ranks[0].MR) : 0, offMS = mm ? boff(c->ranks[0].MS) : 0,
                 offMX = mm ? boff(c->ranks[0].MX) : 0;
    const size_t offMV = mm ? boff(c->ranks[0].MV) : 0;
    const bool hasll = c->ranks[0].llx != nullptr;
    const size_t offLL = hasll ? boff(c->ranks[0].llx) : 0;
    const bool hasllg = c->ranks[0].llg != nullptr;
    const size_t offLLG = hasllg ? boff(c->ranks[0].llg) : 0;
    if (!c->multiprocess) {
        bool ok = true;
        for (auto& a : c->ranks)
            for (auto& b : c->ranks) {
                if (a.dev == b.dev) continue;
                int can = 0;
                KS_CUDA(cudaDeviceCanAccessPeer(&can, a.dev, b.dev));
                if (!can) { ok = false; continue; }
                KS_CUDA(cudaSetDevice(a.dev));
                cudaError_t e = cudaDeviceEnablePeerAccess(b.dev, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else KS_CUDA(e);
            }
        for (auto& a : c->ranks) {
            for (auto& b : c->ranks) {
                a.pp.G_r[b.rank] = b.G_r;
                a.pp.G_v[b.rank] = b.G_v;
                a.pp.S[b.rank] = b.S;
                a.pp.flags[b.rank] = b.flags;
                a.pp.X[b.rank] = b.X;
                a.mpeer.MR[b.rank] = b.MR;
                a.mpeer.MS[b.rank] = b.MS;
                a.mpeer.MX[b.rank] = b.MX;
                a.mpeer.MV[b.rank] = b.MV;
                a.mpeer.flags[b.rank] = b.flags;
                a.llpeer[b.rank] = b.llx;
                a.pp.llg[b.rank] = b.llg;
            }
            a.peer_ok = ok;
        }
        return;
    }
    Rank& r = c->ranks[0];
    KS_CUDA(cudaSetDevice(r.dev));
    cudaIpcMemHandle_t mine;
    KS_CUDA(cudaIpcGetMemHandle(&mine, r.xbuf));
    const size_t hs = sizeof(cudaIpcMemHandle_t);
    char* dbuf = nullptr;
    KS_CUDA(cudaMalloc(reinterpret_cast<void**>(&dbuf), hs * (size_t)c->P));
    KS_CUDA(cudaMemcpy(dbuf + hs * (size_t)r.rank, &mine, hs, cudaMemcpyHostToDevice));
    KS_NCCL(ncclAllGather(dbuf + hs * (size_t)r.rank, dbuf, hs, ncclChar, r.comm, r.stream));
    std::vector<cudaIpcMemHandle_t> all((size_t)c->P);
    KS_CUDA(cudaStreamSynchronize(r.stream));
    KS_CUDA(cudaMemcpy(all.data(), dbuf, hs * (size_t)c->P, cudaMemcpyDeviceToHost));
    KS_CUDA(cudaFree(dbuf));
    bool ok = true;
    for (int g = 0; g < c->P; ++g) {
        if (g == r.rank) continue;
        void* base = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&base, all[(size_t)g], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) { cudaGetLastError(); ok = false; continue; }
        r.ipc_opened.push_back(base);
        char* d = static_cast<char*>(base);
        r.pp.G_r[g] = reinterpret_cast<double*>(d);
        r.pp.G_v[g] = reinterpret_cast<double*>(d + offGv);
        r.pp.S[g] = reinterpret_cast<double*>(d + offS);
        r.pp.flags[g] = reinterpret_cast<unsigned long long*>(d + offF);
        r.pp.X[g] = reinterpret_cast<double*>(d + offX);
        r.mpeer.flags[g] = reinterpret_cast<unsigned long long*>(d + offF);
        if (hasll) r.llpeer[g] = reinterpret_cast<uint64_t*>(d + offLL);
        if (hasllg) r.pp.llg[g] = reinterpret_cast<uint64_t*>(d + offLLG);
        if (mm) {
            r.mpeer.MR[g] = reinterpret_cast<double*>(d + offMR);
            r.mpeer.MS[g] = reinterpret_cast<double*>(d + offMS);
            r.mpeer.MX[g] = reinterpret_cast<double*>(d + offMX);
            r.mpeer.MV[g] = reinterpret_cast<double*>(d + offMV);
        }
    }
    // every rank must agree, or none uses the fused path (collectives must match)
    int* dok = nullptr;
    KS_CUDA(cudaMalloc(reinterpret_cast<void**>(&dok), sizeof(int)));
    int hok = ok ? 1 : 0;
    KS_CUDA(cudaMemcpy(dok, &hok, sizeof(int), cudaMemcpyHostToDevice));
    KS_NCCL(ncclAllReduce(dok, dok, 1, ncclInt, ncclMin, r.comm, r.stream));
    KS_CUDA(cudaStreamSynchronize(r.stream));
    KS_CUDA(cudaMemcpy(&hok, dok, sizeof(int), cudaMemcpyDeviceToHost));
    KS_CUDA(cudaFree(dok));
    r.peer_ok = hok != 0;
}

const double* gemv_t(ks_ctx* c, Rank& r, const double* x_loc, const int* done, long long k,
                     unsigned long long ebase) {
    const int shape = (int)c->opt.gemvt_shape;
    const int64_t rc = gemv_t_chunk_rows(r.m, c->ld, r.num_sms, shape);
    const int64_t nrc = (r.m + rc - 1) / rc;
    const int64_t need = nrc * c->ld;
    if (need > r.upart_cap) {
        retire(r, r.upart);
        retire(r, r.col_ticket);
        r.upart = nullptr;
        r.col_ticket = nullptr;
        dev_alloc_t(&r.upart, (size_t)need);
        dev_alloc_t(&r.col_ticket, (size_t)(c->ld / 512 + 2));
        KS_CUDA(cudaMemset(r.col_ticket, 0, (size_t)(c->ld / 512 + 2) * sizeof(unsigned)));
        r.upart_cap = need;
    }
    if (k > 0 && c->fused()) {            // BiCG loop: reduce-scatter fused into K1T (NEXT-1)
        GemvTPub pub;
        pub.P = c->P;
        const int64_t par = (k & 1) * (int64_t)r.L.P * r.L.chunk;
        for (int g = 0; g < c->P; ++g) {
            pub.dst[g] = r.pp.G_v[g] + par + (int64_t)r.rank * r.L.chunk;
            pub.f_peer[g] = r.pp.flags[g] + kPhaseV * kMaxRanks + r.rank;
        }
        pub.epoch = ebase + (unsigned long long)k;
        pub.ticket = r.col_ticket + c->ld / 512 + 1;
        r.launches += launch_gemv_t(r.A, c->ld, r.m, c->n, x_loc, rc, r.upart, r.col_ticket, r.U, r.L, done,
                                    shape, r.stream, &pub);
        return nullptr;                   // the consumer sums the P slots (k_bicg_update)
    }
    r.launches += launch_gemv_t(r.A, c->ld, r.m, c->n, x_loc, rc, r.upart, r.col_ticket, r.U, r.L, done,
                                shape, r.stream);
    if (c->P == 1) return r.U;
    reduce_scatter_u(c, r);
    return r.qt_loc;
}

GemvConfig gemv_config(const ks_ctx* c, const Rank& r) {
    GemvConfig g = choose_gemv(r.m, c->ld, r.num_sms, (int)c->opt.gemv_rows, (int)c->opt.gemv_split,
                               (int)c->opt.gemv_kernel);
    g.unroll = (int)c->opt.gemv_unroll;
    const int64_t tiles = (r.m + g.rows - 1) / g.rows;
    const int64_t cap = (r.scr.qpart_cap - 2 * tiles - 64) / std::max<int64_t>(1, tiles * g.rows);
    if (g.splits > cap) g.splits = (int)std::max<int64_t>(1, cap);
    return g;
}

}  // namespace ks

void ks_ctx::for_each_rank(const std::function<void(ks::Rank&)>& fn) {
    bool flushed = false;
    int prev = 0;
    for (auto& r : ranks)                 // nothing of this context is in flight between calls
        if (!r.retired.empty()) {
            if (!flushed && cudaGetDevice(&prev) != cudaSuccess) prev = -1;
            flushed = true;
            if (cudaSetDevice(r.dev) == cudaSuccess) ks::flush_retired(r);
        }
    if (flushed && prev >= 0) cudaSetDevice(prev);   // the caller's current device
    if (ranks.size() == 1) {
        ks::cuda_check(cudaSetDevice(ranks[0].dev), "cudaSetDevice");
        cudaGetLastError();   // drop a stale, already-reported non-sticky error (e.g. an OOM)
        fn(ranks[0]);
        return;
    }
    std::vector<std::thread> th;
    std::exception_ptr first;
    std::mutex mu;
    hbar->reset((int)ranks.size());
    for (auto& r : ranks) {
        th.emplace_back([&, rp = &r] {
            try {
                ks::cuda_check(cudaSetDevice(rp->dev), "cudaSetDevice");
                cudaGetLastError();
                fn(*rp);
            } catch (...) {
                {
                    std::lock_guard<std::mutex> g(mu);
                    if (!first) first = std::current_exception();
                }
                hbar->abort();   // peers waiting in a host collective fail instead of blocking
            }
        });
    }
    for (auto& t : th) t.join();
    if (first) std::rethrow_exception(first);
}

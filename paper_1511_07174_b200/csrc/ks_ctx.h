// L3: the opaque context -- "encapsulation of data and distribution and
// communication in opaque objects".  1-D row-block partition of A
// over P GPUs, one Rank per local GPU.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "ks_internal.h"

namespace ks {

struct KsError : std::runtime_error {
    ks_status code;
    KsError(ks_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
void nccl_check(ncclResult_t r, const char* what);
#define KS_CUDA(x) ::ks::cuda_check((x), #x)
#define KS_NCCL(x) ::ks::nccl_check((x), #x)

// Device allocation of library buffers (ks_alloc.cpp): plain cudaMalloc/cudaFree, or
// with KS_GUARD=1 4 KiB canary zones around every buffer for out-of-bounds-write
// detection.  guard_check counts corrupted zones on the given devices (-1: off).
void* dev_alloc(size_t bytes);
void dev_free(void* p);
int64_t guard_check(const std::vector<int>& devs);
template <class T>
inline void dev_alloc_t(T** p, size_t count) { *p = static_cast<T*>(dev_alloc(count * sizeof(T))); }

// Rendezvous of the worker threads of one process (for_each_rank) for the host-driven
// collectives of a context whose ranks share devices (no NCCL communicator: NCCL
// rejects two ranks on one GPU).  abort() releases every waiter with an error when a
// rank failed, so the others cannot block on it.
struct HostBarrier {
    std::mutex mu;
    std::condition_variable cv;
    int n = 0, count = 0;
    unsigned long long gen = 0;
    bool aborted = false;
    void reset(int parties);
    void wait();     // throws KsError(KS_ENCCL) after abort()
    void abort();
};

struct Rank {
    int rank = 0, dev = 0, num_sms = 148;
    int dev_share = 1;          // ranks of this context on the same GPU
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    ncclComm_t comm = nullptr;
    bool own_comm = false;
    Layout L{};
    int64_t m = 0, row0 = 0;

    // device memory (owned)
    double* A = nullptr;        // m x ld
    double* b_full = nullptr;   // ld
    double* x_loc = nullptr;    // m (padded)
    double* p_full = nullptr;   // ld
    double* s_full = nullptr;   // ld
    double* v_full = nullptr;   // ld
    double* q_loc = nullptr;    // m
    double* rhat_loc = nullptr; // m
    double* pt_loc = nullptr;   // m (BiCG)
    double* U = nullptr;        // P * chunk: K1T output (chunk layout)
    double* qt_loc = nullptr;   // chunk: reduce-scattered qt (P > 1)
    // GMRES(m) workspace (lazily sized by the restart length)
    double* gmV = nullptr;
    int64_t gm_ldv = 0;
    int gm_m = 0;
    double* gmH = nullptr;      // (m+1) x m + cs, sn (m) + g (m+1)
    double* gm_hx = nullptr;    // P x kMaxBasis
    GmresState* gm_state = nullptr;
    double* upart = nullptr;    // K1T row-chunk partials (lazily sized)
    unsigned* col_ticket = nullptr;
    int64_t upart_cap = 0;
    // exchange buffers, one allocation (one CUDA IPC handle): G_r, G_v (2 parities
    // x P chunks each), S (2 parities x P x kScalSlot), epoch flags
    double* xbuf = nullptr;
    size_t xbuf_bytes = 0;
    double* G_r = nullptr;      // 2 * P * chunk
    double* G_v = nullptr;      // 2 * P * chunk
    double* S = nullptr;        // 2 * P * kScalSlot
    unsigned long long* flags = nullptr;   // [kNumPhases][kMaxRanks]
    double* X = nullptr;        // ld elements: contiguous full x (end-of-solve gather)
    double *MR = nullptr, *MS = nullptr, *MX = nullptr, *MV = nullptr;   // multi-RHS exchange regions (P > 1)
    uint64_t* llx = nullptr;    // tiny kernels' LL slots in the exchange allocation (P > 1, ld <= 1024)
    uint64_t* llg = nullptr;    // persistent kernels' LL handover region (P > 1, ll_words(ld) words)
    int ll_on = 0;              // KS_OPT_LL_XCHG (effective with the fused exchange)
    const double* x0_full = nullptr;   // the current solve's full x0 on the device (s_full) or NULL
    uint64_t* llpeer[kMaxRanks] = {};
    MultiPeer mpeer{};
    PeerPtrs pp{};
    bool peer_ok = false;       // every rank's exchange buffers are load/store reachable
    unsigned jitter = 0;        // KS_OPT_JITTER seed (also in st->jitter)
    std::vector<void*> ipc_opened;
    unsigned long long epoch_next = 1;
    DevState* st = nullptr;
    double* hist = nullptr;
    int64_t hist_alloc = 0;
    Scratch scr{};
    double* table_tmp = nullptr;
    uint64_t* ll = nullptr;     // LL exchange slots of the tiny kernels (4 * ld words, lazily)
    // multi-RHS CG workspace (lazily sized by the kernel width K and the history cap)
    double *mX = nullptr, *mR = nullptr, *mQ = nullptr, *mP = nullptr, *mhist = nullptr;
    double *mRh = nullptr, *mT = nullptr, *mS = nullptr;   // multi-RHS BiCGSTAB
    MultiState* mstate = nullptr;
    int mK = 0;
    int64_t mhist_cap = 0;

    // host
    int* h_done = nullptr;      // pinned, 2 slots
    double* h_hist = nullptr;   // pinned staging of short histories (kHistStage entries)
    DevState* h_state = nullptr; // pinned
    std::vector<unsigned char> loaded;  // per local row
    int64_t loaded_count = 0;

    // events
    cudaEvent_t ev_poll[2]{};
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
    cudaEvent_t ev_coll[2]{};           // host-driven collectives (shared-device contexts)
    double* rs_stage = nullptr;         // P * chunk: host-driven reduce-scatter staging
    std::vector<void*> retired;         // replaced during a call, freed before the next (retire)
    std::vector<cudaEvent_t> ev_gemv;   // profiling pairs

    // CUDA-graph replay of one poll batch (KS_OPT_USE_GRAPHS)
    long long* kdev = nullptr;            // iteration base read by the captured kernels
    struct GraphCache {
        cudaGraphExec_t exec = nullptr;
        int kind = -1;
        int64_t B = 0, launches = 0;
        const void* hist = nullptr;
        int variant = 0, rows = 0, splits = 0, fused = 0;
    } graphs[2];

    bool bar_zeroed = false;    // the start kernel zeroed the grid-barrier counter
    std::map<long long, int> grid_memo;   // launch geometry (occupancy queries) per kernel kind
    int64_t launches = 0;
    int64_t gemv_launches = 0;
    double gemv_seconds = 0.0;

    VecArgs vargs(bool fused) const;
    VecArgsT<float> vargs_f32(bool fused) const;   // FP32 contexts: buffers hold floats
};

struct Options {
    int64_t true_residual = 1;
    int64_t profile_gemv = 0;
    int64_t poll_batch = 0;   // 0 = auto: whole solve per persistent launch, else 16
    int64_t gemv_rows = 0;
    int64_t gemv_split = 0;
    int64_t gemv_kernel = 0;
    int64_t use_graphs = 0;
    int64_t fused_comm = 1;   // fused NVLink peer-store collectives when available
    int64_t persistent = 2;   // 0 off, 1 on, 2 auto: persistent cooperative kernels
    int64_t gemv_unroll = 0;  // tuning: K1 LDG unroll (0 = default)
    int64_t persist_grid = 0; // tuning: persistent CTAs (0 = auto)
    int64_t gemvt_shape = 204; // tuning: K1T vectors/thread/row * 100 + rows in flight
    int64_t small = 2;        // 0 off, 1 on, 2 auto: small-n shared-memory kernels (P == 1)
    int64_t join_timeout_ms = 120000;   // fused P > 1: solve-start rendezvous bound
    int64_t tiny = 1;         // 1 auto, 0 off: register-resident kernels (P == 1, n <= 1024)
    int64_t jitter = 0;       // race-detection delays at sync points (seed; 0 off)
    int64_t ll_xchg = 1;      // LL handovers in the persistent kernels (P > 1, fused)
};

}  // namespace ks

struct ks_ctx {
    int64_t n = 0, ld = 0;
    ks_dtype dtype = KS_FLOAT64;
    size_t esz = sizeof(double);   // bytes per element of A and the device vectors
    int P = 1;               // global number of ranks
    bool multiprocess = false;
    // some ranks share a GPU (ks_create_on with a repeated device): no NCCL
    // communicator, no fused exchange; the collectives are host-driven peer copies
    bool shared_dev = false;
    std::unique_ptr<ks::HostBarrier> hbar = std::make_unique<ks::HostBarrier>();
    std::vector<ks::Rank> ranks;   // local ranks (1 in multi-process mode)
    ks::Options opt;
    bool poisoned = false;
    std::string last_error;

    // Runs fn(rank) on every local rank: one worker thread per GPU when there is
    // more than one.  Exceptions are collected; the first is rethrown.
    void for_each_rank(const std::function<void(ks::Rank&)>& fn);
    bool writes_host(const ks::Rank& r) const { return multiprocess || r.rank == 0; }
    bool fused() const { return P > 1 && opt.fused_comm && !ranks.empty() && ranks[0].peer_ok; }
    // persistent kernels need P == 1 or the fused exchange (no NCCL inside a kernel)
    bool persistent() const {
        if (opt.persistent == 0) return false;
        if (!(P == 1 || fused())) return false;
        return opt.persistent == 1 || n <= kPersistAutoMaxN;
    }
    static constexpr int64_t kPersistAutoMaxN = 1LL << 62;   // tuned from measurements
    // small-n kernels on when a full vector is <= 32 KiB (FP64 n <= 4096, FP32 n <= 8192):
    // the crossover measured in profiles/r01_small_path.json
    static constexpr int64_t kSmallAutoMaxBytes = 32768;
};

namespace ks {
constexpr int64_t kHistStage = 4096;   // histories up to this long are staged: one sync per solve
void rank_alloc(ks_ctx* c, Rank& r);
void rank_free(Rank& r);
void retire(Rank& r, void* p);     // free at the start of the next call (no cudaFree inside a call)
void flush_retired(Rank& r);
void setup_peers(ks_ctx* c);   // peer access / CUDA IPC of the exchange buffers
void allgather(const ks_ctx* c, Rank& r, double* G, int64_t count_per_rank);   // dtype-aware
void host_launch_once(const ks_ctx* c, Rank& r, const std::function<void()>& launch);   // shared GPU
void copy_chunks_to(const ks_ctx* c, Rank& r, const double* G, double* dst, cudaMemcpyKind kind);
int64_t run_f32(ks_ctx* c, Rank& r, int bicgstab, const double* b, double tol, int64_t maxit,
                double* x, double* hist, int64_t hist_cap, ks_report* rep);
int64_t run_cg(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol, int64_t maxit,
               double* x, double* hist, int64_t hist_cap, ks_report* rep);
int64_t run_bicgstab(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol,
                     int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep);
int64_t run_gmres(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol, int restart,
                  int64_t maxit, double* x, double* hist, int64_t hist_cap, ks_report* rep);
int64_t run_bicg(ks_ctx* c, Rank& r, const double* b, const double* x0, double tol, int64_t maxit,
                 double* x, double* hist, int64_t hist_cap, ks_report* rep);
int64_t run_multi(ks_ctx* c, Rank& r, int bicgstab, int nrhs, const double* B, const double* X0, double tol,
                  int64_t maxit, double* X, double* hist, int64_t hist_cap, ks_report* reps);
// K1T into r.U (chunk layout); for P > 1 reduce-scattered into r.qt_loc.  Returns the
// pointer holding this rank's rows of A^T x.
// k > 0 with the fused exchange (BiCG loop): the reduce-scatter is fused into K1T
// (slots G_v[parity k][rank g's chunk], flag kPhaseV with epoch ebase + k); returns nullptr.
const double* gemv_t(ks_ctx* c, Rank& r, const double* x_loc, const int* done, long long k = 0,
                     unsigned long long ebase = 0);
GemvConfig gemv_config(const ks_ctx* c, const Rank& r);
}  // namespace ks

// Device allocation for every library buffer, with optional guard zones.
//
// compute-sanitizer is not available on the GPU pool, so the library carries its
// own out-of-bounds-write detector: with KS_GUARD=1 in the environment when the
// library is loaded, every buffer allocated here gets a 4 KiB canary zone before
// and after it (filled with 0xA5).  A zone that no longer holds the pattern means
// some kernel wrote outside a buffer.  Zones are verified when a buffer is freed
// and on demand (ks_check_guards); without KS_GUARD the functions are plain
// cudaMalloc / cudaFree.  The exchange buffer (CUDA IPC: peers address it from the
// allocation base) is never guarded.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "ks_ctx.h"

namespace ks {

namespace {

constexpr size_t kGuard = 4096;
constexpr unsigned char kPattern = 0xA5;

struct Entry {
    char* base;
    size_t bytes;    // the caller's exact size
    size_t padded;   // rounded up to 256 bytes (the trailing zone starts at bytes, not here)
    int dev;
};

bool guards_on() {
    static const bool on = [] {
        const char* v = std::getenv("KS_GUARD");
        return v && v[0] && v[0] != '0';
    }();
    return on;
}

std::mutex g_mu;
std::unordered_map<void*, Entry>& registry() {
    static std::unordered_map<void*, Entry> m;
    return m;
}
int64_t g_violations = 0;   // corrupted zones found at free time

// number of corrupted zones of one entry (synchronous; its device must be current)
int zone_errors(const Entry& e) {
    std::vector<unsigned char> h(kGuard);
    int bad = 0;
    // leading zone, then the trailing zone from the exact end of the buffer: the
    // alignment padding [bytes, padded) is canary too (overruns of up to
    // 255 bytes into the padding used to go unseen)
    const size_t tail = e.padded - e.bytes + kGuard;
    std::vector<unsigned char> t(tail);
    if (cudaMemcpy(h.data(), e.base, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    for (unsigned char b : h)
        if (b != kPattern) { ++bad; break; }
    if (cudaMemcpy(t.data(), e.base + kGuard + e.bytes, tail, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    for (unsigned char b : t)
        if (b != kPattern) { ++bad; break; }
    return bad;
}

}  // namespace

void* dev_alloc(size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    if (!guards_on()) {
        void* p = nullptr;
        KS_CUDA(cudaMalloc(&p, bytes));
        return p;
    }
    const size_t padded = (bytes + 255) / 256 * 256;   // keep the user pointer 256-byte aligned
    char* base = nullptr;
    KS_CUDA(cudaMalloc(reinterpret_cast<void**>(&base), padded + 2 * kGuard));
    KS_CUDA(cudaMemset(base, kPattern, kGuard));
    KS_CUDA(cudaMemset(base + kGuard + bytes, kPattern, padded - bytes + kGuard));
    int dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    void* user = base + kGuard;
    // detector self-test (KS_GUARD_SELFTEST=1): one byte past the end of every buffer
    static const bool selftest = [] {
        const char* v = std::getenv("KS_GUARD_SELFTEST");
        return v && v[0] == '1';
    }();
    if (selftest) KS_CUDA(cudaMemset(base + kGuard + bytes, 0, 1));   // the first byte past the buffer
    std::lock_guard<std::mutex> lk(g_mu);
    registry()[user] = Entry{base, bytes, padded, dev};
    return user;
}

void dev_free(void* p) {
    if (!p) return;
    if (!guards_on()) {
        cudaFree(p);
        return;
    }
    Entry e{};
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = registry().find(p);
        if (it == registry().end()) {
            cudaFree(p);
            return;
        }
        e = it->second;
        registry().erase(it);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(e.dev);
    cudaDeviceSynchronize();
    const int bad = zone_errors(e);
    cudaFree(e.base);
    cudaSetDevice(cur);
    std::lock_guard<std::mutex> lk(g_mu);
    g_violations += bad;
}

int64_t guard_check(const std::vector<int>& devs) {
    if (!guards_on()) return -1;
    std::vector<Entry> live;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto& kv : registry())
            for (int d : devs)
                if (kv.second.dev == d) live.push_back(kv.second);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    int64_t bad = 0;
    for (const Entry& e : live) {
        cudaSetDevice(e.dev);
        cudaDeviceSynchronize();
        bad += zone_errors(e);
    }
    cudaSetDevice(cur);
    std::lock_guard<std::mutex> lk(g_mu);
    return bad + g_violations;
}

}  // namespace ks

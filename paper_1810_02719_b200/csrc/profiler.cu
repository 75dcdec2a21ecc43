#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"
#include "profiler.h"

namespace smg {

namespace {
std::atomic<int64_t> g_launches{0};
}

int count_launch() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return 0;
}

int64_t launch_count() { return g_launches.load(); }

// cudaFuncAttributeMaxDynamicSharedMemorySize is per device: cache the largest
// value set per (kernel, device) under a lock, so contexts on several devices
// (or host threads) each get their own call
void ensure_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> have;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    int& cur = have[{func, dev}];
    if (bytes > cur) {
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cur = bytes;
    }
}

Profiler*& active_profiler() {
    thread_local Profiler* p = nullptr;
    return p;
}

void Profiler::clear() {
    std::lock_guard<std::mutex> lock(mu_);
    for (cudaEvent_t e : pool_) cudaEventDestroy(e);
    pool_.clear();
    spans_.clear();
}

int Profiler::new_event(cudaStream_t st) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    cudaEventRecord(e, st);
    pool_.push_back(e);
    return (int)pool_.size() - 1;
}

int Profiler::begin(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) return -1;  // not inside graph capture
    std::lock_guard<std::mutex> lock(mu_);
    return new_event(st);
}

void Profiler::end(const char* stage, int token, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu_);
    const int b = new_event(st);
    if (b >= 0) spans_[stage].push_back({token, b});
}

bool Profiler::read(const std::string& stage, int64_t* launches, double* total_ms) {
    std::lock_guard<std::mutex> lock(mu_);
    auto it = spans_.find(stage);
    if (it == spans_.end()) {
        *launches = 0;
        *total_ms = 0.0;
        return true;
    }
    double t = 0.0;
    for (auto& s : it->second) {
        cudaEventSynchronize(pool_[s.second]);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pool_[s.first], pool_[s.second]);
        t += ms;
    }
    *launches = (int64_t)it->second.size();
    *total_ms = t;
    return true;
}

}  // namespace smg

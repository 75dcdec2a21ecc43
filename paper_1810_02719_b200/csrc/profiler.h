// Per-stage device timing of the library's kernels (diagnostics API
// smg_profile_*).  When a context enables it, every instrumented stage records
// a CUDA event pair on the launching stream; totals are resolved on read.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace smg {

class Profiler {
public:
    ~Profiler() { clear(); }
    void clear();
    int begin(cudaStream_t st);
    void end(const char* stage, int token, cudaStream_t st);
    // sums; synchronises on the recorded events
    bool read(const std::string& stage, int64_t* launches, double* total_ms);

private:
    std::vector<cudaEvent_t> pool_;
    std::map<std::string, std::vector<std::pair<int, int>>> spans_;
    std::mutex mu_;  // chain groups issue from their own host threads
    int new_event(cudaStream_t st);
};

// The active profiler for the calling thread (set for the duration of an API call).
Profiler*& active_profiler();

struct ProfScope {
    const char* stage;
    cudaStream_t st;
    int token = -1;
    ProfScope(const char* s, cudaStream_t stream) : stage(s), st(stream) {
        if (Profiler* p = active_profiler()) token = p->begin(st);
    }
    ~ProfScope() {
        if (token >= 0)
            if (Profiler* p = active_profiler()) p->end(stage, token, st);
    }
};

}  // namespace smg

// Opaque handle definitions shared by the C-ABI translation units.
#pragma once

#include <string>

#include <vector>

#include "../../include/specmesh_gpu.h"
#include "doi.h"
#include "engine.h"
#include "profiler.h"

struct smg_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string error;
    bool profiling = false;
    smg::Profiler prof;
    smg_run_info info{};  // last chain call (smg_last_run_info)
    // DOI step log (smg_doi_trace_*): chain position, c the step ran with, residual
    bool doi_trace = false;
    std::vector<int> trace_pos, trace_c;
    std::vector<double> trace_r;
    void log_doi(const smg::DoiLoop& loop, int pos, int steps) {
        if (!doi_trace) return;
        std::vector<int> c;
        std::vector<double> r;
        loop.read_trace(steps, c, r);
        for (size_t i = 0; i < c.size(); ++i) {
            trace_pos.push_back(pos);
            trace_c.push_back(c[i]);
            trace_r.push_back(r[i]);
        }
    }
};

struct smg_operator {
    smg::TileSet ts;
    smg::FactorSet fs;
    int n = 0, z = 1;
    double delta = 0.0;
};

namespace smg {
// Runs f() for an API call: device selection, profiler activation, exception
// to status translation (exceptions never cross the C ABI).
template <class F>
int guarded_call(smg_context* ctx, F&& f) {
    if (!ctx) return 2;
    struct Activate {
        explicit Activate(smg_context* c) { active_profiler() = c->profiling ? &c->prof : nullptr; }
        ~Activate() { active_profiler() = nullptr; }
    } act(ctx);
    try {
        SMG_CUDA(cudaSetDevice(ctx->device));
        f();
        ctx->error.clear();
        return 0;
    } catch (const Failure& e) {
        ctx->error = e.what();
        return (e.code == 2 || e.code == 4) ? e.code : 3;
    } catch (const std::exception& e) {
        ctx->error = e.what();
        return 3;
    }
}
}  // namespace smg

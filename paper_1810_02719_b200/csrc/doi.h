// K10: dynamic_oi (spectral.hpp:244-287) as a CUDA graph with a conditional
// WHILE node.  One captured body = one DOI iteration:
//   solve (R^z U, device-side c) -> CholeskyQR2 with the rank test ->
//   projection residual e and ||e|| -> decide (grow / shrink / stop, sets the
//   graph condition) -> append e/||e|| as column c when growing.
// The loop runs entirely on the device; the host launches one graph per block
// and reads the final DoiState once.
#pragma once

#include "engine.h"

namespace smg {

struct DoiParams {
    int c_min = 1, c_max = 1, t_max = 0, power = 2;
    double eps_low = 0.0, eps_high = 0.0;
};

class DoiLoop {
public:
    DoiLoop() = default;
    DoiLoop(const DoiLoop&) = delete;
    DoiLoop& operator=(const DoiLoop&) = delete;
    ~DoiLoop();
    // capture the loop for tiles of `ts` with workspace `ws` (batch 1)
    void build(const TileSet& ts, Workspace& ws, const DoiParams& prm, int64_t strideF, cudaStream_t st);
    // run dynamic_oi on the tile: factor slabs (device), coords X (n x 3 row-major,
    // device), bbox scale, permutation (device or null), initial basis in ws.U
    // with c_init columns.  Returns the final state; ws.U holds u (before the
    // final orthonormalize of a pending append, which the caller performs).
    DoiState run(const double* Ff, const double* Fb, const int32_t* perm, const double* X, double bbox, int c_init);
    // per-step (c, residual) of the last run(), r.t entries
    void read_trace(int steps, std::vector<int>& c, std::vector<double>& r) const;

private:
    // one DOI iteration (solve -> CholeskyQR2 -> residual -> decide -> append)
    void issue(cudaStream_t cs, cudaGraphConditionalHandle h, int use_handle);
    bool nograph_ = false;  // SMG_DOI_NOGRAPH=1: host-driven loop (profilers see every kernel)
    const TileSet* ts_ = nullptr;
    Workspace* ws_ = nullptr;
    DoiParams prm_;
    cudaStream_t st_ = nullptr;
    int64_t strideF_ = 0;
    DBuf<double> Ff_, Fb_, X_;
    DBuf<int32_t> P_;
    DBuf<DoiState> state_;
    DBuf<int> trace_c_;
    DBuf<double> trace_r_;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t exec_ = nullptr;
};

}  // namespace smg

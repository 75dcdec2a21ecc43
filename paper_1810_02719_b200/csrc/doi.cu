#include <cstdlib>

#include "doi.h"

namespace smg {

DoiLoop::~DoiLoop() {
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
}

void DoiLoop::issue(cudaStream_t cs, cudaGraphConditionalHandle h, int use_handle) {
    const TileSet& ts = *ts_;
    Workspace& ws = *ws_;
    StepCtx cx{cs, &ts};
    DoiState* state = state_.get();
    const int* dimC = &state->c;
    SolveParams p;
    p.n = ts.n;
    p.Kb = ts.Kb;
    p.z = prm_.power;
    p.c_cap = ws.ccap;
    p.batch = 1;
    p.Ffwd = Ff_.get();
    p.Fbwd = Fb_.get();
    p.strideF = strideF_;
    p.perm = ts.use_perm ? P_.get() : nullptr;
    p.in = ws.U.get();
    p.ldin = ws.ld;
    p.strideIn = ws.mstride();
    p.tmp = ws.T.get();
    p.ldt = ws.ld;
    p.strideT = ws.mstride();
    p.out = ws.V.get();
    p.ldout = ws.ld;
    p.strideOut = ws.mstride();
    p.dimC = dimC;
    p.dimStride = 1;
    solve_block_tridiag(p, ts.W, cs);
    // Two full CholeskyQR passes per DOI step by default.  SMG_DOI_ADAPTIVE=1 lets the probe skip
    // the second pass (C4 485 -> 455 ms), but a DOI trajectory amplifies any change of rounding
    // by ~1/r per growth step: on the reference-generated fixture ref_doi.npz
    // the first block's last decision has a 2.4 % margin and flips (c = 51 instead of 50).
    static const double skip_tol = (std::getenv("SMG_DOI_ADAPTIVE") && std::atoi(std::getenv("SMG_DOI_ADAPTIVE")) == 1)
                                       ? (std::getenv("SMG_ORTH_SKIP_TOL") ? std::atof(std::getenv("SMG_ORTH_SKIP_TOL")) : 1e-13)
                                       : 0.0;
    orth_batch(cx, ws, ws.V.get(), ws.U.get(), ws.ccap, dimC, true, -1, 2, skip_tol);
    project_batch(cx, ws, ws.U.get(), ws.ccap, dimC, X_.get(), 0, nullptr, 0);
    doi_decide(state, 1, ws.stats.get(), 4, h, use_handle, ws.status.get(), cs, trace_c_.get(), trace_r_.get());
    doi_append(state, ws.U.get(), ws.ld, ws.mstride(), ws.e.get(), ws.npad, ts.n, 1, cs);
}

void DoiLoop::build(const TileSet& ts, Workspace& ws, const DoiParams& prm, int64_t strideF, cudaStream_t st) {
    ts_ = &ts;
    ws_ = &ws;
    prm_ = prm;
    st_ = st;
    strideF_ = strideF;
    Ff_.alloc(strideF, st);
    Fb_.alloc(strideF, st);
    X_.alloc((size_t)ts.n * 3, st);
    if (ts.use_perm) P_.alloc(ts.n, st);
    state_.alloc(1, st);
    trace_c_.alloc(std::max(prm.t_max, 1), st);
    trace_r_.alloc(std::max(prm.t_max, 1), st);
    SMG_CUDA(cudaStreamSynchronize(st));

    SMG_CUDA(cudaGraphCreate(&graph_, 0));
    cudaGraphConditionalHandle h;
    SMG_CUDA(cudaGraphConditionalHandleCreate(&h, graph_, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SMG_CUDA(cudaGraphAddNode(&node, graph_, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];

    nograph_ = std::getenv("SMG_DOI_NOGRAPH") != nullptr;
    cudaStream_t cs;
    SMG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    SMG_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    issue(cs, h, 1);
    cudaGraph_t captured;
    SMG_CUDA(cudaStreamEndCapture(cs, &captured));
    SMG_CUDA(cudaStreamDestroy(cs));
    SMG_CUDA(cudaGraphInstantiate(&exec_, graph_, 0));
}

DoiState DoiLoop::run(const double* Ff, const double* Fb, const int32_t* perm, const double* X, double bbox,
                      int c_init) {
    SMG_CUDA(cudaMemcpyAsync(Ff_.get(), Ff, strideF_ * 8, cudaMemcpyDeviceToDevice, st_));
    SMG_CUDA(cudaMemcpyAsync(Fb_.get(), Fb, strideF_ * 8, cudaMemcpyDeviceToDevice, st_));
    SMG_CUDA(cudaMemcpyAsync(X_.get(), X, (size_t)ts_->n * 3 * 8, cudaMemcpyDeviceToDevice, st_));
    if (ts_->use_perm && perm)
        SMG_CUDA(cudaMemcpyAsync(P_.get(), perm, (size_t)ts_->n * 4, cudaMemcpyDeviceToDevice, st_));
    DoiState s{};
    s.c = c_init;
    s.t = 0;
    s.active = prm_.t_max > 0 ? 1 : 0;
    s.c_min = prm_.c_min;
    s.c_max = prm_.c_max;
    s.t_max = prm_.t_max;
    s.eps_low = prm_.eps_low;
    s.eps_high = prm_.eps_high;
    s.scale = bbox == 0.0 ? 1.0 : bbox;  // spectral.hpp:253-254
    SMG_CUDA(cudaMemcpyAsync(state_.get(), &s, sizeof(s), cudaMemcpyHostToDevice, st_));
    if (prm_.t_max > 0 && !nograph_) SMG_CUDA(cudaGraphLaunch(exec_, st_));
    if (prm_.t_max > 0 && nograph_) {
        DoiState h{};
        do {
            issue(st_, cudaGraphConditionalHandle{}, 0);
            SMG_CUDA(cudaMemcpyAsync(&h, state_.get(), sizeof(h), cudaMemcpyDeviceToHost, st_));
            SMG_CUDA(cudaStreamSynchronize(st_));
        } while (h.active);
    }
    DoiState r{};
    SMG_CUDA(cudaMemcpyAsync(&r, state_.get(), sizeof(r), cudaMemcpyDeviceToHost, st_));
    SMG_CUDA(cudaStreamSynchronize(st_));
    return r;
}

void DoiLoop::read_trace(int steps, std::vector<int>& c, std::vector<double>& r) const {
    steps = std::max(0, std::min(steps, prm_.t_max));
    c.resize(steps);
    r.resize(steps);
    if (!steps) return;
    SMG_CUDA(cudaMemcpyAsync(c.data(), trace_c_.get(), (size_t)steps * sizeof(int), cudaMemcpyDeviceToHost, st_));
    SMG_CUDA(cudaMemcpyAsync(r.data(), trace_r_.get(), (size_t)steps * sizeof(double), cudaMemcpyDeviceToHost, st_));
    SMG_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace smg

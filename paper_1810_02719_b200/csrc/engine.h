// Host-side engine of libspecmesh_b200: device buffers, assembled tile sets,
// factor sets, per-batch workspaces and the chain steps built on the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "chain.h"
#include "kernels.h"

namespace smg {

// Library error carrying the C-ABI status (2 InvalidArgument, 3 Error).
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }
inline void require(bool cond, const std::string& msg) {
    if (!cond) fail(2, msg);
}
void cuda_check(cudaError_t e, const char* what);
#define SMG_CUDA(x) ::smg::cuda_check((x), #x)

template <class T>
class DBuf {
public:
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), st_(o.st_) { o.p_ = nullptr; o.n_ = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { reset(); p_ = o.p_; n_ = o.n_; st_ = o.st_; o.p_ = nullptr; o.n_ = 0; }
        return *this;
    }
    ~DBuf() { reset(); }
    void alloc(size_t n, cudaStream_t st) {
        reset();
        st_ = st;
        n_ = n;
        if (n) SMG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), st));
    }
    void zero() {
        if (n_) SMG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), st_));
    }
    void upload(const T* h, size_t n, cudaStream_t st) {
        alloc(n, st);
        if (n) SMG_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, st_));
    }
    void upload(const std::vector<T>& v, cudaStream_t st) {
        upload(v.data(), v.size(), st);
    }
    void reset() {
        if (p_) cudaFreeAsync(p_, st_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    // free on another stream later (objects that outlive the allocating stream)
    void rebind(cudaStream_t st) { st_ = st; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t st_ = 0;
};

template <class T>
std::vector<T> download(const T* d, size_t n, cudaStream_t st) {
    std::vector<T> h(n);
    if (n) SMG_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    return h;
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ------------------------------------------------------------ tiles
struct TileSet {
    int ntiles = 0, n = 0;
    int W = 0, Kb = 0, npad = 0;
    int cpl = 16;  // bound on a row's couplings into the previous block (factor smem stride)
    bool use_perm = false;
    // orderings from the connectivity alone (codec: the decoder has no coordinates,
    // so encoder and decoder must factor identically)
    bool topology_ordering = false;
    int ordering = 0;  // chosen factorisation order: 0 natural, 1 geometric (axis sort), 2 RCM
    int weighting = -1;  // smg_weighting of the assembled tiles (-1: external CSR)
    int64_t total_nnz = 0;
    DBuf<TileRef> refs;
    DBuf<int32_t> nnz, rowptr, cols, perm, bw, blockw;
    DBuf<int64_t> off, detail;
    DBuf<double> vals, trace, delta, shift0, X, bbox;
    DBuf<int> status;
    std::vector<int> status_h;
    std::vector<int64_t> detail_h;

    // assembly + ordering + shifts + coordinate gather; syncs twice (nnz, W)
    void build(const std::vector<TileRef>& tiles, int n, int weighting, double shift_scale, cudaStream_t st);
    // one tile from a host CSR (operator primitives); delta given explicitly
    void build_from_csr(int n, const int32_t* rowptr, const int32_t* cols, const double* vals, double delta,
                        cudaStream_t st);
    void finish_build(double shift_scale, const std::vector<double>* explicit_delta, cudaStream_t st,
                      const double* coords = nullptr);
    const int32_t* perm_of(int tile) const { return use_perm ? perm.get() + (int64_t)tile * n : nullptr; }
    void rebind(cudaStream_t st) {
        refs.rebind(st), nnz.rebind(st), rowptr.rebind(st), cols.rebind(st), perm.rebind(st), bw.rebind(st);
        blockw.rebind(st), off.rebind(st), detail.rebind(st), vals.rebind(st), trace.rebind(st);
        delta.rebind(st), shift0.rebind(st), X.rebind(st), bbox.rebind(st), status.rebind(st);
    }
};

struct FactorSet {
    int first = 0, count = 0;
    int64_t strideF = 0;
    DBuf<double> fwd, bwd;
    DBuf<int> status;
    void factor(const TileSet& ts, int first_tile, int count, const double* shift, cudaStream_t st,
                int* status_out = nullptr);
    const double* f(int tile) const { return fwd.get() + (int64_t)(tile - first) * strideF; }
    const double* b(int tile) const { return bwd.get() + (int64_t)(tile - first) * strideF; }
    void rebind(cudaStream_t st) { fwd.rebind(st), bwd.rebind(st), status.rebind(st); }
};

// ------------------------------------------------------------ workspace
struct Workspace {
    int B = 0, n = 0, npad = 0, ld = 0, ccap = 0;
    int splits = 1;
    DBuf<double> U, V, T, R, G, Gws, Bm, work, rdiag, vnorm, rpart, coeff, sign, e, ppart, ppart2, stats;
    DBuf<double> probe_part, probe_est;  // orthonormality probe of the adaptive CholeskyQR2 (probe.cu)
    DBuf<int> counters;
    DBuf<int> status, errpos, scratch_status, skip, skip2, rneed;
    DBuf<unsigned long long> nmax;
    DBuf<int64_t> detail;
    DBuf<double> H, Hst, Vj, theta, theta_s, Wm, ritz_part, ritz;
    bool proj_ready = false;  // ppart holds the last orth_batch's projection partials (host-side flag)
    void init(int B, int n, int npad, int ccap, cudaStream_t st);
    int64_t mstride() const { return (int64_t)npad * ld; }
};

struct StepCtx {
    cudaStream_t st;
    const TileSet* ts;
};

// Batched building blocks.  `tile0`/`tstride`: tile index of batch entry b is
// tile0 + b * tstride (factor and permutation lookup).
void solve_batch(const StepCtx& cx, Workspace& ws, const FactorSet& fs, int tile0, int tstride, const double* in,
                 double* out, int c, const int* dimC, int z, bool once);
// CholeskyQR2: out = orth(in); sticky per-chain status, error position `pos`.
// skip_tol > 0: adaptive -- a chain whose pass-1 factor Q1 is orthonormal to
// skip_tol (max |Q1^T Q1 - I|, from the pass-2 Gram) keeps Q1 (no second
// Cholesky, no second triangular product).  projX (adaptive path): the
// triangular products also write the projection's partial records for these
// coordinates, and the next project_batch on this workspace skips its pass 1.
void orth_batch(const StepCtx& cx, Workspace& ws, const double* in, double* out, int c, const int* dimC,
                bool rank_test, int pos, int passes = 2, double skip_tol = 0.0, const double* projX = nullptr,
                int64_t strideX = 0);
void project_batch(const StepCtx& cx, Workspace& ws, const double* Q, int c, const int* dimC, const double* X,
                   int64_t strideX, double* xhat, int64_t strideXhat);

}  // namespace smg

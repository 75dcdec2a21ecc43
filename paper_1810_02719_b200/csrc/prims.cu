// L3 primitives of the C ABI (spectral.hpp building blocks) on the same kernels
// as the chain: build_laplacian, ShiftedInverseOperator (+apply/apply_once),
// SpMM, orthonormalize, orthogonal_iteration, dynamic_oi, the first-submesh
// basis, gft / igft.  Host pointers, Eigen column-major layout at the boundary.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/specmesh_gpu.h"
#include "common.cuh"
#include "doi.h"
#include "context.h"
#include "engine.h"
#include "firstbasis.h"

using namespace smg;

namespace {

template <class F>
smg_status guard(smg_context* ctx, F&& f) {
    return static_cast<smg_status>(guarded_call(ctx, std::forward<F>(f)));
}

std::string status_message(int kind, int64_t detail) {
    switch (kind) {
        case kRankDeficient: return "orthonormalize: block is rank deficient at column " + std::to_string(detail);
        case kAllZero: return "orthonormalize: block is rank deficient (all zero)";
        case kFactorFailed: return "sparse factorization of the shifted Laplacian failed";
        default: return "numerical failure (non-finite values)";
    }
}

void check_ws(Workspace& ws, cudaStream_t st) {
    int s = 0;
    int64_t d = 0;
    SMG_CUDA(cudaMemcpyAsync(&s, ws.status.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaMemcpyAsync(&d, ws.detail.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    if (s != 0) fail(3, status_message(s, d));
}

// column-major host block -> ws buffer (row-major)
void put_block(const double* host, int rows, int cols, double* dev_rowmajor, int64_t ld, cudaStream_t st) {
    DBuf<double> tmp;
    tmp.upload(host, (size_t)rows * cols, st);
    transpose_to_rowmajor(tmp.get(), rows, cols, dev_rowmajor, ld, st);
    SMG_CUDA(cudaStreamSynchronize(st));
}

void get_block(const double* dev_rowmajor, int64_t ld, int rows, int cols, const double* sign, double* host,
               cudaStream_t st) {
    DBuf<double> tmp;
    tmp.alloc((size_t)rows * cols, st);
    transpose_to_colmajor(dev_rowmajor, ld, rows, cols, sign, tmp.get(), st);
    if ((size_t)rows * cols)
        SMG_CUDA(cudaMemcpyAsync(host, tmp.get(), sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
}

// sign convention of ws.U's first c columns (projection against zero coords)
void signs_of(const StepCtx& cx, Workspace& ws, int c) {
    DBuf<double> zeros;
    zeros.alloc((size_t)ws.n * 3, cx.st);
    zeros.zero();
    project_batch(cx, ws, ws.U.get(), c, nullptr, zeros.get(), 0, nullptr, 0);
    SMG_CUDA(cudaStreamSynchronize(cx.st));
}

}  // namespace

extern "C" {

smg_status smg_build_laplacian(smg_context* ctx, const smg_mesh* mesh, const int32_t* members, int32_t n,
                               int32_t weighting, int32_t* rowptr, int32_t* cols, double* vals, int64_t nnz_capacity,
                               int64_t* nnz_out, double* trace_out) {
    return guard(ctx, [&] {
        const cudaStream_t st = ctx->stream;
        require(mesh != nullptr && members != nullptr, "mesh / members are null");
        require(n >= 2, "submesh must have at least 2 vertices");
        require(weighting == SMG_WEIGHTING_BINARY || weighting == SMG_WEIGHTING_DISTANCE,
                "unknown weighting (expected binary|distance)");
        DBuf<double> bx, by, bz;
        DBuf<int32_t> bo, bc, bm;
        const double *x = mesh->x, *y = mesh->y, *z = mesh->z;
        const int32_t *offs = mesh->adj_offsets, *acols = mesh->adj_cols, *mem = members;
        if (!mesh->on_device) {
            const int64_t nv = mesh->vertex_count;
            bx.upload(mesh->x, nv, st);
            by.upload(mesh->y, nv, st);
            bz.upload(mesh->z, nv, st);
            bo.upload(mesh->adj_offsets, nv + 1, st);
            bc.upload(mesh->adj_cols, mesh->adj_offsets[nv], st);
            bm.upload(members, n, st);
            x = bx.get();
            y = by.get();
            z = bz.get();
            offs = bo.get();
            acols = bc.get();
            mem = bm.get();
        }
        TileRef t{mem, offs, acols, x, y, z};
        TileSet ts;
        ts.build({t}, n, weighting, 1e-8, st);
        if (ts.status_h[0] == kCoincident) {
            const int64_t key = ts.detail_h[0];
            const int li = (int)(key >> 20), slot = (int)(key & 0xFFFFF);
            int32_t gi = 0, gj = 0, off = 0;
            SMG_CUDA(cudaMemcpy(&gi, mem + li, 4, cudaMemcpyDeviceToHost));
            SMG_CUDA(cudaMemcpy(&off, offs + gi, 4, cudaMemcpyDeviceToHost));
            SMG_CUDA(cudaMemcpy(&gj, acols + off + slot, 4, cudaMemcpyDeviceToHost));
            fail(3, "coincident connected vertices " + std::to_string(gi) + " and " + std::to_string(gj) +
                        " make the distance weight singular");
        }
        if (nnz_out) *nnz_out = ts.total_nnz;
        require(nnz_capacity >= ts.total_nnz, "CSR capacity too small");
        if (rowptr) SMG_CUDA(cudaMemcpyAsync(rowptr, ts.rowptr.get(), 4 * (n + 1), cudaMemcpyDeviceToHost, st));
        if (cols) SMG_CUDA(cudaMemcpyAsync(cols, ts.cols.get(), 4 * ts.total_nnz, cudaMemcpyDeviceToHost, st));
        if (vals) SMG_CUDA(cudaMemcpyAsync(vals, ts.vals.get(), 8 * ts.total_nnz, cudaMemcpyDeviceToHost, st));
        if (trace_out) SMG_CUDA(cudaMemcpyAsync(trace_out, ts.trace.get(), 8, cudaMemcpyDeviceToHost, st));
        SMG_CUDA(cudaStreamSynchronize(st));
    });
}

smg_status smg_operator_create(smg_context* ctx, int32_t n, const int32_t* rowptr, const int32_t* cols,
                               const double* vals, double delta, int32_t z, smg_operator** out) {
    return guard(ctx, [&] {
        require(out != nullptr, "operator output is null");
        *out = nullptr;
        require(delta > 0.0, "shift delta must be positive");
        require(z >= 1, "power z must be at least 1");
        require(rowptr != nullptr && cols != nullptr && vals != nullptr, "CSR arrays are null");
        auto op = std::make_unique<smg_operator>();
        op->n = n;
        op->z = z;
        op->delta = delta;
        op->ts.build_from_csr(n, rowptr, cols, vals, delta, ctx->stream);
        op->fs.factor(op->ts, 0, 1, nullptr, ctx->stream);
        std::vector<int> fst = download(op->fs.status.get(), 1, ctx->stream);
        if (fst[0] != 0) fail(3, "sparse factorization of the shifted Laplacian failed");
        // the operator may outlive the context's stream: free on the default stream
        SMG_CUDA(cudaStreamSynchronize(ctx->stream));
        op->ts.rebind(0);
        op->fs.rebind(0);
        *out = op.release();
    });
}

void smg_operator_destroy(smg_operator* op) { delete op; }

smg_status smg_operator_apply(smg_context* ctx, const smg_operator* op, int32_t c, const double* block, double* out,
                              int32_t once) {
    return guard(ctx, [&] {
        require(op != nullptr, "operator is null");
        require(c >= 1, "operator/block dimension mismatch");
        const cudaStream_t st = ctx->stream;
        Workspace ws;
        ws.init(1, op->n, op->ts.npad, c, st);
        put_block(block, op->n, c, ws.U.get(), ws.ld, st);
        StepCtx cx{st, &op->ts};
        solve_batch(cx, ws, op->fs, 0, 1, ws.U.get(), ws.V.get(), c, nullptr, op->z, once != 0);
        get_block(ws.V.get(), ws.ld, op->n, c, nullptr, out, st);
    });
}

smg_status smg_operator_spmm(smg_context* ctx, const smg_operator* op, int32_t c, const double* block, double* out) {
    return guard(ctx, [&] {
        require(op != nullptr, "operator is null");
        const cudaStream_t st = ctx->stream;
        Workspace ws;
        ws.init(1, op->n, op->ts.npad, c, st);
        put_block(block, op->n, c, ws.U.get(), ws.ld, st);
        SpmmParams sp;
        sp.n = op->n;
        sp.c = c;
        sp.rowptr = op->ts.rowptr.get();
        sp.csr_offsets = op->ts.off.get();
        sp.cols = op->ts.cols.get();
        sp.vals = op->ts.vals.get();
        sp.shift = op->ts.delta.get();
        sp.X = ws.U.get();
        sp.ldx = ws.ld;
        sp.Y = ws.V.get();
        sp.ldy = ws.ld;
        spmm(sp, st);
        get_block(ws.V.get(), ws.ld, op->n, c, nullptr, out, st);
    });
}

smg_status smg_orthonormalize(smg_context* ctx, int32_t rows, int32_t cols, const double* block, double* q) {
    return guard(ctx, [&] {
        require(cols >= 1 && rows >= cols, "block must be tall (rows >= cols >= 1)");
        require(cols <= 512, "block width exceeds the GPU limit of 512");
        const cudaStream_t st = ctx->stream;
        Workspace ws;
        ws.init(1, rows, round_up(rows, 64), cols, st);
        put_block(block, rows, cols, ws.V.get(), ws.ld, st);
        StepCtx cx{st, nullptr};
        orth_batch(cx, ws, ws.V.get(), ws.U.get(), cols, nullptr, true, 0);
        check_ws(ws, st);
        signs_of(cx, ws, cols);
        get_block(ws.U.get(), ws.ld, rows, cols, ws.sign.get(), q, st);
    });
}

smg_status smg_orthonormality_estimate(smg_context* ctx, int32_t rows, int32_t cols, const double* q,
                                       double* estimate) {
    return guard(ctx, [&] {
        require(cols >= 1 && rows >= cols, "block must be tall (rows >= cols >= 1)");
        require(cols <= 512, "block width exceeds the GPU limit of 512");
        require(estimate != nullptr, "estimate is null");
        const cudaStream_t st = ctx->stream;
        Workspace ws;
        ws.init(1, rows, round_up(rows, 64), cols, st);
        put_block(q, rows, cols, ws.V.get(), ws.ld, st);
        orth_probe(ws.V.get(), ws.ld, ws.mstride(), rows, nullptr, cols, 1, 0.0, ws.probe_part.get(), ws.skip.get(),
                   ws.probe_est.get(), st);
        SMG_CUDA(cudaGetLastError());
        SMG_CUDA(cudaMemcpyAsync(estimate, ws.probe_est.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
        SMG_CUDA(cudaStreamSynchronize(st));
    });
}

smg_status smg_orthogonal_iteration(smg_context* ctx, const smg_operator* op, int32_t c, const double* init,
                                    int32_t t_max, double* out) {
    return guard(ctx, [&] {
        require(op != nullptr, "operator is null");
        require(t_max >= 0, "t_max must be nonnegative");
        require(c >= 1 && c <= op->n, "initial basis does not match the operator size");
        const cudaStream_t st = ctx->stream;
        if (t_max == 0) {
            std::memcpy(out, init, sizeof(double) * (size_t)op->n * c);
            return;
        }
        Workspace ws;
        ws.init(1, op->n, op->ts.npad, c, st);
        put_block(init, op->n, c, ws.U.get(), ws.ld, st);
        StepCtx cx{st, &op->ts};
        for (int t = 0; t < t_max; ++t) {
            solve_batch(cx, ws, op->fs, 0, 1, ws.U.get(), ws.V.get(), c, nullptr, op->z, false);
            orth_batch(cx, ws, ws.V.get(), ws.U.get(), c, nullptr, true, t);
        }
        check_ws(ws, st);
        signs_of(cx, ws, c);
        get_block(ws.U.get(), ws.ld, op->n, c, ws.sign.get(), out, st);
    });
}

smg_status smg_dynamic_oi(smg_context* ctx, const smg_operator* op, int32_t c, const double* init,
                          const double* coords, double eps_low, double eps_high, int32_t c_min, int32_t c_max,
                          int32_t t_max, double* basis_out, int32_t* c_out, int32_t* converged, double* residual,
                          int32_t* iterations) {
    return guard(ctx, [&] {
        require(op != nullptr, "operator is null");
        require(eps_low > 0.0 && eps_low < eps_high, "need 0 < eps_low < eps_high");
        require(c_min >= 1 && c_min <= c && c <= c_max, "need c_min <= init subspace size <= c_max");
        require(c_max <= op->n, "c_max cannot exceed the submesh size");
        require(c_max + 1 <= 512, "c_max exceeds the GPU limit of 511");
        const cudaStream_t st = ctx->stream;
        const int n = op->n;
        Workspace ws;
        ws.init(1, n, op->ts.npad, c_max + 1, st);
        put_block(init, n, c, ws.U.get(), ws.ld, st);
        // coords (column-major n x 3 == SoA) -> row-major X + bbox diagonal on the device
        DBuf<double> cd, X, bb;
        DBuf<int32_t> iota;
        cd.upload(coords, (size_t)n * 3, st);
        std::vector<int32_t> io(n);
        for (int i = 0; i < n; ++i) io[i] = i;
        iota.upload(io, st);
        X.alloc((size_t)n * 3, st);
        bb.alloc(1, st);
        TileRef t{iota.get(), nullptr, nullptr, cd.get(), cd.get() + n, cd.get() + 2 * n};
        DBuf<TileRef> tr;
        tr.upload(&t, 1, st);
        gather_coords(tr.get(), 1, n, X.get(), 0, bb.get(), st);
        std::vector<double> bbox = download(bb.get(), 1, st);
        DoiParams dp;
        dp.c_min = c_min;
        dp.c_max = c_max;
        dp.t_max = t_max;
        dp.power = op->z;
        dp.eps_low = eps_low;
        dp.eps_high = eps_high;
        DoiLoop loop;
        loop.build(op->ts, ws, dp, op->fs.strideF, st);
        DoiState r = loop.run(op->fs.f(0), op->fs.b(0), op->ts.perm_of(0), X.get(), bbox[0], c);
        ctx->log_doi(loop, 0, r.t);
        check_ws(ws, st);
        StepCtx cx{st, &op->ts};
        if (r.appended_raw) {
            orth_batch(cx, ws, ws.U.get(), ws.U.get(), r.c, nullptr, true, 0);
            check_ws(ws, st);
        }
        signs_of(cx, ws, r.c);
        get_block(ws.U.get(), ws.ld, n, r.c, ws.sign.get(), basis_out, st);
        if (c_out) *c_out = r.c;
        if (converged) *converged = r.converged;
        if (residual) *residual = r.residual;
        if (iterations) *iterations = r.t;
    });
}

smg_status smg_bottom_subspace(smg_context* ctx, const smg_operator* op, int32_t c, double* basis_out,
                               double* eigenvalues_out) {
    return guard(ctx, [&] {
        require(op != nullptr, "operator is null");
        require(c >= 1 && c <= op->n, "subspace size out of range");
        const cudaStream_t st = ctx->stream;
        const int n = op->n;
        const int m = first_basis_width(n, c);
        require(m <= 512, "subspace size exceeds the GPU limit");
        Workspace ws;
        ws.init(1, n, op->ts.npad, m, st);
        StepCtx cx{st, &op->ts};
        FirstBasisConfig fc;
        fc.dense_limit = 4096;
        first_basis(cx, ws, op->ts, 0, 1, c, fc, &op->fs);
        signs_of(cx, ws, c);
        get_block(ws.U.get(), ws.ld, n, c, ws.sign.get(), basis_out, st);
        if (eigenvalues_out) {
            SMG_CUDA(cudaMemcpyAsync(eigenvalues_out, ws.theta_s.get(), 8 * c, cudaMemcpyDeviceToHost, st));
            SMG_CUDA(cudaStreamSynchronize(st));
        }
    });
}

smg_status smg_gft(smg_context* ctx, int32_t rows, int32_t c, const double* basis, const double* coords,
                   double* coeffs) {
    return guard(ctx, [&] {
        require(rows >= 1 && c >= 1, "coordinate/basis dimension mismatch");
        require(c <= 4096, "subspace size exceeds the GPU limit");
        const cudaStream_t st = ctx->stream;
        Workspace ws;
        ws.init(1, rows, round_up(rows, 64), c, st);
        put_block(basis, rows, c, ws.U.get(), ws.ld, st);
        DBuf<double> X;
        X.alloc((size_t)rows * 3, st);
        put_block(coords, rows, 3, X.get(), 3, st);
        StepCtx cx{st, nullptr};
        project_batch(cx, ws, ws.U.get(), c, nullptr, X.get(), 0, nullptr, 0);
        // coeff is c x 4 row-major (Px Py Pz Ps): copy the first three as column-major c x 3
        std::vector<double> h = download(ws.coeff.get(), (size_t)c * 4, st);
        for (int j = 0; j < c; ++j)
            for (int a = 0; a < 3; ++a) coeffs[(size_t)a * c + j] = h[(size_t)4 * j + a];
    });
}

}  // extern "C"

namespace {
__global__ void igft_kernel(const double* U, int64_t ld, int n, int c, const double* C, double* out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    double a[3] = {0.0, 0.0, 0.0};
    for (int j = lane; j < c; j += 32) {
        const double q = U[(int64_t)warp * ld + j];
        for (int k = 0; k < 3; ++k) a[k] = fma(q, C[(int64_t)k * c + j], a[k]);
    }
    for (int k = 0; k < 3; ++k) {
        const double v = warp_sum(a[k]);
        if (lane == 0) out[(int64_t)k * n + warp] = v;
    }
}
}  // namespace

extern "C" smg_status smg_igft(smg_context* ctx, int32_t rows, int32_t c, const double* basis, const double* coeffs,
                               double* coords) {
    return guard(ctx, [&] {
        require(rows >= 1 && c >= 1, "coefficient/basis dimension mismatch");
        const cudaStream_t st = ctx->stream;
        Workspace ws;
        ws.init(1, rows, round_up(rows, 64), c, st);
        put_block(basis, rows, c, ws.U.get(), ws.ld, st);
        DBuf<double> C, out;
        C.upload(coeffs, (size_t)c * 3, st);
        out.alloc((size_t)rows * 3, st);
        ::smg::count_launch(), igft_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(ws.U.get(), ws.ld, rows, c, C.get(), out.get());
        SMG_CUDA(cudaGetLastError());
        SMG_CUDA(cudaMemcpyAsync(coords, out.get(), 8 * (size_t)rows * 3, cudaMemcpyDeviceToHost, st));
        SMG_CUDA(cudaStreamSynchronize(st));
    });
}

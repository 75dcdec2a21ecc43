// Engine pieces shared by the chain runner and the L3 primitives.
#include <cstdio>

#include <cstdlib>
#include <string>

#include "engine.h"
#include "profiler.h"

namespace smg {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(3, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
}

namespace {
int supported_width(int w) {
    if (w <= 16) return 16;
    if (w <= 32) return 32;
    if (w <= 48) return 48;
    if (w <= 64) return 64;
    return -1;
}
}  // namespace

void TileSet::build(const std::vector<TileRef>& tiles, int n_, int weighting, double shift_scale, cudaStream_t st) {
    ProfScope prof("assemble", st);
    ntiles = (int)tiles.size();
    n = n_;
    this->weighting = weighting;
    require(n >= 2, "submesh must have at least 2 vertices");
    require(n <= 4096, "submesh size exceeds the GPU limit of 4096 vertices");
    refs.upload(tiles, st);
    nnz.alloc(ntiles, st);
    off.alloc(ntiles + 1, st);
    assemble_count(refs.get(), ntiles, n, nnz.get(), st);
    exclusive_scan_i32_to_i64(nnz.get(), off.get(), ntiles, st);
    int64_t tot = 0;
    SMG_CUDA(cudaMemcpyAsync(&tot, off.get() + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    total_nnz = tot;
    rowptr.alloc((size_t)ntiles * (n + 1), st);
    cols.alloc(tot, st);
    vals.alloc(tot, st);
    trace.alloc(ntiles, st);
    status.alloc(ntiles, st);
    status.zero();
    detail.alloc(ntiles, st);
    {
        std::vector<int64_t> big(ntiles, INT64_MAX);
        detail.upload(big, st);
    }
    assemble_fill(refs.get(), ntiles, n, weighting, off.get(), rowptr.get(), cols.get(), vals.get(), trace.get(),
                  status.get(), detail.get(), st);
    X.alloc((size_t)ntiles * n * 3, st);
    bbox.alloc(ntiles, st);
    gather_coords(refs.get(), ntiles, n, X.get(), (int64_t)n * 3, bbox.get(), st);
    finish_build(shift_scale, nullptr, st, X.get());
    status_h = download(status.get(), ntiles, st);
    detail_h = download(detail.get(), ntiles, st);
}

void TileSet::build_from_csr(int n_, const int32_t* rowptr_h, const int32_t* cols_h, const double* vals_h,
                             double delta_h, cudaStream_t st) {
    ntiles = 1;
    n = n_;
    require(n >= 1, "operator size must be positive");
    require(n <= 4096, "submesh size exceeds the GPU limit of 4096 vertices");
    const int64_t nz = rowptr_h[n];
    total_nnz = nz;
    rowptr.upload(rowptr_h, n + 1, st);
    cols.upload(cols_h, nz, st);
    vals.upload(vals_h, nz, st);
    std::vector<int64_t> o = {0, nz};
    off.upload(o, st);
    // trace in index order (spectral.hpp:32-36)
    double t = 0.0;
    for (int i = 0; i < n; ++i)
        for (int64_t e = rowptr_h[i]; e < rowptr_h[i + 1]; ++e)
            if (cols_h[e] == i) t += vals_h[e];
    std::vector<double> th = {t};
    trace.upload(th, st);
    std::vector<double> dh = {delta_h};
    status.alloc(1, st);
    status.zero();
    finish_build(0.0, &dh, st);
}

void TileSet::finish_build(double shift_scale, const std::vector<double>* explicit_delta, cudaStream_t st,
                           const double* coords) {
    // ordering: the narrowest block-tridiagonal width among the natural order,
    // the geometric order along the tile's longest axis (when coordinates are
    // known) and, if neither is supported, RCM
    bw.alloc(ntiles, st);
    blockw.alloc(ntiles, st);
    DBuf<int32_t> lower;
    lower.alloc(ntiles, st);
    auto widest = [&](const int32_t* pm) {
        natural_bandwidth(rowptr.get(), cols.get(), off.get(), pm, ntiles, n, bw.get(), blockw.get(), lower.get(), st);
        std::vector<int32_t> h = download(blockw.get(), ntiles, st);
        int w = 1;
        for (int v : h) w = std::max(w, v);
        return w;
    };
    int wmax = widest(nullptr);
    use_perm = false;
    ordering = 0;
    // SMG_ORDERING=geometric|natural forces a candidate (tests exercise every path)
    const char* force = std::getenv("SMG_ORDERING");
    const bool force_geo = force && std::string(force) == "geometric";
    const bool force_nat = force && std::string(force) == "natural";
    // A narrower W halves the solve's flops and shrinks its per-step slabs, but
    // doubles its sequential steps: worth it when many tiles keep the GPU
    // throughput-bound, not for a few latency-bound chains whose natural order works.
    if (coords && !topology_ordering && !force_nat && (supported_width(wmax) < 0 || ntiles >= 1024 || force_geo)) {
        DBuf<int32_t> ap;
        ap.alloc((size_t)ntiles * n, st);
        axis_order(coords, (int64_t)n * 3, ntiles, n, ap.get(), st);
        const int wa = widest(ap.get());
        const int sn = supported_width(wmax), sa = supported_width(wa);
        if (sa > 0 && (sn < 0 || sa < sn)) {
            perm = std::move(ap);
            use_perm = true;
            ordering = 1;
            wmax = wa;
        }
    }
    if (supported_width(widest(nullptr)) < 0) {
        // the natural order is not block tridiagonal at W <= 64: RCM competes too
        DBuf<int32_t> rp;
        rp.alloc((size_t)ntiles * n, st);
        rcm_order(rowptr.get(), cols.get(), off.get(), ntiles, n, rp.get(), st);
        const int sr = supported_width(widest(rp.get()));
        const int sc = use_perm ? supported_width(wmax) : -1;
        if (sr > 0 && (sc < 0 || sr <= sc)) {
            perm = std::move(rp);
            use_perm = true;
            ordering = 2;
        } else if (sc < 0) {
            perm = std::move(rp);  // unsupported either way: reported below
            use_perm = true;
            ordering = 2;
        }
    }
    wmax = widest(use_perm ? perm.get() : nullptr);  // final order: width and coupling bound
    {
        std::vector<int32_t> lh = download(lower.get(), ntiles, st);
        int lm = 1;
        for (int v : lh) lm = std::max(lm, v);
        cpl = round_up(lm, 2);  // couplings into the previous block <= lower neighbours
    }
    W = supported_width(wmax);
    if (W < 0) fail(2, "submesh bandwidth after RCM ordering exceeds the supported block width 64");
    Kb = (n + W - 1) / W;
    npad = Kb * W;
    if (explicit_delta) {
        delta.upload(*explicit_delta, st);
    } else {
        delta.alloc(ntiles, st);
        compute_delta(trace.get(), ntiles, n, shift_scale, delta.get(), st);
    }
    shift0.alloc((size_t)2 * ntiles, st);  // [shift | Gershgorin upper bound]
    compute_first_shift(rowptr.get(), cols.get(), vals.get(), off.get(), trace.get(), ntiles, n, shift0.get(), st);
}

void FactorSet::factor(const TileSet& ts, int first_tile, int cnt, const double* shift, cudaStream_t st,
                       int* status_out) {
    ProfScope prof("factor", st);
    first = first_tile;
    count = cnt;
    strideF = (int64_t)ts.Kb * 2 * ts.W * factor_row(ts.W);
    if (fwd.size() < (size_t)strideF * cnt) {
        fwd.alloc((size_t)strideF * cnt, st);
        bwd.alloc((size_t)strideF * cnt, st);
        status.alloc(cnt, st);
    }
    status.zero();
    FactorParams p;
    p.ntiles = cnt;
    p.n = ts.n;
    p.W = ts.W;
    p.Kb = ts.Kb;
    p.rowptr = ts.rowptr.get() + (int64_t)first_tile * (ts.n + 1);
    p.cols = ts.cols.get();
    p.vals = ts.vals.get();
    p.csr_offsets = ts.off.get() + first_tile;
    p.perm = ts.use_perm ? ts.perm.get() + (int64_t)first_tile * ts.n : nullptr;
    p.delta = (shift ? shift : ts.delta.get()) + first_tile;
    p.Ffwd = fwd.get();
    p.Fbwd = bwd.get();
    p.strideF = strideF;
    p.cpl = ts.cpl;
    p.status = status_out ? status_out : status.get();
    factor_tiles(p, st);
    SMG_CUDA(cudaGetLastError());
}

void Workspace::init(int B_, int n_, int npad_, int ccap_, cudaStream_t st) {
    B = B_;
    n = n_;
    npad = npad_;
    ccap = ccap_;
    ld = round_up(std::max(ccap, 8), 32);
    const size_t mat = (size_t)B * npad * ld;
    U.alloc(mat, st);
    V.alloc(mat, st);
    T.alloc(mat, st);
    R.alloc(mat, st);
    U.zero();
    V.zero();
    T.zero();
    R.zero();
    const size_t cc = (size_t)B * ld * ld;
    G.alloc(cc, st);
    Bm.alloc(cc, st);
    work.alloc(cc, st);
    // split-K over the n rows for the Gram: ~8 waves of CTAs (4 splits at C5,
    // measured best), splits of >= 64 rows, at most 16 (single chains are
    // latency-bound: 16 splits took C2 27.4 -> 24.2 ms)
    const int tiles = ((ld + 63) / 64) * ((ld + 63) / 64 + 1) / 2;
    splits = std::max(1, std::min(std::min(npad / 64, 16), (1184 + tiles * B - 1) / std::max(1, tiles * B)));
    if (const char* e = std::getenv("SMG_GRAM_SPLITS")) splits = std::max(1, std::min(npad / 64, std::atoi(e)));
    Gws.alloc((size_t)B * splits * ld * ld, st);
    rdiag.alloc((size_t)B * ld, st);
    vnorm.alloc(B, st);
    rpart.alloc((size_t)B * ((npad + 31) / 32) * ld, st);  // rank_check chunks of 32 rows
    counters.alloc((size_t)3 * B, st);  // last-CTA reductions: rank check | projection (2)
    counters.zero();
    coeff.alloc((size_t)B * ld * 4, st);
    sign.alloc((size_t)B * ld, st);
    e.alloc((size_t)B * npad, st);
    ppart.alloc((size_t)B * proj_chunks(n) * ld * 8, st);
    ppart2.alloc((size_t)B * proj_recon_blocks(n, 2) * 2, st);
    stats.alloc((size_t)B * 4, st);
    status.alloc(B, st);
    status.zero();
    probe_part.alloc((size_t)B * orth_probe_chunks(n) * ld * 8, st);
    probe_est.alloc(B, st);
    skip.alloc(B, st);
    skip.zero();
    skip2.alloc(B, st);
    skip2.zero();
    nmax.alloc(B, st);
    errpos.alloc(B, st);
    errpos.zero();
    rneed.alloc(B, st);
    rneed.zero();
    detail.alloc(B, st);
    detail.zero();
}

void solve_batch(const StepCtx& cx, Workspace& ws, const FactorSet& fs, int tile0, int tstride, const double* in,
                 double* out, int c, const int* dimC, int z, bool once) {
    ProfScope prof("solve", cx.st);
    const TileSet& ts = *cx.ts;
    SolveParams p;
    p.n = ts.n;
    p.Kb = ts.Kb;
    p.z = z;
    p.c_cap = c;
    p.batch = ws.B;
    p.Ffwd = fs.f(tile0);
    p.Fbwd = fs.b(tile0);
    p.strideF = (int64_t)tstride * fs.strideF;
    p.perm = ts.perm_of(tile0);
    p.stridePerm = ts.use_perm ? (int64_t)tstride * ts.n : 0;
    p.in = in;
    p.ldin = ws.ld;
    p.strideIn = ws.mstride();
    p.tmp = ws.T.get();
    p.ldt = ws.ld;
    p.strideT = ws.mstride();
    p.out = out;
    p.ldout = ws.ld;
    p.strideOut = ws.mstride();
    p.dimC = dimC;
    p.dimStride = 1;
    p.once = once ? 1 : 0;
    solve_block_tridiag(p, ts.W, cx.st);
    SMG_CUDA(cudaGetLastError());
}

namespace {
void gram(Workspace& ws, const double* V, int c, const int* dimC, int n, cudaStream_t st,
          const int* skip = nullptr) {
    GemmParams g;
    g.skip = skip;
    g.M = c;
    g.N = c;
    g.K = n;
    g.batch = ws.B;
    g.splits = ws.splits;
    g.A = V;
    g.lda = ws.ld;
    g.strideA = ws.mstride();
    g.B = V;
    g.ldb = ws.ld;
    g.strideB = ws.mstride();
    g.syrkUpper = 1;
    g.dimM = dimC;
    g.dimN = dimC;
    g.dimStride = 1;
    if (g.splits > 1) {
        g.C = ws.Gws.get();
        g.ldc = ws.ld;
        g.strideP = (int64_t)ws.ld * ws.ld;
        g.out = ws.G.get();
        g.ldo = ws.ld;
        g.strideC = (int64_t)ws.ld * ws.ld;
    } else {
        g.C = ws.G.get();
        g.ldc = ws.ld;
        g.strideC = (int64_t)ws.ld * ws.ld;
    }
    ProfScope prof("gram", st);
    gemm(g, true, false, st);
}

// out = V D^-1 R~^-1 with R~ / Dinv / d from the last chol()
// Q = V D^-1 R~^-1 from the pass-1 Cholesky (skip_inverse) by the row-parallel solve
void trsm(Workspace& ws, const double* V, double* out, int c, const int* dimC, int n, cudaStream_t st) {
    TrsmParams t;
    t.n = n;
    t.batch = ws.B;
    t.c_cap = c;
    t.V = V;
    t.ldv = ws.ld;
    t.strideV = ws.mstride();
    t.Q = out;
    t.ldq = ws.ld;
    t.strideQ = ws.mstride();
    t.R = ws.work.get();
    t.ldr = ws.ld;
    t.strideR = (int64_t)ws.ld * ws.ld;
    t.Binv = ws.Bm.get();
    t.ldb = ws.ld;
    t.strideB = (int64_t)ws.ld * ws.ld;
    t.dscale = ws.rdiag.get();
    t.strideD = ws.ld;
    t.dimC = dimC;
    t.dimStride = 1;
    t.status = ws.status.get();
    ProfScope prof("trmm", st);
    trsm_right_upper(t, st);
}

// The solve replaces the Cholesky's serial back-substitution by row-parallel
// work; it pays when few chains leave SMs idle during that single-CTA phase
// (small batches), while at large batches the plain GEMM with B = D^-1 R~^-1
// is faster (the back-substitution overlaps the other chain group's kernels).
bool use_trsm(int c, int batch) {
    static const bool off = std::getenv("SMG_NO_TRSM") != nullptr;
    static const int maxb = std::getenv("SMG_TRSM_MAXB") ? std::atoi(std::getenv("SMG_TRSM_MAXB")) : 4;
    return !off && batch <= maxb && trsm_supported(c);
}

void trmm(Workspace& ws, const double* V, double* out, int c, const int* dimC, int n, cudaStream_t st,
          const int* skip = nullptr, const double* projX = nullptr, int64_t strideX = 0) {
    GemmParams g;
    if (projX) {
        g.projX = projX;
        g.strideProjX = strideX;
        g.projPart = ws.ppart.get();
        g.projN = ws.n;
        g.projChunks = proj_chunks(ws.n);
        g.projCcap = c;
    }
    g.skip = skip;
    g.M = n;
    g.N = c;
    g.K = c;
    g.batch = ws.B;
    g.A = V;
    g.lda = ws.ld;
    g.strideA = ws.mstride();
    g.B = ws.Bm.get();
    g.ldb = ws.ld;
    g.strideB = (int64_t)ws.ld * ws.ld;
    g.C = out;
    g.ldc = ws.ld;
    g.strideC = ws.mstride();
    g.upperB = 1;
    g.dimN = dimC;
    g.dimK = dimC;
    g.dimStride = 1;
    ProfScope prof("trmm", st);
    gemm(g, false, false, st);
}

void chol(Workspace& ws, int c, const int* dimC, bool rank_test, bool column_scale, int pos, cudaStream_t st,
          bool near_identity = false, bool skip_inverse = false, const int* skip = nullptr, int* skip_out = nullptr,
          double skip_tol = 0.0) {
    CholParams p;
    p.skip = skip;
    p.skip_out = skip_out;
    p.skip_tol = skip_tol;
    p.batch = ws.B;
    p.c_cap = c;
    p.G = ws.G.get();
    p.ldg = ws.ld;
    p.strideG = (int64_t)ws.ld * ws.ld;
    p.A = ws.work.get();
    p.lda = ws.ld;
    p.strideA = (int64_t)ws.ld * ws.ld;
    p.Binv = ws.Bm.get();
    p.ldb = ws.ld;
    p.strideB = (int64_t)ws.ld * ws.ld;
    p.dscale = ws.rdiag.get();
    p.strideD = ws.ld;
    p.dimC = dimC;
    p.dimStride = 1;
    p.status = ws.status.get();
    p.status_detail = ws.detail.get();
    p.errpos = ws.errpos.get();
    p.pos = pos;
    p.rank_test = rank_test ? 1 : 0;
    p.column_scale = column_scale ? 1 : 0;
    p.vnorm = rank_test ? ws.vnorm.get() : nullptr;
    p.rank_need = rank_test ? ws.rneed.get() : nullptr;
    p.near_identity = near_identity ? 1 : 0;
    p.skip_inverse = skip_inverse ? 1 : 0;
    ProfScope prof("chol", st);
    chol_factor(p, st);
}
}  // namespace

// second CholeskyQR pass: near-identity chains (max |G~ - I| <= 1e-9, the usual
// case) get B to first order on all SMs; only the others run the full Cholesky
void chol_pass2(Workspace& ws, int c, const int* dimC, int pos, cudaStream_t st, const int* skip_in) {
    if (c <= 256) {
        // small c: the single-CTA near-identity scan inside the Cholesky kernel is
        // cheaper than three launches
        chol(ws, c, dimC, false, true, pos, st, true, false, skip_in);
        return;
    }
    ProfScope prof("chol", st);
    const int64_t sG = (int64_t)ws.ld * ws.ld;
    SMG_CUDA(cudaMemsetAsync(ws.nmax.get(), 0, sizeof(unsigned long long) * ws.B, st));
    near_check(ws.G.get(), ws.ld, sG, dimC, c, ws.B, ws.nmax.get(), st);
    near_fill(ws.G.get(), ws.ld, sG, dimC, c, ws.B, ws.nmax.get(), skip_in, ws.skip2.get(), ws.Bm.get(), ws.ld, sG,
              ws.rdiag.get(), ws.ld, st);
    chol(ws, c, dimC, false, true, pos, st, false, false, ws.skip2.get());
}

void orth_batch(const StepCtx& cx, Workspace& ws, const double* in, double* out, int c, const int* dimC,
                bool rank_test, int pos, int passes, double skip_tol, const double* projX, int64_t strideX) {
    ProfScope prof("orthonormalize", cx.st);
    ws.proj_ready = false;
    const int n = ws.npad;
    const bool adaptive = skip_tol > 0.0 && passes == 2;
    if ((rank_test || adaptive) && in == out) {
        // keep the input for the accurate rank test (T is free between solves)
        SMG_CUDA(cudaMemcpyAsync(ws.T.get(), in, sizeof(double) * ws.mstride() * ws.B, cudaMemcpyDeviceToDevice,
                                 cx.st));
        in = ws.T.get();
    }
    gram(ws, in, c, dimC, n, cx.st);
    if (rank_test) SMG_CUDA(cudaMemsetAsync(ws.rneed.get(), 0, sizeof(int) * ws.B, cx.st));
    const bool ts = use_trsm(c, ws.B);
    chol(ws, c, dimC, rank_test, true, pos, cx.st, false, ts);
    auto pass1 = [&](double* dst) {
        if (ts) trsm(ws, in, dst, c, dimC, n, cx.st);
        else trmm(ws, in, dst, c, dimC, n, cx.st);
    };
    if (passes == 1) {  // single CholeskyQR pass (span-only uses: subspace iteration)
        pass1(out);
        SMG_CUDA(cudaGetLastError());
        return;
    }
    if (adaptive) {
        // Q1 straight into out; pass 2 only for chains whose Q1 is not yet
        // orthonormal to skip_tol (their Q = Q1 B2 goes through R and back)
        // the triangular products also emit the projection's partial records
        // (project_batch then skips its read of the basis)
        const bool fuse = projX != nullptr && !ts && dimC == nullptr && std::getenv("SMG_PROJ_FUSE") != nullptr;
        if (fuse) trmm(ws, in, out, c, dimC, n, cx.st, nullptr, projX, strideX);
        else pass1(out);
        // Is Q1 orthonormal already?  Default: a one-pass randomized probe of |Q1^T Q1 - I|_F
        // (probe.cu) against skip_tol * sqrt(c); the chains that fail (and only they) form the
        // second Gram and factor it.  SMG_ORTH_PROBE=0: the exact max-entry test on the full
        // second Gram of every chain, as before.
        static const bool probe = !(std::getenv("SMG_ORTH_PROBE") && std::atoi(std::getenv("SMG_ORTH_PROBE")) == 0);
        if (probe) {
            {
                ProfScope pc("chol", cx.st);
                orth_probe(out, ws.ld, ws.mstride(), ws.n, dimC, c, ws.B, skip_tol * std::sqrt((double)c),
                           ws.probe_part.get(), ws.skip.get(), ws.probe_est.get(), cx.st);
            }
            gram(ws, out, c, dimC, n, cx.st, ws.skip.get());
            chol_pass2(ws, c, dimC, pos, cx.st, ws.skip.get());
        } else if (c <= 256) {
            gram(ws, out, c, dimC, n, cx.st);
            // the single-CTA pass-2 scan decides the skip too (one launch)
            chol(ws, c, dimC, false, true, pos, cx.st, true, false, nullptr, ws.skip.get(), skip_tol);
        } else {
            gram(ws, out, c, dimC, n, cx.st);
            {
                ProfScope pc("chol", cx.st);
                orth_check(ws.G.get(), ws.ld, (int64_t)ws.ld * ws.ld, dimC, 1, c, ws.B, skip_tol, ws.skip.get(), cx.st);
            }
            chol_pass2(ws, c, dimC, pos, cx.st, ws.skip.get());
        }
        trmm(ws, out, ws.R.get(), c, dimC, n, cx.st, ws.skip.get(), fuse ? projX : nullptr, strideX);
        ws.proj_ready = fuse;
        copy_unskipped(ws.R.get(), out, ws.mstride(), ws.mstride(), ws.B, ws.skip.get(), cx.st);
    } else {
        pass1(ws.R.get());
        gram(ws, ws.R.get(), c, dimC, n, cx.st);
        chol_pass2(ws, c, dimC, pos, cx.st, nullptr);
        trmm(ws, ws.R.get(), out, c, dimC, n, cx.st);
    }
    if (rank_test) {
        RankCheckParams r;
        r.n = ws.n;
        r.batch = ws.B;
        r.c_cap = c;
        r.Q = out;
        r.V = in;
        r.ld = ws.ld;
        r.stride = ws.mstride();
        r.dimC = dimC;
        r.dimStride = 1;
        r.vnorm = ws.vnorm.get();
        r.partial = ws.rpart.get();
        r.counter = ws.counters.get();
        r.need = ws.rneed.get();
        r.status = ws.status.get();
        r.status_detail = ws.detail.get();
        r.errpos = ws.errpos.get();
        r.pos = pos;
        rank_check(r, cx.st);
    }
    SMG_CUDA(cudaGetLastError());
}

void project_batch(const StepCtx& cx, Workspace& ws, const double* Q, int c, const int* dimC, const double* X,
                   int64_t strideX, double* xhat, int64_t strideXhat) {
    ProfScope prof("project", cx.st);
    ProjParams p;
    p.n = ws.n;
    p.batch = ws.B;
    p.c_cap = c;
    p.Q = Q;
    p.ldq = ws.ld;
    p.strideQ = ws.mstride();
    p.X = X;
    p.strideX = strideX;
    p.dimC = dimC;
    p.dimStride = 1;
    p.partial = ws.ppart.get();
    p.partial2 = ws.ppart2.get();
    p.coeff = ws.coeff.get();
    p.strideCoef = (int64_t)ws.ld * 4;
    p.sign = ws.sign.get();
    p.strideSign = ws.ld;
    p.xhat = xhat;
    p.strideXhat = strideXhat;
    p.e_out = ws.e.get();
    p.strideE = ws.npad;
    p.stats = ws.stats.get();
    p.strideStats = 4;
    p.rows_per_warp = 2;
    p.counter = ws.counters.get() + ws.B;
    p.partials_ready = ws.proj_ready ? 1 : 0;
    ws.proj_ready = false;
    project(p, cx.st);
    SMG_CUDA(cudaGetLastError());
}

}  // namespace smg

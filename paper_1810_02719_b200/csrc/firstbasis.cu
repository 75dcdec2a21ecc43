// K9: the first-submesh basis on the GPU.
//
// Reference: detail::initial_block_basis (pipeline.hpp:113-120) =
// bottom_subspace(dense_eigendecomposition(L), c) when n_d <= dense_limit, else
// a cold OI start from random_orthonormal_basis with initial_iterations steps.
//
// Dense path replacement: shift-invert subspace iteration on the tile's own
// block factor with m = c + max(16, c/2) guard columns, then Rayleigh-Ritz:
//   Y = L U (CSR SpMM, K4), H = U^T Y, H = W Theta W^T (cluster Jacobi),
//   Z = U W.  The bottom-c Ritz vectors converge at ((lambda_c+s)/(lambda_{m+1}+s))^z
//   per step instead of the ((lambda_c+s)/(lambda_{c+1}+s))^z of plain OI, and the
// loop stops when the Davis-Kahan bound max_j ||L z_j - theta_j z_j|| / (theta_{c+1}
// - theta_c) on the subspace angle is below 1e-12.  The shift s is the Gershgorin
// lower bound of L plus 1e-3 * mean diagonal, so L + sI is positive definite for
// either weighting and the bottom of the spectrum is what the iteration finds.
// Only span(bottom c) is needed downstream: fixed-c OI and the projections
// depend on the span, and the sign convention is re-applied in project.cu.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "engine.h"
#include "firstbasis.h"
#include "profiler.h"

namespace smg {

namespace {

void gemm_nn(Workspace& ws, const double* A, int64_t lda, const double* Bm, int64_t ldb, int64_t strideB, double* C,
             int M, int N, int K, cudaStream_t st) {
    GemmParams g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.batch = ws.B;
    g.A = A;
    g.lda = lda;
    g.strideA = ws.mstride();
    g.B = Bm;
    g.ldb = ldb;
    g.strideB = strideB;
    g.C = C;
    g.ldc = ws.ld;
    g.strideC = ws.mstride();
    gemm(g, false, false, st);
}

}  // namespace

std::vector<double> gaussian_block_colmajor(int rows, int cols, uint64_t seed) {
    // spectral.hpp:135-139 / pipeline.hpp:104-107: std::mt19937_64 + libstdc++'s
    // normal_distribution, column-major fill -- the same draws as the reference.
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> out((size_t)rows * cols);
    for (int j = 0; j < cols; ++j)
        for (int i = 0; i < rows; ++i) out[(size_t)j * rows + i] = gauss(rng);
    return out;
}

namespace {
FirstBasisReport first_basis_impl(const StepCtx& cx, Workspace& ws, const TileSet& ts, int tile0, int tstride, int c,
                                  const FirstBasisConfig& cfg, const FactorSet* op_factor, bool allow_cheb,
                                  bool* broke) {
    FirstBasisReport rep;
    const cudaStream_t st = cx.st;
    const int n = ts.n;
    // recorded as one "first_basis" stage; its inner solves/QRs are not
    // attributed to the chain's per-step stages
    struct Scope {
        Profiler* saved;
        int token;
        cudaStream_t st;
        explicit Scope(cudaStream_t s) : saved(active_profiler()), token(-1), st(s) {
            if (saved) token = saved->begin(st);
            active_profiler() = nullptr;
        }
        ~Scope() {
            active_profiler() = saved;
            if (saved && token >= 0) saved->end("first_basis", token, st);
        }
    } scope(st);
    if (n > cfg.dense_limit) {
        // cold start exactly as the reference: random_orthonormal_basis + OI
        require(op_factor != nullptr, "internal: cold start needs the operator factor");
        std::vector<double> g = gaussian_block_colmajor(n, c, cfg.seed ^ 0x9E3779B97F4A7C15ULL);
        DBuf<double> gd;
        gd.upload(g, st);
        for (int b = 0; b < ws.B; ++b)
            transpose_to_rowmajor(gd.get(), n, c, ws.V.get() + (int64_t)b * ws.mstride(), ws.ld, st);
        orth_batch(cx, ws, ws.V.get(), ws.U.get(), c, nullptr, true, 0);
        for (int t = 0; t < cfg.initial_iterations; ++t) {
            solve_batch(cx, ws, *op_factor, tile0, tstride, ws.U.get(), ws.V.get(), c, nullptr, cfg.power, false);
            orth_batch(cx, ws, ws.V.get(), ws.U.get(), c, nullptr, true, 0);
        }
        rep.iterations = cfg.initial_iterations;
        rep.cold = true;
        return rep;
    }

    const int m = first_basis_width(n, c);
    require(m <= kFirstBasisMaxCols, "first-submesh subspace size exceeds the GPU limit of 480");
    require(m <= ws.ccap, "internal: workspace too small for the first-basis subspace");
    FactorSet fs;
    fs.factor(ts, tile0, (ws.B - 1) * tstride + 1, ts.shift0.get(), st);
    // the factor set covers tiles tile0 .. tile0 + (B-1)*tstride; solve_batch indexes with tstride

    JacobiPlan pl = jacobi_plan(m);
    ws.H.alloc((size_t)ws.B * m * m, st);
    ws.Hst.alloc((size_t)ws.B * pl.stage_elems, st);
    ws.Vj.alloc((size_t)ws.B * m * m, st);
    ws.theta.alloc((size_t)ws.B * m, st);
    ws.theta_s.alloc((size_t)ws.B * m, st);
    ws.Wm.alloc((size_t)ws.B * m * m, st);
    const int nres = std::min(m, c + 1);
    const int rchunks = (n + 127) / 128;
    ws.ritz_part.alloc((size_t)ws.B * rchunks * nres, st);
    ws.ritz.alloc((size_t)ws.B * nres, st);

    randn(ws.V.get(), n, m, ws.ld, ws.mstride(), ws.B, cfg.seed * 0x2545F4914F6CDD1DULL + 17, st);
    orth_batch(cx, ws, ws.V.get(), ws.U.get(), m, nullptr, false, 0);

    FirstBasisConfig fc = cfg;
    {
        double s0 = 0.0;
        SMG_CUDA(cudaMemcpyAsync(&s0, ts.shift0.get() + tile0, sizeof(double), cudaMemcpyDeviceToHost, st));
        SMG_CUDA(cudaStreamSynchronize(st));
        fc.shift_hint = s0;
    }
    // Gershgorin upper bounds of L (Chebyshev interval end), per batch entry
    std::vector<double> upper(ws.B);
    for (int b = 0; b < ws.B; ++b)
        SMG_CUDA(cudaMemcpyAsync(&upper[b], ts.shift0.get() + ts.ntiles + tile0 + (int64_t)b * tstride,
                                 sizeof(double), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    const bool use_cheb =
        allow_cheb && !(std::getenv("SMG_FIRST_BASIS") && std::string(std::getenv("SMG_FIRST_BASIS")) == "si");
    const int deg = std::getenv("SMG_FB_DEG") ? std::max(2, std::atoi(std::getenv("SMG_FB_DEG"))) : 40;
    DBuf<double> dcoef;          // [deg][B] alpha | [deg][B] gamma | [B] shift
    int iters_next = (m == n) ? 0 : (use_cheb ? 4 : 6);
    if (const char* e = std::getenv("SMG_FB_BOOT")) iters_next = std::max(1, std::atoi(e));
    int cheb_apps = 0;
    double prev_bound = INFINITY;
    for (int round = 0; round < fc.max_rounds; ++round) {
        const int tk_it = scope.saved ? scope.saved->begin(st) : -1;
        if (cheb_apps > 0) {
            // Chebyshev-filtered subspace iteration on L (SpMM only): p_d damps
            // [a, b] = [theta_m, Gershgorin bound] and keeps the bottom of the spectrum
            double* bufs[3] = {ws.U.get(), ws.V.get(), ws.T.get()};
            // binary-weight tiles whose pattern fits shared memory run the fused filter
            int max_nnz = 0;
            bool fused = ts.weighting == 0 && !std::getenv("SMG_CHEB_UNFUSED");
            if (fused) {
                std::vector<int32_t> nz = download(ts.nnz.get(), (size_t)ts.ntiles, st);
                for (int b = 0; b < ws.B; ++b) max_nnz = std::max(max_nnz, nz[(size_t)tile0 + (size_t)b * tstride]);
                fused = cheb_filter_supported(n, max_nnz);
            }
            for (int app = 0; app < cheb_apps && fused; ++app) {
                // all deg steps in one launch, iterates in shared memory (bit-identical
                // to the per-step SpMM path below)
                ChebParams cp;
                cp.n = n;
                cp.c = m;
                cp.batch = ws.B;
                cp.deg = deg;
                cp.rowptr = ts.rowptr.get() + (int64_t)tile0 * (n + 1);
                cp.strideRowptr = (int64_t)tstride * (n + 1);
                cp.csr_offsets = ts.off.get() + tile0;
                cp.offStride = tstride;
                cp.cols = ts.cols.get();
                cp.vals = ts.vals.get();
                cp.coef = dcoef.get();
                cp.X = ws.U.get();
                cp.ldx = ws.ld;
                cp.strideX = ws.mstride();
                cp.Y = ws.V.get();
                cp.ldy = ws.ld;
                cp.strideY = ws.mstride();
                {
                    ProfScope ps("fb_filter", st);
                    cheb_filter(cp, max_nnz, st);
                }
                // same CholeskyQR passes as the per-step path, whose iterate lands back
                // in U (in place: full CholeskyQR2) when deg % 3 == 0
                const bool last = app + 1 == cheb_apps;
                orth_batch(cx, ws, ws.V.get(), ws.U.get(), m, nullptr, false, 0, (last || deg % 3 == 0) ? 2 : 1);
                rep.iterations += deg;
            }
            for (int app = 0; app < cheb_apps && !fused; ++app) {
                int x = 0, y = 1;
                for (int i = 1; i <= deg; ++i) {
                    const int z = (i == 1) ? 1 : 3 - x - y;
                    SpmmParams sp;
                    sp.n = n;
                    sp.c = m;
                    sp.batch = ws.B;
                    sp.rowptr = ts.rowptr.get() + (int64_t)tile0 * (n + 1);
                    sp.strideRowptr = (int64_t)tstride * (n + 1);
                    sp.csr_offsets = ts.off.get() + tile0;
                    sp.offStride = tstride;
                    sp.cols = ts.cols.get();
                    sp.vals = ts.vals.get();
                    sp.shift = dcoef.get() + (size_t)2 * deg * ws.B;
                    sp.alpha = dcoef.get() + (size_t)(i - 1) * ws.B;
                    sp.X = bufs[i == 1 ? 0 : y];
                    sp.ldx = ws.ld;
                    sp.strideX = ws.mstride();
                    if (i > 1) {
                        sp.gamma = dcoef.get() + (size_t)deg * ws.B + (size_t)(i - 1) * ws.B;
                        sp.Z = bufs[x];
                        sp.ldz = ws.ld;
                        sp.strideZ = ws.mstride();
                    }
                    sp.Y = bufs[z];
                    sp.ldy = ws.ld;
                    sp.strideY = ws.mstride();
                    spmm(sp, st);
                    if (i == 1) {
                        x = 0;
                        y = 1;
                    } else {
                        x = y;
                        y = z;
                    }
                }
                const bool last = app + 1 == cheb_apps;
                orth_batch(cx, ws, bufs[y], ws.U.get(), m, nullptr, false, 0, (last || y == 0) ? 2 : 1);
                rep.iterations += deg;
            }
        } else {
            for (int t = 0; t < iters_next; ++t) {
                const int z = (round == 0 && t == 0) ? 1 : 2;
                solve_batch(cx, ws, fs, tile0, tstride, ws.U.get(), ws.V.get(), m, nullptr, z, false);
                // intermediate iterates only need their span: one CholeskyQR pass;
                // the iterate entering Rayleigh-Ritz gets the full CholeskyQR2
                orth_batch(cx, ws, ws.V.get(), ws.U.get(), m, nullptr, false, 0, t + 1 == iters_next ? 2 : 1);
                rep.iterations += 1;
            }
        }
        if (tk_it >= 0) scope.saved->end("fb_iterate", tk_it, st);
        const int tk_rr = scope.saved ? scope.saved->begin(st) : -1;
        // Rayleigh-Ritz: Y = L U (into R), H = U^T Y
        SpmmParams sp;
        sp.n = n;
        sp.c = m;
        sp.batch = ws.B;
        sp.rowptr = ts.rowptr.get() + (int64_t)tile0 * (n + 1);
        sp.strideRowptr = (int64_t)tstride * (n + 1);
        sp.csr_offsets = ts.off.get() + tile0;  // per-batch offsets: stride tstride
        sp.cols = ts.cols.get();
        sp.vals = ts.vals.get();
        sp.X = ws.U.get();
        sp.ldx = ws.ld;
        sp.strideX = ws.mstride();
        sp.Y = ws.R.get();
        sp.ldy = ws.ld;
        sp.strideY = ws.mstride();
        sp.offStride = tstride;
        spmm(sp, st);
        GemmParams g;
        g.M = m;
        g.N = m;
        g.K = n;
        g.batch = ws.B;
        g.A = ws.U.get();
        g.lda = ws.ld;
        g.strideA = ws.mstride();
        g.B = ws.R.get();
        g.ldb = ws.ld;
        g.strideB = ws.mstride();
        g.C = ws.H.get();
        g.ldc = m;
        g.strideC = (int64_t)m * m;
        gemm(g, true, false, st);
        JacobiParams jp;
        jp.batch = ws.B;
        jp.H = ws.H.get();
        jp.ldh = m;
        jp.strideH = (int64_t)m * m;
        jp.stage = ws.Hst.get();
        jp.strideStage = pl.stage_elems;
        jp.V = ws.Vj.get();
        jp.ldv = m;
        jp.strideV = (int64_t)m * m;
        jp.theta = ws.theta.get();
        jp.theta_sorted = ws.theta_s.get();
        jp.strideTheta = m;
        jp.W = ws.Wm.get();
        jp.ldw = m;
        jp.strideW = (int64_t)m * m;
        DBuf<int> sweeps;
        sweeps.alloc(ws.B, st);
        jp.sweeps = sweeps.get();
        // the bootstrap round only plans the Chebyshev filter (interval ends, rate);
        // the filter input needs the span, not converged Ritz vectors
        if (round == 0 && use_cheb && c < m && m < n) {  // (m == n: this Rayleigh-Ritz is exact and final)
            jp.max_sweeps = 2;  // the Ritz values only plan the filter (interval ends, rate)
            if (const char* e = std::getenv("SMG_FB_BOOT_SWEEPS")) jp.max_sweeps = std::max(1, std::atoi(e));
        }
        const int jerr = jacobi_eigh(jp, pl, m, st);
        if (jerr != 0) SMG_CUDA((cudaError_t)jerr);
        if (std::getenv("SMG_DEBUG")) {
            std::vector<int> sw = download(sweeps.get(), ws.B, st);
            int mx = 0;
            for (int v : sw) mx = std::max(mx, v);
            std::fprintf(stderr, "[smg] jacobi m %d clusters %d x %d: max sweeps %d\n", m, ws.B, pl.nc, mx);
        }
        // Z = U W (into V), LZ = Y W (into T)
        gemm_nn(ws, ws.U.get(), ws.ld, ws.Wm.get(), m, (int64_t)m * m, ws.V.get(), n, m, m, st);
        gemm_nn(ws, ws.R.get(), ws.ld, ws.Wm.get(), m, (int64_t)m * m, ws.T.get(), n, m, m, st);
        ritz_residual(ws.T.get(), ws.V.get(), ws.theta_s.get(), n, nres, ws.ld, ws.mstride(), m, ws.B,
                      ws.ritz_part.get(), ws.ritz.get(), st);
        std::swap(ws.U, ws.V);
        if (tk_rr >= 0) scope.saved->end("fb_rayleigh_ritz", tk_rr, st);
        rep.rounds = round + 1;
        std::vector<double> th = download(ws.theta_s.get(), (size_t)ws.B * m, st);
        std::vector<double> rs = download(ws.ritz.get(), (size_t)ws.B * nres, st);
        std::vector<int> sts = download(ws.status.get(), ws.B, st);
        bool bad = false;
        for (int b = 0; b < ws.B; ++b) bad |= sts[b] != 0;
        if (bad) {
            // a filter planned from rough bootstrap Ritz values can over-amplify
            // (single-pass CholeskyQR breaks down): the caller retries shift-invert only
            if (use_cheb && broke) {
                *broke = true;
                return rep;
            }
            fail(3, "first-submesh basis: orthonormalization of the subspace iterate broke down");
        }
        double bound = 0.0, worst_rate = 0.0;
        for (int b = 0; b < ws.B; ++b) {
            const double* tb = th.data() + (size_t)b * m;
            const double* rb = rs.data() + (size_t)b * nres;
            double err = 0.0;
            for (int j = 0; j < c; ++j) err = std::max(err, rb[j]);
            const double gap = (c < m) ? tb[c] - tb[c - 1] : INFINITY;
            const double scale = std::max(std::fabs(tb[m - 1]), 1e-300);
            const double bb = (c < m) ? err / std::max(gap, 1e-16 * scale) : err / scale;
            bound = std::max(bound, bb);
            if (c < m) {
                const double s = fc.shift_hint;
                const double rate = std::pow((tb[c - 1] + s) / (tb[m - 1] + s), 2.0);
                worst_rate = std::max(worst_rate, rate);
            }
        }
        rep.bound = bound;
        if (std::getenv("SMG_DEBUG"))
            std::fprintf(stderr, "[smg] first_basis round %d: iterations %d bound %.3e rate %.3e m %d\n", round,
                         rep.iterations, bound, worst_rate, m);
        if (m == n || bound < fc.tol) break;
        if (!(bound < prev_bound * 0.999) && round >= 3) break;  // stagnated at the rounding floor
        prev_bound = bound;
        // Chebyshev plan from the Ritz values: cut a = theta_m, a0 = theta_1
        cheb_apps = 0;
        if (use_cheb && c < m) {
            std::vector<double> coef((size_t)2 * deg * ws.B + ws.B);
            double worst = 0.0;
            bool ok = true;
            for (int b = 0; b < ws.B && ok; ++b) {
                const double* tb = th.data() + (size_t)b * m;
                const double a = tb[m - 1], a0 = tb[0], up = upper[b];
                if (!(up > a && a > a0 && a > tb[c - 1])) {
                    ok = false;
                    break;
                }
                const double e = 0.5 * (up - a), cen = 0.5 * (up + a);
                const double sigma1 = e / (a0 - cen), tau = 2.0 / sigma1;
                double sigma = sigma1;
                coef[(size_t)0 * ws.B + b] = sigma1 / e;
                coef[(size_t)deg * ws.B + b] = 0.0;
                for (int i = 2; i <= deg; ++i) {
                    const double sn = 1.0 / (tau - sigma);
                    coef[(size_t)(i - 1) * ws.B + b] = 2.0 * sn / e;
                    coef[(size_t)deg * ws.B + (size_t)(i - 1) * ws.B + b] = -sigma * sn;
                    sigma = sn;
                }
                coef[(size_t)2 * deg * ws.B + b] = -cen;
                const double xi = std::fabs((tb[c - 1] - cen) / e);
                worst = std::max(worst, 1.0 / std::cosh(deg * std::acosh(std::max(xi, 1.0 + 1e-15))));
            }
            if (ok && worst < 0.5) {
                dcoef.upload(coef, st);
                // a conservative rate: eigenvalues between lambda_m and the cut are
                // amplified as well (and the bootstrap Ritz values are rough), so
                // count each application as worst^0.4 -- an extra filter application
                // is far cheaper than another Rayleigh-Ritz round
                const double need = std::log(fc.tol * 0.1 / bound) / std::log(std::pow(worst, 0.4));
                cheb_apps = (int)std::min(8.0, std::max(1.0, std::ceil(need)));
            }
        }
        if (cheb_apps == 0) {
            // shift-invert iterations to reach the tolerance at the observed rate
            double need = 4.0;
            // plan with a pessimistic rate (the early Ritz values overestimate the gap) so
            // that one more Rayleigh-Ritz round suffices
            if (worst_rate > 0.0 && worst_rate < 1.0)
                need = std::log(fc.tol * 0.1 / bound) / std::log(std::pow(worst_rate, 0.85));
            iters_next = (int)std::min(60.0, std::max(2.0, std::ceil(need)));
        }
        if (std::getenv("SMG_DEBUG"))
            std::fprintf(stderr, "[smg] first_basis plan: chebyshev applications %d (degree %d), si iterations %d\n",
                         cheb_apps, deg, cheb_apps ? 0 : iters_next);
    }
    return rep;
}
}  // namespace

FirstBasisReport first_basis(const StepCtx& cx, Workspace& ws, const TileSet& ts, int tile0, int tstride, int c,
                             const FirstBasisConfig& cfg, const FactorSet* op_factor) {
    bool broke = false;
    FirstBasisReport rep = first_basis_impl(cx, ws, ts, tile0, tstride, c, cfg, op_factor, true, &broke);
    if (!broke) return rep;
    ws.status.zero();
    return first_basis_impl(cx, ws, ts, tile0, tstride, c, cfg, op_factor, false, nullptr);
}

}  // namespace smg

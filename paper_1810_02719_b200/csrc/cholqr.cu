// K6: CholeskyQR building block -- blocked c x c Cholesky of the column-scaled
// Gram matrix with the reference rank test, and B = D^-1 R~^-1 so that the
// orthonormal factor is one triangular GEMM Q = V B (gemm.cu, upperB).
//
// orthonormalize (spectral.hpp:120-132) computes a Householder QR and throws
// "rank deficient at column k" for the first k with |r_kk| < 1e-13 ||block||_F.
// CholeskyQR gives the same R up to column signs: with D = diag(||v_j||) and
// G~ = D^-1 V^T V D^-1 = R~^T R~, R = R~ D, so |r_kk| = r~_kk d_k and ||block||_F
// = sqrt(trace G).  Column scaling keeps the column-graded blocks R^z U
// produces well conditioned (SURVEY.md §0 finding 5).  A scaled pivot below
// 1e-12 (r~_kk < 1e-6, beyond what the Gram resolves) is a rank-test failure
// at that column; columns that pass are re-tested exactly after the QR by
// rank_check (|q_k^T v_k| against the same threshold).
//
// chol_kernel: one CTA per chain, right-looking blocked Cholesky with 32-wide
// panels; the panel row sits in shared memory, its 32x32 diagonal block is
// factored and inverted by all threads (one barrier per column), the panel row solve and
// the trailing SYRK are 32x32x32 DMMA blocks on all warps; finally the block
// upper-triangular inverse X = R~^-1 is formed by block back-substitution
// (DMMA) and stored row-scaled as B = D^-1 X.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace smg {

#ifdef SMG_CHOL_TIMING
__device__ long long g_chol_t[128];
#define SMG_CHOL_T(i) \
    do { \
        if (threadIdx.x == 0 && blockIdx.x == 0) g_chol_t[(i)] = clock64(); \
    } while (0)
#else
#define SMG_CHOL_T(i) \
    do { \
    } while (0)
#endif

namespace {

#ifndef SMG_CHOL_SINGLE_BUFFER
#define SMG_CHOL_SINGLE_BUFFER 0
#endif
constexpr int CNT = 256;
constexpr int CW = CNT / 32;
constexpr int XS = 36;
constexpr int kMaxPanels = 16;  // c <= 512 (the library-wide column limit)  // 32-wide block stride (% 16 == 4: conflict-free fragments)

// 32x32x32 block product on one warp: acc(4x4 tiles of 8x8, 2 values) += op(A) * B
// with op(A)[m][k] = a(m, k), B[k][n] = b(k, n) supplied as functors.
template <class FA, class FB>
SMG_DEV void warp_block_mma(double (&acc)[4][4][2], FA a, FB b, int g, int t) {
#pragma unroll 2
    for (int kk = 0; kk < 32; kk += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = a(8 * i + g, kk + t);
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = b(kk + t, 8 * j + g);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
}

// back-substitution staging double-buffered when both per-warp buffers fit
__host__ __device__ constexpr bool chol_double_buffered(int c_cap) {
    return (32 * ((c_cap + 31) / 32 * 32 + 4) + 32 * XS + 2 * CW * 32 * XS + 2 * ((c_cap + 31) / 32 * 32)) * 8 <= 227 * 1024 &&
           !SMG_CHOL_SINGLE_BUFFER;
}

// cluster helpers (a launch without clusters is a cluster of one CTA)
SMG_DEV unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
SMG_DEV unsigned cl_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}
SMG_DEV void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
SMG_DEV void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
SMG_DEV void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

SMG_DEV void zero_acc(double (&acc)[4][4][2]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// Upper-triangle element ownership for the 32x32 diagonal block: the 528
// elements (i <= k) are enumerated row by row and thread t owns e = t, t + 256,
// t + 512 (at most three).
struct DiagOwn {
    int n = 0;
    int i[3], k[3];
    SMG_DEV void init(int tid) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            int e = tid + q * CNT;
            i[q] = k[q] = 0;
            if (e >= 528) continue;
            int r = 0;
            while (e >= 32 - r) {
                e -= 32 - r;
                ++r;
            }
            i[q] = r;
            k[q] = r + e;
            n = q + 1;
        }
    }
};

__global__ void __launch_bounds__(CNT) chol_kernel(CholParams p) {
    __shared__ double red[32];
    __shared__ double pivs[32];
    __shared__ double rinvd[32];  // 1 / r_ii of the current diagonal block
    __shared__ int fail;
    extern __shared__ __align__(16) double psm[];
    // single chains run on a cluster of CL CTAs: every CTA repeats the serial
    // diagonal-block phases (identical results), the panel row and the trailing
    // update -- the c^3 work -- are split over the cluster through global A
    const int CL = (int)cl_size(), rank = (int)cl_rank();
    const int b = blockIdx.x / CL;
    if (p.status[b] != kOk) return;  // sticky first error of this chain
    if (p.skip && p.skip[b]) return;  // adaptive pass 2: the pass-1 factor is orthonormal already
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int P = (c + 31) / 32, cp = P * 32;
    const double* G = p.G + (int64_t)b * p.strideG;
    SMG_CHOL_T(0);
    double* A = p.A + (int64_t)b * p.strideA;
    double* Bo = p.Binv + (int64_t)b * p.strideB;
    double* d = p.dscale + (int64_t)b * p.strideD;
    const int64_t lda = p.lda, ldb = p.ldb;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int PS = cp + 4;             // panel row stride (% 16 == 4: conflict-free fragments)
    double* Ps = psm;                  // 32 x PS panel row
    double* Xs = psm + 32 * PS;        // 32 x XS diagonal-block inverse
    double* Ts = Xs + 32 * XS;         // CW x 32 x XS per-warp staging
    double* ds = Ts + CW * 32 * XS;    // d_j (cp)
    double* rds = ds + cp;             // 1 / d_j (cp)

    double tr = 0.0;
    for (int j = tid; j < cp; j += CNT) {
        double dj = 1.0;
        if (j < c) {
            const double gjj = G[(int64_t)j * p.ldg + j];
            tr += gjj;
            dj = p.column_scale ? sqrt(gjj) : 1.0;
        }
        d[j] = dj;
        ds[j] = dj;
        rds[j] = dj > 0.0 ? 1.0 / dj : 0.0;
    }
    tr = block_sum(tr, red);
    const double scale = sqrt(tr);
    if (tid == 0) {
        fail = 0;
        if (p.vnorm) p.vnorm[b] = scale;
    }
    auto record = [&](int kind, int64_t col) {
        p.status[b] = kind;
        if (p.status_detail) p.status_detail[b] = col;
        if (p.errpos) p.errpos[b] = p.pos;
    };
    if (!(scale > 0.0) || !isfinite(scale)) {
        if (tid == 0) record(scale == 0.0 ? kAllZero : kNotFinite, -1);
        return;
    }
    const double thresh = 1e-13 * scale;
    __syncthreads();
    if (p.near_identity) {
        double e = 0.0, er = 0.0;
        for (int i = warp; i < c; i += CW)
            for (int k = i + lane; k < c; k += 32) {
                const double gik = G[(int64_t)i * p.ldg + k];
                const double x = fabs(fma(gik * rds[i], rds[k], (i == k) ? -1.0 : 0.0));
                const double xr = fabs(gik - ((i == k) ? 1.0 : 0.0));
                e = (x <= e) ? e : (x == x ? x : INFINITY);  // NaN -> full path
                er = (xr <= er) ? er : (xr == xr ? xr : INFINITY);
            }
        for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
        for (int o = 16; o > 0; o >>= 1) er = fmax(er, __shfl_xor_sync(0xffffffffu, er, o));
        __syncthreads();  // red[] is reused
        if (lane == 0) red[warp] = e;
        __syncthreads();
        e = red[0];
        for (int w = 1; w < CW; ++w) e = fmax(e, red[w]);
        __syncthreads();
        if (lane == 0) red[warp] = er;
        __syncthreads();
        er = red[0];
        for (int w = 1; w < CW; ++w) er = fmax(er, red[w]);
        if (p.skip_out) {
            const bool sk = er <= p.skip_tol;
            if (tid == 0) p.skip_out[b] = sk ? 1 : 0;
            if (sk) return;
        }
        if (e <= 1e-9) {
            for (int i = warp; i < cp; i += CW)
                for (int k = lane; k < cp; k += 32) {
                    double v = (k == i) ? 1.0 : 0.0;
                    if (k > i && k < c) v = -G[(int64_t)i * p.ldg + k] * rds[i] * rds[k];
                    Bo[(int64_t)i * ldb + k] = v * rds[i];
                }
            return;
        }
        __syncthreads();
    }
    // A = D^-1 G D^-1 (upper triangle incl. full diagonal 32-blocks); identity padding
    for (int i = warp; i < cp; i += CW) {
        const double ri = rds[i];
        const int k0 = (i & ~31) + lane;
        double v[kMaxPanels];
#pragma unroll
        for (int u = 0; u < kMaxPanels; ++u) {  // all loads of the row in flight at once
            const int k = k0 + 32 * u;
            v[u] = (k < cp && i < c && k < c) ? G[(int64_t)i * p.ldg + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kMaxPanels; ++u) {
            const int k = k0 + 32 * u;
            if (k < cp) A[(int64_t)i * lda + k] = (i < c && k < c) ? v[u] * ri * rds[k] : (i == k ? 1.0 : 0.0);
        }
    }
    DiagOwn own;
    own.init(tid);
    __syncthreads();
    if (CL > 1) cl_sync();  // every CTA's copy of A is written before any update
    SMG_CHOL_T(1);

    for (int pb = 0; pb < P; ++pb) {
        const int p0 = pb * 32;
        for (int r = warp; r < 32; r += CW)
            for (int k = p0 + lane; k < cp; k += 32) Ps[r * PS + k] = __ldcg(A + (int64_t)(p0 + r) * lda + k);
        __syncthreads();
        // cluster: this CTA's panel-row load is done; no CTA may overwrite the
        // panel row in A (diagonal block, panel-row blocks) before every CTA has
        // loaded it -- the matching wait sits just before the first store, so the
        // diagonal factor below hides the barrier
        if (CL > 1) cl_arrive();
        SMG_CHOL_T(2 + pb * 5);
        // ---- (a) factor the diagonal block with all threads (right-looking, LDL^T
        // form: the pivots are kept and the rows scaled at the end), then invert it.
        double* D = Ps + p0;  // D[i * PS + k]
        for (int j = 0; j < 32; ++j) {
            const double pj = D[j * PS + j];
            if (tid == 0) pivs[j] = pj;
            const double inv = 1.0 / fmax(pj, 1e-300);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (q < own.n && own.i[q] > j) {
                    const double l = D[j * PS + own.i[q]] * inv;
                    D[own.i[q] * PS + own.k[q]] = fma(-l, D[j * PS + own.k[q]], D[own.i[q] * PS + own.k[q]]);
                }
            }
            __syncthreads();
        }
        // rank test on the block's pivots, off the per-column critical path: first
        // failing column of the block (the pivots do not depend on the test)
        if (warp == 0) {
            const int gj = p0 + lane;
            bool badc = false, unsure = false;
            if (gj < c) {
                const double pj = pivs[lane];
                const bool bp = !(pj > (p.rank_test ? 1e-12 : 0.0)) || !isfinite(pj) || !(ds[gj] > 0.0);
                const double rkk = bp ? 0.0 : sqrt(pj) * ds[gj];
                badc = bp || (p.rank_test && rkk < thresh);
                unsure = p.rank_test && !bp && (pj < kRankCertPiv || rkk < kRankCertRel * scale);
            }
            if (p.rank_need && __any_sync(0xffffffffu, unsure) && lane == 0) atomicOr(p.rank_need + b, 1);
            const unsigned m = __ballot_sync(0xffffffffu, badc);
            if (lane == 0 && m) {
                record(p.rank_test ? kRankDeficient : kNotFinite, p0 + __ffs(m) - 1);
                fail = 1;
            }
            rinvd[lane] = 1.0 / sqrt(fmax(pivs[lane], 1e-300));
        }
        __syncthreads();
        if (fail) return;
        SMG_CHOL_T(3 + pb * 5);
        if (CL > 1) cl_wait();
        // rows scaled: R[i][k] = D[i][k] / sqrt(piv_i); X = R^-1 accumulators
        double xacc[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            xacc[q] = 0.0;
            if (q < own.n) {
                const int i = own.i[q], k = own.k[q];
                const double rii = sqrt(fmax(pivs[i], 1e-300));
                const double r = (i == k) ? rii : D[i * PS + k] * rinvd[i];
                D[i * PS + k] = r;
                A[(int64_t)(p0 + i) * lda + p0 + k] = r;
                xacc[q] = (i == k) ? 1.0 : 0.0;
            }
        }
        for (int e = tid; e < 32 * 32; e += CNT) {
            const int i = e >> 5, k = e & 31;
            if (i > k) Xs[i * XS + k] = 0.0;
        }
        __syncthreads();
        // X = R_pp^-1 by rows, bottom-up: X[l][k] = acc / R[l][l], then
        // acc[i][k] -= R[i][l] X[l][k] for i < l <= k
        for (int l = 31; l >= 0; --l) {
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (q < own.n && own.i[q] == l) Xs[l * XS + own.k[q]] = xacc[q] * rinvd[l];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (q < own.n && own.i[q] < l && own.k[q] >= l)
                    xacc[q] = fma(-D[own.i[q] * PS + l], Xs[l * XS + own.k[q]], xacc[q]);
        }
        __syncthreads();
        SMG_CHOL_T(4 + pb * 5);
        // ---- (b) panel row R_{p,q} = X^T A_{p,q}, q > p (smem operands, written back to smem and L2)
        for (int q = pb + 1 + rank + CL * warp; q < P; q += CL * CW) {
            const int q0 = q * 32;
            double acc[4][4][2];
            zero_acc(acc);
            warp_block_mma(
                acc, [&](int m, int k) { return Xs[k * XS + m]; }, [&](int k, int n) { return Ps[k * PS + q0 + n]; },
                g, t);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = 8 * i + g, cc = q0 + 8 * j + 2 * t;
                    Ps[r * PS + cc] = acc[i][j][0];
                    Ps[r * PS + cc + 1] = acc[i][j][1];
                    double* dst = A + (int64_t)(p0 + r) * lda + cc;
                    dst[0] = acc[i][j][0];
                    dst[1] = acc[i][j][1];
                }
        }
        // diagonal block of B: X_pp scaled by 1/d (rows), lower blocks of this row zero
        for (int r = warp; r < 32; r += CW) {
            Bo[(int64_t)(p0 + r) * ldb + p0 + lane] = Xs[r * XS + lane] * rds[p0 + r];
            for (int k = lane; k < p0; k += 32) Bo[(int64_t)(p0 + r) * ldb + k] = 0.0;
        }
        __syncthreads();
        if (CL > 1 && pb + 1 < P) {
            // the panel row blocks the other CTAs computed, through L2
            cl_sync();
            for (int q = pb + 1; q < P; ++q) {
                if ((q - pb - 1) % CL == rank) continue;
                for (int r = warp; r < 32; r += CW)
                    Ps[r * PS + q * 32 + lane] = __ldcg(A + (int64_t)(p0 + r) * lda + q * 32 + lane);
            }
            __syncthreads();
        }
        SMG_CHOL_T(5 + pb * 5);
        // ---- (c) trailing update A_{q,r} -= R_{p,q}^T R_{p,r}, p < q <= r
        const int rem = P - pb - 1;
        const int nblk = rem * (rem + 1) / 2;
        for (int e = rank + CL * warp; e < nblk; e += CL * CW) {
            int q = 0, rowlen = rem, acc_e = e;
            while (acc_e >= rowlen) {
                acc_e -= rowlen;
                ++q;
                --rowlen;
            }
            const int qq = pb + 1 + q, rr = qq + acc_e;
            const int q0 = qq * 32, r0 = rr * 32;
            double acc[4][4][2], old[4][4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i)  // the block's current values load while the product runs
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double2 o = __ldcg(reinterpret_cast<const double2*>(A + (int64_t)(q0 + 8 * i + g) * lda + r0 + 8 * j + 2 * t));
                    old[i][j][0] = o.x;
                    old[i][j][1] = o.y;
                }
            zero_acc(acc);
            warp_block_mma(
                acc, [&](int m, int k) { return Ps[k * PS + q0 + m]; },
                [&](int k, int n) { return Ps[k * PS + r0 + n]; }, g, t);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    double2* dst = reinterpret_cast<double2*>(A + (int64_t)(q0 + 8 * i + g) * lda + r0 + 8 * j + 2 * t);
                    *dst = make_double2(old[i][j][0] - acc[i][j][0], old[i][j][1] - acc[i][j][1]);
                }
        }
        __syncthreads();
        if (CL > 1) cl_sync();  // the trailing blocks of every CTA are in A before the next panel
        SMG_CHOL_T(6 + pb * 5);
    }
    if (p.skip_inverse) return;
    // block columns of X are independent: on a cluster each CTA back-substitutes
    // the columns q = rank (mod CL), no exchange needed (the diagonal blocks X_pp
    // every CTA wrote identically in (b))
    // ---- (d) X = R~^-1 by block back-substitution: X_pq = -X_pp sum_{s=p+1..q} R_ps X_sq.
    // B holds D^-1 X, so X_sq = d_row * B_sq on read.  R's panel row and X_pp sit
    // in shared memory; each X_sq block is staged into the warp's buffer with
    // one coalesced burst before its DMMA block product.
    double* Tw = Ts + warp * 32 * XS;
    // when shared memory allows, a second per-warp buffer lets the next X_sq
    // block stream in (cp.async) under the current block product; the d_row
    // scaling then happens on the operand read (same rounding as staging it)
    const bool dbl = chol_double_buffered(p.c_cap) && ((reinterpret_cast<uintptr_t>(p.Binv) & 15) == 0) &&
                     (ldb % 2 == 0) && (p.strideB % 2 == 0);
    double* Tw2 = rds + cp + warp * 32 * XS;
    for (int pb = P - 2; pb >= 0; --pb) {
        const int p0 = pb * 32;
        for (int r = warp; r < 32; r += CW) {
            for (int k = p0 + lane; k < cp; k += 32) Ps[r * PS + k] = A[(int64_t)(p0 + r) * lda + k];
            Xs[r * XS + lane] = Bo[(int64_t)(p0 + r) * ldb + p0 + lane] * ds[p0 + r];
        }
        __syncthreads();
        const int qfirst = pb + 1 + ((rank - (pb + 1)) % CL + CL) % CL;
        const int nown = qfirst < P ? (P - qfirst + CL - 1) / CL : 0;
        // cluster (few long chains, latency-bound): each column's s-sum is split
        // over S warps (s strided by S) and the part-0 warp adds the partials in
        // part order (deterministic).  Measured: c = 400 592 -> 516 us, c = 320
        // 384 -> 336 us; on one CTA at c = 200 the extra barrier costs more (222 -> 226 us)
        const int S = (CL > 1 && nown > 0 && nown <= CW / 2) ? min(CW / nown, 4) : 1;
        auto accumulate = [&](double(&acc)[4][4][2], int q0, int sb, int q) {
            if (sb > q) return;
            if (dbl) {
                // 16-byte copies: lane -> row (lane >> 4) of a row pair, columns 2 (lane & 15) +{0,1}
                auto stage = [&](double* buf, int s0) {
#pragma unroll
                    for (int k = 0; k < 32; k += 2) {
                        const int r = k + (lane >> 4), cc = 2 * (lane & 15);
                        cp_async16(buf + r * XS + cc, Bo + (int64_t)(s0 + r) * ldb + q0 + cc);
                    }
                    cp_async_commit();
                };
                stage(Tw, sb * 32);
                int it = 0;
                for (int s = sb; s <= q; s += S, ++it) {
                    const int s0 = s * 32;
                    double* cur = (it & 1) ? Tw2 : Tw;
                    double* nxt = (it & 1) ? Tw : Tw2;
                    __syncwarp();  // every lane is done reading nxt (the previous block)
                    if (s + S <= q) {
                        stage(nxt, s0 + 32 * S);
                        cp_async_wait<1>();
                    } else {
                        cp_async_wait<0>();
                    }
                    __syncwarp();
                    warp_block_mma(
                        acc, [&](int m, int k) { return Ps[m * PS + s0 + k]; },
                        [&](int k, int n) { return cur[k * XS + n] * ds[s0 + k]; }, g, t);
                }
            } else {
                for (int s = sb; s <= q; s += S) {
                    const int s0 = s * 32;
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 32; ++k) Tw[k * XS + lane] = Bo[(int64_t)(s0 + k) * ldb + q0 + lane] * ds[s0 + k];
                    __syncwarp();
                    warp_block_mma(
                        acc, [&](int m, int k) { return Ps[m * PS + s0 + k]; }, [&](int k, int n) { return Tw[k * XS + n]; },
                        g, t);
                }
            }
        };
        auto put = [&](const double(&acc)[4][4][2]) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    Tw[(8 * i + g) * XS + 8 * j + 2 * t] = acc[i][j][0];
                    Tw[(8 * i + g) * XS + 8 * j + 2 * t + 1] = acc[i][j][1];
                }
        };
        // X_pq = -X_pp (sum) scaled to B rows
        auto finish = [&](double(&acc)[4][4][2], int q0) {
            __syncwarp();
            put(acc);
            __syncwarp();
            zero_acc(acc);
            warp_block_mma(
                acc, [&](int m, int k) { return Xs[m * XS + k]; }, [&](int k, int n) { return Tw[k * XS + n]; }, g, t);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = p0 + 8 * i + g;
                    double* dst = Bo + (int64_t)r * ldb + q0 + 8 * j + 2 * t;
                    dst[0] = -acc[i][j][0] * rds[r];
                    dst[1] = -acc[i][j][1] * rds[r];
                }
            __syncwarp();
        };
        if (S == 1) {
            for (int q = qfirst + CL * warp; q < P; q += CL * CW) {
                double acc[4][4][2];
                zero_acc(acc);
                accumulate(acc, q * 32, pb + 1, q);
                finish(acc, q * 32);
            }
        } else {
            const int qi = warp % nown, part = warp / nown;
            const bool active = part < S;
            const int q = qfirst + CL * qi;
            double acc[4][4][2];
            zero_acc(acc);
            if (active) accumulate(acc, q * 32, pb + 1 + part, q);
            __syncwarp();
            if (active && part > 0) put(acc);
            __syncthreads();
            if (active && part == 0) {
                for (int pp = 1; pp < S; ++pp) {
                    const double* Tp = Ts + (qi + pp * nown) * 32 * XS;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            acc[i][j][0] += Tp[(8 * i + g) * XS + 8 * j + 2 * t];
                            acc[i][j][1] += Tp[(8 * i + g) * XS + 8 * j + 2 * t + 1];
                        }
                }
                finish(acc, q * 32);
            }
        }
        __syncthreads();
    }
    SMG_CHOL_T(127);
}

// The last chunk CTA of a chain (counter, threadfence reduction pattern) sums
// the chunk partials in chunk order -- deterministic -- and runs the test.
SMG_DEV void rank_test_block(const RankCheckParams& p, int b, int nchunks) {
    __shared__ int first;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    if (threadIdx.x == 0) first = c;
    __syncthreads();
    const double thresh = 1e-13 * p.vnorm[b];
    for (int k = threadIdx.x; k < c; k += blockDim.x) {
        // chunk order (deterministic); 16 loads issued ahead of their adds
        double r = 0.0;
        const double* src = p.partial + (int64_t)b * nchunks * p.c_cap + k;
        int ch = 0;
        for (; ch + 16 <= nchunks; ch += 16) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = __ldcg(src + (int64_t)(ch + u) * p.c_cap);
#pragma unroll
            for (int u = 0; u < 16; ++u) r += v[u];
        }
        for (; ch < nchunks; ++ch) r += __ldcg(src + (int64_t)ch * p.c_cap);
        if (!(fabs(r) >= thresh)) atomicMin(&first, k);
    }
    __syncthreads();
    if (threadIdx.x == 0 && first < c) {
        p.status[b] = kRankDeficient;
        if (p.status_detail) p.status_detail[b] = first;
        if (p.errpos) p.errpos[b] = p.pos;
    }
}

// partial diag(Q^T V) over a chunk of rows, threads over columns (coalesced rows)
constexpr int RC_ROWS = 32;
__global__ void rank_partial_kernel(RankCheckParams p) {
    const int b = blockIdx.y, chunk = blockIdx.x;
    if (p.status[b] != kOk) return;
    if (p.need && !p.need[b]) return;  // every column certified by the pass-1 pivots
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int r0 = chunk * RC_ROWS, r1 = min(p.n, r0 + RC_ROWS);
    const double* Q = p.Q + (int64_t)b * p.stride;
    const double* V = p.V + (int64_t)b * p.stride;
    for (int k = threadIdx.x; k < c; k += blockDim.x) {
        double acc = 0.0;
        if (r1 - r0 == RC_ROWS) {
            // full chunk: constant trip count so the loads are hoisted ahead of
            // the (unchanged, row-ordered) FMA chain -- latency, not bandwidth,
            // bound this kernel
            const double* q = Q + (int64_t)r0 * p.ld + k;
            const double* v = V + (int64_t)r0 * p.ld + k;
#pragma unroll 16
            for (int i = 0; i < RC_ROWS; ++i) acc = fma(q[(int64_t)i * p.ld], v[(int64_t)i * p.ld], acc);
        } else {
            for (int i = r0; i < r1; ++i) acc = fma(Q[(int64_t)i * p.ld + k], V[(int64_t)i * p.ld + k], acc);
        }
        p.partial[((int64_t)b * gridDim.x + chunk) * p.c_cap + k] = acc;
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&p.counter[b], 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    rank_test_block(p, b, gridDim.x);
    if (threadIdx.x == 0) p.counter[b] = 0;
}

// max over the upper triangle of |G - I| (one CTA per chain; independent
// loads, 8 in flight per thread) -> skip flag
__global__ void orth_check_kernel(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int64_t dimStride,
                                  int c_cap, double tol, int* skip) {
    __shared__ double red[32];
    const int b = blockIdx.x;
    const int c = dimC ? dimC[(int64_t)b * dimStride] : c_cap;
    const double* g = G + (int64_t)b * strideG;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double e = 0.0;
    // a warp per row (upper triangle), 8 independent loads in flight per lane
    for (int i = warp; i < c; i += nw) {
        const double* row = g + (int64_t)i * ldg;
        for (int k0 = i + lane; k0 < c; k0 += 256) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = k0 + 32 * u;
                v[u] = k < c ? fabs(__ldcg(row + k) - (i == k ? 1.0 : 0.0)) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) e = (v[u] <= e) ? e : (v[u] == v[u] ? v[u] : INFINITY);  // NaN -> no skip
        }
    }
    e = warp_max(e);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        skip[b] = (m <= tol) ? 1 : 0;
    }
}

// NEAR_ROWS rows per CTA (warp per row), the diagonal's reciprocal square
// roots staged once per CTA: max |G_ik / (d_i d_k) - delta_ik|, k >= i
constexpr int NEAR_ROWS = 8;
constexpr int NEAR_MAXC = 512;
__global__ void near_check_kernel(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int c_cap,
                                  unsigned long long* nmax) {
    __shared__ double rd[NEAR_MAXC];
    const int b = blockIdx.y;
    const int c = dimC ? dimC[b] : c_cap;
    const double* g = G + (int64_t)b * strideG;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x * NEAR_ROWS >= c) return;
    for (int k = threadIdx.x; k < c; k += blockDim.x) rd[k] = 1.0 / sqrt(__ldcg(g + (int64_t)k * ldg + k));
    __syncthreads();
    double e = 0.0;
    const int i = blockIdx.x * NEAR_ROWS + warp;
    if (i < c) {
        const double ri = rd[i];
        for (int k = i + lane; k < c; k += 32) {
            const double x = fabs(__ldcg(g + (int64_t)i * ldg + k) * ri * rd[k] - (i == k ? 1.0 : 0.0));
            e = (x <= e) ? e : (x == x ? x : INFINITY);
        }
    }
    e = warp_max(e);
    if (lane == 0 && e > 0.0) atomicMax(nmax + b, (unsigned long long)__double_as_longlong(e));
}

__global__ void near_fill_kernel(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int c_cap,
                                 const unsigned long long* nmax, const int* skip_in, int* skip_out, double* Bo,
                                 int64_t ldb, int64_t strideB, double* dscale, int64_t strideD) {
    const int b = blockIdx.y;
    const bool skipped = skip_in && skip_in[b];
    const double m = __longlong_as_double((long long)nmax[b]);
    const bool near = !skipped && m <= 1e-9;
    if (blockIdx.x == 0 && threadIdx.x == 0) skip_out[b] = (skipped || near) ? 1 : 0;
    if (!near) return;
    const int c = dimC ? dimC[b] : c_cap;
    const int cp = (c_cap + 31) / 32 * 32;
    const double* g = G + (int64_t)b * strideG;
    double* B = Bo + (int64_t)b * strideB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x * NEAR_ROWS >= cp) return;
    __shared__ double rd[NEAR_MAXC];
    for (int k = threadIdx.x; k < c; k += blockDim.x) rd[k] = 1.0 / sqrt(__ldcg(g + (int64_t)k * ldg + k));
    __syncthreads();
    const int i = blockIdx.x * NEAR_ROWS + warp;
    if (i < cp) {
        const double di = i < c ? sqrt(__ldcg(g + (int64_t)i * ldg + i)) : 1.0;
        const double ri = di > 0.0 ? 1.0 / di : 0.0;
        if (lane == 0) dscale[(int64_t)b * strideD + i] = di;
        for (int k = lane; k < cp; k += 32) {
            double v = (k == i) ? 1.0 : 0.0;
            if (k > i && k < c) v = -__ldcg(g + (int64_t)i * ldg + k) * ri * rd[k];
            B[(int64_t)i * ldb + k] = v * ri;
        }
    }
}

__global__ void copy_unskipped_kernel(const double* src, double* dst, int64_t elems, int64_t stride, const int* skip) {
    const int b = blockIdx.y;
    if (skip[b]) return;
    const double2* s = reinterpret_cast<const double2*>(src + (int64_t)b * stride);
    double2* d = reinterpret_cast<double2*>(dst + (int64_t)b * stride);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < elems / 2; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}

}  // namespace

void orth_check(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int64_t dimStride, int c_cap,
                int batch, double tol, int* skip, cudaStream_t st) {
    ::smg::count_launch(), orth_check_kernel<<<batch, 256, 0, st>>>(G, ldg, strideG, dimC, dimStride, c_cap, tol, skip);
}

void near_check(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int c_cap, int batch,
                unsigned long long* nmax, cudaStream_t st) {
    const int nb = (c_cap + NEAR_ROWS - 1) / NEAR_ROWS;
    ::smg::count_launch(), near_check_kernel<<<dim3(nb, batch), 32 * NEAR_ROWS, 0, st>>>(G, ldg, strideG, dimC, c_cap, nmax);
}

void near_fill(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int c_cap, int batch,
               const unsigned long long* nmax, const int* skip_in, int* skip_out, double* Binv, int64_t ldb,
               int64_t strideB, double* dscale, int64_t strideD, cudaStream_t st) {
    const int nb = ((c_cap + 31) / 32 * 32 + NEAR_ROWS - 1) / NEAR_ROWS;
    ::smg::count_launch(), near_fill_kernel<<<dim3(nb, batch), 32 * NEAR_ROWS, 0, st>>>(
        G, ldg, strideG, dimC, c_cap, nmax, skip_in, skip_out, Binv, ldb, strideB, dscale, strideD);
}

void copy_unskipped(const double* src, double* dst, int64_t elems, int64_t stride, int batch, const int* skip,
                    cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(64, (elems / 2 + 255) / 256);
    ::smg::count_launch(), copy_unskipped_kernel<<<dim3(std::max(blocks, 1), batch), 256, 0, st>>>(src, dst, elems, stride, skip);
}

void rank_check(const RankCheckParams& p, cudaStream_t st) {
    const int chunks = (p.n + RC_ROWS - 1) / RC_ROWS;
    // threads over columns: no idle warps at c = 200 (224 threads)
    const int threads = std::min(256, std::max(32, (p.c_cap + 31) / 32 * 32));
    ::smg::count_launch(), rank_partial_kernel<<<dim3(chunks, p.batch), threads, 0, st>>>(p);
}

int chol_smem_bytes(int c_cap) {
    const int cp = (c_cap + 31) / 32 * 32;
    return (32 * (cp + 4) + 32 * XS + (chol_double_buffered(c_cap) ? 2 : 1) * CW * 32 * XS + 2 * cp) * 8;
}

void chol_factor(const CholParams& p, cudaStream_t st) {
    if (cholx_factor(p, st)) return;
    const int bytes = chol_smem_bytes(p.c_cap);
    ensure_smem((const void*)chol_kernel, bytes);
    // a few chains with c > 224: a cluster of 4 CTAs per chain splits the panel
    // rows and trailing updates (single-chain configs are bound by this kernel)
    const int P = (p.c_cap + 31) / 32;
    static const int minp = std::getenv("SMG_CHOL_CLUSTER_MINP") ? std::atoi(std::getenv("SMG_CHOL_CLUSTER_MINP")) : 8;
    static const int maxb = std::getenv("SMG_CHOL_CLUSTER_MAXB") ? std::atoi(std::getenv("SMG_CHOL_CLUSTER_MAXB")) : 4;
    const bool cluster = p.batch <= maxb && P >= minp && !std::getenv("SMG_CHOL_NOCLUSTER");
    if (!cluster) {
        ::smg::count_launch(), chol_kernel<<<p.batch, CNT, bytes, st>>>(p);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.batch * 4);
    cfg.blockDim = dim3(CNT);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 4;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ::smg::count_launch();
    cudaLaunchKernelEx(&cfg, chol_kernel, p);
}

}  // namespace smg

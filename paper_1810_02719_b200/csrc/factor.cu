// K2: factorisation of L + delta I for every submesh, batched (one CTA per tile).
//
// Replaces the ShiftedInverseOperator constructor (spectral.hpp:147-159:
// `shifted = L + delta*I; SimplicialLDLT::compute`).  Eigen's LDL^T does no
// pivoting and accepts negative pivots (only an exact zero pivot is a
// NumericalIssue); the same algebra is kept as a *signed* block Cholesky
// A = L Sigma L^T (Sigma = diag(+-1)) so indefinite matrices behave the same.
//
// In the chosen ordering (natural for grid tiles, RCM otherwise) the matrix is
// block tridiagonal with W x W blocks D_k (diagonal) and B_k = A_{k,k-1}:
//   L_{k,k-1} = B_k Linv_{k-1}^T Sigma_{k-1}
//   S_k       = D_k - L_{k,k-1} Sigma_{k-1} L_{k,k-1}^T
//   S_k       = L_kk Sigma_k L_kk^T            (signed Cholesky, zero pivot fails)
// and the solve operands are written once per tile:
//   Ffwd_k^T = [Linv_k | -Linv_k L_{k,k-1}]^T
//   Fbwd_k^T = [Linv_k^T Sigma_k | -Linv_k^T L_{k+1,k}^T]^T
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int NT_DEFAULT = 256;
// threads per CTA: the W = 32 factor is barrier-latency bound (a barrier per column), so it runs
// 128-thread CTAs (cheaper barriers; 93 registers, five CTAs per SM: C5 309.2 -> 306.8 ms; forcing
// eight per SM at 63 registers was slower, 314 ms) unless SMG_FACTOR_NT256 is defined
#ifdef SMG_FACTOR_NT256
template <int W> struct FThreads { static constexpr int value = NT_DEFAULT; };
#else
template <int W> struct FThreads { static constexpr int value = W == 32 ? 128 : NT_DEFAULT; };
#endif

// Shared memory: three W x W matrices (S, P and L, where L holds Linv_{k-1}
// until -P Linv_{k-1} is written and then receives Linv_k), the coupling lists
// with a runtime stride (cpl = bound on a row's lower neighbours, from the
// ordering pass) and the inverse permutation only for RCM-ordered tiles -- at
// W = 64 in natural order that is ~106 KB, two CTAs per SM.
template <int W>
struct FactorSmem {
    static constexpr int LD = W + 4;  // LD % 16 == 4: conflict-free DMMA fragment reads
    static constexpr int MAT = W * LD;
    static int bytes(int n, int cpl, bool permuted) {
        return (3 * MAT + 5 * W + 32) * 8 + (permuted ? ((n + 1) & ~1) * 4 : 0) + W * cpl * (8 + 4) + W * 4;
    }
};

// C (W x W, DMMA accumulators of one warp's 2x(W/16)... tiles) helpers.
// Warps tile the W x W output as a 4 x 2 grid of (W/32 x W/16) 8x8 tiles.
template <int W>
struct FTile {
    // 8x8 tiles per warp: W=16 1x1 (4 warps), 32 1x2 (8), 48 2x3 (6), 64 2x4 (8)
    static constexpr int MT = (W == 48 || W == 64) ? 2 : 1;
    static constexpr int NTT = W == 16 ? 1 : (W == 32 ? (FThreads<32>::value == 128 ? 4 : 2) : (W == 48 ? 3 : 4));
    static constexpr int WMG = (W / 8) / MT;  // warps along m
    static constexpr int WNG = (W / 8) / NTT; // warps along n
    static constexpr int ACTIVE = WMG * WNG;
};

// acc[i][j] += sum_k A(m, k) * B(k, n) over k in [k0, k1), A/B as functors of
// (row, col) returning smem values; m = 8*(wm*MT+i)+g, n = 8*(wn*NT+j)+g.
template <int W, class FA, class FB, class FSkip>
SMG_DEV void fblock_mma(double (&acc)[FTile<W>::MT][FTile<W>::NTT][2], FA a, FB b, FSkip skip, int wm, int wn,
                        int g, int t) {
    constexpr int MT = FTile<W>::MT, NT = FTile<W>::NTT;
#pragma unroll 2
    for (int kk = 0; kk < W; kk += 4) {
        double av[MT], bv[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) bv[j] = b(kk + t, 8 * (wn * NT + j) + g);
#pragma unroll
        for (int i = 0; i < MT; ++i) av[i] = a(8 * (wm * MT + i) + g, kk + t);
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            if (skip(wm * MT + i, kk)) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
        }
    }
}

template <int W>
__global__ void __launch_bounds__((FThreads<W>::value)) factor_kernel(FactorParams p) {
    constexpr int NT = FThreads<W>::value;
    constexpr int LD = FactorSmem<W>::LD;
    constexpr int MAT = FactorSmem<W>::MAT;
    extern __shared__ __align__(16) double sm[];
    double* S = sm;              // Schur complement / L_kk (lower)
    double* P = sm + MAT;        // L_{k,k-1}
    double* Lp = sm + 2 * MAT;   // Linv_{k-1}, then (same buffer) Linv_k
    double* Lc = Lp;
    double* sig = sm + 3 * MAT;  // Sigma_k
    double* sigp = sig + W;      // Sigma_{k-1}
    double* piv = sigp + W;      // pivots of the current block
    double* rsc = piv + W;       // 1 / (l_jj sigma_j)
    double* rdv = rsc + W;       // pivot reciprocals, published by the diagonal's owner
    int* flag = reinterpret_cast<int*>(rdv + W);
    const int CPL = p.cpl;
    int* ipos = reinterpret_cast<int*>(rdv + W + 32);                                  // RCM only
    double* cval = reinterpret_cast<double*>(ipos + (p.perm ? ((p.n + 1) & ~1) : 0));  // [W][CPL]
    int* cidx = reinterpret_cast<int*>(cval + W * CPL);                                // [W][CPL]
    int* ccnt = cidx + W * CPL;                                                        // [W]
    using FT = FTile<W>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = warp % FT::WMG, wn = warp / FT::WMG;
    const bool mma_warp = warp < FT::ACTIVE;

    const int tile = blockIdx.x;
    const int n = p.n, Kb = p.Kb, tid = threadIdx.x;
    const int32_t* rowptr = p.rowptr + (int64_t)tile * (n + 1);
    const int64_t base = p.csr_offsets[tile];
    const int32_t* cols = p.cols + base;
    const double* vals = p.vals + base;
    const int32_t* perm = p.perm ? p.perm + (int64_t)tile * n : nullptr;
    const double delta = p.delta[tile];
    double* Ff = p.Ffwd + (int64_t)tile * p.strideF;
    double* Fb = p.Fbwd + (int64_t)tile * p.strideF;
    constexpr int FR = factor_row(W);
    const int64_t slab = (int64_t)2 * W * FR;

    if (perm)
        for (int i = tid; i < n; i += NT) ipos[perm[i]] = i;
    if (tid == 0) flag[0] = 0;
    // ownership of the W x W upper triangle (a <= b), enumerated row by row
    constexpr int NOWN = (W * (W + 1) / 2 + NT - 1) / NT;
    int own_a[NOWN], own_b[NOWN], nown = 0;
#pragma unroll
    for (int q = 0; q < NOWN; ++q) {
        int e = tid + q * NT, a = 0;
        own_a[q] = own_b[q] = 0;
        if (e >= W * (W + 1) / 2) continue;
        while (e >= W - a) {
            e -= W - a;
            ++a;
        }
        own_a[q] = a;
        own_b[q] = a + e;
        nown = q + 1;
    }
    __syncthreads();

    for (int k = 0; k < Kb; ++k) {
        const int r0 = k * W;
        // ---- D_k (+ delta on the diagonal, Eigen: shifted += delta * identity)
        for (int e = tid; e < W * W; e += NT) S[(e / W) * LD + (e % W)] = 0.0;
        __syncthreads();
        // one scan of the block's CSR rows: D_k entries and the coupling B_k into block k-1
        for (int r = tid; r < W; r += NT) {
            const int prow = r0 + r;
            int cnt = 0;
            if (prow >= n) {
                S[r * LD + r] = 1.0;
            } else {
                const int i = perm ? perm[prow] : prow;
                for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                    const int pq = perm ? ipos[cols[e]] : cols[e];
                    const int q = pq - r0;
                    if (q >= 0 && q < W) {
                        S[r * LD + q] = (cols[e] == i) ? vals[e] + delta : vals[e];
                    } else if (q >= -W && q < 0) {
                        if (cnt < CPL) {
                            cidx[r * CPL + cnt] = q + W;
                            cval[r * CPL + cnt] = vals[e];
                        }
                        ++cnt;
                    } else if (q < -W || q >= 2 * W) {
                        flag[0] = 2;  // not block tridiagonal at this width
                    }
                }
            }
            ccnt[r] = cnt;
            if (cnt > CPL) flag[0] = 2;
        }
        __syncthreads();
        if (k > 0) {
            // ---- P = B_k Linv_{k-1}^T Sigma_{k-1}  (= L_{k,k-1}), B_k sparse
            for (int e = tid; e < W * W; e += NT) {
                const int r = e / W, c = e % W;
                const int cnt = min(ccnt[r], CPL);
                double acc = 0.0;
                for (int q = 0; q < cnt; ++q) {
                    const int qq = cidx[r * CPL + q];
                    if (c >= qq) acc += cval[r * CPL + q] * Lp[c * LD + qq];
                }
                P[r * LD + c] = acc * sigp[c];
            }
            __syncthreads();
        // ---- Fbwd_{k-1}^T second half: -(L_{k,k-1} Linv_{k-1}) = -(P Lp), row-major
        if (mma_warp) {
            double* Fp = Fb + (int64_t)(k - 1) * slab;
            double acc[FT::MT][FT::NTT][2] = {};
            fblock_mma<W>(
                acc, [&](int m, int kk) { return P[m * LD + kk]; }, [&](int kk, int nn) { return Lp[kk * LD + nn]; },
                [](int, int) { return false; }, wm, wn, g, t4);
#pragma unroll
            for (int i = 0; i < FT::MT; ++i)
#pragma unroll
                for (int j = 0; j < FT::NTT; ++j) {
                    const int r = 8 * (wm * FT::MT + i) + g, jj = 8 * (wn * FT::NTT + j) + 2 * t4;
                    double2* dst = reinterpret_cast<double2*>(Fp + (int64_t)(W + r) * FR + jj);
                    *dst = make_double2(-acc[i][j][0], -acc[i][j][1]);
                }
        }

            // ---- S -= P Sigma_{k-1} P^T  (DMMA; full block, the lower triangle is used)
            if (mma_warp) {
                double acc[FT::MT][FT::NTT][2] = {};
                fblock_mma<W>(
                    acc, [&](int m, int kk) { return P[m * LD + kk]; },
                    [&](int kk, int nn) { return P[nn * LD + kk] * sigp[kk]; }, [](int, int) { return false; }, wm, wn,
                    g, t4);
#pragma unroll
                for (int i = 0; i < FT::MT; ++i)
#pragma unroll
                    for (int j = 0; j < FT::NTT; ++j) {
                        const int r = 8 * (wm * FT::MT + i) + g, s = 8 * (wn * FT::NTT + j) + 2 * t4;
                        S[r * LD + s] -= acc[i][j][0];
                        S[r * LD + s + 1] -= acc[i][j][1];
                    }
            }
        }
        __syncthreads();
        // ---- signed Cholesky S = L Sigma L^T, right-looking in LDL^T form on the
        // upper triangle (row j is read contiguously): every thread updates the
        // elements it owns, one barrier per column; pivots kept, rows scaled at the end
        // 1 / d of column j + 1 is computed once, by the owner of that diagonal
        // element right after its last update, and read by everyone after the
        // barrier (a double division per thread per column dominated the loop)
        const double rd0 = 1.0 / S[0];
        for (int j = 0; j < W; ++j) {
            const double d = S[j * LD + j];
            if (tid == 0) {
                if (!(d != 0.0) || !isfinite(d)) flag[0] = 1;
                piv[j] = d;
            }
            const double rd = j == 0 ? rd0 : rdv[j];
#pragma unroll
            for (int q = 0; q < NOWN; ++q) {
                const int a = own_a[q], b = own_b[q];
                if (q < nown && a > j) {
                    S[a * LD + b] = fma(-S[j * LD + a] * rd, S[j * LD + b], S[a * LD + b]);
                    if (a == j + 1 && b == a) rdv[a] = 1.0 / S[a * LD + a];
                }
            }
            __syncthreads();
        }
        // L (lower) = scaled transpose of the upper rows; Sigma = sign(pivots)
#pragma unroll
        for (int q = 0; q < NOWN; ++q) {
            if (q >= nown) continue;
            const int a = own_a[q], b = own_b[q];
            const double d = piv[a];
            const double la = sqrt(fabs(d));
            if (a == b) {
                S[a * LD + a] = la;
                rdv[a] = 1.0 / la;  // 1 / l_aa for the inverse below (after the next barrier)
            } else {
                S[b * LD + a] = S[a * LD + b] / (la * (d < 0.0 ? -1.0 : 1.0));
            }
        }
        for (int e = tid; e < W; e += NT) {
            sig[e] = piv[e] < 0.0 ? -1.0 : 1.0;
            rsc[e] = 1.0 / (sqrt(fabs(piv[e])) * (piv[e] < 0.0 ? -1.0 : 1.0));
        }
        // ---- Linv_k = L_kk^-1 by rows (update form, X[b][a] accumulated by the owner of (a, b))
        for (int e = tid; e < W * W; e += NT) Lc[(e / W) * LD + (e % W)] = 0.0;
        __syncthreads();
        {
            double xacc[NOWN];
#pragma unroll
            for (int q = 0; q < NOWN; ++q) xacc[q] = (q < nown && own_a[q] == own_b[q]) ? 1.0 : 0.0;
            for (int i = 0; i < W; ++i) {
                const double rii = rdv[i];
#pragma unroll
                for (int q = 0; q < NOWN; ++q)
                    if (q < nown && own_b[q] == i) Lc[i * LD + own_a[q]] = xacc[q] * rii;
                __syncthreads();
                const double ri = rsc[i];
#pragma unroll
                for (int q = 0; q < NOWN; ++q) {
                    const int a = own_a[q], b = own_b[q];
                    // L[b][i] = U_raw[i][b] / (l_ii sigma_i), read from the upper row i
                    if (q < nown && b > i && a <= i) xacc[q] = fma(-S[i * LD + b] * ri, Lc[i * LD + a], xacc[q]);
                }
            }
        }
        __syncthreads();
        // ---- Ffwd_k^T: rows j<W: Linv_k[:, j]; rows W+j: -M_k[:, j], M_k = Linv_k P
        double* F = Ff + (int64_t)k * slab;
        for (int e = tid; e < W * W; e += NT) {
            const int j = e / W, r = e % W;
            F[(int64_t)j * FR + r] = Lc[r * LD + j];
        }
        if (mma_warp) {
            double acc[FT::MT][FT::NTT][2] = {};
            if (k > 0)  // M_k = Linv_k P (Linv_k lower: skip k-slices right of the m-tile)
                fblock_mma<W>(
                    acc, [&](int m, int kk) { return Lc[m * LD + kk]; },
                    [&](int kk, int nn) { return P[kk * LD + nn]; },
                    [](int ti, int kk) { return kk >= 8 * ti + 8; }, wm, wn, g, t4);
            // stored transposed: F[W + j][r] = -M[r][j]
#pragma unroll
            for (int i = 0; i < FT::MT; ++i)
#pragma unroll
                for (int j = 0; j < FT::NTT; ++j)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int r = 8 * (wm * FT::MT + i) + g, jj = 8 * (wn * FT::NTT + j) + 2 * t4 + q;
                        F[(int64_t)(W + jj) * FR + r] = -acc[i][j][q];
                    }
        }
        // ---- Fbwd_k^T first half: row j = sigma_j * Linv_k[j, :]
        {
            double* Fc = Fb + (int64_t)k * slab;
            for (int e = tid; e < W * W; e += NT) {
                const int j = e / W, r = e % W;
                Fc[(int64_t)j * FR + r] = sig[j] * Lc[j * LD + r];
            }
            if (k == Kb - 1)
                for (int e = tid; e < W * W; e += NT) Fc[(int64_t)(W + e / W) * FR + e % W] = 0.0;
        }
        __syncthreads();
        // ---- carry Sigma_k (Linv_k already sits in the L buffer)
        for (int e = tid; e < W; e += NT) sigp[e] = sig[e];
        __syncthreads();
    }
    if (tid == 0 && p.status) p.status[tile] = flag[0] ? kFactorFailed : kOk;
}

template <int W>
void launch(const FactorParams& p, cudaStream_t st) {
    const int bytes = FactorSmem<W>::bytes(p.n, p.cpl, p.perm != nullptr);
    cudaFuncSetAttribute(factor_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    ::smg::count_launch(), factor_kernel<W><<<p.ntiles, FThreads<W>::value, bytes, st>>>(p);
}

}  // namespace

int factor_smem_bytes(int W) {
    switch (W) {
        case 16: return FactorSmem<16>::bytes(0, 16, false);
        case 32: return FactorSmem<32>::bytes(0, 16, false);
        case 48: return FactorSmem<48>::bytes(0, 16, false);
        default: return FactorSmem<64>::bytes(0, 16, false);
    }
}

void factor_tiles(const FactorParams& p, cudaStream_t st) {
    if (p.ntiles == 0) return;
    switch (p.W) {
        case 16: launch<16>(p, st); break;
        case 32: launch<32>(p, st); break;
        case 48: launch<48>(p, st); break;
        case 64: launch<64>(p, st); break;
        default: break;
    }
}

}  // namespace smg

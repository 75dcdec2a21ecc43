// K3: R^z U = ((L + delta I)^-1)^z U for a block of c columns.
//
// Replaces ShiftedInverseOperator::apply / apply_once (spectral.hpp:166-176,
// z SimplicialLDLT solves).  L + delta I = L Sigma L^T is factored in block
// tridiagonal form with W x W blocks (factor.cu), so one triangular sweep is a
// recurrence over the Kb = n_pad / W blocks:
//   forward   y_k = [Linv_k | -M_k] [b_k ; y_{k-1}]
//   backward  x_k = [Linv_k^T Sigma_k | -N_k] [y_k ; x_{k+1}]
// Every step is one (W x 2W) * (2W x CS) product on the DMMA pipe.  Columns are
// independent through all 2z sweeps, so each CTA owns a slice of CS columns of
// one chain and runs every sweep with only CTA barriers; no grid-wide sync.
// The W x 2W factor slab of the next block streams into shared memory with
// cp.async while the current one is multiplied (double buffer).
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int NT = 256;
constexpr int kSolveWarps = NT / 32;

template <int W, int CS>
struct SolveSmem {
    static constexpr int FS = W + 4;   // padded row of the transposed factor slab
    static constexpr int XS = CS + 4;  // padded row of the right-hand-side slab
    static constexpr int F_ELEMS = 2 * W * FS;
    static constexpr int X_ELEMS = 2 * W * XS;
    static constexpr int BYTES = (2 * F_ELEMS + 2 * X_ELEMS) * 8;
};

// zero-fill variant: src_bytes = 0 writes zeros
SMG_DEV void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

// Warp tiling of the W x CS step output: warps form a WM x WN grid, each owns
// MT x NT tiles of 8x8, so per k-slice it loads MT + NT operand fragments for
// MT * NT DMMAs (shared-memory traffic, not the DMMA pipe, bounds this loop).
template <int W, int CS>
struct SolveTiling {
    static constexpr int MT_ALL = W / 8, NT_ALL = CS / 8;
    // 8 warps (two per SM sub-partition hide the DMMA issue latency); prefer a
    // 4 x 2 warp grid, a full m-column of warps when there is one n-tile
    static constexpr int NW = kSolveWarps;
    static constexpr int WM = (NT_ALL == 1) ? (MT_ALL < NW ? MT_ALL : NW)
                                            : ((MT_ALL % 4 == 0) ? 4 : ((MT_ALL % 2 == 0) ? 2 : 1));
    static constexpr int WN_RAW = NW / WM;
    static constexpr int WN = (NT_ALL % WN_RAW == 0) ? WN_RAW
                                                     : ((NT_ALL % 4 == 0 && WN_RAW >= 4) ? 4 : ((NT_ALL % 2 == 0 && WN_RAW >= 2) ? 2 : 1));
    static constexpr int MT = MT_ALL / WM, NT = NT_ALL / WN;
    static constexpr int ACTIVE = WM * WN;
    // Row-tile of the warp's i-th m tile.  The first half of every step is a
    // triangular block, so contiguous row tiles would give the bottom warps up
    // to 4x the DMMAs of the top ones; pairing tile r with MT_ALL-1-r balances
    // every warp (and so every SM sub-partition).
    static constexpr bool PAIRED = (MT == 2 && MT_ALL == 2 * WM);
    SMG_DEV static int tile(int wm, int i) { return PAIRED ? (i == 0 ? wm : MT_ALL - 1 - wm) : wm * MT + i; }
};

template <int W, int CS, bool FWD>
SMG_DEV void mma_step(const double* __restrict__ fs, const double* __restrict__ xs,
                      double (&acc)[SolveTiling<W, CS>::MT][SolveTiling<W, CS>::NT][2], int warp, int g, int t,
                      bool skip_second) {
    using TL = SolveTiling<W, CS>;
    constexpr int MT = TL::MT, NT = TL::NT;
    constexpr int FS = SolveSmem<W, CS>::FS;
    constexpr int XS = SolveSmem<W, CS>::XS;
    const int wm = warp % TL::WM, wn = warp / TL::WM;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (warp >= TL::ACTIVE) return;
    // first half: triangular block (Linv_k lower for FWD, Linv_k^T Sigma upper for BWD)
    if constexpr (TL::PAIRED) {
        // row tiles lo = wm and hi = MT_ALL-1-wm; the k ranges where a tile's
        // block is nonzero are loop bounds, not predicates (a predicated-off
        // DMMA still occupies the pipe): FWD tile r needs kk < 8r+8, BWD kk >= 8r
        const int lo = wm, hi = TL::MT_ALL - 1 - wm;
        auto both = [&](int k0, int k1) {
#pragma unroll 2
            for (int kk = k0; kk < k1; kk += 4) {
                double a0, a1, b[NT];
#pragma unroll
                for (int j = 0; j < NT; ++j) b[j] = xs[(kk + t) * XS + 8 * (wn * NT + j) + g];
                a0 = fs[(kk + t) * FS + 8 * lo + g];
                a1 = fs[(kk + t) * FS + 8 * hi + g];
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    dmma884(acc[0][j][0], acc[0][j][1], a0, b[j]);
                    dmma884(acc[1][j][0], acc[1][j][1], a1, b[j]);
                }
            }
        };
        auto one = [&](int k0, int k1, int i, int r) {
#pragma unroll 2
            for (int kk = k0; kk < k1; kk += 4) {
                double b[NT];
#pragma unroll
                for (int j = 0; j < NT; ++j) b[j] = xs[(kk + t) * XS + 8 * (wn * NT + j) + g];
                const double a = fs[(kk + t) * FS + 8 * r + g];
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a, b[j]);
            }
        };
        if (FWD) {
            both(0, 8 * lo + 8);
            one(8 * lo + 8, 8 * hi + 8, 1, hi);
        } else {
            one(8 * lo, 8 * hi, 0, lo);
            both(8 * hi, W);
        }
    } else {
#pragma unroll 2
    for (int kk = 0; kk < W; kk += 4) {
        double b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = xs[(kk + t) * XS + 8 * (wn * NT + j) + g];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int ti = TL::tile(wm, i);
            const bool nz = FWD ? (kk < 8 * ti + 8) : (kk + 4 > 8 * ti);
            if (!nz) continue;
            const double a = fs[(kk + t) * FS + 8 * ti + g];
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a, b[j]);
        }
    }
    }
    if (skip_second) return;
#pragma unroll 2
    for (int kk = W; kk < 2 * W; kk += 4) {
        double a[MT], b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = xs[(kk + t) * XS + 8 * (wn * NT + j) + g];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = fs[(kk + t) * FS + 8 * TL::tile(wm, i) + g];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

template <int W, int CS>
__global__ void __launch_bounds__(NT) solve_kernel(SolveParams p) {
    using S = SolveSmem<W, CS>;
    using TL = SolveTiling<W, CS>;
    constexpr int FS = S::FS, XS = S::XS;
    extern __shared__ __align__(16) double smem[];
    double* Fs[2] = {smem, smem + S::F_ELEMS};
    double* Xs[2] = {smem + 2 * S::F_ELEMS, smem + 2 * S::F_ELEMS + S::X_ELEMS};

    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int col0 = blockIdx.x * CS;
    if (col0 >= c) return;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int n = p.n, Kb = p.Kb;
    const int64_t slab = (int64_t)2 * W * W;  // doubles per block in Ffwd/Fbwd
    const double* Ffwd = p.Ffwd + (int64_t)b * p.strideF;
    const double* Fbwd = p.Fbwd + (int64_t)b * p.strideF;
    const int32_t* perm = p.perm ? p.perm + (int64_t)b * p.stridePerm : nullptr;
    const double* in = p.in + (int64_t)b * p.strideIn;
    double* tmp = p.tmp + (int64_t)b * p.strideT;
    double* out = p.out + (int64_t)b * p.strideOut;
    const int sweeps = p.once ? 2 : 2 * p.z;

    // issue async loads of factor slab k and rhs rows of block k for `sweep`
    auto issue = [&](int sweep, int k, int buf) {
#ifdef SMG_SOLVE_NO_LOAD
        return;
#endif
        const double* F = ((sweep & 1) ? Fbwd : Ffwd) + (int64_t)k * slab;
        double* fs = Fs[buf];
        // 2W rows x W doubles -> W/2 16-byte chunks per row
        constexpr int CH = W / 2;
        for (int e = tid; e < 2 * W * CH; e += NT) {
            const int r = e / CH, ch = e % CH;
            cp_async16(fs + r * FS + 2 * ch, F + (int64_t)r * W + 2 * ch);
        }
        double* xs = Xs[buf];
        constexpr int CCH = CS / 2;
        for (int e = tid; e < W * CCH; e += NT) {
            const int r = e / CCH, ch = e % CCH;
            const int prow = k * W + r;
            if (sweep == 0) {
                const bool valid = prow < n;
                const int lrow = valid ? (perm ? perm[prow] : prow) : 0;
                cp_async16_zfill(xs + r * XS + 2 * ch, in + (int64_t)lrow * p.ldin + col0 + 2 * ch, valid);
            } else {
                cp_async16(xs + r * XS + 2 * ch, tmp + (int64_t)prow * p.ldt + col0 + 2 * ch);
            }
        }
        cp_async_commit();
    };

    for (int sweep = 0; sweep < sweeps; ++sweep) {
        const bool fwd = (sweep & 1) == 0;
        const bool last = sweep == sweeps - 1;
        int buf = 0;
        {
            const int k = fwd ? 0 : Kb - 1;
            issue(sweep, k, 0);
            // previous-block rows of the first step are zero
            for (int e = tid; e < W * XS; e += NT) Xs[0][W * XS + e] = 0.0;
        }
        for (int step = 0; step < Kb; ++step) {
            const int k = fwd ? step : Kb - 1 - step;
            cp_async_wait<0>();
            __syncthreads();
            if (step + 1 < Kb) issue(sweep, fwd ? k + 1 : k - 1, buf ^ 1);
            double acc[TL::MT][TL::NT][2];
            const bool skip2 = step == 0;
#ifndef SMG_SOLVE_NO_MMA
            if (fwd) mma_step<W, CS, true>(Fs[buf], Xs[buf], acc, warp, g, t, skip2);
            else mma_step<W, CS, false>(Fs[buf], Xs[buf], acc, warp, g, t, skip2);
#else
            for (int i = 0; i < TL::MT; ++i)
                for (int j = 0; j < TL::NT; ++j) acc[i][j][0] = acc[i][j][1] = Xs[buf][tid];
#endif
            // epilogue: result is the "previous block" of the next step and goes to dst
            double* xnext = Xs[buf ^ 1] + W * XS;
            if (warp < TL::ACTIVE) {
                const int wm = warp % TL::WM, wn = warp / TL::WM;
#pragma unroll
                for (int i = 0; i < TL::MT; ++i)
#pragma unroll
                    for (int j = 0; j < TL::NT; ++j) {
                        const int r = 8 * TL::tile(wm, i) + g, cc = 8 * (wn * TL::NT + j) + 2 * t;
                        xnext[r * XS + cc] = acc[i][j][0];
                        xnext[r * XS + cc + 1] = acc[i][j][1];
                        const int prow = k * W + r;
                        if (last) {
                            if (prow < n && col0 + cc < c) {
                                const int lrow = perm ? perm[prow] : prow;
                                double2* dst =
                                    reinterpret_cast<double2*>(out + (int64_t)lrow * p.ldout + col0 + cc);
                                *dst = make_double2(acc[i][j][0], acc[i][j][1]);
                            }
                        } else {
                            double2* dst = reinterpret_cast<double2*>(tmp + (int64_t)prow * p.ldt + col0 + cc);
                            *dst = make_double2(acc[i][j][0], acc[i][j][1]);
                        }
                    }
            }
            buf ^= 1;
        }
        __threadfence_block();
        __syncthreads();
    }
}

template <int W, int CS>
void launch(const SolveParams& p, cudaStream_t st) {
    const int bytes = SolveSmem<W, CS>::BYTES;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(solve_kernel<W, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        configured = true;
    }
    dim3 grid((p.c_cap + CS - 1) / CS, p.batch);
    ::smg::count_launch(), solve_kernel<W, CS><<<grid, NT, bytes, st>>>(p);
}

}  // namespace

// Column-slice width: narrow slices for latency-bound single chains (more CTAs),
// wide slices when many chains already fill the 148 SMs.
void solve_block_tridiag(const SolveParams& p, int W, cudaStream_t st) {
    const int slices8 = (p.c_cap + 7) / 8;
    const bool wide = (int64_t)p.batch * ((p.c_cap + 31) / 32) >= 148;
    const bool mid = (int64_t)p.batch * ((p.c_cap + 15) / 16) >= 148;
    (void)slices8;
    switch (W) {
        case 16: launch<16, 8>(p, st); break;
        case 32:
            if (wide) launch<32, 32>(p, st);
            else if (mid) launch<32, 16>(p, st);
            else launch<32, 8>(p, st);
            break;
        case 48:
            if (wide) launch<48, 32>(p, st);
            else if (mid) launch<48, 16>(p, st);
            else launch<48, 8>(p, st);
            break;
        case 64:
            if (wide) launch<64, 32>(p, st);
            else if (mid) launch<64, 16>(p, st);
            else launch<64, 8>(p, st);
            break;
        default: break;
    }
}

}  // namespace smg

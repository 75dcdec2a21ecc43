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
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

// 8 DMMA warps + 2 producer warps.  The producers move each step's factor slab
// (one bulk async copy on the TMA engine) and right-hand-side rows (cp.async),
// completion tracked by an mbarrier; the DMMA warps never have loads in flight, so
// their shared-memory fragment reads do not wait on the long scoreboard
// (cp.async issued by the DMMA warps themselves serialised the next slab's
// transfer with the current step's products).
constexpr int kSolveWarps = 8;
constexpr int kRhsWarps = 2;                  // right-hand-side producers
constexpr int kProdWarps = 1 + kRhsWarps;     // + one factor-slab producer
constexpr int NT_MMA = kSolveWarps * 32;
constexpr int NT = NT_MMA + kProdWarps * 32;
constexpr int NT_RHS = kRhsWarps * 32;

// Shared-memory plan: a ring of NSF factor slabs (2W x FS, one bulk copy each),
// a deeper ring of NSR right-hand-side blocks (W x XS, cp.async rows) and a
// double-buffered carry y_{k-1} (W x XS, written by the step epilogue).  The
// rhs ring runs furthest ahead: its rows come from the previous sweep's output
// in HBM (or the permuted input), the slabs mostly from L2.  Two CTAs per SM
// when the plan fits, else one CTA with the deepest rings that fit.
template <int W, int CS>
struct SolveSmem {
    static constexpr int FS = W + 4;   // padded row of the transposed factor slab
    static constexpr int XS = CS + 4;  // padded row of the right-hand-side slab
    static constexpr int F_ELEMS = 2 * W * FS;
    static constexpr int R_ELEMS = W * XS;
    // column-private mode (CS = 64): warp w owns all row tiles of columns 8w..8w+7, so the
    // carry y_{k-1} never crosses warps -- one carry buffer, no CTA-level barrier per step
    static constexpr bool PRIV = (CS == 64);
    // consumer (DMMA) warps: the cooperative tiling uses all 8; column-private warps own 16
    // columns each (4 x 2 tiles of 8 x 8: eight independent accumulator chains saturate the
    // warp's sub-partition, tools/dmma_lat.cu) -- one warp per SM sub-partition
    // 16-column slices at W = 32 (large batches, three CTAs per SM): FOUR DMMA warps, each one row
    // tile x both column tiles (3 operand loads per 2 DMMAs instead of 4, half the per-column scalar
    // work): 359 -> 317 us per 32-chain launch, C5 307 -> 299 ms per step; two warps (2 x 2 tiles
    // each) fall back to 360 us -- too few warps per scheduler; 32-column slices with four 1 x 4 warps: 401 us
#ifndef SMG_SOLVE_NCW16
#define SMG_SOLVE_NCW16 4
#endif
    static constexpr int NCW = PRIV ? CS / 16 : ((W == 32 && CS == 16) ? SMG_SOLVE_NCW16 : kSolveWarps);
    static constexpr int THREADS = (NCW + kProdWarps) * 32;
    static constexpr int FB = F_ELEMS * 8, RB = R_ELEMS * 8, YB = PRIV ? RB : 2 * RB;
    // W = 32, CS = 16 (large batches): a budget for three CTAs per SM (two rhs
    // slots instead of six).  The solve is bound by per-CTA step latency, so a
    // third resident CTA raises the SM's throughput: C5 418 -> 377 us per
    // launch against 32-column slices at two CTAs per SM (which were faster
    // than 16-column slices at two per SM).
    static constexpr int HALF = (W == 32 && CS == 16) ? 75 * 1024 : 113 * 1024, FULL = 226 * 1024;
    static constexpr bool TWO = 2 * FB + 3 * RB + YB <= HALF;
    static constexpr int BUDGET = TWO ? HALF : FULL;
#ifdef SMG_SOLVE_NSF_FORCE  // timing probe: slab ring depth override
    static constexpr int NSF = SMG_SOLVE_NSF_FORCE;
#else
    static constexpr int NSF = (!TWO && 3 * FB + 3 * RB + YB <= FULL) ? 3 : 2;
#endif
    static constexpr int NSR_FIT = (BUDGET - NSF * FB - YB) / RB;
#ifdef SMG_SOLVE_NS_FORCE  // timing probe: rhs ring depth override
    static constexpr int NSR = SMG_SOLVE_NS_FORCE;
#else
    static constexpr int NSR = NSR_FIT > 8 ? 8 : NSR_FIT;
#endif
    static_assert(NSR >= 2, "solve shared-memory plan");
    static constexpr int BYTES = NSF * FB + NSR * RB + YB;
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
    static constexpr bool PRIV = SolveSmem<W, CS>::PRIV;
    // 8 warps (two per SM sub-partition hide the DMMA issue latency); prefer a
    // 4 x 2 warp grid, a full m-column of warps when there is one n-tile
    static constexpr int NW = SolveSmem<W, CS>::NCW;
    static constexpr int WM = PRIV ? 1
                                   : (NT_ALL == 1) ? (MT_ALL < NW ? MT_ALL : NW)
                                                   : ((MT_ALL % 4 == 0 && NW >= 4) ? 4
                                                                                   : ((MT_ALL % 2 == 0 && NW >= 2) ? 2 : 1));
    static constexpr int WN_RAW = NW / WM;
    static constexpr int WN = (NT_ALL % WN_RAW == 0) ? WN_RAW
                                                     : ((NT_ALL % 4 == 0 && WN_RAW >= 4) ? 4 : ((NT_ALL % 2 == 0 && WN_RAW >= 2) ? 2 : 1));
    static constexpr int MT = MT_ALL / WM, NT = NT_ALL / WN;
    static constexpr int ACTIVE = WM * WN;
    // Row-tile of the warp's i-th m tile.  The first half of every step is a
    // triangular block, so contiguous row tiles would give the bottom warps up
    // to 4x the DMMAs of the top ones; pairing tile r with MT_ALL-1-r balances
    // every warp (and so every SM sub-partition).
    static constexpr bool PAIRED = !PRIV && (MT == 2 && MT_ALL == 2 * WM);
    static_assert(!PRIV || (NT == 2 && MT == MT_ALL && WN == NW), "column-private tiling: 16 columns per warp");
    SMG_DEV static int tile(int wm, int i) { return PAIRED ? (i == 0 ? wm : MT_ALL - 1 - wm) : wm * MT + i; }
};

template <int W, int CS, bool FWD>
SMG_DEV void mma_step(const double* __restrict__ fs, const double* __restrict__ xs, const double* __restrict__ ys,
                      double (&acc)[SolveTiling<W, CS>::MT][SolveTiling<W, CS>::NT][2], int warp, int g, int t,
                      int part) {
    // part 1: acc = triangular block x b_k (independent of the carry: computed
    // ahead, while other warps finish the previous step); part 2: acc += the
    // coupling block x y_{k-1} (the step's critical path)
    using TL = SolveTiling<W, CS>;
    constexpr int MT = TL::MT, NT = TL::NT;
    constexpr int FS = SolveSmem<W, CS>::FS;
    constexpr int XS = SolveSmem<W, CS>::XS;
    const int wm = warp % TL::WM, wn = warp / TL::WM;
    if (warp >= TL::ACTIVE) return;
    if (part == 2) goto second;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // first half: triangular block (Linv_k lower for FWD, Linv_k^T Sigma upper for BWD)
    if constexpr (TL::PRIV) {
        // all row tiles of one n-tile: in the 8-wide k block kb only the row tiles
        // i >= kb (FWD) / i <= kb (BWD) are nonzero -- compile-time, fully unrolled
#pragma unroll
        for (int kb = 0; kb < MT; ++kb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int kk = 8 * kb + 4 * h;
                double b[NT];
#pragma unroll
                for (int j = 0; j < NT; ++j) b[j] = xs[(kk + t) * XS + 8 * (wn * NT + j) + g];
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    if (FWD ? (i >= kb) : (i <= kb)) {
                        const double a = fs[(kk + t) * FS + 8 * i + g];
#pragma unroll
                        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a, b[j]);
                    }
            }
    } else if constexpr (TL::PAIRED) {
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
    } else if constexpr (MT == 1) {
        // one row tile: its nonzero k range is a loop bound
        const int r = TL::tile(wm, 0);
        const int k0 = FWD ? 0 : 8 * r, k1 = FWD ? 8 * r + 8 : W;
        // fully unrolled over the block; the tile's zero k range is branched
        // around (no DMMA issued), not predicated
#pragma unroll
        for (int kk = 0; kk < W; kk += 4) {
            if (kk < k0 || kk >= k1) continue;
            double b[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) b[j] = xs[(kk + t) * XS + 8 * (wn * NT + j) + g];
            const double a = fs[(kk + t) * FS + 8 * r + g];
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[0][j][0], acc[0][j][1], a, b[j]);
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
    return;
second:
#pragma unroll
    for (int kk = W; kk < 2 * W; kk += 4) {
        double a[MT], b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = ys[(kk - W + t) * XS + 8 * (wn * NT + j) + g];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = fs[(kk + t) * FS + 8 * TL::tile(wm, i) + g];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

// ---- bulk async copies (TMA engine) with mbarrier completion
SMG_DEV uint32_t smem_u32(const void* ptr) { return static_cast<uint32_t>(__cvta_generic_to_shared(ptr)); }
SMG_DEV void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SMG_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
SMG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
SMG_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

SMG_DEV void mbar_arrive_local(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier over the DMMA warps only (the producers run ahead on mbarriers)
template <int THREADS_MMA>
SMG_DEV void mma_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(THREADS_MMA) : "memory"); }

// Warp-specialised: the DMMA warps run the steps (named barrier among
// themselves for the carry rows); one producer warp streams the factor slabs
// (fullF/consumedF ring), two stream the right-hand-side rows (fullR/consumedR
// ring, deeper).  Producers never meet the DMMA warps at a CTA barrier.  Ring
// slot s of step gs is gs % N, the phase parity of that step (gs / N) & 1.
template <int W, int CS>
__global__ void __launch_bounds__((SolveSmem<W, CS>::THREADS)) solve_kernel(SolveParams p) {
    using S = SolveSmem<W, CS>;
    constexpr int kSolveWarps = S::NCW, NT_MMA = S::NCW * 32;  // shadow the file-scope defaults
    using TL = SolveTiling<W, CS>;
    constexpr int FS = S::FS, XS = S::XS;
    constexpr int NSF = S::NSF, NSR = S::NSR;
    extern __shared__ __align__(16) double smem[];
    auto Fs = [&](int i) { return smem + i * S::F_ELEMS; };
    auto Rs = [&](int i) { return smem + NSF * S::F_ELEMS + i * S::R_ELEMS; };
    auto Ys = [&](int i) { return smem + NSF * S::F_ELEMS + NSR * S::R_ELEMS + (S::PRIV ? 0 : i) * S::R_ELEMS; };

    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int col0 = blockIdx.x * CS;
    if (col0 >= c) return;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int n = p.n, Kb = p.Kb;
    const int64_t slab = (int64_t)2 * W * factor_row(W);  // doubles per block in Ffwd/Fbwd (padded rows)
    static_assert(FS == factor_row(W), "smem slab rows match the global padded rows");
    const double* Ffwd = p.Ffwd + (int64_t)b * p.strideF;
    const double* Fbwd = p.Fbwd + (int64_t)b * p.strideF;
    const int32_t* perm = p.perm ? p.perm + (int64_t)b * p.stridePerm : nullptr;
    const double* in = p.in + (int64_t)b * p.strideIn;
    double* tmp = p.tmp + (int64_t)b * p.strideT;
    double* out = p.out + (int64_t)b * p.strideOut;
    const int sweeps = p.once ? 2 : 2 * p.z;
    const int total = sweeps * Kb;

    __shared__ __align__(8) uint64_t fullF[NSF], consF[NSF], fullR[NSR], consR[NSR];
    if (tid == 0) {
        for (int i = 0; i < NSF; ++i) {
            mbar_init(&fullF[i], 1);            // the slab producer's arrive (+ tx bytes)
            mbar_init(&consF[i], kSolveWarps);  // one arrive per DMMA warp
        }
        for (int i = 0; i < NSR; ++i) {
            mbar_init(&fullR[i], kRhsWarps);    // one arrive per rhs warp (+ its lanes' cp.async)
            mbar_init(&consR[i], kSolveWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // step cursor: (sweep, step) of global step gs, advanced incrementally (no
    // division by the runtime block count in the loops)
    struct Cursor {
        int gs, sweep, step, Kb;
        SMG_DEV int k() const { return (sweep & 1) ? Kb - 1 - step : step; }
        SMG_DEV void next() {
            ++gs;
            if (++step == Kb) {
                step = 0;
                ++sweep;
            }
        }
    };

    if (warp == kSolveWarps) {
        // ---- factor slabs: one bulk copy (TMA engine) per step
        if (lane == 0) {
            for (Cursor cu{0, 0, 0, Kb}; cu.gs < total; cu.next()) {
                const int gs = cu.gs, sl = gs % NSF;
                if (gs >= NSF) mbar_wait(&consF[sl], ((gs - NSF) / NSF) & 1);
                const double* F = ((cu.sweep & 1) ? Fbwd : Ffwd) + (int64_t)cu.k() * slab;
#ifdef SMG_SOLVE_SLAB_DIV  // timing probe: move only 1/DIV of the slab bytes
                constexpr uint32_t kSlabBytes = (2 * W * FS * 8 / SMG_SOLVE_SLAB_DIV + 15) / 16 * 16;
#else
                constexpr uint32_t kSlabBytes = 2 * W * FS * 8;
#endif
                mbar_arrive_expect_tx(&fullF[sl], kSlabBytes);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                bulk_g2s(Fs(sl), F, kSlabBytes, &fullF[sl]);
            }
        }
    } else if (warp > kSolveWarps) {
        // ---- right-hand-side rows: cp.async, NSR steps ahead; sweep 0 gathers
        // the permuted input rows, later sweeps read the previous sweep's output
        const int rt = tid - NT_MMA - 32;
        constexpr int CCH = CS / 2;                              // 16-byte chunks per row
        constexpr int PER = (W * CCH + NT_RHS - 1) / NT_RHS;     // chunks per thread per step
        int pn[PER];                                             // next step's source rows (perm prefetch)
        auto src_rows = [&](const Cursor& c, int (&rows)[PER]) {
            const int k = c.k(), sweep = c.sweep;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = rt + i * NT_RHS, r = e / CCH, prow = k * W + r;
                rows[i] = (e < W * CCH && prow < n && sweep == 0 && perm) ? __ldg(perm + prow) : prow;
            }
        };
        Cursor nx{0, 0, 0, Kb};
        src_rows(nx, pn);
        const int cmax = min(p.ldin, p.ldt);  // a slice wider than the remaining columns stops at the row end
        for (Cursor cu{0, 0, 0, Kb}; cu.gs < total; cu.next()) {
            const int gs = cu.gs, sweep = cu.sweep, step = cu.step, k = cu.k(), sl = gs % NSR;
            int rows[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) rows[i] = pn[i];
            nx.next();
            if (nx.gs < total) src_rows(nx, pn);  // overlaps the waits below
            if (gs >= NSR) mbar_wait(&consR[sl], ((gs - NSR) / NSR) & 1);
            if (step == 0 && gs > 0) {
                // this sweep reads the previous sweep's rows: all of its steps are done
                mbar_wait(&consR[(gs - 1) % NSR], ((gs - 1) / NSR) & 1);
            }
            double* xs = Rs(sl);
            const int nvalid = max(0, min(W, n - k * W));
#ifndef SMG_SOLVE_NO_RHS
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = rt + i * NT_RHS;
                if (e >= W * CCH) break;
                const int r = e / CCH, ch = e % CCH;
                if (r < nvalid && col0 + 2 * ch < cmax) {
                    const double* src = (sweep == 0) ? in + (int64_t)rows[i] * p.ldin + col0
                                                     : tmp + (int64_t)rows[i] * p.ldt + col0;
                    cp_async16(xs + r * XS + 2 * ch, src + 2 * ch);
                } else {
                    cp_async16_zfill(xs + r * XS + 2 * ch, in, false);  // padded rows past n
                }
            }
#endif
            asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&fullR[sl])) : "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&fullR[sl]);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else {
        double acc[TL::MT][TL::NT][2];
        // column-private mode: a warp whose 16 columns lie past c only keeps the rings moving
        const bool live = !S::PRIV || col0 + 16 * warp < c;
        // the independent half of step gs (waits for the step's slab and rhs block)
        auto first = [&](double (&acc)[TL::MT][TL::NT][2], int gs, int sweep) {
            mbar_wait(&fullR[gs % NSR], (gs / NSR) & 1);
            mbar_wait(&fullF[gs % NSF], (gs / NSF) & 1);
            if (!live) return;
#if defined(SMG_SOLVE_NO_TRI)  // timing probe: coupling half only (one dense product per step)
            (void)sweep;
            for (int i = 0; i < TL::MT; ++i)
                for (int j = 0; j < TL::NT; ++j) acc[i][j][0] = acc[i][j][1] = Rs(gs % NSR)[tid & 63];
#elif !defined(SMG_SOLVE_NO_MMA)
            if ((sweep & 1) == 0) mma_step<W, CS, true>(Fs(gs % NSF), Rs(gs % NSR), nullptr, acc, warp, g, t, 1);
            else mma_step<W, CS, false>(Fs(gs % NSF), Rs(gs % NSR), nullptr, acc, warp, g, t, 1);
#else
            for (int i = 0; i < TL::MT; ++i)
                for (int j = 0; j < TL::NT; ++j) acc[i][j][0] = acc[i][j][1] = Rs(gs % NSR)[tid];
#endif
        };
        first(acc, 0, 0);
        Cursor nx{0, 0, 0, Kb};
        for (Cursor cu{0, 0, 0, Kb}; cu.gs < total; cu.next()) {
            const int gs = cu.gs, sweep = cu.sweep, step = cu.step, k = cu.k();
            nx.next();
            const int sf = gs % NSF, sr = gs % NSR;
            const bool last = sweep == sweeps - 1;
            // output rows of the last sweep go through the permutation: fetch them
            // before the products so the loads overlap them
            int lrow[TL::MT];
            {
                const int wm = warp % TL::WM;
#pragma unroll
                for (int i = 0; i < TL::MT; ++i) {
                    const int prow = k * W + 8 * TL::tile(wm, i) + g;
                    lrow[i] = (last && perm && prow < n) ? __ldg(perm + prow) : prow;
                }
            }
            double* ycur = Ys(gs & 1);  // this step's output = next step's carry
            const double* yprev = Ys((gs + 1) & 1);
            // the carry of a sweep's first step is zero
#ifndef SMG_SOLVE_NO_MMA
            if (step != 0 && live) {
                if ((sweep & 1) == 0) mma_step<W, CS, true>(Fs(sf), nullptr, yprev, acc, warp, g, t, 2);
                else mma_step<W, CS, false>(Fs(sf), nullptr, yprev, acc, warp, g, t, 2);
            }
#else
            if (step != 0)
                for (int i = 0; i < TL::MT; ++i)
                    for (int j = 0; j < TL::NT; ++j) acc[i][j][0] += yprev[tid];
#endif
            // the slab and rhs block are read: release them before the epilogue
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_local(&consF[sf]);
                if (step + 1 != Kb) mbar_arrive_local(&consR[sr]);
            }
            if (warp < TL::ACTIVE && live) {
                const int wm = warp % TL::WM, wn = warp / TL::WM;
#pragma unroll
                for (int i = 0; i < TL::MT; ++i)
#pragma unroll
                    for (int j = 0; j < TL::NT; ++j) {
                        const int r = 8 * TL::tile(wm, i) + g, cc = 8 * (wn * TL::NT + j) + 2 * t;
                        *reinterpret_cast<double2*>(ycur + r * XS + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
                        const int prow = k * W + r;
                        if (last) {
                            if (prow < n && col0 + cc < c) {
                                double2* dst = reinterpret_cast<double2*>(out + (int64_t)lrow[i] * p.ldout + col0 + cc);
                                *dst = make_double2(acc[i][j][0], acc[i][j][1]);
                            }
                        } else {
                            double2* dst = reinterpret_cast<double2*>(tmp + (int64_t)prow * p.ldt + col0 + cc);
                            *dst = make_double2(acc[i][j][0], acc[i][j][1]);
                        }
                    }
            }
            if (step + 1 == Kb) {
                // the next sweep's rhs rows (read by the producers) are this sweep's
                // output rows: visible to the async proxy before the release
                __threadfence_block();
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_local(&consR[sr]);
            }
            if (nx.gs < total) first(acc, nx.gs, nx.sweep);  // off the critical path: before the barrier
            // ycur complete before the next step reads it; yprev free for reuse
            if constexpr (S::PRIV) __syncwarp();  // the carry columns are the warp's own: no CTA barrier
            else mma_bar<NT_MMA>();
        }
    }
}

template <int W, int CS>
void launch(const SolveParams& p, cudaStream_t st) {
    const int bytes = SolveSmem<W, CS>::BYTES;
    const int slices = (p.c_cap + CS - 1) / CS;
    ensure_smem((const void*)solve_kernel<W, CS>, bytes);
    dim3 grid(slices, p.batch);
    ::smg::count_launch(), solve_kernel<W, CS><<<grid, SolveSmem<W, CS>::THREADS, bytes, st>>>(p);
}

}  // namespace

// Column-slice width: narrow slices for latency-bound single chains (more CTAs),
// wide slices when many chains already fill the 148 SMs.
void solve_block_tridiag(const SolveParams& p, int W, cudaStream_t st) {
    const int slices8 = (p.c_cap + 7) / 8;
    bool wide = (int64_t)p.batch * ((p.c_cap + 31) / 32) >= 148;
    bool mid = (int64_t)p.batch * ((p.c_cap + 15) / 16) >= 148;
    if (const char* e = std::getenv("SMG_SOLVE_CS")) {  // tuning override: 8, 16 or 32
        const int cs = std::atoi(e);
        wide = cs >= 32;
        mid = cs >= 16;
    }
    (void)slices8;
    switch (W) {
        case 16: launch<16, 8>(p, st); break;
        case 32:
            if (std::getenv("SMG_SOLVE_CS") && std::atoi(std::getenv("SMG_SOLVE_CS")) >= 64) launch<32, 64>(p, st);
            else if (wide && std::getenv("SMG_SOLVE_CS") && std::atoi(std::getenv("SMG_SOLVE_CS")) >= 32) launch<32, 32>(p, st);
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

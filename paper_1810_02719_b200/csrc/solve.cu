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
constexpr int kProdWarps = 2;
constexpr int NT_MMA = kSolveWarps * 32;
constexpr int NT = NT_MMA + kProdWarps * 32;
constexpr int NT_PROD = kProdWarps * 32;

template <int W, int CS>
struct SolveSmem {
    static constexpr int FS = W + 4;   // padded row of the transposed factor slab
    static constexpr int XS = CS + 4;  // padded row of the right-hand-side slab
    static constexpr int F_ELEMS = 2 * W * FS;
    static constexpr int X_ELEMS = 2 * W * XS;
    // pipeline depth: as many stages as fit two CTAs per SM (at least 2); a
    // narrow W has short steps, so its loads need more than one step of lead
    static constexpr int STAGE = (F_ELEMS + X_ELEMS) * 8;
    static constexpr int NS = (4 * STAGE <= 113 * 1024) ? 4 : ((3 * STAGE <= 113 * 1024) ? 3 : 2);
    static constexpr int BYTES = NS * STAGE;
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
    } else if constexpr (MT == 1) {
        // one row tile: its nonzero k range is a loop bound
        const int r = TL::tile(wm, 0);
        const int k0 = FWD ? 0 : 8 * r, k1 = FWD ? 8 * r + 8 : W;
#pragma unroll 2
        for (int kk = k0; kk < k1; kk += 4) {
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

SMG_DEV void bulk_multicast(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
SMG_DEV void mbar_arrive_local(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on the mbarrier at the same offset in cluster CTA `rank`
SMG_DEV void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
        " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}
SMG_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAITC_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
SMG_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
SMG_DEV uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}
SMG_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// named barrier over the DMMA warps only (the producers run ahead on mbarriers)
SMG_DEV void mma_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NT_MMA) : "memory"); }

// Warp-specialised: the DMMA warps run the steps (named barrier among
// themselves for the epilogue rows), the producer warps run one step ahead
// and never meet them at a CTA barrier -- they wait for a buffer to be
// released (consumed[buf], one arrive per DMMA warp) and fill it (full[buf]).
// MC: the column-slice CTAs of one chain form a cluster; every CTA releases a
// buffer by arriving on rank 0's empty[buf], and rank 0 multicasts the factor
// slab (read from L2 once per cluster) into every CTA's buffer.
template <int W, int CS, bool MC>
__global__ void __launch_bounds__(NT) solve_kernel(SolveParams p) {
    using S = SolveSmem<W, CS>;
    using TL = SolveTiling<W, CS>;
    constexpr int FS = S::FS, XS = S::XS;
    extern __shared__ __align__(16) double smem[];
    constexpr int NS = S::NS;
    auto Fs = [&](int i) { return smem + i * S::F_ELEMS; };
    auto Xs = [&](int i) { return smem + NS * S::F_ELEMS + i * S::X_ELEMS; };

    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int col0 = blockIdx.x * CS;
    if (!MC && col0 >= c) return;  // (MC launches only with every slice in range)

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

    const bool producer = tid >= NT_MMA;
    const int ptid = tid - NT_MMA;
    __shared__ __align__(8) uint64_t full[NS], consumed[NS], empty[NS];
    uint32_t csz = 1, crank = 0;
    if (MC) {
        csz = cluster_size();
        crank = cluster_rank();
    }
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], kProdWarps);        // one arrive per producer warp (+ tx bytes, cp.async)
            mbar_init(&consumed[i], kSolveWarps);  // one arrive per DMMA warp
            mbar_init(&empty[i], (int)csz);        // rank 0 (MC): one arrive per cluster CTA
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (MC) cluster_sync_all();  // every CTA's barriers exist before the first remote arrive

    auto block_of = [&](int gs) {
        const int sweep = gs / Kb, step = gs % Kb;
        return (sweep & 1) ? Kb - 1 - step : step;
    };

    if (producer) {
        uint32_t cph[NS], eph[NS];
        for (int i = 0; i < NS; ++i) cph[i] = eph[i] = 0u;
        for (int gs = 0; gs < total; ++gs) {
            const int sweep = gs / Kb, step = gs % Kb, k = block_of(gs), buf = gs % NS;
            // the buffer's previous contents (step gs-NS) are consumed; at a sweep's
            // first step the previous sweep (its tmp rows) is complete
            if (gs >= NS) {
                mbar_wait(&consumed[buf], cph[buf]);
                cph[buf] ^= 1u;
            }
            if (step == 0 && gs > 0) {  // step gs-1 (the sweep's end) is consumed; the regular
                const int pb = (gs - 1) % NS;  // wait of step gs-1+NS re-checks this phase
                mbar_wait(&consumed[pb], cph[pb]);
            }
            const double* F = ((sweep & 1) ? Fbwd : Ffwd) + (int64_t)k * slab;
            double* fs = Fs(buf);
            double* xs = Xs(buf);
            const int nvalid = max(0, min(W, n - k * W));  // rhs rows of the block inside the tile
            constexpr int CCH = CS / 2;
            for (int e = ptid; e < W * CCH; e += NT_PROD) {
                const int r = e / CCH, ch = e % CCH;
                const int prow = k * W + r;
                if (r < nvalid) {
                    const double* src = (sweep == 0) ? in + (int64_t)(perm ? perm[prow] : prow) * p.ldin + col0
                                                     : tmp + (int64_t)prow * p.ldt + col0;
                    cp_async16(xs + r * XS + 2 * ch, src + 2 * ch);
                } else {
                    cp_async16_zfill(xs + r * XS + 2 * ch, in, false);  // padded rows past n
                }
            }
            asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[buf])) : "memory");
            __syncwarp();
            if (ptid == 0) {
                mbar_arrive_expect_tx(&full[buf], (uint32_t)(2 * W * FS * 8));
                if constexpr (MC) {
                    mbar_arrive_remote(&empty[buf], 0);  // this CTA's buffer is free and armed
                    if (crank == 0) {
                        mbar_wait_cluster(&empty[buf], eph[buf]);
                        eph[buf] ^= 1u;
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        bulk_multicast(fs, F, 2 * W * FS * 8, &full[buf], (uint16_t)((1u << csz) - 1u));
                    }
                } else {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    bulk_g2s(fs, F, 2 * W * FS * 8, &full[buf]);
                }
            } else if (lane == 0) {
                mbar_arrive_local(&full[buf]);
            }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else {
        uint32_t fph[NS];
        for (int i = 0; i < NS; ++i) fph[i] = 0u;
        for (int gs = 0; gs < total; ++gs) {
            const int sweep = gs / Kb, step = gs % Kb, k = block_of(gs), buf = gs % NS;
            const bool fwd = (sweep & 1) == 0;
            const bool last = sweep == sweeps - 1;
            // output rows of the last sweep go through the permutation: fetch them
            // before the wait so the loads overlap it and the products
            int lrow[TL::MT];
            {
                const int wm = warp % TL::WM;
#pragma unroll
                for (int i = 0; i < TL::MT; ++i) {
                    const int prow = k * W + 8 * TL::tile(wm, i) + g;
                    lrow[i] = (last && perm && prow < n) ? __ldg(perm + prow) : prow;
                }
            }
            mbar_wait(&full[buf], fph[buf]);
            fph[buf] ^= 1u;
            double acc[TL::MT][TL::NT][2];
            const bool skip2 = step == 0;  // previous-block rows of a sweep's first step are zero
#ifndef SMG_SOLVE_NO_MMA
            if (fwd) mma_step<W, CS, true>(Fs(buf), Xs(buf), acc, warp, g, t, skip2);
            else mma_step<W, CS, false>(Fs(buf), Xs(buf), acc, warp, g, t, skip2);
#else
            for (int i = 0; i < TL::MT; ++i)
                for (int j = 0; j < TL::NT; ++j) acc[i][j][0] = acc[i][j][1] = Xs(buf)[tid];
#endif
            // epilogue: result is the "previous block" of the next step and goes to dst
            double* xnext = Xs((gs + 1) % NS) + W * XS;
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
                // the next sweep's rhs rows (read by the producers) are this sweep's tmp rows
                __threadfence_block();
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
            }
            mma_bar();  // xnext complete before the next step reads it; buf fully read
            if (lane == 0) mbar_arrive_local(&consumed[buf]);
        }
    }
    if (MC) {
        __syncthreads();
        cluster_sync_all();  // no CTA leaves while cluster peers may still address its barriers
    }
}

template <int W, int CS>
void launch(const SolveParams& p, cudaStream_t st) {
    const int bytes = SolveSmem<W, CS>::BYTES;
    const int slices = (p.c_cap + CS - 1) / CS;
    int csz = 0;  // cluster size: largest divisor of the slice count in [2, 8]
    // opt-in (SMG_SOLVE_MC=1): with two slab buffers the per-step cross-CTA
    // release/multicast round trip sits on the critical path and the cluster
    // runs slower than independent CTAs (1.48 ms vs 0.83 ms per C5 launch)
    if (p.dimC == nullptr && std::getenv("SMG_SOLVE_MC"))
        for (int d = 8; d >= 2; --d)
            if (slices % d == 0) {
                csz = d;
                break;
            }
    static bool configured[2] = {false, false};
    const bool mc = csz >= 2;
    if (!configured[mc]) {
        if (mc) cudaFuncSetAttribute(solve_kernel<W, CS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        else cudaFuncSetAttribute(solve_kernel<W, CS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        configured[mc] = true;
    }
    dim3 grid(slices, p.batch);
    ::smg::count_launch();
    if (!mc) {
        solve_kernel<W, CS, false><<<grid, NT, bytes, st>>>(p);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csz;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, solve_kernel<W, CS, true>, p);
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

// Batched FP64 GEMM on the DMMA tensor path (mma.sync m8n8k4 f64).
//
// C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b], row-major operands.
// Used for the Gram V^T V (K5, split-K over the n_d rows, upper tiles only),
// the triangular right-multiply V * B with B upper triangular (K7, the K loop
// stops at the tile's last column), and the Rayleigh-Ritz products of the
// first-submesh basis (K9).
//
// CTA tile 64 x BN (BN = 16 * NJ), four warps of 32 x 8NJ, register prefetch of
// the next K slab while the current one is multiplied.  The column range is
// launched as 64-wide tiles plus one narrow tile (BN = 16..64) over c mod 64
// columns, so c = 200 does not pay for 56 padded columns: DMMAs that are predicated off
// still occupy the pipe, so padding is removed structurally, and the masked
// (predicated) inner loop only runs where the tile crosses a row/column edge,
// the Gram's diagonal or B's diagonal block.  Split-K partials are summed in a
// fixed order by gemm_reduce (deterministic).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int BM = 64, BK = 16, NT = 128;
constexpr int SPX = BK + 4;  // x-major slab row (k contiguous): 20 % 16 == 4, conflict-free

// Shared-memory slab of one operand: BK x XW (k, x).  k-major operands (x
// contiguous in global memory) are stored [k][x], x-major ones [x][k]; both
// strides are 4 mod 16 doubles so fragment reads and stores avoid bank conflicts.
template <int XW, bool KMAJOR, int KB = BK>
struct Slab {
    static constexpr int DEPTH = KB;
    static constexpr int S = KMAJOR ? XW + 4 : KB + 4;
    static constexpr int ELEMS = KMAJOR ? KB * (XW + 4) : XW * (KB + 4);
    static constexpr int PER = XW * KB / NT;  // elements per thread
    double r[PER];
    SMG_DEV static double at(const double* s, int k, int x) { return KMAJOR ? s[k * S + x] : s[x * S + k]; }
    SMG_DEV static void coords(int e, int& k, int& x) {
        if (KMAJOR) {
            k = e / XW;
            x = e % XW;
        } else {
            k = e % KB;
            x = e / KB;
        }
    }
    // element (k, x) lives at ptr[k*ld + x] (KMAJOR) or ptr[x*ld + k]
    SMG_DEV void load(const double* __restrict__ ptr, int64_t ld, int k0, int x0, int kmax, int xmax) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            int k, x;
            coords(threadIdx.x + j * NT, k, x);
            const int gk = k0 + k, gx = x0 + x;
            r[j] = (gk < kmax && gx < xmax) ? __ldg(KMAJOR ? ptr + (int64_t)gk * ld + gx : ptr + (int64_t)gx * ld + gk)
                                            : 0.0;
        }
    }
    SMG_DEV void store(double* __restrict__ s) const {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            int k, x;
            coords(threadIdx.x + j * NT, k, x);
            if (KMAJOR) s[k * S + x] = r[j];
            else s[x * S + k] = r[j];
        }
    }
};

// DMMA products of one BK-deep slab pair (shared by the register-staged and the
// producer-warp kernels).
template <class SA, class SB, int NJ>
SMG_DEV void slab_mma(const double* __restrict__ as, const double* __restrict__ bs, double (&acc)[4][NJ][2],
                      unsigned fmask, unsigned kFull, int k0, int kdiag, int upperB, int wm, int wn, int g, int t) {
    constexpr int KD = SA::DEPTH;
    if (fmask == kFull && k0 + KD <= kdiag) {
            // interior: every fragment active, no predication; m16n8k8 (4x the
            // work per instruction of m8n8k4, same accumulator registers)
#pragma unroll
            for (int kk = 0; kk < KD; kk += 8) {
                double a[2][4], bb[NJ][2];
#pragma unroll
                for (int I = 0; I < 2; ++I) {
                    const int r = wm + 16 * I + g;
                    a[I][0] = SA::at(as, kk + t, r);
                    a[I][1] = SA::at(as, kk + t, r + 8);
                    a[I][2] = SA::at(as, kk + t + 4, r);
                    a[I][3] = SA::at(as, kk + t + 4, r + 8);
                }
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    bb[j][0] = SB::at(bs, kk + t, wn + 8 * j + g);
                    bb[j][1] = SB::at(bs, kk + t + 4, wn + 8 * j + g);
                }
#pragma unroll
                for (int I = 0; I < 2; ++I)
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        dmma1688(acc[2 * I][j][0], acc[2 * I][j][1], acc[2 * I + 1][j][0], acc[2 * I + 1][j][1],
                                 a[I][0], a[I][1], a[I][2], a[I][3], bb[j][0], bb[j][1]);
            }
        } else if (fmask != 0 && k0 < kdiag + 8 * NJ) {
#pragma unroll
            for (int kk = 0; kk < KD; kk += 4) {
                unsigned m = fmask;
                if (upperB) {
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        if (kdiag + 8 * j + 7 < k0 + kk) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) m &= ~(1u << (NJ * i + j));
                        }
                }
                if (m == 0) continue;
                double a[4], bb[NJ];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = SA::at(as, kk + t, wm + 8 * i + g);
#pragma unroll
                for (int j = 0; j < NJ; ++j) bb[j] = SB::at(bs, kk + t, wn + 8 * j + g);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        if (m & (1u << (NJ * i + j))) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
            }
        }
}

// Projection partials of one warp tile (32 rows r0.. = one 32-row chunk of
// project.cu's partial pass, 8NJ columns c0..): lane (g, t) holds rows r0 + 8i + g,
// columns c0 + 8j + 2t + q.  Per column, the lane's 4 rows are combined in row
// order and the 8 lanes of a column group by a fixed xor tree (deterministic);
// the argmax keeps the larger |q|, the smaller row on ties (first index wins,
// spectral.hpp:72-85).
template <int NJ>
SMG_DEV void proj_epilogue(const GemmParams& p, const double (&acc)[4][NJ][2], int b, int r0, int c0, int N, int g,
                           int t) {
    if (r0 >= p.projN) return;  // warp-uniform: rows past n are padding (no chunk)
    const int c = min(N, p.projCcap);
    const double* X = p.projX + (int64_t)b * p.strideProjX;
    double* part = p.projPart + ((int64_t)b * p.projChunks + (r0 >> 5)) * (int64_t)p.projCcap * 8;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            double best = -1.0, bval = 0.0, px = 0.0, py = 0.0, pz = 0.0, ps = 0.0;
            int brow = 1 << 30;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = r0 + 8 * i + g;
                if (row >= p.projN) continue;
                // coordinates re-read per column (L1 hits): keeps the epilogue's
                // live registers at the accumulators
                const double x = __ldg(X + 3 * (int64_t)row), y = __ldg(X + 3 * (int64_t)row + 1),
                             z = __ldg(X + 3 * (int64_t)row + 2);
                const double v = acc[i][j][q], m = fabs(v);
                if (m > best) {
                    best = m;
                    bval = v;
                    brow = row;
                }
                px = fma(v, x, px);
                py = fma(v, y, py);
                pz = fma(v, z, pz);
                ps = fma(v, (x + y) + z, ps);
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
                const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
                if (ob > best || (ob == best && orow < brow)) {
                    best = ob;
                    bval = ov;
                    brow = orow;
                }
                px += __shfl_xor_sync(0xffffffffu, px, o);
                py += __shfl_xor_sync(0xffffffffu, py, o);
                pz += __shfl_xor_sync(0xffffffffu, pz, o);
                ps += __shfl_xor_sync(0xffffffffu, ps, o);
            }
            const int col = c0 + 8 * j + 2 * t + q;
            if (g == 0 && col < c) {
                double4* o4 = reinterpret_cast<double4*>(part + (int64_t)col * 8);
                o4[0] = make_double4(best, bval, px, py);
                o4[1] = make_double4(pz, ps, 0.0, 0.0);
            }
        }
}

template <bool TA, bool TB, int NJ>
__global__ void __launch_bounds__(NT, 4) gemm_kernel(GemmParams p, int n_base, int n_end) {
    constexpr int BN = 16 * NJ;
    // op(A) element (m, k): TA ? A[k*lda + m] : A[m*lda + k]  -> k-major iff TA
    // op(B) element (k, n): TB ? B[n*ldb + k] : B[k*ldb + n]  -> k-major iff !TB
    using SA = Slab<BM, TA>;
    using SB = Slab<BN, !TB>;
    const int splits = p.splits > 0 ? p.splits : 1;
    const int b = blockIdx.z / splits;
    const int s = blockIdx.z % splits;
    if (p.skip && p.skip[b]) return;
    const int M = p.dimM ? p.dimM[(int64_t)b * p.dimStride] : p.M;
    const int N = min(p.dimN ? p.dimN[(int64_t)b * p.dimStride] : p.N, n_end);  // this launch's columns
    const int K = p.dimK ? p.dimK[(int64_t)b * p.dimStride] : p.K;
    const int m0 = blockIdx.y * BM, n0 = n_base + blockIdx.x * BN;
    if (m0 >= M || n0 >= N) return;
    if (p.syrkUpper && (m0 >> 5) > ((n0 + BN - 1) >> 5)) return;  // tile entirely below the diagonal 32-blocks

    int kEnd = K;
    if (p.upperB) kEnd = min(kEnd, n0 + BN);
    const int kchunk = ((kEnd + splits - 1) / splits + BK - 1) / BK * BK;
    const int kBeg = s * kchunk;
    const int kStop = min(kEnd, kBeg + kchunk);

    const double* A = p.A + (int64_t)b * p.strideA;
    const double* B = p.B + (int64_t)b * p.strideB;

    __shared__ __align__(16) double As[2][SA::ELEMS];
    __shared__ __align__(16) double Bs[2][SB::ELEMS];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * (8 * NJ);

    double acc[4][NJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // fragments that carry output: rows < M, cols < N, and for syrkUpper not in a
    // 32-block below the diagonal (the Cholesky reads the upper triangle incl.
    // full 32x32 diagonal blocks)
    constexpr unsigned kFull = (1u << (4 * NJ)) - 1u;
    unsigned fmask = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int r = m0 + wm + 8 * i, cc = n0 + wn + 8 * j;
            bool on = r < M && cc < N;
            if (p.syrkUpper && (r >> 5) > ((cc + 7) >> 5)) on = false;  // tiles need not be 32-aligned
            if (on) fmask |= 1u << (NJ * i + j);
        }
    // first k of the warp's diagonal region of an upper-triangular B (k > col is zero)
    const int kdiag = p.upperB ? n0 + wn : 1 << 30;

    SA la;
    SB lb;
    int buf = 0;
    if (kBeg < kStop) {
        la.load(A, p.lda, kBeg, m0, kStop, M);
        lb.load(B, p.ldb, kBeg, n0, kStop, N);
        la.store(As[0]);
        lb.store(Bs[0]);
    }
    __syncthreads();
    for (int k0 = kBeg; k0 < kStop; k0 += BK) {
        const bool more = k0 + BK < kStop;
        if (more) {
            la.load(A, p.lda, k0 + BK, m0, kStop, M);
            lb.load(B, p.ldb, k0 + BK, n0, kStop, N);
        }
        const double* as = As[buf];
        const double* bs = Bs[buf];
        slab_mma<SA, SB, NJ>(as, bs, acc, fmask, kFull, k0, kdiag, p.upperB, wm, wn, g, t);
        if (more) {
            la.store(As[buf ^ 1]);
            lb.store(Bs[buf ^ 1]);
        }
        __syncthreads();
        buf ^= 1;
    }

    double* C;
    double alpha = p.alpha, beta = p.beta;
    if (splits > 1) {
        C = p.C + ((int64_t)b * splits + s) * p.strideP;
        alpha = 1.0;
        beta = 0.0;
    } else {
        C = p.C + (int64_t)b * p.strideC;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm + 8 * i + g;
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int col = n0 + wn + 8 * j + 2 * t + q;
                if (col >= N) continue;
                double* dst = C + (int64_t)row * p.ldc + col;
                double v = alpha * acc[i][j][q];
                if (beta != 0.0) v += beta * *dst;
                *dst = v;
            }
        }
    }
    if (p.projPart && splits == 1) proj_epilogue<NJ>(p, acc, b, m0 + wm, n0 + wn, N, g, t);
}


// ---- producer-warp pipeline: one warp moves the slabs with cp.async into a
// PNS-stage ring (completion on mbarriers), the four DMMA warps never have
// loads in flight (no register staging, no long-scoreboard coupling of their
// fragment reads to outstanding LDGSTS) and never meet at a CTA barrier.
#ifndef SMG_GEMM_PNS
constexpr int PNS = 3;
#else
constexpr int PNS = SMG_GEMM_PNS;
#endif
#ifndef SMG_GEMM_BKP
constexpr int BKP = 16;  // k depth of a pipeline stage
#else
constexpr int BKP = SMG_GEMM_BKP;
#endif
constexpr int NT_P = NT + 32;

SMG_DEV uint32_t g_smem_u32(const void* ptr) { return static_cast<uint32_t>(__cvta_generic_to_shared(ptr)); }
SMG_DEV void g_mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(g_smem_u32(bar)), "r"(count) : "memory");
}
SMG_DEV void g_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(g_smem_u32(bar)) : "memory");
}
SMG_DEV void g_mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n GWAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra GWAIT_%=;\n}\n" ::"r"(g_smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// cp.async of one BK x XW slab into the Slab<XW, KMAJOR> layout, 16-byte chunks
// (zero-filled past kmax / xmax, partial chunks at odd edges)
template <int XW, bool KMAJOR>
SMG_DEV void issue_slab(double* sl, const double* __restrict__ ptr, int64_t ld, int k0, int x0, int kmax, int xmax,
                        int lane) {
    using SL = Slab<XW, KMAJOR, BKP>;
    constexpr int CH = KMAJOR ? XW / 2 : BKP / 2;  // chunks per smem row
    constexpr int NCH = XW * BKP / 2;
    for (int c = lane; c < NCH; c += 32) {
        int k, x;
        if (KMAJOR) {
            k = c / CH;
            x = (c % CH) * 2;
        } else {
            x = c / CH;
            k = (c % CH) * 2;
        }
        const int gk = k0 + k, gx = x0 + x;
        int valid;
        const double* src;
        if (KMAJOR) {
            valid = (gk < kmax) ? max(0, min(2, xmax - gx)) : 0;
            src = ptr + (int64_t)gk * ld + gx;
        } else {
            valid = (gx < xmax) ? max(0, min(2, kmax - gk)) : 0;
            src = ptr + (int64_t)gx * ld + gk;
        }
        if (valid == 0) src = ptr;
        double* dst = KMAJOR ? sl + k * SL::S + x : sl + x * SL::S + k;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(g_smem_u32(dst)), "l"(src),
                     "r"(valid * 8)
                     : "memory");
    }
}

// MW warps along M: 2 -> 64-row tiles (4 DMMA warps); 1 -> 32-row tiles (2 DMMA
// warps) for launches too small to fill the GPU (single chains)
template <int MW>
struct PipeShape {
    static constexpr int BMv = 32 * MW, NDW = 2 * MW, THREADS = 32 * NDW + 32, MINB = 4;
};

template <bool TA, bool TB, int NJ, int MW = 2, bool PROJ = false>
__global__ void __launch_bounds__(PipeShape<MW>::THREADS, PipeShape<MW>::MINB)
    gemm_pipe_kernel(GemmParams p, int n_base, int n_end) {
    constexpr int BN = 16 * NJ;
    constexpr int BM = PipeShape<MW>::BMv, NDW = PipeShape<MW>::NDW;
    using SA = Slab<BM, TA, BKP>;
    using SB = Slab<BN, !TB, BKP>;
    const int splits = p.splits > 0 ? p.splits : 1;
    const int b = blockIdx.z / splits;
    const int s = blockIdx.z % splits;
    if (p.skip && p.skip[b]) return;
    const int M = p.dimM ? p.dimM[(int64_t)b * p.dimStride] : p.M;
    const int N = min(p.dimN ? p.dimN[(int64_t)b * p.dimStride] : p.N, n_end);
    const int K = p.dimK ? p.dimK[(int64_t)b * p.dimStride] : p.K;
    const int m0 = blockIdx.y * BM, n0 = n_base + blockIdx.x * BN;
    if (m0 >= M || n0 >= N) return;
    if (p.syrkUpper && (m0 >> 5) > ((n0 + BN - 1) >> 5)) return;

    int kEnd = K;
    if (p.upperB) kEnd = min(kEnd, n0 + BN);
    const int kchunk = ((kEnd + splits - 1) / splits + BKP - 1) / BKP * BKP;
    const int kBeg = s * kchunk;
    const int kStop = min(kEnd, kBeg + kchunk);
    const int nsteps = kStop > kBeg ? (kStop - kBeg + BKP - 1) / BKP : 0;

    const double* A = p.A + (int64_t)b * p.strideA;
    const double* B = p.B + (int64_t)b * p.strideB;
    extern __shared__ __align__(16) double gsm[];
    double* As = gsm;
    double* Bs = gsm + PNS * SA::ELEMS;
    // diagonal tile of a Gram (V^T V, both operands the same k-major columns): the B slab
    // would duplicate the A slab -- load once, read twice (half the L2 traffic of that tile)
    const bool same_slab = TA && !TB && BM == BN && p.syrkUpper && p.A == p.B && p.lda == p.ldb &&
                           p.strideA == p.strideB && m0 == n0 && M == N;
    __shared__ __align__(8) uint64_t full[PNS], consumed[PNS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < PNS; ++i) {
            g_mbar_init(&full[i], 1);
            g_mbar_init(&consumed[i], NDW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == NDW) {  // producer
        uint32_t cph[PNS];
        for (int i = 0; i < PNS; ++i) cph[i] = 0u;
        for (int ks = 0; ks < nsteps; ++ks) {
            const int st = ks % PNS, k0 = kBeg + ks * BKP;
            if (ks >= PNS) {
                g_mbar_wait(&consumed[st], cph[st]);
                cph[st] ^= 1u;
            }
            // op(A)(m, k) lives at A[k*lda + m] (TA, k-major) or A[m*lda + k]
            issue_slab<BM, TA>(As + st * SA::ELEMS, A, p.lda, k0, m0, kStop, M, lane);
            if (!same_slab) issue_slab<BN, !TB>(Bs + st * SB::ELEMS, B, p.ldb, k0, n0, kStop, N, lane);
            asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(g_smem_u32(&full[st])) : "memory");
            __syncwarp();
            if (lane == 0) g_mbar_arrive(&full[st]);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        return;
    }

    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp % MW) * 32, wn = (warp / MW) * (8 * NJ);
    double acc[4][NJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr unsigned kFull = (1u << (4 * NJ)) - 1u;
    unsigned fmask = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int r = m0 + wm + 8 * i, cc = n0 + wn + 8 * j;
            bool on = r < M && cc < N;
            if (p.syrkUpper && (r >> 5) > ((cc + 7) >> 5)) on = false;
            if (on) fmask |= 1u << (NJ * i + j);
        }
    const int kdiag = p.upperB ? n0 + wn : 1 << 30;
    uint32_t fph[PNS];
    for (int i = 0; i < PNS; ++i) fph[i] = 0u;
    for (int ks = 0; ks < nsteps; ++ks) {
        const int st = ks % PNS, k0 = kBeg + ks * BKP;
        g_mbar_wait(&full[st], fph[st]);
        fph[st] ^= 1u;
        slab_mma<SA, SB, NJ>(As + st * SA::ELEMS, same_slab ? As + st * SA::ELEMS : Bs + st * SB::ELEMS, acc, fmask,
                             kFull, k0, kdiag, p.upperB, wm, wn, g, t);
        __syncwarp();
        if (lane == 0) g_mbar_arrive(&consumed[st]);
    }

    double* C;
    double alpha = p.alpha, beta = p.beta;
    if (splits > 1) {
        C = p.C + ((int64_t)b * splits + s) * p.strideP;
        alpha = 1.0;
        beta = 0.0;
    } else {
        C = p.C + (int64_t)b * p.strideC;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm + 8 * i + g;
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int col = n0 + wn + 8 * j + 2 * t + q;
                if (col >= N) continue;
                double* dst = C + (int64_t)row * p.ldc + col;
                double v = alpha * acc[i][j][q];
                if (beta != 0.0) v += beta * *dst;
                *dst = v;
            }
        }
    }
    if constexpr (PROJ) proj_epilogue<NJ>(p, acc, b, m0 + wm, n0 + wn, N, g, t);
}

__global__ void gemm_reduce_kernel(GemmParams p) {
    const int b = blockIdx.y;
    if (p.skip && p.skip[b]) return;
    const int M = p.dimM ? p.dimM[(int64_t)b * p.dimStride] : p.M;
    const int N = p.dimN ? p.dimN[(int64_t)b * p.dimStride] : p.N;
    const int64_t total = (int64_t)M * N;
    const double* W = p.C + (int64_t)b * p.splits * p.strideP;
    double* out = p.out + (int64_t)b * p.strideC;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / N), j = (int)(e % N);
        if (p.syrkUpper && (i >> 5) > (j >> 5)) continue;  // the Cholesky reads upper 32-blocks only
        double sum = 0.0;
        for (int s = 0; s < p.splits; ++s) sum += W[(int64_t)s * p.strideP + (int64_t)i * p.ldc + j];
        double v = p.alpha * sum;
        double* dst = out + (int64_t)i * p.ldo + j;
        if (p.beta != 0.0) v += p.beta * *dst;
        *dst = v;
    }
}

template <bool TA, bool TB, int NJ>
void launch_tiles(const GemmParams& p, int n_base, int width, cudaStream_t st) {
    constexpr int BN = 16 * NJ;
    const int gm = (p.M + BM - 1) / BM, gn = (width + BN - 1) / BN;
    dim3 grid(gn, gm, p.batch * p.splits);
    ::smg::count_launch();
    // the cp.async pipeline needs 16-byte aligned chunks: even leading
    // dimensions, strides and tile origins
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool aligned = al(p.A) && al(p.B) && !(p.lda & 1) && !(p.ldb & 1) && !(p.strideA & 1) && !(p.strideB & 1) &&
                         !(n_base & 1) && !std::getenv("SMG_GEMM_NOPIPE");
    if (aligned) {
        // a launch that cannot fill the GPU runs 32-row tiles (twice the CTAs)
        const bool small = (int64_t)gm * gn * p.batch * p.splits < 148 && !std::getenv("SMG_GEMM_NOSMALL");
        // projection partials in the epilogue: plain V * B products only
        constexpr bool CAN_PROJ = !TA && !TB;
        const bool proj = CAN_PROJ && p.projPart != nullptr && p.splits == 1;
        if (small) {
            using SA = Slab<32, TA, BKP>;
            using SB = Slab<BN, !TB, BKP>;
            const int bytes = PNS * (SA::ELEMS + SB::ELEMS) * 8;
            dim3 g2(gn, (p.M + 31) / 32, p.batch * p.splits);
            if (proj) {
                ensure_smem((const void*)gemm_pipe_kernel<TA, TB, NJ, 1, CAN_PROJ>, bytes);
                gemm_pipe_kernel<TA, TB, NJ, 1, CAN_PROJ><<<g2, PipeShape<1>::THREADS, bytes, st>>>(p, n_base, n_base + width);
            } else {
                ensure_smem((const void*)gemm_pipe_kernel<TA, TB, NJ, 1>, bytes);
                gemm_pipe_kernel<TA, TB, NJ, 1><<<g2, PipeShape<1>::THREADS, bytes, st>>>(p, n_base, n_base + width);
            }
            return;
        }
        using SA = Slab<BM, TA, BKP>;
        using SB = Slab<BN, !TB, BKP>;
        const int bytes = PNS * (SA::ELEMS + SB::ELEMS) * 8;
        if (proj) {
            ensure_smem((const void*)gemm_pipe_kernel<TA, TB, NJ, 2, CAN_PROJ>, bytes);
            gemm_pipe_kernel<TA, TB, NJ, 2, CAN_PROJ><<<grid, NT_P, bytes, st>>>(p, n_base, n_base + width);
        } else {
            ensure_smem((const void*)gemm_pipe_kernel<TA, TB, NJ>, bytes);
            gemm_pipe_kernel<TA, TB, NJ><<<grid, NT_P, bytes, st>>>(p, n_base, n_base + width);
        }
        return;
    }
    gemm_kernel<TA, TB, NJ><<<grid, NT, 0, st>>>(p, n_base, n_base + width);
}

template <bool TA, bool TB>
void launch_split(const GemmParams& p, cudaStream_t st) {
    // V * B with B upper triangular: the narrow tile takes the FIRST columns, so
    // its K range is `tail` instead of all of K.  The Gram keeps 32-aligned
    // tiles (unaligned ones straddle the diagonal blocks) and its narrow tile last.
    const int tail = p.N % 64, main = p.N - tail;
    const int t0 = p.upperB ? 0 : main, m0 = p.upperB ? tail : 0;
    switch ((tail + 15) / 16) {
        case 1: launch_tiles<TA, TB, 1>(p, t0, tail, st); break;
        case 2: launch_tiles<TA, TB, 2>(p, t0, tail, st); break;
        case 3: launch_tiles<TA, TB, 3>(p, t0, tail, st); break;
        case 4: launch_tiles<TA, TB, 4>(p, t0, tail, st); break;
        default: break;
    }
    if (main > 0) launch_tiles<TA, TB, 4>(p, m0, main, st);
}

}  // namespace

void gemm(const GemmParams& p0, bool transA, bool transB, cudaStream_t st) {
    GemmParams p = p0;
    if (p.splits < 1) p.splits = 1;
    if (p.M <= 0 || p.N <= 0 || p.batch == 0) return;
    if (transA && !transB) launch_split<true, false>(p, st);
    else if (!transA && !transB) launch_split<false, false>(p, st);
    else if (transA && transB) launch_split<true, true>(p, st);
    else launch_split<false, true>(p, st);
    if (p.splits > 1) {
        dim3 rg((unsigned)std::min<int64_t>(((int64_t)p.M * p.N + 255) / 256, 1024), p.batch);
        ::smg::count_launch(), gemm_reduce_kernel<<<rg, 256, 0, st>>>(p);
    }
}

}  // namespace smg

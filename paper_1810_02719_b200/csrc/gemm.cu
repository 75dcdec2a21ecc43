// Batched FP64 GEMM on the DMMA tensor path (mma.sync m8n8k4 f64).
//
// C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b], row-major operands.
// Used for the Gram V^T V (K5, split-K over the n_d rows, upper tiles only),
// the triangular right-multiply V * R^-1 (K7, B upper triangular so the K loop
// stops at the tile's last column), and the Rayleigh-Ritz products of the
// first-submesh basis (K9).  64x64x16 CTA tiles, 4 warps of 32x32, register
// prefetch of the next K slab while the current one is multiplied; split-K
// partials are summed in a fixed order by gemm_reduce (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128, SP = 68;  // SP: padded smem row (68 % 16 == 4)

template <bool KMAJOR>
struct TileLoader {
    // Loads the BK x 64 slab (k in [k0,k0+BK), x in [x0,x0+64)) of an operand whose
    // element (k, x) lives at ptr[k*ld + x] (KMAJOR) or ptr[x*ld + k] (!KMAJOR).
    double r[8];
    SMG_DEV void load(const double* __restrict__ ptr, int64_t ld, int k0, int x0, int kmax, int xmax) {
        const int tid = threadIdx.x;
        if (KMAJOR) {
            const int x = tid & 63, kb = tid >> 6;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = kb + 2 * j;
                const int gk = k0 + k, gx = x0 + x;
                r[j] = (gk < kmax && gx < xmax) ? __ldg(ptr + (int64_t)gk * ld + gx) : 0.0;
            }
        } else {
            const int k = tid & 15, xb = tid >> 4;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int x = xb + 8 * j;
                const int gk = k0 + k, gx = x0 + x;
                r[j] = (gk < kmax && gx < xmax) ? __ldg(ptr + (int64_t)gx * ld + gk) : 0.0;
            }
        }
    }
    SMG_DEV void store(double* __restrict__ s) const {
        const int tid = threadIdx.x;
        if (KMAJOR) {
            const int x = tid & 63, kb = tid >> 6;
#pragma unroll
            for (int j = 0; j < 8; ++j) s[(kb + 2 * j) * SP + x] = r[j];
        } else {
            const int k = tid & 15, xb = tid >> 4;
#pragma unroll
            for (int j = 0; j < 8; ++j) s[k * SP + xb + 8 * j] = r[j];
        }
    }
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_kernel(GemmParams p) {
    const int splits = p.splits > 0 ? p.splits : 1;
    const int b = blockIdx.z / splits;
    const int s = blockIdx.z % splits;
    const int M = p.dimM ? p.dimM[(int64_t)b * p.dimStride] : p.M;
    const int N = p.dimN ? p.dimN[(int64_t)b * p.dimStride] : p.N;
    const int K = p.dimK ? p.dimK[(int64_t)b * p.dimStride] : p.K;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    if (m0 >= M || n0 >= N) return;
    if (p.syrkUpper && blockIdx.y > blockIdx.x) return;

    int kEnd = K;
    if (p.upperB) kEnd = min(kEnd, n0 + BN);
    const int kchunk = ((kEnd + splits - 1) / splits + BK - 1) / BK * BK;
    const int kBeg = s * kchunk;
    const int kStop = min(kEnd, kBeg + kchunk);

    const double* A = p.A + (int64_t)b * p.strideA;
    const double* B = p.B + (int64_t)b * p.strideB;

    __shared__ __align__(16) double As[2][BK * SP];
    __shared__ __align__(16) double Bs[2][BK * SP];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // op(A) element (m, k): TA ? A[k*lda + m] : A[m*lda + k]  -> k-major iff TA
    // op(B) element (k, n): TB ? B[n*ldb + k] : B[k*ldb + n]  -> k-major iff !TB
    // fragments (8x8 of the warp's 32x32) that carry no output are skipped on the
    // DMMA pipe: rows >= M, cols >= N, and for syrkUpper the 32-blocks below the
    // diagonal (the Cholesky reads the upper triangle incl. full 32x32 diagonal blocks)
    unsigned fmask = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = m0 + wm + 8 * i, cc = n0 + wn + 8 * j;
            bool on = r < M && cc < N;
            if (p.syrkUpper && (r >> 5) > (cc >> 5)) on = false;
            if (on) fmask |= 1u << (4 * i + j);
        }

    TileLoader<TA> la;
    TileLoader<!TB> lb;
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
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = as[(kk + t) * SP + wm + 8 * i + g];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = bs[(kk + t) * SP + wn + 8 * j + g];
            unsigned m = fmask;
            if (p.upperB) {  // B[k][col] = 0 for k > col: fragment column block must reach k0 + kk
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (n0 + wn + 8 * j + 7 < k0 + kk) m &= ~(0x1111u << j);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (m & (1u << (4 * i + j))) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
        }
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
        for (int j = 0; j < 4; ++j) {
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
}

__global__ void gemm_reduce_kernel(GemmParams p) {
    const int b = blockIdx.y;
    const int M = p.dimM ? p.dimM[(int64_t)b * p.dimStride] : p.M;
    const int N = p.dimN ? p.dimN[(int64_t)b * p.dimStride] : p.N;
    const int64_t total = (int64_t)M * N;
    const double* W = p.C + (int64_t)b * p.splits * p.strideP;
    double* out = p.out + (int64_t)b * p.strideC;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / N), j = (int)(e % N);
        if (p.syrkUpper && (i / BM) > (j / BN)) continue;
        double sum = 0.0;
        for (int s = 0; s < p.splits; ++s) sum += W[(int64_t)s * p.strideP + (int64_t)i * p.ldc + j];
        double v = p.alpha * sum;
        double* dst = out + (int64_t)i * p.ldo + j;
        if (p.beta != 0.0) v += p.beta * *dst;
        *dst = v;
    }
}

}  // namespace

void gemm(const GemmParams& p0, bool transA, bool transB, cudaStream_t st) {
    GemmParams p = p0;
    if (p.splits < 1) p.splits = 1;
    const int gm = (p.M + BM - 1) / BM, gn = (p.N + BN - 1) / BN;
    if (gm == 0 || gn == 0 || p.batch == 0) return;
    dim3 grid(gn, gm, p.batch * p.splits);
    if (transA && !transB) ::smg::count_launch(), gemm_kernel<true, false><<<grid, NT, 0, st>>>(p);
    else if (!transA && !transB) ::smg::count_launch(), gemm_kernel<false, false><<<grid, NT, 0, st>>>(p);
    else if (transA && transB) ::smg::count_launch(), gemm_kernel<true, true><<<grid, NT, 0, st>>>(p);
    else ::smg::count_launch(), gemm_kernel<false, true><<<grid, NT, 0, st>>>(p);
    if (p.splits > 1) {
        dim3 rg((unsigned)std::min<int64_t>(((int64_t)p.M * p.N + 255) / 256, 1024), p.batch);
        ::smg::count_launch(), gemm_reduce_kernel<<<rg, 256, 0, st>>>(p);
    }
}

}  // namespace smg

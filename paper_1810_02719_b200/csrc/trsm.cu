// K7b: Q = V D^-1 R~^-1 as a right triangular solve (CholeskyQR pass 1).
//
// householderQ() (spectral.hpp:129) is the thin Q of the reference's QR; with
// the Cholesky factor R~ of the column-scaled Gram (cholqr.cu) it is
// Q = V D^-1 R~^-1.  Row blocks of Q are independent, so each CTA owns 64 rows
// of one chain and sweeps the 32-wide column panels left to right:
//   T   = V[:, p] D_p^-1 - sum_{s<p} Q[:, s] R~_{s,p}
//   Q_p = T X_pp,   X_pp = R~_pp^-1 (written by the Cholesky's diagonal phase)
// with the CTA's finished panels kept in shared memory and each panel's column
// of R~ staged once (64-row CTAs), or -- when a 64-row block of finished panels
// and the whole column would not fit (c > ~280) -- 32-row CTAs that stream the
// column of R~ through shared memory in 64-row chunks.  This replaces the explicit block back-substitution for
// R~^-1 -- a serial single-CTA phase of the Cholesky -- by row-parallel work.
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int TNT = 256;  // 8 warps: 4 (8 MI rows) x 2 (16 columns) over the (32 MI) x 32 panel
constexpr int PS36 = 36;  // 32-wide block stride (% 16 == 4)
constexpr int KC = 64;    // streamed R~ rows per chunk

// MI = 2: 64-row CTAs, whole R~ column staged; MI = 1 (CHUNK): 32-row CTAs,
// R~ column streamed in KC-row chunks
template <int MI, bool CHUNK>
struct TrsmCfg {
    static constexpr int TRB = 32 * MI;
    __host__ __device__ static int qs(int cp) { return cp + 4; }
    // CHUNK: two KC-row buffers (the next chunk streams in by cp.async while the
    // current one is multiplied)
    static int bytes(int cp) { return (TRB * qs(cp) + (CHUNK ? 2 * KC : cp) * PS36 + 32 * PS36 + TRB * PS36) * 8; }
};
using TrsmFull = TrsmCfg<2, false>;
using TrsmStream = TrsmCfg<1, true>;

template <int MI, bool CHUNK>
__global__ void __launch_bounds__(TNT) trsm_kernel(TrsmParams p) {
    using TC = TrsmCfg<MI, CHUNK>;
    constexpr int TRB = TC::TRB;
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y;
    if (p.status && p.status[b] != kOk) return;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int P = (c + 31) / 32, cp = (p.c_cap + 31) / 32 * 32;
    const int QS = TC::qs(cp);
    double* Qs = sm;                         // TRB x QS: finished panels of this row block
    double* Rc = Qs + TRB * QS;              // (cp | 2 x KC) x 36: column panel p of R~ (rows < p0)
    double* Xp = Rc + (CHUNK ? 2 * KC : cp) * PS36;  // 32 x 36: X_pp
    double* Tp = Xp + 32 * PS36;      // TRB x 36: T
    const int r0 = blockIdx.x * TRB;
    const double* V = p.V + (int64_t)b * p.strideV;
    double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* A = p.R + (int64_t)b * p.strideR;
    const double* Bo = p.Binv + (int64_t)b * p.strideB;
    const double* d = p.dscale + (int64_t)b * p.strideD;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;  // rows 8 MI wm .., columns 16 wn ..

    for (int pb = 0; pb < P; ++pb) {
        const int p0 = pb * 32;
        // stage R~[0:p0, p0:p0+32] (whole panel) and X_pp = d_row * B_pp
        if (!CHUNK)
            for (int e = tid; e < p0 * 32; e += TNT) {
                const int r = e >> 5, k = e & 31;
                Rc[r * PS36 + k] = A[(int64_t)r * p.ldr + p0 + k];
            }
        for (int e = tid; e < 32 * 32; e += TNT) {
            const int r = e >> 5, k = e & 31;
            Xp[r * PS36 + k] = Bo[(int64_t)(p0 + r) * p.ldb + p0 + k] * d[p0 + r];
        }
        // T starts as V[:, p] D^-1 (accumulator fragments)
        double acc[MI][2][2];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int row = r0 + 8 * MI * wm + 8 * i + g, col = p0 + 16 * wn + 8 * j + 2 * t + q;
                    acc[i][j][q] = (row < p.n) ? V[(int64_t)row * p.ldv + col] / d[col] : 0.0;
                }
        __syncthreads();
        // T -= Q[:, <p] R~[<p, p]
        // CHUNK: the R~ column streams through two KC-row buffers, chunk i+1
        // copied by cp.async while chunk i is multiplied
        const int nch = CHUNK ? (p0 + KC - 1) / KC : (p0 > 0 ? 1 : 0);
        auto stage = [&](int ci) {
            double* buf = Rc + (ci & 1) * KC * PS36;
            const int k0 = ci * KC, rows = min(KC, p0 - k0);
            for (int e = tid; e < rows * 16; e += TNT) {  // 16 pieces of 16 bytes per 32-double row
                const int r = e >> 4, q = e & 15;
                cp_async16(buf + r * PS36 + 2 * q, A + (int64_t)(k0 + r) * p.ldr + p0 + 2 * q);
            }
            cp_async_commit();
        };
        if (CHUNK && nch > 0) stage(0);
        for (int ci = 0; ci < nch; ++ci) {
            const int k0 = CHUNK ? ci * KC : 0;
            const int k1 = CHUNK ? min(p0, k0 + KC) : p0;
            const double* rc = Rc;
            if (CHUNK) {
                if (ci + 1 < nch) {
                    stage(ci + 1);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();  // chunk ci visible to every warp
                rc = Rc + (ci & 1) * KC * PS36;
            }
            for (int kk = k0; kk < k1; kk += 4) {
                const int kr = CHUNK ? kk - k0 : kk;
                double a[MI], bb[2];
#pragma unroll
                for (int i = 0; i < MI; ++i) a[i] = Qs[(8 * MI * wm + 8 * i + g) * QS + kk + t];
#pragma unroll
                for (int j = 0; j < 2; ++j) bb[j] = -rc[(kr + t) * PS36 + 16 * wn + 8 * j + g];
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
            }
            if (CHUNK) __syncthreads();  // buffer ci & 1 is re-staged at iteration ci + 1
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int r = 8 * MI * wm + 8 * i + g, cc = 16 * wn + 8 * j + 2 * t;
                Tp[r * PS36 + cc] = acc[i][j][0];
                Tp[r * PS36 + cc + 1] = acc[i][j][1];
            }
        __syncthreads();
        // Q_p = T X_pp
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
            double a[MI], bb[2];
#pragma unroll
            for (int i = 0; i < MI; ++i) a[i] = Tp[(8 * MI * wm + 8 * i + g) * PS36 + kk + t];
#pragma unroll
            for (int j = 0; j < 2; ++j) bb[j] = Xp[(kk + t) * PS36 + 16 * wn + 8 * j + g];
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int r = 8 * MI * wm + 8 * i + g, cc = 16 * wn + 8 * j + 2 * t;
                Qs[r * QS + p0 + cc] = acc[i][j][0];
                Qs[r * QS + p0 + cc + 1] = acc[i][j][1];
                const int row = r0 + r, col = p0 + cc;
                if (row < p.n) {
                    if (col < c) Q[(int64_t)row * p.ldq + col] = acc[i][j][0];
                    if (col + 1 < c) Q[(int64_t)row * p.ldq + col + 1] = acc[i][j][1];
                }
            }
        __syncthreads();
    }
}

}  // namespace

int trsm_smem_bytes(int c_cap) {
    const int cp = (c_cap + 31) / 32 * 32;
    const int full = TrsmFull::bytes(cp);
    return full <= 227 * 1024 ? full : TrsmStream::bytes(cp);
}

bool trsm_supported(int c_cap) { return trsm_smem_bytes(c_cap) <= 227 * 1024; }

void trsm_right_upper(const TrsmParams& p, cudaStream_t st) {
    const int cp = (p.c_cap + 31) / 32 * 32;
    const bool full = TrsmFull::bytes(cp) <= 227 * 1024;
    const int bytes = trsm_smem_bytes(p.c_cap);
    if (full) ensure_smem((const void*)trsm_kernel<2, false>, bytes);
    else ensure_smem((const void*)trsm_kernel<1, true>, bytes);
    if (full) {
        dim3 grid((p.n + TrsmFull::TRB - 1) / TrsmFull::TRB, p.batch);
        ::smg::count_launch(), trsm_kernel<2, false><<<grid, TNT, bytes, st>>>(p);
    } else {
        dim3 grid((p.n + TrsmStream::TRB - 1) / TrsmStream::TRB, p.batch);
        ::smg::count_launch(), trsm_kernel<1, true><<<grid, TNT, bytes, st>>>(p);
    }
}

}  // namespace smg

// F3: coarse reconstruction of many frames that share one connectivity and one
// set of tracked bases -- the frames stage of denoise_dynamic
// (denoise.hpp:258-291: bases from the first frame, then
// coarse_reconstruct_points(frame_i, bases, mode) for every frame,
// pipeline.hpp:290-305 + partition.hpp:311-355).
//
// Per submesh id the frames are batched into the columns of one operand, so a
// basis is streamed once per frame batch instead of once per frame:
//   X_t  = [x_1 y_1 z_1 ... x_F y_F z_F] (n_d x 3F, gathered by member id)
//   C_t  = U_t^T X_t   (c x 3F, DMMA GEMM, split-K over n_d when few tiles)
//   X^_t = U_t C_t     (n_d x 3F, DMMA GEMM)
// and the stitch averages every vertex's copies in submesh-id order with the
// local degree (Weighted) or 1 (Simple) as the weight.  U_t is the caller's
// column-major n_d x c basis (Eigen layout), read in place: as a row-major
// c x n_d matrix it is A for the first product and A^T for the second.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "profiler.h"

namespace smg {

namespace {

// local_degrees (partition.hpp:177-184): neighbours of each member inside its
// submesh; members sorted ascending, looked up by binary search in smem.
__global__ void local_degree_kernel(const int32_t* members, int n_d, const int32_t* adj_offsets,
                                    const int32_t* adj_cols, int32_t* deg) {
    extern __shared__ int32_t smem_members[];
    const int32_t* mem = members + (int64_t)blockIdx.x * n_d;
    for (int i = threadIdx.x; i < n_d; i += blockDim.x) smem_members[i] = mem[i];
    __syncthreads();
    for (int i = threadIdx.x; i < n_d; i += blockDim.x) {
        const int g = smem_members[i];
        int d = 0;
        for (int e = adj_offsets[g]; e < adj_offsets[g + 1]; ++e) {
            const int w = adj_cols[e];
            int lo = 0, hi = n_d;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (smem_members[mid] < w) lo = mid + 1;
                else hi = mid;
            }
            d += (lo < n_d && smem_members[lo] == w);
        }
        deg[(int64_t)blockIdx.x * n_d + i] = d;
    }
}

// X_t[i][3f + a] = frame_f.axis_a[members_t[i]]; rows padded to ldx columns (zeros)
__global__ void gather_frames_kernel(const int32_t* members, int n_d, const double* const* xyz, int f0, int F,
                                     double* X, int ldx) {
    const int t = blockIdx.y;
    const int32_t* mem = members + (int64_t)t * n_d;
    double* Xt = X + (int64_t)t * n_d * ldx;
    const int64_t total = (int64_t)n_d * ldx;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / ldx), col = (int)(e % ldx);
        double v = 0.0;
        if (col < 3 * F) {
            const int f = col / 3, a = col % 3;
            v = xyz[3 * (f0 + f) + a][mem[i]];
        }
        Xt[e] = v;
    }
}

// partition.hpp:321-346 for F frames at once; owners of g sorted by submesh id
__global__ void stitch_frames_kernel(int n, int n_d, int weighted, const int32_t* offs, const int64_t* slots,
                                     const int32_t* deg, const double* xhat, int ldx, int f0, int F,
                                     double* const* out) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
        const int s = offs[g], e = offs[g + 1];
        const int copies = e - s;
        for (int f = 0; f < F; ++f) {
            double o[3] = {0.0, 0.0, 0.0}, fb[3] = {0.0, 0.0, 0.0}, ws = 0.0;
            for (int q = s; q < e; ++q) {
                const int64_t slot = slots[q];  // submesh id * n_d + local index
                const double w = weighted ? (double)deg[slot] : 1.0;
                const double* xh = xhat + slot * ldx + 3 * f;
                for (int a = 0; a < 3; ++a) {
                    o[a] += w * xh[a];
                    fb[a] += xh[a];
                }
                ws += w;
            }
            double* dst = out[f0 + f];
            for (int a = 0; a < 3; ++a) {
                double v;
                if (copies == 0) v = 0.0;
                else if (ws > 0.0) v = o[a] / ws;
                else v = fb[a] / (double)copies;
                dst[(int64_t)a * n + g] = v;
            }
        }
    }
}

inline int grid_for(int64_t total, int nt, int cap = 8192) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((total + nt - 1) / nt, cap));
}

}  // namespace

void local_degrees(const int32_t* members, int k, int n_d, const int32_t* adj_offsets, const int32_t* adj_cols,
                   int32_t* deg, cudaStream_t st) {
    if (k <= 0) return;
    ::smg::count_launch(), local_degree_kernel<<<k, 256, sizeof(int32_t) * n_d, st>>>(members, n_d, adj_offsets,
                                                                                      adj_cols, deg);
}

int frames_batch(const FramesParams& p) {
    // X_t and X^_t for one batch: 2 * k * n_d * ldx doubles, kept under ~2 GB
    const int64_t per_frame = (int64_t)p.k * p.n_d * 3 * 8 * 2;
    const int64_t budget = (int64_t)2 << 30;
    if (const char* e = std::getenv("SMG_FRAMES_BATCH")) return std::max(1, std::min(p.frames, std::atoi(e)));
    return (int)std::max<int64_t>(1, std::min<int64_t>(p.frames, std::min<int64_t>(128, budget / per_frame)));
}

void coarse_reconstruct_frames(const FramesParams& p, const FramesWork& w, cudaStream_t st) {
    const int FB = w.batch_frames;
    for (int f0 = 0; f0 < p.frames; f0 += FB) {
        const int F = std::min(FB, p.frames - f0);
        const int ldx = (3 * F + 7) / 8 * 8;
        ::smg::count_launch(), gather_frames_kernel<<<dim3(grid_for((int64_t)p.n_d * ldx, 256, 64), p.k), 256, 0, st>>>(
            p.members, p.n_d, p.xyz, f0, F, w.X, ldx);
        {
            ProfScope ps("frames_gemm", st);
            // C_t = U_t^T X_t: U_t column-major n_d x c == row-major c x n_d (lda = n_d)
            GemmParams g;
            g.M = p.c_cap;
            g.N = 3 * F;
            g.K = p.n_d;
            g.batch = p.k;
            g.A = p.bases;
            g.lda = p.n_d;
            g.strideA = p.strideU;
            g.B = w.X;
            g.ldb = ldx;
            g.strideB = (int64_t)p.n_d * ldx;
            g.dimM = p.dimC;
            g.dimStride = 1;
            const int tiles = ((p.c_cap + 63) / 64) * ((3 * F + 63) / 64) * p.k;
            const int splits = std::max(1, std::min(p.n_d / 256, (2 * 148 + tiles - 1) / std::max(1, tiles)));
            g.splits = splits;
            if (splits > 1) {
                g.C = w.Cws;
                g.ldc = ldx;
                g.strideP = (int64_t)p.c_cap * ldx;
                g.out = w.C;
                g.ldo = ldx;
                g.strideC = (int64_t)p.c_cap * ldx;
            } else {
                g.C = w.C;
                g.ldc = ldx;
                g.strideC = (int64_t)p.c_cap * ldx;
        }
        gemm(g, false, false, st);
        // X^_t = U_t C_t: op(A) = U_t, stored as row-major c x n_d -> transposed
        GemmParams h;
        h.M = p.n_d;
        h.N = 3 * F;
        h.K = p.c_cap;
        h.batch = p.k;
        h.A = p.bases;
        h.lda = p.n_d;
        h.strideA = p.strideU;
        h.B = w.C;
        h.ldb = ldx;
        h.strideB = (int64_t)p.c_cap * ldx;
        h.C = w.Xhat;
        h.ldc = ldx;
        h.strideC = (int64_t)p.n_d * ldx;
        h.dimK = p.dimC;
        h.dimStride = 1;
        gemm(h, true, false, st);
        }
        ::smg::count_launch(), stitch_frames_kernel<<<grid_for(p.n, 256, 4096), 256, 0, st>>>(
            p.n, p.n_d, p.weighted, p.owner_offs, p.owner_slots, p.deg, w.Xhat, ldx, f0, F, p.out);
    }
}

void reconstruct_from_coefficients(const FramesParams& p, const double* C, int ldc, double* Xhat, cudaStream_t st) {
    GemmParams h;
    h.M = p.n_d;
    h.N = 3;
    h.K = p.c_cap;
    h.batch = p.k;
    h.A = p.bases;
    h.lda = p.n_d;
    h.strideA = p.strideU;
    h.B = C;
    h.ldb = ldc;
    h.strideB = (int64_t)p.c_cap * ldc;
    h.C = Xhat;
    h.ldc = ldc;
    h.strideC = (int64_t)p.n_d * ldc;
    h.dimK = p.dimC;
    h.dimStride = 1;
    gemm(h, true, false, st);
    ::smg::count_launch(), stitch_frames_kernel<<<grid_for(p.n, 256, 4096), 256, 0, st>>>(
        p.n, p.n_d, p.weighted, p.owner_offs, p.owner_slots, p.deg, Xhat, ldc, 0, 1, p.out);
}

}  // namespace smg

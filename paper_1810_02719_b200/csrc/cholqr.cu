// K6: c x c Cholesky of the column-scaled Gram matrix, the reference rank test,
// and the scaled triangular inverse used by CholeskyQR2.
//
// orthonormalize (spectral.hpp:120-132) computes a Householder QR and throws
// "rank deficient at column k" for the first k with |r_kk| < 1e-13 ||block||_F.
// CholeskyQR gives the same R up to column signs: with D = diag(||v_j||) and
// G~ = D^-1 V^T V D^-1 = R~^T R~, R = R~ D, so |r_kk| = r~_kk d_k and ||block||_F
// = sqrt(trace G).  Column scaling makes the test exact for the column-graded
// blocks R^z U produces (SURVEY.md §0 finding 5).  A non-positive pivot means
// r~_kk is below rounding, reported as rank deficiency at that column.
// Output Binv = D^-1 R~^-1 (upper), so Q1 = V Binv is one triangular GEMM.
// One CTA per batch entry; the working matrix lives in shared memory when it
// fits (c <= 144) and in L2 otherwise.
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int NT = 512;
constexpr int SMEM_C = 144;

__global__ void __launch_bounds__(NT) chol_kernel(CholParams p) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[32];
    __shared__ double d[512];
    const int b = blockIdx.x;
    if (p.status[b] != kOk) return;  // this chain already failed (sticky first error)
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const double* G = p.G + (int64_t)b * p.strideG;
    double* Bo = p.Binv + (int64_t)b * p.strideB;
    double* rdiag = p.rdiag ? p.rdiag + (int64_t)b * p.strideR : nullptr;
    const bool in_smem = c <= SMEM_C;
    const int ld = in_smem ? c : p.c_cap;
    double* A = in_smem ? sm : p.work + (int64_t)b * p.c_cap * p.c_cap;
    const int tid = threadIdx.x;
    auto record = [&](int kind, int64_t col) {
        p.status[b] = kind;
        if (p.status_detail) p.status_detail[b] = col;
        if (p.errpos) p.errpos[b] = p.pos;
    };

    // column norms and ||V||_F
    double tr = 0.0;
    for (int j = tid; j < c; j += NT) {
        const double gjj = G[(int64_t)j * p.ldg + j];
        d[j] = p.column_scale ? sqrt(gjj) : 1.0;
        tr += gjj;
    }
    tr = block_sum(tr, red);
    const double scale = sqrt(tr);
    if (tid == 0 && p.vnorm) p.vnorm[b] = scale;
    if (!(scale > 0.0) || !isfinite(scale)) {
        if (tid == 0) record(scale == 0.0 ? kAllZero : kNotFinite, -1);
        return;
    }
    const double thresh = 1e-13 * scale;
    // scaled upper triangle
    for (int e = tid; e < c * c; e += NT) {
        const int i = e / c, k = e % c;
        if (k >= i) {
            const double di = d[i], dk = d[k];
            A[i * ld + k] = (di > 0.0 && dk > 0.0) ? G[(int64_t)i * p.ldg + k] / di / dk : 0.0;
        }
    }
    __syncthreads();
    // right-looking Cholesky, upper: A = R~^T R~
    int stop = c;
    for (int j = 0; j < c; ++j) {
        const double piv = A[j * ld + j];
        const double rjj = sqrt(piv);
        // A scaled pivot below 1e-12 means r~_jj < 1e-6: beyond what the Gram
        // resolves, i.e. numerically dependent -- the rank-test verdict.
        const bool bad_piv = !(piv > (p.rank_test ? 1e-12 : 0.0)) || !isfinite(piv) || !(d[j] > 0.0);
        const double rkk = bad_piv ? 0.0 : rjj * d[j];
        if (bad_piv || (p.rank_test && rkk < thresh)) {
            if (tid == 0) {
                record(p.rank_test ? kRankDeficient : kNotFinite, j);
                if (rdiag) rdiag[j] = rkk;
            }
            stop = j;
            break;
        }
        for (int k = j + 1 + tid; k < c; k += NT) A[j * ld + k] /= rjj;
        __syncthreads();
        if (tid == 0) {
            A[j * ld + j] = rjj;
            if (rdiag) rdiag[j] = rkk;
        }
        const int m = c - j - 1;
        for (int e = tid; e < m * m; e += NT) {
            const int i = j + 1 + e / m, k = j + 1 + e % m;
            if (k >= i) A[i * ld + k] -= A[j * ld + i] * A[j * ld + k];
        }
        __syncthreads();
    }
    __syncthreads();
    if (stop < c) return;
    // Binv = R~^-1 row-scaled by 1/d: rows from the bottom; row i depends on rows > i.
    // Stored in Bo (upper, ld p.ldb); lower part zeroed.
    for (int e = tid; e < c * c; e += NT) {
        const int i = e / c, k = e % c;
        if (k < i) Bo[(int64_t)i * p.ldb + k] = 0.0;
    }
    // X = R~^-1 computed in place in the lower-unused layout: use Bo as X (unscaled), scale at the end
    for (int i = c - 1; i >= 0; --i) {
        const double rii = A[i * ld + i];
        for (int k = i + tid; k < c; k += NT) {
            double v;
            if (k == i) {
                v = 1.0 / rii;
            } else {
                double acc = 0.0;
                for (int l = i + 1; l <= k; ++l) acc += A[i * ld + l] * Bo[(int64_t)l * p.ldb + k];
                v = -acc / rii;
            }
            Bo[(int64_t)i * p.ldb + k] = v;
        }
        __syncthreads();
    }
    for (int e = tid; e < c * c; e += NT) {
        const int i = e / c, k = e % c;
        if (k >= i) Bo[(int64_t)i * p.ldb + k] /= d[i];
    }
}

// partial diag(Q^T V) over a chunk of rows, threads over columns (coalesced rows)
constexpr int RC_ROWS = 128;
__global__ void rank_partial_kernel(RankCheckParams p) {
    const int b = blockIdx.y, chunk = blockIdx.x;
    if (p.status[b] != kOk) return;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int r0 = chunk * RC_ROWS, r1 = min(p.n, r0 + RC_ROWS);
    const double* Q = p.Q + (int64_t)b * p.stride;
    const double* V = p.V + (int64_t)b * p.stride;
    for (int k = threadIdx.x; k < c; k += blockDim.x) {
        double acc = 0.0;
        for (int i = r0; i < r1; ++i) acc = fma(Q[(int64_t)i * p.ld + k], V[(int64_t)i * p.ld + k], acc);
        p.partial[((int64_t)b * gridDim.x + chunk) * p.c_cap + k] = acc;
    }
}

__global__ void rank_test_kernel(RankCheckParams p, int nchunks) {
    __shared__ int first;
    const int b = blockIdx.x;
    if (p.status[b] != kOk) return;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    if (threadIdx.x == 0) first = c;
    __syncthreads();
    const double thresh = 1e-13 * p.vnorm[b];
    for (int k = threadIdx.x; k < c; k += blockDim.x) {
        double r = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) r += p.partial[((int64_t)b * nchunks + ch) * p.c_cap + k];
        if (!(fabs(r) >= thresh)) atomicMin(&first, k);
    }
    __syncthreads();
    if (threadIdx.x == 0 && first < c) {
        p.status[b] = kRankDeficient;
        if (p.status_detail) p.status_detail[b] = first;
        if (p.errpos) p.errpos[b] = p.pos;
    }
}

}  // namespace

void rank_check(const RankCheckParams& p, cudaStream_t st) {
    const int chunks = (p.n + RC_ROWS - 1) / RC_ROWS;
    ::smg::count_launch(), rank_partial_kernel<<<dim3(chunks, p.batch), 256, 0, st>>>(p);
    ::smg::count_launch(), rank_test_kernel<<<p.batch, 256, 0, st>>>(p, chunks);
}

void chol_inverse(const CholParams& p, cudaStream_t st) {
    const int bytes = std::min(p.c_cap, SMEM_C) * std::min(p.c_cap, SMEM_C) * 8;
    static int configured = 0;
    if (!configured) {
        cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_C * SMEM_C * 8);
        configured = 1;
    }
    ::smg::count_launch(), chol_kernel<<<p.batch, NT, bytes, st>>>(p);
}

}  // namespace smg

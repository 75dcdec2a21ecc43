// Small device-side controllers of the chain: Ritz residual norms for the
// first-submesh basis (K9) and the DOI grow/shrink/stop decision (K10,
// spectral.hpp:259-283) that runs on the device so the dynamic-c loop needs no
// host round-trip per step (it drives a CUDA-graph conditional while node).
#include "chain.h"
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

__global__ void ritz_partial_kernel(const double* LZ, const double* Z, const double* theta, int n, int ncols,
                                    int64_t ld, int64_t stride, int64_t strideTheta, double* partial, int rows) {
    const int b = blockIdx.y, chunk = blockIdx.x;
    const int r0 = chunk * rows, r1 = min(n, r0 + rows);
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) {
        const double th = theta[(int64_t)b * strideTheta + j];
        double acc = 0.0;
        for (int i = r0; i < r1; ++i) {
            const double r = LZ[(int64_t)b * stride + (int64_t)i * ld + j] - th * Z[(int64_t)b * stride + (int64_t)i * ld + j];
            acc = fma(r, r, acc);
        }
        partial[((int64_t)b * gridDim.x + chunk) * ncols + j] = acc;
    }
}

__global__ void ritz_reduce_kernel(const double* partial, int nchunks, int ncols, double* out) {
    const int b = blockIdx.x;
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nchunks; ++k) s += partial[((int64_t)b * nchunks + k) * ncols + j];
        out[(int64_t)b * ncols + j] = sqrt(s);
    }
}

// spectral.hpp:259-283, one thread per chain.  Called after the OI step and the
// projection of step t: stats[1] = ||e||.  Decides, records DoiResult fields
// and prepares the next step (append e/||e|| as column c, or drop column c-1).
__global__ void doi_decide_kernel(DoiState* states, int batch, const double* stats, int64_t strideStats,
                                  cudaGraphConditionalHandle handle, int use_handle, const int* chain_status,
                                  int* trace_c, double* trace_r) {
    bool any_active = false;
    for (int b = 0; b < batch; ++b) {
        DoiState& s = states[b];
        if (!s.active) continue;
        s.t += 1;
        s.appended_raw = 0;
        s.append_scale = 0.0;
        const double en = stats[(int64_t)b * strideStats + 1];
        s.enorm = en;
        s.residual = en / s.scale;
        if (trace_c && batch == 1) {  // step log for decision-level parity (c before the decision)
            trace_c[s.t - 1] = s.c;
            trace_r[s.t - 1] = s.residual;
        }
        if (chain_status && chain_status[b] != 0) s.status = chain_status[b];
        if (s.status != 0) {
            s.active = 0;
        } else if (s.residual > s.eps_high) {
            if (s.c >= s.c_max) {
                s.active = 0;  // bound hit, still above the band: unconverged
            } else {
                s.append_col = s.c;
                s.append_scale = 1.0 / en;
                s.c += 1;
                s.appended_raw = 1;
            }
        } else if (s.residual < s.eps_low) {
            if (s.c <= s.c_min) {
                s.converged = 1;
                s.active = 0;
            } else {
                s.c -= 1;
            }
        } else {
            s.converged = 1;
            s.active = 0;
        }
        if (s.active && s.t >= s.t_max) s.active = 0;
        if (s.active) any_active = true;
    }
    if (use_handle) cudaGraphSetConditional(handle, any_active ? 1u : 0u);
}

// U[:, append_col] = e / ||e|| for chains that decided to grow.
__global__ void doi_append_kernel(const DoiState* states, double* U, int64_t ldu, int64_t strideU, const double* e,
                                  int64_t strideE, int n) {
    const int b = blockIdx.y;
    const DoiState& s = states[b];
    if (!s.appended_raw) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        U[(int64_t)b * strideU + (int64_t)i * ldu + s.append_col] = e[(int64_t)b * strideE + i] * s.append_scale;
}

__global__ void delta_kernel(const double* trace, int ntiles, int n, double scale, double* delta) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        const double mean_diag = trace[t] / (double)n;
        delta[t] = fmax(scale * mean_diag, 1e-300);  // default_shift, spectral.hpp:193-196
    }
}

// first-basis shift: Gershgorin lower bound of L, then + 1e-3 * mean diagonal;
// shift[ntiles + t] = Gershgorin upper bound (Chebyshev filter interval end)
__global__ void first_shift_kernel(const int32_t* rowptr, const int32_t* cols, const double* vals,
                                   const int64_t* csr_offsets, const double* trace, int ntiles, int n, double* shift) {
    __shared__ double red[32], redh[32];
    const int t = blockIdx.x;
    const int32_t* rp = rowptr + (int64_t)t * (n + 1);
    const double* v = vals + csr_offsets[t];
    const int32_t* c = cols + csr_offsets[t];
    double lo = INFINITY, hi = -INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double diag = 0.0, off = 0.0;
        for (int e = rp[i]; e < rp[i + 1]; ++e) {
            if (c[e] == i) diag = v[e];
            else off += fabs(v[e]);
        }
        lo = fmin(lo, diag - off);
        hi = fmax(hi, diag + off);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = lo;
        redh[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = INFINITY, h = -INFINITY;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            m = fmin(m, red[w]);
            h = fmax(h, redh[w]);
        }
        shift[t] = fmax(0.0, -m) + 1e-3 * (trace[t] / (double)n) + 1e-300;
        shift[ntiles + t] = h;
    }
}

// coefficients out: C = sign * P, column-major c x 3 per submesh
__global__ void coeff_out_kernel(const double* coef, int64_t strideCoef, const double* sign, int64_t strideSign,
                                 const int* dimC, int64_t dimStride, int c_fixed, double* out,
                                 const int64_t* out_offsets, const int32_t* ids) {
    const int b = blockIdx.x;
    const int c = dimC ? dimC[(int64_t)b * dimStride] : c_fixed;
    double* o = out + out_offsets[ids[b]];
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
        const double s = sign[(int64_t)b * strideSign + j];
        for (int a = 0; a < 3; ++a) o[(int64_t)a * c + j] = s * coef[(int64_t)b * strideCoef + 4 * j + a];
    }
}

}  // namespace

void ritz_residual(const double* LZ, const double* Z, const double* theta, int n, int ncols, int64_t ld,
                   int64_t stride, int64_t strideTheta, int batch, double* partial, double* out, cudaStream_t st) {
    const int rows = 128;
    const int chunks = (n + rows - 1) / rows;
    ::smg::count_launch(), ritz_partial_kernel<<<dim3(chunks, batch), 256, 0, st>>>(LZ, Z, theta, n, ncols, ld, stride, strideTheta,
                                                              partial, rows);
    ::smg::count_launch(), ritz_reduce_kernel<<<batch, 256, 0, st>>>(partial, chunks, ncols, out);
}

void doi_decide(DoiState* states, int batch, const double* stats, int64_t strideStats,
                cudaGraphConditionalHandle handle, int use_handle, const int* chain_status, cudaStream_t st,
                int* trace_c, double* trace_r) {
    ::smg::count_launch(), doi_decide_kernel<<<1, 1, 0, st>>>(states, batch, stats, strideStats, handle, use_handle, chain_status,
                                                             trace_c, trace_r);
}

void doi_append(const DoiState* states, double* U, int64_t ldu, int64_t strideU, const double* e, int64_t strideE,
                int n, int batch, cudaStream_t st) {
    ::smg::count_launch(), doi_append_kernel<<<dim3((n + 255) / 256, batch), 256, 0, st>>>(states, U, ldu, strideU, e, strideE, n);
}

void compute_delta(const double* trace, int ntiles, int n, double scale, double* delta, cudaStream_t st) {
    if (ntiles) ::smg::count_launch(), delta_kernel<<<(ntiles + 255) / 256, 256, 0, st>>>(trace, ntiles, n, scale, delta);
}

void compute_first_shift(const int32_t* rowptr, const int32_t* cols, const double* vals, const int64_t* csr_offsets,
                         const double* trace, int ntiles, int n, double* shift, cudaStream_t st) {
    if (ntiles) ::smg::count_launch(), first_shift_kernel<<<ntiles, 256, 0, st>>>(rowptr, cols, vals, csr_offsets, trace, ntiles, n, shift);
}

void coeff_out(const double* coef, int64_t strideCoef, const double* sign, int64_t strideSign, const int* dimC,
               int64_t dimStride, int c_fixed, double* out, const int64_t* out_offsets, const int32_t* ids, int batch,
               cudaStream_t st) {
    ::smg::count_launch(), coeff_out_kernel<<<batch, 128, 0, st>>>(coef, strideCoef, sign, strideSign, dimC, dimStride, c_fixed, out,
                                            out_offsets, ids);
}

}  // namespace smg

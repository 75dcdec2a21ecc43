// Device-side chain state and controller launches (chain.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace smg {

// dynamic_oi loop state (spectral.hpp:244-287), one per chain, device resident.
struct DoiState {
    int c;             // columns of U for the next step (incl. a pending raw append)
    int t;             // OI steps done (DoiResult::iterations)
    int active;        // loop continues
    int appended_raw;  // last decision appended e/||e|| (spectral.hpp:257, :272)
    int converged;
    int append_col;
    int c_min, c_max, t_max;
    int status;        // sticky numerical status of this chain (rank deficiency ...)
    double eps_low, eps_high;
    double scale;      // bounding_box_diagonal or 1
    double residual;   // ||e|| / scale
    double enorm;
    double append_scale;
};

void ritz_residual(const double* LZ, const double* Z, const double* theta, int n, int ncols, int64_t ld,
                   int64_t stride, int64_t strideTheta, int batch, double* partial, double* out, cudaStream_t st);
// trace (optional, batch 1): per step t (0-based) the subspace size the step ran
// with (trace_c[t]) and its residual ||e|| / scale (trace_r[t]), t < t_max
void doi_decide(DoiState* states, int batch, const double* stats, int64_t strideStats,
                cudaGraphConditionalHandle handle, int use_handle, const int* chain_status, cudaStream_t st,
                int* trace_c = nullptr, double* trace_r = nullptr);
void doi_append(const DoiState* states, double* U, int64_t ldu, int64_t strideU, const double* e, int64_t strideE,
                int n, int batch, cudaStream_t st);
void compute_delta(const double* trace, int ntiles, int n, double scale, double* delta, cudaStream_t st);
void compute_first_shift(const int32_t* rowptr, const int32_t* cols, const double* vals, const int64_t* csr_offsets,
                         const double* trace, int ntiles, int n, double* shift, cudaStream_t st);
void coeff_out(const double* coef, int64_t strideCoef, const double* sign, int64_t strideSign, const int* dimC,
               int64_t dimStride, int c_fixed, double* out, const int64_t* out_offsets, const int32_t* ids, int batch,
               cudaStream_t st);

}  // namespace smg

// Common device helpers for the sm_100a OI spectral path.
//
// FP64 arithmetic only.  tcgen05 (UMMA) has no f64 kind, so FP64 tensor work is
// the warp-level DMMA `mma.sync.aligned.m8n8k4.row.col.f64` (37.2 TFLOP/s on
// B200 vs 36.8 for DFMA; profiles/fp64_peak_r01.txt).  Matrices inside the
// library are row-major ("vertex-major": row = local vertex, leading dimension
// ld >= c, ld % 8 == 0); the C ABI converts Eigen's column-major at the boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SMG_DEV __device__ __forceinline__

namespace smg {

// D(8x8) += A(8x4, row) * B(4x8, col).  Lane l: g = l >> 2, t = l & 3 holds
// a = A[g][t], b = B[t][g]; d0 = D[g][2t], d1 = D[g][2t+1].
#ifndef SMG_DMMA_ASM
#define SMG_DMMA_ASM asm volatile
#endif
SMG_DEV void dmma884(double& d0, double& d1, double a, double b) {
    SMG_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// D(16x8) += A(16x8, row) * B(8x8, col), f64 (layout verified on B200 by
// tools/dmma16_layout.cu): a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4],
// a3 = A[g+8][t+4]; b0 = B[t][g], b1 = B[t+4][g]; d0/d1 = D[g][2t, 2t+1],
// d2/d3 = D[g+8][2t, 2t+1] -- i.e. two stacked m8n8k4 accumulator tiles.
SMG_DEV void dmma1688(double& d0, double& d1, double& d2, double& d3, double a0, double a1, double a2, double a3,
                      double b0, double b1) {
    SMG_DMMA_ASM("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+d"(d0), "+d"(d1), "+d"(d2), "+d"(d3)
                 : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

SMG_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

SMG_DEV double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

SMG_DEV void cp_async16(void* smem, const void* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
SMG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
SMG_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Block-wide sum of one double per thread (blockDim.x multiple of 32, <= 1024).
SMG_DEV double block_sum(double v, double* scratch /* >= 32 doubles */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    double r = 0.0;
    if (wid == 0) {
        r = lane < nw ? scratch[lane] : 0.0;
        r = warp_sum(r);
        if (lane == 0) scratch[0] = r;
    }
    __syncthreads();
    r = scratch[0];
    __syncthreads();
    return r;
}

// Rank test certification margins (pass-1 Cholesky of the column-scaled Gram,
// unit diagonal): a scaled pivot >= 1e-8 is known to relative 1e-6 (absolute
// pivot error ~ c * eps), and r_kk >= 1e-9 ||V||_F is 1e4 above the reference
// threshold 1e-13 ||V||_F (spectral.hpp:126-128), so |q_k^T v_k| passes for sure.
constexpr double kRankCertPiv = 1e-8;
constexpr double kRankCertRel = 1e-9;

// Status codes written by kernels into device status words.
enum DeviceStatus : int {
    kOk = 0,
    kRankDeficient = 1,      // detail = column
    kAllZero = 2,            // orthonormalize: block all zero
    kFactorFailed = 3,       // zero pivot in LDL^T
    kCoincident = 4,         // distance weighting singular; detail = pair
    kNotFinite = 5,
};

}  // namespace smg

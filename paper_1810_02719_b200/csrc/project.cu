// K8 (+A9, A16, A20): sign convention, spectral projection, reconstruction and
// the two residuals, fused over the freshly orthonormalised basis.
//
//  * apply_sign_convention (spectral.hpp:72-85): per column argmax |q_ij| with
//    the first index winning ties, flip if negative.  The flip is kept as a sign
//    vector instead of rewriting Q: Q~ Q~^T is sign invariant, the next OI step
//    is too (its QR re-normalises signs), and the sign is applied where the
//    basis or the coefficients leave the library.
//  * gft (spectral.hpp:290-293): C = S Q~^T X  (c x 3).
//  * igft + projection_residual_rms (spectral.hpp:295-298, :223-226):
//    X^ = Q~ (Q~^T X), rms = sqrt(||X - X^||_F^2 / (3 n)).
//  * projection_residual (spectral.hpp:216-220): e = s - Q~ (Q~^T s), s = x+y+z,
//    the DOI control signal, and ||e||.
// Pass 1 (per row chunk, threads over columns, coalesced rows of Q) produces
// partial column maxima and partial Q^T [X | s]; pass 2 reduces them in chunk
// order (deterministic); pass 3 (warp per row) rebuilds X^ and e; pass 4 sums
// the per-CTA residual partials in a fixed order.
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int PNT = 256;

SMG_DEV void reduce_block(const ProjParams& p, int b) {
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const double* part = p.partial + (int64_t)b * p.nchunks * (int64_t)p.c_cap * 8;
    double* coef = p.coeff + (int64_t)b * p.strideCoef;  // c x 4: Px Py Pz Ps (unsigned)
    double* sign = p.sign + (int64_t)b * p.strideSign;
    for (int j = threadIdx.x; j < c; j += PNT) {
        double best = -1.0, bval = 0.0;
        double px = 0.0, py = 0.0, pz = 0.0, ps = 0.0;
        for (int ch = 0; ch < p.nchunks; ++ch) {
            const double* o = part + ((int64_t)ch * p.c_cap + j) * 8;
            if (o[0] > best) {  // chunks in row order: strict > keeps the first index
                best = o[0];
                bval = o[1];
            }
            px += o[3];
            py += o[4];
            pz += o[5];
            ps += o[6];
        }
        sign[j] = bval < 0.0 ? -1.0 : 1.0;
        coef[4 * j + 0] = px;
        coef[4 * j + 1] = py;
        coef[4 * j + 2] = pz;
        coef[4 * j + 3] = ps;
    }
}

__global__ void __launch_bounds__(PNT) partial_kernel(ProjParams p) {
    const int b = blockIdx.y, chunk = blockIdx.x;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int r0 = chunk * p.rows_per_chunk, r1 = min(p.n, r0 + p.rows_per_chunk);
    const double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* X = p.X + (int64_t)b * p.strideX;
    double* part = p.partial + ((int64_t)b * p.nchunks + chunk) * (int64_t)p.c_cap * 8;
    // the chunk's coordinates (and s = (x + y) + z) once in shared memory: one
    // broadcast 32-byte read per row instead of three global loads per element
    __shared__ double4 sx[64];
    for (int i = threadIdx.x; i < r1 - r0; i += PNT) {
        const double x = X[3 * (r0 + i)], y = X[3 * (r0 + i) + 1], z = X[3 * (r0 + i) + 2];
        sx[i] = make_double4(x, y, z, (x + y) + z);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < c; j += PNT) {
        double best = -1.0, bval = 0.0;
        int bidx = 0;
        double px = 0.0, py = 0.0, pz = 0.0, ps = 0.0;
#pragma unroll 8
        for (int i = r0; i < r1; ++i) {
            const double q = Q[(int64_t)i * p.ldq + j];
            const double mag = fabs(q);
            if (mag > best) {
                best = mag;
                bval = q;
                bidx = i;
            }
            const double4 v = sx[i - r0];
            px = fma(q, v.x, px);
            py = fma(q, v.y, py);
            pz = fma(q, v.z, pz);
            ps = fma(q, v.w, ps);
        }
        double* o = part + (int64_t)j * 8;
        o[0] = best;
        o[1] = bval;
        o[2] = (double)bidx;
        o[3] = px;
        o[4] = py;
        o[5] = pz;
        o[6] = ps;
    }
    // the last chunk CTA of a chain reduces the chunks in order (deterministic)
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&p.counter[2 * b], 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    reduce_block(p, b);
    if (threadIdx.x == 0) p.counter[2 * b] = 0;
}

SMG_DEV void stats_block(const ProjParams& p, int b, int nblocks) {
    double a = 0.0, e = 0.0;
    const double* o = p.partial2 + (int64_t)b * nblocks * 2;
    for (int k = 0; k < nblocks; ++k) {
        a += o[2 * k];
        e += o[2 * k + 1];
    }
    double* s = p.stats + (int64_t)b * p.strideStats;
    s[0] = sqrt(a / (3.0 * p.n));  // projection_residual_rms
    s[1] = sqrt(e);                // ||e||
    s[2] = a;
}

// warp per row: x^_i = sum_j q_ij P_j ; e_i = s_i - sum_j q_ij Ps_j
__global__ void __launch_bounds__(PNT) recon_kernel(ProjParams p) {
    __shared__ double red[2][PNT / 32];
    extern __shared__ __align__(16) double scoef[];  // c x 4, staged once per CTA
    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* X = p.X + (int64_t)b * p.strideX;
    for (int e = threadIdx.x; e < 4 * c; e += PNT) scoef[e] = p.coeff[(int64_t)b * p.strideCoef + e];
    __syncthreads();
    const double* coef = scoef;
    double* xhat = p.xhat ? p.xhat + (int64_t)b * p.strideXhat : nullptr;
    double* e_out = p.e_out ? p.e_out + (int64_t)b * p.strideE : nullptr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rows_per_block = PNT / 32 * p.rows_per_warp;
    double res2 = 0.0, e2 = 0.0;
    for (int rr = 0; rr < p.rows_per_warp; ++rr) {
        const int i = blockIdx.x * rows_per_block + warp * p.rows_per_warp + rr;
        if (i >= p.n) break;
        double ax = 0.0, ay = 0.0, az = 0.0, as = 0.0;
#pragma unroll 4
        for (int j = lane; j < c; j += 32) {
            const double q = Q[(int64_t)i * p.ldq + j];
            ax = fma(q, coef[4 * j + 0], ax);
            ay = fma(q, coef[4 * j + 1], ay);
            az = fma(q, coef[4 * j + 2], az);
            as = fma(q, coef[4 * j + 3], as);
        }
        ax = warp_sum(ax);
        ay = warp_sum(ay);
        az = warp_sum(az);
        as = warp_sum(as);
        if (lane == 0) {
            const double x = X[3 * i], y = X[3 * i + 1], z = X[3 * i + 2];
            if (xhat) {
                xhat[3 * i] = ax;
                xhat[3 * i + 1] = ay;
                xhat[3 * i + 2] = az;
            }
            const double dx = x - ax, dy = y - ay, dz = z - az;
            res2 += dx * dx + dy * dy + dz * dz;
            const double e = ((x + y) + z) - as;
            if (e_out) e_out[i] = e;
            e2 += e * e;
        }
    }
    if (lane == 0) {
        red[0][warp] = res2;
        red[1][warp] = e2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, e = 0.0;
        for (int w = 0; w < PNT / 32; ++w) {
            a += red[0][w];
            e += red[1][w];
        }
        double* o = p.partial2 + ((int64_t)b * gridDim.x + blockIdx.x) * 2;
        o[0] = a;
        o[1] = e;
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&p.counter[2 * b + 1], 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    stats_block(p, b, gridDim.x);
    p.counter[2 * b + 1] = 0;
}

}  // namespace

int proj_chunks(int n) { return (n + 63) / 64; }
int proj_recon_blocks(int n, int rows_per_warp) { return (n + (PNT / 32) * rows_per_warp - 1) / ((PNT / 32) * rows_per_warp); }

void project(const ProjParams& p0, cudaStream_t st) {
    ProjParams p = p0;
    p.rows_per_chunk = 64;
    p.nchunks = proj_chunks(p.n);
    if (p.rows_per_warp <= 0) p.rows_per_warp = 2;
    ::smg::count_launch(), partial_kernel<<<dim3(p.nchunks, p.batch), PNT, 0, st>>>(p);
    const int nb = proj_recon_blocks(p.n, p.rows_per_warp);
    ::smg::count_launch(), recon_kernel<<<dim3(nb, p.batch), PNT, 4 * p.c_cap * sizeof(double), st>>>(p);
}

}  // namespace smg

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
// Pass 1 (per row chunk, threads over column pairs, coalesced rows of Q)
// produces partial column maxima and partial Q^T [X | s]; pass 2 reduces them
// in a fixed order (32 columns x 8 contiguous chunk ranges per CTA); pass 3
// (thread = column part x 4 rows) rebuilds X^ and e and the chain's last CTA
// sums the residual partials in block order.  Deterministic.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int PNT = 256;   // recon CTA: 8 column parts x 32 row groups of RPT rows
constexpr int QNT = 128;   // partial CTA: two adjacent columns per thread
constexpr int RPC = 32;    // rows per partial chunk
#ifndef SMG_RECON_UNROLL
#define SMG_RECON_UNROLL 1
#endif
constexpr int kReconUnroll = SMG_RECON_UNROLL;  // column-pair steps unrolled in recon
// rows per recon thread: 4 (coefficients reused across them) when the batch
// fills the GPU, 1 for a single chain (4x the CTAs)

// partial record per (chunk, column): best |q|, its q, Px, Py, Pz, Ps (8 doubles, 64 B)
// one double2 (two adjacent columns) per thread and row: a warp reads 512
// contiguous bytes of a row; 32-row chunks give every chain (n / 32) CTAs
__global__ void __launch_bounds__(QNT) partial_kernel(ProjParams p) {
    const int b = blockIdx.y, chunk = blockIdx.x;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int r0 = chunk * RPC, r1 = min(p.n, r0 + RPC);
    const double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* X = p.X + (int64_t)b * p.strideX;
    double* part = p.partial + ((int64_t)b * p.nchunks + chunk) * (int64_t)p.c_cap * 8;
    // the chunk's coordinates (and s = (x + y) + z) once in shared memory
    __shared__ double4 sx[RPC];
    for (int i = threadIdx.x; i < r1 - r0; i += QNT) {
        const double x = X[3 * (r0 + i)], y = X[3 * (r0 + i) + 1], z = X[3 * (r0 + i) + 2];
        sx[i] = make_double4(x, y, z, (x + y) + z);
    }
    __syncthreads();
    for (int j0 = 2 * threadIdx.x; j0 < c; j0 += 2 * QNT) {
        double best0 = -1.0, bval0 = 0.0, best1 = -1.0, bval1 = 0.0;
        double px0 = 0.0, py0 = 0.0, pz0 = 0.0, ps0 = 0.0, px1 = 0.0, py1 = 0.0, pz1 = 0.0, ps1 = 0.0;
        const double* q0 = Q + (int64_t)r0 * p.ldq + j0;
#pragma unroll 8
        for (int i = 0; i < r1 - r0; ++i) {
            const double2 q = __ldg(reinterpret_cast<const double2*>(q0 + (int64_t)i * p.ldq));
            const double m0 = fabs(q.x), m1 = fabs(q.y);
            const bool u0 = m0 > best0, u1 = m1 > best1;  // rows in order: first index wins
            best0 = u0 ? m0 : best0;
            bval0 = u0 ? q.x : bval0;
            best1 = u1 ? m1 : best1;
            bval1 = u1 ? q.y : bval1;
            const double4 v = sx[i];
            px0 = fma(q.x, v.x, px0);
            py0 = fma(q.x, v.y, py0);
            pz0 = fma(q.x, v.z, pz0);
            ps0 = fma(q.x, v.w, ps0);
            px1 = fma(q.y, v.x, px1);
            py1 = fma(q.y, v.y, py1);
            pz1 = fma(q.y, v.z, pz1);
            ps1 = fma(q.y, v.w, ps1);
        }
        double4* o = reinterpret_cast<double4*>(part + (int64_t)j0 * 8);
        o[0] = make_double4(best0, bval0, px0, py0);
        o[1] = make_double4(pz0, ps0, 0.0, 0.0);
        if (j0 + 1 < c) {
            o[2] = make_double4(best1, bval1, px1, py1);
            o[3] = make_double4(pz1, ps1, 0.0, 0.0);
        }
    }
}

// chunk records -> coefficients and signs: CTA = 32 columns x 8 parts; part q
// combines a contiguous range of chunks in order, then part 0 combines the 8
// part results in order (the first index still wins the argmax; fixed order,
// deterministic).  Replaces one last-arriving CTA reducing every column of a
// chain, which serialised ~nchunks * c records through a single SM.
constexpr int RCOL = 32, RPART = 8;
__global__ void __launch_bounds__(RCOL * RPART) chunk_reduce_kernel(ProjParams p) {
    __shared__ double4 ph[RPART][RCOL], pd[RPART][RCOL];
    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int jj = threadIdx.x % RCOL, part = threadIdx.x / RCOL;
    const int j = blockIdx.x * RCOL + jj;
    const int n0 = (int)((int64_t)p.nchunks * part / RPART), n1 = (int)((int64_t)p.nchunks * (part + 1) / RPART);
    double best = -1.0, bval = 0.0, px = 0.0, py = 0.0, pz = 0.0, ps = 0.0;
    if (j < c) {
        const double* part_b = p.partial + (int64_t)b * p.nchunks * (int64_t)p.c_cap * 8;
        for (int ch0 = n0; ch0 < n1; ch0 += 4) {
            double4 h[4], d[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (ch0 + u < n1) {
                    const double4* o = reinterpret_cast<const double4*>(part_b + ((int64_t)(ch0 + u) * p.c_cap + j) * 8);
                    h[u] = o[0];
                    d[u] = o[1];
                }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (ch0 + u >= n1) break;
                if (h[u].x > best) {
                    best = h[u].x;
                    bval = h[u].y;
                }
                px += h[u].z;
                py += h[u].w;
                pz += d[u].x;
                ps += d[u].y;
            }
        }
    }
    ph[part][jj] = make_double4(best, bval, px, py);
    pd[part][jj] = make_double4(pz, ps, 0.0, 0.0);
    __syncthreads();
    if (part != 0 || j >= c) return;
    best = -1.0;
    bval = px = py = pz = ps = 0.0;
    for (int q = 0; q < RPART; ++q) {
        const double4 h = ph[q][jj], d = pd[q][jj];
        if (h.x > best) {
            best = h.x;
            bval = h.y;
        }
        px += h.z;
        py += h.w;
        pz += d.x;
        ps += d.y;
    }
    double* coef = p.coeff + (int64_t)b * p.strideCoef;
    p.sign[(int64_t)b * p.strideSign + j] = bval < 0.0 ? -1.0 : 1.0;
    coef[4 * j + 0] = px;
    coef[4 * j + 1] = py;
    coef[4 * j + 2] = pz;
    coef[4 * j + 3] = ps;
}

SMG_DEV void stats_block(const ProjParams& p, int b, int nblocks) {
    double a = 0.0, e = 0.0;
    const double2* o = reinterpret_cast<const double2*>(p.partial2 + (int64_t)b * nblocks * 2);
    int k = 0;
    for (; k + 16 <= nblocks; k += 16) {  // block order; 16 loads issued ahead of their adds
        double2 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcg(o + k + u);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a += v[u].x;
            e += v[u].y;
        }
    }
    for (; k < nblocks; ++k) {
        const double2 v = __ldcg(o + k);
        a += v.x;
        e += v.y;
    }
    double* s = p.stats + (int64_t)b * p.strideStats;
    s[0] = sqrt(a / (3.0 * p.n));  // projection_residual_rms
    s[1] = sqrt(e);                // ||e||
    s[2] = a;
}

// x^_i = sum_j q_ij P_j ; e_i = s_i - sum_j q_ij Ps_j.  Thread = (column part,
// group of RPT rows): per column pair it loads the coefficients once from smem
// and RPT double2 of Q (8 lanes of a part group cover 128 contiguous bytes of a
// row); the 8 parts of a row group are 8 consecutive lanes, summed by shuffles.
template <int RPT>
__global__ void __launch_bounds__(PNT) recon_kernel(ProjParams p) {
    constexpr int RROWS = (PNT / 8) * RPT;
    __shared__ double red[2][PNT / 32];
    // coefficients staged once per CTA, swizzled so that the 8 column parts'
    // reads of one 16-byte quarter are 128 contiguous bytes (one wavefront):
    // double2 index ((g * 4 + quarter) * 8 + part) for column pair g * 8 + part,
    // quarters {P_j.xy, P_j.zw, P_j+1.xy, P_j+1.zw}
    extern __shared__ __align__(16) double scoef[];
    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* X = p.X + (int64_t)b * p.strideX;
    {
        const double2* src = reinterpret_cast<const double2*>(p.coeff + (int64_t)b * p.strideCoef);
        double2* dst = reinterpret_cast<double2*>(scoef);
        const int npairs = (c + 1) / 2;
        for (int e = threadIdx.x; e < 4 * npairs; e += PNT) {
            const int pi = e >> 2, quarter = e & 3;
            const int j = 2 * pi + (quarter >> 1);
            const double2 v = j < c ? src[2 * j + (quarter & 1)] : make_double2(0.0, 0.0);  // odd c: the pair's tail
            dst[((pi >> 3) * 4 + quarter) * 8 + (pi & 7)] = v;
        }
    }
    __syncthreads();
    double* xhat = p.xhat ? p.xhat + (int64_t)b * p.strideXhat : nullptr;
    double* e_out = p.e_out ? p.e_out + (int64_t)b * p.strideE : nullptr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int part = threadIdx.x & 7, rg = threadIdx.x >> 3;
    const int i0 = blockIdx.x * RROWS + rg * RPT;
    double acc[RPT][4];
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
    const double2* cf = reinterpret_cast<const double2*>(scoef) + part;
#pragma unroll kReconUnroll
    for (int j = 2 * part; j < c; j += 16, cf += 32) {
        const double2 c0 = cf[0], c1 = cf[8], c2 = cf[16], c3 = cf[24];
        const double4 ca = make_double4(c0.x, c0.y, c1.x, c1.y), cb = make_double4(c2.x, c2.y, c3.x, c3.y);
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            if (i0 + r >= p.n) break;
            double2 q = __ldg(reinterpret_cast<const double2*>(Q + (int64_t)(i0 + r) * p.ldq + j));
            if (j + 1 >= c) q.y = 0.0;  // odd c: the padding column is not part of the basis
            acc[r][0] = fma(q.x, ca.x, acc[r][0]);
            acc[r][1] = fma(q.x, ca.y, acc[r][1]);
            acc[r][2] = fma(q.x, ca.z, acc[r][2]);
            acc[r][3] = fma(q.x, ca.w, acc[r][3]);
            acc[r][0] = fma(q.y, cb.x, acc[r][0]);
            acc[r][1] = fma(q.y, cb.y, acc[r][1]);
            acc[r][2] = fma(q.y, cb.z, acc[r][2]);
            acc[r][3] = fma(q.y, cb.w, acc[r][3]);
        }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double v = acc[r][a];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            acc[r][a] = v;
        }
    double res2 = 0.0, e2 = 0.0;
    if (part == 0) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = i0 + r;
            if (i >= p.n) break;
            const double x = X[3 * i], y = X[3 * i + 1], z = X[3 * i + 2];
            if (xhat) {
                xhat[3 * i] = acc[r][0];
                xhat[3 * i + 1] = acc[r][1];
                xhat[3 * i + 2] = acc[r][2];
            }
            const double dx = x - acc[r][0], dy = y - acc[r][1], dz = z - acc[r][2];
            res2 += dx * dx + dy * dy + dz * dz;
            const double e = ((x + y) + z) - acc[r][3];
            if (e_out) e_out[i] = e;
            e2 += e * e;
        }
    }
    // fixed-order block sum (lanes 0, 8, 16, 24 hold the row groups' sums)
    res2 += __shfl_xor_sync(0xffffffffu, res2, 8);
    e2 += __shfl_xor_sync(0xffffffffu, e2, 8);
    res2 += __shfl_xor_sync(0xffffffffu, res2, 16);
    e2 += __shfl_xor_sync(0xffffffffu, e2, 16);
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

// Reconstruction, warp per RW rows: lane l reads the double2 of columns
// 64k + 2l of each row (a warp instruction = 512 contiguous bytes of one row),
// RW rows x 2 column chunks = 2 RW independent 16-byte loads in flight per lane
// (the older thread-per-column-part kernel had 4 and sat at ~28 % of HBM);
// the RW x 4 lane partials are summed by a halving butterfly (each step sends
// half of the values to the partner lane): V values over 32 lanes in V - 1 + ...
// shuffles, a fixed tree (deterministic); afterwards lane l holds value k(l).

// halving step: keep the half selected by `up`, add the partner's copy of it
template <int V>
SMG_DEV void halve(double (&v)[32], int s, bool up) {
#pragma unroll
    for (int j = 0; j < V / 2; ++j) {
        const double send = up ? v[j] : v[j + V / 2];
        const double keep = up ? v[j + V / 2] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
}

template <int RW, int NCH>
__global__ void __launch_bounds__(PNT) recon_warp_kernel(ProjParams p) {
    static_assert(RW * 4 <= 32, "one lane per (row, output)");
    __shared__ double red[2][PNT / 32];
    extern __shared__ __align__(16) double scoef[];  // c_cap x 4: Px Py Pz Ps
    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* X = p.X + (int64_t)b * p.strideX;
    {
        const double2* src = reinterpret_cast<const double2*>(p.coeff + (int64_t)b * p.strideCoef);
        double2* dst = reinterpret_cast<double2*>(scoef);
        const int cpad = (p.c_cap + 64 * NCH - 1) / (64 * NCH) * (64 * NCH);
        for (int e = threadIdx.x; e < 2 * cpad; e += PNT) dst[e] = (e >> 1) < c ? src[e] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double4* cf = reinterpret_cast<const double4*>(scoef);
    // this CTA's rows: a contiguous range of the chain, in row groups of RW per warp
    const int per = ((p.n + gridDim.x - 1) / gridDim.x + RW * (PNT / 32) - 1) / (RW * (PNT / 32)) * (RW * (PNT / 32));
    const int rbeg = blockIdx.x * per, rend = min(p.n, rbeg + per);
    double res2 = 0.0, e2 = 0.0;
    for (int row0 = rbeg + warp * RW; row0 < rend; row0 += RW * (PNT / 32)) {
        double acc[RW][4];
#pragma unroll
        for (int r = 0; r < RW; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
        for (int base = 0; base < c; base += 64 * NCH) {
            double2 q[NCH][RW];
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
                const int col = base + 64 * h + 2 * lane;
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    const int row = row0 + r;
                    q[h][r] = (col < c && row < rend)
                                  ? __ldg(reinterpret_cast<const double2*>(Q + (int64_t)row * p.ldq + col))
                                  : make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
                const int col = base + 64 * h + 2 * lane;
                const double4 c0 = cf[col], c1 = cf[col + 1];  // zero beyond c (odd c: the padding column too)
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    acc[r][0] = fma(q[h][r].x, c0.x, acc[r][0]);
                    acc[r][1] = fma(q[h][r].x, c0.y, acc[r][1]);
                    acc[r][2] = fma(q[h][r].x, c0.z, acc[r][2]);
                    acc[r][3] = fma(q[h][r].x, c0.w, acc[r][3]);
                    acc[r][0] = fma(q[h][r].y, c1.x, acc[r][0]);
                    acc[r][1] = fma(q[h][r].y, c1.y, acc[r][1]);
                    acc[r][2] = fma(q[h][r].y, c1.z, acc[r][2]);
                    acc[r][3] = fma(q[h][r].y, c1.w, acc[r][3]);
                }
            }
        }
        constexpr int V = RW * 4;
        double v[32];
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int a = 0; a < 4; ++a) v[r * 4 + a] = acc[r][a];
        // halving steps over lane bits 4, 3, ..: afterwards lane l holds value
        // k = bits (4, 3, ..) of l; the remaining lane bits are plain butterflies
        int k = 0;
        {
            int vv = V;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
                if (vv > 1) {
                    const bool up = (lane & s) != 0;
                    if (vv == 32) halve<32>(v, s, up);
                    else if (vv == 16) halve<16>(v, s, up);
                    else if (vv == 8) halve<8>(v, s, up);
                    else if (vv == 4) halve<4>(v, s, up);
                    else halve<2>(v, s, up);
                    vv >>= 1;
                    k = 2 * k + (up ? 1 : 0);
                } else {
                    v[0] += __shfl_xor_sync(0xffffffffu, v[0], s);
                }
            }
        }
        const bool owner = (V == 32) || ((lane & (32 / V - 1)) == 0);  // one lane per value
        if (owner) {
            const double val = v[0];
            const int r = k >> 2, a = k & 3, i = row0 + r;
            if (i < rend) {
                const double* xi = X + 3 * (int64_t)i;
                if (a < 3) {
                    if (p.xhat) p.xhat[(int64_t)b * p.strideXhat + 3 * i + a] = val;
                    const double d = xi[a] - val;
                    res2 += d * d;
                } else {
                    const double e = ((xi[0] + xi[1]) + xi[2]) - val;
                    if (p.e_out) p.e_out[(int64_t)b * p.strideE + i] = e;
                    e2 += e * e;
                }
            }
        }
    }
    res2 = warp_sum(res2);
    e2 = warp_sum(e2);
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

// Reconstruction on the DMMA pipe: [X^ | Ps] (n x 4) = Q (n x c) * C (c x 4),
// one m16n8k8 per 16 rows x 8 columns of Q (B = the coefficients, outputs 4-7
// zero).  The A fragments are read straight from global memory -- lane (g, t)
// loads Q[g][k+t], Q[g+8][k+t], Q[g][k+t+4], Q[g+8][k+t+4], so every warp load
// touches 16 rows x 32 contiguous bytes (whole sectors) -- KU k-steps of loads
// are issued before their products (4 * KU * RT 8-byte loads in flight per
// lane), and the coefficients come from shared memory (16 consecutive doubles
// per fragment, conflict-free).  No shuffles: the accumulator of lane (g, t < 2)
// is exactly (x^, y^) or (z^, s^) of rows g and g + 8.
constexpr int MNT = 256;  // 8 warps
template <int RT>
__global__ void __launch_bounds__(MNT, RT == 1 ? 4 : 3) recon_mma_kernel(ProjParams p) {
    constexpr int KU = RT == 1 ? 4 : 2;  // 16 loads in flight per lane either way
    __shared__ double red[2][MNT / 32];
    // B fragments pre-paired: scoef[(kb * 4 + t) * 8 + g] = (C[8kb+t][g], C[8kb+t+4][g])
    // (outputs g = Px Py Pz Ps, zero for g >= 4 and past c): one 16-byte load per
    // lane and k-step, a warp reads 512 contiguous bytes
    extern __shared__ __align__(16) double2 scoef2[];
    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int kpad = (c + 8 * KU - 1) / (8 * KU) * (8 * KU);
    {
        const double* src = p.coeff + (int64_t)b * p.strideCoef;
        for (int e = threadIdx.x; e < 4 * kpad; e += MNT) {
            const int gg = e & 7, tt = (e >> 3) & 3, kb = e >> 5;
            const int k0 = 8 * kb + tt, k1 = k0 + 4;
            scoef2[e] = make_double2(gg < 4 && k0 < c ? src[4 * k0 + gg] : 0.0, gg < 4 && k1 < c ? src[4 * k1 + gg] : 0.0);
        }
    }
    __syncthreads();
    const double* Q = p.Q + (int64_t)b * p.strideQ;
    const double* X = p.X + (int64_t)b * p.strideX;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int row0 = (blockIdx.x * (MNT / 32) + warp) * 16 * RT;
    double acc[RT][4];
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
    // row pointers of the lane's rows (clamped; masked values are zero)
    const double* qr[RT][2];
    bool rv[RT][2];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = row0 + 16 * r + 8 * h + g;
            rv[r][h] = i < p.n;
            qr[r][h] = Q + (int64_t)(rv[r][h] ? i : 0) * p.ldq + t;
        }
    for (int k0 = 0; k0 < c; k0 += 8 * KU) {
        double a[KU][RT][4];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const int k = k0 + 8 * u;
            const bool c0 = k + t < c, c1 = k + t + 4 < c;
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                a[u][r][0] = (rv[r][0] && c0) ? __ldg(qr[r][0] + k) : 0.0;
                a[u][r][1] = (rv[r][1] && c0) ? __ldg(qr[r][1] + k) : 0.0;
                a[u][r][2] = (rv[r][0] && c1) ? __ldg(qr[r][0] + k + 4) : 0.0;
                a[u][r][3] = (rv[r][1] && c1) ? __ldg(qr[r][1] + k + 4) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const int k = k0 + 8 * u;
            const double2 bb = scoef2[((k >> 3) * 4 + t) * 8 + g];
#pragma unroll
            for (int r = 0; r < RT; ++r)
                dmma1688(acc[r][0], acc[r][1], acc[r][2], acc[r][3], a[u][r][0], a[u][r][1], a[u][r][2], a[u][r][3],
                         bb.x, bb.y);
        }
    }
    // lane (g, 0): (x^, y^), lane (g, 1): (z^, s^) of rows g (acc 0, 1) and g + 8 (acc 2, 3)
    double res2 = 0.0, e2 = 0.0;
    if (t < 2) {
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = row0 + 16 * r + 8 * h + g;
                if (i >= p.n) continue;
                const double v0 = acc[r][2 * h], v1 = acc[r][2 * h + 1];
                const double* xi = X + 3 * (int64_t)i;
                double* xh = p.xhat ? p.xhat + (int64_t)b * p.strideXhat + 3 * (int64_t)i : nullptr;
                if (t == 0) {
                    const double dx = xi[0] - v0, dy = xi[1] - v1;
                    res2 += dx * dx + dy * dy;
                    if (xh) {
                        xh[0] = v0;
                        xh[1] = v1;
                    }
                } else {
                    const double x = xi[0], y = xi[1], z = xi[2];
                    const double dz = z - v0;
                    res2 += dz * dz;
                    const double e = ((x + y) + z) - v1;
                    e2 += e * e;
                    if (xh) xh[2] = v0;
                    if (p.e_out) p.e_out[(int64_t)b * p.strideE + i] = e;
                }
            }
    }
    res2 = warp_sum(res2);
    e2 = warp_sum(e2);
    if (lane == 0) {
        red[0][warp] = res2;
        red[1][warp] = e2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, se = 0.0;
        for (int w = 0; w < MNT / 32; ++w) {
            sa += red[0][w];
            se += red[1][w];
        }
        double* o = p.partial2 + ((int64_t)b * gridDim.x + blockIdx.x) * 2;
        o[0] = sa;
        o[1] = se;
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

int proj_chunks(int n) { return (n + RPC - 1) / RPC; }
int proj_recon_blocks(int n, int /*rows_per_warp*/) { return (n + 15) / 16; }  // upper bound (8 warps x 2 rows)

void project(const ProjParams& p0, cudaStream_t st) {
    ProjParams p = p0;
    p.rows_per_chunk = RPC;
    p.nchunks = proj_chunks(p.n);
    if (!p.partials_ready) ::smg::count_launch(), partial_kernel<<<dim3(p.nchunks, p.batch), QNT, 0, st>>>(p);
    ::smg::count_launch(), chunk_reduce_kernel<<<dim3((p.c_cap + RCOL - 1) / RCOL, p.batch), RCOL * RPART, 0, st>>>(p);
    if (!std::getenv("SMG_RECON_OLD") && !std::getenv("SMG_RECON_WARP")) {
        // DMMA reconstruction: 32 rows per warp when the batch fills the GPU, 16 otherwise
        const int kpad = (p.c_cap + 31) / 32 * 32;
        const int msmem = kpad * 4 * (int)sizeof(double2);
        ensure_smem((const void*)recon_mma_kernel<2>, msmem);
        ensure_smem((const void*)recon_mma_kernel<1>, msmem);
        if ((int64_t)p.batch * ((p.n + 255) / 256) >= 2 * 148) {
            const int nb = (p.n + 255) / 256;
            ::smg::count_launch(), recon_mma_kernel<2><<<dim3(nb, p.batch), MNT, msmem, st>>>(p);
        } else {
            const int nb = (p.n + 127) / 128;
            ::smg::count_launch(), recon_mma_kernel<1><<<dim3(nb, p.batch), MNT, msmem, st>>>(p);
        }
        return;
    }
    if (!std::getenv("SMG_RECON_OLD")) {
        // one row group per warp (measured: 46 us per C5 launch against 63 us for
        // the thread-per-column-part kernel; a persistent sweep over row ranges
        // was slower, 58 us); RW rows x 2 column chunks in flight per lane
        const int wsmem = (p.c_cap + 127) / 128 * 128 * 4 * (int)sizeof(double);
        const int maxb = proj_recon_blocks(p.n, 0);
        if (p.batch >= 8) {
            const int cpc = std::min(maxb, (p.n + 4 * (PNT / 32) - 1) / (4 * (PNT / 32)));
            ::smg::count_launch(), recon_warp_kernel<4, 2><<<dim3(cpc, p.batch), PNT, wsmem, st>>>(p);
        } else {
            const int cpc = std::min(maxb, (p.n + 2 * (PNT / 32) - 1) / (2 * (PNT / 32)));
            ::smg::count_launch(), recon_warp_kernel<2, 2><<<dim3(cpc, p.batch), PNT, wsmem, st>>>(p);
        }
        return;
    }
    const int smem = ((p.c_cap + 1) / 2 + 7) / 8 * 32 * (int)sizeof(double2);
    const int nb4 = (p.n + 4 * (PNT / 8) - 1) / (4 * (PNT / 8));
    if ((int64_t)nb4 * p.batch >= 2 * 148) {
        ::smg::count_launch(), recon_kernel<4><<<dim3(nb4, p.batch), PNT, smem, st>>>(p);
    } else {
        const int nb1 = (p.n + PNT / 8 - 1) / (PNT / 8);
        ::smg::count_launch(), recon_kernel<1><<<dim3(nb1, p.batch), PNT, smem, st>>>(p);
    }
}

}  // namespace smg

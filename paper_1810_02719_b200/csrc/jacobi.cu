// K9 helper: eigendecomposition of the small Rayleigh-Ritz matrix H = Q^T L Q
// (m x m, symmetric positive semidefinite) for the first-submesh basis.
//
// The reference takes the bottom-c eigenvectors of the dense n_d x n_d L from
// Eigen's SelfAdjointEigenSolver (spectral.hpp:92-117).  On the GPU the first
// basis comes from shift-invert subspace iteration on the tile's own factor
// followed by Rayleigh-Ritz (firstbasis.cpp); only this m x m eigenproblem
// (m ~ 1.5 c) needs a dense solver.  It is solved by one-sided (Hestenes)
// block Jacobi: columns a_j of A = H are pairwise orthogonalised, the
// rotations accumulate in V, and at convergence A = H V has orthogonal columns,
// so V holds the eigenvectors and theta_j = v_j^T a_j the eigenvalues.
// One-sided Jacobi only ever touches *columns*, so disjoint column pairs are
// independent: one thread-block cluster per matrix, every CTA owns two blocks of
// b columns (A and V) in shared memory, warps rotate disjoint pairs, and the
// blocks move between CTAs by the round-robin tournament through L2 with one
// cluster barrier per round.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace smg {

namespace {

constexpr int JNT = 512;
constexpr int JWARPS = JNT / 32;

struct JacobiShape {
    int m, mp, b, P;
};

SMG_DEV void rotate_pair(double* __restrict__ ax, double* __restrict__ ay, double* __restrict__ vx,
                         double* __restrict__ vy, int mp, int lane, double tiny2, double& offmax) {
    double alpha = 0.0, beta = 0.0, gamma = 0.0;
    for (int r = lane; r < mp; r += 32) {
        const double x = ax[r], y = ay[r];
        alpha = fma(x, x, alpha);
        beta = fma(y, y, beta);
        gamma = fma(x, y, gamma);
    }
    alpha = warp_sum(alpha);
    beta = warp_sum(beta);
    gamma = warp_sum(gamma);
    if (alpha <= tiny2 || beta <= tiny2) return;
    const double rel = fabs(gamma) / sqrt(alpha * beta);
    if (!(rel > 1e-15)) return;
    offmax = fmax(offmax, rel);
    const double zeta = (beta - alpha) / (2.0 * gamma);
    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    const double c = 1.0 / sqrt(1.0 + t * t);
    const double s = c * t;
    for (int r = lane; r < mp; r += 32) {
        const double x = ax[r], y = ay[r];
        ax[r] = c * x - s * y;
        ay[r] = s * x + c * y;
        const double u = vx[r], w = vy[r];
        vx[r] = c * u - s * w;
        vy[r] = s * u + c * w;
    }
}

// slot holding block `blk` after `r` rotations of slots 1..P-1 (slot 0 fixed)
SMG_DEV int block_at_slot(int slot, int r, int P) {
    if (slot == 0) return 0;
    // block at slot s after r rounds came from slot s - r (mod P-1, within 1..P-1)
    int s = (slot - 1 - r) % (P - 1);
    if (s < 0) s += P - 1;
    return s + 1;
}

__global__ void __launch_bounds__(JNT) jacobi_kernel(JacobiParams p, JacobiShape sh) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    __shared__ double wmax[JWARPS];
    __shared__ double cluster_off;
    const int NC = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int batch = blockIdx.x / NC;
    const int m = sh.m, mp = sh.mp, b = sh.b, P = sh.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // shared layout: [2 blocks][A | V][b columns][mp]
    double* blkA[2] = {sm, sm + 2 * b * mp};
    double* blkV[2] = {sm + b * mp, sm + 3 * b * mp};
    const double* H = p.H + (int64_t)batch * p.strideH;
    double* stage = p.stage + (int64_t)batch * p.strideStage;  // [2 parity][P][2][b][mp]
    const int64_t slot_elems = (int64_t)2 * b * mp;

    // initial load: slot s holds block s; CTA rank holds slots rank and P-1-rank
    int slots[2] = {rank, P - 1 - rank};
    for (int h = 0; h < 2; ++h) {
        const int blk = slots[h];
        for (int e = threadIdx.x; e < b * mp; e += JNT) {
            const int jj = e / mp, r = e % mp;
            const int col = blk * b + jj;
            double a = 0.0;
            if (col < m && r < m) a = H[(int64_t)r * p.ldh + col];  // H symmetric: column = row
            blkA[h][e] = a;
            blkV[h][e] = (r == col) ? 1.0 : 0.0;
        }
    }
    // max |H_rr| by a block reduction (max is order independent: same value as
    // the serial loop every thread used to run)
    double nm = 0.0;
    for (int r = threadIdx.x; r < m; r += JNT) nm = fmax(nm, fabs(H[(int64_t)r * p.ldh + r]));
    nm = warp_max(nm);
    if (lane == 0) wmax[warp] = nm;
    __syncthreads();
    double normmax = 0.0;
    for (int w = 0; w < JWARPS; ++w) normmax = fmax(normmax, wmax[w]);
    const double tiny2 = (1e-15 * normmax) * (1e-15 * normmax) + 1e-300;
    __syncthreads();

    int round_global = 0;
    int sweep = 0;
    for (; sweep < p.max_sweeps; ++sweep) {
        double offmax = 0.0;
        for (int round = 0; round < P - 1; ++round, ++round_global) {
            if (round == 0) {
                // intra-block pairs of both held blocks: circle method on b (+1 dummy if odd)
                const int bb = b + (b & 1);
                for (int sr = 0; sr < bb - 1; ++sr) {
                    // pairs (i, j) of the circle arrangement for this sub-round
                    for (int task = warp; task < bb; task += JWARPS) {
                        const int h = task / (bb / 2);
                        const int k = task % (bb / 2);
                        if (h > 1) continue;
                        auto pos = [&](int q) {
                            if (q == 0) return 0;
                            int v = (q - 1 + sr) % (bb - 1);
                            return v + 1;
                        };
                        const int i = pos(k), j = pos(bb - 1 - k);
                        if (i >= b || j >= b) continue;
                        rotate_pair(blkA[h] + i * mp, blkA[h] + j * mp, blkV[h] + i * mp, blkV[h] + j * mp, mp,
                                    lane, tiny2, offmax);
                    }
                    __syncthreads();
                }
            }
            // inter-block pairs (X_i, Y_{(i+s) mod b})
            for (int s = 0; s < b; ++s) {
                for (int i = warp; i < b; i += JWARPS) {
                    const int j = (i + s) % b;
                    rotate_pair(blkA[0] + i * mp, blkA[1] + j * mp, blkV[0] + i * mp, blkV[1] + j * mp, mp, lane,
                                tiny2, offmax);
                }
                __syncthreads();
            }
            // rotate slots 1..P-1: block at slot q (q>=1) moves to slot q % (P-1) + 1
            double* st_out = stage + (int64_t)(round_global & 1) * P * slot_elems;
            for (int h = 0; h < 2; ++h) {
                const int q = slots[h];
                const int nq = (q == 0) ? 0 : (q % (P - 1)) + 1;
                double* dst = st_out + (int64_t)nq * slot_elems;
                for (int e = threadIdx.x; e < b * mp; e += JNT) {
                    dst[e] = blkA[h][e];
                    dst[b * mp + e] = blkV[h][e];
                }
            }
            __threadfence();
            cluster.sync();
            for (int h = 0; h < 2; ++h) {
                const double* src = st_out + (int64_t)slots[h] * slot_elems;
                for (int e = threadIdx.x; e < b * mp; e += JNT) {
                    blkA[h][e] = src[e];
                    blkV[h][e] = src[b * mp + e];
                }
            }
            __syncthreads();
        }
        // cluster-wide max of the off-diagonal measure
        offmax = warp_max(offmax);
        if (lane == 0) wmax[warp] = offmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = 0.0;
            for (int w = 0; w < JWARPS; ++w) v = fmax(v, wmax[w]);
            wmax[0] = v;
            if (rank == 0) cluster_off = 0.0;
        }
        cluster.sync();
        if (threadIdx.x == 0) {
            double* remote = cluster.map_shared_rank(&cluster_off, 0);
            atomicMax(reinterpret_cast<unsigned long long*>(remote), __double_as_longlong(wmax[0]));
        }
        cluster.sync();
        double off = 0.0;
        if (threadIdx.x == 0) off = *cluster.map_shared_rank(&cluster_off, 0);
        __syncthreads();
        if (threadIdx.x == 0) wmax[0] = off;
        __syncthreads();
        off = wmax[0];
        cluster.sync();
        if (off < p.tol) {
            ++sweep;
            break;
        }
    }
    // write V columns and Rayleigh quotients by original column index
    for (int h = 0; h < 2; ++h) {
        const int blk = block_at_slot(slots[h], round_global, P);
        for (int jj = warp; jj < b; jj += JWARPS) {
            const int col = blk * b + jj;
            if (col >= m) continue;
            const double* a = blkA[h] + jj * mp;
            const double* v = blkV[h] + jj * mp;
            double rq = 0.0, vv = 0.0;
            for (int r = lane; r < mp; r += 32) {
                rq = fma(v[r], a[r], rq);
                vv = fma(v[r], v[r], vv);
            }
            rq = warp_sum(rq);
            vv = warp_sum(vv);
            for (int r = lane; r < m; r += 32) p.V[(int64_t)batch * p.strideV + (int64_t)col * p.ldv + r] = v[r];
            if (lane == 0) p.theta[(int64_t)batch * p.strideTheta + col] = rq / vv;
        }
    }
    if (threadIdx.x == 0 && rank == 0 && p.sweeps) p.sweeps[batch] = sweep;
}

// sort eigenpairs ascending (stable), emit W row-major (m x m): W[:, j] = v_{order[j]}
__global__ void sort_kernel(JacobiParams p, int m) {
    const int batch = blockIdx.x;
    extern __shared__ double th[];
    int* order = reinterpret_cast<int*>(th + m);
    const double* theta = p.theta + (int64_t)batch * p.strideTheta;
    for (int j = threadIdx.x; j < m; j += blockDim.x) th[j] = theta[j];
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        int rank = 0;
        const double t = th[j];
        for (int k = 0; k < m; ++k) rank += (th[k] < t) || (th[k] == t && k < j);
        order[rank] = j;
    }
    __syncthreads();
    const double* V = p.V + (int64_t)batch * p.strideV;  // column j of eigvec stored as row j (col-major)
    double* W = p.W + (int64_t)batch * p.strideW;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int r = e / m, j = e % m;
        W[(int64_t)r * p.ldw + j] = V[(int64_t)order[j] * p.ldv + r];
    }
    double* ts = p.theta_sorted + (int64_t)batch * p.strideTheta;
    for (int j = threadIdx.x; j < m; j += blockDim.x) ts[j] = th[order[j]];
}

}  // namespace

JacobiPlan jacobi_plan(int m) {
    JacobiPlan pl;
    int nc = 2;
    while (nc < 8 && (m + 2 * nc - 1) / (2 * nc) > 12) nc *= 2;
    auto fits = [&](int ncv) {
        const int b = (m + 2 * ncv - 1) / (2 * ncv);
        const int mp = ((2 * ncv * b) + 7) / 8 * 8;
        return (int64_t)4 * b * mp * 8 <= 227 * 1024;
    };
    while (nc < 16 && !fits(nc)) nc *= 2;
    pl.nc = nc;
    pl.b = (m + 2 * nc - 1) / (2 * nc);
    pl.P = 2 * nc;
    pl.mp = ((pl.P * pl.b) + 7) / 8 * 8;
    pl.smem = 4 * pl.b * pl.mp * 8;
    pl.stage_elems = (int64_t)2 * pl.P * 2 * pl.b * pl.mp;
    return pl;
}

int jacobi_eigh(const JacobiParams& p, const JacobiPlan& pl, int m, cudaStream_t st) {
    JacobiShape sh{m, pl.mp, pl.b, pl.P};
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    if (pl.nc > 8) cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.nc * p.batch);
    cfg.blockDim = dim3(JNT);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = pl.nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ::smg::count_launch();
    cudaError_t err = cudaLaunchKernelEx(&cfg, jacobi_kernel, p, sh);
    if (err != cudaSuccess) return (int)err;
    const int sbytes = m * 8 + m * 4;
    ::smg::count_launch(), sort_kernel<<<p.batch, 256, sbytes, st>>>(p, m);
    return (int)cudaGetLastError();
}

}  // namespace smg

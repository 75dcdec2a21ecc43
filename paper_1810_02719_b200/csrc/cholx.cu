// K6x: latency-oriented blocked Cholesky of the column-scaled Gram with the
// whole factor resident in (distributed) shared memory.
//
// Same contract as chol_kernel (cholqr.cu; orthonormalize's rank test,
// spectral.hpp:120-132): A = D^-1 G D^-1 = R~^T R~, the reference rank test on
// the pivots, B = D^-1 R~^-1 for the triangular product Q = V B (or R~ and
// the diagonal-block inverses for the row-parallel solve, skip_inverse).
//
// Where chol_kernel keeps A in global memory and streams one panel row
// through shared memory, here the upper block triangle lives in shared
// memory for the whole factorisation: 32x32 blocks (i <= j), owned
// column-cyclically by the CTAs of a thread-block cluster (block column j on
// rank j % CL), XOR-swizzled so every DMMA fragment load is one wavefront.
// Per 32-column panel p:
//   1. the owner of column p factors the diagonal block on ONE warp: lane k
//      holds column k in registers, the pivot row is broadcast through shared
//      memory (LDL^T, no CTA barrier per column), then inverts it the same
//      way (X_pp = R_pp^-1, lane k = column k) and publishes X_pp;
//   2. cluster barrier; every CTA forms its panel-row blocks R_pq = X_pp^T A_pq
//      (DMMA, in place);
//   3. cluster barrier; every CTA updates its trailing blocks
//      A_qr -= R_pq^T R_pr, reading R_pq from the owner of column q through
//      DSMEM.
// Afterwards (unless skip_inverse) each block column of X = R~^-1 is
// back-substituted by one warp from the shared-memory R (columns are
// independent), X_sq blocks through global B (L2).
#include <cooperative_groups.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace smg {

namespace {

#ifdef SMG_CHOLX_TIMING
__device__ unsigned long long g_cx_t[512];
SMG_DEV unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define CXT(i, cond) \
    do { \
        if ((cond) && blockIdx.x < (unsigned)CL) g_cx_t[(i)] = gtime(); \
    } while (0)
#else
#define CXT(i, cond) \
    do { \
    } while (0)
#endif

constexpr int XNT = 256;  // 8 warps
constexpr int XNW = XNT / 32;
constexpr int kXMaxP = 16;  // c <= 512

// element (r, c) of a 32x32 block: rows of 32 doubles, columns XOR-swizzled so
// 8 rows x 4 columns (A fragments) and 4 rows x 8 columns (B fragments) each
// hit 32 distinct double slots
SMG_DEV int sw(int r, int c) { return r * 32 + (c ^ (((r & 3) << 3) | (((r >> 2) & 1) << 2))); }

template <class FA, class FB>
SMG_DEV void blk_mma(double (&acc)[4][4][2], FA a, FB b, int g, int t) {
#pragma unroll 2
    for (int kk = 0; kk < 32; kk += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = a(8 * i + g, kk + t);
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = b(kk + t, 8 * j + g);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
}

SMG_DEV void zero4(double (&acc)[4][4][2]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// local block index of (i, j), i <= j, on the owner of column j (= j % CL):
// owned columns j = rank, rank + CL, ... are stored one after the other, each
// with its j + 1 blocks
SMG_DEV int lblk(int i, int j, int CL) {
    const int m = j / CL, r = j % CL;  // j = r + m CL; earlier owned columns r + u CL, u < m
    return m * (r + 1) + CL * m * (m - 1) / 2 + i;
}

__host__ __device__ constexpr int owned_blocks(int P, int CL, int rank) {
    int n = 0;
    for (int j = rank; j < P; j += CL) n += j + 1;
    return n;
}

__host__ __device__ constexpr int max_owned_blocks(int P, int CL) {
    int m = 0;
    for (int r = 0; r < CL; ++r) m = owned_blocks(P, CL, r) > m ? owned_blocks(P, CL, r) : m;
    return m;
}

// shared memory: owned blocks | xpub (this CTA's published X_pp) | xloc (copy of
// the current panel's X_pp) | row (pivot-row broadcast, 32) | ds (cp) | rds (cp)
__host__ __device__ constexpr int cholx_bytes(int P, int CL) {
    return (max_owned_blocks(P, CL) * 1024 + 2 * 1024 + 32 + 2 * 32 * P) * 8;
}

template <int CL>
__global__ void __launch_bounds__(XNT, 1) cholx_kernel(CholParams p) {
    extern __shared__ __align__(16) double xsm[];
    __shared__ double red[32];
    __shared__ int fail;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = CL > 1 ? (int)cluster.block_rank() : 0;
    const int b = blockIdx.x / CL;
    if (p.status[b] != kOk) return;  // uniform over the cluster
    if (p.skip && p.skip[b]) return;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c_cap;
    const int P = (c + 31) / 32, cp = P * 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nloc = max_owned_blocks(P, CL);
    double* blk = xsm;                       // nloc x 1024
    double* xpub = blk + (int64_t)nloc * 1024;
    double* xloc = xpub + 1024;
    double* rowb = xloc + 1024;
    double* ds = rowb + 32;
    double* rds = ds + cp;
    const double* G = p.G + (int64_t)b * p.strideG;
    double* Ag = p.A + (int64_t)b * p.strideA;
    double* Bo = p.Binv + (int64_t)b * p.strideB;
    double* dout = p.dscale + (int64_t)b * p.strideD;

    auto sync_cluster = [&]() {
        if (CL > 1) cluster.sync();
        else __syncthreads();
    };
    auto block_of = [&](int i, int j) -> double* {  // local or DSMEM pointer to block (i, j)
        double* loc = blk + (int64_t)lblk(i, j, CL) * 1024;
        if (CL == 1 || j % CL == rank) return loc;
        return cluster.map_shared_rank(loc, j % CL);
    };

    // column norms from the Gram's diagonal (every CTA; identical arithmetic)
    double tr = 0.0;
    for (int j = tid; j < cp; j += XNT) {
        double dj = 1.0;
        if (j < c) {
            const double gjj = G[(int64_t)j * p.ldg + j];
            tr += gjj;
            dj = p.column_scale ? sqrt(gjj) : 1.0;
        }
        ds[j] = dj;
        rds[j] = dj > 0.0 ? 1.0 / dj : 0.0;
        if (rank == 0) dout[j] = dj;
    }
    tr = block_sum(tr, red);
    const double scale = sqrt(tr);
    if (tid == 0) {
        fail = 0;
        if (p.vnorm && rank == 0) p.vnorm[b] = scale;
    }
    auto record = [&](int kind, int64_t col) {
        p.status[b] = kind;
        if (p.status_detail) p.status_detail[b] = col;
        if (p.errpos) p.errpos[b] = p.pos;
    };
    if (!(scale > 0.0) || !isfinite(scale)) {  // uniform: every CTA computed the same scale
        if (tid == 0 && rank == 0) record(scale == 0.0 ? kAllZero : kNotFinite, -1);
        return;
    }
    const double thresh = 1e-13 * scale;
    __syncthreads();
    // owned blocks of A = D^-1 G D^-1 (upper; identity padding)
    for (int j = rank; j < P; j += CL)
        for (int i = 0; i <= j; ++i) {
            double* d = blk + (int64_t)lblk(i, j, CL) * 1024;
            for (int e = tid; e < 1024; e += XNT) {
                const int r = e >> 5, k = e & 31, gi = i * 32 + r, gk = j * 32 + k;
                double v;
                if (gi < c && gk < c) v = (gi <= gk || i < j) ? G[(int64_t)gi * p.ldg + gk] * rds[gi] * rds[gk] : 0.0;
                else v = (gi == gk) ? 1.0 : 0.0;
                d[sw(r, k)] = v;
            }
        }
    __syncthreads();
    CXT(0, tid == 0 && rank == 0);

    for (int pb = 0; pb < P; ++pb) {
        const int owner = pb % CL;
        // ---- 1. diagonal block on one warp of its owner
        CXT(8 + pb * 8 + 0, rank == owner && tid == 0);
        if (rank == owner && warp == 0) {
            double* D = blk + (int64_t)lblk(pb, pb, CL) * 1024;
            double a[32];  // column `lane`: a[i] = D[i][lane], i <= lane
#pragma unroll
            for (int i = 0; i < 32; ++i) a[i] = (i <= lane) ? D[sw(i, lane)] : 0.0;
            double piv = 0.0;
            // right-looking LDL^T: after step j, row j is final
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                rowb[lane] = a[j];  // lanes >= j hold row j
                __syncwarp();
                const double pj = rowb[j];
                if (lane == j) piv = pj;
                const double inv = __drcp_rn(fmax(pj, 1e-300));  // no IEEE division on the serial path
                const double s = a[j] * inv;  // l_jk for lane k > j
#pragma unroll
                for (int i = j + 1; i < 32; ++i)
                    if (i <= lane) a[i] = fma(-rowb[i], s, a[i]);
                __syncwarp();
            }
            // rank test on the pivots (first failing column of the block)
            const int gj = pb * 32 + lane;
            bool badc = false, unsure = false;
            if (gj < c) {
                const bool bp = !(piv > (p.rank_test ? 1e-12 : 0.0)) || !isfinite(piv) || !(ds[gj] > 0.0);
                const double rkk = bp ? 0.0 : sqrt(piv) * ds[gj];
                badc = bp || (p.rank_test && rkk < thresh);
                unsure = p.rank_test && !bp && (piv < kRankCertPiv || rkk < kRankCertRel * scale);
            }
            if (p.rank_need && __any_sync(0xffffffffu, unsure) && lane == 0) atomicOr(p.rank_need + b, 1);
            const unsigned m = __ballot_sync(0xffffffffu, badc);
            if (m) {
                if (lane == 0) {
                    record(p.rank_test ? kRankDeficient : kNotFinite, pb * 32 + __ffs(m) - 1);
                    fail = 1;
                }
            } else {
                // R[i][k] = D[i][k] / sqrt(piv_i); rows scaled through the broadcast
                const double rinv = 1.0 / sqrt(fmax(piv, 1e-300));
                rowb[lane] = rinv;
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i <= lane) a[i] = (i == lane) ? sqrt(fmax(piv, 1e-300)) : a[i] * rowb[i];
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i <= lane) D[sw(i, lane)] = a[i];
                // X = R^-1, column `lane`, bottom-up: x[i] = (delta_ik - sum_{l>i} R[i][l] x[l]) / R[i][i],
                // the division as a product with 1/R[i][i] (rinvb)
                double* rinvb = xloc;  // free until the panel-row phase
                rinvb[lane] = rinv;
                // R is in D (written above): broadcast reads, no per-row barrier; the sum
                // runs from the oldest x (l = 31) to the newest (l = i + 1), so each
                // row's chain waits on the previous row only for its last term
                __syncwarp();
                double x[32];
#pragma unroll
                for (int i = 31; i >= 0; --i) {
                    double s0 = (i == lane) ? 1.0 : 0.0;
#pragma unroll
                    for (int l = 31; l > i; --l)
                        if (l <= lane) s0 = fma(-D[sw(i, l)], x[l], s0);
                    x[i] = (i <= lane) ? s0 * rinvb[i] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) xpub[sw(i, lane)] = x[i];
                // B's diagonal block (rows scaled by 1/d) and, for the row-parallel
                // solve, the same X_pp; lower blocks of B zero
#pragma unroll
                for (int i = 0; i < 32; ++i) Bo[(int64_t)(pb * 32 + i) * p.ldb + pb * 32 + lane] = x[i] * rds[pb * 32 + i];
            }
        }
        CXT(8 + pb * 8 + 1, rank == owner && tid == 0);
        if (rank == owner) {
            // zero the lower blocks of B's block row pb (the triangular product reads whole 64-tiles)
            for (int e = tid; e < 32 * pb * 32; e += XNT) {
                const int r = e / (pb * 32), k = e % (pb * 32);
                Bo[(int64_t)(pb * 32 + r) * p.ldb + k] = 0.0;
            }
        }
        sync_cluster();
        CXT(8 + pb * 8 + 2, rank == 0 && tid == 0);
        // the owner's verdict (uniform exit)
        int f = fail;
        if (CL > 1 && rank != owner) f = *cluster.map_shared_rank(&fail, owner);
        if (f) {
            sync_cluster();  // no CTA leaves while another may still read its shared memory
            return;
        }
        if (pb + 1 == P) break;
        // ---- 2. panel row R_pq = X_pp^T A_pq for the owned columns q > p
        const double* X = xpub;
        if (CL > 1 && rank != owner) {
            const double* xr = cluster.map_shared_rank(xpub, owner);
            for (int e = tid; e < 1024; e += XNT) xloc[e] = xr[e];
            __syncthreads();
            X = xloc;
        }
        {
            // owned q > pb, one block per warp
            int q0 = rank;
            while (q0 <= pb) q0 += CL;
            for (int q = q0 + CL * warp; q < P; q += CL * XNW) {
                double* A_ = blk + (int64_t)lblk(pb, q, CL) * 1024;
                double acc[4][4][2];
                zero4(acc);
                blk_mma(acc, [&](int mm, int k) { return X[sw(k, mm)]; }, [&](int k, int n) { return A_[sw(k, n)]; }, g,
                        t);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int r = 8 * i + g, cc = 8 * j + 2 * t;
                        A_[sw(r, cc)] = acc[i][j][0];
                        A_[sw(r, cc + 1)] = acc[i][j][1];
                        if (p.skip_inverse) {  // R~ for the row-parallel solve
                            double* dst = Ag + (int64_t)(pb * 32 + r) * p.lda + q * 32 + cc;
                            dst[0] = acc[i][j][0];
                            dst[1] = acc[i][j][1];
                        }
                    }
            }
        }
        CXT(8 + pb * 8 + 3, rank == 0 && tid == 0);
        sync_cluster();
        CXT(8 + pb * 8 + 4, rank == 0 && tid == 0);
        // ---- 3. trailing update A_qr -= R_pq^T R_pr, owned columns r > p, p < q <= r
        {
            int r0 = rank;
            while (r0 <= pb) r0 += CL;
            int nown = 0;
            for (int r = r0; r < P; r += CL) nown += r - pb;
            for (int e = warp; e < nown; e += XNW) {
                // e -> (q, r): owned columns in order, q = pb+1 .. r
                int r = r0, ee = e;
                while (ee >= r - pb) {
                    ee -= r - pb;
                    r += CL;
                }
                const int q = pb + 1 + ee;
                const double* Rq = block_of(pb, q);
                const double* Rr = blk + (int64_t)lblk(pb, r, CL) * 1024;
                double* T_ = blk + (int64_t)lblk(q, r, CL) * 1024;
                double acc[4][4][2];
                zero4(acc);
                blk_mma(acc, [&](int mm, int k) { return Rq[sw(k, mm)]; }, [&](int k, int n) { return Rr[sw(k, n)]; },
                        g, t);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int rr = 8 * i + g, cc = 8 * j + 2 * t;
                        T_[sw(rr, cc)] -= acc[i][j][0];
                        T_[sw(rr, cc + 1)] -= acc[i][j][1];
                    }
            }
        }
        __syncthreads();
        CXT(8 + pb * 8 + 5, rank == 0 && tid == 0);
    }
    CXT(1, tid == 0 && rank == 0);
    if (p.skip_inverse) {
        sync_cluster();
        return;
    }
    // ---- back-substitution X = R~^-1 by block columns (independent): the warp
    // owning column q computes X_pq = -X_pp sum_{s=p+1..q} R_ps X_sq for p = q-1..0.
    // X_sq (s > p) of this column are read back from B (written above, L2);
    // B holds D^-1 X, so X_sq = d_row * B_sq.
    sync_cluster();  // every diagonal block of B written; R final everywhere
    double* stage = xloc;  // 32 x 32 staging per warp would exceed smem: one warp at a time per column uses
                           // registers only (A from DSMEM/smem, B from L2)
    (void)stage;
    {
        int q0 = rank;
        for (int q = q0 + CL * warp; q < P; q += CL * XNW) {
            for (int pbb = q - 1; pbb >= 0; --pbb) {
                double acc[4][4][2];
                zero4(acc);
                for (int s = pbb + 1; s <= q; ++s) {
                    const double* Rps = block_of(pbb, s);
                    const double* Xsq = Bo + (int64_t)(s * 32) * p.ldb + q * 32;
                    blk_mma(acc, [&](int mm, int k) { return Rps[sw(mm, k)]; },
                            [&](int k, int n) { return __ldcg(Xsq + (int64_t)k * p.ldb + n) * ds[s * 32 + k]; }, g, t);
                }
                // X_pq = -X_pp (acc): X_pp = d_row * B_pp
                double out[4][4][2];
                zero4(out);
                // stage acc through registers -> need acc as B operand: write to global B block (p, q) first
                double* Bpq = Bo + (int64_t)(pbb * 32) * p.ldb + q * 32;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int rr = 8 * i + g, cc = 8 * j + 2 * t;
                        Bpq[(int64_t)rr * p.ldb + cc] = acc[i][j][0];
                        Bpq[(int64_t)rr * p.ldb + cc + 1] = acc[i][j][1];
                    }
                __syncwarp();
                __threadfence_block();
                const double* Bpp = Bo + (int64_t)(pbb * 32) * p.ldb + pbb * 32;
                blk_mma(out, [&](int mm, int k) { return __ldcg(Bpp + (int64_t)mm * p.ldb + k) * ds[pbb * 32 + mm]; },
                        [&](int k, int n) { return __ldcg(Bpq + (int64_t)k * p.ldb + n); }, g, t);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int rr = 8 * i + g, cc = 8 * j + 2 * t;
                        Bpq[(int64_t)rr * p.ldb + cc] = -out[i][j][0] * rds[pbb * 32 + rr];
                        Bpq[(int64_t)rr * p.ldb + cc + 1] = -out[i][j][1] * rds[pbb * 32 + rr];
                    }
                __syncwarp();
                __threadfence_block();
            }
        }
    }
    sync_cluster();
    CXT(2, tid == 0 && rank == 0);
}

template <int CL>
void launch_cholx(const CholParams& p, int P, cudaStream_t st) {
    const int bytes = cholx_bytes(P, CL);
    ensure_smem((const void*)cholx_kernel<CL>, bytes);
    if (CL > 8) cudaFuncSetAttribute(cholx_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.batch * CL);
    cfg.blockDim = dim3(XNT);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ::smg::count_launch();
    cudaLaunchKernelEx(&cfg, cholx_kernel<CL>, p);
}

}  // namespace

// cluster size for the shared-memory Cholesky: the smallest that fits, more
// CTAs for few chains (latency), 0 when c is out of range
int cholx_cluster(int c_cap, int batch) {
    const int P = (c_cap + 31) / 32;
    // up to 2 panels the old single-CTA kernel is as fast (c = 60: 89 vs 92 us per position)
    if (P < 3 || P > kXMaxP) return 0;
    static const int force = std::getenv("SMG_CHOLX_CL") ? std::atoi(std::getenv("SMG_CHOLX_CL")) : 0;
    const int limit = 227 * 1024;
    // single chains: the widest cluster (latency); small batches: pairs (a wide
    // cluster per chain delays the other chain group's kernels); large: fit
    int want = batch == 1 ? 8 : (batch <= 16 ? 2 : 1);
    if (force > 0) want = force;
    for (int cl : {1, 2, 4, 8}) {
        if (cl < want && cl < P) continue;
        if (cholx_bytes(P, cl) <= limit) return cl;
    }
    return 0;
}

bool cholx_factor(const CholParams& p, cudaStream_t st) {
    if (p.near_identity || std::getenv("SMG_CHOLX_OFF")) return false;
    const int P = (p.c_cap + 31) / 32;
    const int cl = cholx_cluster(p.c_cap, p.batch);
    switch (cl) {
        case 1: launch_cholx<1>(p, P, st); return true;
        case 2: launch_cholx<2>(p, P, st); return true;
        case 4: launch_cholx<4>(p, P, st); return true;
        case 8: launch_cholx<8>(p, P, st); return true;
        default: return false;
    }
}

}  // namespace smg

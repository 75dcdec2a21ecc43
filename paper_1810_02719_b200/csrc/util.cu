// Boundary and data-movement kernels: layout conversion at the C ABI, local
// coordinate gather (Submesh::local_coords, partition.hpp:42-46) with the DOI
// bounding-box diagonal (spectral.hpp:228-231), seeded random blocks, the CSR
// SpMM (K4) and the degree-weighted stitch (K11, partition.hpp:311-355).
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

__global__ void to_rowmajor_kernel(const double* cm, int rows, int cols, double* rm, int64_t ld) {
    const int64_t total = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / rows), i = (int)(e % rows);
        rm[(int64_t)i * ld + j] = cm[e];
    }
}

__global__ void to_colmajor_kernel(const double* rm, int64_t ld, int rows, int cols, const double* sign,
                                   double* cm) {
    const int64_t total = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / rows), i = (int)(e % rows);
        const double s = sign ? sign[j] : 1.0;
        cm[e] = s * rm[(int64_t)i * ld + j];
    }
}

__global__ void fill_kernel(double* p, int64_t count, double v) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        p[e] = v;
}

// one CTA per tile: X (n x 3 row-major) and bbox diagonal
__global__ void gather_kernel(const TileRef* tiles, int n, double* X, int64_t strideX, double* bbox) {
    __shared__ double red[6][32];
    const TileRef t = tiles[blockIdx.x];
    double* out = X + (int64_t)blockIdx.x * strideX;
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int g = t.members[i];
        const double v[3] = {t.x[g], t.y[g], t.z[g]};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            out[3 * i + a] = v[a];
            mn[a] = fmin(mn[a], v[a]);
            mx[a] = fmax(mx[a], v[a]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
        for (int a = 0; a < 3; ++a) {
            red[a][w] = mn[a];
            red[3 + a][w] = mx[a];
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
            for (int a = 0; a < 3; ++a) {
                lo[a] = fmin(lo[a], red[a][k]);
                hi[a] = fmax(hi[a], red[3 + a][k]);
            }
        const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        bbox[blockIdx.x] = n > 0 ? sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)))
                                 : 0.0;
    }
}

SMG_DEV uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__global__ void randn_kernel(double* p, int rows, int cols, int64_t ld, int64_t stride, uint64_t seed) {
    const int b = blockIdx.y;
    const int64_t total = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / cols), j = (int)(e % cols);
        // the same start block for every batch entry: a chain's result must not
        // depend on its position in a batch
        const uint64_t h1 = splitmix(seed ^ splitmix((uint64_t)e * 2));
        const uint64_t h2 = splitmix(h1 + 0x632be59bd9b4e019ULL);
        const double u1 = ((h1 >> 11) + 1) * (1.0 / 9007199254740993.0);
        const double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
        p[(int64_t)b * stride + (int64_t)i * ld + j] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

// K4: Y = (L + shift I) X, warp per row, CSR rows of the CTA staged in smem,
// lanes sweep the row of X (coalesced, double2-vectorised when c is even).
constexpr int SPMM_NT = 256, SPMM_ROWS = 8, SPMM_MAXNZ = 32;
__global__ void __launch_bounds__(SPMM_NT) spmm_kernel(SpmmParams p) {
    __shared__ int32_t scol[SPMM_ROWS][SPMM_MAXNZ];
    __shared__ double sval[SPMM_ROWS][SPMM_MAXNZ];
    __shared__ int snz[SPMM_ROWS];
    const int b = blockIdx.y;
    const int c = p.dimC ? p.dimC[(int64_t)b * p.dimStride] : p.c;
    const int32_t* rowptr = p.rowptr + (int64_t)b * p.strideRowptr;
    const int64_t base = p.csr_offsets ? p.csr_offsets[(int64_t)b * p.offStride] : 0;
    const int32_t* cols = p.cols + base;
    const double* vals = p.vals + base;
    const double shift = p.shift ? p.shift[b] : 0.0;
    const double* X = p.X + (int64_t)b * p.strideX;
    double* Y = p.Y + (int64_t)b * p.strideY;
    const double alpha = p.alpha ? p.alpha[b] : 1.0;
    const double gam = p.gamma ? p.gamma[b] : 0.0;
    const double* Zb = p.Z ? p.Z + (int64_t)b * p.strideZ : nullptr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * SPMM_ROWS + warp;
    int s = 0, nzt = 0;
    if (i < p.n) {
        s = rowptr[i];
        nzt = rowptr[i + 1] - s;
        const int nz = min(nzt, SPMM_MAXNZ);
        for (int q = lane; q < nz; q += 32) {
            scol[warp][q] = cols[s + q];
            sval[warp][q] = vals[s + q] + (cols[s + q] == i ? shift : 0.0);
        }
        if (lane == 0) snz[warp] = nz;
    }
    __syncthreads();
    if (i >= p.n) return;
    const int nz = snz[warp];
    // entries past the staged ones (rows with > SPMM_MAXNZ neighbours) come from L2
    auto col_of = [&](int q) { return q < SPMM_MAXNZ ? scol[warp][q] : cols[s + q]; };
    auto val_of = [&](int q) {
        return q < SPMM_MAXNZ ? sval[warp][q] : vals[s + q] + (cols[s + q] == i ? shift : 0.0);
    };
    if ((c & 1) == 0 && (p.ldx & 1) == 0 && (p.ldy & 1) == 0) {
        // U column groups of 64 per pass: every neighbour row contributes U
        // independent double2 loads per lane, so up to nz*U loads are in flight
        constexpr int U = 4;
        for (int j0 = 2 * lane; j0 < c; j0 += 64 * U) {
            double2 acc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
            auto add_row = [&](double v, int col) {
                const double* xr = X + (int64_t)col * p.ldx;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + 64 * u;
                    if (j < c) {
                        const double2 x = *reinterpret_cast<const double2*>(xr + j);
                        acc[u].x = fma(v, x.x, acc[u].x);
                        acc[u].y = fma(v, x.y, acc[u].y);
                    }
                }
            };
            for (int q = 0; q < nz; ++q) add_row(sval[warp][q], scol[warp][q]);
            for (int q = nz; q < nzt; ++q) add_row(val_of(q), col_of(q));
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + 64 * u;
                if (j >= c) continue;
                double2 a = acc[u];
                a.x *= alpha;
                a.y *= alpha;
                if (Zb) {
                    const double2 z = *reinterpret_cast<const double2*>(Zb + (int64_t)i * p.ldz + j);
                    a.x = fma(gam, z.x, a.x);
                    a.y = fma(gam, z.y, a.y);
                }
                *reinterpret_cast<double2*>(Y + (int64_t)i * p.ldy + j) = a;
            }
        }
    } else {
        for (int j = lane; j < c; j += 32) {
            double acc = 0.0;
            for (int q = 0; q < nzt; ++q) acc = fma(val_of(q), X[(int64_t)col_of(q) * p.ldx + j], acc);
            acc *= alpha;
            if (Zb) acc = fma(gam, Zb[(int64_t)i * p.ldz + j], acc);
            Y[(int64_t)i * p.ldy + j] = acc;
        }
    }
}

// ---- stitch: owners of every global vertex, sorted by submesh id
__global__ void owner_count_kernel(const int32_t* members, int64_t count, int32_t* cnt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[members[e]], 1);
}

__global__ void owner_fill_kernel(const int32_t* members, int64_t count, int n_d, const int32_t* offs,
                                  int32_t* fillpos, int64_t* slots) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const int g = members[e];
        const int at = atomicAdd(&fillpos[g], 1);
        slots[offs[g] + at] = e;  // e = submesh_id * n_d + local index: ordering by e == ordering by id
    }
}

__global__ void owner_sort_kernel(int n, const int32_t* offs, int64_t* slots) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
        const int s = offs[g], e = offs[g + 1];
        for (int a = s + 1; a < e; ++a) {
            const int64_t x = slots[a];
            int b = a - 1;
            while (b >= s && slots[b] > x) {
                slots[b + 1] = slots[b];
                --b;
            }
            slots[b + 1] = x;
        }
    }
}

// partition.hpp:321-346: out = sum_s w x^_s / sum_s w in submesh-id order,
// w = local degree (Weighted) or 1; all-zero weights fall back to the plain mean.
__global__ void stitch_kernel(StitchParams p) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < p.n; g += gridDim.x * blockDim.x) {
        const int s = p.offs[g], e = p.offs[g + 1];
        double o[3] = {0.0, 0.0, 0.0}, f[3] = {0.0, 0.0, 0.0}, ws = 0.0;
        for (int q = s; q < e; ++q) {
            const int64_t slot = p.slots[q];
            const int sid = (int)(slot / p.n_d), li = (int)(slot % p.n_d);
            const int32_t* rp = p.rowptr + (int64_t)sid * (p.n_d + 1);
            const double w = p.weighted ? (double)(rp[li + 1] - rp[li] - 1) : 1.0;
            const double* xh = p.xhat + (int64_t)sid * p.strideXhat + 3 * li;
            for (int a = 0; a < 3; ++a) {
                o[a] += w * xh[a];
                f[a] += xh[a];
            }
            ws += w;
        }
        const int copies = e - s;
        for (int a = 0; a < 3; ++a) {
            double v;
            if (copies == 0) v = 0.0;
            else if (ws > 0.0) v = o[a] / ws;
            else v = f[a] / (double)copies;
            p.out[(int64_t)a * p.n + g] = v;  // SoA (Eigen column-major Points)
        }
    }
}

__global__ void coverage_kernel(int n, const int32_t* offs, int32_t* missing) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x)
        if (offs[g + 1] == offs[g]) atomicAdd(missing, 1);
}

inline int blocks_for(int64_t total, int nt) { return (int)std::min<int64_t>((total + nt - 1) / nt, 8192); }

}  // namespace

void transpose_to_rowmajor(const double* cm, int rows, int cols, double* rm, int64_t ld, cudaStream_t st) {
    const int64_t total = (int64_t)rows * cols;
    if (total) ::smg::count_launch(), to_rowmajor_kernel<<<blocks_for(total, 256), 256, 0, st>>>(cm, rows, cols, rm, ld);
}

void transpose_to_colmajor(const double* rm, int64_t ld, int rows, int cols, const double* sign, double* cm,
                           cudaStream_t st) {
    const int64_t total = (int64_t)rows * cols;
    if (total) ::smg::count_launch(), to_colmajor_kernel<<<blocks_for(total, 256), 256, 0, st>>>(rm, ld, rows, cols, sign, cm);
}

void fill(double* p, int64_t count, double v, cudaStream_t st) {
    if (count) ::smg::count_launch(), fill_kernel<<<blocks_for(count, 256), 256, 0, st>>>(p, count, v);
}

void gather_coords(const TileRef* tiles, int ntiles, int n, double* X, int64_t strideX, double* bbox,
                   cudaStream_t st) {
    if (ntiles) ::smg::count_launch(), gather_kernel<<<ntiles, 256, 0, st>>>(tiles, n, X, strideX, bbox);
}

void randn(double* p, int rows, int cols, int64_t ld, int64_t stride, int batch, uint64_t seed, cudaStream_t st) {
    const int64_t total = (int64_t)rows * cols;
    ::smg::count_launch(), randn_kernel<<<dim3(blocks_for(total, 256), batch), 256, 0, st>>>(p, rows, cols, ld, stride, seed);
}

void spmm(const SpmmParams& p, cudaStream_t st) {
    ::smg::count_launch(), spmm_kernel<<<dim3((p.n + SPMM_ROWS - 1) / SPMM_ROWS, p.batch), SPMM_NT, 0, st>>>(p);
}

// ---- fused Chebyshev filter for binary-weight Laplacians (off-diagonal entries
// exactly -1, diagonal = degree): one CTA per (chain, CSL-column slice) holds
// the tile's CSR pattern, its shifted diagonal and two iterates in shared
// memory and runs all deg steps of X_i = alpha_i (L + s I) X_{i-1} + gamma_i
// X_{i-2} there (X_{i-2} is overwritten in place by the thread that owns its
// row).  The per-element arithmetic is spmm_kernel's: v = vals[q] (+ s on the
// diagonal), acc = fma(v, x, acc) in CSR order, acc * alpha, fma(gamma, z, .).
template <int CSL>
__global__ void __launch_bounds__(1024) cheb_bin_kernel(ChebParams p) {
    extern __shared__ __align__(16) double cbuf[];
    const int b = blockIdx.y, col0 = blockIdx.x * CSL, n = p.n;
    const int64_t half = (int64_t)n * CSL;
    double* dg = cbuf + 2 * half;                           // vals[diag] + shift per row
    int32_t* rp = reinterpret_cast<int32_t*>(dg + n);       // n + 1
    int32_t* cl = rp + n + 1;                               // nnz
    const int32_t* rowptr = p.rowptr + (int64_t)b * p.strideRowptr;
    const int64_t base = p.csr_offsets ? p.csr_offsets[(int64_t)b * p.offStride] : 0;
    const int32_t* cols = p.cols + base;
    const double* vals = p.vals + base;
    const double shift = p.coef[(int64_t)2 * p.deg * p.batch + b];
    for (int i = threadIdx.x; i <= n; i += blockDim.x) rp[i] = rowptr[i];
    __syncthreads();
    const int nnz = rp[n];
    for (int q = threadIdx.x; q < nnz; q += blockDim.x) {
        const int col = cols[q];
        cl[q] = col;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int q = rp[i]; q < rp[i + 1]; ++q)
            if (cols[q] == i) dg[i] = vals[q] + shift;
    const double* X = p.X + (int64_t)b * p.strideX;
    // iterates column-major within the slice ([u][row]): the q-th neighbours of
    // consecutive rows are consecutive rows on a structured tile, so a warp's
    // reads of one column hit consecutive banks
    for (int e = threadIdx.x; e < n * CSL; e += blockDim.x) {
        const int u = e / n, i = e % n, j = col0 + u;
        cbuf[e] = j < p.c ? X[(int64_t)i * p.ldx + j] : 0.0;
    }
    __syncthreads();
    for (int step = 1; step <= p.deg; ++step) {
        const double alpha = p.coef[(int64_t)(step - 1) * p.batch + b];
        const double gam = step > 1 ? p.coef[(int64_t)p.deg * p.batch + (int64_t)(step - 1) * p.batch + b] : 0.0;
        const double* xc = cbuf + ((step - 1) & 1) * half;
        double* xo = cbuf + (step & 1) * half;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double acc[CSL];
#pragma unroll
            for (int u = 0; u < CSL; ++u) acc[u] = 0.0;
            const double di = dg[i];
            for (int q = rp[i]; q < rp[i + 1]; ++q) {
                const int col = cl[q];
                const double v = col == i ? di : -1.0;
#pragma unroll
                for (int u = 0; u < CSL; ++u) acc[u] = fma(v, xc[u * n + col], acc[u]);
            }
#pragma unroll
            for (int u = 0; u < CSL; ++u) {
                double a = acc[u] * alpha;
                if (step > 1) a = fma(gam, xo[u * n + i], a);
                xo[u * n + i] = a;
            }
        }
        __syncthreads();
    }
    const double* res = cbuf + (p.deg & 1) * half;
    double* Y = p.Y + (int64_t)b * p.strideY;
    for (int e = threadIdx.x; e < n * CSL; e += blockDim.x) {
        const int u = e / n, i = e % n, j = col0 + u;
        if (j < p.c) Y[(int64_t)i * p.ldy + j] = res[e];
    }
}

int cheb_bin_bytes(int n, int max_nnz, int csl) {
    return 2 * n * csl * 8 + n * 8 + ((n + 1 + max_nnz + 1) / 2) * 8;
}

bool cheb_filter_supported(int n, int max_nnz) { return cheb_bin_bytes(n, max_nnz, 2) <= 227 * 1024; }

void cheb_filter(const ChebParams& p, int max_nnz, cudaStream_t st) {
    auto go = [&](auto kernel, int csl) {
        const int bytes = cheb_bin_bytes(p.n, max_nnz, csl);
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        ::smg::count_launch(), kernel<<<dim3((p.c + csl - 1) / csl, p.batch), 1024, bytes, st>>>(p);
    };
    if (cheb_bin_bytes(p.n, max_nnz, 4) <= 227 * 1024) go(cheb_bin_kernel<4>, 4);
    else go(cheb_bin_kernel<2>, 2);
}

void Stitcher::build(const int32_t* members, int nsub, int n_d, int n, cudaStream_t st) {
    this->n = n;
    this->n_d = n_d;
    const int64_t count = (int64_t)nsub * n_d;
    cudaMallocAsync(&offs, sizeof(int32_t) * (n + 1), st);
    cudaMallocAsync(&slots, sizeof(int64_t) * std::max<int64_t>(count, 1), st);
    int32_t* cnt;
    cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), st);
    cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), st);
    if (count) ::smg::count_launch(), owner_count_kernel<<<blocks_for(count, 256), 256, 0, st>>>(members, count, cnt);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, offs, n + 1, st);
    void* tmp;
    cudaMallocAsync(&tmp, tmp_bytes, st);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, offs, n + 1, st);
    cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), st);
    if (count) ::smg::count_launch(), owner_fill_kernel<<<blocks_for(count, 256), 256, 0, st>>>(members, count, n_d, offs, cnt, slots);
    ::smg::count_launch(), owner_sort_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, offs, slots);
    cudaMallocAsync(&missing, sizeof(int32_t), st);
    cudaMemsetAsync(missing, 0, sizeof(int32_t), st);
    ::smg::count_launch(), coverage_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, offs, missing);
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(cnt, st);
}

void Stitcher::release(cudaStream_t st) {
    if (offs) cudaFreeAsync(offs, st);
    if (slots) cudaFreeAsync(slots, st);
    if (missing) cudaFreeAsync(missing, st);
    offs = nullptr;
    slots = nullptr;
    missing = nullptr;
}

void stitch(const StitchParams& p, cudaStream_t st) {
    ::smg::count_launch(), stitch_kernel<<<blocks_for(p.n, 256), 256, 0, st>>>(p);
}

}  // namespace smg

// K1: induced-submesh Laplacian assembly (bit-exact CSR) and the orderings.
//
// Replaces detail::build_submesh's adjacency/degree part (partition.hpp:169-184)
// and build_laplacian (spectral.hpp:39-68): L = D - C with D_ii = number of
// in-submesh neighbours and C_ij = 1 (Binary) or 1/||v_i - v_j||^2 (distance,
// squared norm summed ((dx^2 + dy^2) + dz^2) like Eigen's squaredNorm on a
// non-contiguous row).  Eigen's setFromTriplets sorts every column by row; for
// the symmetric L those are our CSR rows with ascending column index.  The
// local order is ascending global id, so a member's local index is its rank in
// the sorted member list (binary search in shared memory, no n-sized map as in
// the reference's local_of vector).  One CTA per submesh; all submeshes of all
// chains are assembled in one launch because assembly depends on connectivity
// (and coordinates only for distance weighting), never on the chain carry.
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int NT = 256;
constexpr int MAXN = 4096;

SMG_DEV int find_local(const int32_t* __restrict__ m, int n, int g) {
    int lo = 0, hi = n - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int v = m[mid];
        if (v == g) return mid;
        if (v < g) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

__global__ void __launch_bounds__(NT) count_kernel(const TileRef* tiles, int n, int32_t* nnz_out) {
    __shared__ int32_t mem[MAXN];
    __shared__ double red[32];
    const TileRef t = tiles[blockIdx.x];
    for (int i = threadIdx.x; i < n; i += NT) mem[i] = t.members[i];
    __syncthreads();
    double cnt = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) {
        const int gi = mem[i];
        int c = 1;
        for (int e = t.adj_offsets[gi]; e < t.adj_offsets[gi + 1]; ++e)
            if (find_local(mem, n, t.adj_cols[e]) >= 0) ++c;
        cnt += c;
    }
    cnt = block_sum(cnt, red);
    if (threadIdx.x == 0) nnz_out[blockIdx.x] = (int32_t)cnt;
}

__global__ void __launch_bounds__(NT) fill_kernel(const TileRef* tiles, int n, int weighting,
                                                  const int64_t* csr_offsets, int32_t* rowptr_all,
                                                  int32_t* cols_all, double* vals_all, double* trace,
                                                  int* status, int64_t* detail) {
    __shared__ int32_t mem[MAXN];
    __shared__ int32_t rcount[MAXN];
    __shared__ int32_t part[NT + 1];
    __shared__ double red[32];
    const int tile = blockIdx.x;
    const TileRef t = tiles[tile];
    int32_t* rowptr = rowptr_all + (int64_t)tile * (n + 1);
    int32_t* cols = cols_all + csr_offsets[tile];
    double* vals = vals_all + csr_offsets[tile];
    for (int i = threadIdx.x; i < n; i += NT) mem[i] = t.members[i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
        const int gi = mem[i];
        int c = 1;
        for (int e = t.adj_offsets[gi]; e < t.adj_offsets[gi + 1]; ++e)
            if (find_local(mem, n, t.adj_cols[e]) >= 0) ++c;
        rcount[i] = c;
    }
    __syncthreads();
    // exclusive scan of rcount over contiguous chunks
    const int chunk = (n + NT - 1) / NT;
    const int b0 = threadIdx.x * chunk, b1 = min(n, b0 + chunk);
    int s = 0;
    for (int i = b0; i < b1; ++i) s += rcount[i];
    part[threadIdx.x + 1] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        part[0] = 0;
        for (int i = 1; i <= NT; ++i) part[i] += part[i - 1];
    }
    __syncthreads();
    int run = part[threadIdx.x];
    for (int i = b0; i < b1; ++i) {
        rowptr[i] = run;
        run += rcount[i];
    }
    if (threadIdx.x == NT - 1) rowptr[n] = part[NT];
    __syncthreads();
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) {
        const int gi = mem[i];
        const int deg = rcount[i] - 1;
        int pos = rowptr[i];
        bool diag_done = false;
        for (int e = t.adj_offsets[gi]; e < t.adj_offsets[gi + 1]; ++e) {
            const int gj = t.adj_cols[e];
            const int j = find_local(mem, n, gj);
            if (j < 0) continue;
            if (!diag_done && j > i) {
                cols[pos] = i;
                vals[pos] = (double)deg;
                ++pos;
                diag_done = true;
            }
            double w = 1.0;
            if (weighting == 1) {
                const double dx = t.x[gi] - t.x[gj];
                const double dy = t.y[gi] - t.y[gj];
                const double dz = t.z[gi] - t.z[gj];
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                const double inv = 1.0 / d2;
                if (!(d2 > 0.0) || !isfinite(inv)) {
                    // first offending (row, neighbour slot) in the reference's loop order
                    const long long key = ((long long)i << 20) | (long long)(e - t.adj_offsets[gi]);
                    atomicMin(reinterpret_cast<unsigned long long*>(detail + tile),
                              (unsigned long long)key);
                    status[tile] = kCoincident;
                }
                w = inv;
            }
            cols[pos] = j;
            vals[pos] = -w;
            ++pos;
        }
        if (!diag_done) {
            cols[pos] = i;
            vals[pos] = (double)deg;
        }
        tr += (double)deg;  // integer degrees: the sum is exact in any order
    }
    tr = block_sum(tr, red);
    if (threadIdx.x == 0) trace[tile] = tr;
}

__global__ void scan_kernel(const int32_t* in, int64_t* out, int count) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t run = 0;
    for (int i = 0; i < count; ++i) {
        out[i] = run;
        run += in[i];
    }
    out[count] = run;
}

// Half-bandwidth and the smallest block width W_t for which the (permuted)
// matrix is block tridiagonal: b - 1 if that works (grid tiles: b = width + 1),
// else b.
__global__ void __launch_bounds__(NT) bandwidth_kernel(const int32_t* rowptr_all, const int32_t* cols_all,
                                                       const int64_t* csr_offsets, const int32_t* perm_all, int n,
                                                       int32_t* bw_out, int32_t* blockw_out, int32_t* lower_out) {
    __shared__ int32_t pos[MAXN];
    __shared__ int red_i[3];
    const int tile = blockIdx.x;
    const int32_t* rowptr = rowptr_all + (int64_t)tile * (n + 1);
    const int32_t* cols = cols_all + csr_offsets[tile];
    const int32_t* perm = perm_all ? perm_all + (int64_t)tile * n : nullptr;
    for (int i = threadIdx.x; i < n; i += NT) pos[perm ? perm[i] : i] = i;
    if (threadIdx.x == 0) {
        red_i[0] = 0;
        red_i[1] = 0;
        red_i[2] = 0;
    }
    __syncthreads();
    int bw = 0, low = 0;
    for (int i = threadIdx.x; i < n; i += NT) {
        int li = 0;
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            bw = max(bw, abs(pos[i] - pos[cols[e]]));
            li += pos[cols[e]] < pos[i];
        }
        low = max(low, li);
    }
    atomicMax(&red_i[0], bw);
    atomicMax(&red_i[2], low);
    __syncthreads();
    const int b = red_i[0];
    const int w = b - 1;
    int bad = 0;
    if (w >= 1) {
        for (int i = threadIdx.x; i < n; i += NT)
            for (int e = rowptr[i]; e < rowptr[i + 1]; ++e)
                if (abs(pos[i] / w - pos[cols[e]] / w) > 1) bad = 1;
    } else {
        bad = 1;
    }
    if (bad) atomicOr(&red_i[1], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        bw_out[tile] = b;
        blockw_out[tile] = red_i[1] ? max(b, 1) : w;
        if (lower_out) lower_out[tile] = red_i[2];
    }
}


// Geometric ordering candidate: local vertices sorted by their coordinate along
// the axis of largest extent, ties by the second-largest axis, then by index.
// On a grid tile this is the lexicographic order along the long side, whose
// bandwidth is the short side + 1 (a 32 x 64 tile: W = 32 instead of 64).
// One CTA per tile, bitonic sort of (key1, key2, index) in shared memory.
__global__ void __launch_bounds__(512) axis_order_kernel(const double* X_all, int64_t strideX, int n, int32_t* perm_all) {
    extern __shared__ __align__(16) double asort[];
    int N2 = 1;
    while (N2 < n) N2 <<= 1;
    double* k1 = asort;
    double* k2 = k1 + N2;
    int* id = reinterpret_cast<int*>(k2 + N2);
    __shared__ double wlo[16][3], whi[16][3];
    __shared__ int axes[2];
    const int tile = blockIdx.x, tid = threadIdx.x;
    const double* X = X_all + (int64_t)tile * strideX;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = tid; i < n; i += blockDim.x)
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], X[(int64_t)i * 3 + d]);
            hi[d] = fmax(hi[d], X[(int64_t)i * 3 + d]);
        }
    for (int d = 0; d < 3; ++d)
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    if ((tid & 31) == 0)
        for (int d = 0; d < 3; ++d) {
            wlo[tid >> 5][d] = lo[d];
            whi[tid >> 5][d] = hi[d];
        }
    __syncthreads();
    if (tid == 0) {
        double e[3];
        for (int d = 0; d < 3; ++d) {
            double l = INFINITY, h = -INFINITY;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                l = fmin(l, wlo[w][d]);
                h = fmax(h, whi[w][d]);
            }
            e[d] = h - l;
        }
        int a0 = 0;
        for (int d = 1; d < 3; ++d)
            if (e[d] > e[a0]) a0 = d;
        int a1 = (a0 == 0) ? 1 : 0;
        for (int d = 0; d < 3; ++d)
            if (d != a0 && e[d] > e[a1]) a1 = d;
        axes[0] = a0;
        axes[1] = a1;
    }
    __syncthreads();
    const int a0 = axes[0], a1 = axes[1];
    for (int i = tid; i < N2; i += blockDim.x) {
        if (i < n) {
            k1[i] = X[(int64_t)i * 3 + a0];
            k2[i] = X[(int64_t)i * 3 + a1];
        } else {
            k1[i] = INFINITY;
            k2[i] = INFINITY;
        }
        id[i] = i;
    }
    __syncthreads();
    auto less = [&](int x, int y) {
        if (k1[x] != k1[y]) return k1[x] < k1[y];
        if (k2[x] != k2[y]) return k2[x] < k2[y];
        return id[x] < id[y];
    };
    for (int size = 2; size <= N2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < N2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    if (less(j, i) == up) {
                        double t1 = k1[i];
                        k1[i] = k1[j];
                        k1[j] = t1;
                        double t2 = k2[i];
                        k2[i] = k2[j];
                        k2[j] = t2;
                        int ti = id[i];
                        id[i] = id[j];
                        id[j] = ti;
                    }
                }
            }
            __syncthreads();
        }
    int32_t* perm = perm_all + (int64_t)tile * n;
    for (int r = tid; r < n; r += blockDim.x) perm[r] = id[r];
}

// Reverse Cuthill-McKee per tile (single-thread BFS in shared memory).
// Start vertex: George-Liu pseudo-peripheral search from the lowest-degree
// vertex; neighbours enqueued by (degree, index); every component restarts
// from its lowest-degree unvisited vertex.
__global__ void rcm_kernel(const int32_t* rowptr_all, const int32_t* cols_all, const int64_t* csr_offsets, int n,
                           int32_t* perm_all) {
    __shared__ int32_t order[MAXN];
    __shared__ int32_t level[MAXN];
    __shared__ int16_t deg[MAXN];
    const int tile = blockIdx.x;
    const int32_t* rowptr = rowptr_all + (int64_t)tile * (n + 1);
    const int32_t* cols = cols_all + csr_offsets[tile];
    int32_t* perm = perm_all + (int64_t)tile * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) deg[i] = (int16_t)(rowptr[i + 1] - rowptr[i] - 1);
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int i = 0; i < n; ++i) level[i] = -1;
    int placed = 0;
    while (placed < n) {
        // lowest-degree unvisited vertex
        int start = -1;
        for (int i = 0; i < n; ++i)
            if (level[i] < 0 && (start < 0 || deg[i] < deg[start])) start = i;
        // George-Liu: BFS from start, move to a min-degree vertex of the last level
        int ecc_prev = -1;
        for (int rep = 0; rep < 6; ++rep) {
            // BFS using order[placed..] as queue, marking with level base 1<<20 (temporary)
            int head = placed, tail = placed;
            order[tail++] = start;
            level[start] = (1 << 20);
            int last_begin = placed, last_end = tail, cur = 0;
            while (head < tail) {
                const int lvl_end = tail;
                last_begin = head;
                last_end = lvl_end;
                for (; head < lvl_end; ++head) {
                    const int v = order[head];
                    for (int e = rowptr[v]; e < rowptr[v + 1]; ++e) {
                        const int w = cols[e];
                        if (level[w] < 0) {
                            level[w] = (1 << 20) + cur + 1;
                            order[tail++] = w;
                        }
                    }
                }
                ++cur;
            }
            const int ecc = cur - 1;
            // reset temporary marks
            for (int q = placed; q < tail; ++q) level[order[q]] = -1;
            int cand = order[last_begin];
            for (int q = last_begin; q < last_end; ++q)
                if (deg[order[q]] < deg[cand] || (deg[order[q]] == deg[cand] && order[q] < cand)) cand = order[q];
            if (ecc <= ecc_prev) break;
            ecc_prev = ecc;
            start = cand;
        }
        // Cuthill-McKee from `start`
        int head = placed, tail = placed;
        order[tail++] = start;
        level[start] = 0;
        while (head < tail) {
            const int v = order[head++];
            const int first = tail;
            for (int e = rowptr[v]; e < rowptr[v + 1]; ++e) {
                const int w = cols[e];
                if (level[w] < 0) {
                    level[w] = 0;
                    order[tail++] = w;
                }
            }
            // insertion sort the new entries by (degree, index)
            for (int a = first + 1; a < tail; ++a) {
                const int x = order[a];
                int b = a - 1;
                while (b >= first && (deg[order[b]] > deg[x] || (deg[order[b]] == deg[x] && order[b] > x))) {
                    order[b + 1] = order[b];
                    --b;
                }
                order[b + 1] = x;
            }
        }
        placed = tail;
    }
    for (int p = 0; p < n; ++p) perm[p] = order[n - 1 - p];
}

}  // namespace

void assemble_count(const TileRef* tiles, int ntiles, int n, int32_t* nnz_out, cudaStream_t st) {
    if (ntiles) ::smg::count_launch(), count_kernel<<<ntiles, NT, 0, st>>>(tiles, n, nnz_out);
}

void assemble_fill(const TileRef* tiles, int ntiles, int n, int weighting, const int64_t* csr_offsets,
                   int32_t* rowptr, int32_t* cols, double* vals, double* trace, int* status,
                   int64_t* status_detail, cudaStream_t st) {
    if (ntiles)
        ::smg::count_launch(), fill_kernel<<<ntiles, NT, 0, st>>>(tiles, n, weighting, csr_offsets, rowptr, cols, vals, trace, status,
                                           status_detail);
}

void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int count, cudaStream_t st) {
    ::smg::count_launch(), scan_kernel<<<1, 32, 0, st>>>(in, out, count);
}

void natural_bandwidth(const int32_t* rowptr, const int32_t* cols, const int64_t* csr_offsets, const int32_t* perm,
                       int ntiles, int n, int32_t* bw_out, int32_t* blockw_out, int32_t* lower_out, cudaStream_t st) {
    if (ntiles)
        ::smg::count_launch(), bandwidth_kernel<<<ntiles, NT, 0, st>>>(rowptr, cols, csr_offsets, perm, n, bw_out,
                                                                      blockw_out, lower_out);
}

void axis_order(const double* X, int64_t strideX, int ntiles, int n, int32_t* perm, cudaStream_t st) {
    int N2 = 1;
    while (N2 < n) N2 <<= 1;
    const int bytes = N2 * (8 + 8 + 4);
    ensure_smem((const void*)axis_order_kernel, bytes);
    if (ntiles) ::smg::count_launch(), axis_order_kernel<<<ntiles, 512, bytes, st>>>(X, strideX, n, perm);
}

void rcm_order(const int32_t* rowptr, const int32_t* cols, const int64_t* csr_offsets, int ntiles, int n,
               int32_t* perm, cudaStream_t st) {
    if (ntiles) ::smg::count_launch(), rcm_kernel<<<ntiles, 128, 0, st>>>(rowptr, cols, csr_offsets, n, perm);
}

}  // namespace smg

// F4: two-stage bilateral fine denoising (denoise.hpp:11-180, mesh.hpp:87-116).
//
//  face_geometry        geom_kernel: centroid ((a+b)+c)/3, unit normal of
//                       (b-a) x (c-a), area 0.5 |cross|, degenerate flag -- one
//                       thread per face, explicitly rounded products/sums (no FMA
//                       contraction) so the geometry is the reference's doubles
//  faces_of_vertex      CSR by atomic count + scan + fill, lists sorted ascending
//  face_ring_adjacency  per face the union of its vertices' face lists (a 3-way
//                       merge with dedup); depth d > 1 unions the previous rings
//                       of the ring's faces (k-way merge); count pass + fill pass
//  default_sigma_spatial  per-face sums over ring members g > f, then a fixed-
//                       order device reduction (deterministic)
//  bilateral_normals    Jacobi sweeps, one thread per face, ring in ascending
//                       order, zero-area faces skipped, degenerate faces kept
//  update_vertices      per pass: centroids from the current vertices, then per
//                       vertex the mean of n_f (n_f . (m_f - v)) over its faces
// Face data is AoS double4 ({centroid, area}, {normal, 0}) so a ring gather is
// two 32-byte loads; vertices are AoS double4 inside the kernels.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "engine.h"
#include "kernels.h"
#include "profiler.h"

namespace smg {

namespace {

SMG_DEV double sq3(double x, double y, double z) { return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)); }

__global__ void to_aos_kernel(int64_t n, const double* x, const double* y, const double* z, double4* v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = make_double4(x[i], y[i], z[i], 0.0);
}

__global__ void to_soa_kernel(int64_t n, const double4* v, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double4 a = v[i];
        out[i] = a.x;
        out[n + i] = a.y;
        out[2 * n + i] = a.z;
    }
}

__global__ void check_faces_kernel(int64_t nf, const int32_t* faces, int64_t n, int* bad) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const int v = faces[3 * f + k];
            if (v < 0 || v >= n) atomicMin(bad, (int)f);
        }
}

SMG_DEV double4 centroid(const double4 a, const double4 b, const double4 c) {
    return make_double4(__ddiv_rn(__dadd_rn(__dadd_rn(a.x, b.x), c.x), 3.0),
                        __ddiv_rn(__dadd_rn(__dadd_rn(a.y, b.y), c.y), 3.0),
                        __ddiv_rn(__dadd_rn(__dadd_rn(a.z, b.z), c.z), 3.0), 0.0);
}

// mesh.hpp:94-116
__global__ void geom_kernel(int64_t nf, const int32_t* faces, const double4* v, double4* cen_area, double4* nrm,
                            int* degenerate) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const double4 a = v[faces[3 * f]], b = v[faces[3 * f + 1]], c = v[faces[3 * f + 2]];
        double4 m = centroid(a, b, c);
        const double ux = __dsub_rn(b.x, a.x), uy = __dsub_rn(b.y, a.y), uz = __dsub_rn(b.z, a.z);
        const double vx = __dsub_rn(c.x, a.x), vy = __dsub_rn(c.y, a.y), vz = __dsub_rn(c.z, a.z);
        const double cx = __dsub_rn(__dmul_rn(uy, vz), __dmul_rn(uz, vy));
        const double cy = __dsub_rn(__dmul_rn(uz, vx), __dmul_rn(ux, vz));
        const double cz = __dsub_rn(__dmul_rn(ux, vy), __dmul_rn(uy, vx));
        const double norm = __dsqrt_rn(sq3(cx, cy, cz));
        m.w = __dmul_rn(0.5, norm);
        cen_area[f] = m;
        if (norm > 0.0) {
            nrm[f] = make_double4(__ddiv_rn(cx, norm), __ddiv_rn(cy, norm), __ddiv_rn(cz, norm), 0.0);
            degenerate[f] = 0;
        } else {
            nrm[f] = make_double4(0.0, 0.0, 0.0, 0.0);
            degenerate[f] = 1;
        }
    }
}

__global__ void fov_count_kernel(int64_t nf, const int32_t* faces, int32_t* cnt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 3 * nf; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[faces[e]], 1);
}

__global__ void fov_fill_kernel(int64_t nf, const int32_t* faces, const int32_t* offs, int32_t* fill, int32_t* list) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 3 * nf; e += (int64_t)gridDim.x * blockDim.x) {
        const int v = faces[e];
        list[offs[v] + atomicAdd(&fill[v], 1)] = (int32_t)(e / 3);
    }
}

// sort each CSR row ascending (short rows: insertion sort)
__global__ void sort_rows_kernel(int64_t rows, const int32_t* offs, int32_t* list) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int s = offs[r], e = offs[r + 1];
        for (int a = s + 1; a < e; ++a) {
            const int32_t x = list[a];
            int b = a - 1;
            while (b >= s && list[b] > x) {
                list[b + 1] = list[b];
                --b;
            }
            list[b + 1] = x;
        }
    }
}

constexpr int kMaxUnion = 128;  // lists merged per face

// union of the sorted lists src_list[src_offs[id] ..] for the ids of face f:
// depth 1: ids = the face's 3 vertices (lists = faces of a vertex); depth > 1:
// ids = the face's previous ring (lists = previous rings).  out == nullptr: count.
template <int KMAX>
__global__ void ring_union_kernel(int64_t nf, const int32_t* id_offs, const int32_t* ids, const int32_t* faces,
                                  const int32_t* src_offs, const int32_t* src_list, const int32_t* out_offs,
                                  int32_t* out, int32_t* count, int* overflow) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        int head[KMAX], end[KMAX];
        int k = 0;
        if (faces) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int v = faces[3 * f + q];
                head[k] = src_offs[v];
                end[k] = src_offs[v + 1];
                ++k;
            }
        } else {
            const int s = id_offs[f], e = id_offs[f + 1];
            if (e - s > KMAX) {
                atomicExch(overflow, 1);
                continue;
            }
            for (int q = s; q < e; ++q) {
                const int g = ids[q];
                head[k] = src_offs[g];
                end[k] = src_offs[g + 1];
                ++k;
            }
        }
        int written = 0, last = -1;
        const int base = out ? out_offs[f] : 0;
        while (true) {
            int best = INT32_MAX;
#pragma unroll
            for (int q = 0; q < (KMAX == 3 ? 3 : k); ++q)
                if (head[q] < end[q]) best = min(best, src_list[head[q]]);
            if (best == INT32_MAX) break;
#pragma unroll
            for (int q = 0; q < (KMAX == 3 ? 3 : k); ++q)
                if (head[q] < end[q] && src_list[head[q]] == best) ++head[q];
            if (best != last) {
                if (out) out[base + written] = best;
                ++written;
                last = best;
            }
        }
        if (!out) count[f] = written;
    }
}

// denoise.hpp:67-83, per face: sum of |c_f - c_g| over ring members g > f (ascending)
__global__ void sigma_partial_kernel(int64_t nf, const int32_t* offs, const int32_t* ring, const double4* ca,
                                     double* sum, int32_t* cnt) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const double4 a = ca[f];
        double s = 0.0;
        int c = 0;
        for (int q = offs[f]; q < offs[f + 1]; ++q) {
            const int g = ring[q];
            if (g <= f) continue;
            const double4 b = ca[g];
            s = __dadd_rn(s, __dsqrt_rn(sq3(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z))));
            ++c;
        }
        sum[f] = s;
        cnt[f] = c;
    }
}

__global__ void sigma_final_kernel(const double* total, const int64_t* count, double* sigma, double given) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *sigma = given > 0.0 ? given : (*count > 0 ? *total / (double)*count : 0.0);
}

// denoise.hpp:87-127, one Jacobi sweep
__global__ void bilateral_kernel(int64_t nf, const int32_t* offs, const int32_t* ring, const double4* ca,
                                 const double4* cur, double4* next, const int* degenerate, const double* sigma_s,
                                 double sigma_r) {
    const double ss = *sigma_s;
    const double two_s = __dmul_rn(__dmul_rn(2.0, ss), ss);
    const double two_r = __dmul_rn(__dmul_rn(2.0, sigma_r), sigma_r);
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const double4 nf_ = cur[f];
        if (degenerate[f]) {
            next[f] = nf_;
            continue;
        }
        const double4 cf = ca[f];
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int q = offs[f]; q < offs[f + 1]; ++q) {
            const int g = ring[q];
            const double4 cg = ca[g];
            if (cg.w <= 0.0) continue;  // zero-area faces do not contribute
            const double4 ng = cur[g];
            const double ks = exp(-__ddiv_rn(sq3(__dsub_rn(cf.x, cg.x), __dsub_rn(cf.y, cg.y), __dsub_rn(cf.z, cg.z)), two_s));
            const double kr =
                exp(-__ddiv_rn(sq3(__dsub_rn(nf_.x, ng.x), __dsub_rn(nf_.y, ng.y), __dsub_rn(nf_.z, ng.z)), two_r));
            const double w = __dmul_rn(__dmul_rn(cg.w, ks), kr);
            ax = __dadd_rn(ax, __dmul_rn(w, ng.x));
            ay = __dadd_rn(ay, __dmul_rn(w, ng.y));
            az = __dadd_rn(az, __dmul_rn(w, ng.z));
        }
        const double norm = __dsqrt_rn(sq3(ax, ay, az));
        next[f] = norm > 0.0 ? make_double4(__ddiv_rn(ax, norm), __ddiv_rn(ay, norm), __ddiv_rn(az, norm), 0.0) : nf_;
    }
}

__global__ void centroid_kernel(int64_t nf, const int32_t* faces, const double4* v, double4* cen) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x)
        cen[f] = centroid(v[faces[3 * f]], v[faces[3 * f + 1]], v[faces[3 * f + 2]]);
}

// denoise.hpp:155-163
__global__ void vertex_update_kernel(int64_t n, const int32_t* offs, const int32_t* fov, const double4* nrm,
                                     const double4* cen, const double4* cur, double4* next) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const double4 p = cur[v];
        const int s = offs[v], e = offs[v + 1];
        if (s == e) {
            next[v] = p;
            continue;
        }
        double dx = 0.0, dy = 0.0, dz = 0.0;
        for (int q = s; q < e; ++q) {
            const int f = fov[q];
            const double4 nn = nrm[f], m = cen[f];
            const double d = __dadd_rn(__dadd_rn(__dmul_rn(nn.x, __dsub_rn(m.x, p.x)), __dmul_rn(nn.y, __dsub_rn(m.y, p.y))),
                                       __dmul_rn(nn.z, __dsub_rn(m.z, p.z)));
            dx = __dadd_rn(dx, __dmul_rn(nn.x, d));
            dy = __dadd_rn(dy, __dmul_rn(nn.y, d));
            dz = __dadd_rn(dz, __dmul_rn(nn.z, d));
        }
        const double k = (double)(e - s);
        next[v] = make_double4(__dadd_rn(p.x, __ddiv_rn(dx, k)), __dadd_rn(p.y, __ddiv_rn(dy, k)),
                               __dadd_rn(p.z, __ddiv_rn(dz, k)), 0.0);
    }
}

inline int grid_for(int64_t total, int nt = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((total + nt - 1) / nt, 148 * 32));
}

void scan_i32(const int32_t* in, int32_t* out, int64_t count, cudaStream_t st) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)count, st);
    DBuf<char> tmp;
    tmp.alloc(std::max<size_t>(bytes, 1), st);
    cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, (int)count, st);
}

template <class T>
T read1(const T* d, cudaStream_t st) {
    T h{};
    SMG_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

void fine_denoise(const FineParams& p, cudaStream_t st) {
    const int64_t n = p.n, nf = p.nf;
    require(n >= 0 && nf >= 0, "mesh sizes must be nonnegative");
    require(n < INT32_MAX && nf < INT32_MAX / 3, "mesh exceeds the 32-bit index range");
    auto sz = [](int64_t c) { return (size_t)std::max<int64_t>(c, 1); };
    if (nf > 0) {
        DBuf<int> bad;
        bad.alloc(1, st);
        const int big = INT32_MAX;
        SMG_CUDA(cudaMemcpyAsync(bad.get(), &big, sizeof(int), cudaMemcpyHostToDevice, st));
        ::smg::count_launch(), check_faces_kernel<<<grid_for(nf), 256, 0, st>>>(nf, p.faces, n, bad.get());
        const int b = read1(bad.get(), st);
        if (b != big) fail(2, "face " + std::to_string(b) + " references a vertex out of range");
    }
    DBuf<double4> v0, v1, ca, n0, n1;
    DBuf<int> degen, overflow;
    v0.alloc(sz(n), st);
    v1.alloc(sz(n), st);
    ca.alloc(sz(nf), st);
    n0.alloc(sz(nf), st);
    n1.alloc(sz(nf), st);
    degen.alloc(sz(nf), st);
    overflow.alloc(1, st);
    ::smg::count_launch(), to_aos_kernel<<<grid_for(n), 256, 0, st>>>(n, p.x, p.y, p.z, v0.get());
    {
        ProfScope ps("fine_geometry", st);
        ::smg::count_launch(), geom_kernel<<<grid_for(nf), 256, 0, st>>>(nf, p.faces, v0.get(), ca.get(), n0.get(),
                                                                         degen.get());
    }
    // faces of each vertex (ascending) and the face rings
    DBuf<int32_t> fcnt, foffs, ffill, flist, roffs, rcnt, ring;
    fcnt.alloc(n + 1, st);
    foffs.alloc(n + 1, st);
    ffill.alloc(n + 1, st);
    flist.alloc(sz(3 * nf), st);
    roffs.alloc(nf + 1, st);
    rcnt.alloc(nf + 1, st);
    {
        ProfScope ps("fine_rings", st);
        fcnt.zero();
        ffill.zero();
        overflow.zero();
        if (nf) ::smg::count_launch(), fov_count_kernel<<<grid_for(3 * nf), 256, 0, st>>>(nf, p.faces, fcnt.get());
        scan_i32(fcnt.get(), foffs.get(), n + 1, st);
        if (nf)
            ::smg::count_launch(), fov_fill_kernel<<<grid_for(3 * nf), 256, 0, st>>>(nf, p.faces, foffs.get(),
                                                                                    ffill.get(), flist.get());
        ::smg::count_launch(), sort_rows_kernel<<<grid_for(n), 256, 0, st>>>(n, foffs.get(), flist.get());
        for (int d = 0; d < p.ring_depth; ++d) {
            const bool first = d == 0;
            const int32_t* ido = first ? nullptr : roffs.get();
            const int32_t* ids = first ? nullptr : ring.get();
            const int32_t* so = first ? foffs.get() : roffs.get();
            const int32_t* sl = first ? flist.get() : ring.get();
            const int32_t* fc = first ? p.faces : nullptr;
            SMG_CUDA(cudaMemsetAsync(rcnt.get() + nf, 0, sizeof(int32_t), st));
            auto launch_union = [&](const int32_t* oo, int32_t* o, int32_t* cnt) {
                if (first)
                    ::smg::count_launch(), ring_union_kernel<3><<<grid_for(nf, 128), 128, 0, st>>>(
                        nf, ido, ids, fc, so, sl, oo, o, cnt, overflow.get());
                else
                    ::smg::count_launch(), ring_union_kernel<kMaxUnion><<<grid_for(nf, 128), 128, 0, st>>>(
                        nf, ido, ids, fc, so, sl, oo, o, cnt, overflow.get());
            };
            launch_union(nullptr, nullptr, rcnt.get());
            DBuf<int32_t> noffs, nring;
            noffs.alloc(nf + 1, st);
            scan_i32(rcnt.get(), noffs.get(), nf + 1, st);
            const int32_t total = read1(noffs.get() + nf, st);
            if (read1(overflow.get(), st)) fail(3, "face ring exceeds the GPU limit of 128 merged lists");
            nring.alloc(sz(total), st);
            launch_union(noffs.get(), nring.get(), nullptr);
            roffs = std::move(noffs);
            ring = std::move(nring);
        }
    }
    // sigma_spatial: given, or the mean adjacent-centroid distance (deterministic reduction)
    DBuf<double> sigma, tot;
    DBuf<int64_t> totc;
    sigma.alloc(1, st);
    tot.alloc(1, st);
    totc.alloc(1, st);
    if (p.sigma_spatial > 0.0) {
        ::smg::count_launch(), sigma_final_kernel<<<1, 32, 0, st>>>(tot.get(), totc.get(), sigma.get(), p.sigma_spatial);
    } else {
        ProfScope ps("fine_sigma", st);
        DBuf<double> fsum;
        DBuf<int32_t> fc;
        fsum.alloc(sz(nf), st);
        fc.alloc(sz(nf), st);
        if (nf)
            ::smg::count_launch(), sigma_partial_kernel<<<grid_for(nf), 256, 0, st>>>(nf, roffs.get(), ring.get(),
                                                                                      ca.get(), fsum.get(), fc.get());
        size_t b1 = 0, b2 = 0;
        cub::DeviceReduce::Sum(nullptr, b1, fsum.get(), tot.get(), (int)nf, st);
        cub::DeviceReduce::Sum(nullptr, b2, fc.get(), totc.get(), (int)nf, st);
        DBuf<char> tmp;
        tmp.alloc(std::max<size_t>(std::max(b1, b2), 1), st);
        cub::DeviceReduce::Sum(tmp.get(), b1, fsum.get(), tot.get(), (int)nf, st);
        cub::DeviceReduce::Sum(tmp.get(), b2, fc.get(), totc.get(), (int)nf, st);
        if (nf == 0 || read1(totc.get(), st) <= 0) fail(2, "mesh has no adjacent face pairs");
        ::smg::count_launch(), sigma_final_kernel<<<1, 32, 0, st>>>(tot.get(), totc.get(), sigma.get(), 0.0);
    }
    double4 *na = n0.get(), *nb = n1.get();
    {
        ProfScope ps("fine_normals", st);
        for (int it = 0; it < p.normal_iterations; ++it) {
            ::smg::count_launch(), bilateral_kernel<<<grid_for(nf), 256, 0, st>>>(
                nf, roffs.get(), ring.get(), ca.get(), na, nb, degen.get(), sigma.get(), p.sigma_range);
            std::swap(na, nb);
        }
    }
    if (p.normals_out) ::smg::count_launch(), to_soa_kernel<<<grid_for(nf), 256, 0, st>>>(nf, na, p.normals_out);
    double4 *va = v0.get(), *vb = v1.get();
    {
        ProfScope ps("fine_vertices", st);
        for (int it = 0; it < p.vertex_iterations; ++it) {
            ::smg::count_launch(), centroid_kernel<<<grid_for(nf), 256, 0, st>>>(nf, p.faces, va, ca.get());
            ::smg::count_launch(), vertex_update_kernel<<<grid_for(n), 256, 0, st>>>(n, foffs.get(), flist.get(), na,
                                                                                    ca.get(), va, vb);
            std::swap(va, vb);
        }
    }
    ::smg::count_launch(), to_soa_kernel<<<grid_for(n), 256, 0, st>>>(n, va, p.out);
    SMG_CUDA(cudaGetLastError());
}

}  // namespace smg

// TEST INFRASTRUCTURE ONLY.  C entry points over the reference's OWN headers
// (compiled unmodified from /root/reference/proj/include, never copied into this
// repository) with oracle/eigen_shim standing in for the absent Eigen dependency
// (see oracle/eigen_shim/Eigen/mini_eigen.hpp for what that does and does not pin).
// Built by `make refharness` into oracle/_ref/libspecmesh_ref.so (git-ignored);
// used by tests/golden/make_ref_fixtures.py to generate the committed golden
// vectors and, when present, by the CPU tests to check the numpy oracle directly.
#include "specmesh/compress.hpp"
#include "specmesh/denoise.hpp"
#include "specmesh/pipeline.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

using namespace specmesh;

namespace {

thread_local std::string g_error;

struct RefMesh {
    Mesh mesh;
    EdgeSet edges;
};

struct RefSeg {
    Segmentation seg;
};

struct RefBases {
    BlockBases bb;
};

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_error.clear();
        return 0;
    } catch (const InvalidArgument& e) {
        g_error = e.what();
        return 2;
    } catch (const ParseError& e) {
        g_error = e.what();
        return 4;
    } catch (const Error& e) {
        g_error = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_error = std::string("unexpected: ") + e.what();
        return 1;
    }
}

Eigen::MatrixXd from_colmajor(const double* p, int rows, int cols) {
    Eigen::MatrixXd m(rows, cols);
    std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(rows) * cols);
    return m;
}

void to_colmajor(const Eigen::Mat<double>& m, double* out) {
    std::memcpy(out, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
}

}  // namespace

extern "C" {

// mirrors specmesh::PipelineConfig (pipeline.hpp:41-68) field for field
struct ref_config {
    int part_count;
    double growth;
    int basis_mode;  // 0 OI, 1 DOI, 2 SVD
    int weighting;   // 0 Binary, 1 InverseSquaredDistance
    int subspace_size;
    double eps_low, eps_high;
    int c_min, c_max, power, iterations, initial_iterations, doi_iterations;
    unsigned long long seed;
    int dense_limit;
    double shift_scale;
    unsigned threads;
};

const char* ref_last_error() { return g_error.c_str(); }

void ref_default_config(ref_config* out) {
    const PipelineConfig c;
    out->part_count = c.part_count;
    out->growth = c.growth;
    out->basis_mode = static_cast<int>(c.basis_mode);
    out->weighting = c.weighting == Weighting::Binary ? 0 : 1;
    out->subspace_size = c.subspace_size;
    out->eps_low = c.eps_low;
    out->eps_high = c.eps_high;
    out->c_min = c.c_min;
    out->c_max = c.c_max;
    out->power = c.power;
    out->iterations = c.iterations;
    out->initial_iterations = c.initial_iterations;
    out->doi_iterations = c.doi_iterations;
    out->seed = c.seed;
    out->dense_limit = c.dense_limit;
    out->shift_scale = c.shift_scale;
    out->threads = c.threads;
}

static PipelineConfig to_cfg(const ref_config* c) {
    PipelineConfig cfg;
    cfg.part_count = c->part_count;
    cfg.growth = c->growth;
    cfg.basis_mode = static_cast<BasisMode>(c->basis_mode);
    cfg.weighting = c->weighting == 0 ? Weighting::Binary : Weighting::InverseSquaredDistance;
    cfg.subspace_size = c->subspace_size;
    cfg.eps_low = c->eps_low;
    cfg.eps_high = c->eps_high;
    cfg.c_min = c->c_min;
    cfg.c_max = c->c_max;
    cfg.power = c->power;
    cfg.iterations = c->iterations;
    cfg.initial_iterations = c->initial_iterations;
    cfg.doi_iterations = c->doi_iterations;
    cfg.seed = c->seed;
    cfg.dense_limit = c->dense_limit;
    cfg.shift_scale = c->shift_scale;
    cfg.threads = c->threads;
    return cfg;
}

// ---- mesh + edges (mesh.hpp:18-70); vertices and faces row-major n x 3
int ref_mesh_create(int n, const double* xyz, int nf, const int* faces, void** out) {
    return guarded([&] {
        auto m = std::make_unique<RefMesh>();
        m->mesh.vertices.resize(n, 3);
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) m->mesh.vertices(i, a) = xyz[3 * i + a];
        m->mesh.faces.resize(nf, 3);
        for (int f = 0; f < nf; ++f)
            for (int a = 0; a < 3; ++a) m->mesh.faces(f, a) = faces[3 * f + a];
        m->mesh.validate();
        m->edges = build_edges(m->mesh);
        *out = m.release();
    });
}
void ref_mesh_destroy(void* m) { delete static_cast<RefMesh*>(m); }
long long ref_mesh_edge_entries(void* m) {
    long long t = 0;
    for (const auto& l : static_cast<RefMesh*>(m)->edges.neighbors) t += static_cast<long long>(l.size());
    return t;
}
void ref_mesh_edges_csr(void* m, long long* offsets, int* cols) {
    const auto& nb = static_cast<RefMesh*>(m)->edges.neighbors;
    long long at = 0;
    for (std::size_t v = 0; v < nb.size(); ++v) {
        offsets[v] = at;
        for (int w : nb[v]) cols[at++] = w;
    }
    offsets[nb.size()] = at;
}

// ---- segmentation: the reference's own segment_mesh (pipeline.hpp:131-138), or
// an external one built with detail::build_submesh (partition.hpp:169-197)
int ref_segment_mesh(void* mesh, const ref_config* cfg, void** out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        auto s = std::make_unique<RefSeg>();
        s->seg = segment_mesh(m->mesh, m->edges, to_cfg(cfg));
        *out = s.release();
    });
}
int ref_segmentation_from_members(void* mesh, int count, const long long* offsets, const int* members,
                                  const int* sequence, void** out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        auto s = std::make_unique<RefSeg>();
        for (int id = 0; id < count; ++id) {
            std::vector<int> mem(members + offsets[id], members + offsets[id + 1]);
            s->seg.submeshes.push_back(detail::build_submesh(m->mesh, m->edges, std::move(mem)));
        }
        s->seg.order.sequence.assign(sequence, sequence + count);
        *out = s.release();
    });
}
void ref_seg_destroy(void* s) { delete static_cast<RefSeg*>(s); }
int ref_seg_count(void* s) { return static_cast<int>(static_cast<RefSeg*>(s)->seg.submeshes.size()); }
int ref_seg_part_count(void* s) { return static_cast<RefSeg*>(s)->seg.partition.part_count; }
void ref_seg_assignment(void* s, int* out) {
    const auto& a = static_cast<RefSeg*>(s)->seg.partition.assignment;
    for (Eigen::Index i = 0; i < a.size(); ++i) out[i] = a(i);
}
int ref_seg_size(void* s, int id) { return static_cast<RefSeg*>(s)->seg.submeshes[id].size(); }
void ref_seg_members(void* s, int id, int* out) {
    const auto& g = static_cast<RefSeg*>(s)->seg.submeshes[id].global_indices;
    std::copy(g.begin(), g.end(), out);
}
void ref_seg_order(void* s, int* out) {
    const auto& q = static_cast<RefSeg*>(s)->seg.order.sequence;
    std::copy(q.begin(), q.end(), out);
}
long long ref_seg_adjacency_entries(void* s, int id) {
    long long t = 0;
    for (const auto& l : static_cast<RefSeg*>(s)->seg.submeshes[id].local_adjacency) t += static_cast<long long>(l.size());
    return t;
}

// ---- Laplacian (spectral.hpp:39-68) as CSR (= CSC of the symmetric matrix), trace, shift
int ref_laplacian(void* mesh, void* seg, int id, int weighting, double shift_scale, int* offsets, int* cols,
                  double* vals, double* trace, double* delta) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Submesh& sub = static_cast<RefSeg*>(seg)->seg.submeshes[id];
        const Laplacian lap = build_laplacian(sub, m->mesh.vertices,
                                              weighting == 0 ? Weighting::Binary : Weighting::InverseSquaredDistance);
        const int n = static_cast<int>(lap.size());
        std::copy(lap.matrix.outerIndexPtr(), lap.matrix.outerIndexPtr() + n + 1, offsets);
        std::copy(lap.matrix.innerIndexPtr(), lap.matrix.innerIndexPtr() + lap.matrix.nonZeros(), cols);
        std::copy(lap.matrix.valuePtr(), lap.matrix.valuePtr() + lap.matrix.nonZeros(), vals);
        *trace = lap.trace();
        *delta = default_shift(lap, shift_scale);
    });
}
long long ref_laplacian_nnz(void* seg, int id) {
    const Submesh& sub = static_cast<RefSeg*>(seg)->seg.submeshes[id];
    return ref_seg_adjacency_entries(seg, id) + sub.size();
}

// ---- primitives; matrices column-major
int ref_orthonormalize(int rows, int cols, const double* in, double* out) {
    return guarded([&] { to_colmajor(orthonormalize(from_colmajor(in, rows, cols)), out); });
}
int ref_apply(void* mesh, void* seg, int id, int weighting, double shift_scale, int z, int cols, const double* in,
              double* out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Submesh& sub = static_cast<RefSeg*>(seg)->seg.submeshes[id];
        const Laplacian lap = build_laplacian(sub, m->mesh.vertices,
                                              weighting == 0 ? Weighting::Binary : Weighting::InverseSquaredDistance);
        const ShiftedInverseOperator op(lap, default_shift(lap, shift_scale), z);
        to_colmajor(op.apply(from_colmajor(in, sub.size(), cols)), out);
    });
}
int ref_bottom_subspace(void* mesh, void* seg, int id, int weighting, int c, double* eigenvalues, double* basis) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Submesh& sub = static_cast<RefSeg*>(seg)->seg.submeshes[id];
        const Laplacian lap = build_laplacian(sub, m->mesh.vertices,
                                              weighting == 0 ? Weighting::Binary : Weighting::InverseSquaredDistance);
        const Spectrum sp = dense_eigendecomposition(lap);
        for (Eigen::Index i = 0; i < sp.eigenvalues.size(); ++i) eigenvalues[i] = sp.eigenvalues(i);
        to_colmajor(bottom_subspace(sp, c).vectors, basis);
    });
}
// orthogonal_iteration (spectral.hpp:204-211) from a given basis
int ref_orthogonal_iteration(void* mesh, void* seg, int id, int weighting, double shift_scale, int z, int c,
                             const double* init, int t_max, double* out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Submesh& sub = static_cast<RefSeg*>(seg)->seg.submeshes[id];
        const Laplacian lap = build_laplacian(sub, m->mesh.vertices,
                                              weighting == 0 ? Weighting::Binary : Weighting::InverseSquaredDistance);
        const ShiftedInverseOperator op(lap, default_shift(lap, shift_scale), z);
        const SpectralBasis res = orthogonal_iteration(op, SpectralBasis{from_colmajor(init, sub.size(), c)}, t_max);
        to_colmajor(res.vectors, out);
    });
}
// dynamic_oi (spectral.hpp:244-287); out_basis holds n_d x c_max doubles
int ref_dynamic_oi(void* mesh, void* seg, int id, int weighting, double shift_scale, int z, int c, const double* init,
                   double eps_low, double eps_high, int c_min, int c_max, int t_max, double* out_basis, int* out_c,
                   int* out_iterations, int* out_converged, double* out_residual) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Submesh& sub = static_cast<RefSeg*>(seg)->seg.submeshes[id];
        const Laplacian lap = build_laplacian(sub, m->mesh.vertices,
                                              weighting == 0 ? Weighting::Binary : Weighting::InverseSquaredDistance);
        const ShiftedInverseOperator op(lap, default_shift(lap, shift_scale), z);
        const DoiResult r = dynamic_oi(op, SpectralBasis{from_colmajor(init, sub.size(), c)},
                                       sub.local_coords(m->mesh.vertices), eps_low, eps_high, c_min, c_max, t_max);
        to_colmajor(r.basis.vectors, out_basis);
        *out_c = r.basis.subspace_size();
        *out_iterations = r.iterations;
        *out_converged = r.converged ? 1 : 0;
        *out_residual = r.residual;
    });
}
int ref_max_principal_angle(int rows, int cols, const double* a, const double* b, double* out) {
    return guarded([&] { *out = max_principal_angle(from_colmajor(a, rows, cols), from_colmajor(b, rows, cols)); });
}
int ref_resize_basis(int rows, int cols, const double* in, int new_size, unsigned long long seed, double* out) {
    return guarded([&] {
        to_colmajor(resize_basis(SpectralBasis{from_colmajor(in, rows, cols)}, new_size, seed).vectors, out);
    });
}

// ---- chains (pipeline.hpp:144-194 with an external segmentation; :198-285 whole entry)
int ref_chain_fixed(void* mesh, void* seg, const ref_config* cfg, const int* sizes_in_order, void** out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Segmentation& s = static_cast<RefSeg*>(seg)->seg;
        std::vector<int> sizes(sizes_in_order, sizes_in_order + s.order.sequence.size());
        auto b = std::make_unique<RefBases>();
        b->bb = compute_block_bases_fixed_sizes(m->mesh, m->edges, to_cfg(cfg), s, sizes);
        *out = b.release();
    });
}
int ref_chain(void* mesh, const ref_config* cfg, void** out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        auto b = std::make_unique<RefBases>();
        b->bb = compute_block_bases(m->mesh, m->edges, to_cfg(cfg));
        *out = b.release();
    });
}
// The DOI chain over an EXTERNAL segmentation (the reference's DOI branch always
// segments internally, pipeline.hpp:201, but C4 prescribes its 64x64 tiles).  The
// loop below restates pipeline.hpp:245-285 around the reference's own functions
// (build_laplacian, ShiftedInverseOperator, initial_block_basis, resize_basis,
// dynamic_oi, projection_residual_rms), which do all the work.
int ref_chain_doi_external(void* mesh, void* seg, const ref_config* c, void** out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const PipelineConfig cfg = to_cfg(c);
        auto b = std::make_unique<RefBases>();
        BlockBases& result = b->bb;
        result.submeshes = static_cast<RefSeg*>(seg)->seg.submeshes;
        result.order = static_cast<RefSeg*>(seg)->seg.order;
        const int k = static_cast<int>(result.submeshes.size());
        result.bases.resize(k);
        result.stats.resize(k);
        result.block_size = result.submeshes.empty() ? 0 : result.submeshes.front().size();
        SpectralBasis previous;
        for (std::size_t pos = 0; pos < result.order.sequence.size(); ++pos) {
            const int id = result.order.sequence[pos];
            const Submesh& sub = result.submeshes[id];
            const int c_max = cfg.resolve_c_max(sub.size());
            const int doi_t_max = cfg.resolve_doi_iterations(c_max);
            const Laplacian laplacian = build_laplacian(sub, m->mesh.vertices, cfg.weighting);
            const ShiftedInverseOperator op(laplacian, default_shift(laplacian, cfg.shift_scale), cfg.power);
            SpectralBasis init;
            if (pos == 0) {
                init = detail::initial_block_basis(laplacian, op, std::clamp(cfg.subspace_size, cfg.c_min, c_max), cfg);
            } else {
                init = resize_basis(previous, std::clamp(previous.subspace_size(), cfg.c_min, c_max),
                                    cfg.seed + 0x5851f42d4c957f2dULL * pos);
            }
            DoiResult doi = dynamic_oi(op, init, sub.local_coords(m->mesh.vertices), cfg.eps_low, cfg.eps_high,
                                       cfg.c_min, c_max, doi_t_max);
            result.stats[id].subspace_size = doi.basis.subspace_size();
            result.stats[id].doi_residual = doi.residual;
            result.stats[id].converged = doi.converged;
            result.stats[id].oi_iterations = doi.iterations;
            result.stats[id].residual_rms = projection_residual_rms(doi.basis, sub.local_coords(m->mesh.vertices));
            previous = doi.basis;
            result.bases[id] = std::move(doi.basis);
            if (std::getenv("REF_PROGRESS"))
                std::fprintf(stderr, "tile %d c=%d t=%d conv=%d r=%.6e\n", id, result.stats[id].subspace_size,
                             doi.iterations, int(doi.converged), doi.residual);
        }
        *out = b.release();
    });
}
void ref_bases_destroy(void* b) { delete static_cast<RefBases*>(b); }
int ref_bases_count(void* b) { return static_cast<int>(static_cast<RefBases*>(b)->bb.submeshes.size()); }
int ref_bases_block_size(void* b) { return static_cast<RefBases*>(b)->bb.block_size; }
int ref_bases_size(void* b, int id) { return static_cast<RefBases*>(b)->bb.submeshes[id].size(); }
void ref_bases_members(void* b, int id, int* out) {
    const auto& g = static_cast<RefBases*>(b)->bb.submeshes[id].global_indices;
    std::copy(g.begin(), g.end(), out);
}
void ref_bases_order(void* b, int* out) {
    const auto& q = static_cast<RefBases*>(b)->bb.order.sequence;
    std::copy(q.begin(), q.end(), out);
}
int ref_bases_c(void* b, int id) { return static_cast<RefBases*>(b)->bb.bases[id].subspace_size(); }
void ref_bases_basis(void* b, int id, double* out) { to_colmajor(static_cast<RefBases*>(b)->bb.bases[id].vectors, out); }
// stats: subspace_size, residual_rms, doi_residual, converged, oi_iterations
void ref_bases_stats(void* b, int id, double* out) {
    const BlockStats& s = static_cast<RefBases*>(b)->bb.stats[id];
    out[0] = s.subspace_size;
    out[1] = s.residual_rms;
    out[2] = s.doi_residual;
    out[3] = s.converged ? 1.0 : 0.0;
    out[4] = s.oi_iterations;
}
// gft coefficients of block id (c x 3, column-major) -- spectral.hpp:290-293
int ref_bases_coefficients(void* b, void* mesh, int id, double* out) {
    return guarded([&] {
        const BlockBases& bb = static_cast<RefBases*>(b)->bb;
        auto* m = static_cast<RefMesh*>(mesh);
        to_colmajor(gft(bb.bases[id], bb.submeshes[id].local_coords(m->mesh.vertices)), out);
    });
}
// coarse_reconstruct_points (pipeline.hpp:300-305); out row-major n x 3
int ref_bases_reconstruct(void* b, void* mesh, int weighted, double* out) {
    return guarded([&] {
        auto* m = static_cast<RefMesh*>(mesh);
        const Points p = coarse_reconstruct_points(m->mesh, static_cast<RefBases*>(b)->bb,
                                                   weighted ? AverageMode::Weighted : AverageMode::Simple);
        for (Eigen::Index i = 0; i < p.rows(); ++i)
            for (int a = 0; a < 3; ++a) out[3 * i + a] = p(i, a);
    });
}
double ref_bases_timing(void* b, const char* stage) { return static_cast<RefBases*>(b)->bb.timings.get(stage); }


// ---- F2: the spectral codec (compress.hpp:152-219, :378-474): SPECMSH1 bytes
int ref_compress(void* mesh, const ref_config* cfg, int quant_bits, unsigned char* out, long long cap,
                 long long* out_len) {
    return guarded([&] {
        CompressionConfig cc;
        cc.pipeline = to_cfg(cfg);
        cc.quant_bits = quant_bits;
        const std::vector<std::uint8_t> bytes =
            serialize_encoded_mesh(compress_mesh(static_cast<RefMesh*>(mesh)->mesh, cc));
        *out_len = static_cast<long long>(bytes.size());
        if (static_cast<long long>(bytes.size()) <= cap) std::copy(bytes.begin(), bytes.end(), out);
    });
}
// decompress_mesh(parse_encoded_mesh(bytes)) -> vertices row-major n x 3
int ref_decompress(const unsigned char* bytes, long long len, double* out, int n_expected) {
    return guarded([&] {
        const Mesh m = decompress_mesh(parse_encoded_mesh(std::vector<std::uint8_t>(bytes, bytes + len)));
        require(m.vertex_count() == n_expected, "vertex count mismatch");
        for (Eigen::Index i = 0; i < m.vertices.rows(); ++i)
            for (int a = 0; a < 3; ++a) out[3 * i + a] = m.vertices(i, a);
    });
}

// ---- F4: fine_denoise (denoise.hpp:175-180); out row-major n x 3, normals nf x 3
int ref_fine_denoise(void* mesh, double sigma_spatial, double sigma_range, int normal_iterations,
                     int vertex_iterations, int ring_depth, double* out, double* out_normals) {
    return guarded([&] {
        const Mesh& m = static_cast<RefMesh*>(mesh)->mesh;
        BilateralParams p;
        p.sigma_spatial = sigma_spatial;
        p.sigma_range = sigma_range;
        p.normal_iterations = normal_iterations;
        p.vertex_iterations = vertex_iterations;
        p.ring_depth = ring_depth;
        p.validate();
        const Mesh r = fine_denoise(m, p);
        for (Eigen::Index i = 0; i < r.vertices.rows(); ++i)
            for (int a = 0; a < 3; ++a) out[3 * i + a] = r.vertices(i, a);
        if (out_normals) {
            const Points nrm = bilateral_normals(face_geometry(m), face_ring_adjacency(m, p.ring_depth), p);
            for (Eigen::Index f = 0; f < nrm.rows(); ++f)
                for (int a = 0; a < 3; ++a) out_normals[3 * f + a] = nrm(f, a);
        }
    });
}

// ---- F3: denoise_dynamic (denoise.hpp:258-291); frames row-major F x n x 3 sharing the mesh's faces
int ref_denoise_dynamic(void* mesh, int frames, const double* xyz, const ref_config* cfg, int weighted, double* out,
                        int* blocks_computed) {
    return guarded([&] {
        const Mesh& first = static_cast<RefMesh*>(mesh)->mesh;
        const int n = static_cast<int>(first.vertex_count());
        std::vector<Mesh> seq(static_cast<std::size_t>(frames));
        for (int f = 0; f < frames; ++f) {
            seq[f].faces = first.faces;
            seq[f].vertices.resize(n, 3);
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 3; ++a) seq[f].vertices(i, a) = xyz[(static_cast<std::size_t>(f) * n + i) * 3 + a];
        }
        const DynamicDenoiseResult r =
            denoise_dynamic(seq, to_cfg(cfg), weighted ? AverageMode::Weighted : AverageMode::Simple);
        for (int f = 0; f < frames; ++f)
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 3; ++a) out[(static_cast<std::size_t>(f) * n + i) * 3 + a] = r.frames[f].vertices(i, a);
        *blocks_computed = r.basis_blocks_computed;
    });
}

}  // extern "C"

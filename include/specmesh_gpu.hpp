// specmesh_gpu.hpp -- C++ adapter over the C ABI (specmesh_gpu.h).
//
// Two layers:
//   1. specmesh_gpu:: -- std::vector typed C++ (no Eigen): RAII context,
//      exceptions carrying the reference's message texts, and the chain calls
//      with the reference's argument meaning (pipeline.hpp:144-201).  Compiled
//      and exercised by tests/cpp/abi_chain.cpp.
//   2. specmesh_gpu::ref:: (only when the reference headers are visible, i.e.
//      <specmesh/pipeline.hpp> and Eigen are on the include path) -- the exact
//      reference signature
//          BlockBases compute_block_bases_fixed_sizes(const Mesh&, const EdgeSet&,
//              const PipelineConfig&, Segmentation, const std::vector<int>&)
//      (pipeline.hpp:144-147), so a caller (compress_mesh compress.hpp:171-174,
//      decompress_mesh :228-230, coarse_denoise denoise.hpp:194-195) switches by
//      changing the namespace of one call.  Eigen is absent from this image and
//      the GPU box (profiles/eigen_probe_r02.txt), so this layer is compiled only
//      where the reference builds.
#ifndef SPECMESH_GPU_HPP
#define SPECMESH_GPU_HPP

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "specmesh_gpu.h"

namespace specmesh_gpu {

// core.hpp:18-34: Error / InvalidArgument / ParseError, same what() texts
struct Error : std::runtime_error {
    int status;
    Error(const std::string& m, int s = SMG_ERROR) : std::runtime_error(m), status(s) {}
};
struct InvalidArgument : Error {
    explicit InvalidArgument(const std::string& m) : Error(m, SMG_INVALID_ARGUMENT) {}
};
struct ParseError : Error {
    explicit ParseError(const std::string& m) : Error(m, SMG_PARSE_ERROR) {}
};

inline void check(smg_context* ctx, smg_status st) {
    if (st == SMG_OK) return;
    const std::string m = smg_last_error(ctx);
    if (st == SMG_INVALID_ARGUMENT) throw InvalidArgument(m);
    if (st == SMG_PARSE_ERROR) throw ParseError(m);
    throw Error(m, st);
}

// One device + stream (smg_create); move-only.
class Context {
public:
    explicit Context(int device = 0) {
        const smg_status st = smg_create(device, &h_);
        if (st != SMG_OK) throw Error("smg_create failed on device " + std::to_string(device) + ": no usable sm_100 GPU", st);
    }
    Context(Context&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Context& operator=(Context&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ~Context() {
        if (h_) smg_destroy(h_);
    }
    smg_context* get() const { return h_; }

private:
    smg_context* h_ = nullptr;
};

// Mesh (mesh.hpp:18-37) + EdgeSet (mesh.hpp:40-50) as host arrays: vertices
// column-major n x 3 (Eigen's MatrixX3d storage), neighbour lists as CSR.
struct Mesh {
    std::vector<double> vertices;  // x[0..n) | y[0..n) | z[0..n)
    std::vector<int32_t> adj_offsets, adj_cols;
    int64_t vertex_count() const { return (int64_t)vertices.size() / 3; }
};

// Segmentation (pipeline.hpp:125-129): sorted member lists + visiting order.
struct Segmentation {
    std::vector<std::vector<int32_t>> submeshes;
    std::vector<int32_t> sequence;
};

// BlockStats (pipeline.hpp:70-76)
struct BlockStats {
    int subspace_size = 0;
    double residual_rms = 0.0, doi_residual = 0.0;
    bool converged = true;
    int oi_iterations = 0;
};

// BlockBases (pipeline.hpp:78-92) + project_blocks' coefficients and
// coarse_reconstruct_points' result (pipeline.hpp:290-305), indexed by id.
struct BlockBases {
    int block_size = 0;
    std::vector<std::vector<double>> bases;         // n_d x c_id column-major (if requested)
    std::vector<std::vector<double>> coefficients;  // c_id x 3 column-major (gft)
    std::vector<BlockStats> stats;
    std::vector<double> reconstruction;             // n x 3 column-major (Weighted)
    double timings[6] = {0, 0, 0, 0, 0, 0};         // laplacian factorize basis basis_total project total
};

inline smg_pipeline_config default_config() {
    smg_pipeline_config c;
    smg_default_config(&c);
    return c;
}

namespace detail {
struct Views {
    std::vector<int32_t> moffs, members;
    smg_mesh mesh{};
    smg_segmentation seg{};
};
inline void make_views(const Mesh& m, const Segmentation& s, Views& v) {
    const int64_t n = m.vertex_count();
    v.mesh = smg_mesh{n, m.vertices.data(), m.vertices.data() + n, m.vertices.data() + 2 * n,
                      m.adj_offsets.data(), m.adj_cols.data(), 0};
    v.moffs.assign(1, 0);
    v.members.clear();
    for (const auto& sub : s.submeshes) {
        v.members.insert(v.members.end(), sub.begin(), sub.end());
        v.moffs.push_back((int32_t)v.members.size());
    }
    v.seg = smg_segmentation{(int32_t)s.submeshes.size(), v.moffs.data(), v.members.data(),
                             (int32_t)s.sequence.size(), s.sequence.data(), 0};
}
struct Out {
    std::vector<int32_t> ss, conv, its;
    std::vector<double> rms, doi, coef, bases, recon;
    std::vector<int64_t> coff, boff;
    smg_chain_output o{};
    void init(int k, int n_d, int64_t n, int c_cap, bool want_bases) {
        ss.assign(k, 0);
        conv.assign(k, 0);
        its.assign(k, 0);
        rms.assign(k, 0.0);
        doi.assign(k, 0.0);
        coef.assign((size_t)k * c_cap * 3, 0.0);
        coff.assign(k + 1, 0);
        recon.assign((size_t)n * 3, 0.0);
        o = smg_chain_output{};
        o.subspace_size = ss.data();
        o.residual_rms = rms.data();
        o.doi_residual = doi.data();
        o.converged = conv.data();
        o.oi_iterations = its.data();
        o.reconstruction = recon.data();
        o.coefficients = coef.data();
        o.coefficients_capacity = (int64_t)coef.size();
        o.coefficient_offsets = coff.data();
        if (want_bases) {
            bases.assign((size_t)k * n_d * c_cap, 0.0);
            boff.assign(k + 1, 0);
            o.bases = bases.data();
            o.bases_capacity = (int64_t)bases.size();
            o.basis_offsets = boff.data();
        }
    }
    BlockBases result(int k, int n_d) {
        BlockBases r;
        r.block_size = n_d;
        r.stats.resize(k);
        r.coefficients.resize(k);
        if (o.bases) r.bases.resize(k);
        for (int id = 0; id < k; ++id) {
            r.stats[id] = BlockStats{ss[id], rms[id], doi[id], conv[id] != 0, its[id]};
            r.coefficients[id].assign(coef.begin() + coff[id], coef.begin() + coff[id + 1]);
            if (o.bases) r.bases[id].assign(bases.begin() + boff[id], bases.begin() + boff[id + 1]);
        }
        r.reconstruction = std::move(recon);
        std::copy(o.timings, o.timings + 6, r.timings);
        return r;
    }
};
inline int block_size_of(const Segmentation& s) {
    if (s.submeshes.empty()) throw InvalidArgument("cannot process an empty submesh list");
    return (int)s.submeshes.front().size();
}
}  // namespace detail

// compute_block_bases_fixed_sizes (pipeline.hpp:144-194) + project_blocks +
// coarse_reconstruct_points (Weighted)
inline BlockBases compute_block_bases_fixed_sizes(Context& ctx, const Mesh& mesh, const smg_pipeline_config& cfg,
                                                  const Segmentation& seg, const std::vector<int>& sizes_in_order,
                                                  bool want_bases = false) {
    detail::Views v;
    detail::make_views(mesh, seg, v);
    const int k = (int)seg.submeshes.size(), n_d = detail::block_size_of(seg);
    const int c_cap = sizes_in_order.empty() ? 1 : *std::max_element(sizes_in_order.begin(), sizes_in_order.end());
    detail::Out out;
    out.init(k, n_d, mesh.vertex_count(), std::max(c_cap, 1), want_bases);
    std::vector<int32_t> sizes(sizes_in_order.begin(), sizes_in_order.end());
    check(ctx.get(), smg_compute_block_bases_fixed_sizes(ctx.get(), &v.mesh, &v.seg, &cfg, sizes.data(), &out.o));
    return out.result(k, n_d);
}

// compute_block_bases (pipeline.hpp:198-287), OI or DOI by cfg.basis_mode, over
// an external Segmentation (the reference segments internally at :201)
inline BlockBases compute_block_bases(Context& ctx, const Mesh& mesh, const smg_pipeline_config& cfg,
                                      const Segmentation& seg, bool want_bases = false) {
    detail::Views v;
    detail::make_views(mesh, seg, v);
    const int k = (int)seg.submeshes.size(), n_d = detail::block_size_of(seg);
    int c_cap = cfg.subspace_size;
    if (cfg.basis_mode == SMG_BASIS_DOI) c_cap = std::min(cfg.c_max > 0 ? cfg.c_max : std::max(64, 2 * cfg.subspace_size), n_d);
    detail::Out out;
    out.init(k, n_d, mesh.vertex_count(), std::max(c_cap, 1), want_bases);
    check(ctx.get(), smg_compute_block_bases(ctx.get(), &v.mesh, &v.seg, &cfg, &out.o));
    return out.result(k, n_d);
}

// segment_mesh (pipeline.hpp:131-138) on the GPU: sorted member lists of
// n_d vertices per submesh id + the SubmeshOrder sequence (assignment optional)
inline Segmentation segment_mesh(Context& ctx, const Mesh& mesh, int part_count, double growth, uint64_t seed,
                                 std::vector<int32_t>* assignment = nullptr) {
    detail::Views v;
    detail::make_views(mesh, Segmentation{{std::vector<int32_t>(1, 0)}, {0}}, v);
    int32_t nd = 0;
    std::vector<int32_t> seq(std::max(part_count, 1));
    // first call sizes the member buffer (InvalidArgument "members capacity too small" with n_d set)
    const smg_status st0 = smg_segment_mesh(ctx.get(), &v.mesh, part_count, growth, seed, nullptr, nullptr, 0, &nd,
                                            seq.data());
    if (nd <= 0) check(ctx.get(), st0);
    std::vector<int32_t> mem((size_t)part_count * nd);
    if (assignment) assignment->resize((size_t)mesh.vertex_count());
    check(ctx.get(), smg_segment_mesh(ctx.get(), &v.mesh, part_count, growth, seed,
                                      assignment ? assignment->data() : nullptr, mem.data(), (int64_t)mem.size(), &nd,
                                      seq.data()));
    Segmentation s;
    for (int p = 0; p < part_count; ++p) s.submeshes.emplace_back(mem.begin() + (size_t)p * nd, mem.begin() + (size_t)(p + 1) * nd);
    s.sequence = std::move(seq);
    return s;
}

// compute_block_bases(mesh, edges, cfg) (pipeline.hpp:198-201): segments
// internally like the reference (cfg.part_count, cfg.growth, cfg.seed)
inline BlockBases compute_block_bases(Context& ctx, const Mesh& mesh, const smg_pipeline_config& cfg) {
    return compute_block_bases(ctx, mesh, cfg, segment_mesh(ctx, mesh, cfg.part_count, cfg.growth, cfg.seed));
}

}  // namespace specmesh_gpu

// ------------------------------------------------------------------ reference-typed layer
#if defined(__has_include)
#if __has_include(<specmesh/pipeline.hpp>)
#include <specmesh/pipeline.hpp>

namespace specmesh_gpu {
namespace ref {

inline Context& thread_context() {
    thread_local Context ctx(0);
    return ctx;
}

inline smg_pipeline_config to_c(const specmesh::PipelineConfig& cfg) {
    smg_pipeline_config c = default_config();
    c.weighting = cfg.weighting == specmesh::Weighting::Binary ? SMG_WEIGHTING_BINARY : SMG_WEIGHTING_DISTANCE;
    c.basis_mode = cfg.basis_mode == specmesh::BasisMode::DOI ? SMG_BASIS_DOI : SMG_BASIS_OI;
    c.subspace_size = cfg.subspace_size;
    c.eps_low = cfg.eps_low;
    c.eps_high = cfg.eps_high;
    c.c_min = cfg.c_min;
    c.c_max = cfg.c_max;
    c.power = cfg.power;
    c.iterations = cfg.iterations;
    c.initial_iterations = cfg.initial_iterations;
    c.doi_iterations = cfg.doi_iterations;
    c.seed = cfg.seed;
    c.dense_limit = cfg.dense_limit;
    c.shift_scale = cfg.shift_scale;
    c.part_count = cfg.part_count;
    c.growth = cfg.growth;
    return c;
}

// drop-in for specmesh::compute_block_bases_fixed_sizes (pipeline.hpp:144-147)
inline specmesh::BlockBases compute_block_bases_fixed_sizes(const specmesh::Mesh& mesh, const specmesh::EdgeSet& edges,
                                                            const specmesh::PipelineConfig& cfg,
                                                            specmesh::Segmentation seg,
                                                            const std::vector<int>& sizes_in_order) {
    Mesh m;
    const auto& V = mesh.vertices;
    m.vertices.assign(V.data(), V.data() + V.size());  // column-major n x 3
    m.adj_offsets.assign(1, 0);
    for (const auto& nb : edges.neighbors) {
        m.adj_cols.insert(m.adj_cols.end(), nb.begin(), nb.end());
        m.adj_offsets.push_back((int32_t)m.adj_cols.size());
    }
    Segmentation s;
    for (const auto& sub : seg.submeshes) s.submeshes.emplace_back(sub.global_indices.begin(), sub.global_indices.end());
    s.sequence.assign(seg.order.sequence.begin(), seg.order.sequence.end());
    BlockBases b;
    try {
        b = specmesh_gpu::compute_block_bases_fixed_sizes(thread_context(), m, to_c(cfg), s, sizes_in_order, true);
    } catch (const InvalidArgument& e) {
        throw specmesh::InvalidArgument(e.what());
    } catch (const Error& e) {
        throw specmesh::Error(e.what());
    }
    specmesh::BlockBases r;
    r.submeshes = std::move(seg.submeshes);
    r.order = std::move(seg.order);
    r.block_size = b.block_size;
    const int k = (int)b.stats.size();
    r.bases.resize(k);
    r.stats.resize(k);
    for (int id = 0; id < k; ++id) {
        const auto& st = b.stats[id];
        r.bases[id].vectors = Eigen::Map<const Eigen::MatrixXd>(b.bases[id].data(), b.block_size, st.subspace_size);
        r.stats[id] = specmesh::BlockStats{st.subspace_size, st.residual_rms, st.doi_residual, st.converged,
                                           st.oi_iterations};
    }
    return r;
}

// drop-in for specmesh::segment_mesh (pipeline.hpp:131-138), on the GPU
inline specmesh::Segmentation segment_mesh(const specmesh::Mesh& mesh, const specmesh::EdgeSet& edges,
                                           const specmesh::PipelineConfig& cfg) {
    Mesh m;
    m.vertices.assign(mesh.vertices.data(), mesh.vertices.data() + mesh.vertices.size());
    m.adj_offsets.assign(1, 0);
    for (const auto& nb : edges.neighbors) {
        m.adj_cols.insert(m.adj_cols.end(), nb.begin(), nb.end());
        m.adj_offsets.push_back((int32_t)m.adj_cols.size());
    }
    std::vector<int32_t> assignment;
    Segmentation s = specmesh_gpu::segment_mesh(thread_context(), m, cfg.part_count, cfg.growth, cfg.seed, &assignment);
    specmesh::Segmentation r;
    r.partition.part_count = cfg.part_count;
    r.partition.assignment = Eigen::Map<const Eigen::VectorXi>(assignment.data(), (Eigen::Index)assignment.size());
    for (auto& mem : s.submeshes)
        r.submeshes.push_back(specmesh::detail::build_submesh(mesh, edges, std::vector<int>(mem.begin(), mem.end())));
    r.order.sequence.assign(s.sequence.begin(), s.sequence.end());
    return r;
}

}  // namespace ref
}  // namespace specmesh_gpu
#endif
#endif

#endif  // SPECMESH_GPU_HPP

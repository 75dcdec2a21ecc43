// Compiled C++ caller of the C ABI through include/specmesh_gpu.hpp (no Python):
// reads a mesh + segmentation + config written by tests/test_cpp_abi.py, runs
// smg_compute_block_bases_fixed_sizes (pipeline.hpp:144-194) or the DOI chain
// (compute_block_bases, pipeline.hpp:245-285), and writes the stats,
// coefficients and reconstruction back for comparison with the Python path.
//
// input  (little endian): i64 n, i32 nnz_adj, i32 k, i32 n_d, i32 mode (0 OI, 1 DOI),
//        i32 c, i32 t, i32 c_min, i32 c_max, f64 eps_low, f64 eps_high, f64 shift_scale,
//        f64 x[n] y[n] z[n], i32 adj_offsets[n+1], i32 adj_cols[nnz_adj],
//        i32 members[k*n_d], i32 sequence[k]
// output: i32 status, then (status 0) per id: i32 c, f64 rms, f64 doi, i32 conv, i32 its,
//         f64 coefficients[c*3]; then f64 reconstruction[3n]; else the error text.
// exit code: the smg status (0 ok, 2 InvalidArgument, 3 Error).
#include <cstdio>
#include <cstring>
#include <vector>

#include "specmesh_gpu.hpp"

namespace {
template <class T>
void rd(FILE* f, T* p, size_t n) {
    if (n && fread(p, sizeof(T), n, f) != n) throw specmesh_gpu::InvalidArgument("short input file");
}
template <class T>
void wr(FILE* f, const T* p, size_t n) {
    fwrite(p, sizeof(T), n, f);
}
}  // namespace

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
        return 2;
    }
    FILE* out = std::fopen(argv[2], "wb");
    if (!out) return 2;
    int32_t status = 0;
    try {
        FILE* in = std::fopen(argv[1], "rb");
        if (!in) throw specmesh_gpu::InvalidArgument("cannot open input");
        int64_t n;
        int32_t hdr[8];
        double eps[3];
        rd(in, &n, 1);
        rd(in, hdr, 8);
        rd(in, eps, 3);
        const int nnz = hdr[0], k = hdr[1], nd = hdr[2], mode = hdr[3], c = hdr[4], t = hdr[5];
        specmesh_gpu::Mesh mesh;
        mesh.vertices.resize(3 * n);
        mesh.adj_offsets.resize(n + 1);
        mesh.adj_cols.resize(nnz);
        rd(in, mesh.vertices.data(), 3 * n);
        rd(in, mesh.adj_offsets.data(), n + 1);
        rd(in, mesh.adj_cols.data(), nnz);
        specmesh_gpu::Segmentation seg;
        seg.submeshes.assign(k, std::vector<int32_t>(nd));
        for (auto& s : seg.submeshes) rd(in, s.data(), nd);
        seg.sequence.resize(k);
        rd(in, seg.sequence.data(), k);
        std::fclose(in);

        specmesh_gpu::Context ctx(0);
        smg_pipeline_config cfg = specmesh_gpu::default_config();
        cfg.weighting = SMG_WEIGHTING_BINARY;
        cfg.subspace_size = c;
        cfg.iterations = t;
        cfg.c_min = hdr[6];
        cfg.c_max = hdr[7];
        cfg.eps_low = eps[0];
        cfg.eps_high = eps[1];
        cfg.shift_scale = eps[2];
        specmesh_gpu::BlockBases bb;
        if (mode == 0) {
            bb = specmesh_gpu::compute_block_bases_fixed_sizes(ctx, mesh, cfg, seg, std::vector<int>(k, c));
        } else {
            cfg.basis_mode = SMG_BASIS_DOI;
            bb = specmesh_gpu::compute_block_bases(ctx, mesh, cfg, seg);
        }
        wr(out, &status, 1);
        for (int id = 0; id < k; ++id) {
            const auto& st = bb.stats[id];
            const int32_t ci = st.subspace_size, conv = st.converged, its = st.oi_iterations;
            wr(out, &ci, 1);
            wr(out, &st.residual_rms, 1);
            wr(out, &st.doi_residual, 1);
            wr(out, &conv, 1);
            wr(out, &its, 1);
            wr(out, bb.coefficients[id].data(), bb.coefficients[id].size());
        }
        wr(out, bb.reconstruction.data(), bb.reconstruction.size());
    } catch (const specmesh_gpu::Error& e) {
        status = e.status;
        wr(out, &status, 1);
        std::fputs(e.what(), out);
    }
    std::fclose(out);
    return status;
}

// Host-side launch interfaces of the sm_100a kernels (internal to the library).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace smg {

// Every kernel launch site calls this (comma-prefixed); read via the
// diagnostics API as the "launches" stage.
int count_launch();
int64_t launch_count();
// raise a kernel's dynamic shared-memory limit on the current device (cached per device)
void ensure_smem(const void* func, int bytes);

// ------------------------------------------------------------------ GEMM (gemm.cu)
struct GemmParams {
    int M = 0, N = 0, K = 0, batch = 1, splits = 1;
    const double* A = nullptr;
    int64_t lda = 0, strideA = 0;
    const double* B = nullptr;
    int64_t ldb = 0, strideB = 0;
    double* C = nullptr;  // destination (splits == 1) or split-K workspace (ld = ldc)
    int64_t ldc = 0, strideC = 0;
    int64_t strideP = 0;    // workspace stride per (batch, split)
    double* out = nullptr;  // destination when splits > 1 (batch stride strideC)
    int64_t ldo = 0;
    double alpha = 1.0, beta = 0.0;
    const int* dimM = nullptr;  // optional device-side dims (per batch, stride dimStride)
    const int* dimN = nullptr;
    const int* dimK = nullptr;
    int64_t dimStride = 0;
    int upperB = 0;     // B upper triangular (square): k < n0 + 64
    int syrkUpper = 0;  // only tiles with tile_m <= tile_n
    const int* skip = nullptr;  // optional per batch entry: nonzero -> no work (adaptive CholeskyQR2)
    // optional projection partials in the epilogue of a plain (unsplit) product
    // C = A B whose rows are basis rows (the CholeskyQR triangular product): per
    // 32-row chunk and column the record of project.cu's partial pass -- best
    // |q| (first row wins ties), its q, and q^T [x y z (x+y)+z] over the chunk
    // -- so the projection need not re-read the basis
    const double* projX = nullptr;  // n x 3 local coordinates per batch entry
    int64_t strideProjX = 0;
    double* projPart = nullptr;     // batch * projChunks * projCcap * 8
    int projN = 0, projChunks = 0, projCcap = 0;
};
void gemm(const GemmParams& p, bool transA, bool transB, cudaStream_t st);

// ------------------------------------------------------------------ assembly (assemble.cu)
struct TileRef {             // one submesh of one chain
    const int32_t* members;  // sorted ascending global ids (n)
    const int32_t* adj_offsets;
    const int32_t* adj_cols;
    const double* x;
    const double* y;
    const double* z;
};
void assemble_count(const TileRef* tiles, int ntiles, int n, int32_t* nnz_out, cudaStream_t st);
void assemble_fill(const TileRef* tiles, int ntiles, int n, int weighting, const int64_t* csr_offsets,
                   int32_t* rowptr, int32_t* cols, double* vals, double* trace, int* status,
                   int64_t* status_detail, cudaStream_t st);
void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int count, cudaStream_t st);
void natural_bandwidth(const int32_t* rowptr, const int32_t* cols, const int64_t* csr_offsets, const int32_t* perm,
                       int ntiles, int n, int32_t* bw_out, int32_t* blockw_out, int32_t* lower_out, cudaStream_t st);
void axis_order(const double* X, int64_t strideX, int ntiles, int n, int32_t* perm, cudaStream_t st);
void rcm_order(const int32_t* rowptr, const int32_t* cols, const int64_t* csr_offsets, int ntiles, int n,
               int32_t* perm, cudaStream_t st);

// ------------------------------------------------------------------ factor (factor.cu)
// Row stride of the (2W x W) solve operand slabs in global memory: padded to
// W + 4 doubles (% 16 == 4) so one bulk copy lands a slab in the solve's
// bank-conflict-free shared-memory layout.
__host__ __device__ constexpr int factor_row(int W) { return W + 4; }
struct FactorParams {
    int ntiles = 0, n = 0, W = 0, Kb = 0;
    const int32_t* rowptr = nullptr;  // per tile (n+1) entries at tile*(n+1)
    const int32_t* cols = nullptr;
    const double* vals = nullptr;
    const int64_t* csr_offsets = nullptr;
    const int32_t* perm = nullptr;  // per tile n entries (nullptr: natural)
    const double* delta = nullptr;  // per tile
    double* Ffwd = nullptr;
    double* Fbwd = nullptr;
    int64_t strideF = 0;  // doubles per tile
    int* status = nullptr;
    int cpl = 16;  // bound on a row's couplings into the previous block (lower neighbours)
};
void factor_tiles(const FactorParams& p, cudaStream_t st);
int factor_smem_bytes(int W);

// ------------------------------------------------------------------ solve (solve.cu)
struct SolveParams {
    int n = 0, Kb = 0, z = 2, c_cap = 0, batch = 1;
    const double* Ffwd = nullptr;
    const double* Fbwd = nullptr;
    int64_t strideF = 0;
    const int32_t* perm = nullptr;
    int64_t stridePerm = 0;
    const double* in = nullptr;
    int64_t ldin = 0, strideIn = 0;
    double* tmp = nullptr;
    int64_t ldt = 0, strideT = 0;
    double* out = nullptr;
    int64_t ldout = 0, strideOut = 0;
    const int* dimC = nullptr;
    int64_t dimStride = 0;
    int once = 0;
};
void solve_block_tridiag(const SolveParams& p, int W, cudaStream_t st);

// ------------------------------------------------------------------ CholeskyQR (cholqr.cu)
struct CholParams {
    int batch = 1, c_cap = 0;
    const double* G = nullptr;  // Gram (upper 64-tiles valid)
    int64_t ldg = 0, strideG = 0;
    double* A = nullptr;  // scaled Gram -> R~ (upper), ld multiple of 32 (>= c rounded to 32)
    int64_t lda = 0, strideA = 0;
    double* Binv = nullptr;  // B = D^-1 R~^-1 (upper, lower blocks zero), ld = ldb
    int64_t ldb = 0, strideB = 0;
    double* dscale = nullptr;  // column norms d_j (rounded-up length)
    int64_t strideD = 0;
    const int* dimC = nullptr;
    int64_t dimStride = 0;
    int* status = nullptr;           // sticky per-chain status (first error wins)
    int64_t* status_detail = nullptr;
    int* errpos = nullptr;           // chain position of the first error
    int pos = 0;
    double* vnorm = nullptr;         // ||V||_F per batch entry (rank-test scale)
    int rank_test = 1;
    // rank test: set to 1 (atomicOr, zeroed by the caller) when some pivot is not
    // far enough above the reference threshold for the Cholesky to certify it
    // (scaled pivot < 1e-8 or r_kk < 1e-9 ||V||_F): only then does the exact
    // |q_k^T v_k| test (rank_check) have anything to decide
    int* rank_need = nullptr;
    int column_scale = 1;
    // second CholeskyQR pass: when max|G~ - I| <= 1e-9 the factor is taken to
    // first order, R~ = I + triu(G~ - I, 1) (error O(|E|^2) <= c * 1e-18), and
    // B = D^-1 (I - triu(G~ - I, 1)) is written without the serial Cholesky
    int near_identity = 0;
    // skip the block back-substitution for R~^-1 (off-diagonal blocks of B); the
    // caller forms Q with trsm_right_upper instead
    int skip_inverse = 0;
    const int* skip = nullptr;  // optional per chain: nonzero -> nothing to do (pass 2 not needed)
    // adaptive CholeskyQR2 decided inside the near-identity scan (pass 2, single
    // CTA path): skip_out[b] = max |G - I| <= skip_tol (unscaled; the pass-1
    // factor is then kept and nothing else is written)
    int* skip_out = nullptr;
    double skip_tol = 0.0;
};
void chol_factor(const CholParams& p, cudaStream_t st);
// the shared-memory (cluster) Cholesky (cholx.cu); false when it does not apply
bool cholx_factor(const CholParams& p, cudaStream_t st);
// Adaptive CholeskyQR2: skip[b] = 1 when the pass-1 factor is already
// orthonormal to tol, max_{i<=k<c} |G_ik - delta_ik| <= tol (G = Q1^T Q1, upper)
void orth_check(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int64_t dimStride, int c_cap,
                int batch, double tol, int* skip, cudaStream_t st);
// Second CholeskyQR pass, near-identity case on all SMs: nmax[b] = max over the
// upper triangle of |G~ - I| (G~ = D^-1 G D^-1, D = sqrt(diag G); NaN -> inf;
// nmax zeroed by the caller), then for chains not skipped (skip_in) with
// nmax <= 1e-9: B = D^-1 (I - triu(G~ - I, 1)) (the factor to first order,
// error <= c * 1e-18) and d = D; skip_out[b] = skip_in[b] || near (the full
// Cholesky then runs only for the rest)
void near_check(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int c_cap, int batch,
                unsigned long long* nmax, cudaStream_t st);
void near_fill(const double* G, int64_t ldg, int64_t strideG, const int* dimC, int c_cap, int batch,
               const unsigned long long* nmax, const int* skip_in, int* skip_out, double* Binv, int64_t ldb,
               int64_t strideB, double* dscale, int64_t strideD, cudaStream_t st);
// dst_b = src_b for the batch entries with skip[b] == 0 (n x ld row-major blocks)
// Orthonormality probe (probe.cu): skip[b] = (estimated |Q^T Q - I|_F <= tol) from 8 fixed
// +-1 probe vectors in one pass over Q; part holds batch * orth_probe_chunks(n) * c_cap * 8.
int orth_probe_chunks(int n);
void orth_probe(const double* Q, int64_t ldq, int64_t strideQ, int n, const int* dimC, int c_cap, int batch, double tol,
                double* part, int* skip, double* est_out, cudaStream_t st);
void copy_unskipped(const double* src, double* dst, int64_t elems, int64_t stride, int batch, const int* skip,
                    cudaStream_t st);
int chol_smem_bytes(int c_cap);
// Q = V D^-1 R~^-1 by a row-parallel right triangular solve (trsm.cu), from the
// Cholesky's R~ (upper blocks in R) and diagonal-block inverses (diag of Binv).
struct TrsmParams {
    int n = 0, batch = 1, c_cap = 0;
    const double* V = nullptr;
    int64_t ldv = 0, strideV = 0;
    double* Q = nullptr;
    int64_t ldq = 0, strideQ = 0;
    const double* R = nullptr;
    int64_t ldr = 0, strideR = 0;
    const double* Binv = nullptr;
    int64_t ldb = 0, strideB = 0;
    const double* dscale = nullptr;
    int64_t strideD = 0;
    const int* dimC = nullptr;
    int64_t dimStride = 0;
    const int* status = nullptr;
};
void trsm_right_upper(const TrsmParams& p, cudaStream_t st);
bool trsm_supported(int c_cap);
int trsm_smem_bytes(int c_cap);
// Accurate reference rank test after CholeskyQR2: |r_kk| = |q_k^T v_k| against
// 1e-13 ||V||_F (first failing column, sticky status).
struct RankCheckParams {
    int n = 0, batch = 1, c_cap = 0;
    const double* Q = nullptr;
    const double* V = nullptr;
    int64_t ld = 0, stride = 0;
    const int* dimC = nullptr;
    int64_t dimStride = 0;
    const double* vnorm = nullptr;
    double* partial = nullptr;  // batch * chunks * c_cap
    int* status = nullptr;
    int64_t* status_detail = nullptr;
    int* errpos = nullptr;
    int pos = 0;
    int* counter = nullptr;  // per batch, zero: the last chunk CTA of a chain runs the test
    const int* need = nullptr;  // optional per batch: 0 -> the pass-1 pivots certified every column
};
void rank_check(const RankCheckParams& p, cudaStream_t st);

// ------------------------------------------------------------------ projection (project.cu)
struct ProjParams {
    int n = 0, batch = 1, c_cap = 0;
    const double* Q = nullptr;
    int64_t ldq = 0, strideQ = 0;
    const double* X = nullptr;  // n x 3 row-major
    int64_t strideX = 0;
    const int* dimC = nullptr;
    int64_t dimStride = 0;
    double* partial = nullptr;   // batch * nchunks * c_cap * 8
    double* partial2 = nullptr;  // batch * recon_blocks * 2
    int nchunks = 0, rows_per_chunk = 64, rows_per_warp = 2;
    int partials_ready = 0;  // the partial records were written by the CholeskyQR product (gemm projPart)
    double* coeff = nullptr;  // c_cap x 4 per batch: Px Py Pz Ps (unsigned)
    int64_t strideCoef = 0;
    double* sign = nullptr;  // per batch, stride strideSign
    int64_t strideSign = 0;
    double* xhat = nullptr;  // n x 3 row-major per batch
    int64_t strideXhat = 0;
    double* e_out = nullptr;
    int64_t strideE = 0;
    double* stats = nullptr;  // per batch: [0] residual_rms [1] ||e|| [2] ||X-X^||^2
    int* counter = nullptr;   // 2 per batch, zero: last-CTA reductions of the partial / recon passes
    int64_t strideStats = 4;
};
int proj_chunks(int n);
int proj_recon_blocks(int n, int rows_per_warp);
void project(const ProjParams& p, cudaStream_t st);

// ------------------------------------------------------------------ Jacobi RR (jacobi.cu)
struct JacobiParams {
    int batch = 1;
    const double* H = nullptr;
    int64_t ldh = 0, strideH = 0;
    double* stage = nullptr;
    int64_t strideStage = 0;
    double* V = nullptr;  // eigenvectors, column j contiguous at V + j*ldv
    int64_t ldv = 0, strideV = 0;
    double* theta = nullptr;
    double* theta_sorted = nullptr;
    int64_t strideTheta = 0;
    double* W = nullptr;  // sorted eigenvectors, row-major m x m
    int64_t ldw = 0, strideW = 0;
    int* sweeps = nullptr;
    int max_sweeps = 40;
    double tol = 1e-14;
};
struct JacobiPlan {
    int nc = 2, b = 1, P = 4, mp = 8, smem = 0;
    int64_t stage_elems = 0;
};
JacobiPlan jacobi_plan(int m);
int jacobi_eigh(const JacobiParams& p, const JacobiPlan& pl, int m, cudaStream_t st);

// ------------------------------------------------------------------ utilities (util.cu)
void transpose_to_rowmajor(const double* colmajor, int rows, int cols, double* rowmajor, int64_t ld,
                           cudaStream_t st);
void transpose_to_colmajor(const double* rowmajor, int64_t ld, int rows, int cols, const double* sign,
                           double* colmajor, cudaStream_t st);
void fill(double* p, int64_t count, double v, cudaStream_t st);
void gather_coords(const TileRef* tiles, int ntiles, int n, double* X, int64_t strideX, double* bbox,
                   cudaStream_t st);
void randn(double* p, int rows, int cols, int64_t ld, int64_t stride, int batch, uint64_t seed, cudaStream_t st);

struct SpmmParams {
    int n = 0, c = 0, batch = 1;
    const int32_t* rowptr = nullptr;
    int64_t strideRowptr = 0;
    const int64_t* csr_offsets = nullptr;  // per batch offset into cols/vals (nullptr: 0)
    int64_t offStride = 1;                 // csr_offsets index stride per batch entry
    const int32_t* cols = nullptr;
    const double* vals = nullptr;
    const double* shift = nullptr;  // per batch diagonal shift (nullptr: 0)
    // Chebyshev-step form Y = alpha_b (L + shift_b I) X + gamma_b Z (nullptr: alpha 1, no Z term)
    const double* alpha = nullptr;
    const double* gamma = nullptr;
    const double* Z = nullptr;
    int64_t ldz = 0, strideZ = 0;
    const double* X = nullptr;
    int64_t ldx = 0, strideX = 0;
    double* Y = nullptr;
    int64_t ldy = 0, strideY = 0;
    const int* dimC = nullptr;
    int64_t dimStride = 0;
};
void spmm(const SpmmParams& p, cudaStream_t st);

// The whole Chebyshev filter of one application (deg steps of the three-term
// recurrence X_i = alpha_i (L + s I) X_{i-1} + gamma_i X_{i-2}) for binary-weight
// Laplacians, with the CSR pattern and the iterates of a column slice held in
// shared memory: the same per-element arithmetic as deg spmm() calls.
struct ChebParams {
    int n = 0, c = 0, batch = 1, deg = 0;
    const int32_t* rowptr = nullptr;
    int64_t strideRowptr = 0;
    const int64_t* csr_offsets = nullptr;
    int64_t offStride = 1;
    const int32_t* cols = nullptr;
    const double* vals = nullptr;
    const double* coef = nullptr;  // [deg][batch] alpha | [deg][batch] gamma | [batch] shift
    const double* X = nullptr;     // X_0
    int64_t ldx = 0, strideX = 0;
    double* Y = nullptr;           // X_deg
    int64_t ldy = 0, strideY = 0;
};
bool cheb_filter_supported(int n, int max_nnz);
void cheb_filter(const ChebParams& p, int max_nnz, cudaStream_t st);

struct Stitcher {
    int n = 0, n_d = 0;
    int32_t* offs = nullptr;
    int64_t* slots = nullptr;
    int32_t* missing = nullptr;
    void build(const int32_t* members, int nsub, int n_d, int n, cudaStream_t st);
    void release(cudaStream_t st);
};
struct StitchParams {
    int n = 0, n_d = 0, weighted = 1;
    const int32_t* offs = nullptr;
    const int64_t* slots = nullptr;
    const int32_t* rowptr = nullptr;  // per submesh id (n_d+1)
    const double* xhat = nullptr;     // per submesh id n_d x 3 row-major
    int64_t strideXhat = 0;
    double* out = nullptr;  // SoA n x 3
};
void stitch(const StitchParams& p, cudaStream_t st);

// ------------------------------------------------------------------ frames (frames.cu)
// coarse_reconstruct_points for many frames over one set of bases (F3,
// denoise_dynamic's frames stage, denoise.hpp:280-288)
struct FramesParams {
    int n = 0;                 // mesh vertex count
    int k = 0, n_d = 0;        // submeshes (ids 0..k-1), block size
    const int32_t* members = nullptr;  // k * n_d, sorted per submesh
    const double* bases = nullptr;     // per id n_d x c column-major, stride strideU
    int64_t strideU = 0;
    const int* dimC = nullptr;         // per id c (device)
    int c_cap = 0;
    int frames = 0;
    const double* const* xyz = nullptr;  // device table: x_0 y_0 z_0 x_1 ... (3 * frames)
    double* const* out = nullptr;        // device table: frames SoA n x 3 outputs
    int weighted = 1;
    const int32_t* deg = nullptr;        // k * n_d local degrees
    const int32_t* owner_offs = nullptr; // Stitcher owners
    const int64_t* owner_slots = nullptr;
};
struct FramesWork {
    int batch_frames = 1;
    double* X = nullptr;     // k * n_d * ldx
    double* Xhat = nullptr;  // k * n_d * ldx
    double* C = nullptr;     // k * c_cap * ldx
    double* Cws = nullptr;   // split-K workspace k * splits * c_cap * ldx (splits <= n_d / 256)
};
int frames_batch(const FramesParams& p);
void local_degrees(const int32_t* members, int k, int n_d, const int32_t* adj_offsets, const int32_t* adj_cols,
                   int32_t* deg, cudaStream_t st);
void coarse_reconstruct_frames(const FramesParams& p, const FramesWork& w, cudaStream_t st);

// ------------------------------------------------------------------ codec (codec.cu)
// per block in SubmeshOrder position order (EncodedMesh.blocks, compress.hpp:108)
struct CodecParams {
    int blocks = 0, quant_bits = 12;
    const int* c = nullptr;               // subspace size per position
    const double* const* coef = nullptr;  // encode: c x 3 column-major coefficients per position
    uint16_t* values = nullptr;           // 3c per position, axis-major (EncodedBlock.values)
    const int64_t* value_off = nullptr;
    double* lo = nullptr;                 // 3 per position (coeff_min)
    double* hi = nullptr;                 // 3 per position (coeff_max)
    uint8_t* flags = nullptr;             // constant_axis bits
    int64_t* payload_bytes = nullptr;     // encode: packed bytes per position
    uint8_t* payload = nullptr;
    const int64_t* payload_off = nullptr;
    const int* dest = nullptr;            // unpack: submesh id of the position
    double* C = nullptr;                  // unpack: c x ldc row-major per submesh id
    int64_t strideC = 0;
    int ldc = 0;
};
void codec_encode(const CodecParams& p, cudaStream_t st);
void codec_pack(const CodecParams& p, cudaStream_t st);
void codec_unpack(const CodecParams& p, cudaStream_t st);
// igft + stitch of given coefficients (decompress_mesh's decode + reconstruct_weighted)
void reconstruct_from_coefficients(const FramesParams& p, const double* C, int ldc, double* Xhat,
                                   cudaStream_t st);

// ------------------------------------------------------------------ fine denoising (fine.cu)
// fine_denoise (denoise.hpp:172-178): face_geometry, face_ring_adjacency,
// bilateral_normals, update_vertices; device pointers
struct FineParams {
    int64_t n = 0, nf = 0;
    const double* x = nullptr;  // SoA vertices
    const double* y = nullptr;
    const double* z = nullptr;
    const int32_t* faces = nullptr;  // nf x 3 row-major
    double sigma_spatial = 0.0, sigma_range = 0.35;
    int normal_iterations = 5, vertex_iterations = 10, ring_depth = 1;
    double* out = nullptr;          // SoA n x 3
    double* normals_out = nullptr;  // optional SoA nf x 3 (filtered normals)
};
void fine_denoise(const FineParams& p, cudaStream_t st);

}  // namespace smg

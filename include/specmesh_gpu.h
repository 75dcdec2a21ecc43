/*
 * specmesh_gpu.h -- C ABI of the B200-native OI spectral path (libspecmesh_b200.so).
 *
 * Drop-in boundary for the reference's per-submesh spectral chain
 * (/root/reference/proj/include/specmesh; header-only C++ over Eigen, no FFI of
 * its own -- SURVEY.md §8(b)).  Each entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only; exceptions never cross
 * the boundary: every call returns a status and smg_last_error() holds the
 * reference's message text ("orthonormalize: block is rank deficient at column 14").
 *
 * Conventions
 *   - Status codes follow the SPEC CLI exit codes: 0 ok,
 *     2 InvalidArgument (core.hpp:24-28, `require` preconditions), 3 Error
 *     (numerical failures, core.hpp:18-22).
 *   - Dense matrices cross the ABI column-major (Eigen's default storage of
 *     MatrixXd / MatrixX3d): an n x c basis is c contiguous columns of n doubles,
 *     Points (n x 3) are x[0..n) | y[0..n) | z[0..n).
 *   - The Laplacian crosses as CSR with int32 indices; for the symmetric L these
 *     are exactly Eigen's compressed-column arrays (spectral.hpp:63-66).
 *   - `on_device` = 0: host pointers (copied in/out inside the call);
 *     1: device pointers on the context's device (no host copies).
 *   - A context owns one CUDA device and one stream; it is thread-compatible
 *     (one context per host thread).
 *   - There is no CPU fallback: every compute call runs sm_100a kernels and
 *     fails with status 3 if the device cannot run them.
 */
#ifndef SPECMESH_GPU_H
#define SPECMESH_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMG_ABI_VERSION 2

/* 2 = InvalidArgument, 3 = Error, 4 = ParseError (core.hpp:18-34) */
typedef enum { SMG_OK = 0, SMG_INVALID_ARGUMENT = 2, SMG_ERROR = 3, SMG_PARSE_ERROR = 4 } smg_status;

/* spectral.hpp:22 Weighting */
typedef enum { SMG_WEIGHTING_BINARY = 0, SMG_WEIGHTING_DISTANCE = 1 } smg_weighting;
/* pipeline.hpp:12 BasisMode (SVD is the non-OI comparison baseline: out of scope) */
typedef enum { SMG_BASIS_OI = 0, SMG_BASIS_DOI = 1 } smg_basis_mode;

typedef struct smg_context smg_context;
typedef struct smg_operator smg_operator;
typedef struct smg_comm smg_comm;

/* Mesh (mesh.hpp:18-37) + EdgeSet (mesh.hpp:40-50, neighbour lists sorted ascending). */
typedef struct {
    int64_t vertex_count;
    const double* x;            /* vertex_count */
    const double* y;
    const double* z;
    const int32_t* adj_offsets; /* vertex_count + 1 */
    const int32_t* adj_cols;    /* adj_offsets[vertex_count] */
    int32_t on_device;
} smg_mesh;

/* Segmentation (pipeline.hpp:125-129) reduced to what the path reads: the
 * submeshes' member lists (partition.hpp:34-47; sorted ascending = local order)
 * and the SubmeshOrder sequence (partition.hpp:49-51). */
typedef struct {
    int32_t submesh_count;
    const int32_t* member_offsets; /* submesh_count + 1 */
    const int32_t* members;
    int32_t sequence_length;
    const int32_t* sequence;       /* permutation of submesh ids */
    int32_t on_device;
} smg_segmentation;

/* PipelineConfig (pipeline.hpp:41-68), path fields only, field for field. */
typedef struct {
    int32_t weighting;          /* smg_weighting; reference default distance */
    int32_t basis_mode;         /* smg_basis_mode */
    int32_t subspace_size;      /* fixed c; initial c in DOI mode (16) */
    double eps_low;             /* DOI band, relative to bbox diagonal (0.004) */
    double eps_high;            /* (0.04) */
    int32_t c_min;              /* (2) */
    int32_t c_max;              /* 0: derived, resolve_c_max (pipeline.hpp:60-63) */
    int32_t power;              /* z (2) */
    int32_t iterations;         /* t_max per OI update (2) */
    int32_t initial_iterations; /* cold-start OI when n_d > dense_limit (60) */
    int32_t doi_iterations;     /* 0: derived, resolve_doi_iterations (pipeline.hpp:64-67) */
    uint64_t seed;              /* (1) */
    int32_t dense_limit;        /* (4096) */
    double shift_scale;         /* delta = shift_scale * trace(L)/n_d (1e-8) */
    /* segmentation (segment_mesh, pipeline.hpp:131-138): used when a chain call
     * gets no Segmentation (seg == NULL), as the reference always segments */
    int32_t part_count;         /* k (8) */
    double growth;              /* overlap factor, n_d = floor(growth * max part) (1.15) */
} smg_pipeline_config;

/* Results of a chain: BlockBases.stats (pipeline.hpp:70-92) plus the optional
 * coefficient / reconstruction / basis outputs.  Arrays are indexed by submesh
 * id.  Optional pointers may be NULL. */
typedef struct {
    int32_t* subspace_size;   /* [submesh_count] */
    double* residual_rms;     /* [submesh_count] projection_residual_rms */
    double* doi_residual;     /* [submesh_count] */
    int32_t* converged;       /* [submesh_count] */
    int32_t* oi_iterations;   /* [submesh_count] */
    /* coarse_reconstruct_points (pipeline.hpp:300-305), Weighted mode: vertex_count x 3 */
    double* reconstruction;
    /* gft coefficients C = U^T X (spectral.hpp:290-293), c_id x 3 column-major per
     * submesh id, packed at coefficient_offsets[id] (offsets written by the call) */
    double* coefficients;
    int64_t coefficients_capacity;  /* doubles available in `coefficients` */
    int64_t* coefficient_offsets;   /* [submesh_count + 1] */
    /* tracked bases n_d x c_id column-major at basis_offsets[id] */
    double* bases;
    int64_t bases_capacity;         /* doubles available in `bases` */
    int64_t* basis_offsets;         /* [submesh_count + 1] */
    int32_t on_device;              /* applies to reconstruction/coefficients/bases */
    /* StageTimings (core.hpp:41-68), device-event seconds:
     * [0] laplacian [1] factorize [2] basis (first submesh) [3] basis_total
     * [4] project (gft+igft+stitch) [5] total */
    double timings[6];
    /* the segmentation the call used (optional; filled when the call segmented
     * the mesh itself, seg == NULL): SubmeshOrder sequence [submesh_count],
     * sorted member lists (submesh_count x block_size, row = submesh id) */
    int32_t* sequence_out;
    int32_t* members_out;
    int64_t members_capacity;
    int32_t block_size;       /* n_d (always written) */
} smg_chain_output;

int smg_abi_version(void);
const char* smg_last_error(const smg_context* ctx);

/* Context on CUDA device `device`.  Fails (status 3) without a usable sm_100 device. */
smg_status smg_create(int device, smg_context** out);
void smg_destroy(smg_context* ctx);

/* PipelineConfig defaults (pipeline.hpp:41-58). */
void smg_default_config(smg_pipeline_config* cfg);

/* ---------------------------------------------------------------- L4 chain */

/* compute_block_bases_fixed_sizes (pipeline.hpp:144-194) followed, when the
 * output requests it, by project_blocks + coarse_reconstruct_points
 * (pipeline.hpp:290-305).  sizes_in_order: one c per order position (host). */
smg_status smg_compute_block_bases_fixed_sizes(smg_context* ctx, const smg_mesh* mesh,
                                               const smg_segmentation* seg,
                                               const smg_pipeline_config* cfg,
                                               const int32_t* sizes_in_order,
                                               smg_chain_output* out);

/* compute_block_bases (pipeline.hpp:198-287) for basis_mode OI or DOI, over an
 * EXTERNAL segmentation (the reference segments internally at :201; the
 * configs supply their own tiles). */
/* seg == NULL: the mesh is segmented on the GPU first (segment_mesh with
 * cfg->part_count, cfg->growth, cfg->seed -- the reference's own flow,
 * pipeline.hpp:198-201); out arrays then hold cfg->part_count submeshes. */
smg_status smg_compute_block_bases(smg_context* ctx, const smg_mesh* mesh,
                                   const smg_segmentation* seg,
                                   const smg_pipeline_config* cfg, smg_chain_output* out);

/* n_chains independent fixed-size chains (one per mesh) processed in lockstep
 * on this context's device; all submeshes of all chains must share n_d and c.
 * meshes/segs/outs are arrays of n_chains.  This is config 5's per-GPU shard. */
smg_status smg_run_chains(smg_context* ctx, int32_t n_chains, const smg_mesh* meshes,
                          const smg_segmentation* segs, const smg_pipeline_config* cfg,
                          const int32_t* sizes_in_order, smg_chain_output* outs);

/* ------------------------------------------------------ F3 dynamic meshes */

/* AverageMode (partition.hpp:53). */
typedef enum { SMG_AVERAGE_SIMPLE = 0, SMG_AVERAGE_WEIGHTED = 1 } smg_average_mode;

/* BlockBases.bases (pipeline.hpp:78-92) in the layout smg_chain_output writes:
 * the basis of submesh id is n_d x subspace_size[id], column-major, at
 * data + offsets[id].  subspace_size/offsets are host arrays. */
typedef struct {
    int32_t submesh_count;
    const int32_t* subspace_size; /* [submesh_count] */
    const int64_t* offsets;       /* [submesh_count + 1] */
    const double* data;
    int32_t on_device;
} smg_bases;

/* coarse_reconstruct_points(frame, bases, mode) (pipeline.hpp:300-305) for
 * frame_count frames that share `topology`'s connectivity (its coordinates are
 * not read; x/y/z may be NULL) -- the frames stage of denoise_dynamic
 * (denoise.hpp:280-288).  frames_xyz: 3 * frame_count pointers x_0, y_0, z_0,
 * x_1, ... of vertex_count doubles; out: frame_count pointers, each a SoA
 * vertex_count x 3 result.  Uncovered vertices -> status 2 with the reference
 * message (partition.hpp:347-353). */
smg_status smg_coarse_reconstruct_frames(smg_context* ctx, const smg_mesh* topology,
                                         const smg_segmentation* seg, const smg_bases* bases,
                                         int32_t frame_count, const double* const* frames_xyz,
                                         int32_t frames_on_device, int32_t average_mode,
                                         double* const* out, int32_t out_on_device);

/* denoise_dynamic (denoise.hpp:258-291) over an EXTERNAL segmentation: the
 * bases of frames[0] (fixed sizes_in_order when given, else compute_block_bases
 * by cfg->basis_mode), then every frame's coarse reconstruction.  Every frame
 * must share frames[0]'s connectivity (status 2, "frame i does not share the
 * sequence connectivity").  *basis_blocks_computed = number of bases (k).
 * timings (optional, 3 doubles, device-event seconds): [0] shared_basis
 * [1] frames [2] total. */
smg_status smg_denoise_dynamic(smg_context* ctx, int32_t frame_count, const smg_mesh* frames,
                               const smg_segmentation* seg, const smg_pipeline_config* cfg,
                               const int32_t* sizes_in_order, int32_t average_mode,
                               double* const* out, int32_t out_on_device,
                               int32_t* basis_blocks_computed, double* timings);

/* ------------------------------------------------------------ F2 spectral codec */

/* EncodedBlock (compress.hpp:17-25) of every block in SubmeshOrder sequence
 * order, plus the block payloads exactly as serialize_encoded_mesh packs them
 * (compress.hpp:415-423: non-constant axes' values, quant_bits each, MSB first,
 * each block padded to a byte).  Host arrays. */
typedef struct {
    int32_t block_count;
    int32_t quant_bits;
    uint32_t* submesh_id;     /* [block_count] */
    uint32_t* subspace_size;  /* [block_count] */
    double* coeff_min;        /* [3 * block_count] */
    double* coeff_max;        /* [3 * block_count] */
    uint8_t* constant_axis;   /* [block_count]: bit a = axis a constant (the serialized flags byte) */
    uint16_t* values;         /* optional [3 * sum c]: block i's 3c values (axis-major) at 3 * (sum of earlier c) */
    uint8_t* payload;
    int64_t payload_capacity; /* bytes; sum over blocks of ceil(3 c quant_bits / 8) always suffices */
    int64_t* payload_offsets; /* [block_count + 1] */
} smg_encoded_blocks;

/* compress_mesh's basis and encode stages (compress.hpp:152-219) over an
 * EXTERNAL segmentation: Binary weighting (forced, as the reference does);
 * sizes_in_order (host, one c per position) when given, else cfg->basis_mode:
 * OI -> subspace_size for every block, DOI -> the sizes a DOI probe chain picks
 * (compress.hpp:162-166); then the fixed-size OI chain, gft and encode_block
 * (compress.hpp:33-62) per block.  quant_bits in [1, 16]. */
smg_status smg_compress_blocks(smg_context* ctx, const smg_mesh* mesh, const smg_segmentation* seg,
                               const smg_pipeline_config* cfg, const int32_t* sizes_in_order,
                               int32_t quant_bits, smg_encoded_blocks* out);

/* decompress_mesh (compress.hpp:221-256) over an external segmentation: replays
 * the chain from `topology`'s connectivity alone (coordinates not read; Binary
 * weighting, the blocks' sizes), decodes every block (dequantize_block +
 * igft, compress.hpp:64-89) and stitches with degree weights.  `in->payload`
 * and the per-block headers are read; `in->values` may be NULL.  A block count
 * or order that does not match the segmentation -> status 4 (ParseError) with
 * the reference message.  out: SoA vertex_count x 3. */
smg_status smg_decompress_blocks(smg_context* ctx, const smg_mesh* topology, const smg_segmentation* seg,
                                 const smg_pipeline_config* cfg, const smg_encoded_blocks* in,
                                 double* out, int32_t out_on_device);

/* ------------------------------------------------------ F4 fine denoising */

/* BilateralParams (denoise.hpp:11-24). */
typedef struct {
    double sigma_spatial;       /* 0: mean adjacent-centroid distance (default_sigma_spatial) */
    double sigma_range;         /* (0.35) */
    int32_t normal_iterations;  /* (5) */
    int32_t vertex_iterations;  /* (10) */
    int32_t ring_depth;         /* (1) */
} smg_bilateral_params;

void smg_default_bilateral_params(smg_bilateral_params* params);

/* fine_denoise (denoise.hpp:172-178): face_geometry (mesh.hpp:94-116),
 * face_ring_adjacency (denoise.hpp:39-65), bilateral_normals (:87-127) and
 * update_vertices (:133-165).  Vertices SoA (x, y, z: vertex_count each),
 * faces face_count x 3 row-major; out: SoA vertex_count x 3; normals_out
 * (optional): the filtered face normals, SoA face_count x 3.  All pointers
 * host (on_device = 0) or device.  The reference's validate() and
 * "mesh has no adjacent face pairs" errors -> status 2. */
smg_status smg_fine_denoise(smg_context* ctx, int64_t vertex_count, const double* x, const double* y,
                            const double* z, int64_t face_count, const int32_t* faces,
                            const smg_bilateral_params* params, double* out, double* normals_out,
                            int32_t on_device);

/* ------------------------------------------------------------ multi-GPU
 * Independent chains shard over ranks, one process per GPU, no exchange during
 * compute; per-mesh results are all-gathered (NCCL over NVLink / NVSwitch).
 * NCCL is loaded at run time (libnccl.so.2; SMG_NCCL_LIB overrides). */

/* the contiguous balanced slice of `total` chains owned by `rank` (the first
 * total % world ranks get one extra) */
smg_status smg_shard_range(int32_t total, int32_t world, int32_t rank, int32_t* first, int32_t* count);
/* rank 0: a 128-byte NCCL unique id for the caller to broadcast */
smg_status smg_comm_unique_id(smg_context* ctx, uint8_t* id);
smg_status smg_comm_create(smg_context* ctx, const uint8_t* id, int32_t world, int32_t rank, smg_comm** out);
void smg_comm_destroy(smg_comm* comm);
/* all-gather of per-mesh rows in global mesh order: `local` = this rank's
 * shard (smg_shard_range rows of row_doubles, device), `out` = total rows
 * (device), on the context stream; ragged shards are padded internally */
smg_status smg_gather_meshes(smg_context* ctx, smg_comm* comm, int32_t total, int64_t row_doubles,
                             const double* local, double* out);

/* ------------------------------------------------------------ segmentation (F1)
 * The step before the path, on the GPU and bit-exact with the reference's tie
 * rules.  Host or device mesh (mesh->on_device); outputs are host or device
 * pointers (any, copied with cudaMemcpyDefault).  InvalidArgument texts are
 * the reference's ("part count k must satisfy 1 <= k <= n/4", "partition
 * failed: k is incompatible with the mesh connectivity (...)", "overlap growth
 * must be >= 1.0", "partition has an empty part", ...). */

/* partition_mesh (partition.hpp:84-159): assignment[n] = part id. */
smg_status smg_partition_mesh(smg_context* ctx, const smg_mesh* mesh, int32_t part_count, uint64_t seed,
                              int32_t* assignment);
/* expand_overlaps (partition.hpp:205-253): part_count sorted member lists of
 * n_d = floor(growth * max part size) vertices (row = part id); *block_size = n_d. */
smg_status smg_expand_overlaps(smg_context* ctx, const smg_mesh* mesh, const int32_t* assignment,
                               int32_t part_count, double growth, int32_t* members,
                               int64_t members_capacity, int32_t* block_size);
/* order_submeshes (partition.hpp:258-307): host member lists (offsets). */
smg_status smg_order_submeshes(smg_context* ctx, int32_t submesh_count, const int32_t* member_offsets,
                               const int32_t* members, uint64_t seed, int32_t* sequence);
/* segment_mesh (pipeline.hpp:131-138) = the three above; assignment optional. */
smg_status smg_segment_mesh(smg_context* ctx, const smg_mesh* mesh, int32_t part_count, double growth,
                            uint64_t seed, int32_t* assignment, int32_t* members,
                            int64_t members_capacity, int32_t* block_size, int32_t* sequence);

/* ------------------------------------------------------------ L3 primitives
 * Host pointers, column-major.  They run the same kernels as the chain. */

/* detail::build_submesh adjacency (partition.hpp:169-184) + build_laplacian
 * (spectral.hpp:39-68) for one submesh.  Writes CSR (rowptr n+1, cols/vals nnz);
 * nnz_capacity bounds cols/vals; *nnz_out gets the count; *trace_out = trace(L)
 * (spectral.hpp:32-36).  Coincident connected vertices under distance weighting
 * -> status 3 with the reference message. */
smg_status smg_build_laplacian(smg_context* ctx, const smg_mesh* mesh, const int32_t* members,
                               int32_t n, int32_t weighting, int32_t* rowptr, int32_t* cols,
                               double* vals, int64_t nnz_capacity, int64_t* nnz_out,
                               double* trace_out);

/* default_shift (spectral.hpp:193-196). */
double smg_default_shift(double trace, int32_t n, double scale);

/* ShiftedInverseOperator (spectral.hpp:145-190): factor L + delta I (host CSR). */
smg_status smg_operator_create(smg_context* ctx, int32_t n, const int32_t* rowptr,
                               const int32_t* cols, const double* vals, double delta, int32_t z,
                               smg_operator** out);
void smg_operator_destroy(smg_operator* op);
/* apply (z solves, spectral.hpp:172-176) or apply_once (:166-169). */
smg_status smg_operator_apply(smg_context* ctx, const smg_operator* op, int32_t c,
                              const double* block, double* out, int32_t once);
/* (L + delta I) X  -- CSR SpMM (no reference symbol; residual / verification). */
smg_status smg_operator_spmm(smg_context* ctx, const smg_operator* op, int32_t c,
                             const double* block, double* out);

/* orthonormalize (spectral.hpp:120-132): thin Q with the reference rank test and
 * sign convention.  Status 3 "orthonormalize: block is rank deficient at column k". */
smg_status smg_orthonormalize(smg_context* ctx, int32_t rows, int32_t cols, const double* block,
                              double* q);

/* orthogonal_iteration (spectral.hpp:204-211). */
smg_status smg_orthogonal_iteration(smg_context* ctx, const smg_operator* op, int32_t c,
                                    const double* init, int32_t t_max, double* out);

/* dynamic_oi (spectral.hpp:244-287).  basis_out holds n x c_max doubles; the
 * final c is written to *c_out. coords: n x 3 column-major. */
smg_status smg_dynamic_oi(smg_context* ctx, const smg_operator* op, int32_t c,
                          const double* init, const double* coords, double eps_low,
                          double eps_high, int32_t c_min, int32_t c_max, int32_t t_max,
                          double* basis_out, int32_t* c_out, int32_t* converged,
                          double* residual, int32_t* iterations);

/* bottom_subspace(dense_eigendecomposition(L), c) (spectral.hpp:92-117): the
 * first-submesh basis, produced on the GPU by shift-invert subspace iteration +
 * Rayleigh-Ritz on the operator's factor (K9).  eigenvalues_out
 * (optional, c doubles) gets the ascending Ritz values. */
smg_status smg_bottom_subspace(smg_context* ctx, const smg_operator* op, int32_t c,
                               double* basis_out, double* eigenvalues_out);

/* gft / igft (spectral.hpp:290-298). */
smg_status smg_gft(smg_context* ctx, int32_t rows, int32_t c, const double* basis,
                   const double* coords, double* coeffs);
smg_status smg_igft(smg_context* ctx, int32_t rows, int32_t c, const double* basis,
                    const double* coeffs, double* coords);

/* ------------------------------------------------------------ diagnostics
 * Per-stage device time (CUDA events on the context stream) of the library's
 * kernels, the StageTimings analogue at kernel granularity.  Stages:
 * "assemble", "factor", "solve", "orthonormalize" (= "gram" + "chol" + "trmm"
 * + rank test), "project"; nested scopes are inclusive.  Enabling clears the
 * record. */
smg_status smg_profile_enable(smg_context* ctx, int32_t on);
smg_status smg_profile_read(smg_context* ctx, const char* stage, int64_t* launches, double* total_ms);

/* What the last chain call (smg_compute_block_bases*, smg_run_chains) chose:
 * the factorisation's block width W (the block-tridiagonal solve's half-band
 * is W + 1) and ordering (0 natural, 1 geometric = sort along the tile's
 * longest axis, 2 RCM), the chain groups (streams) and the batch shape. */
typedef struct {
    int32_t block_width;
    int32_t ordering;
    int32_t chain_groups;
    int32_t chains;
    int32_t positions;
} smg_run_info;
smg_status smg_last_run_info(smg_context* ctx, smg_run_info* info);

/* DOI step log (decision-level parity of dynamic_oi, spectral.hpp:259-283):
 * while enabled, every dynamic_oi step of smg_compute_block_bases (DOI mode)
 * and smg_dynamic_oi appends (chain position, subspace size the step ran
 * with, residual ||e||/bbox_diag that decided it).  Enabling or disabling
 * clears the log.  smg_doi_trace_read with capacity 0 returns the count only. */
smg_status smg_doi_trace_enable(smg_context* ctx, int32_t on);
smg_status smg_doi_trace_read(smg_context* ctx, int64_t capacity, int32_t* position,
                              int32_t* subspace_size, double* residual, int64_t* count);

/* The one-pass orthonormality probe of the adaptive CholeskyQR2 (probe.cu): an estimate of
 * ||Q^T Q - I||_F from 8 fixed +-1 vectors, for a column-major rows x cols block.  In the fixed-c
 * chain a pass-1 factor whose estimate is <= 1e-13 sqrt(c) skips the second pass; this entry
 * exposes the estimator so tests can hold it against the exact norm.  No reference counterpart
 * (HouseholderQR, spectral.hpp:125-129, needs no second pass). */
smg_status smg_orthonormality_estimate(smg_context* ctx, int32_t rows, int32_t cols, const double* q,
                                       double* estimate);

#ifdef __cplusplus
}
#endif

#endif /* SPECMESH_GPU_H */

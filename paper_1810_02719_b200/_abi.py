"""ctypes binding of the C ABI in include/specmesh_gpu.h (libspecmesh_b200.so).

This is the Python-side equivalent of the FFI stub a maintainer would add to
call the library.  No torch types cross the boundary: plain
pointers and sizes only.  Loading fails loudly when the shared library is
missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libspecmesh_b200.so")

SMG_OK, SMG_INVALID_ARGUMENT, SMG_ERROR, SMG_PARSE_ERROR = 0, 2, 3, 4
WEIGHTING = {"binary": 0, "distance": 1}
BASIS_MODE = {"oi": 0, "doi": 1}

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)


class smg_mesh(C.Structure):
    _fields_ = [("vertex_count", C.c_int64), ("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p),
                ("adj_offsets", C.c_void_p), ("adj_cols", C.c_void_p), ("on_device", C.c_int32)]


class smg_segmentation(C.Structure):
    _fields_ = [("submesh_count", C.c_int32), ("member_offsets", C.c_void_p), ("members", C.c_void_p),
                ("sequence_length", C.c_int32), ("sequence", C.c_void_p), ("on_device", C.c_int32)]


class smg_pipeline_config(C.Structure):
    _fields_ = [("weighting", C.c_int32), ("basis_mode", C.c_int32), ("subspace_size", C.c_int32),
                ("eps_low", C.c_double), ("eps_high", C.c_double), ("c_min", C.c_int32), ("c_max", C.c_int32),
                ("power", C.c_int32), ("iterations", C.c_int32), ("initial_iterations", C.c_int32),
                ("doi_iterations", C.c_int32), ("seed", C.c_uint64), ("dense_limit", C.c_int32),
                ("shift_scale", C.c_double), ("part_count", C.c_int32), ("growth", C.c_double)]


class smg_chain_output(C.Structure):
    _fields_ = [("subspace_size", C.c_void_p), ("residual_rms", C.c_void_p), ("doi_residual", C.c_void_p),
                ("converged", C.c_void_p), ("oi_iterations", C.c_void_p), ("reconstruction", C.c_void_p),
                ("coefficients", C.c_void_p), ("coefficients_capacity", C.c_int64),
                ("coefficient_offsets", C.c_void_p), ("bases", C.c_void_p), ("bases_capacity", C.c_int64),
                ("basis_offsets", C.c_void_p), ("on_device", C.c_int32), ("timings", C.c_double * 6),
                ("sequence_out", C.c_void_p), ("members_out", C.c_void_p), ("members_capacity", C.c_int64),
                ("block_size", C.c_int32)]


class smg_bases(C.Structure):
    _fields_ = [("submesh_count", C.c_int32), ("subspace_size", C.c_void_p), ("offsets", C.c_void_p),
                ("data", C.c_void_p), ("on_device", C.c_int32)]


class smg_encoded_blocks(C.Structure):
    _fields_ = [("block_count", C.c_int32), ("quant_bits", C.c_int32), ("submesh_id", C.c_void_p),
                ("subspace_size", C.c_void_p), ("coeff_min", C.c_void_p), ("coeff_max", C.c_void_p),
                ("constant_axis", C.c_void_p), ("values", C.c_void_p), ("payload", C.c_void_p),
                ("payload_capacity", C.c_int64), ("payload_offsets", C.c_void_p)]


class smg_bilateral_params(C.Structure):
    _fields_ = [("sigma_spatial", C.c_double), ("sigma_range", C.c_double), ("normal_iterations", C.c_int32),
                ("vertex_iterations", C.c_int32), ("ring_depth", C.c_int32)]


class smg_run_info(C.Structure):
    _fields_ = [("block_width", C.c_int32), ("ordering", C.c_int32), ("chain_groups", C.c_int32),
                ("chains", C.c_int32), ("positions", C.c_int32)]


AVERAGE_MODE = {"simple": 0, "weighted": 1}

# every symbol include/specmesh_gpu.h declares (checked by the CPU test suite)
EXPORTED = [
    "smg_abi_version", "smg_last_error", "smg_create", "smg_destroy", "smg_default_config",
    "smg_compute_block_bases_fixed_sizes", "smg_compute_block_bases", "smg_run_chains",
    "smg_build_laplacian", "smg_default_shift", "smg_operator_create", "smg_operator_destroy",
    "smg_operator_apply", "smg_operator_spmm", "smg_orthonormalize", "smg_orthogonal_iteration",
    "smg_dynamic_oi", "smg_bottom_subspace", "smg_gft", "smg_igft", "smg_profile_enable", "smg_profile_read",
    "smg_coarse_reconstruct_frames", "smg_denoise_dynamic", "smg_compress_blocks", "smg_decompress_blocks",
    "smg_default_bilateral_params", "smg_fine_denoise", "smg_doi_trace_enable", "smg_doi_trace_read",
    "smg_last_run_info", "smg_partition_mesh", "smg_expand_overlaps", "smg_order_submeshes", "smg_segment_mesh",
    "smg_shard_range", "smg_comm_unique_id", "smg_comm_create", "smg_comm_destroy", "smg_gather_meshes",
    "smg_orthonormality_estimate",
]

_lib: Optional[C.CDLL] = None


def load(path: Optional[str] = None) -> C.CDLL:
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"libspecmesh_b200.so not built ({p}); run `make` or __graft_entry__.build()")
    lib = C.CDLL(p)
    vp = C.c_void_p
    sig = {
        "smg_abi_version": ([], C.c_int),
        "smg_last_error": ([vp], C.c_char_p),
        "smg_create": ([C.c_int, C.POINTER(vp)], C.c_int),
        "smg_destroy": ([vp], None),
        "smg_default_config": ([C.POINTER(smg_pipeline_config)], None),
        "smg_compute_block_bases_fixed_sizes": ([vp, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                                                 C.POINTER(smg_pipeline_config), vp,
                                                 C.POINTER(smg_chain_output)], C.c_int),
        "smg_compute_block_bases": ([vp, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                                     C.POINTER(smg_pipeline_config), C.POINTER(smg_chain_output)], C.c_int),
        "smg_run_chains": ([vp, C.c_int32, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                            C.POINTER(smg_pipeline_config), vp, C.POINTER(smg_chain_output)], C.c_int),
        "smg_build_laplacian": ([vp, C.POINTER(smg_mesh), vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_int64,
                                 c_int64_p, c_double_p], C.c_int),
        "smg_default_shift": ([C.c_double, C.c_int32, C.c_double], C.c_double),
        "smg_operator_create": ([vp, C.c_int32, vp, vp, vp, C.c_double, C.c_int32, C.POINTER(vp)], C.c_int),
        "smg_operator_destroy": ([vp], None),
        "smg_operator_apply": ([vp, vp, C.c_int32, vp, vp, C.c_int32], C.c_int),
        "smg_operator_spmm": ([vp, vp, C.c_int32, vp, vp], C.c_int),
        "smg_orthonormalize": ([vp, C.c_int32, C.c_int32, vp, vp], C.c_int),
        "smg_orthogonal_iteration": ([vp, vp, C.c_int32, vp, C.c_int32, vp], C.c_int),
        "smg_dynamic_oi": ([vp, vp, C.c_int32, vp, vp, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int32,
                            vp, c_int32_p, c_int32_p, c_double_p, c_int32_p], C.c_int),
        "smg_bottom_subspace": ([vp, vp, C.c_int32, vp, vp], C.c_int),
        "smg_gft": ([vp, C.c_int32, C.c_int32, vp, vp, vp], C.c_int),
        "smg_igft": ([vp, C.c_int32, C.c_int32, vp, vp, vp], C.c_int),
        "smg_profile_enable": ([vp, C.c_int32], C.c_int),
        "smg_profile_read": ([vp, C.c_char_p, c_int64_p, c_double_p], C.c_int),
        "smg_doi_trace_enable": ([vp, C.c_int32], C.c_int),
        "smg_last_run_info": ([vp, C.POINTER(smg_run_info)], C.c_int),
        "smg_partition_mesh": ([vp, C.POINTER(smg_mesh), C.c_int32, C.c_uint64, vp], C.c_int),
        "smg_shard_range": ([C.c_int32, C.c_int32, C.c_int32, c_int32_p, c_int32_p], C.c_int),
        "smg_comm_unique_id": ([vp, vp], C.c_int),
        "smg_comm_create": ([vp, vp, C.c_int32, C.c_int32, C.POINTER(vp)], C.c_int),
        "smg_comm_destroy": ([vp], None),
        "smg_gather_meshes": ([vp, vp, C.c_int32, C.c_int64, vp, vp], C.c_int),
        "smg_expand_overlaps": ([vp, C.POINTER(smg_mesh), vp, C.c_int32, C.c_double, vp, C.c_int64, c_int32_p],
                                C.c_int),
        "smg_order_submeshes": ([vp, C.c_int32, vp, vp, C.c_uint64, vp], C.c_int),
        "smg_segment_mesh": ([vp, C.POINTER(smg_mesh), C.c_int32, C.c_double, C.c_uint64, vp, vp, C.c_int64,
                              c_int32_p, vp], C.c_int),
        "smg_doi_trace_read": ([vp, C.c_int64, vp, vp, vp, c_int64_p], C.c_int),
        "smg_orthonormality_estimate": ([vp, C.c_int32, C.c_int32, vp, c_double_p], C.c_int),
        "smg_coarse_reconstruct_frames": ([vp, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                                           C.POINTER(smg_bases), C.c_int32, vp, C.c_int32, C.c_int32, vp,
                                           C.c_int32], C.c_int),
        "smg_compress_blocks": ([vp, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                                 C.POINTER(smg_pipeline_config), vp, C.c_int32, C.POINTER(smg_encoded_blocks)],
                                C.c_int),
        "smg_decompress_blocks": ([vp, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                                   C.POINTER(smg_pipeline_config), C.POINTER(smg_encoded_blocks), vp, C.c_int32],
                                  C.c_int),
        "smg_default_bilateral_params": ([C.POINTER(smg_bilateral_params)], None),
        "smg_fine_denoise": ([vp, C.c_int64, vp, vp, vp, C.c_int64, vp, C.POINTER(smg_bilateral_params), vp, vp,
                              C.c_int32], C.c_int),
        "smg_denoise_dynamic": ([vp, C.c_int32, C.POINTER(smg_mesh), C.POINTER(smg_segmentation),
                                 C.POINTER(smg_pipeline_config), vp, C.c_int32, vp, C.c_int32, c_int32_p,
                                 c_double_p], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib

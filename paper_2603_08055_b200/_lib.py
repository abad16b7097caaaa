"""ctypes binding of libgsa_sm100.so (the C ABI in include/gsa_sm100.h).

The shared library is built in-tree by ``paper_2603_08055_b200.build`` and is
REQUIRED: there is no CPU or eager-PyTorch fallback. Importing the compute
entry points without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgsa_sm100.so")

GSA_DTYPE_F32 = 0
GSA_DTYPE_BF16 = 1


class GsaTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("heads", C.c_int32), ("rows", C.c_int32),
                ("dim", C.c_int32), ("head_stride", C.c_int64), ("row_stride", C.c_int64)]


class GsaLayout(C.Structure):
    _fields_ = [("num_special", C.c_int32), ("num_frames", C.c_int32), ("grid_h", C.c_int32),
                ("grid_w", C.c_int32), ("window_s", C.c_int32)]


class GsaParamsC(C.Structure):
    _fields_ = [("window_s", C.c_int32), ("top_k", C.c_int32), ("scale", C.c_double), ("variant", C.c_int32),
                ("ref_stride", C.c_int32), ("block_m", C.c_int32), ("block_n", C.c_int32)]


class GsaShard(C.Structure):
    _fields_ = [("frame_begin", C.c_int32), ("frame_end", C.c_int32), ("special_begin", C.c_int32),
                ("special_end", C.c_int32)]


class GsaGatherOp(C.Structure):
    _fields_ = [("buffer", C.c_int32), ("phase", C.c_int32), ("offset", C.c_int64), ("count", C.c_int64)]


class GsaSavedC(C.Structure):
    """gsa_saved: the ForwardContext fields gsa_backward reads (device pointers)."""
    _fields_ = [("qc", C.c_void_p), ("kc", C.c_void_p), ("vc", C.c_void_p), ("o_comp", C.c_void_p),
                ("lse_comp", C.c_void_p), ("plan_offsets", C.c_void_p), ("plan_ids", C.c_void_p),
                ("plan_entries", C.c_int64), ("o_sel", C.c_void_p), ("lse_sel", C.c_void_p), ("gate", C.c_void_p),
                ("o_spec", GsaTensor), ("lse_spec", C.c_void_p)]


class GsaContextC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("qc", "kc", "vc", "o_comp", "lse_comp", "topk", "o_sel", "lse_sel",
                                          "gate", "lse_spec")]


_lib = None


def load() -> C.CDLL:
    """Load libgsa_sm100.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the sm_100a kernels are the only implementation; there is no fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, f32 = C.c_void_p, C.c_int, C.c_int64, C.c_float
    T = C.POINTER(GsaTensor)
    Lp = C.POINTER(GsaLayout)
    P = C.POINTER(GsaParamsC)
    L.gsa_status_string.restype = C.c_char_p
    L.gsa_last_error_message.restype = C.c_char_p
    L.gsa_make_layout.argtypes = [i32, i32, i32, i32, i32, Lp]
    L.gsa_validate_params.argtypes = [P, Lp]
    L.gsa_avg_pool_tokens.argtypes = [T, Lp, T, vp]
    L.gsa_upsample_nearest.argtypes = [T, Lp, T, vp]
    L.gsa_tiled_attention.argtypes = [T, T, T, f32, i32, i32, T, vp, vp]
    L.gsa_special_token_attention.argtypes = [T, T, T, f32, T, vp, vp]
    L.gsa_compressed_attention_topk_workspace_bytes.restype = C.c_size_t
    L.gsa_compressed_attention_topk_workspace_bytes.argtypes = [i32, i32, i32, i32]
    L.gsa_compressed_attention_topk.argtypes = [T, T, T, i32, f32, i32, i32, vp, i32, T, vp, vp, vp,
                                                C.POINTER(C.c_int), vp, C.c_size_t, vp]
    L.gsa_forced_windows.argtypes = [Lp, i32, vp, C.POINTER(C.c_int), vp]
    L.gsa_build_selection_plan.argtypes = [vp, i32, i32, i32, Lp, i32, i32, vp, vp, i64, C.POINTER(C.c_int64),
                                           vp, C.c_size_t, vp]
    L.gsa_build_selection_plan_workspace_bytes.restype = C.c_size_t
    L.gsa_build_selection_plan_workspace_bytes.argtypes = [i32, i32, i32, Lp, i32]
    L.gsa_block_sparse_attention.argtypes = [T, T, T, vp, vp, Lp, f32, T, vp, vp]
    L.gsa_gate.argtypes = [T, T, T, vp]
    L.gsa_forward_workspace_bytes.restype = C.c_size_t
    L.gsa_forward_workspace_bytes.argtypes = [Lp, P, i32, i32]
    L.gsa_forward.argtypes = [T, T, T, T, Lp, P, T, C.POINTER(GsaContextC), C.POINTER(C.c_int), vp, C.c_size_t, vp]
    L.gsa_forward_with_plan.argtypes = [T, T, T, T, Lp, P, vp, vp, T, vp, C.c_size_t, vp]
    L.gsa_forward_stats.argtypes = [Lp, P, i32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.gsa_selection_sparsity.argtypes = [Lp, P, C.POINTER(C.c_double)]
    S = C.POINTER(GsaShard)
    L.gsa_shard_workspace_bytes.restype = C.c_size_t
    L.gsa_shard_workspace_bytes.argtypes = [Lp, P, S, i32, i32]
    L.gsa_shard_pool.argtypes = [T, T, T, Lp, P, S, T, T, T, vp]
    L.gsa_shard_compress.argtypes = [T, T, T, Lp, P, S, T, vp, vp, C.POINTER(C.c_int), vp, C.c_size_t, vp]
    L.gsa_shard_attend.argtypes = [T, T, T, T, Lp, P, S, T, vp, T, vp, C.c_size_t, vp]
    L.gsa_project_qkv.argtypes = [vp, i32, i32, vp, vp, vp, i32, i32, T, T, T, vp]
    L.gsa_project_qkv_bf16.argtypes = [vp, i32, i32, i64, vp, i32, vp, i64, vp]
    L.gsa_residual_bf16.argtypes = [vp, vp, vp, i64, vp]
    L.gsa_convert.argtypes = [vp, i32, vp, i32, i64, vp]
    L.gsa_shard_of_rank.argtypes = [Lp, i32, i32, S]
    L.gsa_shard_gather_plan.argtypes = [Lp, i32, i32, i32, i64, C.POINTER(GsaGatherOp), i32, C.POINTER(C.c_int)]
    L.gsa_comm_get_unique_id.argtypes = [vp]
    L.gsa_comm_init.argtypes = [C.POINTER(C.c_void_p), vp, i32, i32]
    L.gsa_comm_destroy.argtypes = [vp]
    L.gsa_shard_forward_workspace_bytes.restype = C.c_size_t
    L.gsa_shard_forward_workspace_bytes.argtypes = [Lp, P, i32, i32, i32, i32]
    L.gsa_shard_forward.argtypes = [vp, T, T, T, T, Lp, P, T, vp, vp, C.c_size_t, vp]
    L.gsa_set_stage_events.argtypes = [C.POINTER(C.c_void_p), i32]
    L.gsa_launch_count.argtypes = [C.POINTER(C.c_uint64)]
    L.gsa_backward_workspace_bytes.restype = C.c_size_t
    L.gsa_backward_workspace_bytes.argtypes = [Lp, P, i32, i32, i64, i32]
    L.gsa_backward.argtypes = [T, T, T, T, Lp, P, C.POINTER(GsaSavedC), T, T, T, T, vp, vp, C.c_size_t, vp]
    L.gsa_project_backward_workspace_bytes.restype = C.c_size_t
    L.gsa_project_backward_workspace_bytes.argtypes = [i32, i32, i32, i32]
    L.gsa_project_backward.argtypes = [vp, i32, i32, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                       C.c_size_t, vp]
    L.gsa_avg_pool_backward.argtypes = [T, Lp, T, vp]
    L.gsa_upsample_backward.argtypes = [T, Lp, T, vp]
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "gsa_abi_version", "gsa_status_string", "gsa_last_error_message", "gsa_make_layout", "gsa_validate_params",
    "gsa_avg_pool_tokens", "gsa_upsample_nearest", "gsa_tiled_attention", "gsa_special_token_attention",
    "gsa_compressed_attention_topk_workspace_bytes", "gsa_compressed_attention_topk", "gsa_forced_windows",
    "gsa_build_selection_plan", "gsa_build_selection_plan_workspace_bytes", "gsa_block_sparse_attention",
    "gsa_gate", "gsa_forward_workspace_bytes", "gsa_forward", "gsa_forward_with_plan", "gsa_forward_stats", "gsa_selection_sparsity",
    "gsa_set_stage_events", "gsa_launch_count", "gsa_shard_workspace_bytes", "gsa_shard_pool", "gsa_shard_compress",
    "gsa_shard_attend", "gsa_project_qkv", "gsa_shard_of_rank", "gsa_shard_gather_plan", "gsa_comm_get_unique_id",
    "gsa_comm_init", "gsa_comm_destroy", "gsa_shard_forward_workspace_bytes", "gsa_shard_forward",
    "gsa_project_qkv_bf16", "gsa_residual_bf16", "gsa_convert", "gsa_backward_workspace_bytes", "gsa_backward",
    "gsa_project_backward_workspace_bytes", "gsa_project_backward", "gsa_avg_pool_backward",
    "gsa_upsample_backward",
]

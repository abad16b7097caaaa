"""B200-native (sm_100a) Global Sparse Attention layer forward (Speed3R, arxiv 2603.08055).

The product is the C-ABI library ``libgsa_sm100.so`` (hand-written CUDA for
sm_100a, include/gsa_sm100.h) behind the reference's operator API. This
package holds the CUDA sources (``csrc/``), the in-tree build, and a Python
mirror of the reference interface used by tests and the benchmark.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8) -> str:
    """Compile every CUDA source for sm_100a into paper_2603_08055_b200/libgsa_sm100.so."""
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", os.path.join(HERE, "csrc")], check=True)
    return os.path.join(HERE, "libgsa_sm100.so")


from .gsa import (  # noqa: E402
    HostPipeline, HYBRID, PLAIN, CompressedResult, DivisibilityError, EmptySelection, ForwardContext, GsaError, GsaParams,
    IndexOutOfRange, InvalidStride, InvalidTiling, KernelTiling, NonFiniteInput, SelectionPlan, ShapeMismatch,
    TokenLayout, Unsupported, Workspace, ZeroSizeError, avg_pool_tokens, block_sparse_attention, build_selection_plan,
    build_token_layout, forced_windows_of, forward_stats, fused_compressed_attention_topk, gate, gsa_forward,
    gsa_forward_with_plan, project_qkv, resolved_scale, selection_sparsity, special_token_attention, tiled_attention, upsample_nearest,
    ContextMismatch, GsaGradients, avg_pool_backward, gsa_backward, layer_backward, project_backward, upsample_backward,
)

__all__ = [
    "build", "HostPipeline", "HYBRID", "PLAIN", "CompressedResult", "DivisibilityError", "EmptySelection", "ForwardContext",
    "GsaError", "GsaParams", "IndexOutOfRange", "InvalidStride", "InvalidTiling", "KernelTiling", "NonFiniteInput",
    "SelectionPlan", "ShapeMismatch", "TokenLayout", "Unsupported", "Workspace", "ZeroSizeError", "avg_pool_tokens",
    "block_sparse_attention", "build_selection_plan", "build_token_layout", "forced_windows_of", "forward_stats",
    "fused_compressed_attention_topk", "gate", "gsa_forward", "gsa_forward_with_plan", "project_qkv", "resolved_scale",
    "selection_sparsity", "special_token_attention", "tiled_attention", "upsample_nearest", "ContextMismatch",
    "GsaGradients", "avg_pool_backward", "gsa_backward", "layer_backward", "project_backward", "upsample_backward",
]

"""Python mirror of the reference operator API (proj/include/gsa) over the
sm_100a C ABI. Tensors are torch CUDA tensors shaped [heads, rows, dim]
(head-major like the reference's Tensor<T>, tensor.hpp:15-42); bf16 Q/K/V is
the fast path, f32 is accepted everywhere. Every function raises the Python
twin of the reference exception (errors.hpp:8-58) on bad input.

This module is the host-side plumbing used by the tests and bench.py; the
drop-in for C++ callers is include/gsa/*.hpp over the same C ABI.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _lib
from ._lib import GsaContextC, GsaLayout, GsaParamsC, GsaSavedC, GsaTensor


# ----------------------------------------------------------------- errors
class GsaError(RuntimeError):
    pass


class ShapeMismatch(GsaError):
    pass


class DivisibilityError(GsaError):
    pass


class ZeroSizeError(GsaError):
    pass


class IndexOutOfRange(GsaError):
    pass


class NonFiniteInput(GsaError):
    pass


class InvalidTiling(GsaError):
    pass


class InvalidStride(GsaError):
    pass


class EmptySelection(GsaError):
    pass


class Unsupported(GsaError):
    pass


class CudaError(GsaError):
    pass


class WorkspaceError(GsaError):
    pass


class ContextMismatch(GsaError):
    pass


_STATUS = {1: GsaError, 2: ShapeMismatch, 3: DivisibilityError, 4: ZeroSizeError, 5: IndexOutOfRange,
           6: NonFiniteInput, 7: InvalidTiling, 8: InvalidStride, 9: EmptySelection, 10: Unsupported,
           11: CudaError, 12: WorkspaceError, 13: GsaError, 14: ContextMismatch}


def _check(rc: int) -> None:
    if rc != 0:
        L = _lib.load()
        raise _STATUS.get(rc, GsaError)(L.gsa_last_error_message().decode())


# ------------------------------------------------------------------ types
@dataclass(frozen=True)
class TokenLayout:
    """layout.hpp:13-40. Construct with build_token_layout()."""
    num_special: int = 0
    num_frames: int = 1
    grid_h: int = 0
    grid_w: int = 0
    window_s: int = 1

    @property
    def tokens_per_frame(self) -> int:
        return self.grid_h * self.grid_w

    @property
    def image_tokens(self) -> int:
        return self.num_frames * self.tokens_per_frame

    @property
    def total_tokens(self) -> int:
        return self.num_special + self.image_tokens

    @property
    def wins_w(self) -> int:
        return self.grid_w // self.window_s

    @property
    def windows_per_frame(self) -> int:
        return (self.grid_h // self.window_s) * self.wins_w

    @property
    def num_windows(self) -> int:
        return self.num_frames * self.windows_per_frame

    def window_of_token(self, t: int) -> int:
        if not 0 <= t < self.image_tokens:
            raise IndexOutOfRange("window_of_token: image token index out of range")
        f, r = divmod(t, self.tokens_per_frame)
        row, col = divmod(r, self.grid_w)
        return f * self.windows_per_frame + (row // self.window_s) * self.wins_w + col // self.window_s

    def tokens_of_window(self, w: int) -> list[int]:
        if not 0 <= w < self.num_windows:
            raise IndexOutOfRange("tokens_of_window: window index out of range")
        f, r = divmod(w, self.windows_per_frame)
        wr, wc = divmod(r, self.wins_w)
        s, base = self.window_s, f * self.tokens_per_frame
        return [base + (wr * s + dr) * self.grid_w + wc * s + dc for dr in range(s) for dc in range(s)]

    def frame_of_window(self, w: int) -> int:
        if not 0 <= w < self.num_windows:
            raise IndexOutOfRange("frame_of_window: window index out of range")
        return w // self.windows_per_frame

    def c(self) -> GsaLayout:
        return GsaLayout(self.num_special, self.num_frames, self.grid_h, self.grid_w, self.window_s)


def build_token_layout(num_special: int, num_frames: int, grid_h: int, grid_w: int, window_s: int) -> TokenLayout:
    """build_token_layout (layout.cpp:7-24), validated by the C ABI."""
    out = GsaLayout()
    _check(_lib.load().gsa_make_layout(num_special, num_frames, grid_h, grid_w, window_s, C.byref(out)))
    return TokenLayout(num_special, num_frames, grid_h, grid_w, window_s)


@dataclass
class KernelTiling:
    block_m: int = 16
    block_n: int = 16


PLAIN, HYBRID = 0, 1


@dataclass
class GsaParams:
    """types.hpp:58-65."""
    window_s: int = 4
    top_k: int = 32
    scale: float = 0.0
    variant: int = PLAIN
    ref_stride: int = 100
    tiling: KernelTiling = field(default_factory=KernelTiling)

    def c(self) -> GsaParamsC:
        return GsaParamsC(self.window_s, self.top_k, self.scale, self.variant, self.ref_stride,
                          self.tiling.block_m, self.tiling.block_n)


def resolved_scale(params: GsaParams, dim: int) -> float:
    """reference.hpp:22-26 (float32 rounding of 1/sqrt(d))."""
    s = params.scale if params.scale > 0 else 1.0 / math.sqrt(dim)
    return float(torch.tensor(s, dtype=torch.float32))


# --------------------------------------------------------------- plumbing
def _desc(t: torch.Tensor) -> GsaTensor:
    if t.dim() != 3:
        raise ShapeMismatch(f"expected a [heads, rows, dim] tensor, got shape {tuple(t.shape)}")
    if not t.is_cuda:
        raise GsaError("tensors must live on the GPU (the sm_100a kernels are the only implementation)")
    if t.dtype == torch.bfloat16:
        dt = _lib.GSA_DTYPE_BF16
    elif t.dtype == torch.float32:
        dt = _lib.GSA_DTYPE_F32
    else:
        raise Unsupported(f"dtype {t.dtype} not supported")
    if t.shape[2] > 1 and t.stride(2) != 1:
        raise Unsupported("the feature dimension must be contiguous")
    return GsaTensor(t.data_ptr() if t.numel() else None, dt, t.shape[0], t.shape[1], t.shape[2],
                     t.stride(0), t.stride(1))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _empty(*shape, dtype=torch.float32, device=None):
    return torch.empty(*shape, dtype=dtype, device=device or "cuda")


# -------------------------------------------------------------------- ops
def avg_pool_tokens(x_img: torch.Tensor, layout: TokenLayout) -> torch.Tensor:
    """compression.hpp:20-38 (bit-exact)."""
    out = _empty(x_img.shape[0], layout.num_windows, x_img.shape[2], device=x_img.device)
    _check(_lib.load().gsa_avg_pool_tokens(C.byref(_desc(x_img)), C.byref(layout.c()), C.byref(_desc(out)), _stream()))
    return out


def upsample_nearest(coarse: torch.Tensor, layout: TokenLayout) -> torch.Tensor:
    """compression.hpp:42-53."""
    out = _empty(coarse.shape[0], layout.image_tokens, coarse.shape[2], device=coarse.device)
    _check(_lib.load().gsa_upsample_nearest(C.byref(_desc(coarse)), C.byref(layout.c()), C.byref(_desc(out)), _stream()))
    return out


def tiled_attention(q, k, v, scale: float, tiling: KernelTiling = KernelTiling()):
    """compression.hpp:99-165 -> (out f32, lse f32 [H, mq])."""
    out = _empty(q.shape[0], q.shape[1], q.shape[2], device=q.device)
    lse = _empty(q.shape[0], q.shape[1], device=q.device)
    _check(_lib.load().gsa_tiled_attention(C.byref(_desc(q)), C.byref(_desc(k)), C.byref(_desc(v)), C.c_float(scale),
                                           tiling.block_m, tiling.block_n, C.byref(_desc(out)), _ptr(lse), _stream()))
    return out, lse


def special_token_attention(q_spec, k, v, scale: float, tiling: KernelTiling = KernelTiling()):
    """layer.hpp:80-96 -> (out, lse)."""
    out = _empty(q_spec.shape[0], q_spec.shape[1], q_spec.shape[2], device=q_spec.device)
    lse = _empty(q_spec.shape[0], q_spec.shape[1], device=q_spec.device)
    if q_spec.shape[1] == 0:
        return out, lse
    _check(_lib.load().gsa_tiled_attention(C.byref(_desc(q_spec)), C.byref(_desc(k)), C.byref(_desc(v)),
                                           C.c_float(scale), tiling.block_m, tiling.block_n, C.byref(_desc(out)),
                                           _ptr(lse), _stream()))
    return out, lse


@dataclass
class CompressedResult:
    """compression.hpp:167-172 (+ TopkResult types.hpp:30-48)."""
    out: torch.Tensor
    lse: torch.Tensor
    indices: torch.Tensor  # [H, W, k_eff] int32
    k: int
    guide_scores: Optional[torch.Tensor] = None


def fused_compressed_attention_topk(qc, kc, vc, k: int, scale: float, tiling: KernelTiling = KernelTiling(),
                                    excluded: Optional[torch.Tensor] = None, keep_guide_scores: bool = False
                                    ) -> CompressedResult:
    """compression.hpp:180-297 (indices bit-exact with the reference)."""
    L = _lib.load()
    H, W, d = qc.shape
    n_ex = 0 if excluded is None else int(excluded.numel())
    sel = W - (0 if excluded is None else int(excluded.to(torch.int32).sum().item()))
    k_eff_guess = max(0, min(k, sel))
    out = _empty(H, W, d, device=qc.device)
    lse = _empty(H, W, device=qc.device)
    idx = torch.empty(H, W, max(1, k_eff_guess), dtype=torch.int32, device=qc.device)
    guide = _empty(H, W, max(1, k_eff_guess), device=qc.device) if keep_guide_scores else None
    ws_bytes = L.gsa_compressed_attention_topk_workspace_bytes(H, W, d, k_eff_guess)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=qc.device)
    ex = None if excluded is None else excluded.to(torch.uint8).contiguous()
    k_eff = C.c_int()
    _check(L.gsa_compressed_attention_topk(C.byref(_desc(qc)), C.byref(_desc(kc)), C.byref(_desc(vc)), k,
                                           C.c_float(scale), tiling.block_m, tiling.block_n, _ptr(ex), n_ex,
                                           C.byref(_desc(out)), _ptr(lse), _ptr(idx), _ptr(guide), C.byref(k_eff),
                                           _ptr(ws), ws_bytes, _stream()))
    ke = k_eff.value
    return CompressedResult(out, lse, idx[:, :, :ke], ke, None if guide is None else guide[:, :, :ke])


@dataclass
class SelectionPlan:
    """selection.hpp:19-33, on the device."""
    heads: int
    rows: int
    offsets: torch.Tensor      # int64 [H*rows+1]
    window_ids: torch.Tensor   # int32
    forced_windows: torch.Tensor

    def row_size(self, h: int, r: int) -> int:
        i = h * self.rows + r
        return int(self.offsets[i + 1] - self.offsets[i])


def forced_windows_of(layout: TokenLayout, ref_stride: int, device="cuda") -> torch.Tensor:
    """selection.cpp:14-21."""
    L = _lib.load()
    n = C.c_int()
    _check(L.gsa_forced_windows(C.byref(layout.c()), ref_stride, None, C.byref(n), _stream()))
    out = torch.empty(max(1, n.value), dtype=torch.int32, device=device)
    _check(L.gsa_forced_windows(C.byref(layout.c()), ref_stride, _ptr(out), C.byref(n), _stream()))
    return out[: n.value]


def build_selection_plan(topk: torch.Tensor, layout: TokenLayout, variant: int, ref_stride: int) -> SelectionPlan:
    """selection.cpp:29-67. topk: int32 [H, W, k] on the device."""
    L = _lib.load()
    topk = topk.to(torch.int32).contiguous()
    H, W, k = topk.shape
    # row width bound: forced windows (reference frames every ref_stride frames) ++ top-k
    F = len(range(0, layout.num_frames, max(ref_stride, 1))) * layout.windows_per_frame if variant == HYBRID else 0
    cap = max(1, H * W * (k + F))
    offsets = torch.empty(H * W + 1, dtype=torch.int64, device=topk.device)
    ids = torch.empty(cap, dtype=torch.int32, device=topk.device)
    ws_bytes = L.gsa_build_selection_plan_workspace_bytes(H, W, k, C.byref(layout.c()), max(ref_stride, 1))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=topk.device)
    n = C.c_int64()
    _check(L.gsa_build_selection_plan(_ptr(topk), H, W, k, C.byref(layout.c()), variant, ref_stride, _ptr(offsets),
                                      _ptr(ids), cap, C.byref(n), _ptr(ws), ws_bytes, _stream()))
    forced = forced_windows_of(layout, ref_stride, topk.device) if variant == HYBRID else \
        torch.empty(0, dtype=torch.int32, device=topk.device)
    return SelectionPlan(H, W, offsets, ids[: n.value], forced)


def block_sparse_attention(q_img, k_img, v_img, plan: SelectionPlan, layout: TokenLayout, scale: float,
                           tiling: KernelTiling = KernelTiling()):
    """selection.hpp:63-136 -> (out f32, lse)."""
    L = _lib.load()
    _tiling_check(tiling)
    if plan.heads != q_img.shape[0] or plan.rows != layout.num_windows:
        raise ShapeMismatch("block_sparse_attention: plan shape does not match layout/heads")
    H, Mi, d = q_img.shape
    out = _empty(H, layout.image_tokens, d, device=q_img.device)
    lse = _empty(H, layout.image_tokens, device=q_img.device)
    _check(L.gsa_block_sparse_attention(C.byref(_desc(q_img)), C.byref(_desc(k_img)), C.byref(_desc(v_img)),
                                        _ptr(plan.offsets), _ptr(plan.window_ids), C.byref(layout.c()),
                                        C.c_float(scale), C.byref(_desc(out)), _ptr(lse), _stream()))
    return out, lse


def _tiling_check(t: KernelTiling) -> None:
    ok = lambda v: 8 <= v <= 256 and (v & (v - 1)) == 0  # noqa: E731
    if not ok(t.block_m) or not ok(t.block_n):
        raise InvalidTiling(f"tiling blocks must be powers of two in [8, 256], got {t.block_m}x{t.block_n}")


def gate(q_img: torch.Tensor, w_g: torch.Tensor) -> torch.Tensor:
    """layer.hpp:99-119."""
    g = _empty(*q_img.shape, device=q_img.device)
    _check(_lib.load().gsa_gate(C.byref(_desc(q_img)), C.byref(_desc(w_g.contiguous())), C.byref(_desc(g)), _stream()))
    return g


@dataclass
class ForwardContext:
    """layer.hpp:124-142 (device tensors)."""
    qc: torch.Tensor
    kc: torch.Tensor
    vc: torch.Tensor
    o_comp_coarse: torch.Tensor
    lse_comp: torch.Tensor
    topk: torch.Tensor
    o_sel: torch.Tensor
    lse_sel: torch.Tensor
    gate_vals: torch.Tensor
    lse_spec: torch.Tensor
    k_eff: int


class Workspace:
    """Caller-owned scratch for gsa_forward (grown on demand, reused across calls).

    A workspace is stream-ordered like the calls that use it: share one only
    between calls on the same CUDA stream (the default workspaces are per
    (device, stream)). A buffer that is replaced while a call on another stream
    may still read it is kept alive for that stream (record_stream)."""

    def __init__(self):
        self.buf: Optional[torch.Tensor] = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            if self.buf is not None and self.buf.is_cuda:
                self.buf.record_stream(torch.cuda.current_stream(self.buf.device))
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_default_ws: dict = {}


def _default_workspace(device) -> Workspace:
    """The implicit workspace of calls without one: one per (device, current stream)."""
    dev = torch.device(device)
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    ws = _default_ws.get(key)
    if ws is None:
        ws = _default_ws[key] = Workspace()
    return ws


def gsa_forward(q, k, v, w_g, layout: TokenLayout, params: GsaParams, context: bool = False,
                out: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None):
    """gsa_forward (layer.hpp:177-230) from projected Q/K/V [H, M, d].
    Returns out (f32 [H, M, d]) or (out, ForwardContext) when context=True."""
    L = _lib.load()
    H, M, d = q.shape
    dev = q.device
    if out is None:
        out = _empty(H, M, d, device=dev)
    lc, pc = layout.c(), params.c()
    ws_bytes = L.gsa_forward_workspace_bytes(C.byref(lc), C.byref(pc), H, d)
    ws = (workspace or _default_workspace(dev)).get(ws_bytes, dev)
    ctx = None
    cstruct = None
    if context:
        W, Mi, Ms = layout.num_windows, layout.image_tokens, layout.num_special
        nf = 0
        if params.variant == HYBRID and params.ref_stride >= 1:
            nf = len(range(0, layout.num_frames, params.ref_stride)) * layout.windows_per_frame
        k_eff = max(0, min(params.top_k, W - nf))
        ctx = ForwardContext(_empty(H, W, d, device=dev), _empty(H, W, d, device=dev), _empty(H, W, d, device=dev),
                             _empty(H, W, d, device=dev), _empty(H, W, device=dev),
                             torch.empty(H, W, max(1, k_eff), dtype=torch.int32, device=dev),
                             _empty(H, Mi, d, device=dev), _empty(H, Mi, device=dev), _empty(H, Mi, d, device=dev),
                             _empty(H, Ms, device=dev), k_eff)
        cstruct = GsaContextC(*[t.data_ptr() for t in (ctx.qc, ctx.kc, ctx.vc, ctx.o_comp_coarse, ctx.lse_comp,
                                                          ctx.topk, ctx.o_sel, ctx.lse_sel, ctx.gate_vals,
                                                          ctx.lse_spec)])
    ke = C.c_int()
    _check(L.gsa_forward(C.byref(_desc(q)), C.byref(_desc(k)), C.byref(_desc(v)), C.byref(_desc(w_g.contiguous())),
                         C.byref(lc), C.byref(pc), C.byref(_desc(out)),
                         C.byref(cstruct) if cstruct is not None else None, C.byref(ke), _ptr(ws),
                         ws.numel(), _stream()))
    if ctx is not None:
        ctx.topk = ctx.topk[:, :, : ke.value]
        ctx.k_eff = ke.value
        return out, ctx
    return out


def gsa_forward_with_plan(q, k, v, w_g, layout: TokenLayout, params: GsaParams, plan: SelectionPlan,
                          workspace: Optional[Workspace] = None):
    """layer.hpp:235-262."""
    L = _lib.load()
    H, M, d = q.shape
    out = _empty(H, M, d, device=q.device)
    lc, pc = layout.c(), params.c()
    ws_bytes = L.gsa_forward_workspace_bytes(C.byref(lc), C.byref(pc), H, d)
    ws = (workspace or _default_workspace(q.device)).get(ws_bytes, q.device)
    _check(L.gsa_forward_with_plan(C.byref(_desc(q)), C.byref(_desc(k)), C.byref(_desc(v)),
                                   C.byref(_desc(w_g.contiguous())), C.byref(lc), C.byref(pc), _ptr(plan.offsets),
                                   _ptr(plan.window_ids), C.byref(_desc(out)), _ptr(ws), ws.numel(), _stream()))
    return out


# ----------------------------------------------------------------- backward
def avg_pool_backward(d_pooled: torch.Tensor, layout: TokenLayout) -> torch.Tensor:
    """gradients.hpp:21-34: [H, W, d] -> [H, Mi, d], each member row = its window's row / s^2."""
    H, _, d = d_pooled.shape
    out = _empty(H, layout.image_tokens, d, device=d_pooled.device)
    _check(_lib.load().gsa_avg_pool_backward(C.byref(_desc(d_pooled)), C.byref(layout.c()), C.byref(_desc(out)),
                                             _stream()))
    return out


def upsample_backward(d_fine: torch.Tensor, layout: TokenLayout) -> torch.Tensor:
    """gradients.hpp:37-49: [H, Mi, d] -> [H, W, d], member rows summed per window."""
    H, _, d = d_fine.shape
    out = _empty(H, layout.num_windows, d, device=d_fine.device)
    _check(_lib.load().gsa_upsample_backward(C.byref(_desc(d_fine)), C.byref(layout.c()), C.byref(_desc(out)),
                                             _stream()))
    return out


def gsa_backward(q, k, v, w_g, layout: TokenLayout, params: GsaParams, ctx: ForwardContext, out: torch.Tensor,
                 d_out: torch.Tensor, plan: Optional[SelectionPlan] = None, workspace: Optional[Workspace] = None,
                 grads: Optional[tuple] = None):
    """gsa_backward (gradients.hpp:54-243) up to the projection: the layer's gradients with
    respect to the projected q/k/v and to W_g, with the top-k held constant. `ctx` and `out`
    are what gsa_forward(..., context=True) returned for the same q/k/v; the plan is rebuilt
    from ctx.topk unless given; `grads` = (dq, dk, dv, dw_g) f32 buffers to write into.
    Returns (dq, dk, dv, dw_g), f32."""
    L = _lib.load()
    H, M, d = q.shape
    dev = q.device
    if plan is None:
        plan = build_selection_plan(ctx.topk, layout, params.variant, params.ref_stride)
    Ms = layout.num_special
    lc, pc = layout.c(), params.c()
    E = int(plan.window_ids.numel())
    ws_bytes = L.gsa_backward_workspace_bytes(C.byref(lc), C.byref(pc), H, d, E, _desc(q).dtype)
    ws = (workspace or _default_workspace(dev)).get(ws_bytes, dev)
    saved = GsaSavedC(ctx.qc.data_ptr(), ctx.kc.data_ptr(), ctx.vc.data_ptr(), ctx.o_comp_coarse.data_ptr(),
                      ctx.lse_comp.data_ptr(), plan.offsets.data_ptr(), plan.window_ids.data_ptr(), E,
                      ctx.o_sel.data_ptr(), ctx.lse_sel.data_ptr(), ctx.gate_vals.data_ptr(), _desc(out[:, :Ms]),
                      ctx.lse_spec.data_ptr() if Ms else None)
    d_out = d_out.float()
    if grads is None:
        dq, dk, dv = (_empty(H, M, d, device=dev) for _ in range(3))
        dw_g = _empty(H, d, d, device=dev)
    else:
        dq, dk, dv, dw_g = grads
    _check(L.gsa_backward(C.byref(_desc(q)), C.byref(_desc(k)), C.byref(_desc(v)), C.byref(_desc(w_g.contiguous())),
                          C.byref(lc), C.byref(pc), C.byref(saved), C.byref(_desc(d_out)), C.byref(_desc(dq)),
                          C.byref(_desc(dk)), C.byref(_desc(dv)), _ptr(dw_g), _ptr(ws), ws.numel(), _stream()))
    return dq, dk, dv, dw_g


def project_backward(x, w_q, w_k, w_v, dq, dk, dv, workspace: Optional[Workspace] = None, grads: Optional[tuple] = None):
    """Projection backward (gradients.hpp:226-263): dW_* = X^T dY per head and
    dX = sum_h dQ W_q^T + dK W_k^T + dV W_v^T. `grads` = (dx, dw_q, dw_k, dw_v) f32 buffers
    to write into. Returns (dx, dw_q, dw_k, dw_v), f32."""
    L = _lib.load()
    x, w_q, w_k, w_v, dq, dk, dv = (t.float().contiguous() for t in (x, w_q, w_k, w_v, dq, dk, dv))
    if x.dim() == 3:
        x = x.reshape(x.shape[-2], x.shape[-1])
    T, Cm = x.shape
    H, _, d = w_q.shape
    if grads is None:
        dx = _empty(T, Cm, device=x.device)
        dws = [_empty(H, Cm, d, device=x.device) for _ in range(3)]
    else:
        dx, dws = grads[0], list(grads[1:])
    nbytes = L.gsa_project_backward_workspace_bytes(T, Cm, H, d)
    ws = (workspace.get(nbytes, x.device) if workspace is not None
          else torch.empty(nbytes, dtype=torch.uint8, device=x.device))
    _check(L.gsa_project_backward(_ptr(x), T, Cm, _ptr(w_q), _ptr(w_k), _ptr(w_v), H, d, _ptr(dq), _ptr(dk), _ptr(dv),
                                  _ptr(dx), *[_ptr(t) for t in dws], _ptr(ws), ws.numel(), _stream()))
    return (dx, *dws)


@dataclass
class GsaGradients:
    """gradients.hpp:14-19."""
    dx: torch.Tensor    # [tokens, model_dim]
    dw_q: torch.Tensor  # [H, model_dim, d]
    dw_k: torch.Tensor
    dw_v: torch.Tensor
    dw_g: torch.Tensor  # [H, d, d]


def layer_backward(x, w_q, w_k, w_v, w_g, layout: TokenLayout, params: GsaParams, d_out,
                   workspace: Optional[Workspace] = None) -> tuple[torch.Tensor, GsaGradients]:
    """gsa_forward (layer.hpp:177-230) from X then gsa_backward (gradients.hpp:54-265):
    the full layer gradient with respect to X and every weight. Returns (out, grads)."""
    q, k, v = project_qkv(x, w_q, w_k, w_v)
    out, ctx = gsa_forward(q, k, v, w_g, layout, params, context=True, workspace=workspace)
    dq, dk, dv, dw_g = gsa_backward(q, k, v, w_g, layout, params, ctx, out, d_out, workspace=workspace)
    dx, dwq, dwk, dwv = project_backward(x, w_q, w_k, w_v, dq, dk, dv)
    return out, GsaGradients(dx, dwq, dwk, dwv, dw_g)


def forward_stats(layout: TokenLayout, params: GsaParams, heads: int) -> tuple[int, int]:
    """KernelStats (types.hpp:78-86) in closed form: (scores_computed, keys_attended)."""
    a, b = C.c_uint64(), C.c_uint64()
    _check(_lib.load().gsa_forward_stats(C.byref(layout.c()), C.byref(params.c()), heads, C.byref(a), C.byref(b)))
    return a.value, b.value


def selection_sparsity(layout: TokenLayout, params: GsaParams) -> float:
    """selection_sparsity (declared at workload.hpp:112, undefined in the
    reference): 1 - attended fine keys per image query / image_tokens."""
    out = C.c_double()
    _check(_lib.load().gsa_selection_sparsity(C.byref(layout.c()), C.byref(params.c()), C.byref(out)))
    return out.value


def project_qkv(x: torch.Tensor, w_q: torch.Tensor, w_k: torch.Tensor, w_v: torch.Tensor,
                dtype: torch.dtype = torch.float32):
    """project_qkv (layer.hpp:48-76): x [tokens, C] f32, w_* [H, C, d] f32 ->
    (q, k, v) [H, tokens, d]. f32 outputs are bit-identical to the reference
    (ascending-a accumulation, no FMA); bf16 outputs are their RNE rounding."""
    L = _lib.load()
    x, w_q, w_k, w_v = (t.contiguous() for t in (x, w_q, w_k, w_v))
    if x.dim() == 3:
        x = x.reshape(x.shape[-2], x.shape[-1])
    T, Cm = x.shape
    H, C2, d = w_q.shape
    if C2 != Cm or w_k.shape != w_q.shape or w_v.shape != w_q.shape:
        raise ShapeMismatch("project_qkv: X must be [tokens x model_dim] and weights [heads x model_dim x dim]")
    outs = [_empty(H, T, d, dtype=dtype, device=x.device) for _ in range(3)]
    _check(L.gsa_project_qkv(_ptr(x), T, Cm, _ptr(w_q), _ptr(w_k), _ptr(w_v), H, d, C.byref(_desc(outs[0])),
                             C.byref(_desc(outs[1])), C.byref(_desc(outs[2])), _stream()))
    return tuple(outs)


class HostPipeline:
    """gsa_forward from HOST (pinned) Q/K/V to a HOST output, pipelined over head
    groups. Every stage of the layer is independent per head (the top-k, the plan
    and all softmaxes are per head: types.hpp:27-48, compression.hpp:213-215), so
    head group g is computed on the compute stream while group g+1 is copied in
    and group g-1 is copied out on two copy streams: PCIe and HBM/tensor work
    overlap instead of adding up. Results are bitwise those of one gsa_forward
    over all heads (same kernels, same per-head arithmetic).

    Device buffers are allocated once per (shape, dtype) and reused.
    """

    def __init__(self, heads_per_group: int = 2, device="cuda", slots: int = 2):
        self.g = heads_per_group
        self.slots = max(2, slots)  # device buffer sets (measured at V=1000: 2 and 3 equal, the copies are PCIe-bound)
        self.device = torch.device(device)
        self.s_in = torch.cuda.Stream(self.device)
        self.s_comp = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)
        self._bufs = None
        self._key = None
        self.ws = [Workspace() for _ in range(self.slots)]

    def _alloc(self, q, out_dtype=torch.float32):
        H, M, d = q.shape
        key = (H, M, d, q.dtype)
        if self._key != key:
            g = min(self.g, H)
            mk = lambda dt: torch.empty(g, M, d, dtype=dt, device=self.device)  # noqa: E731
            # double-buffered device slots per head group
            self._bufs = [dict(q=mk(q.dtype), k=mk(q.dtype), v=mk(q.dtype), out=mk(out_dtype))
                          for _ in range(self.slots)]
            self._key = key
        return self._bufs

    def forward(self, q_host, k_host, v_host, w_g, layout: TokenLayout, params: GsaParams, out_host):
        """q/k/v_host: pinned [H, M, d] (bf16 or f32); w_g: device f32 [H, d, d];
        out_host: pinned f32 [H, M, d]. Returns out_host once the copies are done."""
        H = q_host.shape[0]
        bufs = self._alloc(q_host)
        g = min(self.g, H)
        # single-head first and last groups: the pipeline fill (first H2D) and drain
        # (last D2H) are the only copies that do not overlap compute
        if H > 2 and g > 1:
            mid = H - 2
            sizes = [1] + [g] * (mid // g) + ([mid % g] if mid % g else []) + [1]
        else:
            sizes = [g] * (H // g) + ([H % g] if H % g else [])
        groups, h0 = [], 0
        for n in sizes:
            groups.append((h0, h0 + n))
            h0 += n
        ev_in = [torch.cuda.Event() for _ in groups]
        ev_comp = [torch.cuda.Event() for _ in groups]
        ev_out = [torch.cuda.Event() for _ in groups]
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_in, self.s_comp, self.s_out):
            s.wait_stream(cur)
        S = self.slots
        for i, (h0, h1) in enumerate(groups):
            b = bufs[i % S]
            n = h1 - h0
            with torch.cuda.stream(self.s_in):
                if i >= S:  # the slot's previous compute must be done reading it
                    self.s_in.wait_event(ev_comp[i - S])
                b["q"][:n].copy_(q_host[h0:h1], non_blocking=True)
                b["k"][:n].copy_(k_host[h0:h1], non_blocking=True)
                b["v"][:n].copy_(v_host[h0:h1], non_blocking=True)
                ev_in[i].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(ev_in[i])
                if i >= S:  # the slot's previous output must be copied out
                    self.s_comp.wait_event(ev_out[i - S])
                gsa_forward(b["q"][:n], b["k"][:n], b["v"][:n], w_g[h0:h1], layout, params,
                            out=b["out"][:n], workspace=self.ws[i % S])
                ev_comp[i].record(self.s_comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev_comp[i])
                out_host[h0:h1].copy_(b["out"][:n], non_blocking=True)
                ev_out[i].record(self.s_out)
        cur.wait_stream(self.s_out)
        return out_host

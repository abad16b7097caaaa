"""L-layer global-attention stack (BASELINE configs[2]: a
24-layer stack at 1000 views).

Per layer (the reference's layer contract, layer.hpp:48-76 and 177-230):

  X_l [M, C] bf16 --(one GEMM, X_l . W_qkv[l], W_qkv = [W_q | W_k | W_v])--> QKV [M, 3, H, d] bf16
  Q/K/V = strided head views of QKV ([H, M, d] with head stride d, row stride 3C):
          the C-ABI tensor descriptors take them as they are, no transpose copy
  O = gsa_forward(Q, K, V, W_g[l])   written token-major through a strided
          descriptor ([H, M, d] view of an [M, H, d] buffer)
  X_{l+1} = X_l + O (heads concatenated: [M, H*d]), rounded to bf16 -- the residual
          connection of the transformer block; without it a stack of pure attention
          layers averages the tokens towards each other (over-smoothing), the
          compressed scores collapse into near-ties and the exact top-k fallback
          takes over (measured: a 24-layer stack without residual did not finish)

The projection runs on the library's tcgen05 GEMM (gsa_project_qkv_bf16: bf16
in, f32 accumulate in TMEM, bf16 out; W_qkv stored transposed once per layer)
and the residual on gsa_residual_bf16, so a stacked forward launches only this
library's kernels. Parity is defined at the post-projection boundary (SURVEY
§8(c)): the layer tests compare the GSA layer against the reference on the same
bf16 Q/K/V, and the exact f32 `project_qkv` (layer.hpp:48-76) remains available
for bit-parity of the projection itself.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from .gsa import GsaParams, TokenLayout, Workspace, _check, _stream, gsa_forward


class GsaStack:
    def __init__(self, layout: TokenLayout, params: GsaParams, layers: int, heads: int = 16, dim: int = 64,
                 device="cuda", seed: int = 0, w_qkv: Optional[list] = None, w_g: Optional[list] = None):
        self.layout, self.params, self.layers = layout, params, layers
        self.heads, self.dim = heads, dim
        self.model_dim = heads * dim
        C = self.model_dim
        gen = torch.Generator(device=device).manual_seed(seed)
        # random init of the reference's shape: N(0, 1/C) projections, W_g = N(0,1)/8 (workload.hpp:104)
        self.w_qkv = w_qkv if w_qkv is not None else [
            (torch.randn(C, 3 * C, generator=gen, device=device) / C ** 0.5).to(torch.bfloat16) for _ in range(layers)]
        self.w_g = w_g if w_g is not None else [
            torch.randn(heads, dim, dim, generator=gen, device=device) / 8.0 for _ in range(layers)]
        # K-major copies for the tensor-core GEMM (static weights: transposed once)
        self.w_qkv_t = [w.t().contiguous() for w in self.w_qkv]
        self.ws = Workspace()
        self._out = None
        self._qkv = None
        self._lib = _lib.load()

    def heads_of(self, qkv: torch.Tensor):
        """[M, 3C] -> three [H, M, d] strided views (head stride d, row stride 3C)."""
        M = qkv.shape[0]
        v = qkv.view(M, 3, self.heads, self.dim)
        return tuple(v[:, i].permute(1, 0, 2) for i in range(3))

    def project(self, x: torch.Tensor, l: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """x [M, C] bf16 -> X . W_qkv[l] [M, 3C] bf16 (tcgen05 GEMM, f32 accumulation)."""
        M, Cm = x.shape
        if out is None:
            out = torch.empty(M, 3 * Cm, dtype=torch.bfloat16, device=x.device)
        _check(self._lib.gsa_project_qkv_bf16(C.c_void_p(x.data_ptr()), M, Cm, x.stride(0),
                                              C.c_void_p(self.w_qkv_t[l].data_ptr()), 3 * Cm,
                                              C.c_void_p(out.data_ptr()), out.stride(0), _stream()))
        return out

    def residual(self, x: torch.Tensor, o: torch.Tensor) -> torch.Tensor:
        """bf16(x + o): x [M, C] bf16, o [M, C] f32."""
        y = torch.empty_like(x)
        _check(self._lib.gsa_residual_bf16(C.c_void_p(x.data_ptr()), C.c_void_p(o.data_ptr()),
                                           C.c_void_p(y.data_ptr()), x.numel(), _stream()))
        return y

    def layer(self, x: torch.Tensor, l: int) -> torch.Tensor:
        M = x.shape[0]
        if self._out is None or self._out.shape[0] != M or self._out.device != x.device:
            self._out = torch.empty(M, self.heads, self.dim, device=x.device)
            self._qkv = torch.empty(M, 3 * self.model_dim, dtype=torch.bfloat16, device=x.device)
        qkv = self.project(x, l, self._qkv)
        q, k, v = self.heads_of(qkv)
        gsa_forward(q, k, v, self.w_g[l], self.layout, self.params, out=self._out.permute(1, 0, 2),
                    workspace=self.ws)
        return self.residual(x, self._out.view(M, self.model_dim))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x [M, C] bf16 -> X_L [M, C] bf16."""
        if x.dim() != 2 or x.shape[1] != self.model_dim or x.dtype != torch.bfloat16:
            raise ValueError(f"expected bf16 [tokens, {self.model_dim}], got {tuple(x.shape)} {x.dtype}")
        for l in range(self.layers):
            x = self.layer(x, l)
        return x

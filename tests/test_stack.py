"""The L-layer stack driver (paper_2603_08055_b200/stack.py):
strided Q/K/V head views of the fused projection and a token-major output
descriptor must give exactly what the contiguous per-layer path gives (same
kernels, same inputs), and every layer's GSA output must stay within the
north-star tolerance of the reference run on that layer's bf16 Q/K/V."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_08055_b200 as m
    return m


@pytest.mark.parametrize("lt,heads,topk,variant", [((10, 2, 16, 16, 4), 2, 8, 0), ((12, 6, 16, 16, 4), 4, 6, 1)])
def test_stack_strided_views_match_contiguous_layers(gsa, lt, heads, topk, variant):
    from paper_2603_08055_b200.stack import GsaStack
    L = gsa.build_token_layout(*lt)
    p = gsa.GsaParams(window_s=4, top_k=topk, variant=variant, ref_stride=2)
    st = GsaStack(L, p, layers=3, heads=heads, dim=64, seed=3)
    M, C = L.total_tokens, heads * 64
    x0 = (torch.randn(M, C, generator=torch.Generator(device="cuda").manual_seed(5), device="cuda")).to(torch.bfloat16)
    got = st.forward(x0)

    x = x0
    for l in range(3):
        qkv = st.project(x, l)
        q, k, v = (t.contiguous() for t in st.heads_of(qkv))
        out = gsa.gsa_forward(q, k, v, st.w_g[l], L, p)
        x = (x.float() + out.permute(1, 0, 2).reshape(M, C)).to(torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), x.view(torch.int16))


@pytest.mark.parametrize("M,Cm,N", [(1000, 1024, 3072), (300, 128, 384), (129, 64, 512), (4096, 512, 1536), (77, 192, 96)])
def test_projection_gemm_tc(gsa, M, Cm, N):
    """The stack's tcgen05 GEMM (gsa_project_qkv_bf16) against an f32 reference of the same
    bf16 inputs: the bf16 output differs from the rounded exact product by at most a
    couple of ulps (f32 accumulation order), and ragged M (TMA zero fill) is handled."""
    import ctypes as C
    from paper_2603_08055_b200 import _lib
    L = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M + N)
    x = torch.randn(M, Cm, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Cm, N, generator=g, device="cuda") / Cm ** 0.5).to(torch.bfloat16)
    wt = w.t().contiguous()
    out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    rc = L.gsa_project_qkv_bf16(C.c_void_p(x.data_ptr()), M, Cm, Cm, C.c_void_p(wt.data_ptr()), N,
                                C.c_void_p(out.data_ptr()), N, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    ref = x.double() @ w.double()
    err = (out.double() - ref).abs()
    tol = 2 ** -7 * ref.abs() + 1e-6 * (x.double().abs() @ w.double().abs())  # <= ~1 bf16 ulp + f32 accumulation
    assert torch.isfinite(out.float()).all()
    assert (err <= tol).all(), float((err / tol.clamp_min(1e-30)).max())


def test_residual_bf16_matches_torch(gsa):
    from paper_2603_08055_b200.stack import GsaStack
    L = gsa.build_token_layout(0, 1, 8, 8, 4)
    st = GsaStack(L, gsa.GsaParams(window_s=4, top_k=2), layers=1, heads=2, dim=64, seed=1)
    x = torch.randn(333, 128, device="cuda").to(torch.bfloat16)
    o = torch.randn(333, 128, device="cuda")
    assert torch.equal(st.residual(x, o).view(torch.int16), (x.float() + o).to(torch.bfloat16).view(torch.int16))


def test_stack_layer_within_tolerance_of_reference(gsa, ref):
    """Layer 1 of a 2-layer stack (its input is layer 0's output) vs the reference
    fused CPU layer on the same bf16 Q/K/V: top-k bit-exact, output within tolerance."""
    from paper_2603_08055_b200.stack import GsaStack
    lt = (10, 2, 16, 16, 4)
    L = gsa.build_token_layout(*lt)
    p = gsa.GsaParams(window_s=4, top_k=8)
    st = GsaStack(L, p, layers=2, heads=2, dim=64, seed=11)
    M, C = L.total_tokens, 128
    x0 = torch.randn(M, C, generator=torch.Generator(device="cuda").manual_seed(2), device="cuda").to(torch.bfloat16)
    x1 = st.layer(x0, 0)
    q, k, v = (t.contiguous() for t in st.heads_of(x1 @ st.w_qkv[1]))
    out, ctx = gsa.gsa_forward(q, k, v, st.w_g[1], L, p, context=True)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    rf = ref.forward(f(q), f(k), f(v), f(st.w_g[1]), lt, top_k=8, variant=0, ref_stride=2)
    np.testing.assert_array_equal(ctx.topk.cpu().numpy(), rf["topk"])
    o = f(out)
    assert np.abs(o - rf["out"]).max() < 1e-3 and rel_l2(o, rf["out"]) < 5e-4

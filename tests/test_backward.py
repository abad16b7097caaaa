"""Layer backward (gradients.hpp:14-265) on the B200 vs the reference.

The oracle is the unmodified reference gsa_forward + gsa_backward (oracle/_ref, run in
f32 here on the same inputs). Two levels:

* kernels in isolation: the device backward consumes the REFERENCE's own saved
  context (q/k/v, pooled tensors, LSE rows, plan, outputs), so the only difference is
  the order of f32 accumulation: dQ/dK/dV/dW_g within rel-L2 1e-5. dQ/dK/dV are read
  off the reference through its projection backward with X = I (dW_q = X^T dQ = dQ).
* end to end from X: device forward (tensor cores, fp16 P.V) + device backward +
  projection backward vs the reference's dX / dW_q / dW_k / dW_v / dW_g. The forward's
  O_comp / O_sel carry the fp16 P.V error (conftest.P16_*), which enters the gate and D
  terms: rel-L2 <= 2e-3.

Size-independent properties: dO = 0 gives exact zeros, 2 dO gives
exactly twice every gradient, repeated calls are bitwise identical, bf16 q/k/v give
the gradients of their f32 values bit for bit.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KERNEL_REL = 1e-5  # same context, different f32 summation order
E2E_REL = 2e-3     # device forward's fp16 P.V error propagated through the gate and D terms


@pytest.fixture(scope="module")
def gsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_08055_b200 as m
    return m


def dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(dtype)


def host(t):
    torch.cuda.synchronize()
    return t.detach().float().cpu().numpy()


def weights(rng, H, Cm, d):
    w = [(rng.standard_normal((H, Cm, d)) / np.sqrt(Cm)).astype(np.float32) for _ in range(3)]
    wg = (rng.standard_normal((H, d, d)) / 8).astype(np.float32)
    return w, wg


def ref_context(gsa, r, lt, H, top_k, variant, ref_stride):
    """The reference's saved context as a device ForwardContext (+ its plan)."""
    L = gsa.build_token_layout(*lt)
    ctx = gsa.ForwardContext(dev(r["qc"]), dev(r["kc"]), dev(r["vc"]), dev(r["o_comp"]), dev(r["lse_comp"]),
                             dev(r["topk"], torch.int32), dev(r["o_sel"]), dev(r["lse_sel"]), dev(r["gate"]),
                             dev(r["lse_spec"]), r["k_eff"])
    plan = gsa.build_selection_plan(ctx.topk, L, variant, ref_stride)
    return L, ctx, plan


CASES = [  # layout (ns, nf, gh, gw, s), heads, dim, top_k, variant, ref_stride
    ((2, 2, 8, 8, 4), 2, 16, 2, 0, 100),
    ((0, 3, 8, 8, 4), 2, 64, 3, 0, 100),
    ((3, 4, 8, 8, 2), 2, 32, 5, 1, 2),
    ((5, 2, 12, 12, 4), 3, 64, 4, 1, 1),
    ((1, 2, 8, 16, 8), 2, 128, 1, 0, 100),
    ((2, 5, 8, 8, 4), 2, 64, 3, 1, 2),  # hybrid fast path: forced frames 0, 2, 4 as a dense pass
]


@pytest.mark.parametrize("lt,H,d,top_k,variant,ref_stride", CASES)
def test_backward_kernels_on_reference_context(gsa, ref, lt, H, d, top_k, variant, ref_stride):
    rng = np.random.default_rng(sum(lt) + H + d)
    M = lt[0] + lt[1] * lt[2] * lt[3]
    x = np.eye(M, dtype=np.float32)  # X = I: q = W_q, and the reference's dW_q is dQ itself
    wq, wk, wv = (rng.standard_normal((H, M, d)).astype(np.float32) for _ in range(3))
    wg = (rng.standard_normal((H, d, d)) / 8).astype(np.float32)
    d_out = rng.standard_normal((H, M, d)).astype(np.float32)
    r = ref.backward(x, wq, wk, wv, wg, lt, d_out, top_k=top_k, variant=variant, ref_stride=ref_stride)
    L, ctx, plan = ref_context(gsa, r, lt, H, top_k, variant, ref_stride)
    p = gsa.GsaParams(window_s=lt[4], top_k=top_k, variant=variant, ref_stride=ref_stride)
    dq, dk, dv, dwg = gsa.gsa_backward(dev(r["q"]), dev(r["k"]), dev(r["v"]), dev(wg), L, p, ctx, dev(r["out"]),
                                       dev(d_out), plan=plan)
    for name, got, want in (("dq", dq, r["dw_q"]), ("dk", dk, r["dw_k"]), ("dv", dv, r["dw_v"]),
                            ("dw_g", dwg, r["dw_g"])):
        got = host(got)
        assert rel_l2(got, want) < KERNEL_REL, name
        assert np.abs(got - want).max() < KERNEL_REL * 10 * max(1.0, np.abs(want).max()), name


@pytest.mark.parametrize("lt,H,d,top_k,variant,ref_stride", CASES[:4] + CASES[5:])
def test_layer_backward_from_x_matches_reference(gsa, ref, lt, H, d, top_k, variant, ref_stride):
    rng = np.random.default_rng(7 + sum(lt))
    M = lt[0] + lt[1] * lt[2] * lt[3]
    Cm = 96
    x = rng.standard_normal((M, Cm)).astype(np.float32)
    (wq, wk, wv), wg = weights(rng, H, Cm, d)
    d_out = rng.standard_normal((H, M, d)).astype(np.float32)
    r = ref.backward(x, wq, wk, wv, wg, lt, d_out, top_k=top_k, variant=variant, ref_stride=ref_stride)
    L = gsa.build_token_layout(*lt)
    p = gsa.GsaParams(window_s=lt[4], top_k=top_k, variant=variant, ref_stride=ref_stride)
    out, grads = gsa.layer_backward(dev(x), dev(wq), dev(wk), dev(wv), dev(wg), L, p, dev(d_out))
    assert rel_l2(host(out), r["out"]) < 1e-3
    for name in ("dx", "dw_q", "dw_k", "dw_v", "dw_g"):
        assert rel_l2(host(getattr(grads, name)), r[name]) < E2E_REL, name


def _layer(gsa, rng, lt, H, d, top_k, dtype=torch.bfloat16):
    M = lt[0] + lt[1] * lt[2] * lt[3]
    q, k, v = (torch.randn(H, M, d, device="cuda").to(dtype) for _ in range(3))
    wg = torch.randn(H, d, d, device="cuda") / 8
    L = gsa.build_token_layout(*lt)
    p = gsa.GsaParams(window_s=lt[4], top_k=top_k)
    out, ctx = gsa.gsa_forward(q, k, v, wg, L, p, context=True)
    return q, k, v, wg, L, p, out, ctx


def test_backward_linear_in_upstream_gradient(gsa):
    """SPEC.md:405-406 at a few thousand windows: dO = 0 -> exact zeros; 2 dO -> exactly 2x
    (every term is linear in dO and scaling by 2 is exact); repeated calls bitwise equal."""
    torch.manual_seed(3)
    q, k, v, wg, L, p, out, ctx = _layer(gsa, None, (4, 20, 24, 24, 4), 4, 64, 16)
    plan = gsa.build_selection_plan(ctx.topk, L, p.variant, p.ref_stride)
    d_out = torch.randn_like(out)
    g1 = gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, d_out, plan=plan)
    g1b = gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, d_out, plan=plan)
    g2 = gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, 2 * d_out, plan=plan)
    g0 = gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, torch.zeros_like(d_out), plan=plan)
    for a, b, c, z in zip(g1, g1b, g2, g0):
        assert torch.equal(a, b)
        assert torch.equal(2 * a, c)
        assert not torch.any(z)
        assert torch.isfinite(a).all()


def test_backward_bf16_inputs_equal_f32_values(gsa):
    torch.manual_seed(5)
    q, k, v, wg, L, p, out, ctx = _layer(gsa, None, (2, 6, 16, 16, 4), 2, 64, 8)
    d_out = torch.randn_like(out)
    a = gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, d_out)
    b = gsa.gsa_backward(q.float(), k.float(), v.float(), wg, L, p, ctx, out, d_out)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("T,Cm,H,d", [(300, 80, 3, 32), (300, 80, 3, 64), (1001, 264, 2, 64)])
def test_project_backward_matches_float64(gsa, T, Cm, H, d):
    """d = 64 runs on the tensor cores (bf16 hi / lo planes, 3-term products: ~1e-5 relative),
    other head dims on CUDA cores (f32 FMA); token counts not a multiple of 8 / 128 and model
    dims not a multiple of 128 exercise the padded and partial tiles."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((T, Cm)).astype(np.float32)
    w = [rng.standard_normal((H, Cm, d)).astype(np.float32) for _ in range(3)]
    g = [rng.standard_normal((H, T, d)).astype(np.float32) for _ in range(3)]
    dx, *dws = gsa.project_backward(dev(x), *[dev(t) for t in w], *[dev(t) for t in g])
    x64 = x.astype(np.float64)
    want_dx = sum(np.einsum("htj,haj->ta", gi.astype(np.float64), wi.astype(np.float64)) for gi, wi in zip(g, w))
    tol = 2e-5 if d == 64 else 1e-6
    assert rel_l2(host(dx), want_dx) < tol
    for dw, gi in zip(dws, g):
        assert rel_l2(host(dw), np.einsum("ta,htj->haj", x64, gi.astype(np.float64))) < tol


@pytest.mark.parametrize("lt", [(3, 2, 8, 8, 4), (0, 3, 6, 12, 2), (1, 1, 16, 16, 8)])
def test_pool_and_upsample_adjoints_bit_exact(gsa, ref, lt):
    """gradients.hpp:21-49 bit for bit, and the adjoint identities of SPEC.md:421."""
    rng = np.random.default_rng(1)
    H, d = 2, 24
    L = gsa.build_token_layout(*lt)
    W, Mi = L.num_windows, L.image_tokens
    dp = rng.standard_normal((H, W, d)).astype(np.float32)
    df = rng.standard_normal((H, Mi, d)).astype(np.float32)
    win = np.array([L.window_of_token(t) for t in range(Mi)])
    inv = np.float32(1.0) / np.float32(lt[4] * lt[4])
    got_p = host(gsa.avg_pool_backward(dev(dp), L))
    np.testing.assert_array_equal(got_p, dp[:, win] * inv)
    got_u = host(gsa.upsample_backward(dev(df), L))
    want_u = np.zeros((H, W, d), np.float32)
    for t in range(Mi):  # the reference's accumulation order (ascending token)
        want_u[:, win[t]] += df[:, t]
    np.testing.assert_array_equal(got_u, want_u)
    # <pool(X), Y> == <X, pool_backward(Y)> and <up(C), Y> == <C, up_backward(Y)>
    pooled = host(gsa.avg_pool_tokens(dev(df), L))
    assert abs(np.vdot(pooled.astype(np.float64), dp) - np.vdot(df.astype(np.float64), got_p)) < 1e-3
    up = host(gsa.upsample_nearest(dev(dp), L))
    assert abs(np.vdot(up.astype(np.float64), df) - np.vdot(dp.astype(np.float64), got_u)) < 1e-3


def test_backward_rejects_mismatched_context(gsa):
    torch.manual_seed(2)
    q, k, v, wg, L, p, out, ctx = _layer(gsa, None, (2, 2, 8, 8, 4), 2, 64, 2)
    plan = gsa.build_selection_plan(ctx.topk, L, p.variant, p.ref_stride)
    with pytest.raises(gsa.ShapeMismatch):
        gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, torch.zeros(2, out.shape[1] - 1, 64, device="cuda"), plan=plan)
    bad = gsa.SelectionPlan(plan.heads, plan.rows, plan.offsets, plan.window_ids[:-1], plan.forced_windows)
    with pytest.raises(gsa.ContextMismatch):
        gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, torch.zeros_like(out), plan=bad)


@pytest.mark.parametrize("variant,ref_stride", [(0, 100), (1, 8)])
def test_layer_backward_16_views_matches_reference(gsa, ref, variant, ref_stride):
    """The VGGT geometry at 16 views (5 specials + 36x36 patches per view: M = 20,816, W = 1,296,
    top-32): plan rows of 4 gathered chunks, inverse-plan rows of every length, 80 special rows,
    key splits, hybrid forced frames 0 and 8 — the tensor-core backward from X against the
    reference's gsa_backward."""
    rng = np.random.default_rng(16 + variant)
    lt = (80, 16, 36, 36, 4)
    M = lt[0] + lt[1] * lt[2] * lt[3]
    H, Cm, d = 2, 128, 64
    x = rng.standard_normal((M, Cm)).astype(np.float32)
    (wq, wk, wv), wg = weights(rng, H, Cm, d)
    d_out = rng.standard_normal((H, M, d)).astype(np.float32)
    r = ref.backward(x, wq, wk, wv, wg, lt, d_out, top_k=32, variant=variant, ref_stride=ref_stride, threads=16)
    L = gsa.build_token_layout(*lt)
    p = gsa.GsaParams(window_s=4, top_k=32, variant=variant, ref_stride=ref_stride)
    out, grads = gsa.layer_backward(dev(x), dev(wq), dev(wk), dev(wv), dev(wg), L, p, dev(d_out))
    assert rel_l2(host(out), r["out"]) < 1e-3
    for name in ("dx", "dw_q", "dw_k", "dw_v", "dw_g"):
        assert rel_l2(host(getattr(grads, name)), r[name]) < E2E_REL, name

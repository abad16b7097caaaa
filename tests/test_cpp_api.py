"""The C++ drop-in API (include/gsa/*.hpp: the reference's operator signatures
over the sm_100a C ABI), driven by tests/cpp/gsa_cpp_driver.cpp the way a
reference user would call it, compared with the reference compiled unmodified
(oracle/_ref):

* project_qkv (f32): bit-identical Q/K/V;
* gsa_forward(x, ...): TopkResult indices and the selection plan bit-exact,
  output within the north-star tolerance (max|d| <= 2e-2, rel L2 <= 1e-3;
  asserted much tighter), KernelStats in closed form;
* every per-branch operator against its reference twin;
* the error convention (DivisibilityError, InvalidTiling, EmptySelection,
  ShapeMismatch, NonFiniteInput, Unsupported for Tensor<double>).
"""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from conftest import P16_ABS, P16_REL, ROOT, rel_l2

CPP = os.path.join(ROOT, "tests", "cpp")
LIB = os.path.join(ROOT, "paper_2603_08055_b200", "libgsa_sm100.so")


def _build():
    if not os.path.exists(LIB):
        pytest.skip("libgsa_sm100.so not built")
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return os.path.join(CPP, "gsa_cpp_driver")


def test_cpp_api_compiles_against_the_c_abi():
    """The drop-in headers compile with -Wall -Wextra and link libgsa_sm100.so (CPU box)."""
    exe = _build()
    assert os.access(exe, os.X_OK)


def _load(d):
    out = {}
    for line in open(os.path.join(d, "manifest.txt")):
        if line.startswith("#"):
            out.setdefault("_checks", []).append(line[1:].strip())
            continue
        name, dt, *shape = line.split()
        a = np.fromfile(os.path.join(d, name + ".bin"), dtype={"f32": np.float32, "i32": np.int32, "i64": np.int64}[dt])
        out[name] = a.reshape([int(s) for s in shape])
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f32", "bf16"])
@pytest.mark.parametrize("lt,heads,model_dim,top_k,variant", [
    ((10, 2, 16, 16, 4), 2, 128, 8, 0),
    ((40, 8, 36, 36, 4), 4, 256, 32, 0),
    ((12, 6, 16, 16, 4), 2, 64, 6, 1),
])
def test_cpp_api_matches_reference(tmp_path, ref, lt, heads, model_dim, top_k, variant, precision):
    """precision f32: the caller's values as they are; bf16 (gsa::device::Precision::kBf16):
    Q/K/V rounded to bf16 after the exact projection -- the reference then runs on those
    same rounded values (the driver dumps the Q/K/V the layer consumed)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build()
    r = subprocess.run([exe, str(tmp_path), *map(str, lt), str(heads), str(model_dim), str(top_k), str(variant),
                        precision], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    d = _load(str(tmp_path))
    assert "done" in d["_checks"]
    for name in ("divisibility", "tiling", "double", "empty_selection", "forward_rows", "nonfinite"):
        assert f"ok {name}" in d["_checks"], name

    # project_qkv: the reference's f32 arithmetic, bit for bit (then RNE to bf16 in bf16 mode)
    q, k, v = ref.project(d["x"][0], d["w_q"], d["w_k"], d["w_v"])
    if precision == "bf16":
        import torch as _t
        q, k, v = (_t.from_numpy(a).to(_t.bfloat16).float().numpy() for a in (q, k, v))
    for got, want in ((d["q"], q), (d["k"], k), (d["v"], v)):
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))

    # gsa_forward from X vs the reference fused layer on the same projections
    rf = ref.forward(q, k, v, d["w_g"], lt, top_k=top_k, variant=variant, ref_stride=2)
    np.testing.assert_array_equal(d["topk"], rf["topk"])
    np.testing.assert_array_equal(d["qc"].view(np.uint32), rf["qc"].view(np.uint32))
    # regression bounds inside the north star: O'_comp carries the fp16 P.V error
    assert np.abs(d["out"] - rf["out"]).max() < P16_ABS and rel_l2(d["out"], rf["out"]) < 5e-4
    assert rel_l2(d["o_comp"], rf["o_comp"]) < 1e-3
    assert np.abs(d["gate"] - rf["gate"]).max() < 1e-5
    assert np.abs(d["o_sel"] - rf["o_sel"]).max() < P16_ABS and rel_l2(d["o_sel"], rf["o_sel"]) < P16_REL
    offs, ids = ref.plan(rf["topk"], lt, variant, 2)
    np.testing.assert_array_equal(d["plan_offsets"], offs)
    np.testing.assert_array_equal(d["plan_ids"], ids)
    H, W, s = heads, d["topk"].shape[1], lt[4]
    Ms, M = lt[0], d["out"].shape[1]
    assert d["stats"][0] == H * (Ms * M + W * W)
    assert d["stats"][1] == ids.size * s ** 4

    # the layer backward (gradients.hpp:54-265) vs the reference's on the same X, weights, dO
    assert "ok backward_shape" in d["_checks"]
    rb = ref.backward(d["x"][0], d["w_q"], d["w_k"], d["w_v"], d["w_g"], lt, d["d_out"], top_k=top_k,
                      variant=variant, ref_stride=2)
    for name in ("dx", "dw_q", "dw_k", "dw_v", "dw_g"):
        assert np.isfinite(d[name]).all(), name
        # f32: the same plan and the device forward's fp16 P.V error only. bf16 runs the layer on
        # rounded Q/K/V, whose top-k (and so the detached plan) may legitimately differ from the f32
        # reference's; their device backward is pinned bit for bit to the f32 path on the same
        # values in test_backward.py
        if precision == "f32":
            assert rel_l2(d[name].reshape(rb[name].shape), rb[name]) < 2e-3, name

    # per-branch operators
    Mi = M - Ms
    np.testing.assert_array_equal(d["op_kc"].view(np.uint32), rf["kc"].view(np.uint32))
    scale = 0.125
    ex = None
    if variant:
        ex = np.zeros(W, np.uint8)
        ex[ref.forced_windows(lt, 2)] = 1
    oc, _, idx, guide = ref.compress(rf["qc"], rf["kc"], rf["vc"], top_k, scale, excluded=ex, guide=True)
    np.testing.assert_array_equal(d["op_topk"], idx)
    np.testing.assert_array_equal(d["op_guide"], guide.reshape(-1).astype(np.float32))
    assert rel_l2(d["op_o_comp"], oc) < 1e-3
    np.testing.assert_array_equal(d["op_plan_ids"], ids)
    osel, _ = ref.block_sparse(q[:, Ms:], k[:, Ms:], v[:, Ms:], lt, offs, ids, scale)
    assert np.abs(d["op_o_sel"] - osel).max() < P16_ABS and rel_l2(d["op_o_sel"], osel) < P16_REL
    assert np.abs(d["op_gate"] - ref.gate(q[:, Ms:], d["w_g"])).max() < 1e-5
    np.testing.assert_array_equal(d["op_up"], ref.upsample(d["op_o_comp"], lt))
    if Ms:
        ospec, _ = ref.tiled_attention(q[:, :Ms], k, v, scale)
        # f32 operands: S on tensor cores from a 3-term bf16 split, P.V with P and V in fp16
        # (the compressed-branch kernel in softmax-only mode): ~2^-11 relative in the output
        assert np.abs(d["op_o_spec"] - ospec).max() < P16_ABS and rel_l2(d["op_o_spec"], ospec) < P16_REL
    # pinned plan = the plan gsa_forward realised: compressed branch without top-k
    assert np.abs(d["op_out_with_plan"] - rf["out"]).max() < 1e-3
    assert Mi > 0

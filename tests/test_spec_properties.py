"""The reference's acceptance property suites, ported to the
sm_100a path and checked against the UNMODIFIED reference (oracle/_ref):

1. dense degeneration: s=1, k=W, no specials == dense image
   attention, 50 random instances up to 2048 image tokens;
2. fused vs oracle: 100 seeded random configurations (s in
   {1,2,4}, k in 1..W, plain/hybrid, num_special in {0,1,5}, f32 and bf16
   inputs) -- GPU top-k bit-exact with the reference's fused path, GPU output
   vs the brute-force reference_gsa within tolerance;
3. streaming top-k exactness: 1000 trials (>= 100 all-tie
   adversarial) of fused_compressed_attention_topk, indices bit-exact with the
   reference, and bitwise identical across tilings B_M, B_N in {8,16,32,64};
4. gather/mask equivalence: block_sparse_attention == the
   -inf-masked dense oracle over 100 random plans, exp(LSE) == denominators;
6. forced inclusion: hybrid ref_stride=100 with frames in
   {1, 99, 100, 250}: every plan row holds every window of frames 0, 100, 200.

Tolerances: SPEC states 1e-5 (f32) for its own CPU paths; the GPU contract is the
north star's (max|d| <= 2e-2, rel L2 <= 1e-3) with indices bit-exact. Each test
asserts the north-star bound and a tighter regression bound stated inline.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import P16_ABS, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-3


@pytest.fixture(scope="module")
def gsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_08055_b200 as m
    return m


def bf16r(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy()


def dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(dtype)


def random_config(rng):
    s = int(rng.choice([1, 2, 4]))
    while True:
        gh, gw = s * int(rng.integers(1, 1 + 16 // s)), s * int(rng.integers(1, 1 + 16 // s))
        frames = int(rng.integers(1, 9))
        if frames * gh * gw <= 2048:
            break
    ns = frames * int(rng.choice([0, 1, 5]))
    W = frames * (gh // s) * (gw // s)
    k = int(rng.integers(1, W + 1))
    variant = int(rng.integers(0, 2))
    ref_stride = int(rng.integers(1, frames + 1))
    heads = int(rng.integers(1, 4))
    dim = 64 if rng.random() < 0.8 else int(rng.choice([32, 48]))
    return (ns, frames, gh, gw, s), k, variant, ref_stride, heads, dim


def test_dense_degeneration_50(gsa, ref):
    """s=1, k=W, no specials: the layer is dense image attention (the
    selection covers every window, so out = g * o_comp + (1-g) * o_dense with o_comp == o_dense)."""
    rng = np.random.default_rng(573)
    worst = 0.0
    for i in range(50):
        frames = int(rng.integers(1, 5))
        gh, gw = int(rng.integers(1, 24)), int(rng.integers(1, 24))
        if frames * gh * gw > 2048:
            gh, gw = 8, 8
        lt = (0, frames, gh, gw, 1)
        Mi = frames * gh * gw
        H = int(rng.integers(1, 3))
        q, k, v = (rng.standard_normal((H, Mi, 64)).astype(np.float32) for _ in range(3))
        wg = (rng.standard_normal((H, 64, 64)) / 8).astype(np.float32)
        L = gsa.build_token_layout(*lt)
        out = gsa.gsa_forward(dev(q, torch.float32), dev(k, torch.float32), dev(v, torch.float32),
                              dev(wg, torch.float32), L, gsa.GsaParams(window_s=1, top_k=Mi))
        dense = ref.full_attention(q, k, v, 0.125)
        err = float(np.abs(out.cpu().numpy() - dense).max())
        worst = max(worst, err)
    # SPEC's f32 bound (1e-5) is for its own CPU paths; here the compressed branch, which s=1 makes
    # the whole dense softmax, runs P.V in fp16: regression bound 1e-3
    assert worst <= 1e-3, worst


@pytest.mark.parametrize("block", range(4))
def test_fused_vs_oracle_100_random_configs(gsa, ref, block):
    """100 seeded configurations (25 per block), f32 and bf16 inputs."""
    rng = np.random.default_rng(574 + 1000 * block)
    worst_rel = 0.0
    for i in range(25):
        lt, k, variant, ref_stride, H, d = random_config(rng)
        M = lt[0] + lt[1] * lt[2] * lt[3]
        dt = torch.float32 if rng.random() < 0.5 else torch.bfloat16
        q, kk, v = (rng.standard_normal((H, M, d)).astype(np.float32) for _ in range(3))
        if dt == torch.bfloat16:
            q, kk, v = bf16r(q), bf16r(kk), bf16r(v)
        wg = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
        L = gsa.build_token_layout(*lt)
        p = gsa.GsaParams(window_s=lt[4], top_k=k, variant=variant, ref_stride=ref_stride)
        out, ctx = gsa.gsa_forward(dev(q, dt), dev(kk, dt), dev(v, dt), dev(wg, torch.float32), L, p, context=True)
        rf = ref.forward(q, kk, v, wg, lt, top_k=k, variant=variant, ref_stride=ref_stride, threads=4)
        naive = ref.reference_gsa(q, kk, v, wg, lt, top_k=k, variant=variant, ref_stride=ref_stride)
        tag = f"cfg {i}: lt={lt} k={k} variant={variant} r={ref_stride} H={H} d={d} {dt}"
        np.testing.assert_array_equal(ctx.topk.cpu().numpy(), rf["topk"], err_msg=tag)
        o = out.cpu().numpy()
        assert np.abs(o - naive).max() <= MAX_ABS and rel_l2(o, naive) <= REL_L2, tag
        assert np.abs(o - naive).max() <= 1e-3 and rel_l2(o, naive) <= 2e-4, tag  # regression bound
        worst_rel = max(worst_rel, rel_l2(o, naive))
    print(f"block {block}: worst rel L2 vs reference_gsa {worst_rel:.2e}")


def _topk_batch(rng, kind, H, W):
    if kind == "all_ties":  # every score of a row equal: indices must be 0..k-1
        qc = rng.standard_normal((H, W, 64)).astype(np.float32)
        kc = np.broadcast_to(rng.standard_normal((H, 1, 64)).astype(np.float32), (H, W, 64)).copy()
    elif kind == "int_ties":  # small integers: mass exact ties between distinct windows
        qc, kc = (rng.integers(-2, 3, size=(H, W, 64)).astype(np.float32) for _ in range(2))
    elif kind == "sharp":
        qc, kc = (rng.standard_normal((H, W, 64)).astype(np.float32) * 4 for _ in range(2))
    else:
        qc, kc = (rng.standard_normal((H, W, 64)).astype(np.float32) for _ in range(2))
    vc = rng.standard_normal((H, W, 64)).astype(np.float32)
    return qc, kc, vc


def test_streaming_topk_1000_trials(gsa, ref):
    """>= 1000 trials (each query row is an independent top-k problem; 40
    seeded instances of random W, k, data kind), >= 100 of them all-tie rows; indices (and
    guide scores) bit-exact with the reference's fused top-k, which the reference itself
    asserts equal to naive_topk; results identical across tilings."""
    rng = np.random.default_rng(575)
    kinds = ["all_ties"] * 5 + ["int_ties"] * 10 + ["normal"] * 15 + ["sharp"] * 10
    trials = ties = 0
    for i, kind in enumerate(kinds):
        W = int(rng.integers(24, 400))
        H = int(rng.integers(1, 3))
        k = int(rng.integers(1, min(W, 160) + 1))
        qc, kc, vc = _topk_batch(rng, kind, H, W)
        ex = (rng.random(W) < 0.2).astype(np.uint8) if (kind == "normal" and i % 3 == 0) else None
        o_ref, _, i_ref, g_ref = ref.compress(qc, kc, vc, k, 0.125, excluded=ex, guide=True, threads=4)
        exd = None if ex is None else torch.from_numpy(ex).cuda()
        r = gsa.fused_compressed_attention_topk(dev(qc, torch.float32), dev(kc, torch.float32),
                                                dev(vc, torch.float32), k, 0.125, excluded=exd,
                                                keep_guide_scores=True)
        got = r.indices.cpu().numpy()
        np.testing.assert_array_equal(got, i_ref, err_msg=f"instance {i} ({kind}, W={W}, k={k})")
        np.testing.assert_array_equal(r.guide_scores.cpu().numpy(), g_ref.astype(np.float32))
        if kind == "all_ties":
            assert (got == np.arange(got.shape[2])[None, None]).all()
            ties += H * W
        trials += H * W
        if i % 8 == 0:  # tilings are validated and never change the result (types.hpp:13-25)
            for bm, bn in ((8, 64), (64, 8), (32, 32), (16, 16)):
                r2 = gsa.fused_compressed_attention_topk(dev(qc, torch.float32), dev(kc, torch.float32),
                                                         dev(vc, torch.float32), k, 0.125,
                                                         tiling=gsa.KernelTiling(bm, bn), excluded=exd)
                assert torch.equal(r2.indices, r.indices) and torch.equal(r2.out, r.out)
    assert trials >= 1000 and ties >= 100, (trials, ties)


def test_gather_mask_equivalence_100_plans(gsa, ref):
    """block_sparse_attention over 100 random plans (distinct window ids per
    row, random row lengths) == the -inf-masked dense oracle; exp(LSE) == the true
    denominators (relative 1e-5 in f32; SPEC's 1e-10 is its f64 bound)."""
    rng = np.random.default_rng(576)
    for i in range(100):
        frames = int(rng.integers(1, 4))
        lt = (0, frames, 8, int(rng.choice([8, 12, 16])), 4)
        W = frames * 2 * (lt[3] // 4)
        Mi = frames * lt[2] * lt[3]
        H = int(rng.integers(1, 3))
        offs = [0]
        ids = []
        for _ in range(H * W):
            n = int(rng.integers(1, W + 1))
            ids.extend(rng.choice(W, n, replace=False).tolist())
            offs.append(len(ids))
        offs, ids = np.array(offs, np.int64), np.array(ids, np.int32)
        dt = torch.float32 if i % 2 else torch.bfloat16
        q, k, v = (bf16r(rng.standard_normal((H, Mi, 64))) for _ in range(3))
        gl = gsa.build_token_layout(*lt)
        plan = gsa.SelectionPlan(H, W, torch.from_numpy(offs).cuda(), torch.from_numpy(ids).cuda(),
                                 torch.empty(0, dtype=torch.int32, device="cuda"))
        out, lse = gsa.block_sparse_attention(dev(q, dt), dev(k, dt), dev(v, dt), plan, gl, 0.125)
        o_m, den = ref.masked_attention(q, k, v, lt, offs, ids, 0.125)
        assert np.abs(out.cpu().numpy() - o_m).max() <= P16_ABS, i
        rel = np.abs(np.exp(lse.cpu().numpy().astype(np.float64)) / den - 1.0).max()
        assert rel <= 1e-5, (i, rel)


@pytest.mark.parametrize("frames", [1, 99, 100, 250])
def test_forced_inclusion(gsa, frames):
    """hybrid, ref_stride=100: every plan row holds every window of
    frames 0, 100, 200, ... (ascending, first), exhaustive over the rows."""
    lt = (0, frames, 8, 8, 4)
    L = gsa.build_token_layout(*lt)
    W, wpf = L.num_windows, L.windows_per_frame
    rng = np.random.default_rng(frames)
    H, k = 2, 3
    topk = np.stack([np.stack([rng.choice(W, min(k, W), replace=False) for _ in range(W)]) for _ in range(H)])
    plan = gsa.build_selection_plan(torch.from_numpy(topk.astype(np.int32)).cuda(), L, 1, 100)
    offs, ids = plan.offsets.cpu().numpy(), plan.window_ids.cpu().numpy()
    forced = np.array([f * wpf + w for f in range(0, frames, 100) for w in range(wpf)], np.int32)
    for r in range(H * W):
        row = ids[offs[r]:offs[r + 1]]
        np.testing.assert_array_equal(row[: forced.size], forced)
        assert len(set(row.tolist())) == row.size

"""CPU tests of the parity checker itself: the C restatement (oracle/) must
reproduce the reference's known answers (SPEC.md examples), the committed golden
fixtures made by the unmodified reference (tests/golden/), and — where
oracle/_ref is built — the reference on fresh random instances."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_NAMES, load_golden, rel_l2
from oracle import Layout, make_inputs


# ---------------------------------------------------------- SPEC known answers
def test_naive_topk_known_answer(orc):
    # SPEC.md:121  naive_topk([3,1,3,2], 2) -> [0, 2]
    assert orc.topk_row(np.array([3, 1, 3, 2], np.float32), 2).tolist() == [0, 2]
    # SPEC.md:200  all-equal scores, k=3 -> [0,1,2]
    assert orc.topk_row(np.zeros(9, np.float32), 3).tolist() == [0, 1, 2]


def test_layout_known_answers():
    # SPEC.md:53-55, 65
    assert Layout(0, 2, 4, 4, 4).num_windows == 2
    L = Layout(5, 10, 36, 36, 4)
    assert L.image_tokens == 12960 and L.num_windows == 810
    assert Layout(0, 1, 8, 8, 4).window_of_token(5 * 8 + 6) == 3


def test_pool_known_answer(orc):
    # a 2x2 window holding 0,1,2,3 pools to 1.5
    x = np.arange(4, dtype=np.float32).reshape(1, 4, 1)
    assert orc.pool(x, Layout(0, 1, 2, 2, 2))[0, 0, 0] == 1.5


def test_forced_frames_known_answer(orc):
    # 250 frames, stride 100 -> frames {0,100,200}
    L = Layout(0, 250, 4, 4, 4)
    fw = orc.forced_windows(L, 100)
    assert fw.tolist() == [0, 100, 200]


def test_hybrid_plan_known_answer(orc):
    # frames=3, 8x8, s=4 (4 windows/frame), stride 100, top-k row
    # [5,2,9] -> plan row [0,1,2,3,5,9]
    L = Layout(0, 3, 8, 8, 4)
    topk = np.array([[[5, 2, 9]] * L.num_windows], np.int32)
    offs, ids = orc.build_plan(topk, L, 1, 100)
    assert ids[offs[0]:offs[1]].tolist() == [0, 1, 2, 3, 5, 9]


def test_single_window_known_answer(orc):
    # one window -> output == Vc row, indices == [0]
    rng = np.random.default_rng(0)
    qc, kc, vc = (rng.standard_normal((1, 1, 8)).astype(np.float32) for _ in range(3))
    out, lse, idx = orc.compress_topk(qc, kc, vc, 4, 0.5)
    assert idx.tolist() == [[[0]]]
    np.testing.assert_array_equal(out, vc)


# --------------------------------------------------- oracle vs reference pins
def test_scaled_dot_matches_reference_bitwise(orc, ref):
    rng = np.random.default_rng(1)
    for n in (1, 3, 4, 7, 16, 63, 64, 65, 129):
        for _ in range(20):
            a = rng.standard_normal(n).astype(np.float32)
            b = rng.standard_normal(n).astype(np.float32)
            s = np.float32(rng.uniform(0.01, 2))
            assert np.float32(orc.scaled_dot(a, b, s)).tobytes() == np.float32(ref.scaled_dot(a, b, s)).tobytes()


def test_topk_tie_rule_matches_reference(orc, ref):
    # 10^3 trials including exact ties
    rng = np.random.default_rng(2)
    for t in range(1000):
        n = int(rng.integers(1, 80))
        k = int(rng.integers(0, n + 3))
        scores = rng.integers(-3, 4, size=n).astype(np.float32) if t % 2 else rng.standard_normal(n).astype(np.float32)
        ex = (rng.random(n) < 0.2).astype(np.uint8) if t % 3 == 0 else None
        kk = min(k, n - (0 if ex is None else int(ex.sum())))
        assert orc.topk_row(scores, kk, ex).tolist() == ref.naive_topk(scores, kk, ex).tolist()


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_oracle_reproduces_golden(orc, name):
    g = load_golden(name)
    L = Layout(*g["layout"])
    r = orc.gsa_forward(g["q"], g["k"], g["v"], g["w_g"], L, top_k=g["top_k"], variant=g["variant"],
                        ref_stride=g["ref_stride"])
    np.testing.assert_array_equal(r["topk"], g["topk"])
    Ms = g["layout"][0]
    np.testing.assert_array_equal(orc.pool(g["q"][:, Ms:], L), g["qc"])
    np.testing.assert_array_equal(orc.pool(g["k"][:, Ms:], L), g["kc"])
    assert np.abs(r["out"] - g["out"]).max() < 1e-5
    assert np.abs(r["o_comp"] - g["o_comp"]).max() < 1e-5
    assert np.abs(r["lse_sel"] - g["lse_sel"]).max() < 1e-4


def test_parity_digests_reproduced_by_oracle(orc):
    meta = json.load(open(os.path.join(GOLDEN, "parity_digests.json")))
    for name, m in meta.items():
        L = Layout(*m["layout"])
        kind = m["kind"]
        q, k, v, wg = make_inputs(orc, L, heads=m["heads"], dim=64, seed=m["seed"],
                                  kind="uniform" if kind == "uniform" else "normal",
                                  sharp=3.0 if kind == "sharp" else 1.0)
        r = orc.gsa_forward(q, k, v, wg, L, top_k=m["top_k"], variant=m["variant"], ref_stride=m["ref_stride"])
        assert r["k_eff"] == m["k_eff"]
        assert hashlib.sha256(r["topk"].astype(np.int32).tobytes()).hexdigest() == m["topk_sha256"], name
        assert abs(float(r["out"].astype(np.float64).sum()) - m["out_sum"]) < 1e-3 * max(1.0, m["out_abs_sum"] * 1e-3)


@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_random(orc, ref, seed):
    # fused vs oracle over random configurations (s in {1,2,4},
    # ns in {0,1,5}, plain/hybrid, k from 1 to all windows)
    rng = np.random.default_rng(100 + seed)
    s = [1, 2, 4][seed % 3]
    ns = [0, 1, 5][(seed // 3) % 3]
    nf = int(rng.integers(1, 4))
    g = s * int(rng.integers(1, 4)) * (2 if s == 1 else 1)
    lt = (ns, nf, g, g, s)
    L = Layout(*lt)
    variant = seed % 2
    k = int(rng.integers(1, L.num_windows + 2))
    q, kk, v, wg = make_inputs(orc, L, heads=2, dim=64, seed=seed)
    a = ref.forward(q, kk, v, wg, lt, top_k=k, variant=variant, ref_stride=2, threads=2)
    b = orc.gsa_forward(q, kk, v, wg, L, top_k=k, variant=variant, ref_stride=2)
    np.testing.assert_array_equal(a["topk"], b["topk"])
    assert rel_l2(b["out"], a["out"]) < 1e-5


def test_reference_errors_mirrored(ref):
    assert ref.build_layout(0, 1, 5, 5, 4)[0] == -3  # DivisibilityError
    assert ref.build_layout(0, 0, 4, 4, 4)[0] == -4  # ZeroSizeError


@pytest.mark.parametrize("variant,specials", [(0, 5), (1, 0)])
def test_sampled_checker_matches_full_reference_layer(orc, ref, variant, specials):
    """The sampled-row checker (oracle/sampled.py -> gsa_ref_sampled_head) must reproduce the
    full reference fused layer (gsa_ref_forward) on the rows it samples: top-k bit-exact and
    outputs to float rounding. This pins the checker used at V >= 100 (tests/test_scale_parity.py,
    bench.py's post-timing parity) against the reference run in full."""
    torch = pytest.importorskip("torch")
    from oracle import Layout
    from oracle.sampled import sampled_parity
    lt = (specials * 6, 6, 16, 16, 4)
    L = Layout(*lt)
    q, k, v, wg = make_inputs(orc, L, heads=3, dim=64, seed=17)
    rf = ref.forward(q, k, v, wg, lt, top_k=9, variant=variant, ref_stride=4)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731  (CPU tensors stand in for device ones)
    res = sampled_parity(T(q), T(k), T(v), T(wg), lt, 9, T(rf["out"]), T(rf["topk"]), variant=variant, ref_stride=4,
                         o_comp=T(rf["o_comp"]), lse_comp=T(rf["lse_comp"]), o_sel=T(rf["o_sel"]),
                         lse_sel=T(rf["lse_sel"]), frac=0.25, spec_frac=0.5, threads=4)
    assert res["rows_checked"] == 3 * int(np.ceil(0.25 * L.num_windows))
    assert res["topk_mismatches"] == 0
    assert res["rel_l2"] < 1e-6 and res["max_abs"] < 1e-6
    assert res["o_comp_rel_l2"] < 1e-5 and res["lse_comp_max_abs"] < 1e-5
    assert res["o_sel_rel_l2"] < 1e-6 and res["lse_sel_max_abs"] < 1e-6
    if specials:
        assert res["special_rows_checked"] > 0 and res["special_rel_l2"] < 1e-6
    # a corrupted GPU row is caught
    bad = rf["topk"].copy()
    bad[1, 5, [0, 1]] = bad[1, 5, [1, 0]]
    res2 = sampled_parity(T(q), T(k), T(v), T(wg), lt, 9, T(rf["out"]), T(bad), variant=variant, ref_stride=4,
                          frac=1.0, threads=4)
    assert res2["topk_mismatches"] == 1

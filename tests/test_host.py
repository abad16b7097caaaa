"""Host-side pieces of the C ABI that need no GPU."""
from __future__ import annotations


def test_selection_sparsity_spec_examples():
    """selection_sparsity (declared, never defined, in the reference's
    workload.hpp:112): the SPEC's worked examples and its monotonicity properties.
    Host arithmetic in the C ABI: runs without a GPU."""
    import paper_2603_08055_b200 as gsa
    L = gsa.build_token_layout(0, 10, 36, 36, 4)
    assert abs(gsa.selection_sparsity(L, gsa.GsaParams(window_s=4, top_k=32)) - (1 - 512 / 12960)) < 1e-12
    hyb = gsa.GsaParams(window_s=4, top_k=32, variant=gsa.HYBRID, ref_stride=100)
    assert abs(gsa.selection_sparsity(L, hyb) - (1 - (81 + 32) * 16 / 12960)) < 1e-12
    assert gsa.selection_sparsity(L, gsa.GsaParams(window_s=4, top_k=L.num_windows)) == 0.0
    prev = 1.0
    for k in (1, 2, 8, 32, 128, 810):
        s = gsa.selection_sparsity(L, gsa.GsaParams(window_s=4, top_k=k))
        assert s <= prev
        prev = s
    for frames in (2, 4, 8, 16):  # non-decreasing in image tokens at fixed k
        a = gsa.selection_sparsity(gsa.build_token_layout(0, frames, 36, 36, 4), gsa.GsaParams(window_s=4, top_k=32))
        b = gsa.selection_sparsity(gsa.build_token_layout(0, frames * 2, 36, 36, 4), gsa.GsaParams(window_s=4, top_k=32))
        assert b >= a

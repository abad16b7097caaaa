"""Host-side pieces of the C ABI that need no GPU."""
from __future__ import annotations

import pytest


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


def test_bench_cli_exponent_fit_and_seeds():
    """SPEC.md:522-529 known answers of fit_scaling_exponent; seed' = hash(seed, size) is
    stable and size-dependent."""
    from paper_2603_08055_b200.cli import DegenerateInput, fit_scaling_exponent, size_seed
    ns = [1000, 2000, 4000, 8000]
    assert abs(fit_scaling_exponent([(n, 3e-9 * n * n) for n in ns]) - 2.0) < 1e-9
    assert abs(fit_scaling_exponent([(n, 5e-6 * n) for n in ns]) - 1.0) < 1e-9
    for bad in ([(1, 1.0), (2, 2.0)], [(1, 1.0), (2, 2.0), (2, 3.0)], [(1, 1.0), (2, -2.0), (3, 3.0)]):
        with pytest.raises(DegenerateInput):
            fit_scaling_exponent(bad)
    assert size_seed(7, 8) == size_seed(7, 8) and size_seed(7, 8) != size_seed(7, 16) != size_seed(8, 16)


def test_bench_cli_csv_schema_and_flags(tmp_path):
    """The CSV header is SPEC's exact column order; f64 and --backward on a
    mode without a backward are rejected loudly rather than silently downgraded."""
    from paper_2603_08055_b200 import cli
    assert cli.CSV_COLUMNS == ["mode", "frames", "image_tokens", "window_s", "top_k", "variant", "repeats",
                               "median_s", "mean_s", "stddev_s"]
    with pytest.raises(SystemExit):
        cli.main(["--backward", "--mode", "dense"])
    cfg = tmp_path / "c.cfg"
    cfg.write_text("bogus_key = 3\n")
    with pytest.raises(SystemExit):
        cli.main(["--config", str(cfg)])

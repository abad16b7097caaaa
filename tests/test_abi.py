"""CPU-side checks of the drop-in boundary: libgsa_sm100.so loads without a GPU,
exports every entry point include/gsa_sm100.h declares, and its host-only
validation mirrors the reference's error classes. No compute calls here."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "gsa_sm100.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2603_08055_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libgsa_sm100.so not built: run __graft_entry__.build()")
    return _lib.load()


def declared_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsa_[a-z_0-9]+)\s*\(", src)))


def test_header_and_library_agree(lib):
    from paper_2603_08055_b200 import _lib
    decl = declared_functions()
    assert len(decl) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gsa_[a-z_0-9]+)", out))
    missing = [f for f in decl if f not in exported]
    assert not missing, f"declared but not exported: {missing}"
    assert sorted(_lib.EXPORTED_SYMBOLS) == sorted(decl)
    for f in decl:
        getattr(lib, f)


def test_no_cxx_symbols_leak_into_abi(lib):
    # the boundary is plain C: every gsa_* symbol is unmangled
    from paper_2603_08055_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "gsa_forward" in out


def test_status_strings(lib):
    lib.gsa_status_string.restype = C.c_char_p
    names = [lib.gsa_status_string(i).decode() for i in range(14)]
    assert names[:10] == ["ok", "GsaError", "ShapeMismatch", "DivisibilityError", "ZeroSizeError",
                          "IndexOutOfRange", "NonFiniteInput", "InvalidTiling", "InvalidStride", "EmptySelection"]
    assert lib.gsa_abi_version() == 1


def test_layout_validation_mirrors_reference():
    import paper_2603_08055_b200 as gsa
    L = gsa.build_token_layout(5, 10, 36, 36, 4)
    assert L.num_windows == 810 and L.image_tokens == 12960
    with pytest.raises(gsa.DivisibilityError):
        gsa.build_token_layout(0, 1, 5, 5, 4)  # layout.cpp:13-16
    with pytest.raises(gsa.ZeroSizeError):
        gsa.build_token_layout(0, 0, 4, 4, 4)
    with pytest.raises(gsa.ZeroSizeError):
        gsa.build_token_layout(-1, 1, 4, 4, 4)
    with pytest.raises(gsa.IndexOutOfRange):
        L.window_of_token(L.image_tokens)
    assert L.window_of_token(0) == 0 and len(L.tokens_of_window(809)) == 16


def test_layout_matches_reference_harness(ref):
    import paper_2603_08055_b200 as gsa
    lt = (3, 2, 12, 8, 4)
    L = gsa.build_token_layout(*lt)
    for t in range(0, L.image_tokens, 7):
        assert L.window_of_token(t) == ref.window_of_token(lt, t)
    for w in range(L.num_windows):
        assert L.tokens_of_window(w) == ref.tokens_of_window(lt, w).tolist()


def test_params_validation(lib):
    import paper_2603_08055_b200 as gsa
    from paper_2603_08055_b200 import _lib
    L = gsa.build_token_layout(0, 1, 8, 8, 4)

    def rc(**kw):
        p = gsa.GsaParams(**kw)
        return lib.gsa_validate_params(C.byref(p.c()), C.byref(L.c()))

    assert rc() == 0
    assert rc(top_k=0) == 1                               # GsaError (types.hpp:68)
    assert rc(scale=-1.0) == 1
    assert rc(variant=1, ref_stride=0) == 8               # InvalidStride
    assert rc(tiling=gsa.KernelTiling(12, 16)) == 7       # InvalidTiling
    assert rc(tiling=gsa.KernelTiling(512, 16)) == 7
    assert rc(window_s=2) == 2                            # ShapeMismatch (layer.hpp:182)
    del _lib


def test_forward_stats_closed_form():
    # at the parity geometry scores_computed = 13,379,584 and
    # keys_attended = 84,934,656 (KernelStats, types.hpp:78-86)
    import paper_2603_08055_b200 as gsa
    L = gsa.build_token_layout(40, 8, 36, 36, 4)
    sc, ka = gsa.forward_stats(L, gsa.GsaParams(), 16)
    assert sc == 13_379_584
    assert ka == 84_934_656


def test_backward_host_validation(lib):
    """gsa_backward / gsa_project_backward / the pool adjoints reject bad calls on the host
    (before any device work) with the reference's classes: ContextMismatch for an
    incomplete saved context (errors.hpp:44), ShapeMismatch for a dO of the wrong shape
    (gradients.hpp:66-67) and for adjoint inputs of the wrong row count (:23-24, :39-40)."""
    import paper_2603_08055_b200 as gsa
    from paper_2603_08055_b200._lib import GsaSavedC, GsaTensor
    L = gsa.build_token_layout(2, 2, 8, 8, 4)
    H, d, M, W, Mi = 2, 64, L.total_tokens, L.num_windows, L.image_tokens
    fake = 256  # never dereferenced: validation fails first

    def t(rows, dim=d, heads=H, dtype=0):
        return GsaTensor(fake, dtype, heads, rows, dim, rows * dim, dim)

    p = gsa.GsaParams(top_k=2).c()
    lc = L.c()
    wg = GsaTensor(fake, 0, H, d, d, d * d, d)
    full = GsaSavedC(*([fake] * 5), fake, fake, H * W * 2, fake, fake, fake, t(2), fake)
    empty = GsaSavedC()
    q = t(M)

    def bwd(saved, d_out):
        return lib.gsa_backward(C.byref(q), C.byref(q), C.byref(q), C.byref(wg), C.byref(lc), C.byref(p),
                                C.byref(saved), C.byref(d_out), C.byref(t(M)), C.byref(t(M)), C.byref(t(M)),
                                C.c_void_p(fake), None, 0, None)

    assert bwd(empty, t(M)) == 14                     # ContextMismatch: incomplete context
    assert bwd(full, t(M - 1)) == 2                   # ShapeMismatch: dO rows
    bad_spec = GsaSavedC(*([fake] * 5), fake, fake, H * W * 2, fake, fake, fake, t(1), fake)
    assert bwd(bad_spec, t(M)) == 14                  # o_spec must be [H][Ms][d]
    assert bwd(full, t(M)) == 12                      # WorkspaceError: no workspace given
    assert lib.gsa_avg_pool_backward(C.byref(t(W + 1)), C.byref(lc), C.byref(t(Mi)), None) == 2
    assert lib.gsa_upsample_backward(C.byref(t(Mi - 1)), C.byref(lc), C.byref(t(W)), None) == 2
    assert lib.gsa_project_backward(None, M, 32, None, None, None, H, d, None, None, None, None, None, None, None,
                                    None, 0, None) == 1  # null pointers: GsaError
    assert lib.gsa_backward_workspace_bytes(C.byref(lc), C.byref(p), H, d, H * W * 2, 1) > \
        lib.gsa_backward_workspace_bytes(C.byref(lc), C.byref(p), H, d, H * W * 2, 0)  # bf16 adds f32 copies
